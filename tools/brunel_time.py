"""Brunel at SYNAPSES on the default engine (environment knobs apply): device
ms per biological second after WARM warm-up steps, over STEPS steps, plus the
final membrane-state digest (variants must agree bit for bit).
    python tools/brunel_time.py [SYNAPSES] [WARM] [STEPS]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

syn = float(sys.argv[1]) if len(sys.argv) > 1 else 1e9
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
sim = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True), synapses=int(syn))
sim.run(warm)
_, k0 = sim.device_time()
sim.run(steps)
_, k1 = sim.device_time()
dig = hashlib.sha256(sim.neuron_field(0).tobytes()).hexdigest()[:16]
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SYNQ_"))
print(f"[{env or 'default'}] engine={sim.engine}: {(k1 - k0) / steps * 1e7:.2f} ms per bio-s in step kernels, "
      f"V digest {dig}", flush=True)
