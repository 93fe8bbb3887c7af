"""A/B of the persistent schedules on one network: serial k_persistent vs the
pipelined kernel at several leads.  Every variant must produce bit-identical
counters and membrane state (both are exact); prints us per timestep.

    python tools/ab_pipeline.py [MODEL] [SYNAPSES] [STEPS] [LEADS...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

model = sys.argv[1] if len(sys.argv) > 1 else "brunel"
syn = float(sys.argv[2]) if len(sys.argv) > 2 else 1e9
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
leads = [int(x) for x in sys.argv[4:]] or [2, 4, 8]
prof = os.environ.get("SYNQ_PROFILE") == "1"

# (name, pipeline mode, lead, environment for the engine setup)
variants = [("serial", 0, 0, {})]
for L in leads:
    variants.append((f"ell lead={L}", 1, L, {"SYNQ_BITMAP": "0"}))
    variants.append((f"bitmap lead={L}", 1, L, {"SYNQ_BITMAP": "1"}))
if os.environ.get("AB_NO_SERIAL"):
    variants = variants[1:]
if os.environ.get("AB_ONLY"):
    variants = [v for v in variants if v[0].startswith(os.environ["AB_ONLY"])]
ref = None
for name, mode, lead, env in variants:
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    sim = synq.Sim(model, opts=synq.Opts(seed=1, deterministic=True, pipeline=mode, lead=lead, profile=prof),
                   synapses=int(syn))
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    assert sim.pipelined == bool(mode), (name, sim.pipelined)
    sim.run(500)  # warm-up
    d0, k0 = sim.device_time()
    sim.run(steps)
    d1, k1 = sim.device_time()
    c = sim.counters()
    v = sim.neuron_field(0).view(np.uint32).copy()
    line = (f"{name:14s} us/step={(k1 - k0) / steps * 1e6:8.2f}  spikes={c['spikes']} deliveries={c['deliveries']} "
            f"events/s={c['deliveries'] / max(k1, 1e-12) * (steps / (steps + 500)):.3e}")
    if prof:
        pc = sim.phase_cycles()
        line += f"  phases(mean)={ {k: round(x) for k, x in pc['mean'].items()} } pacing={pc['pacing']} pipe={pc['pipeline']}"
    print(line, flush=True)
    key = (c["spikes"], c["deliveries"], v.tobytes())
    if ref is None:
        ref = key
    else:
        assert key == ref, f"{name}: differs from the serial kernel"
    del sim
print("all variants bit-identical")
