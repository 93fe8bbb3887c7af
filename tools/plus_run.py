"""Brunel+ driver for ncu launch lists: python tools/plus_run.py SYNAPSES STEPS [fast]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

syn, steps = float(sys.argv[1]), int(sys.argv[2])
det = not (len(sys.argv) > 3 and sys.argv[3] == "fast")
sim = synq.Sim("brunel+", opts=synq.Opts(seed=1, deterministic=det), synapses=int(syn))
sim.run(steps)
c = sim.counters()
d, _ = sim.device_time()
print(f"brunel+ syn={sim.synapses} n={sim.neurons} steps={steps} {d / steps * 1e6:.1f} us/step "
      f"spikes={c['spikes']} deliveries={c['deliveries']} synapse_updates={c['synapse_updates']}")
