"""Per-step cost of short persistent launches (the sharded exchange runs
delay-1 = 14 steps per launch) vs the default 1000-step batches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

for b in [int(x) for x in os.environ.get('BATCHES', '1000,100,14,7').split(',')]:
    sim = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True, batch_steps=b), synapses=int(1e9))
    sim.run(2000)
    d0, k0 = sim.device_time()
    sim.run(4200)
    d1, k1 = sim.device_time()
    print(f"batch {b:5d}: {(d1 - d0) / 4200 * 1e6:.2f} us/step device, {(k1 - k0) / 4200 * 1e6:.2f} us/step kernel",
          flush=True)
    sim.close()
