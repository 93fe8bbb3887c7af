"""Setup-time breakdown of Brunel 1e9 on one B200: construction (plan +
expansion + rounding fix-ups) vs the rest of Sim creation (partition,
receive-window bitmaps, engine setup, init)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (context + NCCL library first, as bench.py does)

import paper_1912_07423_b200 as synq

torch.cuda.init()
torch.zeros(1, device="cuda")
for rep in range(2):
    t0 = time.perf_counter()
    sim = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True), synapses=int(1e9))
    wall = time.perf_counter() - t0
    print(f"rep {rep}: Sim() {wall:.3f} s: construct {sim.seconds('construct'):.3f} s, "
          f"init_neurons {sim.seconds('init_neurons'):.3f} s, fixups {sim.construction_fixups()}", flush=True)
    sim.close()
