"""Peer-exchange shards on one GPU vs the unsharded engine: W shards of
Brunel at SYNAPSES, each with 148 // W CTAs, running side by side and
exchanging frames through each other's rings (Opts(shard_peer=True)).
Prints ms per biological second (device time of the slowest shard) and
checks the merged state against the unsharded run.

    python tools/peer_probe.py [SYNAPSES] [STEPS] [W...]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq
from paper_1912_07423_b200 import shard

syn = int(float(sys.argv[1])) if len(sys.argv) > 1 else int(1e9)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
worlds = [int(x) for x in sys.argv[3:]] or [2]
BIO = 10000

ref = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True), synapses=syn)
ref.run(500)
d0, _ = ref.device_time()
ref.run(steps)
d1, _ = ref.device_time()
rv = ref.neuron_field(0).view(np.uint32).copy()
print(f"unsharded engine={ref.engine}: {(d1 - d0) / steps * BIO * 1e3:.2f} ms per bio-s", flush=True)
ref.close()
for W in worlds:
    t0 = time.time()
    g = shard.PeerGroup("brunel", 0, W, tiles=148 // W, synapses=syn, seed=1, deterministic=True)
    print(f"W={W} setup {time.time() - t0:.1f} s, engines {[s.engine for s in g.sims]}", flush=True)
    g.run(500)
    a = [s.device_time()[0] for s in g.sims]
    w0 = time.time()
    g.run(steps)
    wall = time.time() - w0
    b = [s.device_time()[0] for s in g.sims]
    dev = max(y - x for x, y in zip(a, b))
    same = np.array_equal(g.neuron_field(0).view(np.uint32), rv)
    print(f"W={W} peer shards ({148 // W} CTAs each): {dev / steps * BIO * 1e3:.2f} ms per bio-s device, "
          f"{wall / steps * BIO * 1e3:.2f} wall; state equal to unsharded: {same}", flush=True)
    g.close()
