"""Where do peer shards differ from the unsharded engine? (debugging aid)
python tools/peer_diff.py W BATCH [TILES] [RUNS...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq
from paper_1912_07423_b200 import shard

W, batch = int(sys.argv[1]), int(sys.argv[2])
tiles = int(sys.argv[3]) if len(sys.argv) > 3 else 16
runs = [int(x) for x in sys.argv[4:]] or [1, 250, 949]
n = 20000
ref = synq.Sim("brunel", n, synq.Opts(seed=3, deterministic=True, record=True))
ref.run(sum(runs))
rc, rids = ref.frames()
rv = ref.neuron_field(0).view(np.uint32).copy()
g = shard.PeerGroup("brunel", n, W, tiles=tiles, seed=3, deterministic=True, record=True, batch_steps=batch)
for k in runs:
    g.run(k)
print("delay", g.delay, "state equal:", np.array_equal(g.neuron_field(0).view(np.uint32), rv))
for r, s in enumerate(g.sims):
    c, ids = s.frames()
    bad = np.nonzero(c != rc)[0]
    print(f"shard {r}: range {s.shard_range()} frames differing: {len(bad)} first {bad[:10]} "
          f"got {c[bad[:5]]} want {rc[bad[:5]]}")
    if len(bad):
        f = bad[0]
        off, roff = int(c[:f].sum()), int(rc[:f].sum())
        got, want = set(ids[off:off + c[f]].tolist()), set(rids[roff:roff + rc[f]].tolist())
        print("   missing", sorted(want - got)[:20], "extra", sorted(got - want)[:20])
