"""Debug driver: W in-process shards on one GPU (python tools/shard_dbg.py model n W steps [tiles])."""
import sys; sys.path.insert(0, '.')
from paper_1912_07423_b200 import shard
model, n, W, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
kw = {"tiles": int(sys.argv[5])} if len(sys.argv) > 5 else {}
g = shard.ShardGroup(model, n, W, record=True, seed=1, deterministic=True, **kw)
done = 0
try:
    while done < steps:
        g.run(7)
        done += 7
    print(model, n, W, kw, "ok", sum(len(f) for f in g.frames))
except Exception as e:
    print(model, n, W, kw, "FAIL at", done, e)
