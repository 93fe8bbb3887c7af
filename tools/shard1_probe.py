"""Per-GPU cost of the shard exchange on one B200: Brunel 1e9 as a one-rank
shard, against the unsharded engine, after the bench's warm-up (WARM steps,
default 30000 = 3 biological seconds) over STEPS timed steps (default 10000):
  * nccl shard: 14-step launches + export_bits + ncclAllGather + import per batch;
  * peer shard: NVLink peer exchange (frames stored into the peers' rings by
    the step kernel; 1000-step launches), wired by hand (PeerGroup);
  * nccl+peer shard: the same, IPC handles allgathered over NCCL by the engine
    (the bench's multi-GPU wiring with --exchange peer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq
from paper_1912_07423_b200 import shard

STEPS = int(os.environ.get("STEPS", "10000"))
WARM = int(os.environ.get("WARM", "30000"))
which = sys.argv[1:] or ["unsharded", "nccl", "peer", "nccl+peer"]
for name in which:
    if name == "peer":
        g = shard.PeerGroup("brunel", 0, 1, tiles=148, synapses=int(1e9), seed=1, deterministic=True)
        sim = g.sims[0]
    else:
        kw = {}
        if name.startswith("nccl"):
            kw["shard_nccl"] = (0, 1, synq.nccl_unique_id())
        if name == "nccl+peer":
            kw["shard_peer"] = True
        sim = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True, **kw), synapses=int(1e9))
    sim.run(WARM)
    d0, k0 = sim.device_time()
    l0 = sim.kernel_launches()
    sim.run(STEPS)
    d1, k1 = sim.device_time()
    print(f"{name:12s}: {(d1 - d0) / STEPS * 1e7:.1f} ms per bio-s device ({(k1 - k0) / STEPS * 1e7:.1f} ms in step "
          f"kernels), {sim.kernel_launches() - l0} launches for {STEPS} steps, engine {sim.engine}", flush=True)
    sim.close()
