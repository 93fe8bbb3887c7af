"""Per-GPU cost of the in-engine NCCL shard loop on one B200: Brunel 1e9 as
a one-rank NCCL shard (14-step launches + export_bits + ncclAllGather +
import per batch) vs the unsharded engine (1000-step launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

# SHARD_ONLY=1: just the shard; STEPS: timed steps (default 10000)
ONLY = os.environ.get("SHARD_ONLY") == "1"
STEPS = int(os.environ.get("STEPS", "10000"))
cases = [("nccl shard (1 rank)", {"shard_nccl": (0, 1, synq.nccl_unique_id())})]
if not ONLY:
    cases.insert(0, ("unsharded", {}))
for name, kw in cases:
    sim = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True, **kw), synapses=int(1e9))
    sim.run(2000 if not ONLY else 140)
    d0, k0 = sim.device_time()
    sim.run(STEPS)
    d1, k1 = sim.device_time()
    print(f"{name:22s}: {(d1 - d0) * 1e3:.1f} ms per bio-s device ({(k1 - k0) * 1e3:.1f} ms in step kernels), "
          f"launches {sim.kernel_launches()}", flush=True)
    sim.close()
