"""BASELINE config 5 (Brunel ~1.2e10 synapses: B8) instantiated
on ONE B200: the 8 target-partitioned shards of an 8-GPU run, held side by
side in one process (each stores only its own sub-rows), exchanging the
in-engine bitmask blocks by hand, against the same network unsharded
(ELL delivery, ~50 GB).  Merged frames must be identical; per-shard
storage, setup and step times are printed.  STEPS (default 420)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1912_07423_b200 as synq
from paper_1912_07423_b200 import shard

STEPS = int(os.environ.get("STEPS", "420"))
W = int(os.environ.get("WORLD", "8"))
SYN = float(os.environ.get("SYN", "1.2e10"))
n = synq.solve_neurons("brunel", int(SYN))
out = {"neurons": n, "world": W, "steps": STEPS}
t0 = time.perf_counter()
g = shard.ShardGroup("brunel", n, W, record=True, exchange="bits", seed=1, deterministic=True)
out["shard_setup_s"] = round(time.perf_counter() - t0, 2)
out["shard_synapses"] = [s.synapses for s in g.sims]
out["shard_engine"] = [s.engine for s in g.sims]
out["shard_total_bytes"] = [s.memory_actual()["total_bytes"] for s in g.sims]
g.run(STEPS)
frames = g.frames
k = [s.device_time()[0] for s in g.sims]
out["shard_device_ms_per_step"] = [round(x / STEPS * 1e3, 4) for x in k]
out["shard_spikes"] = int(sum(len(f) for f in frames))
g.close()
print(json.dumps(out), flush=True)
t0 = time.perf_counter()
ref = synq.Sim("brunel", n, synq.Opts(seed=1, deterministic=True, record=True))
out["full_setup_s"] = round(time.perf_counter() - t0, 2)
out["full_synapses"] = ref.synapses
out["full_engine"] = ref.engine
ref.run(STEPS)
counts, ids = ref.frames()
out["full_device_ms_per_step"] = round(ref.device_time()[0] / STEPS * 1e3, 4)
out["sum_shard_synapses_equal"] = sum(out["shard_synapses"]) == ref.synapses
out["frames_equal"] = bool(np.array_equal(np.array([len(f) for f in frames]), counts)
                           and np.array_equal(np.concatenate(frames), ids))
print(json.dumps(out), flush=True)
