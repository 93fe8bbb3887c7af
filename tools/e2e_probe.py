"""Where the end-to-end (recording) time goes for Brunel 1e9: device time vs
run() wall time with recording vs raster() copy-out."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

sim = synq.Sim("brunel", opts=synq.Opts(seed=1, deterministic=True), synapses=int(1e9))
sim.run(20000)
for rec in (False, True, True, True):
    sim.set_record(rec)
    d0, k0 = sim.device_time()
    t0 = time.perf_counter()
    sim.run(10000)
    t1 = time.perf_counter()
    d1, k1 = sim.device_time()
    t2 = time.perf_counter()
    n = 0
    if rec:
        if not hasattr(sim, "_bufs"):
            import numpy as np
            sim._bufs = (np.zeros(6_000_000, np.int64), np.zeros(6_000_000, np.uint32))
        st, ids = sim.raster(out=sim._bufs)
        n = len(ids)
    t3 = time.perf_counter()
    print(f"record={rec}: run wall {1e3*(t1-t0):.1f} ms, device {1e3*(d1-d0):.1f} ms, kernel {1e3*(k1-k0):.1f} ms, "
          f"raster() {1e3*(t3-t2):.1f} ms ({n} spikes), launches {sim.kernel_launches()}", flush=True)
