"""Brunel+ (STDP on E->E, BASELINE config 3) on the B200 (generic per-step
graph engine: update, lazy STDP catch-up, receive) vs the reference CPU
simulator (oracle/_ref, parallel mode, all host threads) on the same network.
    python tools/plus_probe.py SYNAPSES GPU_STEPS CPU_STEPS"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1912_07423_b200 as synq

syn = float(sys.argv[1]) if len(sys.argv) > 1 else 1e8
gsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
csteps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
for det in (True, False):
    sim = synq.Sim("brunel+", opts=synq.Opts(seed=1, deterministic=det), synapses=int(syn))
    sim.run(200)
    d0, _ = sim.device_time()
    c0 = sim.counters()
    sim.run(gsteps)
    d1, _ = sim.device_time()
    c1 = sim.counters()
    ev = c1["deliveries"] - c0["deliveries"]
    su = c1["synapse_updates"] - c0["synapse_updates"]
    print(f"B200 brunel+ syn={sim.synapses} n={sim.neurons} {'ordered(exact)' if det else 'fast'}: "
          f"{(d1 - d0) / gsteps * 1e4 * 1e3:.1f} ms per bio-s, {ev / (d1 - d0):.3e} events/s, "
          f"{su / (d1 - d0):.3e} synapse updates/s, engine={sim.engine}", flush=True)
    sim.close()
ref = oracle.RefLib()
L = ref.L
threads = os.cpu_count() or 1
o = L.synq_opts_new()
L.synq_opts_seed(o, 1)
L.synq_opts_threads(o, threads)
L.synq_opts_deterministic(o, 0)
s = C.c_void_p()
assert L.synq_sim_new_for_synapses(b"brunel+", int(syn), o, C.byref(s)) == 0, L.synq_last_error()
L.synq_sim_run(s, 20)
t0 = time.perf_counter()
L.synq_sim_run(s, csteps)
dt = time.perf_counter() - t0
print(f"CPU reference brunel+ parallel, {threads} threads: {dt / csteps * 1e4 * 1e3:.1f} ms per bio-s "
      f"(sample of {csteps} steps)", flush=True)
