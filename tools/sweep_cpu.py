"""CPU baseline of the synthetic sweep (BASELINE config 4): the UNMODIFIED
reference (oracle/_ref/synq_golden sweep_time: the sweep model of
include/synq/models/sweep.hpp compiled against the reference's network<M>)
at S synapses per (p, rate) point, deterministic 1 thread (the reference's
fastest mode for population models), timed over SAMPLE steps
after WARM steps.  Test/baseline infrastructure: it runs the oracle.
    python tools/sweep_cpu.py [S] [SAMPLE] [WARM] [THREADS] [DET]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "oracle", "_ref", "synq_golden")
S = float(sys.argv[1]) if len(sys.argv) > 1 else 1e9
SAMPLE = int(sys.argv[2]) if len(sys.argv) > 2 else 200
WARM = int(sys.argv[3]) if len(sys.argv) > 3 else 20
THREADS = int(sys.argv[4]) if len(sys.argv) > 4 else 1
DET = int(sys.argv[5]) if len(sys.argv) > 5 else 1
out = []
for p in (0.1, 0.01, 0.001):
    for rate in (1.0, 10.0, 100.0):
        r = subprocess.run([TOOL, "sweep_time", str(S), str(p), str(rate), "1", str(WARM), str(SAMPLE), str(THREADS),
                            str(DET)], capture_output=True, text=True, check=True)
        kv = dict(line.split("=", 1) for line in r.stdout.split())
        sim = float(kv["sim_s"])
        rec = {"p": p, "rate_hz": rate, "neurons": int(kv["neurons"]), "synapses": int(kv["synapses"]),
               "sample_steps": SAMPLE, "events_per_s": int(kv["events"]) / sim if sim > 0 else None,
               "ms_per_bio_s": sim / SAMPLE * 1e4 * 1e3, "construct_s": float(kv["construct_s"]),
               "threads": THREADS, "deterministic": bool(DET)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
