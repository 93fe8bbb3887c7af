"""Long-run rate goldens for the statistical parity test (SURVEY.md 8(d),
north star: "population firing rates must match within a stated statistical
bound").  Generated HERE from the UNMODIFIED reference (oracle/_ref/
libsynq_ref.so, its own C ABI): deterministic mode, 1 thread, 1 biological
second (10,000 steps of 0.1 ms), the reference's 500 ms warm-up dropped
(measure.warmup_ms, model_defaults.cfg:5), seeds 1..8.

    python tests/golden/make_rates.py      # writes tests/golden/rates.json

Rate = synq_sim_firing_rate (spikes per measured neuron per step, stimulus
excluded; analysis.cpp:41-50, sim_runtime.cpp:62-66) / dt, in Hz.
"""
import ctypes as C
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

CASES = [("brunel+", 4000), ("brunel", 20000), ("vogels", 4000)]
SEEDS = list(range(1, 9))
STEPS = 10000


def one(args):
    import oracle
    model, n, seed = args
    L = oracle.RefLib().L
    o = L.synq_opts_new()
    L.synq_opts_seed(o, seed)
    L.synq_opts_threads(o, 1)
    L.synq_opts_deterministic(o, 1)
    h = C.c_void_p()
    if L.synq_sim_new(model.encode(), n, o, C.byref(h)) != 0:
        raise RuntimeError(L.synq_last_error())
    L.synq_sim_run(h, STEPS)
    r = C.c_double()
    L.synq_sim_firing_rate(h, C.byref(r))
    L.synq_sim_free(h)
    L.synq_opts_free(o)
    return model, n, seed, r.value / 1e-4


def main():
    jobs = [(m, n, s) for m, n in CASES for s in SEEDS]
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        res = list(ex.map(one, jobs))
    out = {"steps": STEPS, "dt_ms": 0.1, "warmup_ms": 500, "seeds": SEEDS, "mode": "reference deterministic, 1 thread",
           "rates_hz": {}}
    for m, n, s, hz in res:
        out["rates_hz"].setdefault(f"{m}:{n}", []).append(hz)
    with open(os.path.join(HERE, "rates.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for k, v in out["rates_hz"].items():
        import statistics
        print(k, round(statistics.mean(v), 3), "+-", round(statistics.stdev(v), 3))


if __name__ == "__main__":
    main()
