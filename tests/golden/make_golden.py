"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists) after `make -C oracle`:

    python tests/golden/make_golden.py

Every vector is produced by oracle/_ref/synq_golden, which links the
reference's own sources (proj/src/*.cpp) and calls its public C++ API
(random.hpp, adjacency.hpp, engine.hpp, benchmarks.hpp).  The fixtures pin
both the C restatement (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_parity.py) to the reference without needing /root/reference
at test time.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rng_vectors():
    out = {}
    for seed in (1, 42, 2**63 + 5, 0):
        out[f"xs_{seed}"] = np.frombuffer(O.golden("rng", seed, 64), np.uint32)
    out["uniform_7"] = np.frombuffer(O.golden("uniform", 7, 32), np.float64)
    pairs = [(1, 0), (1, 1), (1, 2**32), (1, 2**32 + 141420), (123, 9999), (2**64 - 1, 3)]
    out["derive_pairs"] = np.array(pairs, np.uint64)
    out["derive_vals"] = np.array([int(O.golden("derive", m, i)) for m, i in pairs], np.uint64)
    cases = [(99, 500, 0.12, 200), (1, 3200, 0.02, 200), (5, 56568, 0.1, 40), (3, 100, 0.0, 4),
             (3, 100, 1.0, 4), (8, 0, 0.5, 4)]
    for k, (s, m, p, n) in enumerate(cases):
        out[f"binom_{k}"] = np.frombuffer(O.golden("binomial", s, m, p, n), np.uint32)
    out["binom_cases"] = np.array([(s, m, p, n) for s, m, p, n in cases], np.float64)
    scases = [(50, 0, 5000, 2024), (6, 10, 30, 9), (1000, 100, 60000, 5), (10, 20, 30, 11),
              (1, 7, 8, 3), (0, 5, 10, 3), (3000, 0, 3200, 77)]
    for k, (n, a, b, s) in enumerate(scases):
        out[f"sorted_{k}"] = np.frombuffer(O.golden("sorted", n, a, b, s), np.uint32)
    out["sorted_cases"] = np.array(scases, np.uint64)
    raw = O.golden("fig2")
    out["fig2_trace"] = np.frombuffer(raw[: 8 * 5 * 8], np.float64).reshape(8, 5)
    out["fig2_out"] = np.frombuffer(raw[8 * 5 * 8:], np.uint32)
    np.savez_compressed(os.path.join(HERE, "rng_construct.npz"), **out)


def plan_vectors():
    out = {}
    import tempfile
    for tag, model, n, seed in (("pp42", "pingpong", 0, 42), ("v400", "vogels", 400, 1),
                                ("b1000", "brunel", 1000, 3)):
        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "plan.bin")
            O.golden("plan", model, n, seed, p)
            raw = open(p, "rb").read()
        njobs, deg_max, pitch, neurons = np.frombuffer(raw[:16], np.uint32)
        total = np.frombuffer(raw[16:24], np.uint64)[0]
        rec = np.dtype([("n", "<u4"), ("a", "<u4"), ("b", "<u4"), ("o", "<u8")])
        jobs = np.frombuffer(raw[24: 24 + 20 * njobs], rec)
        deg = np.frombuffer(raw[24 + 20 * njobs:], np.uint32)
        out[f"{tag}_hdr"] = np.array([njobs, deg_max, pitch, neurons, total], np.uint64)
        out[f"{tag}_jobs"] = np.stack([jobs["n"], jobs["a"], jobs["b"], jobs["o"]], 1).astype(np.uint64)
        out[f"{tag}_deg"] = deg
    np.savez_compressed(os.path.join(HERE, "plans.npz"), **out)


ADJ = [("vogels", 400, 1, True), ("pingpong", 0, 42, True), ("vogels", 4000, 1, False),
       ("brunel", 2000, 7, False), ("brunel", 20000, 1, False)]


def adj_vectors():
    out, meta = {}, {}
    for model, n, seed, full in ADJ:
        nn, pitch, deg_max, cells = O.reference_adjacency(model, n, seed)
        tag = f"{model.replace('+', 'p')}_{n}_s{seed}"
        deg = (cells != 0xFFFFFFFF).sum(1).astype(np.uint32)
        out[f"{tag}_deg"] = deg
        if full:
            out[f"{tag}_cells"] = cells
        meta[tag] = {"model": model, "neurons": n, "seed": seed, "pitch": pitch,
                     "deg_max": deg_max, "rows": nn, "edges": int(deg.sum()),
                     "sha256": sha(cells)}
    np.savez_compressed(os.path.join(HERE, "adjacency.npz"), **out)
    return meta


RUNS = [
    # model, neurons, seed, steps, history, dt, delay
    ("pingpong", 0, 42, 200, 0, 0, 0),
    ("pingpong", 0, 5, 1000, 0, 0, 0),
    ("vogels", 1000, 99, 3000, 0, 0, 0),
    ("vogels", 4000, 1, 10000, 0, 0, 0),
    ("brunel", 2000, 99, 3000, 0, 0, 0),
    ("brunel", 20000, 1, 2000, 0, 0, 0),
    ("brunel+", 400, 99, 1000, 0, 0, 0),
    ("brunel+", 120, 2024, 400, 0, 0, 0),
    ("brunel+", 80, 7, 200, 1, 0, 0),
    ("brunel+", 90, 99, 333, 23, 0, 0),
    ("vogels", 500, 3, 500, 0, 0.25, 3),
]


def run_vectors():
    out, meta = {}, {}
    for model, n, seed, steps, hist, dt, delay in RUNS:
        r = O.reference_run(model, n, seed, steps, hist, dt, delay)
        tag = f"{model.replace('+', 'p')}_{n}_s{seed}_t{steps}_h{hist}_d{delay}"
        out[f"{tag}_counts"] = r.counts
        out[f"{tag}_ids"] = r.ids
        for i, f in enumerate(r.fields):
            out[f"{tag}_f{i}"] = f
        if r.syn is not None:
            for i, f in enumerate(r.syn):
                out[f"{tag}_syn{i}"] = f
            out[f"{tag}_ages"] = r.ages
        meta[tag] = {"model": model, "neurons": n, "seed": seed, "steps": steps,
                     "history": hist, "dt": dt, "delay": delay, "counters": r.counters}
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)
    return meta


# the benchmarked configuration (BASELINE.json configs[1]): Brunel sized for
# ~1e9 synapses through solve_neurons (synq_sim_new_for_synapses), seed 1,
# one full biological second (10,000 steps; past the step-2,213 point where
# the reference's own parallel and deterministic modes part)
BIG = [("brunel", 1_000_000_000, 1, 10_000)]


def frame_digests(counts: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """u64 per step: the first 8 bytes (little endian) of sha256 of the
    frame's ids as u32 LE (tests/test_gpu_parity_big.py recomputes it)."""
    out = np.empty(len(counts), np.uint64)
    off = 0
    for k, c in enumerate(counts):
        h = hashlib.sha256(np.ascontiguousarray(ids[off:off + c], "<u4").tobytes()).digest()
        out[k] = int.from_bytes(h[:8], "little")
        off += c
    return out


def big_vectors(workdir: str = "/tmp/synq_big"):
    """Reference run at the bench configuration, reduced to fixtures: the
    adjacency (sha256 of the whole table, per-1024-row block digests, the
    degree vector), per-step frame counts and digests, final V / ACC / REF
    (sha256 + the first 4096 values) and the counters."""
    os.makedirs(workdir, exist_ok=True)
    out, meta = {}, {}
    for model, syn, seed, steps in BIG:
        tag = f"{model.replace('+', 'p')}_{syn:.0e}_s{seed}_t{steps}".replace("+", "")
        base = os.path.join(workdir, tag)
        if not os.path.exists(base + ".counters"):
            O.golden("big", model, syn, seed, steps, base)
        raw = np.memmap(base + ".adj", np.uint32, "r")
        neurons, pitch, deg_max, sentinel = (int(x) for x in raw[:4])
        cells = raw[4:4 + neurons * pitch].reshape(neurons, pitch)
        h = hashlib.sha256()
        blocks = []
        deg = np.empty(neurons, np.uint32)
        for r0 in range(0, neurons, 1024):
            blk = np.ascontiguousarray(cells[r0:r0 + 1024])
            b = blk.tobytes()
            h.update(b)
            blocks.append(int.from_bytes(hashlib.sha256(b).digest()[:8], "little"))
            deg[r0:r0 + len(blk)] = (blk != sentinel).sum(1)
        fr = np.fromfile(base + ".frames", np.uint32)
        counts, parts, off = [], [], 0
        while off < len(fr):
            c = int(fr[off])
            counts.append(c)
            parts.append(fr[off + 1: off + 1 + c])
            off += 1 + c
        counts = np.array(counts, np.uint32)
        ids = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
        st = np.fromfile(base + ".state", np.uint32).reshape(3, neurons)
        counters = {}
        for line in open(base + ".counters"):
            k, v = line.strip().split("=")
            counters[k] = int(v)
        out[f"{tag}_deg"] = deg
        out[f"{tag}_blocks"] = np.array(blocks, np.uint64)
        out[f"{tag}_counts"] = counts
        out[f"{tag}_digests"] = frame_digests(counts, ids)
        for i in range(3):
            out[f"{tag}_f{i}_head"] = st[i, :4096].copy()
        meta[tag] = {"model": model, "synapses": syn, "seed": seed, "steps": steps, "neurons": neurons,
                     "pitch": pitch, "deg_max": deg_max, "edges": int(deg.sum()), "adj_sha256": h.hexdigest(),
                     "state_sha256": [hashlib.sha256(st[i].tobytes()).hexdigest() for i in range(3)],
                     "counters": counters}
    np.savez_compressed(os.path.join(HERE, "big.npz"), **out)
    return meta


# Brunel+ (BASELINE.json configs[2]) at scale, short horizons: frames,
# neuron state, ages and the synapse state after flush (sha256 per field)
BIGP = [("brunel+", 100_000_000, 1, 400), ("brunel+", 1_000_000_000, 1, 100)]


def bigp_vectors(workdir: str = "/tmp/synq_bigp"):
    os.makedirs(workdir, exist_ok=True)
    out, meta = {}, {}
    for model, syn, seed, steps in BIGP:
        tag = f"brunelp_{syn:.0e}_s{seed}_t{steps}".replace("+", "")
        base = os.path.join(workdir, tag)
        if not os.path.exists(base + ".counters"):
            O.golden("big", model, syn, seed, steps, base)
        hdr = np.fromfile(base + ".adj", np.uint32, count=4)
        neurons, pitch, deg_max = int(hdr[0]), int(hdr[1]), int(hdr[2])
        counts, ids = O.split_frames(np.fromfile(base + ".frames", np.uint32))
        st = np.fromfile(base + ".state", np.uint32).reshape(3, neurons)
        ages = np.fromfile(base + ".ages", np.uint32)
        syn_sha = []
        cap = neurons * deg_max
        mm = np.memmap(base + ".syn", np.uint32, "r")
        for f in range(3):
            h = hashlib.sha256()
            for a in range(f * cap, (f + 1) * cap, 1 << 26):
                h.update(np.ascontiguousarray(mm[a:min((f + 1) * cap, a + (1 << 26))]).tobytes())
            syn_sha.append(h.hexdigest())
        counters = {}
        for fn in (".counters", ".preflush"):
            for line in open(base + fn):
                k, v = line.strip().split("=")
                counters[("preflush_" if fn == ".preflush" else "") + k] = int(v)
        out[f"{tag}_counts"] = counts
        out[f"{tag}_digests"] = frame_digests(counts, ids)
        meta[tag] = {"model": model, "synapses": syn, "seed": seed, "steps": steps, "neurons": neurons,
                     "deg_max": deg_max, "pitch": pitch,
                     "state_sha256": [hashlib.sha256(st[i].tobytes()).hexdigest() for i in range(3)],
                     "ages_sha256": hashlib.sha256(ages.tobytes()).hexdigest(), "syn_sha256": syn_sha,
                     "counters": counters}
    np.savez_compressed(os.path.join(HERE, "bigp.npz"), **out)
    return meta


# synthetic sweep (BASELINE.json configs[3]) at a reduced budget: every
# (p, rate) point of the bench grid, S = 1e6 synapses, seed 1, 2000 steps
SWEEP_S, SWEEP_STEPS = 1_000_000, 2000
SWEEP = [(p, r) for p in (0.1, 0.01, 0.001) for r in (1.0, 10.0, 100.0)]


# the same model at S = 1e8 (N up to 316,228: the streamed-state ELL engine
# of the sparse points), 100 Hz, 300 steps
SWEEP_BIG_S, SWEEP_BIG_STEPS = 100_000_000, 300
SWEEP_BIG = [(0.1, 100.0), (0.01, 100.0), (0.001, 100.0)]


def sweep_vectors(S=None, steps=None, points=None, name="sweep.npz"):
    """Reference runs of the sweep model (include/synq/models/sweep.hpp built
    against the reference headers): per-step counts + digests, final ACC
    (sha256), counters."""
    import tempfile
    S = S or SWEEP_S
    steps = steps or SWEEP_STEPS
    out, meta = {}, {}
    for p, rate in (points or SWEEP):
        tag = f"sweep_p{p:g}_r{rate:g}"
        with tempfile.TemporaryDirectory() as td:
            base = os.path.join(td, "run")
            O.golden("sweep", S, p, rate, 1, steps, base)
            counts, ids = O.split_frames(np.fromfile(base + ".frames", np.uint32))
            acc = np.fromfile(base + ".state", np.uint32)
            counters = {}
            for line in open(base + ".counters"):
                k, v = line.strip().split("=")
                counters[k] = int(v)
        out[f"{tag}_counts"] = counts
        out[f"{tag}_digests"] = frame_digests(counts, ids)
        meta[tag] = {"S": S, "p": p, "rate": rate, "seed": 1, "steps": steps,
                     "acc_sha256": hashlib.sha256(acc.tobytes()).hexdigest(), "counters": counters}
    np.savez_compressed(os.path.join(HERE, name), **out)
    return meta


def main():
    if not O.have_reference():
        raise SystemExit("oracle/_ref not built (needs /root/reference): make -C oracle")
    if sys.argv[1:] and sys.argv[1] in ("big", "sweep", "bigp", "sweepbig"):
        path = os.path.join(HERE, "golden.json")
        meta = json.load(open(path))
        if sys.argv[1] == "big":
            meta["big"] = big_vectors()
        elif sys.argv[1] == "bigp":
            meta["bigp"] = bigp_vectors()
        elif sys.argv[1] == "sweepbig":
            meta["sweep_big"] = sweep_vectors(SWEEP_BIG_S, SWEEP_BIG_STEPS, SWEEP_BIG, "sweep_big.npz")
        else:
            meta["sweep"] = sweep_vectors()
        with open(path, "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        print("big fixtures written to", HERE)
        return
    rng_vectors()
    plan_vectors()
    meta = {"adjacency": adj_vectors(), "runs": run_vectors(), "big": big_vectors(),
            "sweep": sweep_vectors(), "bigp": bigp_vectors()}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
