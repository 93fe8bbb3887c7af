"""Synthetic sweep (BASELINE.json configs[3], SURVEY.md 8 "SW") vs the
reference: the sweep model (include/synq/models/sweep.hpp) is compiled
against the reference's headers for the goldens (oracle/_ref/synq_golden
sweep) and against this repo's device engine here (build/sweep dump, the
C++ network<Model> API).  Every (p, rate) point of the bench grid at a
reduced budget S = 1e6: per-step spike counts and id digests over 2000
steps, final ACC bits and the delivery counter, bit for bit.
Tolerance: none.
"""
import hashlib
import os
import subprocess

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "sweep")


def digests(counts, ids):
    out = np.empty(len(counts), np.uint64)
    off = 0
    for k, c in enumerate(counts):
        h = hashlib.sha256(np.ascontiguousarray(ids[off:off + c], "<u4").tobytes()).digest()
        out[k] = int.from_bytes(h[:8], "little")
        off += int(c)
    return out


def test_sweep_points_bit_exact(golden, tmp_path):
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", ROOT, "build/sweep"], check=True)
    sw = np.load(os.path.join(ROOT, "tests", "golden", "sweep.npz"))
    for tag, m in golden["meta"]["sweep"].items():
        base = str(tmp_path / tag)
        subprocess.run([BIN, "dump", str(m["S"]), repr(m["p"]), repr(m["rate"]), str(m["seed"]), str(m["steps"]),
                        base], check=True, timeout=300)
        counts, ids = O.split_frames(np.fromfile(base + ".frames", np.uint32))
        assert np.array_equal(counts, sw[f"{tag}_counts"]), tag
        assert np.array_equal(digests(counts, ids), sw[f"{tag}_digests"]), tag
        acc = np.fromfile(base + ".state", np.uint32)
        assert hashlib.sha256(acc.tobytes()).hexdigest() == m["acc_sha256"], tag
        got = dict(line.strip().split("=") for line in open(base + ".counters"))
        for k in ("spikes", "deliveries", "frames_consumed", "edges", "neurons"):
            assert int(got[k]) == m["counters"][k], (tag, k)


def test_sweep_points_at_1e8_bit_exact(golden, tmp_path):
    """S = 1e8, 100 Hz, 300 steps (tests/golden/make_golden.py sweepbig):
    N = 31,623 / 100,000 / 316,228 — the bitmap engine and the
    streamed-state ELL engine of the sparse points at scale."""
    if "sweep_big" not in golden["meta"]:
        pytest.skip("sweep_big goldens not generated")
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", ROOT, "build/sweep"], check=True)
    sw = np.load(os.path.join(ROOT, "tests", "golden", "sweep_big.npz"))
    for tag, m in golden["meta"]["sweep_big"].items():
        base = str(tmp_path / tag)
        subprocess.run([BIN, "dump", str(m["S"]), repr(m["p"]), repr(m["rate"]), str(m["seed"]), str(m["steps"]),
                        base], check=True, timeout=600)
        counts, ids = O.split_frames(np.fromfile(base + ".frames", np.uint32))
        assert np.array_equal(counts, sw[f"{tag}_counts"]), tag
        assert np.array_equal(digests(counts, ids), sw[f"{tag}_digests"]), tag
        acc = np.fromfile(base + ".state", np.uint32)
        assert hashlib.sha256(acc.tobytes()).hexdigest() == m["acc_sha256"], tag
        got = dict(line.strip().split("=") for line in open(base + ".counters"))
        for k in ("spikes", "deliveries", "frames_consumed", "edges", "neurons"):
            assert int(got[k]) == m["counters"][k], (tag, k)
