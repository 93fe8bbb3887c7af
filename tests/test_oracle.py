"""Pin the C restatement (oracle/synq_oracle.c) to the reference.

Two anchors, as the parity plan requires:
* the reference's own known-answer tests (proj/tests/test_sorted_random.cpp,
  test_adjacency.cpp, test_models.cpp, test_lazy.cpp), restated here;
* golden vectors generated from the UNMODIFIED reference build by
  tests/golden/make_golden.py (committed under tests/golden/).
"""
import hashlib

import numpy as np
import pytest

import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ RNG
def test_xorshift_streams_match_reference(golden):
    g = golden["rng"]
    for seed in (1, 42, 2**63 + 5, 0):
        assert (O.xorshift(seed, 64) == g[f"xs_{seed}"]).all()


def test_derive_seed_matches_reference(golden):
    g = golden["rng"]
    for (m, i), v in zip(g["derive_pairs"], g["derive_vals"]):
        assert O.derive_seed(int(m), int(i)) == int(v)


def test_binomial_matches_reference(golden):
    g = golden["rng"]
    for k, (s, m, p, n) in enumerate(g["binom_cases"]):
        assert (O.binomial(int(s), int(m), float(p), int(n)) == g[f"binom_{k}"]).all()


def test_binomial_boundaries():
    # proj/tests/test_random.cpp:41-46
    assert (O.binomial(1, 100, 0.0, 3) == 0).all()
    assert (O.binomial(1, 100, 1.0, 3) == 100).all()
    assert (O.binomial(1, 0, 0.5, 3) == 0).all()


# -------------------------------------------------------- sorted_random
def test_fig2_worked_example():
    # proj/tests/test_sorted_random.cpp:23-51 (frozen to 1e-4 there)
    draws = [0.46, 0.97, 0.22, 0.81, 0.98, 0.38, 0.70, 0.18]
    out, tr = O.sorted_random_replay(6, 0, 100, draws)
    exp_e = [0.776529, 0.030459, 1.514128, 0.210721, 0.020203, 0.967584, 0.356675, 1.714798]
    exp_p = [0.0, 0.776529, 0.806988, 2.321116, 2.531837, 2.552040, 3.519624, 3.876299]
    exp_n = [0.0, 0.200327, 0.208185, 0.598797, 0.653158, 0.658370, 0.907986, 1.0]
    assert np.allclose(tr[0], exp_e, rtol=1e-4)
    assert np.allclose(tr[1], exp_p, rtol=1e-4)
    assert np.allclose(tr[2], exp_n, rtol=1e-4, atol=1e-12)
    assert list(tr[3]) == [0, 19, 20, 56, 61, 62, 85, 94]
    assert list(out) == [19, 21, 58, 64, 66, 90]


def test_fig2_matches_reference_trace(golden):
    g = golden["rng"]
    draws = g["fig2_trace"][:, 0]
    out, tr = O.sorted_random_replay(6, 0, 100, draws)
    assert (out == g["fig2_out"]).all()
    assert (tr[0] == g["fig2_trace"][:, 1]).all()  # bit-exact exponentials
    assert (tr[1] == g["fig2_trace"][:, 2]).all()
    assert (tr[2] == g["fig2_trace"][:, 3]).all()
    assert (tr[3] == g["fig2_trace"][:, 4]).all()


def test_padding_draw_has_no_effect():
    # proj/tests/test_sorted_random.cpp:53-61
    a, _ = O.sorted_random_replay(6, 0, 100, [0.46, 0.97, 0.22, 0.81, 0.98, 0.38, 0.70, 0.18])
    b, _ = O.sorted_random_replay(6, 0, 100, [0.46, 0.97, 0.22, 0.81, 0.98, 0.38, 0.70, 0.55])
    assert (a == b).all()


def test_sorted_random_matches_reference(golden):
    g = golden["rng"]
    for k, (n, a, b, s) in enumerate(g["sorted_cases"]):
        got = O.sorted_random(int(n), int(a), int(b), int(s))
        assert (got == g[f"sorted_{k}"]).all()


def test_sorted_random_preconditions():
    # proj/tests/test_sorted_random.cpp:90-95
    with pytest.raises(ValueError):
        O.sorted_random(6, 10, 10, 1)
    with pytest.raises(ValueError):
        O.sorted_random(6, 10, 12, 1)


def test_sorted_random_full_interval():
    # proj/tests/test_sorted_random.cpp:83-88
    assert list(O.sorted_random(10, 20, 30, 11)) == list(range(20, 30))


# --------------------------------------------------------- construction
def _desc_for(model, n):
    if model == "pingpong":
        return O.SoDesc.make([100, 100], [(0, 1, 0.01), (1, 0, 0.01)], 1.0, 1)
    if model == "vogels":
        ne = int(round(0.8 * n))
        return O.SoDesc.make([ne, n - ne], [(s, t, 0.02) for s in (0, 1) for t in (0, 1)], 0.1, 8)
    ne, ni = int(np.floor(0.4 * n + 0.5)), int(np.floor(0.1 * n + 0.5))
    conns = [(0, 0, .1), (0, 1, .1), (1, 0, .1), (1, 1, .1), (2, 0, .1), (2, 1, .1)]
    return O.SoDesc.make([ne, ni, n - ne - ni], conns, 0.1, 15)


@pytest.mark.parametrize("tag,model,n,seed", [("pp42", "pingpong", 0, 42),
                                              ("v400", "vogels", 400, 1),
                                              ("b1000", "brunel", 1000, 3)])
def test_plan_matches_reference(golden, tag, model, n, seed):
    g = golden["plans"]
    p = O.plan_graph(_desc_for(model, n), seed)
    njobs, deg_max, pitch, neurons, total = (int(x) for x in g[f"{tag}_hdr"])
    assert (p.deg_max, p.pitch, p.neurons, p.edges) == (deg_max, pitch, neurons, total)
    assert len(p.jobs) == njobs
    assert (p.jobs == g[f"{tag}_jobs"]).all()
    assert (p.degree == g[f"{tag}_deg"]).all()


def test_adjacency_matches_reference(golden):
    adj, meta = golden["adj"], golden["meta"]["adjacency"]
    for tag, m in meta.items():
        if m["neurons"] > 5000:
            continue  # the large ones are covered by the slow test below
        g = O.build_graph(_desc_for(m["model"], m["neurons"]), m["seed"])
        assert g.pitch == m["pitch"] and g.deg_max == m["deg_max"] and g.edges == m["edges"]
        assert (g.degree == adj[f"{tag}_deg"]).all()
        assert sha(g.cells) == m["sha256"], tag
        if f"{tag}_cells" in adj:
            assert (g.cells == adj[f"{tag}_cells"]).all()


@pytest.mark.slow
def test_adjacency_large_matches_reference(golden):
    adj, meta = golden["adj"], golden["meta"]["adjacency"]
    for tag, m in meta.items():
        g = O.build_graph(_desc_for(m["model"], m["neurons"]), m["seed"])
        assert sha(g.cells) == m["sha256"], tag


def test_adjacency_invariants():
    # proj/tests/test_adjacency.cpp:63-85 rows sorted, unique, sentinel padded, pitch%32
    d = O.SoDesc.make([200, 300], [(0, 0, .05), (0, 1, .1), (1, 0, .02), (1, 1, 0.0)])
    g = O.build_graph(d, 99)
    assert g.pitch % 32 == 0 and g.pitch >= g.deg_max
    for i in range(500):
        row = g.cells[i]
        k = g.degree[i]
        assert (np.diff(row[:k].astype(np.int64)) > 0).all()
        assert (row[:k] < 500).all() and (row[k:] == 0xFFFFFFFF).all()
    # p = 1 forces the full interval (test_adjacency.cpp:49-61)
    g = O.build_graph(O.SoDesc.make([20, 30], [(0, 1, 1.0)]), 7)
    assert g.deg_max == 30
    assert (g.cells[:20, :30] == np.arange(20, 50)).all()
    # p = 0: all sentinel (test_adjacency.cpp:39-47)
    g = O.build_graph(O.SoDesc.make([50], [(0, 0, 0.0)]), 7)
    assert g.edges == 0 and g.deg_max == 0


# ------------------------------------------------------------ simulation
def _run_cases(golden):
    for tag, m in golden["meta"]["runs"].items():
        yield tag, m


def test_runs_match_reference(golden):
    runs = golden["runs"]
    for tag, m in _run_cases(golden):
        s = O.Sim(m["model"], m["neurons"], m["seed"], m["history"], m["dt"], m["delay"])
        s.run(m["steps"])
        counts, ids = s.frames()
        assert (counts == runs[f"{tag}_counts"]).all(), tag
        assert (ids == runs[f"{tag}_ids"]).all(), tag
        nf = 1 if m["model"] == "pingpong" else 3
        for i in range(nf):
            assert (s.field(i) == runs[f"{tag}_f{i}"]).all(), (tag, i)
        c = s.counters()
        rc = m["counters"]
        for k in ("spikes", "deliveries", "frames_consumed", "expiry_batches"):
            key = k if m["model"] != "brunel+" or k not in ("expiry_batches",) else "preflush_" + k
            assert c[k] == rc.get(key, rc[k]), (tag, k)
        if m["model"] == "brunel+":
            assert c["synapse_updates"] == rc["preflush_synapse_updates"]
            assert (s.ages() == runs[f"{tag}_ages"]).all()
            s.flush()
            for i in range(3):
                assert (s.syn_field(i).view(np.uint32) ==
                        runs[f"{tag}_syn{i}"].view(np.uint32)).all(), (tag, i)
            assert s.counters()["synapse_updates"] == rc["synapse_updates"]


def test_lazy_updates_equal_eager_work_after_flush():
    # proj/tests/test_lazy.cpp:73-85
    s = O.Sim("brunel+", 100, 5)
    s.run(500)
    assert s.counters()["synapse_updates"] <= s.graph().edges * 500
    s.flush()
    assert s.counters()["synapse_updates"] == s.graph().edges * 500


def test_lif_decay_kat():
    # proj/tests/test_models.cpp:63-68: V=10, rest 0, tau 20, dt 1 -> 9.5
    v = np.float32(10.0)
    v = np.float32(v + (np.float32(1.0) * (-(v - np.float32(0.0)) / np.float32(20.0)) + np.float32(0)))
    assert abs(float(v) - 9.5) < 1e-6


def test_big_fixture_is_self_consistent(golden):
    """tests/golden/big.npz (Brunel 1e9 from the reference) agrees with its
    own metadata: degrees sum to the edges, counts to the spikes."""
    for tag, m in golden["meta"]["big"].items():
        big = golden["big"]
        assert int(big[f"{tag}_deg"].astype(np.uint64).sum()) == m["edges"] == m["counters"]["edges"]
        assert int(big[f"{tag}_counts"].astype(np.uint64).sum()) == m["counters"]["spikes"]
        assert len(big[f"{tag}_digests"]) == m["steps"]
        assert int(big[f"{tag}_deg"].max()) == m["deg_max"]
        assert m["pitch"] % 32 == 0 and m["pitch"] >= m["deg_max"]
