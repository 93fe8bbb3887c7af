"""Every schedule of the persistent engine against the reference goldens.

The pipelined kernel (include/synq/detail/pipeline.cuh) changes WHEN
deliveries happen (warp-specialised update / delivery, count ring, batched
passes, lead / lag flow control) and HOW they are counted (ELL chunks with
one shared-memory atomic per delivery, or receive-window bitmaps counted by
warp bit-transposes).  None of that may change a single bit: frames, neuron
state and counters are compared with the golden vectors produced by the
UNMODIFIED reference (tests/golden), for
  * serial / pipelined-ELL / pipelined-bitmap engines,
  * 4 / 8 / 16 update warps (512- and 1024-thread CTAs),
  * leads 1 .. delay and delivery lags 0 .. 2,
  * bitmap windows of 1, 2, 4 and 8 uint4 (tile counts 148 .. 10),
  * recording on (ordered frame log) and off, batch boundaries.
Engine knobs are read from the environment when a network is built.
"""
import os

import numpy as np
import pytest

import paper_1912_07423_b200 as synq

pytestmark = pytest.mark.gpu


def build(m, env, monkeypatch, **kw):
    for k in ("SYNQ_BITMAP", "SYNQ_UW", "SYNQ_LAG", "SYNQ_LEAD", "SYNQ_PREFETCH", "SYNQ_STREAM", "SYNQ_WORKQ", "SYNQ_SOLO", "SYNQ_CLUSTER", "SYNQ_CLUSTER_SIZE"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    opts = synq.Opts(seed=m["seed"], deterministic=True, record=kw.pop("record", True),
                     dt=m["dt"] or None, delay=m["delay"] or None, **kw)
    return synq.Sim(m["model"], m["neurons"], opts)


def check(sim, golden, tag, steps=None, chunks=None):
    m = golden["meta"]["runs"][tag]
    runs = golden["runs"]
    if chunks:
        for c in chunks:
            sim.run(c)
    else:
        sim.run(steps or m["steps"])
    counts, ids = sim.frames()
    assert np.array_equal(counts, runs[f"{tag}_counts"]), (tag, "counts")
    assert np.array_equal(ids, runs[f"{tag}_ids"]), (tag, "ids")
    for i in range(3):
        assert np.array_equal(sim.neuron_field(i).view(np.uint32), runs[f"{tag}_f{i}"]), (tag, "field", i)
    c = sim.counters()
    assert c["spikes"] == m["counters"]["spikes"] and c["deliveries"] == m["counters"]["deliveries"], tag
    assert c["frames_consumed"] == m["counters"]["frames_consumed"], tag


ENGINES = [
    ("serial", dict(pipeline=0), {}, "persistent"),
    ("ell", dict(pipeline=1), {"SYNQ_BITMAP": 0}, "pipelined"),
    ("bitmap", dict(pipeline=1), {"SYNQ_BITMAP": 2}, "pipelined-bitmap"),
]


@pytest.mark.parametrize("tag", ["brunel_20000_s1_t2000_h0_d0", "brunel_2000_s99_t3000_h0_d0",
                                 "vogels_1000_s99_t3000_h0_d0", "vogels_500_s3_t500_h0_d3"])
@pytest.mark.parametrize("engine", ENGINES, ids=[e[0] for e in ENGINES])
def test_engines_bit_exact(golden, monkeypatch, tag, engine):
    _, kw, env, want = engine
    sim = build(golden["meta"]["runs"][tag], env, monkeypatch, **kw)
    assert sim.engine == want, (tag, sim.engine)
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("uw", [4, 8, 16])
@pytest.mark.parametrize("bitmap", [0, 2])
def test_update_warps(golden, monkeypatch, uw, bitmap):
    tag = "brunel_20000_s1_t2000_h0_d0"
    sim = build(golden["meta"]["runs"][tag], {"SYNQ_UW": uw, "SYNQ_BITMAP": bitmap}, monkeypatch, pipeline=1)
    assert sim.pipelined
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("lead,lag", [(1, 0), (2, 1), (3, 2), (8, 1), (15, 0), (15, 2)])
def test_lead_and_lag(golden, monkeypatch, lead, lag):
    tag = "brunel_20000_s1_t2000_h0_d0"
    sim = build(golden["meta"]["runs"][tag], {"SYNQ_LAG": lag, "SYNQ_PREFETCH": 1}, monkeypatch,
                pipeline=1, lead=lead)
    assert sim.engine == "pipelined-bitmap"
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("tiles", [10, 20, 40, 148])  # receive windows of 8 / 4 / 2 / 1 uint4
def test_bitmap_window_widths(golden, monkeypatch, tiles):
    tag = "brunel_20000_s1_t2000_h0_d0"
    sim = build(golden["meta"]["runs"][tag], {"SYNQ_BITMAP": 2}, monkeypatch, pipeline=1, tiles=tiles)
    assert sim.engine == "pipelined-bitmap"
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("engine", ENGINES[1:], ids=[e[0] for e in ENGINES[1:]])
def test_batch_boundaries_and_recording(golden, monkeypatch, engine):
    """Uneven run() chunks (launch boundaries inside the delay window), and
    recording switched on mid-run, leave every bit unchanged."""
    _, kw, env, _ = engine
    tag = "brunel_2000_s99_t3000_h0_d0"
    m = golden["meta"]["runs"][tag]
    sim = build(m, env, monkeypatch, batch_steps=37, **kw)
    check(sim, golden, tag, chunks=[1, 2, 13, 14, 15, 16, 500, 1439, 1000])
    sim.close()
    # no recording: counters and state still exact
    sim = build(m, env, monkeypatch, record=False, **kw)
    sim.run(m["steps"])
    for i in range(3):
        assert np.array_equal(sim.neuron_field(i).view(np.uint32), golden["runs"][f"{tag}_f{i}"])
    assert sim.counters()["deliveries"] == m["counters"]["deliveries"]
    sim.close()


@pytest.mark.parametrize("tag", ["brunel_20000_s1_t2000_h0_d0", "brunel_2000_s99_t3000_h0_d0",
                                 "vogels_1000_s99_t3000_h0_d0", "vogels_500_s3_t500_h0_d3"])
@pytest.mark.parametrize("bitmap", [0, 2])
def test_streamed_state(golden, monkeypatch, tag, bitmap):
    """Streamed update (neuron state in HBM, loaded / stored every step; the
    mode for more neurons per CTA than registers hold, e.g. the p <= 0.01
    sweep networks), forced on the golden networks."""
    sim = build(golden["meta"]["runs"][tag], {"SYNQ_STREAM": 1, "SYNQ_BITMAP": bitmap}, monkeypatch, pipeline=1)
    assert sim.pipelined
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("tag", ["brunel_20000_s1_t2000_h0_d0", "brunel_2000_s99_t3000_h0_d0",
                                 "vogels_1000_s99_t3000_h0_d0"])
@pytest.mark.parametrize("uw", [4, 16])
def test_workqueue_delivery(golden, monkeypatch, tag, uw):
    """Barrier-free bitmap delivery (SYNQ_WORKQ=1: a poller warp claims
    frames, worker warps take 32-spike blocks from a linear work space) —
    experimental schedule, must be bit-exact like every other."""
    sim = build(golden["meta"]["runs"][tag], {"SYNQ_WORKQ": 1, "SYNQ_BITMAP": 2, "SYNQ_UW": uw}, monkeypatch,
                pipeline=1)
    assert sim.engine == "pipelined-bitmap"
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("tag", ["brunel_2000_s99_t3000_h0_d0", "vogels_1000_s99_t3000_h0_d0",
                                 "vogels_500_s3_t500_h0_d3", "vogels_4000_s1_t10000_h0_d0"])
@pytest.mark.parametrize("chunks", [None, "uneven"])
def test_solo_engine_bit_exact(golden, monkeypatch, tag, chunks):
    """Single-CTA engine (detail/solo.cuh, SYNQ_SOLO=1, <= 4096 neurons):
    bit-exact, also when run() is cut into launches of odd sizes (the frames
    of an earlier launch are delivered from global memory)."""
    m = golden["meta"]["runs"][tag]
    sim = build(m, {"SYNQ_SOLO": 1}, monkeypatch)
    assert sim.engine == "solo", sim.engine
    cuts = None
    if chunks:
        left, cuts = m["steps"], []
        for c in (1, 2, 13, 7, 301):
            c = min(c, left)
            cuts.append(c)
            left -= c
        cuts.append(left)
    check(sim, golden, tag, chunks=cuts)
    sim.close()


def test_solo_engine_is_opt_in(golden, monkeypatch):
    tag = "vogels_1000_s99_t3000_h0_d0"
    sim = build(golden["meta"]["runs"][tag], {}, monkeypatch)
    assert sim.engine != "solo"
    check(sim, golden, tag)
    sim.close()


@pytest.mark.parametrize("tag", ["brunel_2000_s99_t3000_h0_d0", "vogels_1000_s99_t3000_h0_d0",
                                 "vogels_500_s3_t500_h0_d3", "vogels_4000_s1_t10000_h0_d0"])
@pytest.mark.parametrize("size", [8, 16])
@pytest.mark.parametrize("chunks", [None, "uneven"])
def test_cluster_engine_bit_exact(golden, monkeypatch, tag, size, chunks):
    """One thread-block cluster (detail/cluster.cuh, SYNQ_CLUSTER=1): frames
    through distributed shared memory, bit-exact; uneven run() chunks make
    launches start from frames of an earlier launch."""
    m = golden["meta"]["runs"][tag]
    sim = build(m, {"SYNQ_CLUSTER": 1, "SYNQ_CLUSTER_SIZE": size}, monkeypatch)
    assert sim.engine == "cluster", sim.engine
    cuts = None
    if chunks:
        left, cuts = m["steps"], []
        for c in (1, 2, 13, 7, 301):
            c = min(c, left)
            cuts.append(c)
            left -= c
        cuts.append(left)
    check(sim, golden, tag, chunks=cuts)
    sim.close()
