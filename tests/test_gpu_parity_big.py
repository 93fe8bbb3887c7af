"""Parity at the benchmarked configuration (BASELINE.json configs[1]):
Brunel sized for ~1e9 synapses (141,421 neurons, 999,981,220 synapses),
seed 1, one full biological second (10,000 steps), built and run through
the C ABI exactly as bench.py does (synq_sim_new_for_synapses).

The goldens come from the UNMODIFIED reference at this size
(tests/golden/make_golden.py big -> oracle/_ref/synq_golden big), reduced
to hashes so they fit the repo:
  * adjacency: sha256 of the whole padded ELL table (adjacency.cpp:29-109),
    per-1024-row block digests (to locate a difference), degree vector;
  * frames: spike count and a sha256-based digest of the ascending ids of
    every one of the 10,000 steps (engine.hpp:188-218); the reference's own
    parallel and deterministic modes part at step 2,213 at this size;
  * final V / ACC / REF bits (sha256) and the counters.
Tolerance: none.  Float state is compared as raw bits.
"""
import hashlib

import numpy as np
import pytest

import paper_1912_07423_b200 as synq

pytestmark = pytest.mark.gpu

TAG = "brunel_1e09_s1_t10000"


def digests(counts, ids):
    out = np.empty(len(counts), np.uint64)
    off = 0
    for k, c in enumerate(counts):
        h = hashlib.sha256(np.ascontiguousarray(ids[off:off + c], "<u4").tobytes()).digest()
        out[k] = int.from_bytes(h[:8], "little")
        off += int(c)
    return out


@pytest.fixture(scope="module")
def big_sim(golden):
    m = golden["meta"]["big"][TAG]
    sim = synq.Sim(m["model"], opts=synq.Opts(seed=m["seed"], record=True), synapses=m["synapses"])
    yield m, sim
    sim.close()


def test_brunel_1e9_adjacency_matches_reference(golden, big_sim):
    m, sim = big_sim
    big = golden["big"]
    assert sim.neurons == m["neurons"] and sim.synapses == m["edges"]
    cells = sim.graph()
    assert cells.shape == (m["neurons"], m["pitch"])
    deg = (cells != 0xFFFFFFFF).sum(1).astype(np.uint32)
    assert np.array_equal(deg, big[f"{TAG}_deg"])
    h = hashlib.sha256()
    blocks = []
    for r0 in range(0, m["neurons"], 1024):
        b = np.ascontiguousarray(cells[r0:r0 + 1024]).tobytes()
        h.update(b)
        blocks.append(int.from_bytes(hashlib.sha256(b).digest()[:8], "little"))
    bad = np.nonzero(np.array(blocks, np.uint64) != big[f"{TAG}_blocks"])[0]
    assert len(bad) == 0, f"adjacency differs in 1024-row blocks {bad[:10].tolist()}"
    assert h.hexdigest() == m["adj_sha256"]
    del cells


def test_brunel_1e9_full_second_bit_exact(golden, big_sim):
    m, sim = big_sim
    big = golden["big"]
    assert sim.persistent and sim.exact
    sim.run(m["steps"])
    counts, ids = sim.frames()
    want_c = big[f"{TAG}_counts"]
    assert len(counts) == len(want_c) == m["steps"]
    diff = np.nonzero(counts != want_c)[0]
    assert len(diff) == 0, f"spike counts first differ at step {diff[0]}"
    got_d = digests(counts, ids)
    diff = np.nonzero(got_d != big[f"{TAG}_digests"])[0]
    assert len(diff) == 0, f"spike ids first differ at step {diff[0]}"
    for i in range(3):
        f = sim.neuron_field(i).view(np.uint32)
        assert np.array_equal(f[:4096], big[f"{TAG}_f{i}_head"]), i
        assert hashlib.sha256(f.tobytes()).hexdigest() == m["state_sha256"][i], i
    c, rc = sim.counters(), m["counters"]
    assert c["spikes"] == rc["spikes"]
    assert c["deliveries"] == rc["deliveries"]
    assert c["frames_consumed"] == rc["frames_consumed"]


# ---- Brunel+ (BASELINE.json configs[2]) at 1e8 and 1e9 synapses, short
# horizons (tests/golden/make_golden.py bigp): frames, neuron state, ages,
# then the synapse state after flush (sha256 per field), ordered mode.
@pytest.mark.parametrize("tag", ["brunelp_1e08_s1_t400", "brunelp_1e09_s1_t100"])
def test_brunel_plus_at_scale_bit_exact(golden, tag):
    if "bigp" not in golden["meta"] or tag not in golden["meta"]["bigp"]:
        pytest.skip("bigp goldens not generated")
    m = golden["meta"]["bigp"][tag]
    big = golden["bigp"]
    sim = synq.Sim("brunel+", opts=synq.Opts(seed=m["seed"], deterministic=True, record=True),
                   synapses=m["synapses"])
    assert sim.neurons == m["neurons"] and sim.exact
    sim.run(m["steps"])
    counts, ids = sim.frames()
    diff = np.nonzero(counts != big[f"{tag}_counts"])[0]
    assert len(diff) == 0, f"spike counts first differ at step {diff[0]}"
    diff = np.nonzero(digests(counts, ids) != big[f"{tag}_digests"])[0]
    assert len(diff) == 0, f"spike ids first differ at step {diff[0]}"
    for i in range(3):
        f = sim.neuron_field(i).view(np.uint32)
        assert hashlib.sha256(f.tobytes()).hexdigest() == m["state_sha256"][i], i
    assert hashlib.sha256(sim.ages().tobytes()).hexdigest() == m["ages_sha256"]
    c, rc = sim.counters(), m["counters"]
    assert c["synapse_updates"] == rc["preflush_synapse_updates"]
    sim.flush()
    for i in range(3):
        f = sim.synapse_field(i).view(np.uint32)
        assert hashlib.sha256(f.tobytes()).hexdigest() == m["syn_sha256"][i], i
        del f
    c = sim.counters()
    assert c["spikes"] == rc["spikes"] and c["deliveries"] == rc["deliveries"]
    assert c["synapse_updates"] == rc["synapse_updates"]
    sim.close()


@pytest.mark.timeout(900, method="thread")
def test_brunel_1e9_peer_shards_full_second_bit_exact(golden):
    """The bench network as two NVLink-peer shards (Opts(shard_peer=True)),
    side by side on this GPU with 74 CTAs each, one run() of the whole
    biological second: each shard stores only its targets' sub-rows, the
    step kernels store their frames into each other's rings, and every
    shard's engine log (the merged frames) and the assembled state equal the
    reference's, step for step."""
    from paper_1912_07423_b200 import shard

    m = golden["meta"]["big"][TAG]
    big = golden["big"]
    g = shard.PeerGroup(m["model"], 0, 2, tiles=74, synapses=m["synapses"], seed=m["seed"], deterministic=True,
                        record=True)
    assert sum(s.synapses for s in g.sims) == m["edges"]
    g.run(m["steps"])
    for r, s in enumerate(g.sims):
        counts, ids = s.frames()
        diff = np.nonzero(counts != big[f"{TAG}_counts"])[0]
        assert len(diff) == 0, f"shard {r}: spike counts first differ at step {diff[0]}"
        diff = np.nonzero(digests(counts, ids) != big[f"{TAG}_digests"])[0]
        assert len(diff) == 0, f"shard {r}: spike ids first differ at step {diff[0]}"
    for i in range(3):
        f = g.neuron_field(i).view(np.uint32)
        assert hashlib.sha256(f.tobytes()).hexdigest() == m["state_sha256"][i], i
    g.close()
