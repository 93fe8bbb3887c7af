"""Target-partitioned shards on the B200 vs the reference.

W shards of one network (each a persistent engine that updates and receives
only its own id ranges) exchange frames every delay-1 steps; the merged
frames, the assembled neuron state and the summed counters must equal the
reference's unsharded run bit for bit (tests/golden).  One GPU holds all W
shards here; the NCCL transport is the same exchange with device buffers.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import paper_1912_07423_b200 as synq
from paper_1912_07423_b200 import shard

pytestmark = pytest.mark.gpu


def population_runs(golden):
    for tag, m in golden["meta"]["runs"].items():
        if m["model"] in ("vogels", "brunel") and not m["history"]:
            yield tag, m


def group(m, world, exchange="words", **kw):
    return shard.ShardGroup(m["model"], m["neurons"], world, record=True, seed=m["seed"], exchange=exchange,
                            deterministic=True, dt=m["dt"] or None, delay=m["delay"] or None, **kw)


@pytest.mark.parametrize("exchange", ["words", "bits"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_bit_exact(golden, world, exchange):
    """exchange="bits": the fixed-size bitmask blocks of the in-engine NCCL
    exchange (k_export_bits -> allgather -> k_import_bits), gathered by hand
    into one device buffer on this GPU."""
    runs = golden["runs"]
    n_cases = 0
    for tag, m in population_runs(golden):
        g = group(m, world, exchange)
        assert all(s.persistent for s in g.sims)
        g.run(m["steps"])
        counts = np.array([len(f) for f in g.frames])
        assert np.array_equal(counts, runs[f"{tag}_counts"]), (tag, world)
        assert np.array_equal(np.concatenate(g.frames), runs[f"{tag}_ids"]), (tag, world)
        for i in range(3):
            got = g.neuron_field(i).view(np.uint32)
            assert np.array_equal(got, runs[f"{tag}_f{i}"]), (tag, world, i)
        c, rc = g.counters(), m["counters"]
        assert c["spikes"] == rc["spikes"] and c["deliveries"] == rc["deliveries"], (tag, world)
        # every id range is owned by exactly one shard
        owned = sorted(r for s in g.sims for r in s.shard_range() if r[1] > r[0])
        assert owned[0][0] == 0 and owned[-1][1] == m["neurons"]
        assert all(a[1] == b[0] for a, b in zip(owned, owned[1:]))
        g.close()
        n_cases += 1
    assert n_cases >= 2


def test_sharded_tiles_invariance(golden):
    """Forcing different CTA counts per shard changes nothing."""
    tag, m = next(iter(population_runs(golden)))
    ref = None
    for tiles in (1, 3, 7):
        g = group(m, 2, tiles=tiles)
        g.run(m["steps"])
        ids = np.concatenate(g.frames)
        if ref is None:
            ref = ids
        assert np.array_equal(ids, ref), tiles
        g.close()


def test_export_format_matches_frames(golden):
    tag, m = next(iter(population_runs(golden)))
    g = group(m, 2)
    g.run(2 * (g.delay - 1) + 1)
    s0 = g.sims[0]
    (a0, a1), (b0, b1) = s0.shard_range()
    # a fresh export of the last (1-step) batch is consistent with the record
    words = s0.shard_export()
    (fa, fb), = shard.unpack_frames(words)
    assert np.all((fa >= a0) & (fa < a1)) and np.all((fb >= b0) & (fb < b1))
    last = g.frames[-1]
    assert set(fa.tolist()) | set(fb.tolist()) == set(last[((last >= a0) & (last < a1)) | ((last >= b0) & (last < b1))].tolist())
    assert len(words) <= s0.shard_capacity()
    g.close()


def test_shard_guards(golden):
    tag, m = next(iter(population_runs(golden)))
    opts = dict(seed=m["seed"], deterministic=True, dt=m["dt"] or None, delay=m["delay"] or None)
    s = synq.Sim(m["model"], m["neurons"], synq.Opts(shard=(0, 2), **opts))
    d = s.delay
    with pytest.raises(synq.SynqError):  # more than delay-1 steps between exchanges
        s.run(d)
    s.run(d - 1)
    with pytest.raises(synq.SynqError):  # frames of rank 1 not imported yet
        s.run(1)
    with pytest.raises(synq.SynqError):
        s.shard_import(np.array([0], np.uint32), 0)  # own rank
    s.close()
    with pytest.raises(synq.SynqError):
        synq.Opts(shard=(2, 2))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, m, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ss = shard.ShardedSim(m["model"], m["neurons"], record=True, seed=m["seed"], deterministic=True,
                              dt=m["dt"] or None, delay=m["delay"] or None)
        ss.run(m["steps"])
        c = ss.counters()
        rng = ss.sim.shard_range()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=np.concatenate(ss.frames),
                 counts=np.array([len(f) for f in ss.frames]), spikes=c["spikes"],
                 deliveries=c["deliveries"], rng=np.array(rng).reshape(-1), v=ss.sim.neuron_field(0))
        ss.close()
    finally:
        dist.destroy_process_group()


def test_sharded_processes_gloo(golden):
    """Two processes, one shard each, exchanging over torch.distributed."""
    import torch.multiprocessing as mp

    runs = golden["runs"]
    tag, m = next(iter(population_runs(golden)))
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), m, d), nprocs=2, join=True, start_method="spawn")
        parts = []
        for r in range(2):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            assert np.array_equal(z["counts"], runs[f"{tag}_counts"])
            assert np.array_equal(z["ids"], runs[f"{tag}_ids"])
            assert int(z["spikes"]) == m["counters"]["spikes"]
            assert int(z["deliveries"]) == m["counters"]["deliveries"]
            rg = z["rng"]
            parts.append((((rg[0], rg[1]), (rg[2], rg[3])), z["v"]))
        v = shard.assemble_field(parts)
        assert np.array_equal(v.view(np.uint32), runs[f"{tag}_f0"])


def test_nccl_in_engine_single_rank(golden):
    """The in-engine exchange end to end on one GPU: a one-rank NCCL
    communicator, export -> ncclAllGather -> import on the engine stream after
    every batch of delay-1 steps, recording through the shard's own frame
    log.  Frames, state and counters stay bit-exact with the reference."""
    runs = golden["runs"]
    for tag, m in population_runs(golden):
        uid = synq.nccl_unique_id()
        opts = synq.Opts(seed=m["seed"], deterministic=True, record=True, dt=m["dt"] or None,
                         delay=m["delay"] or None, shard_nccl=(0, 1, uid))
        sim = synq.Sim(m["model"], m["neurons"], opts)
        assert sim.persistent and sim.shard_capacity() > 0
        sim.run(m["steps"])  # any number of steps: the engine exchanges internally
        counts, ids = sim.frames()
        assert np.array_equal(counts, runs[f"{tag}_counts"]), tag
        assert np.array_equal(ids, runs[f"{tag}_ids"]), tag
        for i in range(3):
            assert np.array_equal(sim.neuron_field(i).view(np.uint32), runs[f"{tag}_f{i}"]), (tag, i)
        assert sim.counters()["deliveries"] == m["counters"]["deliveries"], tag
        sim.close()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_engine_log_segments_merged_frames(golden, world):
    """Every shard records through its own engine log (CTA 0 logs the merged
    frame, remote ranks' pieces included).  The log must be cut into steps by
    the merged per-frame counts, not by the shard's local spike counts: each
    shard's raster equals the reference frames up to the last delivered one."""
    runs = golden["runs"]
    for tag, m in population_runs(golden):
        g = group(m, world, "bits", engine_record=True)
        g.run(m["steps"])
        done = m["steps"] - g.delay + 1  # frames delivered (the rest await the next exchange)
        want_c = runs[f"{tag}_counts"][:done]
        want_ids = runs[f"{tag}_ids"][: int(want_c.sum())]
        for s in g.sims:
            counts, ids = s.frames()
            assert np.array_equal(counts[:done], want_c), (tag, world)
            assert np.array_equal(ids[: int(want_c.sum())], want_ids), (tag, world)
            assert counts[done:].sum() == 0
        g.close()


@pytest.mark.parametrize("world", [2, 4])
def test_shard_stores_only_its_sub_rows(world):
    """A shard builds only the sub-rows of its own targets:
    each row of its table is the full row restricted to the shard's receive
    range (still sorted, same ids), the sub-rows add up to the whole network,
    and the per-shard adjacency storage is about 1/W of the unsharded one."""
    n = 12000
    full = synq.Sim("brunel", n, synq.Opts(seed=5, deterministic=True))
    g = full.graph()
    deg = (g != 0xFFFFFFFF).sum(axis=1)
    grp = shard.ShardGroup("brunel", n, world, seed=5, deterministic=True)
    total = 0
    for s in grp.sims:
        lo, hi = s.shard_range()[0]
        sub = s.graph()
        sdeg = (sub != 0xFFFFFFFF).sum(axis=1)
        for r in range(0, n, 997):
            row = g[r, : deg[r]]
            want = row[(row >= lo) & (row < hi)]
            assert np.array_equal(sub[r, : sdeg[r]], want), (world, r)
        assert int(sdeg.sum()) == s.synapses
        total += s.synapses
        # padded sub-rows: pitch ~ deg_max / W (the ELL table is N x pitch)
        assert sub.shape[1] <= 1.3 * g.shape[1] / world + 32, (sub.shape, g.shape)
    assert total == full.synapses
    # the merged run is still bit-identical to the unsharded one
    grp.record = True
    ref = synq.Sim("brunel", n, synq.Opts(seed=5, deterministic=True, record=True))
    ref.run(3 * (grp.delay - 1))
    grp.run(3 * (grp.delay - 1))
    counts, ids = ref.frames()
    assert np.array_equal(np.array([len(f) for f in grp.frames]), counts)
    assert np.array_equal(np.concatenate(grp.frames), ids)
    grp.close()


@pytest.mark.timeout(600, method="thread")
@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_exchange_bit_exact(golden, world):
    """NVLink peer exchange (Opts(shard_peer=True)): the shards' step kernels
    store their frames into each other's rings, run side by side on this GPU
    (W x 8 CTAs), and every shard runs all steps in one run() call — no
    exchange between launches.  Frames (each shard's engine log holds the
    merged frames), state and counters equal the reference bit for bit."""
    runs = golden["runs"]
    n_cases = 0
    for tag, m in population_runs(golden):
        g = shard.PeerGroup(m["model"], m["neurons"], world, seed=m["seed"], deterministic=True, record=True,
                            dt=m["dt"] or None, delay=m["delay"] or None)
        assert all(s.persistent and s.pipelined for s in g.sims)
        g.run(m["steps"])
        for s in g.sims:
            counts, ids = s.frames()
            assert np.array_equal(counts, runs[f"{tag}_counts"]), (tag, world)
            assert np.array_equal(ids, runs[f"{tag}_ids"]), (tag, world)
        for i in range(3):
            assert np.array_equal(g.neuron_field(i).view(np.uint32), runs[f"{tag}_f{i}"]), (tag, world, i)
        c, rc = g.counters(), m["counters"]
        assert c["spikes"] == rc["spikes"] and c["deliveries"] == rc["deliveries"], (tag, world)
        g.close()
        n_cases += 1
    assert n_cases >= 2


@pytest.mark.timeout(600, method="thread")
@pytest.mark.parametrize("world", [2, 4])
def test_peer_exchange_batches_and_brunel_scale(world):
    """Peer shards across many launches (batch_steps 7 and 1000, runs cut
    at odd sizes) and at a network whose frames carry hundreds of ids: the
    merged raster equals the unsharded engine's."""
    n = 20000
    ref = synq.Sim("brunel", n, synq.Opts(seed=3, deterministic=True, record=True))
    ref.run(1200)
    rc, rids = ref.frames()
    rv = ref.neuron_field(0).view(np.uint32).copy()
    ref.close()
    for batch in (7, 1000):
        g = shard.PeerGroup("brunel", n, world, tiles=16, seed=3, deterministic=True, record=True, batch_steps=batch)
        for k in (1, 250, 949):
            g.run(k)
        counts, ids = g.sims[1].frames()
        assert np.array_equal(counts, rc), batch
        assert np.array_equal(ids, rids), batch
        assert np.array_equal(g.neuron_field(0).view(np.uint32), rv), batch
        g.close()


def _peer_worker(rank, world, port, m, out_dir):
    """One peer shard per process: IPC handles swapped over gloo, then the
    step kernels exchange frames through each other's memory."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sim = synq.Sim(m["model"], m["neurons"], synq.Opts(shard=(rank, world), shard_peer=True, tiles=4,
                                                           record=True, seed=m["seed"], deterministic=True,
                                                           dt=m["dt"] or None, delay=m["delay"] or None))
        handles = [None] * world
        dist.all_gather_object(handles, sim.peer_ipc_handle())
        sim.peer_connect_ipc(handles)
        dist.barrier()
        sim.run(m["steps"])
        counts, ids = sim.frames()
        rng = sim.shard_range()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids, counts=counts, rng=np.array(rng).reshape(-1),
                 v=sim.neuron_field(0))
        dist.barrier()  # the peer's ring stays mapped until both are done
        sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300, method="thread")
def test_peer_exchange_ipc_processes(golden):
    """Two processes on this GPU, one peer shard each, connected through
    cudaIpc handles (the multi-GPU wiring; here the two contexts share the
    device by time-slicing, so only a short run).  Each process's engine log
    holds the merged frames of the reference."""
    import torch.multiprocessing as mp

    runs = golden["runs"]
    tag, m = next(iter(population_runs(golden)))
    m = dict(m, steps=min(m["steps"], 200))
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_peer_worker, args=(2, _free_port(), m, d), nprocs=2, join=True, start_method="spawn")
        want_c = runs[f"{tag}_counts"][: m["steps"]]
        want_ids = runs[f"{tag}_ids"][: int(want_c.sum())]
        parts = []
        for r in range(2):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            assert np.array_equal(z["counts"], want_c), r
            assert np.array_equal(z["ids"], want_ids), r
            rg = z["rng"]
            parts.append((((rg[0], rg[1]), (rg[2], rg[3])), z["v"]))
        assert len(shard.assemble_field(parts)) == m["neurons"]
