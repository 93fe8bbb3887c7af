"""Multi-GPU shard protocol on CPU.

The wire format, batching over delay-1 steps, the torch.distributed exchange
(gloo, world_size 2) and the merge of the gathered frames are exercised with
an oracle-backed stand-in shard: every rank runs the whole network in the
oracle (test infrastructure only), exports the frames of its own id range in
the engine's export format and checks every frame it imports against its own
replica.  The merged frames must equal the oracle's unsharded frames.  The
same driver runs the CUDA shards in tests/test_gpu_shard.py.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_1912_07423_b200 import shard


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(3)
    fa = [np.sort(rng.choice(1000, rng.integers(0, 40), replace=False)).astype(np.uint32) for _ in range(7)]
    fb = [np.sort(rng.choice(1000, rng.integers(0, 5), replace=False)).astype(np.uint32) for _ in range(7)]
    w = shard.pack_frames(fa, fb)
    assert w[0] == 7 and len(w) == 1 + 14 + sum(map(len, fa)) + sum(map(len, fb))
    back = shard.unpack_frames(w)
    for (a, b), x, y in zip(back, fa, fb):
        assert np.array_equal(a, x) and np.array_equal(b, y)
    with pytest.raises(ValueError):
        shard.unpack_frames(np.concatenate([w, [1]]))


def test_empty_batch_and_merge():
    assert shard.unpack_frames(shard.pack_frames([], [])) == []
    w0 = shard.pack_frames([[5, 1]], [[900]])
    w1 = shard.pack_frames([[3]], [[]])
    (m,) = shard.merge_frames([w0, w1])
    assert m.tolist() == [1, 3, 5, 900]
    with pytest.raises(ValueError):
        shard.merge_frames([w0, shard.pack_frames([[3], [4]], [[], []])])


def test_assemble_field():
    a = np.arange(10, dtype=np.float32)
    b = -a
    out = shard.assemble_field([(((0, 4), (8, 9)), a), (((4, 8), (9, 10)), b)])
    assert out.tolist() == [0, 1, 2, 3, -4, -5, -6, -7, 8, -9]
    with pytest.raises(ValueError):
        shard.assemble_field([(((0, 4), (8, 8)), a)])


class OracleShard:
    """Stand-in with the CUDA shard's interface (run / shard_export /
    shard_import / shard_capacity / delay / counters), backed by a full
    oracle replica; rank r owns ids [r*n/W, (r+1)*n/W)."""

    def __init__(self, model, n, seed, rank, world):
        self.sim = oracle.Sim(model, n, seed)
        self.rank, self.world, self.n = rank, world, n
        self.delay = self.sim.delay
        self.lo = [q * n // world for q in range(world + 1)]
        self.imported = [0] * world
        self.batch = (0, 0)
        self.checked = 0

    def _frames(self, t0, b, q):
        counts, ids = self.sim.frames()
        off = np.concatenate([np.zeros(1, np.int64), np.cumsum(counts, dtype=np.int64)])
        out = []
        for t in range(t0, t0 + b):
            f = ids[off[t]:off[t + 1]]
            out.append(f[(f >= self.lo[q]) & (f < self.lo[q + 1])].astype(np.uint32))
        return out

    def run(self, b):
        t = self.sim.now()
        assert 0 < b <= self.delay - 1
        for q in range(self.world):  # the engine's guard (engine.hpp run())
            assert q == self.rank or self.imported[q] >= t + b - self.delay + 1
        self.sim.run(b)
        self.batch = (t, b)

    def shard_capacity(self):
        return 1 + 2 * self.delay + self.delay * (self.lo[self.rank + 1] - self.lo[self.rank])

    def shard_export(self):
        t0, b = self.batch
        fa = self._frames(t0, b, self.rank)
        return shard.pack_frames(fa, [np.empty(0, np.uint32)] * b)

    def shard_import(self, words, q):
        frames = shard.unpack_frames(words)
        mine = self._frames(self.imported[q], len(frames), q)
        for (a, bb), m in zip(frames, mine):
            assert len(bb) == 0 and np.array_equal(a, m)
            self.checked += 1
        self.imported[q] += len(frames)

    def counters(self):
        counts, ids = self.sim.frames()
        own = ids[(ids >= self.lo[self.rank]) & (ids < self.lo[self.rank + 1])]
        return {"spikes": int(len(own))}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, steps, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sim = OracleShard("vogels", 1000, 99, rank, world)
        ss = shard.ShardedSim("vogels", 1000, record=True, sim=sim)
        ss.run(steps)
        c = ss.counters()
        assert sim.checked == len(ss.frames) * (world - 1)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), spikes=c["spikes"],
                 counts=np.array([len(f) for f in ss.frames]),
                 ids=np.concatenate(ss.frames) if ss.frames else np.empty(0, np.uint32))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_exchange_matches_unsharded(world):
    steps = 157  # not a multiple of delay-1: the last batch is short
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), steps, d), nprocs=world,
                           join=True, start_method="spawn")
        ref = oracle.Sim("vogels", 1000, 99)
        ref.run(steps)
        rc, rids = ref.frames()
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            assert np.array_equal(z["counts"], rc)
            assert np.array_equal(z["ids"], _sorted_frames(rc, rids))
            assert int(z["spikes"]) == int(rc.sum())


def _sorted_frames(counts, ids):
    off = np.concatenate([np.zeros(1, np.int64), np.cumsum(counts, dtype=np.int64)])
    return np.concatenate([np.sort(ids[off[t]:off[t + 1]]) for t in range(len(counts))])
