"""Target-partitioned multi-GPU shards.

One process per GPU.  Shard r owns a contiguous range of the receiving
neurons and of the update-only neurons; it updates only those, and delivers
every spike of the network only onto its own targets.  The one exchange step
is the spike frame: a spike produced at step t is due at t+delay, so a shard
can run delay-1 steps ahead before it needs the other shards' frames of that
batch (the engine's look-ahead keeps one frame in flight, hence delay-1 and
not delay).  Per batch each shard

    run(b)  ->  export (its frames of the b steps)  ->  allgather  ->  import

The reference parallelises the same pipeline over threads of one address
space (proj/include/synq/engine.hpp:181-224: update / exchange / receive per
step, the spike queue shared by all threads); here the shared queue becomes
the allgathered frame buffer.

Export wire format (uint32 words, written by k_export in
include/synq/detail/persistent.cuh): [b, (a_0, b_0), …, (a_{b-1}, b_{b-1}),
ids of step 0 (receiving piece, then update-only piece), ids of step 1, …].

Drivers: `ShardGroup` holds all W shards in one process (one GPU; the
bit-exact check of the protocol against the unsharded engine);
`ShardedSim` is one process's shard, exchanging through `TorchTransport` over
torch.distributed — NCCL with device buffers (the words never leave HBM), or
gloo with host buffers.
"""
from __future__ import annotations

import numpy as np

from . import Opts, Sim


# ---------------------------------------------------------------------------
# wire format
def pack_frames(frames_a, frames_b) -> np.ndarray:
    """Pack per-step (receiving ids, update-only ids) into export words."""
    b = len(frames_a)
    assert len(frames_b) == b
    head = np.empty(1 + 2 * b, np.uint32)
    head[0] = b
    head[1::2] = [len(x) for x in frames_a]
    head[2::2] = [len(x) for x in frames_b]
    body = [np.asarray(x, np.uint32) for pair in zip(frames_a, frames_b) for x in pair]
    return np.concatenate([head] + body) if body else head


def unpack_frames(words):
    """Inverse of pack_frames: list of (receiving ids, update-only ids)."""
    w = np.asarray(words, np.uint32)
    b = int(w[0])
    ca, cb = w[1:1 + 2 * b:2].astype(np.int64), w[2:2 + 2 * b:2].astype(np.int64)
    pos = 1 + 2 * b
    out = []
    for k in range(b):
        a = w[pos:pos + ca[k]]
        pos += ca[k]
        bb = w[pos:pos + cb[k]]
        pos += cb[k]
        out.append((a, bb))
    if pos != len(w):
        raise ValueError(f"frame words: {len(w)} given, {pos} described")
    return out


# ---------------------------------------------------------------------------
class TorchTransport:
    """torch.distributed allgather of each shard's export.

    With the NCCL backend the export is written straight into a device
    buffer and the gathered frames are imported from device memory; with
    gloo the words go through host tensors.  Two collectives per batch: the
    word counts, then the words padded to the largest count.
    """

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = (torch.device("cuda", torch.cuda.current_device())
                       if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        self.bufs = None

    def _ensure(self, cap):
        torch = self.torch
        if self.bufs is None or self.bufs[0].numel() < cap:
            self.bufs = (torch.empty(cap, dtype=torch.int32, device=self.device),
                         torch.empty(self.world * cap, dtype=torch.int32, device=self.device))
        return self.bufs

    def max_capacity(self, cap: int) -> int:
        t = self.torch.tensor([cap], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def exchange_sim(self, sim: Sim, cap: int):
        """Export sim's last batch, allgather, import every other rank's
        frames.  Returns (gathered words, words per rank, padded stride)."""
        torch, dist = self.torch, self.dist
        send, recv = self._ensure(cap)
        if self.device.type == "cuda":
            torch.cuda.current_stream().synchronize()
            n = sim.shard_export(device_ptr=send.data_ptr(), capacity=cap)
        else:
            w = sim.shard_export()
            n = len(w)
            send[:n] = torch.from_numpy(w.view(np.int32))
        counts = torch.tensor([n], dtype=torch.int64, device=self.device)
        allc = torch.empty(self.world, dtype=counts.dtype, device=self.device)
        dist.all_gather_into_tensor(allc, counts, group=self.group)
        allc = [int(x) for x in allc.tolist()]
        m = max(allc)
        out = recv[: self.world * m]
        dist.all_gather_into_tensor(out, send[:m].contiguous(), group=self.group)
        if self.device.type == "cuda":
            torch.cuda.current_stream().synchronize()
        for q in range(self.world):
            if q == self.rank:
                continue
            seg = out[q * m: q * m + allc[q]]
            if self.device.type == "cuda":
                sim.shard_import(None, q, device_ptr=seg.data_ptr(), nwords=allc[q])
            else:
                sim.shard_import(seg.numpy().view(np.uint32), q)
        return out, allc, m

    def allreduce_sum(self, values):
        t = self.torch.tensor(values, dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, group=self.group)
        return [int(x) for x in t.tolist()]


# ---------------------------------------------------------------------------
class ShardGroup:
    """W shards of one network driven from one process (one GPU).

    Each shard is a full synq engine restricted to its range; frames move
    between them through host memory.  Used to check the sharded protocol
    bit-exactly against the unsharded engine on a single B200, and as the
    one-GPU stand-in for a multi-GPU run.
    """

    def __init__(self, model: str, neurons: int, world: int, record: bool = False, exchange: str = "words",
                 engine_record: bool = False, **opts):
        # record: merge the exported frames here; engine_record: every shard
        # also records the merged frames through its own engine log
        self.world = world
        self.sims = [Sim(model, neurons, Opts(shard=(r, world), record=engine_record or None, **opts))
                     for r in range(world)]
        self.delay = self.sims[0].delay
        self.record = record
        self.exchange = exchange  # "words" (host wire format) or "bits" (the in-engine bitmask blocks)
        self.frames: list[np.ndarray] = []
        self._gathered = None

    def _bits_exchange(self):
        """What ncclAllGather does for the in-engine exchange: every rank's
        bitmask block side by side in one device buffer, imported by all."""
        import torch

        words = self.sims[0].shard_bits_words()
        if self._gathered is None:
            self._gathered = torch.zeros(self.world * words, dtype=torch.int32, device="cuda")
        g = self._gathered
        for r, s in enumerate(self.sims):
            s.shard_export_bits(g.data_ptr() + 4 * r * words)
        for s in self.sims:
            s.shard_import_bits(g.data_ptr())

    def run(self, steps: int):
        batch = self.delay - 1
        while steps > 0:
            b = min(steps, batch)
            for s in self.sims:
                s.run(b)
            if self.exchange == "bits":
                words = [s.shard_export() for s in self.sims] if self.record else None
                self._bits_exchange()
            else:
                words = [s.shard_export() for s in self.sims]
                for r, s in enumerate(self.sims):
                    for q in range(self.world):
                        if q != r:
                            s.shard_import(words[q], q)
            if self.record:
                self.frames.extend(merge_frames(words))
            steps -= b

    def neuron_field(self, f: int, dtype=np.float32) -> np.ndarray:
        return assemble_field([(s.shard_range(), s.neuron_field(f, dtype)) for s in self.sims])

    def counters(self) -> dict:
        out: dict = {}
        for s in self.sims:
            for k, v in s.counters().items():
                out[k] = out.get(k, 0) + v
        return out

    def close(self):
        for s in self.sims:
            s.close()


class PeerGroup:
    """W peer-exchange shards of one network in one process (one GPU).

    Opts(shard_peer=True): every shard's step kernel stores its frames into
    the other shards' queue rings and releases them there
    (include/synq/detail/persistent.cuh peer_export), so run(steps) is one
    run() per shard with no exchange between launches.  The W kernels wait
    on each other's frames and must run side by side: each shard gets
    `tiles` CTAs (W x tiles <= the SM count), and the shards run from one
    host thread each.  Across GPUs the same kernels run one per device,
    connected through IPC handles (Sim.peer_ipc_handle / peer_connect_ipc).
    """

    def __init__(self, model: str, neurons: int, world: int, tiles: int = 8, synapses: int | None = None, **opts):
        self.world = world
        self.sims = [Sim(model, neurons, Opts(shard=(r, world), shard_peer=True, tiles=tiles, **opts),
                         synapses=synapses) for r in range(world)]
        self.delay = self.sims[0].delay
        eps = [s.peer_endpoint() for s in self.sims]
        for s in self.sims:
            s.peer_connect(eps)

    def run(self, steps: int):
        import threading

        errors: list[BaseException] = []

        def go(s):
            try:
                s.run(steps)
            except BaseException as e:  # re-raised below
                errors.append(e)

        threads = [threading.Thread(target=go, args=(s,)) for s in self.sims]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]

    def neuron_field(self, f: int, dtype=np.float32) -> np.ndarray:
        return assemble_field([(s.shard_range(), s.neuron_field(f, dtype)) for s in self.sims])

    def counters(self) -> dict:
        out: dict = {}
        for s in self.sims:
            for k, v in s.counters().items():
                out[k] = out.get(k, 0) + v
        return out

    def close(self):
        for s in self.sims:
            s.close()


class ShardedSim:
    """This process's shard of a network, exchanging frames over
    torch.distributed (launch one process per GPU with torchrun)."""

    def __init__(self, model: str, neurons: int, transport: TorchTransport | None = None,
                 record: bool = False, sim=None, **opts):
        self.transport = transport or TorchTransport()
        self.rank, self.world = self.transport.rank, self.transport.world
        # `sim` lets a test substitute any object with the shard interface
        self.sim = sim if sim is not None else Sim(model, neurons, Opts(shard=(self.rank, self.world), **opts))
        self.delay = self.sim.delay
        self.cap = self.transport.max_capacity(self.sim.shard_capacity())
        self.record = record
        self.frames: list[np.ndarray] = []

    def run(self, steps: int):
        batch = self.delay - 1
        while steps > 0:
            b = min(steps, batch)
            self.sim.run(b)
            out, allc, m = self.transport.exchange_sim(self.sim, self.cap)
            if self.record:
                host = out.cpu().numpy().view(np.uint32)
                self.frames.extend(merge_frames([host[q * m: q * m + allc[q]] for q in range(self.world)]))
            steps -= b

    def counters(self) -> dict:
        c = self.sim.counters()
        keys = sorted(c)
        return dict(zip(keys, self.transport.allreduce_sum([int(c[k]) for k in keys])))

    def close(self):
        self.sim.close()


def merge_frames(words_by_rank) -> list[np.ndarray]:
    """Global frames of one batch: the union of every shard's ids per step,
    in id order (the order the unsharded engine's pieces tile the id space)."""
    per = [unpack_frames(w) for w in words_by_rank]
    b = len(per[0])
    if any(len(p) != b for p in per):
        raise ValueError("shards exported different batch lengths")
    return [np.sort(np.concatenate([x for p in per for x in p[k]])) for k in range(b)]


def assemble_field(parts) -> np.ndarray:
    """Global neuron field from each shard's (range, full-size array), taking
    every shard's own receiving and update-only ranges."""
    (ra, ub), arr = parts[0]
    out = np.empty_like(arr)
    covered = np.zeros(len(arr), bool)
    for ((a0, a1), (b0, b1)), arr in parts:
        out[a0:a1] = arr[a0:a1]
        out[b0:b1] = arr[b0:b1]
        covered[a0:a1] = True
        covered[b0:b1] = True
    if not covered.all():
        raise ValueError("shard ranges do not cover the network")
    return out
