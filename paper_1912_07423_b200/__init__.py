"""B200-native synq: ctypes host binding of the C ABI in include/synq/synq.h.

This is the Python-side mirror of the reference's C interface
(/root/reference/proj/include/synq/synq.h): the same entry points, argument
meaning and status codes, loaded from the in-tree libsynq.so.1 that the
Makefile builds for sm_100a.  There is no CPU fallback: if the library is
missing, or no CUDA device is usable, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("SYNQ_LIB") or os.path.join(PKG_DIR, "lib", "libsynq.so.1")
HEADER = os.path.join(ROOT, "include", "synq", "synq.h")

SYNQ_OK = 0
STATUS = {0: "ok", 1: "invalid argument", 2: "unknown model", 3: "io error",
          4: "out of memory", 5: "internal error"}
PHASES = {"construct": 0, "init_neurons": 1, "init_synapses": 2, "simulate": 3}


class SynqError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"synq status {status} ({STATUS.get(status, '?')}): {message}")
        self.status = status
        self.message = message


def build(jobs: int = 8) -> None:
    """Compile libsynq.so.1 for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", ROOT, f"-j{jobs}", "lib"], check=True)


def declared_symbols() -> list[str]:
    """Every function declared in include/synq/synq.h."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(synq_[a-z_0-9]+)\s*\(", text)))


class _Memory(C.Structure):
    _fields_ = [(k, C.c_double) for k in (
        "neuron_fields", "neuron_spikes", "neuron_bitmasks", "neuron_ages",
        "neuron_expirations", "synapse_adjacency", "synapse_fields", "neuron_total",
        "synapse_total", "total_bytes")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `make lib` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i64, dbl, cs = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int64, C.c_double, C.c_char_p
    st = C.c_int

    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)

    sig("synq_version", cs)
    sig("synq_status_name", cs, st)
    sig("synq_last_error", cs)
    sig("synq_opts_new", vp)
    sig("synq_opts_free", None, vp)
    sig("synq_opts_seed", st, vp, u64)
    sig("synq_opts_threads", st, vp, u32)
    sig("synq_opts_deterministic", st, vp, C.c_int)
    sig("synq_opts_dt", st, vp, dbl)
    sig("synq_opts_delay", st, vp, u32)
    sig("synq_opts_record", st, vp, C.c_int)
    sig("synq_opts_defaults_file", st, vp, cs)
    sig("synq_opts_param", st, vp, cs, dbl)
    sig("synq_sim_new", st, cs, u32, vp, C.POINTER(vp))
    sig("synq_sim_new_for_synapses", st, cs, u64, vp, C.POINTER(vp))
    sig("synq_sim_new_from_file", st, cs, cs, vp, C.POINTER(vp))
    sig("synq_sim_free", None, vp)
    sig("synq_sim_step", st, vp)
    sig("synq_sim_run", st, vp, i64)
    sig("synq_sim_flush", st, vp)
    sig("synq_sim_neurons", u32, vp)
    sig("synq_sim_synapses", u64, vp)
    sig("synq_sim_ages", st, vp, vp, u64)
    sig("synq_sim_synapse_capacity", u64, vp)
    sig("synq_sim_now", i64, vp)
    sig("synq_sim_dt", dbl, vp)
    sig("synq_sim_delay", u32, vp)
    sig("synq_sim_seed", u64, vp)
    sig("synq_sim_scaling", dbl, vp)
    sig("synq_sim_firing_rate", st, vp, C.POINTER(dbl))
    sig("synq_sim_spike_count", st, vp, C.POINTER(u64))
    sig("synq_sim_seconds", dbl, vp, C.c_int)
    sig("synq_sim_write_raster", st, vp, cs)
    sig("synq_sim_write_stats", st, vp, cs)
    sig("synq_memory_estimate", st, cs, u64, u64, C.POINTER(_Memory))
    sig("synq_sim_memory_actual", st, vp, C.POINTER(_Memory))
    sig("synq_scaling_constant", st, cs, u64, C.POINTER(dbl))
    sig("synq_solve_neurons", st, cs, u64, C.POINTER(u32))
    # B200 extensions
    sig("synq_opts_batch_steps", st, vp, u32)
    sig("synq_opts_persistent", st, vp, C.c_int)
    sig("synq_opts_tiles", st, vp, u32)
    sig("synq_opts_pipeline", st, vp, C.c_int, u32)
    sig("synq_sim_engine", C.c_int, vp)
    sig("synq_sim_exact", C.c_int, vp)
    sig("synq_sim_counters", st, vp, vp)
    sig("synq_sim_raster_size", st, vp, C.POINTER(u64))
    sig("synq_sim_raster_copy", st, vp, vp, vp, u64)
    sig("synq_sim_step_spikes", st, vp, vp, u64)
    sig("synq_sim_neuron_field", st, vp, u32, vp, u64)
    sig("synq_sim_synapse_field", st, vp, u32, vp, u64)
    sig("synq_sim_graph_shape", st, vp, C.POINTER(u32), C.POINTER(u32))
    sig("synq_sim_graph_cells", st, vp, vp, u64)
    sig("synq_sim_construction_fixups", u64, vp)
    sig("synq_sim_device_time", st, vp, vp)
    sig("synq_sim_kernel_launches", u64, vp)
    sig("synq_sim_transfer_bytes", st, vp, vp)
    sig("synq_sim_set_record", st, vp, C.c_int)
    sig("synq_opts_profile", st, vp, C.c_int)
    sig("synq_opts_shard", st, vp, u32, u32)
    sig("synq_sim_shard_capacity", u64, vp)
    sig("synq_sim_shard_range", st, vp, C.POINTER(u32))
    sig("synq_sim_shard_export", st, vp, vp, u64, C.c_int, C.POINTER(u64))
    sig("synq_sim_shard_import", st, vp, vp, u64, u32, C.c_int)
    sig("synq_sim_phase_cycles", st, vp, vp, C.POINTER(u32))
    sig("synq_nccl_unique_id", st, vp)
    sig("synq_opts_shard_nccl", st, vp, u32, u32, vp)
    sig("synq_sim_shard_bits_words", u64, vp)
    sig("synq_sim_shard_export_bits", st, vp, vp)
    sig("synq_sim_shard_import_bits", st, vp, vp)
    sig("synq_opts_shard_peer", st, vp, C.c_int)
    sig("synq_sim_peer_endpoint", st, vp, C.POINTER(PeerEndpoint))
    sig("synq_sim_peer_connect", st, vp, C.POINTER(PeerEndpoint), u32)
    sig("synq_sim_peer_ipc_handle", st, vp, vp)
    sig("synq_sim_peer_connect_ipc", st, vp, vp, u32)
    _lib = L
    return L


def check(status: int) -> None:
    if status != SYNQ_OK:
        raise SynqError(status, lib().synq_last_error().decode(errors="replace"))


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Opts:
    """synq_opts (synq.h:33-47) plus the B200 extensions."""

    def __init__(self, seed=None, threads=None, deterministic=None, dt=None, delay=None,
                 record=None, defaults_file=None, params=None, batch_steps=None,
                 persistent=None, tiles=None, profile=None, shard=None, pipeline=None, lead=0,
                 shard_nccl=None, shard_peer=None):
        self._L = lib()  # kept: module globals may be gone when __del__ runs at exit
        self.h = self._L.synq_opts_new()
        if not self.h:
            raise MemoryError("synq_opts_new")
        L = lib()
        if seed is not None:
            check(L.synq_opts_seed(self.h, seed))
        if threads is not None:
            check(L.synq_opts_threads(self.h, threads))
        if deterministic is not None:
            check(L.synq_opts_deterministic(self.h, int(deterministic)))
        if dt is not None:
            check(L.synq_opts_dt(self.h, dt))
        if delay is not None:
            check(L.synq_opts_delay(self.h, delay))
        if record is not None:
            check(L.synq_opts_record(self.h, int(record)))
        if defaults_file is not None:
            check(L.synq_opts_defaults_file(self.h, defaults_file.encode()))
        for k, v in (params or {}).items():
            check(L.synq_opts_param(self.h, k.encode(), float(v)))
        if batch_steps is not None:
            check(L.synq_opts_batch_steps(self.h, batch_steps))
        if persistent is not None:
            check(L.synq_opts_persistent(self.h, persistent))
        if tiles is not None:
            check(L.synq_opts_tiles(self.h, tiles))
        if pipeline is not None:
            check(L.synq_opts_pipeline(self.h, int(pipeline), int(lead)))
        if profile is not None:
            check(L.synq_opts_profile(self.h, int(profile)))
        if shard is not None:
            check(L.synq_opts_shard(self.h, int(shard[0]), int(shard[1])))
        if shard_nccl is not None:  # (rank, world, 128-byte NCCL unique id)
            _prefer_torch_nccl()
            rank, world, uid = shard_nccl
            buf = C.create_string_buffer(bytes(uid), 128)
            check(L.synq_opts_shard_nccl(self.h, int(rank), int(world), buf))
        if shard_peer is not None:  # NVLink peer exchange (after shard / shard_nccl)
            check(L.synq_opts_shard_peer(self.h, int(shard_peer)))

    def __del__(self):
        if getattr(self, "h", None):
            self._L.synq_opts_free(self.h)
            self.h = None


class Sim:
    """synq_sim (synq.h:51-122) on the B200."""

    def __init__(self, model: str, neurons: int = 0, opts: Opts | None = None,
                 synapses: int | None = None, desc_path: str | None = None):
        h = C.c_void_p()
        o = opts.h if opts is not None else None
        L = lib()
        if desc_path is not None:
            check(L.synq_sim_new_from_file(model.encode(), desc_path.encode(), o, C.byref(h)))
        elif synapses is not None:
            check(L.synq_sim_new_for_synapses(model.encode(), synapses, o, C.byref(h)))
        else:
            check(L.synq_sim_new(model.encode(), neurons, o, C.byref(h)))
        self._L = lib()
        self.h = h
        self._opts = opts

    def close(self):
        if getattr(self, "h", None):
            self._L.synq_sim_free(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # stepping
    def step(self):
        check(lib().synq_sim_step(self.h))

    def run(self, steps: int):
        check(lib().synq_sim_run(self.h, steps))

    def flush(self):
        check(lib().synq_sim_flush(self.h))

    # queries
    @property
    def neurons(self):
        return int(lib().synq_sim_neurons(self.h))

    @property
    def synapses(self):
        return int(lib().synq_sim_synapses(self.h))

    @property
    def synapse_capacity(self):
        return int(lib().synq_sim_synapse_capacity(self.h))

    def now(self):
        return int(lib().synq_sim_now(self.h))

    @property
    def dt(self):
        return float(lib().synq_sim_dt(self.h))

    @property
    def delay(self):
        return int(lib().synq_sim_delay(self.h))

    @property
    def seed(self):
        return int(lib().synq_sim_seed(self.h))

    @property
    def scaling(self):
        return float(lib().synq_sim_scaling(self.h))

    @property
    def persistent(self) -> bool:
        return bool(lib().synq_sim_engine(self.h))

    @property
    def pipelined(self) -> bool:
        return lib().synq_sim_engine(self.h) >= 2

    @property
    def engine(self) -> str:
        return {0: "graph", 1: "persistent", 2: "pipelined", 3: "pipelined-bitmap", 4: "solo", 5: "cluster"}[
            lib().synq_sim_engine(self.h)]

    @property
    def exact(self) -> bool:
        return bool(lib().synq_sim_exact(self.h))

    def firing_rate(self) -> float:
        r = C.c_double()
        check(lib().synq_sim_firing_rate(self.h, C.byref(r)))
        return r.value

    def spike_count(self) -> int:
        r = C.c_uint64()
        check(lib().synq_sim_spike_count(self.h, C.byref(r)))
        return r.value

    def seconds(self, phase: str = "simulate") -> float:
        return float(lib().synq_sim_seconds(self.h, PHASES[phase]))

    def counters(self) -> dict:
        c = np.zeros(6, np.uint64)
        check(lib().synq_sim_counters(self.h, _p(c)))
        return dict(zip(["steps", "spikes", "deliveries", "synapse_updates", "expiry_batches",
                         "frames_consumed"], (int(x) for x in c)))

    def write_raster(self, path: str):
        check(lib().synq_sim_write_raster(self.h, path.encode()))

    def write_stats(self, path: str = "-"):
        check(lib().synq_sim_write_stats(self.h, path.encode()))

    def memory_actual(self) -> dict:
        m = _Memory()
        check(lib().synq_sim_memory_actual(self.h, C.byref(m)))
        return m.as_dict()

    def raster(self, out=None):
        """(steps, ids) of the recorded raster.  `out` = (int64, uint32) arrays
        to fill (grown when too small) lets a caller reuse its buffers."""
        n = C.c_uint64()
        check(lib().synq_sim_raster_size(self.h, C.byref(n)))
        if out is not None and len(out[0]) >= n.value and len(out[1]) >= n.value:
            steps, ids = out
        else:
            steps = np.empty(max(n.value, 1), np.int64)
            ids = np.empty(max(n.value, 1), np.uint32)
        check(lib().synq_sim_raster_copy(self.h, _p(steps), _p(ids), n.value))
        return steps[: n.value], ids[: n.value]

    def step_spikes(self) -> np.ndarray:
        out = np.empty(max(self.now(), 1), np.uint32)
        check(lib().synq_sim_step_spikes(self.h, _p(out), len(out)))
        return out[: self.now()]

    def frames(self):
        """(counts per step, concatenated sorted ids) from the recorded raster."""
        steps, ids = self.raster()
        counts = np.bincount(steps, minlength=self.now()).astype(np.uint32) if len(steps) else \
            np.zeros(self.now(), np.uint32)
        return counts, ids

    def neuron_field(self, f: int, dtype=np.float32) -> np.ndarray:
        out = np.empty(self.neurons, dtype)
        check(lib().synq_sim_neuron_field(self.h, f, _p(out), out.nbytes))
        return out

    def synapse_field(self, f: int, dtype=np.float32) -> np.ndarray:
        out = np.empty(max(self.synapse_capacity, 1), dtype)
        check(lib().synq_sim_synapse_field(self.h, f, _p(out), out.nbytes))
        return out[: self.synapse_capacity]

    def ages(self) -> np.ndarray:
        out = np.empty(max(self.neurons, 1), np.uint32)
        check(lib().synq_sim_ages(self.h, _p(out), len(out)))
        return out[: self.neurons]

    def graph(self) -> np.ndarray:
        pitch, dmax = C.c_uint32(), C.c_uint32()
        check(lib().synq_sim_graph_shape(self.h, C.byref(pitch), C.byref(dmax)))
        out = np.empty(max(self.neurons * pitch.value, 1), np.uint32)
        check(lib().synq_sim_graph_cells(self.h, _p(out), len(out)))
        return out[: self.neurons * pitch.value].reshape(self.neurons, pitch.value)

    def construction_fixups(self) -> int:
        return int(lib().synq_sim_construction_fixups(self.h))

    def device_time(self):
        """(device seconds of run/step, seconds inside the step kernels)"""
        out = np.zeros(2, np.float64)
        check(lib().synq_sim_device_time(self.h, _p(out)))
        return float(out[0]), float(out[1])

    def phase_cycles(self) -> dict:
        out = np.zeros(15, np.float64)
        tiles = C.c_uint32()
        check(lib().synq_sim_phase_cycles(self.h, _p(out), C.byref(tiles)))
        names = ["update", "publish", "poll", "gather", "deliver"]
        d = {"mean": dict(zip(names, (round(float(x)) for x in out[:5]))),
             "pacing": dict(zip(names, (round(float(x)) for x in out[5:10]))),
             "update_detail": {"own_work": round(float(out[10])), "to_first_barrier": round(float(out[11]))},
             "producer": dict(zip(["poll", "ids", "splits", "rebase", "issue"],
                                  (round(float(x)) for x in out[10:15]))),
             "pipeline": dict(zip(["deliver_wait", "passes", "update_bar1", "update_scan", "prefix_chunklist"],
                                  (round(float(x), 2) for x in out[10:15]))), "tiles": tiles.value}
        return d

    # ---- multi-GPU shard exchange
    def shard_range(self):
        """((receiving lo, hi), (update-only lo, hi)) neuron ids of this shard."""
        out = (C.c_uint32 * 4)()
        check(lib().synq_sim_shard_range(self.h, out))
        return (out[0], out[1]), (out[2], out[3])

    def shard_capacity(self) -> int:
        return int(lib().synq_sim_shard_capacity(self.h))

    def shard_export(self, buf=None, device_ptr: int | None = None, capacity: int | None = None):
        """Pack the last run's frames.  With device_ptr the words go to device
        memory (e.g. a torch tensor's data_ptr()); otherwise into a numpy
        array (returned)."""
        words = C.c_uint64()
        if device_ptr is not None:
            check(lib().synq_sim_shard_export(self.h, C.c_void_p(device_ptr), capacity, 1, C.byref(words)))
            return int(words.value)
        cap = self.shard_capacity()
        out = np.empty(max(cap, 1), np.uint32)
        check(lib().synq_sim_shard_export(self.h, _p(out), cap, 0, C.byref(words)))
        return out[: words.value].copy()

    def shard_import(self, words, from_rank: int, device_ptr: int | None = None, nwords: int | None = None):
        if device_ptr is not None:
            check(lib().synq_sim_shard_import(self.h, C.c_void_p(device_ptr), nwords, from_rank, 1))
        else:
            w = np.ascontiguousarray(words, np.uint32)
            check(lib().synq_sim_shard_import(self.h, _p(w), len(w), from_rank, 0))

    def set_record(self, on: bool):
        check(lib().synq_sim_set_record(self.h, int(on)))

    # ---- bitmask frame exchange (the in-engine NCCL path does this itself)
    def shard_bits_words(self) -> int:
        return int(lib().synq_sim_shard_bits_words(self.h))

    def shard_export_bits(self, device_ptr: int):
        check(lib().synq_sim_shard_export_bits(self.h, C.c_void_p(device_ptr)))

    def shard_import_bits(self, device_ptr: int):
        check(lib().synq_sim_shard_import_bits(self.h, C.c_void_p(device_ptr)))

    # ---- NVLink peer exchange (Opts(shard_peer=True))
    def peer_endpoint(self) -> "PeerEndpoint":
        e = PeerEndpoint()
        check(lib().synq_sim_peer_endpoint(self.h, C.byref(e)))
        return e

    def peer_connect(self, endpoints):
        """endpoints[q]: every rank's peer_endpoint() (same process)."""
        arr = (PeerEndpoint * len(endpoints))(*endpoints)
        check(lib().synq_sim_peer_connect(self.h, arr, len(endpoints)))

    def peer_ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        check(lib().synq_sim_peer_ipc_handle(self.h, buf))
        return buf.raw

    def peer_connect_ipc(self, handles):
        """handles[q]: every rank's peer_ipc_handle() (other processes)."""
        blob = b"".join(bytes(h) for h in handles)
        check(lib().synq_sim_peer_connect_ipc(self.h, C.create_string_buffer(blob, len(blob)), len(handles)))

    def kernel_launches(self) -> int:
        return int(lib().synq_sim_kernel_launches(self.h))

    def transfer_bytes(self):
        out = np.zeros(2, np.uint64)
        check(lib().synq_sim_transfer_bytes(self.h, _p(out)))
        return int(out[0]), int(out[1])


PEER_HANDLE_BYTES = 136  # synq.h SYNQ_PEER_HANDLE_BYTES


class PeerEndpoint(C.Structure):
    """synq_peer_endpoint: a shard's queue ring and frame words."""
    _fields_ = [("queue", C.c_void_p), ("finfo", C.c_void_p), ("publishers", C.c_uint32),
                ("reserved", C.c_uint32)]


def _prefer_torch_nccl():
    """libsynq opens NCCL on first use and reuses a libnccl.so.2 already in the
    process: load torch's (newer) one first when torch is installed, so both
    share it."""
    try:
        import torch  # noqa: F401
    except Exception:
        pass


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id for synq_opts_shard_nccl (make it on one
    rank and broadcast it)."""
    _prefer_torch_nccl()
    buf = C.create_string_buffer(128)
    check(lib().synq_nccl_unique_id(buf))
    return buf.raw


def memory_estimate(model: str, neurons: int, synapses: int) -> dict:
    m = _Memory()
    check(lib().synq_memory_estimate(model.encode(), neurons, synapses, C.byref(m)))
    return m.as_dict()


def scaling_constant(model: str, neurons: int) -> float:
    r = C.c_double()
    check(lib().synq_scaling_constant(model.encode(), neurons, C.byref(r)))
    return r.value


def solve_neurons(model: str, synapses: int) -> int:
    r = C.c_uint32()
    check(lib().synq_solve_neurons(model.encode(), synapses, C.byref(r)))
    return r.value


def version() -> str:
    return lib().synq_version().decode()
