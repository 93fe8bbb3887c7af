"""CPU oracle for the synq hot path — TEST INFRASTRUCTURE ONLY.

Two checkers live here:

* ``liboracle.so`` — a plain-C restatement (oracle/synq_oracle.c) of the
  reference algorithm: RNG streams, plan_jobs/expand_jobs construction and the
  deterministic step loop of the four benchmark models.
* ``_ref/libsynq_ref.so`` and ``_ref/synq_golden`` — the UNMODIFIED reference
  compiled from /root/reference/proj by oracle/Makefile.  These travel to the
  GPU box inside the repo snapshot, so the reference itself is available there
  as a checker and as the CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product library (libsynq.so.1) never links
or calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import tempfile
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
GOLDEN_TOOL = os.path.join(REF_DIR, "synq_golden")
REF_LIB = os.path.join(REF_DIR, "libsynq_ref.so")

MODELS = {"pingpong": 0, "vogels": 1, "brunel": 2, "brunel+": 3}


def build() -> None:
    """(Re)build the oracle artefacts (C restatement always; the reference
    build only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _XS(C.Structure):
    _fields_ = [("x", C.c_uint32), ("y", C.c_uint32), ("z", C.c_uint32), ("w", C.c_uint32)]


class SoDesc(C.Structure):
    _fields_ = [
        ("npops", C.c_uint32),
        ("pop", C.c_uint32 * 16),
        ("nconn", C.c_uint32),
        ("csrc", C.c_uint32 * 64),
        ("cdst", C.c_uint32 * 64),
        ("cp", C.c_double * 64),
        ("dt", C.c_double),
        ("delay", C.c_uint32),
    ]

    @staticmethod
    def make(pops, conns, dt=1.0, delay=1) -> "SoDesc":
        d = SoDesc()
        d.npops = len(pops)
        for i, p in enumerate(pops):
            d.pop[i] = p
        d.nconn = len(conns)
        for i, (s, t, p) in enumerate(conns):
            d.csrc[i], d.cdst[i], d.cp[i] = s, t, p
        d.dt = dt
        d.delay = delay
        return d


class _Job(C.Structure):
    _fields_ = [("n", C.c_uint32), ("a", C.c_uint32), ("b", C.c_uint32), ("pad", C.c_uint32),
                ("o", C.c_uint64)]


class _Graph(C.Structure):
    _fields_ = [
        ("neurons", C.c_uint32), ("deg_max", C.c_uint32), ("pitch", C.c_uint32),
        ("edges", C.c_uint64), ("njobs", C.c_uint64), ("jobs", C.POINTER(_Job)),
        ("degree", C.POINTER(C.c_uint32)), ("cells", C.POINTER(C.c_uint32)),
    ]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        u32, u64, i64, dbl, vp = C.c_uint32, C.c_uint64, C.c_int64, C.c_double, C.c_void_p
        L.so_derive_seed.restype = u64
        L.so_derive_seed.argtypes = [u64, u64]
        L.so_xs_fill.argtypes = [u64, vp, C.c_size_t]
        L.so_binomial_fill.argtypes = [u64, u32, dbl, vp, C.c_size_t]
        L.so_xs_seed.argtypes = [C.POINTER(_XS), u64]
        L.so_sorted_random.argtypes = [u32, u32, u32, C.POINTER(_XS), vp]
        L.so_sorted_random_replay.argtypes = [u32, u32, u32, vp, vp, vp]
        L.so_build_graph.restype = C.POINTER(_Graph)
        L.so_build_graph.argtypes = [C.POINTER(SoDesc), u64, u32]
        L.so_plan_graph.restype = C.POINTER(_Graph)
        L.so_plan_graph.argtypes = [C.POINTER(SoDesc), u64, u32]
        L.so_graph_free.argtypes = [C.POINTER(_Graph)]
        L.so_sim_new.restype = vp
        L.so_sim_new.argtypes = [C.c_int, u32, u64, u32, dbl, u32]
        L.so_sim_new_desc.restype = vp
        L.so_sim_new_desc.argtypes = [C.c_int, C.POINTER(SoDesc), u64, u32]
        L.so_sim_free.argtypes = [vp]
        L.so_sim_run.argtypes = [vp, i64]
        L.so_sim_flush.argtypes = [vp]
        L.so_sim_graph.restype = C.POINTER(_Graph)
        L.so_sim_graph.argtypes = [vp]
        for fn in ("so_sim_neurons", "so_sim_delay", "so_sim_history"):
            getattr(L, fn).restype = u32
            getattr(L, fn).argtypes = [vp]
        L.so_sim_now.restype = i64
        L.so_sim_now.argtypes = [vp]
        L.so_sim_counters.argtypes = [vp, vp]
        L.so_sim_field.argtypes = [vp, C.c_int, vp]
        L.so_sim_syn_field.argtypes = [vp, C.c_int, vp]
        L.so_sim_ages.argtypes = [vp, vp]
        L.so_sim_frame_words.restype = u64
        L.so_sim_frame_words.argtypes = [vp]
        L.so_sim_frames.argtypes = [vp, vp]
        L.so_sim_constants.argtypes = [vp, vp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- RNG
def derive_seed(master: int, index: int) -> int:
    return int(lib().so_derive_seed(master, index))


def xorshift(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    lib().so_xs_fill(seed, _ptr(out), n)
    return out


def binomial(seed: int, m: int, p: float, n: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    lib().so_binomial_fill(seed, m, p, _ptr(out), n)
    return out


def sorted_random(n: int, a: int, b: int, seed: int) -> np.ndarray:
    r = _XS()
    lib().so_xs_seed(C.byref(r), seed)
    out = np.empty(max(n, 1), np.uint32)
    if lib().so_sorted_random(n, a, b, C.byref(r), _ptr(out)) != 0:
        raise ValueError("sorted_random precondition violated")
    return out[:n]


def sorted_random_replay(n: int, a: int, b: int, draws):
    d = np.ascontiguousarray(draws, np.float64)
    out = np.empty(max(n, 1), np.uint32)
    trace = np.empty(4 * (n + 2), np.float64)
    if lib().so_sorted_random_replay(n, a, b, _ptr(d), _ptr(out), _ptr(trace)) != 0:
        raise ValueError("sorted_random precondition violated")
    return out[:n], trace.reshape(4, n + 2)


# --------------------------------------------------------- construction
@dataclass
class Graph:
    neurons: int
    deg_max: int
    pitch: int
    edges: int
    degree: np.ndarray
    cells: np.ndarray | None
    jobs: np.ndarray  # (njobs, 4) [n, a, b, o]


def _graph_from(gp, with_cells=True) -> Graph:
    g = gp.contents
    n = g.neurons
    deg = np.ctypeslib.as_array(g.degree, shape=(max(n, 1),))[:n].copy()
    cells = None
    if with_cells and g.cells:
        cells = np.ctypeslib.as_array(g.cells, shape=(max(n * g.pitch, 1),))[: n * g.pitch]
        cells = cells.reshape(n, g.pitch).copy() if g.pitch else np.zeros((n, 0), np.uint32)
    jobs = np.zeros((g.njobs, 4), np.uint64)
    for i in range(g.njobs):
        j = g.jobs[i]
        jobs[i] = (j.n, j.a, j.b, j.o)
    return Graph(n, g.deg_max, g.pitch, g.edges, deg, cells, jobs)


def build_graph(desc: SoDesc, seed: int, pitch_align: int = 32) -> Graph:
    gp = lib().so_build_graph(C.byref(desc), seed, pitch_align)
    try:
        return _graph_from(gp)
    finally:
        lib().so_graph_free(gp)


def plan_graph(desc: SoDesc, seed: int, pitch_align: int = 32) -> Graph:
    gp = lib().so_plan_graph(C.byref(desc), seed, pitch_align)
    try:
        return _graph_from(gp, with_cells=False)
    finally:
        lib().so_graph_free(gp)


# ----------------------------------------------------------- simulation
@dataclass
class RunResult:
    counts: np.ndarray  # per-step spike count
    ids: np.ndarray  # concatenated frames
    counters: dict
    fields: list = field(default_factory=list)  # raw u32 views of the neuron fields
    syn: list | None = None
    ages: np.ndarray | None = None

    def frame(self, t: int) -> np.ndarray:
        off = int(self.counts[:t].sum())
        return self.ids[off: off + int(self.counts[t])]


def split_frames(words: np.ndarray):
    counts, ids, i = [], [], 0
    n = len(words)
    while i < n:
        c = int(words[i])
        counts.append(c)
        ids.append(words[i + 1: i + 1 + c])
        i += 1 + c
    return (np.asarray(counts, np.uint32),
            np.concatenate(ids).astype(np.uint32) if ids else np.zeros(0, np.uint32))


class Sim:
    """Deterministic CPU restatement of network<M> (engine.hpp:188-436)."""

    def __init__(self, model: str, neurons: int = 0, seed: int = 1, history: int = 0,
                 dt: float = 0.0, delay: int = 0, desc: SoDesc | None = None):
        self.model = model
        if desc is not None:
            self.h = lib().so_sim_new_desc(MODELS[model], C.byref(desc), seed, history)
        else:
            self.h = lib().so_sim_new(MODELS[model], neurons, seed, history, dt, delay)
        if not self.h:
            raise ValueError("oracle: cannot build model")

    def __del__(self):
        if getattr(self, "h", None):
            lib().so_sim_free(self.h)
            self.h = None

    @property
    def n(self):
        return int(lib().so_sim_neurons(self.h))

    @property
    def delay(self):
        return int(lib().so_sim_delay(self.h))

    @property
    def history(self):
        return int(lib().so_sim_history(self.h))

    def now(self):
        return int(lib().so_sim_now(self.h))

    def run(self, steps: int):
        lib().so_sim_run(self.h, steps)

    def flush(self):
        lib().so_sim_flush(self.h)

    def graph(self) -> Graph:
        return _graph_from(lib().so_sim_graph(self.h))

    def counters(self) -> dict:
        c = np.zeros(6, np.uint64)
        lib().so_sim_counters(self.h, _ptr(c))
        keys = ["steps", "spikes", "deliveries", "synapse_updates", "expiry_batches",
                "frames_consumed"]
        return {k: int(v) for k, v in zip(keys, c)}

    def field(self, f: int) -> np.ndarray:
        out = np.empty(self.n, np.uint32)
        lib().so_sim_field(self.h, f, _ptr(out))
        return out

    def field_f32(self, f: int) -> np.ndarray:
        return self.field(f).view(np.float32)

    def syn_field(self, f: int) -> np.ndarray:
        g = self.graph()
        out = np.empty(self.n * g.deg_max, np.float32)
        lib().so_sim_syn_field(self.h, f, _ptr(out))
        return out

    def ages(self) -> np.ndarray:
        out = np.empty(self.n, np.uint32)
        lib().so_sim_ages(self.h, _ptr(out))
        return out

    def frames(self):
        n = int(lib().so_sim_frame_words(self.h))
        w = np.empty(max(n, 1), np.uint32)
        lib().so_sim_frames(self.h, _ptr(w))
        return split_frames(w[:n])

    def constants(self) -> np.ndarray:
        out = np.zeros(6, np.float64)
        lib().so_sim_constants(self.h, _ptr(out))
        return out


# ------------------------------------------------- the reference itself
def have_reference() -> bool:
    return os.path.exists(GOLDEN_TOOL) and os.path.exists(REF_LIB)


def golden(*args, out_bytes=True) -> bytes:
    """Run the reference-linked dumper (oracle/_ref/synq_golden)."""
    r = subprocess.run([GOLDEN_TOOL, *map(str, args)], check=True, capture_output=True)
    return r.stdout


def reference_run(model: str, neurons: int, seed: int, steps: int, history: int = 0,
                  dt: float = 0.0, delay: int = 0, desc_path: str | None = None) -> RunResult:
    """Deterministic run of the UNMODIFIED reference network<M> via synq_golden."""
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "run")
        if desc_path:
            golden("run_desc", model, desc_path, seed, steps, out)
        else:
            golden("run", model, neurons, seed, steps, out, history, dt, delay)
        words = np.fromfile(out + ".frames", np.uint32)
        counts, ids = split_frames(words)
        counters = {}
        with open(out + ".counters") as fh:
            for line in fh:
                k, v = line.strip().split("=")
                counters[k] = int(v)
        n = counters["neurons"]
        st = np.fromfile(out + ".state", np.uint8)
        fields = []
        if model == "pingpong":
            fields = [st[:n].astype(np.uint32)]
        else:
            w = st.view(np.uint32)
            fields = [w[i * n:(i + 1) * n].copy() for i in range(3)]
        syn = ages = None
        if os.path.exists(out + ".syn"):
            s = np.fromfile(out + ".syn", np.float32)
            cap = len(s) // 3
            syn = [s[i * cap:(i + 1) * cap].copy() for i in range(3)]
            ages = np.fromfile(out + ".ages", np.uint32)
            with open(out + ".preflush") as fh:
                for line in fh:
                    k, v = line.strip().split("=")
                    counters["preflush_" + k] = int(v)
        return RunResult(counts, ids, counters, fields, syn, ages)


def reference_adjacency(model: str, neurons: int, seed: int):
    """(neurons, pitch, deg_max, cells[neurons, pitch]) from the reference build."""
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "adj.bin")
        golden("adj", model, neurons, seed, p)
        raw = np.fromfile(p, np.uint32)
    n, pitch, deg_max, sent = (int(x) for x in raw[:4])
    assert sent == 0xFFFFFFFF
    return n, pitch, deg_max, raw[4:].reshape(n, pitch) if pitch else np.zeros((n, 0), np.uint32)


# --------------------------------------- the reference C ABI (CPU baseline)
class RefLib:
    """ctypes binding of the reference's own C ABI (oracle/_ref/libsynq_ref.so)."""

    def __init__(self, path: str = REF_LIB):
        L = C.CDLL(path)
        vp, u32, u64, i64, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int64, C.c_double
        L.synq_opts_new.restype = vp
        L.synq_opts_free.argtypes = [vp]
        for fn, t in (("synq_opts_seed", u64), ("synq_opts_threads", u32),
                      ("synq_opts_deterministic", C.c_int), ("synq_opts_record", C.c_int),
                      ("synq_opts_dt", dbl), ("synq_opts_delay", u32)):
            getattr(L, fn).argtypes = [vp, t]
        L.synq_opts_param.argtypes = [vp, C.c_char_p, dbl]
        L.synq_sim_new.argtypes = [C.c_char_p, u32, vp, C.POINTER(vp)]
        L.synq_sim_new_for_synapses.argtypes = [C.c_char_p, u64, vp, C.POINTER(vp)]
        L.synq_sim_free.argtypes = [vp]
        L.synq_sim_run.argtypes = [vp, i64]
        L.synq_sim_step.argtypes = [vp]
        L.synq_sim_flush.argtypes = [vp]
        L.synq_sim_neurons.argtypes = [vp]
        L.synq_sim_neurons.restype = u32
        L.synq_sim_synapses.argtypes = [vp]
        L.synq_sim_synapses.restype = u64
        L.synq_sim_seconds.argtypes = [vp, C.c_int]
        L.synq_sim_seconds.restype = dbl
        L.synq_sim_spike_count.argtypes = [vp, C.POINTER(u64)]
        L.synq_sim_firing_rate.argtypes = [vp, C.POINTER(dbl)]
        L.synq_sim_write_stats.argtypes = [vp, C.c_char_p]
        L.synq_sim_write_raster.argtypes = [vp, C.c_char_p]
        L.synq_last_error.restype = C.c_char_p
        self.L = L
