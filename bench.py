#!/usr/bin/env python3
"""Headline benchmark: Brunel balanced network at ~1e9 synapses on B200.

Metric (BASELINE.json): synaptic events/sec and wall time per 1 s of
biological time.  One bench "step" = 1 s of biological time = 10,000
simulation timesteps (dt = 0.1 ms) of synq::network<brunel_model>, run through
the C ABI (libsynq.so.1).  Events = the engine's delivery counter, exactly the
reference's `deliveries` (proj/include/synq/engine.hpp:408).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl synq|reference]

* value: events/s over all ranks, device-timed (CUDA events recorded by the
  library on its own stream around every run; max over ranks).
* e2e: the same workload through the C ABI with spike recording on and the
  raster copied into host buffers each step (device->host bytes counted).
* roofline: the persistent step kernel (update + receive, warp-specialised) —
  algorithmic bytes per launch / kernel time vs the measured HBM copy bandwidth.
* cpu_baseline: the UNMODIFIED reference (oracle/_ref/libsynq_ref.so, built
  from /root/reference by oracle/Makefile) on a bounded sample of the same
  network, on this host's cores.
* --impl reference: the reference's own CPU simulator on this host: deterministic
  (1 thread) and parallel (all threads) modes, the faster reported.
Inputs are larger than L2 (4.2 GB adjacency vs 126 MB L2), so no L2 flush.
Under torchrun (N > 1) the ranks shard ONE network of N x 1e9 synapses
(target-partitioned, spike frames allgathered over NCCL every delay-1 steps;
weak scaling); `--replicas` runs independent 1e9-synapse replicas instead.
Rank 0 prints the JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "synaptic events/sec & wall time per 1 s bio time (Brunel, 1/2/4/8 B200)"
UNIT = "events/s"
BIO_STEPS = 10000  # 1 s of biological time at dt = 0.1 ms


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="synq", choices=["synq", "reference"])
    ap.add_argument("--synapses", type=float, default=1e9)
    ap.add_argument("--workload", default="weak", choices=["weak", "b8"],
                    help="N>1: 'weak' = one network of N x --synapses (weak scaling); 'b8' = BASELINE "
                         "config 5, one Brunel network of 1.2e10 synapses over the N GPUs (strong scaling)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample-steps", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary BASELINE configs (Vogels 4000, Brunel+ 1e8) reported beside the headline")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent 1e9-synapse replicas instead of one sharded network")
    ap.add_argument("--exchange", default="bitmask", choices=["bitmask", "peer"],
                    help="N>1 with --backend nccl: bitmask = in-engine ncclAllGather of spike bitmasks every "
                         "delay-1 steps; peer = NVLink peer exchange (the step kernel stores each frame into every "
                         "peer's ring; IPC handles allgathered over NCCL; one launch per 1000 steps)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 frame exchange (gloo: host buffers, e.g. several ranks on one GPU)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def ensure_world(args) -> None:
    """--gpus N is the world size.  Without torchrun env vars and N > 1 this
    process re-launches itself under torch.distributed.run (one rank per
    GPU, rendezvous on 127.0.0.1); under torchrun WORLD_SIZE must equal N."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    if args.impl == "synq" and not (args.backend == "gloo"):
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have} "
                             "(one rank per GPU; NCCL refuses two ranks on one device)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.out, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        self.out.flush()
        self.out.seek(0)
        rows = [r.split(",") for r in self.out.read().strip().splitlines() if r.strip()]
        rows = [[x.strip() for x in r] for r in rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        busy = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        mhz = [int(r[1]) for r in busy if r[1].isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in busy:
            for k, name in enumerate(names):
                if r[3 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(mhz) if mhz else None,
                "sm_max_mhz": int(rows[0][2]) if rows[0][2].isdigit() else None,
                "reasons": sorted(reasons), "samples": len(busy)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic_per_step():
    """dram bytes per simulation timestep of the persistent kernel, from the
    committed ncu --set full capture summary (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            s = json.load(fh)
        return float(s["dram_bytes_per_timestep"]), s.get("source")
    except Exception:
        return None, None


# ------------------------------------------------------------ CPU baseline
def cpu_reference_sample(synapses: float, seed: int, sample_steps: int, threads: int,
                         deterministic: bool, warm_steps: int = 200):
    """Run the unmodified reference on a bounded sample; returns dict."""
    import oracle

    ref = oracle.RefLib()
    L = ref.L
    opts = L.synq_opts_new()
    L.synq_opts_seed(opts, seed)
    L.synq_opts_deterministic(opts, 1 if deterministic else 0)
    L.synq_opts_threads(opts, threads)
    sim = C.c_void_p()
    st = L.synq_sim_new_for_synapses(b"brunel", int(synapses), opts, C.byref(sim))
    if st != 0:
        raise RuntimeError("reference: " + L.synq_last_error().decode())
    L.synq_sim_run(sim, warm_steps)
    t_sim0 = L.synq_sim_seconds(sim, 3)
    d0 = _ref_deliveries(L, sim)
    L.synq_sim_run(sim, sample_steps)
    t_sim = L.synq_sim_seconds(sim, 3) - t_sim0
    d = _ref_deliveries(L, sim) - d0
    out = {"events": d, "sim_s": t_sim, "steps": sample_steps,
           "construct_s": L.synq_sim_seconds(sim, 0), "neurons": int(L.synq_sim_neurons(sim)),
           "synapses": int(L.synq_sim_synapses(sim))}
    L.synq_sim_free(sim)
    L.synq_opts_free(opts)
    return out


def _ref_deliveries(L, sim) -> int:
    with tempfile.NamedTemporaryFile("r", suffix=".txt") as fh:
        L.synq_sim_write_stats(sim, fh.name.encode())
        for line in open(fh.name):
            if line.startswith("deliveries="):
                return int(line.split("=")[1])
    raise RuntimeError("reference stats lack deliveries")


def _reference_mode(L, args, sample, threads, deterministic):
    """Build the reference Brunel network and time K samples of `sample`
    timesteps after W warm-up samples; returns (events, seconds, sim)."""
    opts = L.synq_opts_new()
    L.synq_opts_seed(opts, args.seed)
    L.synq_opts_threads(opts, threads)
    L.synq_opts_deterministic(opts, 1 if deterministic else 0)
    sim = C.c_void_p()
    if L.synq_sim_new_for_synapses(b"brunel", int(args.synapses), opts, C.byref(sim)) != 0:
        raise RuntimeError(L.synq_last_error().decode())
    L.synq_opts_free(opts)
    for _ in range(args.warmup):
        L.synq_sim_run(sim, sample)
    t0 = L.synq_sim_seconds(sim, 3)
    d0 = _ref_deliveries(L, sim)
    for _ in range(args.steps):
        L.synq_sim_run(sim, sample)
    secs = L.synq_sim_seconds(sim, 3) - t0
    events = _ref_deliveries(L, sim) - d0
    return events, secs, sim


def run_reference_arm(args):
    """The reference's own CPU simulator on this host: both of its modes on
    the same Brunel network — deterministic (1 thread, its fastest for this
    model) and parallel (all host threads) — reporting the faster."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    try:
        import oracle

        if not oracle.have_reference():
            raise FileNotFoundError("oracle/_ref not built")
        ref = oracle.RefLib()
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"reference build missing: {e}"}))
        return 0
    L = ref.L
    threads = os.cpu_count() or 1
    sample = max(100, int(os.environ.get("SYNQ_REF_SAMPLE_STEPS", 500)))
    modes = {}
    info = {}
    for name, thr, det in (("deterministic", 1, True), ("parallel", threads, False)):
        try:
            ev, secs, sim = _reference_mode(L, args, sample, thr, det)
            modes[name] = (ev / secs, thr, ev, secs)
            info = {"synapses": int(L.synq_sim_synapses(sim)), "neurons": int(L.synq_sim_neurons(sim))}
            L.synq_sim_free(sim)
        except Exception as e:  # reported, the other mode still counts
            modes[name] = (0.0, thr, 0, 0.0)
            info.setdefault("errors", []).append(f"{name}: {e}")
    best = max(modes, key=lambda k: modes[k][0])
    value, cores, events, secs = modes[best]
    if value <= 0:
        print(json.dumps({"impl": "reference", "unavailable": "reference runs failed: %s" % info}))
        return 0
    bio_per_step = sample / BIO_STEPS
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1000.0,
        "wall_s_per_bio_s": secs / (args.steps * bio_per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference builder, seed %d)" % args.seed,
        "config": {"workload": "brunel_1e9" if args.synapses == 1e9 else "brunel", **info,
                   "bio_ms_per_step": sample * 0.1, "mode": f"reference {best}, {cores} thread(s)",
                   "modes_events_per_s": {k: v[0] for k, v in modes.items()}},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} x {sample} timesteps of Brunel 1e9 after "
                                   f"{args.warmup} warm-up samples; faster of deterministic (1 thread) "
                                   f"and parallel ({threads} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------ B200 arm
def secondary_configs(synq):
    """BASELINE configs 1 and 3 measured in the same run (device-timed, after
    warm-up; not the headline): Vogels-Abbott 4000 over one biological second
    and Brunel+ 1e8 (STDP) over 0.2 s.  Parity of both: tests/test_gpu_parity*.py."""
    out = {}
    try:
        sim = synq.Sim("vogels", 4000, synq.Opts(seed=1, deterministic=True))
        sim.run(2000)
        d0, _ = sim.device_time()
        c0 = sim.counters()["deliveries"]
        sim.run(BIO_STEPS)
        d1, _ = sim.device_time()
        ev = sim.counters()["deliveries"] - c0
        out["vogels_4000"] = {"ms_per_bio_s": (d1 - d0) * 1e3, "events_per_s": ev / (d1 - d0),
                              "engine": sim.engine, "exact": sim.exact}
        sim.close()
    except Exception as e:  # reported, never fatal
        out["vogels_4000"] = {"error": str(e)}
    try:
        sim = synq.Sim("brunel+", opts=synq.Opts(seed=1, deterministic=True), synapses=int(1e8))
        sim.run(500)
        d0, _ = sim.device_time()
        c0 = sim.counters()
        steps = 2000
        sim.run(steps)
        d1, _ = sim.device_time()
        c1 = sim.counters()
        out["brunel_plus_1e8"] = {"ms_per_bio_s": (d1 - d0) / steps * BIO_STEPS * 1e3,
                                  "events_per_s": (c1["deliveries"] - c0["deliveries"]) / (d1 - d0),
                                  "synapse_updates_per_s": (c1["synapse_updates"] - c0["synapse_updates"]) / (d1 - d0),
                                  "synapses": sim.synapses, "engine": sim.engine, "exact": sim.exact,
                                  "sample_steps": steps}
        sim.close()
    except Exception as e:
        out["brunel_plus_1e8"] = {"error": str(e)}
    return out


def main():
    args = parse()
    ensure_world(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    rank, world, local = dist_env()
    torch = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        dist.init_process_group(args.backend)
        if not args.replicas:
            return run_sharded(args, rank, world, local)
    os.environ.setdefault("CUDA_DEVICE_ORDER", "PCI_BUS_ID")
    import paper_1912_07423_b200 as synq

    # the CUDA runtime picks the device from the current context: bind it
    if world > 1:
        torch.cuda.synchronize()

    t_setup = time.perf_counter()
    opts = synq.Opts(seed=args.seed + rank, deterministic=True)
    sim = synq.Sim("brunel", opts=opts, synapses=int(args.synapses))
    setup_s = time.perf_counter() - t_setup
    assert sim.persistent, "brunel must run on the persistent engine"

    sim.run(args.warmup * BIO_STEPS)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    barrier()
    dev0, ker0 = sim.device_time()
    c0 = sim.counters()
    l0 = sim.kernel_launches()
    with ClockSampler(local) as clocks:
        sim.run(args.steps * BIO_STEPS)
    dev1, ker1 = sim.device_time()
    c1 = sim.counters()
    l1 = sim.kernel_launches()
    barrier()
    secs = dev1 - dev0
    kern = ker1 - ker0
    events = c1["deliveries"] - c0["deliveries"]
    spikes = c1["spikes"] - c0["spikes"]

    # e2e: spike recording on, raster copied to host buffers every step
    import numpy as np

    sim.set_record(True)
    # one untimed recorded second first: the host raster grows to its working
    # size (first-touch page faults), later seconds reuse the pages
    sim.run(BIO_STEPS)
    st_w, ids_w = sim.raster()
    bufs = (np.empty(2 * len(st_w) + 1024, np.int64), np.empty(2 * len(ids_w) + 1024, np.uint32))
    bufs[0].fill(0)  # touch the host pages once, outside the timed region
    bufs[1].fill(0)
    sim.set_record(True)
    h0, d0b = sim.transfer_bytes()
    ce0 = sim.counters()["deliveries"]
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        sim.run(BIO_STEPS)
        steps_arr, ids_arr = sim.raster(out=bufs)
        sim.set_record(True)  # clears the host raster, keeps recording
    e2e_s = time.perf_counter() - t0
    h1, d1b = sim.transfer_bytes()
    e2e_events = sim.counters()["deliveries"] - ce0
    raster_bytes_host = int(steps_arr.nbytes + ids_arr.nbytes)
    sim.set_record(False)

    if world > 1:
        import torch
        import torch.distributed as dist

        t = torch.tensor([secs, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs, e2e_s = float(t[0]), float(t[1])
        e = torch.tensor([events, e2e_events, spikes], dtype=torch.float64, device="cuda")
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        events, e2e_events, spikes = float(e[0]), float(e[1]), float(e[2])

    if rank != 0:
        return 0

    n = sim.neurons
    n_exc = int(round(0.4 * n))
    n_rec = n_exc + int(round(0.1 * n))
    n_stim = n - n_rec
    timesteps = args.steps * BIO_STEPS
    launches = l1 - l0
    # algorithmic bytes of the fused step kernel: 4 B per
    # delivery (target id), 24 B per LIF neuron-step, 32 B per Poisson
    # neuron-step (16 B stream read + write), 4 B per queued spike
    alg = 4.0 * events + (24.0 * n_rec + 32.0 * n_stim) * timesteps * world + 4.0 * spikes
    peak, peak_src = measured_peaks()
    achieved = alg / kern / 1e9 / world if kern > 0 else 0.0
    traffic_step, traffic_src = ncu_traffic_per_step()
    per_launch_steps = timesteps / max(1, launches)
    line = {
        "metric": METRIC,
        "value": events / secs,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1000.0,
        "wall_s_per_bio_s": secs / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic: Brunel network built on device from seed %d (reference RNG streams)" % args.seed,
        "config": {
            "workload": "brunel_1e9" if args.synapses == 1e9 else "brunel",
            "synapses": sim.synapses, "neurons": n, "bio_s_per_step": 1.0, "dt_ms": 0.1,
            "delay_steps": sim.delay, "parallelism": f"dp{world} (replicas)" if world > 1 else "single",
            "engine": f"{sim.engine} (exact)", "tiles": None,
            "l2": "inputs larger than L2 (adjacency %.2f GB)" % (sim.synapses * 4 / 1e9),
            "setup_s": round(setup_s, 2), "construction_fixups": sim.construction_fixups(),
        },
        "gpu_launches": launches,
        "spikes_per_bio_s": spikes / args.steps / world,
        "events_per_bio_s": events / args.steps / world,
        "roofline": {
            "bound": "hbm",
            "kernel": ("synq::dev::k_pipeline<brunel_model, UW, NPT, bitmap> (warp-specialised update + receive)"
                       if sim.engine == "pipelined-bitmap" else f"synq::dev step kernel ({sim.engine})"),
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": (traffic_step * per_launch_steps) if traffic_step else None,
            "traffic_source": traffic_src,
            "alg_bytes_per_launch": alg / world / max(1, launches),
            "alg_bytes_definition": "SURVEY.md 8(d): 4 B per delivery (u32 target id) + 24 B per LIF and "
                                    "32 B per Poisson neuron-step + 4 B per spike; the bitmap receive "
                                    "format moves ~1.3 B per delivery of it",
            "receive_only_GBps": 4.0 * events / world / kern / 1e9 if kern > 0 else 0.0,
            "kernel_s": kern,
            "peak_source": peak_src,
        },
        "e2e": {
            "value": e2e_events / e2e_s,
            "unit": UNIT,
            "h2d_bytes_per_step": (h1 - h0) / args.e2e_steps,
            "d2h_bytes_per_step": (d1b - d0b) / args.e2e_steps,
            "how": "C ABI synq_sim_run(10000) with recording (the kernel writes the ordered spike "
                   "log into pinned host memory, batches pipelined) + synq_sim_raster_copy into host "
                   "numpy buffers per step, wall clock, after one untimed recorded second",
            "raster_bytes_last_step": raster_bytes_host,
            "inputs": "no per-step host inputs: the network is built on the device from the seed "
                      "(h2d counts only control words); the per-step output is the spike raster",
        },
        "clocks": clocks.summary(),
    }
    # the CPU reference sample runs after every GPU timed region (it builds a
    # 4.2 GB network and would share host memory bandwidth with the e2e leg)
    sim.close()
    if rank == 0 and world == 1 and not args.no_secondary:
        line["secondary"] = secondary_configs(synq)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_result = {}
        try:
            cpu_result.update(cpu_reference_sample(args.synapses, args.seed, args.cpu_sample_steps, 1, True))
        except Exception as e:  # reported, never fatal
            cpu_result["error"] = str(e)
        if "error" in cpu_result:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": "failed: " + cpu_result["error"]}
        else:
            v = cpu_result["events"] / cpu_result["sim_s"]
            line["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"{cpu_result['steps']} timesteps (after 200 warm-up) of the same Brunel "
                          f"1e9 network ({cpu_result['synapses']} synapses), reference deterministic "
                          f"mode, 1 thread; construction {cpu_result['construct_s']:.1f} s",
                "wall_s_per_bio_s": cpu_result["sim_s"] * BIO_STEPS / cpu_result["steps"],
            }
    print(json.dumps(line))
    return 0


def run_sharded(args, rank, world, local):
    """N>1: ONE Brunel network of N x `--synapses` synapses,
    target-partitioned over the N GPUs (weak scaling: ~1e9 synapses and the
    same deliveries per step per GPU).  Every rank updates its own neurons and
    delivers every spike of the network onto its own targets; the spike
    frames are exchanged with an allgather (NCCL over NVLink, device buffers)
    every delay-1 steps, which is exact because a spike is due delay steps
    after it fires."""
    import torch
    import torch.distributed as dist

    import paper_1912_07423_b200 as synq
    from paper_1912_07423_b200 import shard

    b8 = args.workload == "b8"
    total = int(1.2e10) if b8 else int(args.synapses * world)
    in_engine = args.backend == "nccl"
    t_setup = time.perf_counter()
    if in_engine:
        # the engine allgathers the frames itself (ncclAllGather on its own
        # stream after every batch): one NCCL id, broadcast from rank 0
        uid = [synq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        peer = args.exchange == "peer"
        sim = synq.Sim("brunel", opts=synq.Opts(seed=args.seed, deterministic=True,
                                                shard_nccl=(rank, world, uid[0]), shard_peer=peer or None),
                       synapses=total)

        class _Engine:  # the ShardedSim surface bench needs
            record = False
            frames: list = []

            def run(self, steps):
                sim.run(steps)

            def close(self):
                sim.close()

        ss = _Engine()
    else:
        sim = synq.Sim("brunel", opts=synq.Opts(seed=args.seed, deterministic=True, shard=(rank, world)),
                       synapses=total)
        ss = shard.ShardedSim("brunel", 0, transport=shard.TorchTransport(), sim=sim)
    setup_s = time.perf_counter() - t_setup
    ss.run(args.warmup * BIO_STEPS)

    def sync_all():
        torch.cuda.synchronize()
        dist.barrier()

    sync_all()
    c0, l0 = sim.counters(), sim.kernel_launches()
    _, ker0 = sim.device_time()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    with ClockSampler(local % max(1, torch.cuda.device_count())) as clocks:
        ss.run(args.steps * BIO_STEPS)
        torch.cuda.synchronize()
    ev1.record()
    ev1.synchronize()
    secs = ev0.elapsed_time(ev1) * 1e-3
    c1, l1 = sim.counters(), sim.kernel_launches()
    _, ker1 = sim.device_time()
    sync_all()

    # e2e: the global spike raster on the host (in-engine: every rank's
    # engine logs the merged frames into pinned memory and rank 0 copies the
    # raster out through the C ABI; host path: frames merged from the gathered
    # words), one untimed second first
    if in_engine:
        if rank == 0:
            sim.set_record(True)
        ss.run(BIO_STEPS)
        if rank == 0:
            sim.raster()
            sim.set_record(True)
    else:
        ss.record = True
        ss.run(BIO_STEPS)
        ss.frames.clear()
    sync_all()
    e0 = sim.counters()["deliveries"]
    h0, d0b = sim.transfer_bytes()
    t0 = time.perf_counter()
    gathered = 0
    for _ in range(args.e2e_steps):
        ss.run(BIO_STEPS)
        if in_engine:
            if rank == 0:
                st, ids = sim.raster()
                gathered += int(st.nbytes + ids.nbytes)
                sim.set_record(True)
        else:
            gathered += sum(int(f.nbytes) for f in ss.frames)
            ss.frames.clear()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if in_engine and rank == 0:
        sim.set_record(False)
    e2e_ev = sim.counters()["deliveries"] - e0
    h1, d1b = sim.transfer_bytes()

    dev = torch.device("cuda") if args.backend == "nccl" else torch.device("cpu")
    mx = torch.tensor([secs, e2e_s, ker1 - ker0], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = torch.tensor([c1["deliveries"] - c0["deliveries"], c1["spikes"] - c0["spikes"], e2e_ev, l1 - l0,
                       (d1b - d0b) + gathered, sim.synapses], dtype=torch.float64, device=dev)
    # each rank stores only its own targets' sub-rows: the network's synapses
    # are the sum over ranks, the largest per-GPU share is reported beside it
    ms = torch.tensor([sim.synapses], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    max_syn = int(ms.item())
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    secs, e2e_s, kern = (float(x) for x in mx.tolist())
    events, spikes, e2e_events, launches, d2h, total_syn = (float(x) for x in sm.tolist())
    total_syn = int(total_syn)
    if rank != 0:
        ss.close()
        return 0
    n = sim.neurons
    n_exc = int(round(0.4 * n))
    n_rec = n_exc + int(round(0.1 * n))
    timesteps = args.steps * BIO_STEPS
    alg = 4.0 * events + (24.0 * n_rec + 32.0 * (n - n_rec)) * timesteps + 4.0 * spikes
    peak, peak_src = measured_peaks()
    achieved = alg / world / kern / 1e9 if kern > 0 else 0.0
    line = {
        "metric": METRIC, "value": events / secs, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1000.0, "wall_s_per_bio_s": secs / args.steps,
        "higher_is_better": True, "scaling": "strong" if b8 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: Brunel network built on device from seed %d (reference RNG streams)" % args.seed,
        "config": {"workload": "brunel_1.2e10_sharded (BASELINE config 5)" if b8 else f"brunel_{world}x1e9_sharded",
                   "synapses": total_syn, "neurons": n, "synapses_per_gpu_max": max_syn,
                   "bio_s_per_step": 1.0, "dt_ms": 0.1, "delay_steps": sim.delay,
                   "parallelism": f"shard{world} (target-partitioned; " + (
                       "NVLink peer exchange: the step kernel stores every frame into each peer's ring, "
                       "system-scope release; IPC handles over NCCL)" if in_engine and args.exchange == "peer" else
                       f"in-engine ncclAllGather of spike bitmasks every {sim.delay - 1} steps)" if in_engine else
                       f"host-driven {args.backend} allgather of spike frames every {sim.delay - 1} steps)"),
                   "engine": f"{sim.engine} shard (exact)", "setup_s": round(setup_s, 2),
                   "l2": "inputs larger than L2"},
        "gpu_launches": int(launches),
        "spikes_per_bio_s": spikes / args.steps, "events_per_bio_s": events / args.steps,
        "roofline": {"bound": "hbm", "kernel": f"synq::dev step kernel ({sim.engine}), per GPU",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel_s": kern, "peak_source": peak_src,
                     "alg_bytes_definition": "SURVEY.md 8(d), whole network / N GPUs"},
        "e2e": {"value": e2e_events / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0.0,
                "d2h_bytes_per_step": d2h / max(1, args.e2e_steps + 1) / world,
                "how": "sharded run; the global spike raster copied to host numpy buffers every bio-second"},
        "clocks": clocks.summary(),
    }
    print(json.dumps(line))
    ss.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
