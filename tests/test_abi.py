"""C-ABI boundary checks that need no GPU.

* libsynq.so.1 loads and exports every function include/synq/synq.h declares
  (the 37 reference entry points of proj/include/synq/synq.h + extensions);
* the host-only entry points behave like the reference's
  (proj/tests/test_capi.cpp:29-49, 154-166);
* without a CUDA device, simulation creation fails loudly with
  SYNQ_ERR_INTERNAL — there is no CPU fallback.
"""
import ctypes as C
import os
import subprocess

import pytest

import paper_1912_07423_b200 as synq

REFERENCE_ABI = [
    "synq_version", "synq_status_name", "synq_last_error", "synq_opts_new", "synq_opts_free",
    "synq_opts_seed", "synq_opts_threads", "synq_opts_deterministic", "synq_opts_dt",
    "synq_opts_delay", "synq_opts_record", "synq_opts_defaults_file", "synq_opts_param",
    "synq_sim_new", "synq_sim_new_for_synapses", "synq_sim_new_from_file", "synq_sim_free",
    "synq_sim_step", "synq_sim_run", "synq_sim_flush", "synq_sim_neurons", "synq_sim_synapses",
    "synq_sim_synapse_capacity", "synq_sim_now", "synq_sim_dt", "synq_sim_delay", "synq_sim_seed",
    "synq_sim_scaling", "synq_sim_firing_rate", "synq_sim_spike_count", "synq_sim_seconds",
    "synq_sim_write_raster", "synq_sim_write_stats", "synq_memory_estimate",
    "synq_sim_memory_actual", "synq_scaling_constant", "synq_solve_neurons",
]


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_reference_abi_has_37_entry_points():
    assert len(REFERENCE_ABI) == 37


def test_header_declares_reference_abi():
    declared = synq.declared_symbols()
    missing = [s for s in REFERENCE_ABI if s not in declared]
    assert not missing, missing


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", synq.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in synq.declared_symbols() if s not in exported]
    assert not missing, missing


def test_soname():
    out = subprocess.run(["readelf", "-d", synq.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "libsynq.so.1" in out


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", synq.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_status_strings():
    L = synq.lib()
    assert L.synq_version()
    assert L.synq_status_name(0) == b"ok"
    assert L.synq_status_name(2) == b"unknown model"


def test_unknown_model_is_reported():
    h = C.c_void_p()
    st = synq.lib().synq_sim_new(b"izhikevich", 100, None, C.byref(h))
    assert st == 2 and not h.value
    assert b"izhikevich" in synq.lib().synq_last_error()


def test_null_handles_rejected():
    L = synq.lib()
    assert L.synq_sim_step(None) == 1
    assert L.synq_opts_seed(None, 1) == 1
    assert L.synq_sim_neurons(None) == 0
    d = C.c_double()
    assert L.synq_sim_firing_rate(None, C.byref(d)) == 1


def test_memory_estimate_and_scaling():
    m = synq.memory_estimate("brunel+", 1000, 10000)
    assert m["neuron_total"] == 82.25 and m["synapse_total"] == 16.0
    assert m["total_bytes"] == pytest.approx(82.25 * 1000 + 16.0 * 10000)
    assert synq.memory_estimate("vogels", 1, 1)["neuron_total"] == 48.0
    assert synq.memory_estimate("brunel", 1, 1)["neuron_total"] == 68.0
    with pytest.raises(synq.SynqError) as e:
        synq.memory_estimate("pingpong", 10, 10)
    assert e.value.status == 1
    assert synq.scaling_constant("vogels", 4000) == 1.0
    assert synq.scaling_constant("brunel", 20000) == 1.0
    assert synq.scaling_constant("vogels", 8000) == pytest.approx(0.25)
    with pytest.raises(synq.SynqError) as e:
        synq.scaling_constant("nosuch", 4000)
    assert e.value.status == 2


def test_solve_neurons():
    assert synq.solve_neurons("vogels", 320000) == 4000
    assert synq.solve_neurons("brunel", 20000000) == 20000
    assert synq.solve_neurons("brunel", 1000000000) == 141421
    with pytest.raises(synq.SynqError):
        synq.solve_neurons("pingpong", 1000)


def test_opts_validation():
    o = synq.Opts()
    L = synq.lib()
    assert L.synq_opts_dt(o.h, 0.0) == 1
    assert L.synq_opts_delay(o.h, 0) == 1
    assert L.synq_opts_param(o.h, b"", 1.0) == 1
    assert L.synq_opts_defaults_file(o.h, b"/nonexistent/params.cfg") == 3
    assert L.synq_opts_persistent(o.h, 7) == 1


def test_defaults_file_matches_builtins(tmp_path):
    # configs/model_defaults.cfg runs unchanged: merging it must be accepted
    cfg = tmp_path / "defaults.cfg"
    cfg.write_text("brunel.g = 5.0\n# comment\nvogels.p = 0.02\n")
    o = synq.Opts()
    assert synq.lib().synq_opts_defaults_file(o.h, str(cfg).encode()) == 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    h = C.c_void_p()
    st = synq.lib().synq_sim_new(b"vogels", 400, None, C.byref(h))
    assert st == 5, synq.lib().synq_last_error()
    assert not h.value
