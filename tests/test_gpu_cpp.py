"""C++ model-API tests on the B200 (tests/cpp/test_network.cu, built by
`make tests`): user-defined models compiled into the device engine, checked
against the reference's engine / lazy-STDP properties."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_network")

pytestmark = pytest.mark.gpu

CASES = ["delay_property", "pingpong_flag_reference", "silent_expiry", "ages_bound", "reinit",
         "span_writeback", "accumulation_modes", "debug_checks", "lazy", "plan", "plan_large"]


@pytest.mark.parametrize("case", CASES)
def test_cpp_model_api(case):
    assert os.path.exists(BIN), "build/test_network missing: run `make tests`"
    r = subprocess.run([BIN, case], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
