"""bench.py's reference arm on the CPU (no GPU needed): the UNMODIFIED
reference (oracle/_ref/libsynq_ref.so) runs a small Brunel network through
its own C ABI, and the JSON line keeps the driver's contract."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not oracle.have_reference(), reason="oracle/_ref not built")
def test_reference_arm_contract():
    env = dict(os.environ, SYNQ_REF_SAMPLE_STEPS="100")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--synapses", "2e6",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600,
                         check=True).stdout.strip().splitlines()
    line = json.loads(out[-1])
    assert line["impl"] == "reference" and line["unit"] == "events/s" and line["value"] > 0
    assert line["metric"].startswith("synaptic events/sec")
    for k in ("n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "dtype", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
