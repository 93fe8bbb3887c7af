"""`build/synq` command line runner (tools/cli/synq.cpp), the replacement for
the reference CLI (proj/tools/synq.cpp:60-189).

CPU: option parsing, --help/--version, and the reference's usage errors.
GPU: a Vogels-4000 run written as a raster file matches the golden spike
train bit for bit, and --sweep writes the Fig.-3 CSV."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "synq")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", ROOT, "build/synq"], check=True)
    return BIN


def run(cli, *args, timeout=600):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=timeout)


def test_help_and_version(cli):
    r = run(cli, "--help")
    assert r.returncode == 0
    for opt in ("--model", "--neurons", "--synapses", "--duration", "--dt", "--delay", "--seed", "--threads",
                "--deterministic", "--raster", "--stats", "--param", "--defaults", "--net", "--sweep", "--out"):
        assert opt in r.stdout
    v = run(cli, "--version")
    assert v.returncode == 0 and v.stdout.strip()


@pytest.mark.parametrize("args,code,msg", [
    ([], 2, "--model is required"),
    (["--model", "brunel", "--bogus", "1"], 2, "unknown option"),
    (["--model", "brunel", "--neurons", "x"], 2, "not a non-negative integer"),
    (["--model", "brunel", "--neurons"], 2, "needs a value"),
    (["--model", "brunel", "--deterministic=1", "--neurons", "10"], 2, "takes no value"),
    (["--model", "brunel"], 1, "needs --neurons, --synapses or --net"),
    (["--model", "brunel", "--neurons", "10", "--synapses", "1e6"], 1, "not both"),
    (["--model", "brunel", "--sweep", "1e6,1e7", "--neurons", "10"], 1, "--sweep cannot be combined"),
    (["--model", "brunel", "--neurons", "10", "--duration", "0"], 1, "--duration must be > 0"),
    (["--model", "brunel", "--sweep", "1e6"], 1, "at least two sizes"),
    (["--model", "brunel", "--sweep", "1e6,0.5"], 1, "sweep sizes must be >= 1"),
    (["--model", "brunel", "--neurons", "10", "--param", "noequals"], 1, "bad --param"),
    (["--model", "brunel", "--neurons", "10", "--param", "j=abc"], 1, "bad --param value"),
    (["--model", "brunel", "--neurons", "10", "--delay", "4294967297"], 1, "--delay must fit 32 bits"),
    (["--model", "brunel", "--neurons", "10", "--threads", "4294967296"], 1, "--threads must fit 32 bits"),
])
def test_usage_errors(cli, args, code, msg):
    r = run(cli, *args)
    assert r.returncode == code, r.stderr
    assert r.stderr.startswith("synq: error: ") and msg in r.stderr, r.stderr


@pytest.mark.gpu
def test_raster_matches_golden(cli, tmp_path, golden):
    raster = tmp_path / "v4k.txt"
    stats = tmp_path / "v4k.stats"
    r = run(cli, "--model", "vogels", "--neurons", "4000", "--seed", "1", "--duration", "1", "--deterministic",
            "--raster", str(raster), "--stats", str(stats))
    assert r.returncode == 0, r.stderr
    lines = raster.read_text().splitlines()
    assert lines[0].startswith("# dt=")
    rec = np.array([ln.split("\t") for ln in lines[1:]], dtype=np.int64)
    runs = golden["runs"]
    tag = "vogels_4000_s1_t10000_h0_d0"
    counts = np.bincount(rec[:, 0], minlength=10000)
    assert np.array_equal(counts, runs[f"{tag}_counts"])
    assert np.array_equal(rec[:, 1].astype(np.uint32), runs[f"{tag}_ids"])
    assert stats.read_text().strip()


@pytest.mark.gpu
def test_sweep_csv(cli, tmp_path):
    out = tmp_path / "sweep.csv"
    r = run(cli, "--model", "brunel", "--sweep", "1e6,4e6", "--duration", "0.1", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = out.read_text().splitlines()
    assert rows[0] == "synapses,setup_s,sim_s,bytes"
    assert len(rows) == 3
    syn = [int(x.split(",")[0]) for x in rows[1:]]
    assert 0.8e6 < syn[0] < 1.2e6 and 3.2e6 < syn[1] < 4.8e6
    for row in rows[1:]:
        _, setup, sim, nbytes = row.split(",")
        assert float(setup) > 0 and float(sim) > 0 and int(nbytes) > 0
