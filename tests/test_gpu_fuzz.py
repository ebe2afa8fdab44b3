"""Fixed-seed slices of the randomised stress tools (tests/stress/fuzz.py, fuzz_api.py, extreme.py,
fuzz_threads.py) in the GPU suite: random shapes, masks, plan options and entry points against the
oracle, with guard zones, repeat runs, sdnn_tune and serialize round trips.  The long runs that found the
session-4 persistent-CTA bug are recorded in profiles/r02_s4_fuzz.log; these slices keep that coverage in
every round-end run (a failure prints the offending case line)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_tool(args, timeout):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    bad = [ln for ln in r.stdout.splitlines() if "FAIL" in ln]
    assert r.returncode == 0 and not bad, "\n".join(bad[:10]) + "\n" + r.stdout[-1500:] + r.stderr[-1500:]
    return r.stdout


@pytest.mark.parametrize("extra", [["--n", "150", "--seed", "101"], ["--n", "40", "--seed", "102", "--wide-n", "--max-gflop", "8"]])
def test_fuzz_spmm(extra):
    out = run_tool([os.path.join("tests", "stress", "fuzz.py"), *extra], 900)
    assert "0 failed" in out.splitlines()[-1]


def test_fuzz_api():
    out = run_tool([os.path.join("tests", "stress", "fuzz_api.py"), "--n", "120", "--seed", "103"], 900)
    assert "0 failed" in out.splitlines()[-1]


def test_extreme_shapes():
    out = run_tool([os.path.join("tests", "stress", "extreme.py")], 900)
    assert "0 failed" in out.splitlines()[-1]


def test_threads_share_a_handle():
    out = run_tool([os.path.join("tests", "stress", "fuzz_threads.py"), "--threads", "4", "--iters", "30"], 600)
    assert out.splitlines()[-1].startswith("# 0 failures")
