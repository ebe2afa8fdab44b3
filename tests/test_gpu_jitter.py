"""Pipeline-protocol stress (a substitute for compute-sanitizer racecheck / synccheck, which is closed
on the GPU pool — DESIGN.md "Sanitizers"): with SDNN_JITTER=1 every producer, TMEM issuer and
consumer warp sleeps a pseudo-random 0-2 µs at the mbarrier hand-off points (stage full / empty,
TMEM half full / free, metadata slots), so the warps interleave in orders the free-running kernels
rarely produce.  A missing wait or arrive, a parity slip or a reused slot would change or corrupt Y;
the results must be bitwise identical to the undisturbed run for every pipeline: row kernel (with
split rows summed in shared memory), row split-K, TMEM-R (plain, 1×4 runs, split-K), the row-pair TMEM kernel and the V = 8
TMEM kernel.  (In the TMEM-R kernels the issuer warps are perturbed — a consumer-side hook cost the
bench kernel 2.4 % even when off — so the consumers see the chunks arrive at perturbed times.)"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import sdnn_synth as synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [  # (problem, N, handle options)
    ("c2_768x768", 1024, {}),                               # row kernel + split rows (V = 4)
    ("c2_768x768", 64, {}),                                 # split rows, V = 2 tiles
    ("c2_3072x768", 4096, dict(kernel="row")),              # split rows, 8-row panels, V = 8 tiles
    ("c3_256x128", 128, dict(kernel="row")),                # row kernel, split-K
    ("c3_512x512", 6272, dict(kernel="tmem")),              # TMEM-R
    ("c4_2048x512_s95", 1024, dict(kernel="tmem")),         # TMEM-R with 1×4 runs
    ("c3_1024x512", 6272, dict(kernel="tmem")),             # 245 items: several per CTA when persistent
    ("tsplit", 128, {}),                                    # TMEM-R split-K (4096², N = 128)
    ("c3_512x512", 1024, dict(kernel="tmemp")),             # row pairs
    ("c1", 1024, dict(kernel="tmem8")),                     # V = 8 TMEM kernel
    ("c4_2048x512_s80", 12544, dict(kernel="tmem")),        # TMEM-R, persistent by default (882 items, 8 chunks)
]

SCRIPT = r'''
import importlib.util, os, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
spec = importlib.util.spec_from_file_location("jt", os.path.join(sys.argv[1], "tests", "test_gpu_jitter.py"))
jt = importlib.util.module_from_spec(spec)
spec.loader.exec_module(jt)
CASES, problem = jt.CASES, jt.problem
out = {}
for i, (key, N, opts) in enumerate(CASES):
    p = problem(key, N)
    h = sdnn.Handle.from_problem(p, **opts)
    X = torch.from_numpy(p.x_cols(0, N) if key == "tsplit" else p.x()[:, :N].copy()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    for rep in range(3):
        out[f"{i}_{rep}"] = h.spmm(X, b, act=1).cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def problem(key, N):
    if key == "tsplit":
        return synth.make_problem("tsplit", 4096, 4096, N, 0.9)
    return synth.config_problem(key, N=N)


def test_jittered_pipelines_bitwise(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "jitter.npz"
    env = dict(os.environ, SDNN_JITTER="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(out)], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    got = np.load(out)
    sys.path.insert(0, ROOT)
    import paper_2101_07948_b200 as sdnn
    for i, (key, N, opts) in enumerate(CASES):
        p = problem(key, N)
        h = sdnn.Handle.from_problem(p, **opts)
        X = torch.from_numpy(p.x_cols(0, N) if key == "tsplit" else p.x()[:, :N].copy()).cuda()
        ref = h.spmm(X, torch.from_numpy(p.bias).cuda(), act=1).cpu().numpy()
        for rep in range(3):
            np.testing.assert_array_equal(got[f"{i}_{rep}"], ref, err_msg=f"{key} {opts} rep {rep}")


def test_persistent_tmem_ctas_bitwise(tmp_path):
    """SDNN_TMEM_PERSIST=1 (forced; by default only short K ranges over ≥ 4 items per SM): one CTA per
    SM runs its (row block, N tile) items through one chunk pipeline — same per-row order, so Y is
    bitwise the default launch's (TMEM-R cases only)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "persist.npz"
    env = dict(os.environ, SDNN_TMEM_PERSIST="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(out)], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    got = np.load(out)
    sys.path.insert(0, ROOT)
    import paper_2101_07948_b200 as sdnn
    for i, (key, N, opts) in enumerate(CASES):
        p = problem(key, N)
        h = sdnn.Handle.from_problem(p, **opts)
        X = torch.from_numpy(p.x_cols(0, N) if key == "tsplit" else p.x()[:, :N].copy()).cuda()
        ref = h.spmm(X, torch.from_numpy(p.bias).cuda(), act=1).cpu().numpy()
        np.testing.assert_array_equal(got[f"{i}_0"], ref, err_msg=f"{key} {opts}")


def test_local_pieces_bitwise_vs_workspace(tmp_path):
    """Split rows summed by the row kernel in shared memory (CTA-local pieces, the default) against the
    workspace + split_reduce_kernel form (SDNN_LOCAL_PIECES=0): the same additions in the same order,
    so Y is bitwise equal — V = 2 / 4 / 8 tiles."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "ws.npz"
    env = dict(os.environ, SDNN_LOCAL_PIECES="0", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(out)], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    got = np.load(out)
    sys.path.insert(0, ROOT)
    import paper_2101_07948_b200 as sdnn
    for i, (key, N, opts) in enumerate(CASES[:3]):
        p = problem(key, N)
        h = sdnn.Handle.from_problem(p, **opts)
        assert h.info()["num_split_rows"] > 0
        X = torch.from_numpy(p.x()[:, :N].copy()).cuda()
        ref = h.spmm(X, torch.from_numpy(p.bias).cuda(), act=1).cpu().numpy()
        np.testing.assert_array_equal(got[f"{i}_0"], ref, err_msg=f"{key} N={N} {opts}")
