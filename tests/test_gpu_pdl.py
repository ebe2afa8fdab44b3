"""Programmatic dependent launch (the row, TMEM-R and reduction kernels run their prologue while the
previous kernel on the stream drains, and touch X / bias / Y only after `griddepcontrol.wait`):
dependent calls must see each other's complete results.

* a dependent two-layer chain (layer 2 reads layer 1's Y; a third kernel then overwrites layer 1's Y)
  captured in a CUDA graph and replayed, eagerly on one stream, and alternated between two streams
  with events: Y2 bitwise equal to the synchronised calls, on every plan kind the chain takes (row
  plan with split rows, TMEM-R, TMEM-R split-K with its reduction kernel, persistent TMEM-R);
* the same Y with `SDNN_PDL=0` (plain launches) in a subprocess: bitwise equal."""
import os
import subprocess
import sys

import numpy as np
import pytest

import sdnn_synth as synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (layer-1 problem, layer-2 problem, N): layer 2's K = layer 1's M
CHAINS = [
    ("c2_3072x768", "c2_768x3072", 1024),   # TMEM-R, then TMEM-R split-K + splitk_reduce_kernel
    ("c2_768x768", "c2_768x768", 1024),     # row plans with split rows (summed in the kernel)
    ("c2_768x768", "c2_768x768", 102),      # ragged N: generic path, workspace + split_reduce_kernel
    ("c4_512x2048_s80", "c4_2048x512_s80", 12544),  # TMEM-R, then persistent TMEM-R (short K, many items)
]


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


def _layers(sdnn, k1, k2, N):
    p1 = synth.config_problem(k1)
    p2 = synth.config_problem(k2)
    assert p2.K == p1.M
    h1, h2 = sdnn.Handle.from_problem(p1), sdnn.Handle.from_problem(p2)
    X = torch.from_numpy(np.ascontiguousarray(p1.x()[:, :N])).cuda()
    b1, b2 = torch.from_numpy(p1.bias).cuda(), torch.from_numpy(p2.bias).cuda()
    return h1, h2, X, b1, b2


def _reference(h1, h2, X, b1, b2):
    Y1 = h1.spmm(X, b1, act=1)
    torch.cuda.synchronize()
    Y2 = h2.spmm(Y1, b2, act=1)
    torch.cuda.synchronize()
    return Y2


@pytest.mark.parametrize("k1,k2,N", CHAINS)
def test_dependent_chain_graph_eager_streams(sdnn, k1, k2, N):
    h1, h2, X, b1, b2 = _layers(sdnn, k1, k2, N)
    ref = _reference(h1, h2, X, b1, b2)
    Y1 = torch.empty((h1.M, N), device="cuda")
    Y2 = torch.full_like(ref, float("nan"))

    def chain():
        h1.spmm(X, b1, act=1, out=Y1)
        h2.spmm(Y1, b2, act=1, out=Y2)
        Y1.fill_(float("nan"))  # overwritten after layer 2 read it: a late reader would see NaN

    # eager, one stream, back to back
    for _ in range(3):
        chain()
    torch.cuda.synchronize()
    assert torch.equal(Y2, ref)
    # CUDA graph (programmatic edges between the captured kernels), replayed
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        chain()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    Y2.fill_(float("nan"))
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            chain()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Y2, ref)
    # two streams, layer 2 on the second after an event
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        Y2.fill_(float("nan"))
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            h1.spmm(X, b1, act=1, out=Y1)
        ev = torch.cuda.Event()
        ev.record(s1)
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            h2.spmm(Y1, b2, act=1, out=Y2)
        torch.cuda.synchronize()
        assert torch.equal(Y2, ref)


SCRIPT = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
import paper_2101_07948_b200 as sdnn
import test_gpu_pdl as t
out = {}
for i, (k1, k2, N) in enumerate(t.CHAINS):
    h1, h2, X, b1, b2 = t._layers(sdnn, k1, k2, N)
    out[str(i)] = t._reference(h1, h2, X, b1, b2).cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def test_plain_launches_bitwise(sdnn, tmp_path):
    out = tmp_path / "nopdl.npz"
    env = dict(os.environ, SDNN_PDL="0", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(out)], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    got = np.load(out)
    for i, (k1, k2, N) in enumerate(CHAINS):
        h1, h2, X, b1, b2 = _layers(sdnn, k1, k2, N)
        np.testing.assert_array_equal(got[str(i)], _reference(h1, h2, X, b1, b2).cpu().numpy(), err_msg=f"{k1}->{k2} N={N}")
