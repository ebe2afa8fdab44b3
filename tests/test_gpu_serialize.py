"""Prepared-handle serialization (sdnn_serialize / sdnn_deserialize; the paper's reusable preparation,
P:41; SURVEY §5 checkpoint/resume): a handle rebuilt from its blob — without Algorithm 1 or the
packing — gives bitwise the original's results on every plan it keeps; corrupt blobs are rejected."""
import numpy as np
import pytest

import sdnn_synth as synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


@pytest.mark.parametrize("key,opts,Ns", [
    ("c2_768x768", {}, (1024, 100)),                       # auto: row plan (split rows) + TMEM plan
    ("narrow", {}, (128, 2048, 68)),                        # auto with the narrow plan, split-K at N = 128
    ("c3_512x512", dict(kernel="tmem"), (6272, 96)),       # explicit TMEM (+ its ragged fallback)
    ("c1", dict(kernel="group"), (128,)),
    ("c1", dict(kernel="tmem8", permuted_output=True), (1024,)),
])
def test_roundtrip_bitwise(sdnn, key, opts, Ns):
    p = synth.make_problem("ser_nw", 2048, 1024, 2048, 0.9) if key == "narrow" else synth.config_problem(key, N=max(Ns))
    h = sdnn.Handle.from_problem(p, **opts)
    blob = h.serialize()
    h2 = sdnn.Handle.deserialize(blob)
    assert h2.info() == h.info()
    np.testing.assert_array_equal(h2.permutation(), h.permutation())
    assert h2.serialize() == blob  # stable
    b = torch.from_numpy(p.bias).cuda()
    for N in Ns:
        X = torch.from_numpy(np.ascontiguousarray(p.x_cols(0, N))).cuda()
        assert h2.kernel_for(N, X.data_ptr()) == h.kernel_for(N, X.data_ptr())
        np.testing.assert_array_equal(h2.spmm(X, b, act=1).cpu().numpy(), h.spmm(X, b, act=1).cpu().numpy())


def test_corrupt_blobs_rejected(sdnn):
    p = synth.config_problem("c1")
    blob = sdnn.Handle.from_problem(p).serialize()
    for bad in (b"", blob[:7], b"XXXXXXXX" + blob[8:], blob[:len(blob) // 2], blob + b"\0",
                blob[:8] + (2).to_bytes(4, "little") + blob[12:]):
        with pytest.raises(sdnn.SdnnError):
            sdnn.Handle.deserialize(bad)


def test_codegen_not_serialized(sdnn):
    p = synth.config_problem("c1")
    with pytest.raises(sdnn.SdnnError) as e:
        sdnn.Handle.from_problem(p, kernel="codegen").serialize()
    assert e.value.status == 3
