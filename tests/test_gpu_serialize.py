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
    ("c3_512x512", dict(kernel="tmemp"), (6272, 100)),          # Algorithm 1 row pairs (+ ragged fallback)
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
                blob[:8] + (99).to_bytes(4, "little") + blob[12:]):
        with pytest.raises(sdnn.SdnnError):
            sdnn.Handle.deserialize(bad)


def test_codegen_not_serialized(sdnn):
    p = synth.config_problem("c1")
    with pytest.raises(sdnn.SdnnError) as e:
        sdnn.Handle.from_problem(p, kernel="codegen").serialize()
    assert e.value.status == 3


# blob layout (sdnn_spmm.cu plan_fields): scalar fields, then length-prefixed vectors
_SCALARS = [("M", "i4"), ("K", "i4"), ("nnz", "i8"), ("permuted", "i4"), ("permuted_output", "i4"),
            ("no_split_k", "i4"), ("kernel", "i4"), ("group_entries", "i8"), ("group_sb", "i4"),
            ("group_subblocks", "i8"), ("panel_rows", "i4"), ("cta_panels", "i4"), ("num_panels", "i4"),
            ("num_row_blocks", "i4"), ("k_chunk", "i4"), ("num_chunks", "i4"), ("max_block_bytes", "i4"),
            ("max_panel_nnz", "i8"), ("tmem_fill", "i4")]
_VECTORS = [("perm", "i4"), ("row_orig", "i4"), ("blk_off", "i8"), ("meta", "u1"), ("piece_row", "i4"),
            ("piece_begin", "i4"), ("piece_end", "i4"), ("split_row", "i4"), ("split_first", "i4"),
            ("split_count", "i4")]


def _index(blob: bytes):
    """{(plan index, field): (byte offset, dtype, count)} of every plan in a blob."""
    off, out = 16, {}
    nplans = int.from_bytes(blob[12:16], "little")
    for i in range(nplans):
        out[(i, "role")] = (off, "u4", 1)
        off += 4
        for name, dt in _SCALARS:
            out[(i, name)] = (off, dt, 1)
            off += np.dtype(dt).itemsize
        for name, dt in _VECTORS:
            n = int.from_bytes(blob[off:off + 8], "little")
            out[(i, name)] = (off + 8, dt, n)
            off += 8 + n * np.dtype(dt).itemsize
    assert off == len(blob)
    return out


def _patch(blob: bytes, idx, plan: int, field: str, value, at: int = 0) -> bytes:
    off, dt, n = idx[(plan, field)]
    assert at < n
    size = np.dtype(dt).itemsize
    b = bytearray(blob)
    b[off + at * size:off + (at + 1) * size] = np.array([value], dtype=dt).tobytes()
    return bytes(b)


def test_corrupt_fields_rejected(sdnn):
    """Structural corruptions the kernels would turn into out-of-bounds accesses are rejected by the
    deserializer: split-row targets, split / piece table bounds, panel geometry, plan kind
    per role, metadata segment bounds and TMEM columns."""
    p = synth.config_problem("c2_768x768")  # auto: row plan with split rows (role 0) + TMEM plan (role 1)
    blob = sdnn.Handle.from_problem(p).serialize()
    idx = _index(blob)
    roles = {int(np.frombuffer(blob, "u4", 1, idx[(i, "role")][0])[0]): i for i in range(len({k[0] for k in idx}))}
    row, tm = roles[0], roles[1]
    assert idx[(row, "split_row")][2] > 0  # the fixture really has split rows
    meta_off, _, _ = idx[(tm, "meta")]
    hdr_bytes = 10 * 24 * 4
    first_entry = int(np.frombuffer(blob, "u4", 1, meta_off)[0]) >> 16
    bad = [
        _patch(blob, idx, row, "split_row", p.M),                        # reduction writes past Y
        _patch(blob, idx, row, "split_row", -1),
        _patch(blob, idx, row, "split_first", 10**6),                   # beyond the piece table
        _patch(blob, idx, row, "split_count", 0),
        _patch(blob, idx, row, "num_panels", 1),                        # != row blocks × CTA panels
        _patch(blob, idx, row, "panel_rows", 6),                        # not a compiled geometry
        _patch(blob, idx, tm, "cta_panels", 6),                         # TMEM kernel: 24 warps
        _patch(blob, idx, tm, "kernel", 1),                             # role 1 must be a TMEM plan
        _patch(blob, idx, tm, "max_block_bytes", 200 * 1024),           # stage ring beyond shared memory
        _patch(blob, idx, tm, "meta", 0xFF, at=2),                      # slot 0: start 0x..FF.. beyond block
        _patch(blob, idx, tm, "meta", 0x7F, at=hdr_bytes + 8 * first_entry + 1),  # TMEM column ≥ 512
    ]
    for i, b in enumerate(bad):
        with pytest.raises(sdnn.SdnnError) as e:
            sdnn.Handle.deserialize(b)
        assert e.value.status == 1, i  # SDNN_ERR_INVALID_ARGUMENT
    sdnn.Handle.deserialize(blob).close()  # the unmodified blob still loads


def test_second_tmem_plan_round_trip(sdnn):
    """An auto handle's second TMEM plan (more row blocks, picked per call by wave fill) travels in the
    blob as role 4, so the deserialized handle holds the same plans, and a role-4 plan without its
    role-1 partner, of another shape or of another kernel is rejected."""
    p = synth.config_problem("c2_3072x768")  # tmem_pick takes the second plan at N = 1024
    h = sdnn.Handle.from_problem(p)
    blob = h.serialize()
    idx = _index(blob)
    nplans = len({k[0] for k in idx})
    roles = {int(np.frombuffer(blob, "u4", 1, idx[(i, "role")][0])[0]): i for i in range(nplans)}
    assert 1 in roles and 4 in roles
    rb = lambda i: int(np.frombuffer(blob, "i4", 1, idx[(i, "num_row_blocks")][0])[0])
    assert rb(roles[4]) > rb(roles[1])
    h2 = sdnn.Handle.deserialize(blob)
    assert h2.serialize() == blob  # every plan, the second TMEM plan included, came back
    X = torch.from_numpy(p.x()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    assert h2.kernel_for(p.N, X.data_ptr()) == h.kernel_for(p.N, X.data_ptr()) == 4
    np.testing.assert_array_equal(h2.spmm(X, b, act=1).cpu().numpy(), h.spmm(X, b, act=1).cpu().numpy())
    for bad in (_patch(blob, idx, roles[4], "kernel", 1), _patch(blob, idx, roles[4], "M", p.M - 1),
                _patch(blob, idx, roles[4], "role", 1), _patch(blob, idx, roles[1], "role", 4)):
        with pytest.raises(sdnn.SdnnError):
            sdnn.Handle.deserialize(bad)
