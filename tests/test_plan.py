"""Host-side preparation checks (no GPU): the C++ inverted-index Algorithm 1 against the oracle
 and the packing invariants of the execution-ordered format."""
import numpy as np
import pytest

import paper_2101_07948_b200 as sdnn
import sdnn_synth as synth


def decode(p, plan):
    """Decode the exported plan back into (orig_row, col, val) triples, checking the layout."""
    info = plan.info()
    if info["kernel"] == 2:
        return decode_group(p, plan)
    if info["kernel"] == 6:
        return decode_pairs(p, plan)
    row_orig, blk_off, meta = plan.export()
    rw, wc, kc, nch, nrb = (info[k] for k in ("panel_rows", "cta_panels", "k_chunk", "num_chunks", "num_row_blocks"))
    V = {4: 4, 5: 8}.get(info["kernel"], 0)
    if V:  # kernel 4: 24 warps with their own panels (replicated TMEM lane quarters); kernel 5: 6 slots
        assert (rw, wc, kc) == ((10, 24, 64) if V == 4 else (5, 6, 32))
    rcta = rw * wc
    hdr_bytes = (rcta * 4 + 15) // 16 * 16
    assert blk_off[0] == 0 and blk_off[-1] == meta.size and np.all(np.diff(blk_off) > 0)
    assert np.all(blk_off % 16 == 0)
    assert np.diff(blk_off).max() <= info["max_block_bytes"]
    triples = []
    last_col = {}
    runs = []
    prow, pbeg, pend = plan.export_pieces() if info["num_pieces"] else ([], [], [])
    for b in range(nrb):
        for j in range(nch):
            blk = meta[blk_off[b * nch + j]:blk_off[b * nch + j + 1]]
            hdr = blk[:rcta * 4].view(np.uint32)
            ent = blk[hdr_bytes:]
            for s in range(rcta):
                start, cnt = int(hdr[s] >> 16), int(hdr[s] & 0xFFFF)
                nrun = 0
                if V:  # TMEM format: count in bits 0..7, leading aligned 1×4 runs in bits 8..15
                    cnt, nrun = cnt & 0xFF, cnt >> 8
                    assert V == 4 or nrun == 0
                    assert 4 * nrun <= cnt
                    for u in range(nrun):
                        runs.append((b, j, start + 4 * u))
                assert start % 2 == 0
                orow = int(row_orig[b * rcta + s])
                key = orow
                if orow <= -2:  # a piece of a split row (row plan): CSR entries [pbeg, pend) of prow
                    pid = -2 - orow
                    orow, key = int(prow[pid]), (int(prow[pid]), pid)
                if orow < 0:
                    assert cnt == 0
                    continue
                if V:  # TMEM format: segments padded to whole pairs
                    assert cnt % 2 == 0
                elif cnt % 2:  # row format: an odd segment's partner slot is the zero entry the kernels read
                    assert not np.any(ent[(start + cnt) * 8:(start + cnt) * 8 + 8])
                for i in range(cnt):
                    e = ent[(start + i) * 8:(start + i) * 8 + 8]
                    cl = int(e[:4].view(np.uint32)[0])
                    w = e[4:].view(np.float32)[0]
                    if V:  # column field = V·col_local + 256·(chunk parity): the TMEM column of X[col]
                        # (kernel 4: | TMEM lane base of the slot's warp quarter, (32·(warp % 4)) << 16)
                        lane_base = ((32 * ((s // rw) % 4)) << 16) if V == 4 else 0
                        assert cl & ~0xFFFF == lane_base
                        cl &= 0xFFFF
                        half = 256 * (j & 1)
                        if w == 0:
                            assert cl == half  # padding entry
                            continue
                        assert (cl - half) % V == 0 and 0 <= cl - half < 256
                        cl = (cl - half) // V
                    assert 0 <= cl < kc
                    col = j * kc + cl
                    assert col > last_col.get(key, -1)  # ascending column order per row (per piece)
                    last_col[key] = col
                    triples.append((orow, col, w))
    for b, j, at in runs:  # a run is 4 consecutive columns k..k+3, k % 4 == 0
        blk = meta[blk_off[b * nch + j]:blk_off[b * nch + j + 1]]
        cols = [int(blk[hdr_bytes + (at + t) * 8:hdr_bytes + (at + t) * 8 + 4].view(np.uint32)[0]) & 0xFFFF
                for t in range(4)]
        assert cols == [cols[0] + 4 * t for t in range(4)] and (cols[0] % 256) % 16 == 0
    decode.runs = len(runs)
    # pieces of a row: consecutive ids q = 0..P-1, piece q = entries row_ptr[r] + q, + P, … (interleaved)
    pid = 0
    while pid < len(prow):
        r = int(prow[pid])
        P = int(np.sum(prow == r))
        assert list(prow[pid:pid + P]) == [r] * P and P >= 2
        for q in range(P):
            assert pbeg[pid + q] == p.row_ptr[r] + q and pend[pid + q] == p.row_ptr[r + 1]
        pid += P
    return info, row_orig, triples


def decode_pairs(p, plan):
    """Kernel 6 (TMEM, Algorithm 1 row pairs): per slot pair, shared columns {col, w_a, w_b, 0}, then
    each row's own columns, each list ascending, with the warp's TMEM lane base in every column."""
    info = plan.info()
    row_orig, blk_off, meta = plan.export()
    rw, wc, kc, nch, nrb = (info[k] for k in ("panel_rows", "cta_panels", "k_chunk", "num_chunks", "num_row_blocks"))
    assert (rw, wc, kc) == (10, 24, 64)
    rcta = rw * wc
    hdr_bytes = (rcta * 4 + 15) // 16 * 16
    assert blk_off[0] == 0 and blk_off[-1] == meta.size and np.all(blk_off % 16 == 0)
    triples, shared = [], 0
    perm = sdnn.permutation(p.row_ptr, p.col_idx, p.M, p.K) if info["permuted"] else np.arange(p.M)
    decode_pairs.pos = np.empty(p.M, int)
    decode_pairs.pos[perm] = np.arange(p.M)
    for b in range(nrb):
        for j in range(nch):
            blk = meta[blk_off[b * nch + j]:blk_off[b * nch + j + 1]]
            hdr = blk[:rcta * 4].view(np.uint32)
            ent = blk[hdr_bytes:]

            def entry(i):
                cl = int(ent[i * 8:i * 8 + 4].view(np.uint32)[0])
                lane_base = (32 * ((s // rw) % 4)) << 16
                assert cl & ~0xFFFF == lane_base
                cl &= 0xFFFF
                half = 256 * (j & 1)
                assert (cl - half) % 4 == 0 and 0 <= cl - half < 256
                return (cl - half) // 4, ent[i * 8 + 4:i * 8 + 8].view(np.float32)[0]
            for s in range(0, rcta, 2):
                ha, hb = int(hdr[s]), int(hdr[s + 1])
                start, ns, na, b0, nb = ha >> 16, (ha >> 8) & 0xFF, ha & 0xFF, hb >> 16, hb & 0xFF
                assert start % 2 == 0 and na % 2 == 0 and nb % 2 == 0 and b0 == start + 2 * ns + na
                ra, rb = int(row_orig[b * rcta + s]), int(row_orig[b * rcta + s + 1])
                if ra >= 0 and rb >= 0:  # a pair = two consecutive Algorithm 1 positions (2i, 2i + 1)
                    assert decode_pairs.pos[rb] == decode_pairs.pos[ra] + 1 and decode_pairs.pos[ra] % 2 == 0
                cols_a, cols_b = [], []
                for i in range(ns):
                    c, wa = entry(start + 2 * i)
                    wb = ent[(start + 2 * i + 1) * 8:(start + 2 * i + 1) * 8 + 4].view(np.float32)[0]
                    assert ra >= 0 and rb >= 0
                    triples += [(ra, j * kc + c, wa), (rb, j * kc + c, wb)]
                    cols_a.append(c), cols_b.append(c)
                    shared += 1
                for r, n0, n in ((ra, start + 2 * ns, na), (rb, b0, nb)):
                    own = []
                    for i in range(n):
                        c, w = entry(n0 + i)
                        if w == 0:
                            assert c == 0  # padding entry (column 0 of the half)
                            continue
                        assert r >= 0
                        triples.append((r, j * kc + c, w))
                        own.append(c)
                    assert own == sorted(own)
                assert cols_a == sorted(cols_a)
    decode_pairs.shared = shared
    return info, row_orig, triples


def decode_group(p, plan):
    info = plan.info()
    row_orig, blk_off, meta = plan.export()
    wc, kc, nch, nrb, sb = (info[k] for k in ("cta_panels", "k_chunk", "num_chunks", "num_row_blocks", "group_sb"))
    assert info["panel_rows"] == 16 and sb in (1, 2, 4)
    assert blk_off[0] == 0 and blk_off[-1] == meta.size and np.all(blk_off % 16 == 0)
    triples, last_col, entries, nsb = [], {}, 0, 0
    for b in range(nrb):
        for j in range(nch):
            blk = meta[blk_off[b * nch + j]:blk_off[b * nch + j + 1]].view(np.uint32)
            for w in range(wc):
                hoff, n, woff = int(blk[4 * w]), int(blk[4 * w + 1]), int(blk[4 * w + 2])
                assert hoff % 4 == 0 and woff % 4 == 0  # 16-byte aligned heads and weights
                wts = blk[woff:].view(np.float32)
                wi, prev = 0, -1
                for e in range(n):
                    h = int(blk[hoff + e])
                    cl, sbm = h & 0xFFFF, h >> 16
                    assert 0 <= cl < kc and cl > prev and sbm != 0 and sbm < (1 << (16 // sb))
                    prev = cl
                    entries += 1
                    for s_ in range(16 // sb):
                        if not sbm >> s_ & 1:
                            continue
                        nsb += 1
                        for i in range(sb):
                            r = s_ * sb + i
                            wv = wts[wi]
                            wi += 1
                            orow = int(row_orig[(b * wc + w) * 16 + r])
                            if wv == 0:  # padding slot (generators never emit explicit zeros)
                                continue
                            assert orow >= 0
                            col = j * kc + cl
                            assert col > last_col.get(orow, -1)
                            last_col[orow] = col
                            triples.append((orow, col, wv))
    assert abs(entries * 1000 // max(p.nnz, 1) - info["group_entries_per_nnz_x1000"]) <= 1
    assert abs(nsb * 1000 // max(p.nnz, 1) - info["group_subblocks_per_nnz_x1000"]) <= 1
    return info, row_orig, triples


def csr_triples(p):
    r = np.repeat(np.arange(p.M), np.diff(p.row_ptr))
    return sorted(zip(r.tolist(), p.col_idx.tolist(), p.vals.tolist()))


@pytest.mark.parametrize("key", ["c1", "c2_768x768", "c3_128x64", "c4_512x2048_s95"])
def test_c_alg1_equals_oracle_on_configs(oracle_mod, key):
    p = synth.config_problem(key, N=4)
    np.testing.assert_array_equal(sdnn.permutation(p.row_ptr, p.col_idx, p.M, p.K),
                                  oracle_mod.alg1(p.row_ptr, p.col_idx, p.M, p.K))


@pytest.mark.parametrize("seed", range(100))
def test_c_alg1_equals_bruteforce_random(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    mask = rng.random((M, K)) < rng.uniform(0, 0.7)
    if seed % 5 == 0:
        mask[M // 2:] = mask[:M - M // 2]
    rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum(mask.sum(1))
    ci = np.nonzero(mask)[1].astype(np.int32)
    order = sdnn.permutation(rp, ci, M, K).tolist()
    assert order == oracle_mod.alg1_bruteforce([set(np.flatnonzero(mask[i]).tolist()) for i in range(M)])


@pytest.mark.parametrize("M,K,per_row,seed", [(3000, 50, 3, 0), (5000, 8, 1, 1), (2000, 400, 2, 2), (4000, 64, 0.3, 3),
                                              (1500, 1500, 40, 4), (2500, 30, 6, 5)])
def test_c_alg1_tall_sparse_equals_oracle(oracle_mod, M, K, per_row, seed):
    """Algorithm 1's two argmax modes (rows touched by the previous row when they are few, a plain scan
    otherwise) and its list compaction give the oracle's order on tall sparse matrices, where steps switch
    between the modes — with duplicate rows (ties: lowest index), empty rows and runs of rows that share
    no column with their predecessor (the lowest-remaining-index pointer)."""
    rng = np.random.default_rng(seed)
    counts = np.minimum(K, rng.poisson(per_row, size=M))
    counts[rng.integers(0, M, M // 10)] = 0                     # empty rows
    cols = [np.sort(rng.choice(K, size=int(n), replace=False)) for n in counts]
    for dst, src in zip(rng.integers(0, M, M // 8), rng.integers(0, M, M // 8)):  # duplicates → ties
        cols[dst] = cols[src]
    rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum([len(c) for c in cols])
    ci = (np.concatenate(cols) if rp[-1] else np.zeros(0)).astype(np.int32)
    order = sdnn.permutation(rp, ci, M, K)
    assert sorted(order.tolist()) == list(range(M))
    np.testing.assert_array_equal(order, oracle_mod.alg1(rp, ci, M, K))


@pytest.mark.parametrize("key,opts", [
    ("c1", {}), ("c1", dict(permute=False)), ("c2_768x3072", {}), ("c3_128x64", dict(panel_rows=8, cta_panels=3)),
    ("c4_512x2048_s80", dict(k_chunk=8)), ("c3_256x128", dict(k_chunk=96, cta_panels=1)),
    ("c1", dict(kernel="group")), ("c2_768x3072", dict(kernel="group")), ("c3_128x64", dict(kernel="group", cta_panels=3)),
    ("c4_2048x512_s95", dict(kernel="group", k_chunk=16)), ("c2_768x768", dict(kernel="group", permute=False)),
    ("c2_768x768", dict(kernel="group", group_sb=1)), ("c3_512x512", dict(kernel="group", group_sb=2)),
    ("c4_512x2048_s80", dict(kernel="group", group_sb=4)),
    ("c1", dict(kernel="tmem")), ("c2_768x3072", dict(kernel="tmem")), ("c4_2048x512_s95", dict(kernel="tmem", permute=False)),
    ("c1", dict(kernel="tmem8")), ("c2_768x768", dict(kernel="tmem8")), ("c4_512x2048_s80", dict(kernel="tmem8")),
    ("c1", dict(kernel="tmemp")), ("c2_768x3072", dict(kernel="tmemp")), ("c4_2048x512_s80", dict(kernel="tmemp")),
    ("c3_512x512", dict(kernel="tmemp", permute=False)),
])
def test_packing_invariants(oracle_mod, key, opts):
    p = synth.config_problem(key, N=4)
    plan = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, **opts)
    info, row_orig, triples = decode(p, plan)
    # every nonzero appears exactly once with its original row, column and value
    assert sorted(triples) == csr_triples(p)
    perm = sdnn.permutation(p.row_ptr, p.col_idx, p.M, p.K) if opts.get("permute", True) else np.arange(p.M)
    if info["kernel"] == 2:
        # group kernel: panels tile the Algorithm 1 order, then empty slots
        np.testing.assert_array_equal(row_orig[:p.M], perm)
        assert np.all(row_orig[p.M:] == -1)
    else:
        # row kernel: every row in exactly one slot (or split into pieces); rows of a warp keep their
        # Algorithm 1 order
        prow = plan.export_pieces()[0] if info["num_pieces"] else np.zeros(0, np.int32)
        assert sorted(row_orig[row_orig >= 0].tolist() + sorted(set(prow.tolist()))) == list(range(p.M))
        assert sorted((-2 - row_orig[row_orig <= -2]).tolist()) == list(range(len(prow)))
        pos = np.empty(p.M, int); pos[perm] = np.arange(p.M)
        for w in range(info["num_panels"]):
            rs = [r for r in row_orig[w * info["panel_rows"]:(w + 1) * info["panel_rows"]] if r >= 0]
            assert list(pos[rs]) == sorted(pos[rs])
        if info["num_pieces"]:
            return  # load balance of split plans: test_split_rows_balance
        # LPT balance: max warp load <= mean load + heaviest row
        loads = [sum(int(np.diff(p.row_ptr)[r]) for r in row_orig[w * info["panel_rows"]:(w + 1) * info["panel_rows"]] if r >= 0)
                 for w in range(info["num_panels"])]
        assert max(loads) <= p.nnz / info["num_panels"] + np.diff(p.row_ptr).max() + info["panel_rows"]
    assert info["num_row_blocks"] * info["panel_rows"] * info["cta_panels"] >= p.M
    cnt = np.diff(p.row_ptr)
    assert info["max_panel_nnz"] >= cnt.max()


def test_split_rows_balance():
    """Log-normal rows (c2, up to K nonzeros): heavy rows are cut into pieces so that no warp's load
    exceeds the mean by more than one piece; uniform masks (c3-c5) are never split; the flag turns
    it off."""
    for key in ("c2_768x768", "c2_768x3072", "c2_3072x768"):
        p = synth.config_problem(key, N=4)
        plan = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="row")
        info = plan.info()
        assert info["num_split_rows"] > 0 and info["num_pieces"] > info["num_split_rows"]
        mean = p.nnz / info["num_panels"]
        T = max(64, -(-p.nnz // (info["num_panels"])))
        assert info["max_panel_nnz"] <= 1.2 * mean + T, key
        off = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="row", split_rows=False).info()
        assert off["num_pieces"] == 0 and off["max_panel_nnz"] >= np.diff(p.row_ptr).max()
        decode(p, plan)
    for key in ("c3_512x512", "c4_2048x512_s80"):
        p = synth.config_problem(key, N=4)
        assert sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="row").info()["num_pieces"] == 0


def test_split_row_pieces_share_a_row_block():
    """The pieces of a split row sit on distinct warps of ONE row block (so the row kernel adds them in
    shared memory at its end), at most one piece per warp of the block, consecutive piece ids."""
    for key in ("c2_768x768", "c2_768x3072", "c2_3072x768"):
        p = synth.config_problem(key, N=4)
        plan = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="row")
        info = plan.info()
        rw, wc = info["panel_rows"], info["cta_panels"]
        row_orig = plan.export()[0]
        prow = plan.export_pieces()[0]
        where = {}
        for sl, o in enumerate(row_orig):
            if o <= -2:
                where[-2 - int(o)] = (sl // (rw * wc), sl // rw)
        assert sorted(where) == list(range(len(prow)))
        for r in np.unique(prow):
            pids = np.flatnonzero(prow == r)
            assert np.all(np.diff(pids) == 1) and 2 <= len(pids) <= wc
            blocks = {where[int(i)][0] for i in pids}
            warps = {where[int(i)][1] for i in pids}
            assert len(blocks) == 1 and len(warps) == len(pids), (key, r)


def test_auto_kernel_choice_and_alg1_benefit():
    """The cost model picks the group kernel where 16-row unions are small, and Algorithm 1 shrinks
    the unions on structured masks (the paper's reason for the permutation)."""
    for key in ("c2_768x768", "c4_2048x512_s80"):
        p = synth.config_problem(key, N=4)
        a = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="group").info()
        b = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="group", permute=False).info()
        assert a["group_entries_per_nnz_x1000"] < b["group_entries_per_nnz_x1000"], key
        assert sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K).info()["kernel"] == 1


def test_degenerate_shapes():
    for M, K, dens in [(1, 1, 1.0), (1, 300, 0.5), (300, 1, 0.5), (5, 7, 0.0), (33, 65, 1.0)]:
        rng = np.random.default_rng(M * K)
        mask = rng.random((M, K)) < dens
        rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum(mask.sum(1))
        ci = np.nonzero(mask)[1].astype(np.int32)
        v = rng.standard_normal(ci.size).astype(np.float32)
        p = synth.Problem("d", M, K, 1, 0, "x", rp, ci, v, None, 0, 0)
        v[v == 0] = 1.0  # decode treats 0.0 weights as padding
        for kernel, sb in (("row", 0), ("group", 1), ("group", 2), ("group", 4), ("tmem", 0), ("tmem8", 0), ("tmemp", 0)):
            plan = sdnn.Plan(rp, ci, v, M, K, kernel=kernel, group_sb=sb)
            _, _, triples = decode(p, plan)
            assert sorted(triples) == csr_triples(p)


def test_tmem_runs_marked_on_block_clustered_masks():
    """c4's 1×4 runs are counted as leading runs of their row segments (one tcgen05.ld.x16 each)."""
    p = synth.config_problem("c4_2048x512_s95", N=4)
    plan = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="tmem")
    _, _, triples = decode(p, plan)
    assert sorted(triples) == csr_triples(p)
    assert decode.runs == p.nnz // 4
    p = synth.config_problem("c3_512x512", N=4)
    decode(p, sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="tmem"))
    assert decode.runs < p.nnz // 500  # chance leading runs of a uniform 85 % mask


def test_tmem_plan_options():
    p = synth.config_problem("c1", N=4)
    with pytest.raises(sdnn.SdnnError):
        sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="tmem", panel_rows=11)
    with pytest.raises(sdnn.SdnnError):
        sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="tmem8", panel_rows=4)
    # kernel 4, panel_rows = r: about r rows per warp (more row blocks of 24 ten-slot panels)
    q = synth.config_problem("c2_3072x768", N=4)
    i10 = sdnn.Plan(q.row_ptr, q.col_idx, q.vals, q.M, q.K, kernel="tmem").info()
    i8 = sdnn.Plan(q.row_ptr, q.col_idx, q.vals, q.M, q.K, kernel="tmem", panel_rows=8).info()
    assert (i10["num_row_blocks"], i8["num_row_blocks"]) == (13, 16) and i8["panel_rows"] == 10
    plan8 = sdnn.Plan(q.row_ptr, q.col_idx, q.vals, q.M, q.K, kernel="tmem", panel_rows=8)
    assert sorted(decode(q, plan8)[2]) == csr_triples(q)
    with pytest.raises(sdnn.SdnnError):
        sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="tmem8", k_chunk=64)
    assert sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="tmem8", k_chunk=32).info()["kernel"] == 5


def test_plan_deterministic():
    p = synth.config_problem("c2_768x768", N=4)
    a = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K).export()
    b = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K).export()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_codegen_plan_and_ptx(tmp_path):
    """Codegen plan: panels partition the Algorithm 1 order; the generated PTX has one FFMA with an
    immediate weight per nonzero of the panel (P:139 registers named by position) and assembles."""
    import shutil
    import subprocess
    p = synth.config_problem("c3_512x512", N=4)
    plan = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="codegen")
    info = plan.info()
    row_orig, _, _ = plan.export()
    perm = sdnn.permutation(p.row_ptr, p.col_idx, p.M, p.K)
    np.testing.assert_array_equal(row_orig[row_orig >= 0], perm)
    assert info["kernel"] == 3 and info["panel_rows"] <= 128 and 296 % info["num_panels"] == 0
    ptx = plan.codegen_ptx(p.row_ptr, p.col_idx, p.vals, 0)
    rows0 = [r for r in row_orig[:info["panel_rows"]] if r >= 0]
    nnz0 = int(sum(np.diff(p.row_ptr)[rows0]))
    assert ptx.count("fma.rn.f32 ") == nnz0
    import struct
    w = struct.unpack("<I", struct.pack("<f", p.vals[p.row_ptr[rows0[0]]]))[0]
    assert f"0f{w:08X}" in ptx
    ptxas = shutil.which("ptxas") or "/usr/local/cuda/bin/ptxas"
    f = tmp_path / "p0.ptx"
    f.write_text(ptx)
    r = subprocess.run([ptxas, "-arch=sm_100a", "-O1", str(f), "-o", str(tmp_path / "p0.cubin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
