"""N > 1 host logic on CPU with world_size-2 gloo: column sharding covers N exactly,
max-over-ranks timing, the prepared-plan hash agrees across ranks, and concatenated per-rank
results equal the unsharded result (oracle, column independence)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import sdnn_synth as synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2101_07948_b200 as sdnn
        p = synth.make_problem("mr", 300, 200, 1000, 0.9, mask="lognormal", seed=3)
        c0, c1 = bench.shard_range(p.N, rank, world)
        t = bench.max_over_ranks(float(rank + 1), dist)
        plan = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K)
        # the hash covers the packed arrays (meta, blk_off, row_orig, split tables), not just the info:
        # a one-byte difference in one rank's metadata must be caught
        arrays = [*plan.export(), *plan.export_pieces()]
        packed = b"".join(np.ascontiguousarray(a).tobytes() for a in arrays)
        same = bench.check_same_across_ranks(bench.plan_hash(packed), dist)
        meta = arrays[2].copy()
        meta[len(meta) // 2] ^= 1 if rank == 1 else 0
        tampered = b"".join(np.ascontiguousarray(a).tobytes() for a in [arrays[0], arrays[1], meta, *arrays[3:]])
        caught = not bench.check_same_across_ranks(bench.plan_hash(tampered), dist)
        differ = bench.check_same_across_ranks(f"rank{rank}", dist)
        Y, _ = oracle.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, p.x_cols(c0, c1), p.bias, act=1, want_scale=False)
        parts = [None] * world
        dist.all_gather_object(parts, (c0, c1, Y))
        # unfused Y all-gather (gather.nccl_gather; gloo here): every rank gets the full M×N Y
        from paper_2101_07948_b200.gather import column_bounds, nccl_gather
        import torch
        Yg = nccl_gather(torch.from_numpy(Y), column_bounds(p.N, world)).numpy()
        Yfull, _ = oracle.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, p.x(), p.bias, act=1, want_scale=False)
        assert np.array_equal(Yg, Yfull)
        q.put((rank, c0, c1, t, same and caught, differ, parts if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def _gather_worker(rank, world, port, N, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2101_07948_b200.gather import column_bounds, nccl_gather
        bounds = column_bounds(N, world)
        c0, c1 = bounds[rank]
        full = torch.arange(5 * N, dtype=torch.float32).reshape(5, N)
        got = nccl_gather(full[:, c0:c1].contiguous(), bounds)
        q.put((rank, bool(torch.equal(got, full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,world", [(10, 3), (9, 2)])
def test_nccl_gather_ragged_shards(N, world):
    """Unequal (and empty) column blocks are padded for the collective and trimmed after."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, N, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok for _, ok in res)


def test_two_rank_gloo(oracle_mod):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (_, a0, a1, t0, s0, d0, parts), (_, b0, b1, t1, s1, d1, _) = res
    assert (a0, a1, b0, b1) == (0, 500, 500, 1000)
    assert t0 == t1 == 2.0
    assert s0 and s1 and not d0 and not d1
    p = synth.make_problem("mr", 300, 200, 1000, 0.9, mask="lognormal", seed=3)
    Yfull, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, p.x(), p.bias, act=1, want_scale=False)
    np.testing.assert_array_equal(np.concatenate([y for _, _, y in parts], 1), Yfull)


@pytest.mark.parametrize("N,world", [(262144, 1), (262144, 8), (1000, 3), (10, 4), (7, 2)])
def test_shard_range_partition(N, world):
    rs = [bench.shard_range(N, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == N
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c and a <= b
    assert all(a % 4 == 0 for a, _ in rs)
