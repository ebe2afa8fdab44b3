"""Fused Y all-gather plumbing on one GPU: a one-rank NCCL group, the full Y in
symmetric memory, sdnn_spmm_multi through the peers' buffer addresses + the symmetric-memory
barrier.  The result must equal sdnn_spmm bitwise (same kernel, same per-column order).  The N > 1
exchange itself needs several GPUs; its host logic is covered by tests/test_multirank.py."""
import socket

import pytest
import torch

import sdnn_synth as synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def one_rank_group():
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["peer", "auto"])
@pytest.mark.parametrize("kernel", ["auto", "row", "tmem"])
@pytest.mark.parametrize("key", ["c2_768x768", "c1"])
def test_fused_gather_one_rank(one_rank_group, sdnn, kernel, key, mode):
    """Both store paths of the fused gather (per-peer sdnn_spmm_multi; multicast sdnn_spmm_multicast
    where the one-rank group has a multicast address — `auto` reports which it took) give sdnn_spmm's
    Y bitwise."""
    from paper_2101_07948_b200.gather import FusedGather, column_bounds
    p = synth.config_problem(key)
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    X = torch.from_numpy(p.x()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    ref = h.spmm(X, b, act=1)
    fg = FusedGather(p.M, p.N, column_bounds(p.N, 1), mode=mode)
    print(f"fused gather mode={mode} -> {fg.mode}")
    fg.Y.fill_(float("nan"))
    Y = fg.spmm(h, X, b, act=1)
    torch.cuda.synchronize()
    assert torch.equal(Y, ref)
    with pytest.raises(ValueError):
        fg.spmm(h, X[:, :-4].contiguous(), b, act=1)


def test_multicast_entry_errors(sdnn):
    """sdnn_spmm_multicast rejects a NULL multicast address and bad column windows before launching
    (a multimem.st to an address that is not a multicast object is undefined, so none is issued)."""
    p = synth.config_problem("c1")
    h = sdnn.Handle.from_problem(p)
    X = torch.from_numpy(p.x()).cuda()
    with pytest.raises(sdnn.SdnnError) as e:
        h.spmm_multicast(X, 0, ldy=p.N, col0=0)
    assert e.value.status == 1
    Y = torch.empty((p.M, p.N), device="cuda")
    with pytest.raises(sdnn.SdnnError):
        h.spmm_multicast(X, Y.data_ptr(), ldy=p.N - 4, col0=0)  # ldy < col0 + N
    with pytest.raises(sdnn.SdnnError):
        sdnn.Handle.from_problem(p, kernel="codegen").spmm_multicast(X, Y.data_ptr(), ldy=p.N, col0=0)
