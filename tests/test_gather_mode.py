"""Store-path selection of the fused Y all-gather: NVLink SHARP multicast
(sdnn_spmm_multicast, one multimem.st per element) when the symmetric-memory handle has a multicast
address, else per-peer stores (sdnn_spmm_multi).  Host logic only."""
import pytest

from paper_2101_07948_b200.gather import gather_mode


@pytest.mark.parametrize("requested,has_mc,ptr,expect", [
    ("auto", True, 0x7f0000000000, "multicast"),
    ("auto", True, 0, "peer"),          # support flag without an address: no multicast object
    ("auto", False, 0x7f0000000000, "peer"),
    ("auto", False, 0, "peer"),
    ("peer", True, 0x7f0000000000, "peer"),
    ("multicast", True, 0x7f0000000000, "multicast"),
])
def test_gather_mode(requested, has_mc, ptr, expect):
    assert gather_mode(requested, has_mc, ptr) == expect


def test_gather_mode_errors():
    with pytest.raises(RuntimeError):
        gather_mode("multicast", False, 0)
    with pytest.raises(ValueError):
        gather_mode("nvshmem", True, 1)
