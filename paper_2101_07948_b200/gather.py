"""Optional Y all-gather across ranks (collective 2): every rank ends with the full M×N Y.

The SpMM shards along N with no exchange (column independence, P5): rank r owns columns
[c0_r, c1_r) of X and Y.  When every rank needs the whole Y (e.g. the next layer is sharded
differently), two forms:

* ``FusedGather`` — the B200 form.  Y lives in a symmetric-memory buffer (one M×N row-major copy per
  rank, mapped into every peer's address space over NVLink).  Where the group has an NVLink SHARP
  multicast address (``has_multicast_support``), ``sdnn_spmm_multicast`` stores each float4 of the
  rank's shard once with ``multimem.st.global.v4.f32`` and NVSwitch replicates it into every rank's
  Y; otherwise ``sdnn_spmm_multi`` is given all ranks' buffer addresses and stores every float4 to
  each of them.  Either way leading dimension N and column offset c0_r place the shard, the stores
  happen in the epilogue while later row panels are still computing — the transfer overlaps the FMA
  loop tile by tile, there is no separate collective kernel and no [g][M][N/g] → M×N permute-copy.
  Symmetric-memory barriers before (no peer still reading the previous Y) and after the kernel.
* ``nccl_gather`` — the unfused baseline: ``sdnn_spmm`` into the local shard, then an all-gather of
  the (padded) shards and a column concatenation.  Also the path for groups without symmetric memory
  (gloo on CPU in the tests).

Host logic only: every byte of Y is computed by the CUDA kernels behind the C ABI.
"""
from __future__ import annotations


def column_bounds(N: int, world: int) -> list[tuple[int, int]]:
    """Contiguous column block per rank: every shard but the last has ⌊N/g⌋ rounded down to a
    multiple of 4 columns (so each starts 16-B aligned in a row of X or Y); the last takes the rest."""
    if world < 1 or N < 0:
        raise ValueError("need world >= 1 and N >= 0")
    base = (N // world) // 4 * 4
    starts = [r * base for r in range(world)] + [N]
    return [(starts[r], starts[r + 1]) for r in range(world)]


def nccl_gather(Y_shard, bounds, group=None):
    """All-gather the column shards (M × (c1_r − c0_r) each, rank order) into one M×N tensor.
    Unequal widths are padded to the widest shard for the collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist

    world = len(bounds)
    widths = [b - a for a, b in bounds]
    wmax = max(widths)
    M = Y_shard.shape[0]
    send = Y_shard
    if Y_shard.shape[1] != wmax:
        send = torch.zeros((M, wmax), dtype=Y_shard.dtype, device=Y_shard.device)
        send[:, :Y_shard.shape[1]] = Y_shard
    parts = [torch.empty((M, wmax), dtype=Y_shard.dtype, device=Y_shard.device) for _ in range(world)]
    dist.all_gather(parts, send.contiguous(), group=group)
    return torch.cat([parts[r][:, :widths[r]] for r in range(world)], dim=1)


def gather_mode(requested: str, has_multicast: bool, multicast_ptr: int) -> str:
    """Store path of the fused gather: "multicast" (one multimem.st per element through the group's
    NVLink SHARP multicast address; NVSwitch writes every rank's buffer) when the symmetric-memory
    handle supports it, else "peer" (the epilogue stores every element to each rank's buffer over
    NVLink).  `requested` is "auto", "multicast" (an error without support) or "peer"."""
    if requested not in ("auto", "multicast", "peer"):
        raise ValueError("mode must be auto, multicast or peer")
    mc = bool(has_multicast) and int(multicast_ptr or 0) != 0
    if requested == "multicast" and not mc:
        raise RuntimeError("multicast requested but the symmetric-memory handle has no multicast address")
    if requested == "peer":
        return "peer"
    return "multicast" if mc else "peer"


class FusedGather:
    """Full-Y symmetric-memory buffer for a group; ``spmm`` runs the rank's shard with the
    all-gather fused into the epilogue (see the module docstring)."""

    def __init__(self, M: int, N: int, bounds, group=None, device=None, mode: str = "auto"):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if len(bounds) != self.world:
            raise ValueError("one column block per rank")
        if self.world > 8:
            raise ValueError("sdnn_spmm_multi writes at most 8 destinations")
        self.M, self.N, self.bounds = M, N, list(bounds)
        if self.bounds[0][0] != 0 or self.bounds[-1][1] != N or any(
                b != c for (_, b), (c, _) in zip(self.bounds, self.bounds[1:])):
            raise ValueError("column blocks must tile [0, N)")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.Y = symm_mem.empty((M, N), dtype=torch.float32, device=dev)
        self._hdl = symm_mem.rendezvous(self.Y, self.group)
        self.ptrs = [int(self._hdl.buffer_ptrs[r]) for r in range(self.world)]
        try:
            has_mc = bool(self._hdl.has_multicast_support())
            mc_ptr = int(self._hdl.multicast_ptr) if has_mc else 0
        except Exception:  # older symmetric-memory builds: no multicast attributes
            has_mc, mc_ptr = False, 0
        self.mode = gather_mode(mode, has_mc, mc_ptr)
        self.mc_ptr = mc_ptr

    def spmm(self, h, X, bias=None, act="relu", stream=None):
        """Y[:, c0:c1] = act(W·X + b) on every rank's copy of Y: a barrier first (no rank may still be
        reading the previous Y when the peers' stores arrive), the kernel storing through the multicast
        address or to every peer, then a barrier so that on return (stream order) this rank's Y holds
        every rank's columns.  Both barriers run on `stream` (default: the current stream)."""
        import contextlib

        import torch
        c0, c1 = self.bounds[self.rank]
        if X.shape[1] != c1 - c0:
            raise ValueError(f"X shard has {X.shape[1]} columns, rank {self.rank} owns {c1 - c0}")
        ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            self._hdl.barrier(channel=0)
            if self.mode == "multicast":
                h.spmm_multicast(X, self.mc_ptr, ldy=self.N, col0=c0, bias=bias, act=act, stream=stream)
            else:
                h.spmm_multi(X, self.ptrs, ldy=self.N, col0=c0, bias=bias, act=act, stream=stream)
            self._hdl.barrier(channel=0)
        return self.Y
