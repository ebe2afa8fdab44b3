"""paper_2101_07948_b200 — thin Python binding of libsdnn (include/sdnn.h).

Argument marshalling only: every step of the hot path (Algorithm 1, packing, the SpMM kernel, the
fused epilogue) runs inside libsdnn.so.  PyTorch supplies device memory and streams.  There is no
CPU fallback: if the in-tree library is missing this module raises on import; build it with
`python paper_2101_07948_b200/build.py` or `__graft_entry__.build()`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsdnn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsdnn.so not built at {LIB_PATH}; run `python paper_2101_07948_b200/build.py`")

_lib = ctypes.CDLL(LIB_PATH)

ACT_NONE, ACT_RELU = 0, 1
STATUS = {0: "SDNN_OK", 1: "SDNN_ERR_INVALID_ARGUMENT", 2: "SDNN_ERR_INVALID_CSR", 3: "SDNN_ERR_UNSUPPORTED",
          4: "SDNN_ERR_OUT_OF_MEMORY", 5: "SDNN_ERR_CUDA", 6: "SDNN_ERR_DEVICE_MISMATCH", 7: "SDNN_ERR_INTERNAL"}

# exported symbols (must match include/sdnn.h; checked by tests/test_abi.py)
EXPORTS = ["sdnn_prepare", "sdnn_destroy", "sdnn_spmm", "sdnn_spmm_multi", "sdnn_spmm_multicast", "sdnn_conv2d", "sdnn_serialize", "sdnn_tune", "sdnn_conv2d_tune",
           "sdnn_deserialize", "sdnn_spmm_host", "sdnn_spmm_kernel",
           "sdnn_get_permutation",
           "sdnn_get_info",
           "sdnn_permutation", "sdnn_csr_permute_columns", "sdnn_plan_create", "sdnn_plan_get_info", "sdnn_plan_export", "sdnn_plan_export_pieces",
           "sdnn_plan_destroy",
           "sdnn_plan_codegen_ptx", "sdnn_status_string", "sdnn_last_error_message", "sdnn_abi_version"]


class SdnnError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.sdnn_last_error_message().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class PermOpts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("permute", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("panel_rows_max", ctypes.c_int32),
                ("cta_panels", ctypes.c_int32), ("k_chunk", ctypes.c_int32), ("group_sb", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class Info(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("M", ctypes.c_int32), ("K", ctypes.c_int32),
                ("nnz", ctypes.c_int64), ("device", ctypes.c_int32), ("permuted", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("group_entries_per_nnz_x1000", ctypes.c_int32),
                ("group_sb", ctypes.c_int32), ("group_subblocks_per_nnz_x1000", ctypes.c_int32),
                ("panel_rows", ctypes.c_int32), ("cta_panels", ctypes.c_int32), ("num_panels", ctypes.c_int32),
                ("num_row_blocks", ctypes.c_int32), ("k_chunk", ctypes.c_int32), ("num_chunks", ctypes.c_int32),
                ("meta_bytes", ctypes.c_int64), ("max_block_bytes", ctypes.c_int32), ("alt_kernel", ctypes.c_int32),
                ("max_panel_nnz", ctypes.c_int64), ("num_split_rows", ctypes.c_int32), ("num_pieces", ctypes.c_int32),
                ("narrow_row_blocks", ctypes.c_int32), ("narrow4_row_blocks", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "struct_size"}


_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib.sdnn_prepare.argtypes = [_vp, _vp, _vp, _i32, _i32, ctypes.POINTER(PermOpts), ctypes.POINTER(_vp)]
_lib.sdnn_destroy.argtypes = [_vp]
_lib.sdnn_spmm.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _vp]
_lib.sdnn_spmm_multi.argtypes = [_vp, _vp, _i64, _vp, _i32, ctypes.POINTER(_vp), _i32, _i64, _i64, _vp]
_lib.sdnn_spmm_multicast.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _i64, _i64, _vp]
_lib.sdnn_spmm_host.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _i64]
_lib.sdnn_get_permutation.argtypes = [_vp, _vp]
_lib.sdnn_spmm_kernel.argtypes = [_vp, _i64, _vp, _vp, ctypes.POINTER(_i32)]
_lib.sdnn_get_info.argtypes = [_vp, ctypes.POINTER(Info)]
_lib.sdnn_permutation.argtypes = [_vp, _vp, _i32, _i32, _vp]
_lib.sdnn_csr_permute_columns.argtypes = [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]
_lib.sdnn_conv2d_tune.argtypes = [_vp, _vp] + [_i32] * 8 + [_vp, _vp, ctypes.POINTER(_i32), ctypes.POINTER(ctypes.c_float)]
_lib.sdnn_tune.argtypes = [_vp, _vp, _i64, _vp, _vp, ctypes.POINTER(_i32), ctypes.POINTER(ctypes.c_float)]
_lib.sdnn_serialize.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_size_t)]
_lib.sdnn_deserialize.argtypes = [_vp, ctypes.c_size_t, ctypes.POINTER(_vp)]
_lib.sdnn_conv2d.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp]
_lib.sdnn_plan_create.argtypes = [_vp, _vp, _vp, _i32, _i32, ctypes.POINTER(PermOpts), ctypes.POINTER(_vp)]
_lib.sdnn_plan_get_info.argtypes = [_vp, ctypes.POINTER(Info)]
_lib.sdnn_plan_export.argtypes = [_vp, _vp, _vp, _vp]
_lib.sdnn_plan_export_pieces.argtypes = [_vp, _vp, _vp, _vp]
_lib.sdnn_plan_destroy.argtypes = [_vp]
_lib.sdnn_plan_codegen_ptx.argtypes = [_vp, _vp, _vp, _vp, _i32, _vp, ctypes.POINTER(_i64)]
_lib.sdnn_status_string.restype = ctypes.c_char_p
_lib.sdnn_last_error_message.restype = ctypes.c_char_p
_lib.sdnn_abi_version.restype = ctypes.c_int32
for _f in EXPORTS:
    if _f not in ("sdnn_status_string", "sdnn_last_error_message", "sdnn_abi_version"):
        getattr(_lib, _f).restype = ctypes.c_int


def _check(st: int, where: str):
    if st != 0:
        raise SdnnError(st, where)


def _np_ptr(a):
    return None if a is None else a.ctypes.data


def _csr(row_ptr, col_idx, vals):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.float32)
    return rp, ci, v


KERNELS = {"auto": 0, "row": 1, "group": 2, "codegen": 3, "tmem": 4, "tmem8": 5, "tmemp": 6}


FLAG_NO_ROW_SPLIT = 1
FLAG_PERMUTED_OUTPUT = 2
FLAG_NO_SPLIT_K = 4


def _opts(permute=True, kernel="auto", panel_rows=0, cta_panels=0, k_chunk=0, group_sb=0, split_rows=True,
          permuted_output=False, split_k=True):
    k = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    flags = ((0 if split_rows else FLAG_NO_ROW_SPLIT) | (FLAG_PERMUTED_OUTPUT if permuted_output else 0)
             | (0 if split_k else FLAG_NO_SPLIT_K))
    return PermOpts(ctypes.sizeof(PermOpts), int(bool(permute)), k, int(panel_rows), int(cta_panels), int(k_chunk),
                    int(group_sb), flags)


def _act(act) -> int:
    if isinstance(act, str):
        return {"none": ACT_NONE, "relu": ACT_RELU}[act.lower()]
    return int(act)


def permutation(row_ptr, col_idx, M: int, K: int) -> np.ndarray:
    """Algorithm 1 on host via libsdnn (no GPU needed)."""
    rp, ci, _ = _csr(row_ptr, col_idx, None)
    order = np.empty(M, dtype=np.int32)
    _check(_lib.sdnn_permutation(_np_ptr(rp), _np_ptr(ci), M, K, _np_ptr(order)), "sdnn_permutation")
    return order


def permute_columns(row_ptr, col_idx, vals, M: int, K: int, order) -> tuple[np.ndarray, np.ndarray]:
    """CSR of W·P (sdnn_csr_permute_columns): column order[i] moves to position i, rows re-sorted.
    Returns (col_idx', vals'); row_ptr is unchanged."""
    rp, ci, v = _csr(row_ptr, col_idx, vals)
    order = np.ascontiguousarray(order, dtype=np.int32)
    if order.shape != (K,):
        raise ValueError("order must have K entries")
    oc = np.empty_like(ci)
    ov = np.empty_like(v)
    _check(_lib.sdnn_csr_permute_columns(_np_ptr(rp), _np_ptr(ci), _np_ptr(v), M, K, _np_ptr(order), _np_ptr(oc),
                                         _np_ptr(ov)), "sdnn_csr_permute_columns")
    return oc, ov


class Plan:
    """Host-only plan (sdnn_plan_*): the prepared execution-ordered format without a device."""

    def __init__(self, row_ptr, col_idx, vals, M: int, K: int, **opts):
        rp, ci, v = _csr(row_ptr, col_idx, vals)
        h = _vp()
        o = _opts(**opts)
        _check(_lib.sdnn_plan_create(_np_ptr(rp), _np_ptr(ci), _np_ptr(v), M, K, ctypes.byref(o), ctypes.byref(h)),
               "sdnn_plan_create")
        self._h = h

    def info(self) -> dict:
        i = Info()
        i.struct_size = ctypes.sizeof(Info)
        _check(_lib.sdnn_plan_get_info(self._h, ctypes.byref(i)), "sdnn_plan_get_info")
        return i.as_dict()

    def codegen_ptx(self, row_ptr, col_idx, vals, panel: int) -> str:
        """Generated PTX of one codegen panel (plan created with kernel="codegen")."""
        rp, ci, v = _csr(row_ptr, col_idx, vals)
        n = _i64(0)
        _check(_lib.sdnn_plan_codegen_ptx(self._h, _np_ptr(rp), _np_ptr(ci), _np_ptr(v), panel, None, ctypes.byref(n)),
               "sdnn_plan_codegen_ptx")
        buf = ctypes.create_string_buffer(n.value)
        _check(_lib.sdnn_plan_codegen_ptx(self._h, _np_ptr(rp), _np_ptr(ci), _np_ptr(v), panel, buf, ctypes.byref(n)),
               "sdnn_plan_codegen_ptx")
        return buf.value.decode()

    def export_pieces(self):
        """Split rows of a row plan: (row, begin, end) per piece (CSR entry ranges)."""
        n = self.info()["num_pieces"]
        row, begin, end = (np.empty(n, np.int32) for _ in range(3))
        _check(_lib.sdnn_plan_export_pieces(self._h, _np_ptr(row), _np_ptr(begin), _np_ptr(end)), "sdnn_plan_export_pieces")
        return row, begin, end

    def export(self):
        i = self.info()
        row_orig = np.empty(i["num_panels"] * i["panel_rows"], np.int32)
        blk_off = np.empty(i["num_row_blocks"] * i["num_chunks"] + 1, np.int64)
        meta = np.empty(i["meta_bytes"], np.uint8)
        _check(_lib.sdnn_plan_export(self._h, _np_ptr(row_orig), _np_ptr(blk_off), _np_ptr(meta)), "sdnn_plan_export")
        return row_orig, blk_off, meta

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.sdnn_plan_destroy(self._h)
            self._h = None


class Handle:
    """sdnn_prepare on the current CUDA device; .spmm runs the kernel on torch CUDA tensors."""

    def __init__(self, row_ptr, col_idx, vals, M: int, K: int, **opts):
        rp, ci, v = _csr(row_ptr, col_idx, vals)
        self.M, self.K = int(M), int(K)
        h = _vp()
        o = _opts(**opts)
        _check(_lib.sdnn_prepare(_np_ptr(rp), _np_ptr(ci), _np_ptr(v), M, K, ctypes.byref(o), ctypes.byref(h)),
               "sdnn_prepare")
        self._h = h

    @classmethod
    def from_problem(cls, p, **opts):
        return cls(p.row_ptr, p.col_idx, p.vals, p.M, p.K, **opts)

    @classmethod
    def for_conv(cls, row_ptr, col_idx, vals, OC: int, IC: int, FY: int, FX: int, **opts):
        """A handle for sdnn_conv2d: filters as the OC × (IC·FY·FX) CSR, no split rows, and K chunks of
        whole input channels when a multiple of FY·FX fits the chunk rules (72 for 3×3: 8-12 % faster,
        profiles/r01_conv_kchunk.log), and 8 panels per CTA from 64 output channels up: taller CTAs
        stage each input patch for more filters (graph-timed, profiles/r01_conv_cta.log: 256 channels
        at 56 px 483 → 393 µs, 128 at 14 px 21 → 19 µs; 64 at 28 px 3 % slower)."""
        import math
        fyx = FY * FX
        kc = fyx * 8 // math.gcd(fyx, 8)  # lcm(FY·FX, 8)
        opts.setdefault("k_chunk", kc if kc <= 128 and IC * fyx >= 2 * kc else 0)
        if OC >= 64 and not opts.get("panel_rows") and not opts.get("cta_panels"):
            opts["cta_panels"] = 8
        opts.setdefault("split_rows", False)
        try:
            return cls(row_ptr, col_idx, vals, OC, IC * fyx, **opts)
        except SdnnError as e:
            # a whole-channel chunk that does not fit the stage ring (e.g. 3×5 filters: 120 columns): the
            # library's own chunk choice instead
            if e.status != 3 or not opts.get("k_chunk") or opts["k_chunk"] != kc:
                raise
            opts["k_chunk"] = 0
            return cls(row_ptr, col_idx, vals, OC, IC * fyx, **opts)

    def conv2d_tune(self, X, FY: int = 3, FX: int = 3, pad: int = 1, stride: int = 1, stream=None) -> dict:
        """sdnn_conv2d_tune for X's geometry: {"pixels": 2 | 4 | 0 (rules) | -2 (explicit form: virtual
        operand written out + TMEM-R SpMM), "split_k": slices, "us": µs}."""
        import torch
        IC, B, H, W = X.shape
        Ho, Wo = (H + 2 * pad - FY) // stride + 1, (W + 2 * pad - FX) // stride + 1
        out = torch.empty((self.M, B, Ho, Wo), dtype=torch.float32, device=X.device)
        s = torch.cuda.current_stream(X.device) if stream is None else stream
        ch, us = _i32(0), ctypes.c_float(0)
        _check(_lib.sdnn_conv2d_tune(self._h, X.data_ptr(), B, IC, H, W, FY, FX, pad, stride, out.data_ptr(),
                                     s.cuda_stream, ctypes.byref(ch), ctypes.byref(us)), "sdnn_conv2d_tune")
        if ch.value == -2:  # the explicit form (virtual operand written out, TMEM-R SpMM)
            return {"pixels": -2, "split_k": 0, "us": us.value}
        if ch.value < 0:
            return {"pixels": 0, "split_k": 0, "us": us.value}
        return {"pixels": ch.value // 16, "split_k": ch.value % 16, "us": us.value}

    def tune(self, X, out=None, stream=None) -> dict:
        """sdnn_tune: measure every path for X's N and keep the fastest for later calls with that N.
        Returns {"path": "tmem" | "row" | "narrow" | "narrow4", "split_k": slices, "us": µs per call}."""
        import torch
        if X.dim() != 2 or X.shape[0] != self.K or X.dtype != torch.float32 or not X.is_cuda or not X.is_contiguous():
            raise ValueError(f"X must be a contiguous CUDA float32 tensor of shape ({self.K}, N)")
        N = X.shape[1]
        if out is None:
            out = torch.empty((self.M, N), dtype=torch.float32, device=X.device)
        s = torch.cuda.current_stream(X.device) if stream is None else stream
        path, us = _i32(0), ctypes.c_float(0)
        _check(_lib.sdnn_tune(self._h, X.data_ptr(), N, out.data_ptr(), s.cuda_stream, ctypes.byref(path),
                              ctypes.byref(us)), "sdnn_tune")
        if path.value < 0:
            return {"path": "auto", "split_k": 0, "us": us.value}
        return {"path": ("tmem", "row", "narrow", "narrow4")[path.value // 16], "split_k": path.value % 16, "us": us.value}

    def serialize(self) -> bytes:
        """The prepared handle as a blob (sdnn_serialize): reload with Handle.deserialize."""
        n = ctypes.c_size_t(0)
        _check(_lib.sdnn_serialize(self._h, None, ctypes.byref(n)), "sdnn_serialize")
        buf = ctypes.create_string_buffer(n.value)
        _check(_lib.sdnn_serialize(self._h, buf, ctypes.byref(n)), "sdnn_serialize")
        return buf.raw[:n.value]

    @classmethod
    def deserialize(cls, blob: bytes) -> "Handle":
        """A handle from sdnn_serialize's blob, on the current CUDA device (no Algorithm 1, no packing)."""
        h = _vp()
        _check(_lib.sdnn_deserialize(blob, len(blob), ctypes.byref(h)), "sdnn_deserialize")
        self = cls.__new__(cls)
        self._h = h
        i = self.info()
        self.M, self.K = i["M"], i["K"]
        return self

    def info(self) -> dict:
        i = Info()
        i.struct_size = ctypes.sizeof(Info)
        _check(_lib.sdnn_get_info(self._h, ctypes.byref(i)), "sdnn_get_info")
        return i.as_dict()

    def kernel_for(self, N: int, x_ptr: int = 0, y_ptr: int = 0) -> int:
        """Kernel id sdnn_spmm launches for N columns at these X/Y addresses (negative = generic)."""
        k = _i32(0)
        _check(_lib.sdnn_spmm_kernel(self._h, int(N), x_ptr or None, y_ptr or None, ctypes.byref(k)), "sdnn_spmm_kernel")
        return k.value

    def permutation(self) -> np.ndarray:
        out = np.empty(self.M, np.int32)
        _check(_lib.sdnn_get_permutation(self._h, _np_ptr(out)), "sdnn_get_permutation")
        return out

    def spmm(self, X, bias=None, act="relu", out=None, stream=None):
        """Y = act(W·X + b) for a CUDA float32 K×N tensor X (row-major contiguous)."""
        import torch
        if X.dim() != 2 or X.shape[0] != self.K or X.dtype != torch.float32 or not X.is_cuda:
            raise ValueError(f"X must be a CUDA float32 tensor of shape ({self.K}, N)")
        if not X.is_contiguous():
            raise ValueError("X must be contiguous (row-major K×N)")
        N = X.shape[1]
        if out is None:
            out = torch.empty((self.M, N), dtype=torch.float32, device=X.device)
        elif out.shape != (self.M, N) or out.dtype != torch.float32 or not out.is_contiguous():
            raise ValueError("out must be a contiguous float32 (M, N) tensor")
        if bias is not None and (bias.numel() != self.M or bias.dtype != torch.float32 or not bias.is_cuda
                                 or not bias.is_contiguous()):
            raise ValueError("bias must be a contiguous CUDA float32 tensor of M elements")
        s = torch.cuda.current_stream(X.device) if stream is None else stream
        _check(_lib.sdnn_spmm(self._h, X.data_ptr(), N, None if bias is None else bias.data_ptr(), _act(act),
                              out.data_ptr(), s.cuda_stream), "sdnn_spmm")
        return out

    def conv2d(self, X, FY: int = 3, FX: int = 3, pad: int = 1, stride: int = 1, bias=None, act="relu", out=None,
               stream=None):
        """Sparse convolution (sdnn_conv2d): X CUDA float32 [IC][B][H][W] → [OC][B][Ho][Wo]; the handle
        holds the filters as the OC × (IC·FY·FX) CSR (prepare with split_rows=False)."""
        import torch
        if X.dim() != 4 or X.dtype != torch.float32 or not X.is_cuda or not X.is_contiguous():
            raise ValueError("X must be a contiguous CUDA float32 [IC][B][H][W] tensor")
        IC, B, H, W = X.shape
        Ho, Wo = (H + 2 * pad - FY) // stride + 1, (W + 2 * pad - FX) // stride + 1
        if out is None:
            out = torch.empty((self.M, B, Ho, Wo), dtype=torch.float32, device=X.device)
        elif out.shape != (self.M, B, Ho, Wo) or out.dtype != torch.float32 or not out.is_contiguous():
            raise ValueError("out must be a contiguous float32 [OC][B][Ho][Wo] tensor")
        if bias is not None and (bias.numel() != self.M or bias.dtype != torch.float32 or not bias.is_cuda):
            raise ValueError("bias must be a CUDA float32 tensor of OC elements")
        s = torch.cuda.current_stream(X.device) if stream is None else stream
        _check(_lib.sdnn_conv2d(self._h, X.data_ptr(), B, IC, H, W, FY, FX, pad, stride,
                                None if bias is None else bias.data_ptr(), _act(act), out.data_ptr(), s.cuda_stream),
               "sdnn_conv2d")
        return out

    def spmm_multi(self, X, dst_ptrs, ldy: int, col0: int, bias=None, act="relu", stream=None):
        """Y = act(W·X + b) into every destination (device addresses, e.g. peers' symmetric-memory
        buffers), each M×ldy row-major, columns [col0, col0 + N) — sdnn_spmm_multi."""
        import torch
        if X.dim() != 2 or X.shape[0] != self.K or X.dtype != torch.float32 or not X.is_cuda or not X.is_contiguous():
            raise ValueError(f"X must be a contiguous CUDA float32 tensor of shape ({self.K}, N)")
        if bias is not None and (bias.numel() != self.M or bias.dtype != torch.float32 or not bias.is_cuda):
            raise ValueError("bias must be a CUDA float32 tensor of M elements")
        arr = (_vp * len(dst_ptrs))(*[int(d) for d in dst_ptrs])
        s = torch.cuda.current_stream(X.device) if stream is None else stream
        _check(_lib.sdnn_spmm_multi(self._h, X.data_ptr(), X.shape[1], None if bias is None else bias.data_ptr(),
                                    _act(act), arr, len(dst_ptrs), int(ldy), int(col0), s.cuda_stream),
               "sdnn_spmm_multi")

    def spmm_multicast(self, X, mc_ptr: int, ldy: int, col0: int, bias=None, act="relu", stream=None):
        """Y = act(W·X + b) stored once through a multicast address (multimem.st; NVSwitch writes every
        rank's buffer), M×ldy row-major, columns [col0, col0 + N) — sdnn_spmm_multicast."""
        import torch
        if X.dim() != 2 or X.shape[0] != self.K or X.dtype != torch.float32 or not X.is_cuda or not X.is_contiguous():
            raise ValueError(f"X must be a contiguous CUDA float32 tensor of shape ({self.K}, N)")
        if bias is not None and (bias.numel() != self.M or bias.dtype != torch.float32 or not bias.is_cuda):
            raise ValueError("bias must be a CUDA float32 tensor of M elements")
        s = torch.cuda.current_stream(X.device) if stream is None else stream
        _check(_lib.sdnn_spmm_multicast(self._h, X.data_ptr(), X.shape[1], None if bias is None else bias.data_ptr(),
                                        _act(act), int(mc_ptr), int(ldy), int(col0), s.cuda_stream),
               "sdnn_spmm_multicast")

    def spmm_host(self, X: np.ndarray, bias: np.ndarray | None = None, act="relu", out: np.ndarray | None = None,
                  block_cols: int = 0):
        """The same operation on host arrays (sdnn_spmm_host); synchronous."""
        if X.dtype != np.float32 or X.ndim != 2 or X.shape[0] != self.K or not X.flags.c_contiguous:
            raise ValueError("X must be a C-contiguous float32 (K, N) array")
        N = X.shape[1]
        if out is None:
            out = np.empty((self.M, N), np.float32)
        if out.dtype != np.float32 or out.shape != (self.M, N) or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 (M, N) array")
        if bias is not None:
            bias = np.ascontiguousarray(bias, dtype=np.float32)
        _check(_lib.sdnn_spmm_host(self._h, X.ctypes.data, N, _np_ptr(bias), _act(act), out.ctypes.data,
                                   int(block_cols)), "sdnn_spmm_host")
        return out

    def spmm_host_ptr(self, x_ptr: int, N: int, bias_ptr, act, y_ptr: int, block_cols: int = 0):
        """sdnn_spmm_host on raw host pointers (e.g. pinned torch CPU tensors)."""
        _check(_lib.sdnn_spmm_host(self._h, x_ptr, N, bias_ptr, _act(act), y_ptr, int(block_cols)), "sdnn_spmm_host")

    def close(self):
        if getattr(self, "_h", None):
            try:
                _lib.sdnn_destroy(self._h)
            except (AttributeError, TypeError):  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    def __del__(self):
        self.close()


def abi_version() -> int:
    return _lib.sdnn_abi_version()


class Chain:
    """Layers Y_{l+1} = act_l(W_l·Y_l + b_l) run back to back.

    Every layer but the last is prepared with SDNN_FLAG_PERMUTED_OUTPUT, so its output rows stay in
    that layer's Algorithm 1 order and nothing is un-permuted between layers; the next layer's
    columns are relabelled the same way at preparation (sdnn_csr_permute_columns), and its bias is
    taken in its own plan order.  The last layer writes the original row order.  Intermediates are
    preallocated per N and reused (the GPU form of the paper's buffer reuse; at the BERT FFN shapes
    they stay in the 126 MB L2).  layers: [(row_ptr, col_idx, vals, M, K, bias | None, act), ...].
    """

    def __init__(self, layers, **opts):
        import torch
        self.handles, self.biases, self.acts = [], [], []
        prev_order, prev_M = None, None
        for i, (rp, ci, v, M, K, bias, act) in enumerate(layers):
            if prev_M is not None and K != prev_M:
                raise ValueError(f"layer {i}: K = {K} but the previous layer has M = {prev_M}")
            if prev_order is not None:
                ci, v = permute_columns(rp, ci, v, M, K, prev_order)
            last = i == len(layers) - 1
            h = Handle(rp, ci, v, M, K, permuted_output=not last, **opts)
            order = h.permutation()
            b = None
            if bias is not None:
                b = np.ascontiguousarray(np.asarray(bias, np.float32) if last else np.asarray(bias, np.float32)[order])
                b = torch.from_numpy(b).cuda()
            self.handles.append(h)
            self.biases.append(b)
            self.acts.append(act)
            prev_order, prev_M = order, M
        self.K = layers[0][4]
        self.M = layers[-1][3]
        self._bufs = {}

    def forward(self, X, out=None, stream=None):
        """X: CUDA float32 (K_0, N); returns the last layer's (M_L, N) output in original row order."""
        import torch
        N = X.shape[1]
        bufs = self._bufs.get(N)
        if bufs is None:
            bufs = [torch.empty((h.M, N), dtype=torch.float32, device=X.device) for h in self.handles[:-1]]
            self._bufs = {N: bufs}
        cur = X
        for i, h in enumerate(self.handles):
            last = i == len(self.handles) - 1
            dst = out if last else bufs[i]
            cur = h.spmm(cur, self.biases[i], act=self.acts[i], out=dst, stream=stream)
        return cur

