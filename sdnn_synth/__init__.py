"""Seeded synthetic inputs for the sparse-weight SpMM  Y = act(W·X + b).

This module holds ONLY input generation (masks, values, activations, bias).  It contains none of the
method's arithmetic, and it is the one module that both the CPU oracle side (`oracle/`, `tests/`)
and the CUDA product side (`bench.py`, the binding's users) import.

Recipe (SURVEY.md §8(c) readings C11-C16, §8(d) config table):
  * W is M×K, CSR with int32 row_ptr/col_idx (strictly increasing columns per row) and fp32 values.
  * nnz is exact: density d‰ = round(1000·(1−s)); nnz = (d‰·M·K + 500) div 1000        (C11)
  * masks: "uniform" (exact-nnz uniform positions, BASELINE configs[0], [2], [4]);
           "lognormal" (row nnz ∝ exp(z), z~N(0,1), largest-remainder apportioned, capped at K,
                        then uniform columns per row; C14, BASELINE configs[1]);
           "block4" (random 1×4 runs aligned to multiples of 4 along K; C15, BASELINE configs[3]);
           "threshold" (the paper's own suite model: unit Gaussian, keep the nnz largest magnitudes,
                        P:173 §4.1; values are the surviving Gaussians).
  * values N(0, 0.05) (σ, C12), exact zeros redrawn (C6); X ~ N(0,1); bias ~ N(0, 0.1).
  * seeds: numpy SeedSequence([seed, crc32(config key), tensor id(, block)]) (C16); X is generated in
    8192-column blocks so any column shard is identical for every GPU count.
"""
from __future__ import annotations

import dataclasses
import zlib

import numpy as np

T_MASK, T_VALS, T_X, T_BIAS = 0, 1, 2, 3
X_BLOCK = 8192

ACT_NONE, ACT_RELU = 0, 1


def density_permille(sparsity: float) -> int:
    d = int(round(1000.0 * (1.0 - float(sparsity))))
    if not (0 <= d <= 1000):
        raise ValueError(f"sparsity {sparsity} outside [0, 1]")
    return d


def nnz_target(M: int, K: int, sparsity: float) -> int:
    """C11: nnz = round((1-s)·M·K), computed in integers with half-up rounding."""
    return (density_permille(sparsity) * M * K + 500) // 1000


def _rng(seed: int, key: str, tensor: int, *extra: int) -> np.random.Generator:
    ss = np.random.SeedSequence([int(seed), zlib.crc32(key.encode()), int(tensor), *[int(e) for e in extra]])
    return np.random.Generator(np.random.PCG64(ss))


def _csr_from_sorted_linear(lin: np.ndarray, M: int, K: int):
    lin = np.sort(lin.astype(np.int64))
    rows = lin // K
    cols = (lin % K).astype(np.int32)
    row_ptr = np.zeros(M + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr.astype(np.int32), cols


def mask_uniform(M, K, nnz, rng):
    lin = rng.choice(M * K, size=nnz, replace=False)
    return _csr_from_sorted_linear(lin, M, K)


def lognormal_row_counts(M, K, nnz, rng, sigma=1.0):
    """C14: row weights s_i = exp(σ z_i); largest-remainder apportionment of nnz, capped at K,
    overflow redistributed over uncapped rows (ties → lowest row)."""
    if nnz > M * K:
        raise ValueError("nnz > M*K")
    s = np.exp(sigma * rng.standard_normal(M))
    counts = np.zeros(M, dtype=np.int64)
    remaining = nnz
    active = np.ones(M, dtype=bool)
    while remaining > 0:
        idx = np.nonzero(active)[0]
        w = s[idx]
        quota = remaining * w / w.sum()
        base = np.floor(quota).astype(np.int64)
        short = remaining - int(base.sum())
        rem = quota - base
        order = np.lexsort((idx, -rem))  # largest remainder first, ties -> lowest row
        base[order[:short]] += 1
        counts[idx] += base
        over = np.maximum(counts - K, 0)
        remaining = int(over.sum())
        counts -= over
        active = counts < K
    return counts


def mask_lognormal(M, K, nnz, rng, sigma=1.0):
    counts = lognormal_row_counts(M, K, nnz, rng, sigma)
    row_ptr = np.zeros(M + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(counts)
    cols = np.empty(nnz, dtype=np.int32)
    for i in range(M):
        c = int(counts[i])
        if c:
            cols[row_ptr[i]:row_ptr[i + 1]] = np.sort(rng.choice(K, size=c, replace=False))
    return row_ptr.astype(np.int32), cols


def mask_block4(M, K, sparsity, rng):
    """C15: round((1-s)·M·K/4) distinct 1×4 runs from the M × K/4 grid of aligned slots."""
    if K % 4:
        raise ValueError("block4 mask needs K % 4 == 0")
    nb = (density_permille(sparsity) * M * (K // 4) + 500) // 1000
    blk = rng.choice(M * (K // 4), size=nb, replace=False)
    r = blk // (K // 4)
    c0 = (blk % (K // 4)) * 4
    lin = (r[:, None] * K + c0[:, None] + np.arange(4)[None, :]).reshape(-1)
    return _csr_from_sorted_linear(lin, M, K)


def weight_values(nnz, rng, sigma=0.05):
    v = (sigma * rng.standard_normal(nnz)).astype(np.float32)
    while True:  # C6: generators never emit explicit zeros
        z = np.nonzero(v == 0)[0]
        if z.size == 0:
            return v
        v[z] = (sigma * rng.standard_normal(z.size)).astype(np.float32)


def threshold_matrix(M, K, nnz, rng):
    """unit-Gaussian dense matrix, values below the magnitude threshold set to zero; the
    threshold is the empirical quantile keeping exactly nnz entries (S:71 reading)."""
    d = rng.standard_normal((M, K)).astype(np.float32)
    flat = np.abs(d).reshape(-1)
    keep = np.argsort(-flat, kind="stable")[:nnz]
    row_ptr, cols = _csr_from_sorted_linear(keep, M, K)
    lin = np.sort(keep)
    return row_ptr, cols, d.reshape(-1)[lin].astype(np.float32)


@dataclasses.dataclass
class Problem:
    name: str
    M: int
    K: int
    N: int
    sparsity: float
    mask: str
    row_ptr: np.ndarray  # int32[M+1]
    col_idx: np.ndarray  # int32[nnz]
    vals: np.ndarray     # float32[nnz]
    bias: np.ndarray | None  # float32[M]
    act: int
    seed: int

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def x_block(self, b: int) -> np.ndarray:
        """Columns [b·X_BLOCK, (b+1)·X_BLOCK) ∩ [0, N) of X (K × width, float32, row-major)."""
        c0 = b * X_BLOCK
        w = min(X_BLOCK, self.N - c0)
        return _rng(self.seed, self.name, T_X, b).standard_normal((self.K, w), dtype=np.float32)

    def x_cols(self, c0: int, c1: int, out: np.ndarray | None = None) -> np.ndarray:
        """X[:, c0:c1] as a contiguous K × (c1-c0) float32 array (block-seeded, shard-invariant)."""
        if out is None:
            out = np.empty((self.K, c1 - c0), dtype=np.float32)
        b0, b1 = c0 // X_BLOCK, (c1 - 1) // X_BLOCK if c1 > c0 else c0 // X_BLOCK - 1
        for b in range(b0, b1 + 1):
            blk = self.x_block(b)
            s0 = max(c0, b * X_BLOCK)
            s1 = min(c1, b * X_BLOCK + blk.shape[1])
            out[:, s0 - c0:s1 - c0] = blk[:, s0 - b * X_BLOCK:s1 - b * X_BLOCK]
        return out

    def x(self) -> np.ndarray:
        return self.x_cols(0, self.N)

    def dense_w(self) -> np.ndarray:
        d = np.zeros((self.M, self.K), dtype=np.float32)
        r = np.repeat(np.arange(self.M), np.diff(self.row_ptr))
        d[r, self.col_idx] = self.vals
        return d


def make_problem(name: str, M: int, K: int, N: int, sparsity: float, mask: str = "uniform",
                 bias: bool = True, act: int = ACT_RELU, seed: int = 0) -> Problem:
    nnz = nnz_target(M, K, sparsity)
    rm = _rng(seed, name, T_MASK)
    if mask == "uniform":
        row_ptr, cols = mask_uniform(M, K, nnz, rm)
        vals = weight_values(nnz, _rng(seed, name, T_VALS))
    elif mask == "lognormal":
        row_ptr, cols = mask_lognormal(M, K, nnz, rm)
        vals = weight_values(nnz, _rng(seed, name, T_VALS))
    elif mask == "block4":
        row_ptr, cols = mask_block4(M, K, sparsity, rm)
        vals = weight_values(int(row_ptr[-1]), _rng(seed, name, T_VALS))
    elif mask == "threshold":
        row_ptr, cols, vals = threshold_matrix(M, K, nnz, rm)
    else:
        raise ValueError(f"unknown mask {mask!r}")
    b = (0.1 * _rng(seed, name, T_BIAS).standard_normal(M)).astype(np.float32) if bias else None
    return Problem(name, M, K, N, float(sparsity), mask, row_ptr.astype(np.int32), cols.astype(np.int32),
                   vals.astype(np.float32), b, act, seed)


# BASELINE.json configs.  key -> (M, K, N, sparsity, mask)
CONFIGS: dict[str, tuple[int, int, int, float, str]] = {
    "c1": (256, 256, 128, 0.90, "uniform"),
    "c2_768x768": (768, 768, 1024, 0.90, "lognormal"),
    "c2_3072x768": (3072, 768, 1024, 0.90, "lognormal"),
    "c2_768x3072": (768, 3072, 1024, 0.90, "lognormal"),
    "c3_128x64": (128, 64, 6272, 0.85, "uniform"),
    "c3_256x128": (256, 128, 6272, 0.85, "uniform"),
    "c3_512x512": (512, 512, 6272, 0.85, "uniform"),
    "c3_1024x512": (1024, 512, 6272, 0.85, "uniform"),
    "c4_2048x512_s80": (2048, 512, 12544, 0.80, "block4"),
    "c4_512x2048_s80": (512, 2048, 12544, 0.80, "block4"),
    "c4_2048x512_s95": (2048, 512, 12544, 0.95, "block4"),
    "c4_512x2048_s95": (512, 2048, 12544, 0.95, "block4"),
    "c5": (4096, 4096, 262144, 0.90, "uniform"),
}


def config_problem(key: str, seed: int = 0, N: int | None = None, act: int = ACT_RELU, bias: bool = True) -> Problem:
    M, K, n, s, mask = CONFIGS[key]
    return make_problem(key, M, K, n if N is None else N, s, mask, bias=bias, act=act, seed=seed)


def desk_grid():
    """S:510 acceptance grid: {64,256,512}² × {0.7,0.8,0.9,0.95} × N∈{32,128} × 3 seeds."""
    for n in (64, 256, 512):
        for s in (0.7, 0.8, 0.9, 0.95):
            for N in (32, 128):
                for seed in range(3):
                    yield dict(name=f"desk_{n}_{int(round(s * 100))}_{N}", M=n, K=n, N=N, sparsity=s, seed=seed)


# ----------------------------------------------------------------------------- sparse convolution
@dataclasses.dataclass
class ConvProblem:
    """Sparse k×k convolution: filters OC×IC×FY×FX stored as
    the CSR of the OC × (IC·FY·FX) matrix (column = (ic·FY + fy)·FX + fx), activations in
    the C×(B·H·W) layout of the 1×1 convs (reading C17): X[ic][b][y][x], Y[oc][b][oy][ox]."""
    name: str
    OC: int
    IC: int
    H: int
    W: int
    B: int
    FY: int
    FX: int
    pad: int
    stride: int
    sparsity: float
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    bias: np.ndarray | None
    act: int
    seed: int

    @property
    def K(self) -> int:
        return self.IC * self.FY * self.FX

    @property
    def Ho(self) -> int:
        return (self.H + 2 * self.pad - self.FY) // self.stride + 1

    @property
    def Wo(self) -> int:
        return (self.W + 2 * self.pad - self.FX) // self.stride + 1

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def x(self) -> np.ndarray:
        """Input activations, float32 [IC][B][H][W], N(0, 1)."""
        return _rng(self.seed, self.name, T_X).standard_normal((self.IC, self.B, self.H, self.W), dtype=np.float32)


def make_conv_problem(name: str, OC: int, IC: int, H: int, W: int, B: int, sparsity: float, FY: int = 3,
                      FX: int = 3, pad: int = 1, stride: int = 1, bias: bool = True, act: int = ACT_RELU,
                      seed: int = 0) -> ConvProblem:
    """The paper's conv suite: random (uniform-mask) sparse filters at 90 / 95 %, IC/OC 32-256,
    images 7/14/28/56, 3×3, pad 1; values N(0, 0.05) like the SpMM weights."""
    K = IC * FY * FX
    nnz = nnz_target(OC, K, sparsity)
    row_ptr, cols = mask_uniform(OC, K, nnz, _rng(seed, name, T_MASK))
    vals = weight_values(nnz, _rng(seed, name, T_VALS))
    b = (0.1 * _rng(seed, name, T_BIAS).standard_normal(OC)).astype(np.float32) if bias else None
    return ConvProblem(name, OC, IC, H, W, B, FY, FX, pad, stride, float(sparsity), row_ptr.astype(np.int32),
                       cols.astype(np.int32), vals.astype(np.float32), b, act, seed)
