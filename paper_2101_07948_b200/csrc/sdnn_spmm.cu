// sdnn_spmm.cu — device side of libsdnn for B200 (sm_100a): upload of the prepared plan
// (sdnn_prepare), the SpMM kernels and their launch (sdnn_spmm, sdnn_spmm_host).
//
// Kernel: one CTA owns a row block of W_c warp panels (R_w permuted rows each)
// and one N tile of TN = 32·V columns.  A producer warp streams the reduction dimension in chunks of
// KC rows ("split-K" tiling along the reduction dimension): per chunk one TMA tile
// load of X[k0:k0+KC, n0:n0+TN] plus one bulk copy of the chunk's execution-ordered metadata block
// into a ring of shared-memory stages, completed on an mbarrier.  Each consumer warp then,
// for every nonzero of its rows in the chunk, broadcasts the weight and FMAs it with the X row slice
// read from shared memory into statically indexed accumulator registers (the SpMM microkernel of
// P:135 fig:spmm / P:139 §3.2.2), in ascending column order.  The fused epilogue adds the bias,
// applies ReLU (§3.1) and stores each row to its ORIGINAL position (inverse of the Algorithm 1
// permutation).  No tensor cores (unstructured sparsity is not a dense contraction; north_star).
//
// Map of this file:
//   * helpers (mbarrier, TMA, bulk / cp.async copies), parameter blocks (KParams / KParamsY / YOut);
//   * row / group kernels (spmm_tma_kernel: TMA ring, V = 2/4/8 columns per lane, optional split-K
//     slice via blockIdx.y), their generic bounds-checked twin, the split-row and split-K reductions;
//   * sparse convolution (spmm_conv2_kernel: patch staged per tile; spmm_conv_kernel: gather form);
//   * TMEM kernel (spmm_tmem_kernel: X tile in tensor memory, filler / consumer warps, optional
//     multi-destination epilogue and split-K slice, each a separate template instance);
//   * host side: upload (prepare_one), per-call path rules (launch_auto: TMEM / TMEM split-K /
//     narrow / row / split-K), tuned paths (launch_path, sdnn_tune, sdnn_conv2d_tune), the C entry
//     points, the host-buffer pipeline, serialization.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <type_traits>
#include <new>
#include <string>
#include <vector>

#include "sdnn_internal.h"
#include "group_entry.inc"

#ifndef SDNN_DIAG
#define SDNN_DIAG 0  // diagnostics builds only (kernel 5: 1 no TMEM loads, 2 no FFMA2; TMEM-R: 3 no consumer
                     // entry loop, 4 no tcgen05.cp fill); never set in the product
#endif

namespace sdnn {
void plan_fill_info(const Plan& p, int32_t device, sdnn_info* info);
}
using namespace sdnn;

// Persistent state of the host-buffer entry point: 3 streams (H2D, kernel, D2H), their events and
// two device X/Y column-block buffers.
#ifndef SDNN_HOST_BUFS  // sdnn_spmm_host pipeline depth (X/Y block buffers)
#define SDNN_HOST_BUFS 2  // 3 or 4 measured no faster (profiles/r01_host_bufs.log): PCIe-bound
#endif
constexpr int kHostBufs = SDNN_HOST_BUFS;
struct HostStage {
  cudaStream_t s[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev[3][kHostBufs] = {};
  float* x[kHostBufs] = {};
  float* y[kHostBufs] = {};
  float* bias = nullptr;
  int64_t cols = 0;
};

struct sdnn_handle_s {
  Plan plan;            // host copy (meta cleared after upload to save memory)
  int32_t device = -1;
  uint8_t* d_meta = nullptr;
  int64_t* d_blk_off = nullptr;
  int32_t* d_row_orig = nullptr;
  int32_t* d_split = nullptr;  // split-row table {rows, first piece, count} (row plan)
  // split rows whose pieces all sit in one row block: per slot {pk, target row} (row_pre), so the row
  // kernel adds the pieces in shared memory; null when some row's pieces span row blocks
  int2* d_slotpk = nullptr;
  int32_t pieces_per_cta = 0;  // most pieces in one row block (shared-memory slots the sum needs)
  cudaMemPool_t ws_pool = nullptr;  // split-row workspaces: stream-ordered, memory kept between calls
  // codegen kernel: one JIT module per panel, one stream per panel (all panels run concurrently)
  std::vector<CUmodule> cg_mods;
  std::vector<CUfunction> cg_funcs;
  std::vector<cudaStream_t> cg_streams;
  std::vector<cudaEvent_t> cg_join;
  cudaEvent_t cg_fork = nullptr;
  int32_t cg_ctas = 1;  // persistent CTAs per panel kernel
  std::mutex cg_mu;     // the per-panel streams are shared by concurrent calls on one handle
  // auto handles (kernel = 0): the TMEM plan prepared beside the row plan; sdnn_spmm takes it when
  // the call fits its fast path and fills at least one wave of CTAs (tmem_worth)
  sdnn_handle_s* alt = nullptr;
  // auto handles: the same TMEM plan with ~25 % more row blocks (fewer rows per warp) — taken per call
  // when its grid fills the GPU's waves better (tmem_pick); blob role 4
  sdnn_handle_s* alt2 = nullptr;
  // auto handles: a row plan with more, smaller row blocks, for row-plan calls whose grid on the
  // main row plan is under one wave (small N: one or two N tiles)
  sdnn_handle_s* narrow = nullptr;
  // and, when narrow has more than 4 panels per CTA, a plan of 4-panel (16-row) row blocks for the
  // calls whose TN = 128 grid on it is one to three waves (narrow_pick)
  sdnn_handle_s* narrow4 = nullptr;
  // sdnn_tune: measured best path per N (fast-path calls: one 16-byte-aligned destination)
  struct Tuned {
    int32_t path = -1;  // 0 TMEM plan, 1 row plan, 2 narrow row plan, 3 narrow4 row plan
    int32_t ks = 1;     // split-K slices
  };
  std::map<int64_t, Tuned> tuned;
  // sdnn_conv2d_tune: per geometry {B, IC, H, W, FY, FX, pad, stride} → (pixels per lane, slices)
  std::map<std::array<int32_t, 8>, std::pair<int32_t, int32_t>> conv_tuned;
  mutable std::mutex tune_mu;
  int32_t sms = 148;
  bool tmem_runs = true;  // kernel 4 plan with aligned 1×4 runs in its metadata (else the run-free consumer)
  bool tmem_runs_only = false;  // ... and nothing else (every row segment is whole runs)
  HostStage hs;         // sdnn_spmm_host staging (created on first use)
  std::mutex host_mu;
};

// ------------------------------------------------------------------------------------------------
// PTX helpers (mbarrier, TMA, bulk copy)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Programmatic dependent launch (PDL): the row, TMEM-R and reduction kernels are launched with
// programmatic stream serialization (launch_k), so a call's grid is scheduled while the previous
// kernel on the stream drains and runs its prologue (mbarrier init, TMEM allocation, the first
// metadata copies: plan memory, immutable after sdnn_prepare) in that kernel's shadow.
// pdl_wait() blocks until every prerequisite grid has completed and its writes are visible — every
// thread calls it before its first access to caller memory (X, bias, Y) or a workspace; without a
// programmatic prerequisite it returns at once.  pdl_trigger() lets the next grid launch as soon as
// every CTA of this one has started (it still waits for this grid's completion in its pdl_wait).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Timing perturbation for the pipeline-protocol tests (SDNN_JITTER=1 → KParams::dbg bit 8): a
// pseudo-random 0-2 µs sleep at the mbarrier hand-off points of the TMA / TMEM pipelines, so that
// producers, issuers and consumers interleave in orders the free-running kernel rarely produces; the
// results must stay bitwise identical (tests/test_gpu_jitter.py).  One predictable branch otherwise.
__device__ __forceinline__ void jitter(int32_t dbg, uint32_t salt) {
  if (dbg & 256) {
    uint32_t h = (salt ^ (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x >> 5) * 0x85EBCA6Bu) * 2654435761u;
    h ^= h >> 15;
    __nanosleep(h & 2047u);
  }
}
// Same, but each try_wait may suspend the thread until the phase completes (time hint in ns), so a
// warp that waits long (a filler ahead of the consumers) does not spin on issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 1000000;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Output destinations of a launch: Y is written to every y[d] (d < n), row-major with leading
// dimension ld, at columns col0 .. col0 + N − 1 (sdnn_spmm: one destination, ld = N, col0 = 0;
// sdnn_spmm_multi: e.g. the symmetric buffers of all ranks for a fused all-gather).
constexpr int kMaxDst = 8;
struct YOut {
  float* y[kMaxDst];
  int32_t n;
  int32_t mc;  // 1: y[0] is a multicast address (sdnn_spmm_multicast): stores are multimem.st, which
               // NVSwitch replicates into every rank's buffer
  int64_t ld, col0;
};
// Y written as sdnn_spmm writes it: one plain destination, leading dimension N, no offset
static bool y_plain(const YOut& o, int64_t N) { return o.n == 1 && o.ld == N && o.col0 == 0 && !o.mc; }
// stores of output elements: plain (streaming) or multimem (multicast destination)
__device__ __forceinline__ void y_st4(float* p, float a, float b, float c, float d, bool mc) {
  if (mc)
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  else
    __stcs(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}
__device__ __forceinline__ void y_st2(float* p, float a, float b, bool mc) {
  if (mc)
    asm volatile("multimem.st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
  else
    __stcs(reinterpret_cast<float2*>(p), make_float2(a, b));
}
__device__ __forceinline__ void y_st1(float* p, float a, bool mc) {
  if (mc)
    asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
  else
    *p = a;
}
static YOut y_single(float* Y, int64_t N) {
  YOut o{};
  o.y[0] = Y;
  o.n = 1;
  o.ld = N;
  o.col0 = 0;
  return o;
}
static bool y_aligned16(const YOut& o) {
  if (o.ld % 4 || o.col0 % 4) return false;
  for (int d = 0; d < o.n; ++d)
    if (reinterpret_cast<uintptr_t>(o.y[d]) % 16) return false;
  return true;
}

struct KParams {
  const uint8_t* meta;
  const int64_t* blk_off;
  const int32_t* row_orig;
  const float* X;  // fallback kernel only
  const float* bias;
  float* Y;  // the single destination (ld = N, col0 = 0); yo.y[0] as well
  int64_t N;
  int32_t K, nch, kc, wc, nrb, stages;
  int32_t x_stage_bytes, m_stage_bytes, hdr_bytes;
  int32_t act;
  float* ws;    // split-row workspace (pieces × N), row plans only
  int32_t dbg;  // TMEM kernels, diagnostics only (SDNN_DEBUG_TMEM): bit 0 skip the X loads, bit 1 skip the FMAs,
               // bit 2 skip the smem → TMEM fill
};
// Row/group/generic kernels and the multi-destination TMEM kernel: KParams + every destination.  The
// single-destination TMEM kernel takes plain KParams — its register allocation (72 regs, bound by
// __launch_bounds__) shifts with the parameter block size and a larger block measured 8 % slower on c5.
struct KParamsY : KParams {
  float* kws;   // split-K (row kernel): raw partial sums, slice blockIdx.y at kws + blockIdx.y·M·N, else NULL
  const int2* slotpk;  // row kernel, CTA-local split rows: per slot {pk, target row} (pieces summed in
                       // shared memory at the kernel's end); NULL: pieces go to the workspace p.ws
  int32_t M;
  YOut yo;  // every destination (sdnn_spmm_multi); p.Y = yo.y[0] when there is just one of ld = N, col0 = 0
};
template <bool MULTI> using TmemParams = std::conditional_t<MULTI, KParamsY, KParams>;

// acc[0..1] (4 columns of one row) += w · x
__device__ __forceinline__ void fma4(float2 (&acc)[2], float w, const float4& x) {
  const float2 w2 = make_float2(w, w);
  acc[0] = __ffma2_rn(w2, make_float2(x.x, x.y), acc[0]);
  acc[1] = __ffma2_rn(w2, make_float2(x.z, x.w), acc[1]);
}
// Consume one chunk: for each of the warp's RW rows, every (col, w) entry of the chunk:
// acc[r] += w · X_stage[col][lane·4 .. +4] (and +128 for V = 8), ascending column order.
// TF = log2 of the TMEM-kernel metadata scale (column field = 2^TF·col_local + 256·half; 0 = row format),
// read by the generic fallback of a TMEM plan.
template <int RW, int V, int TF = 0>
__device__ __forceinline__ void consume_chunk(float2 (&acc)[RW][V / 2], const float* __restrict__ xs,
                                              const uint8_t* __restrict__ ms, int warp, int lane, int hdr_bytes) {
  constexpr int TN = 32 * V;
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(ms) + warp * RW;
  const float4* ent = reinterpret_cast<const float4*>(ms + hdr_bytes);
  const float* xl = xs + lane * (V == 2 ? 2 : 4);
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const uint32_t h = hdr[r];
    const int cnt = int(TF ? (h & 0xffu) : (h & 0xffffu));
    if constexpr (V == 2) {  // 2 columns of N per lane (TN = 64): small-N calls, twice the warps
      const float4* e2 = ent + (h >> 16) / 2;
      for (int i = 0; i < cnt; i += 2) {
        const float4 ee = e2[i >> 1];
        acc[r][0] = __ffma2_rn(make_float2(ee.y, ee.y), *reinterpret_cast<const float2*>(xl + __float_as_int(ee.x) * TN),
                               acc[r][0]);
        if (i + 1 < cnt)
          acc[r][0] = __ffma2_rn(make_float2(ee.w, ee.w),
                                 *reinterpret_cast<const float2*>(xl + __float_as_int(ee.z) * TN), acc[r][0]);
      }
      continue;
    }  // TMEM format: bits 8..15 count leading runs
    const float4* e = ent + (h >> 16) / 2;
    for (int i = 0; i < cnt; i += 2) {
      const float4 ee = e[i >> 1];
      {
        const float* xp = xl + (TF ? ((__float_as_int(ee.x) & 255) >> TF) : __float_as_int(ee.x)) * TN;
        const float2 w2 = make_float2(ee.y, ee.y);
        const float4 x0 = *reinterpret_cast<const float4*>(xp);
        acc[r][0] = __ffma2_rn(w2, make_float2(x0.x, x0.y), acc[r][0]);
        acc[r][1] = __ffma2_rn(w2, make_float2(x0.z, x0.w), acc[r][1]);
        if constexpr (V == 8) {
          const float4 x1 = *reinterpret_cast<const float4*>(xp + 128);
          acc[r][2] = __ffma2_rn(w2, make_float2(x1.x, x1.y), acc[r][2]);
          acc[r][3] = __ffma2_rn(w2, make_float2(x1.z, x1.w), acc[r][3]);
        }
      }
      {  // an odd count's partner slot is the packing's zero entry (column 0, weight 0): no test, no
         // divergence bookkeeping (c2 +5-7 %, c3 256×128 +13 %); 0·x leaves the sum unchanged
         // (up to the sign of an exact zero, reading P5)
        const float* xp = xl + (TF ? ((__float_as_int(ee.z) & 255) >> TF) : __float_as_int(ee.z)) * TN;
        const float2 w2 = make_float2(ee.w, ee.w);
        const float4 x0 = *reinterpret_cast<const float4*>(xp);
        acc[r][0] = __ffma2_rn(w2, make_float2(x0.x, x0.y), acc[r][0]);
        acc[r][1] = __ffma2_rn(w2, make_float2(x0.z, x0.w), acc[r][1]);
        if constexpr (V == 8) {
          const float4 x1 = *reinterpret_cast<const float4*>(xp + 128);
          acc[r][2] = __ffma2_rn(w2, make_float2(x1.x, x1.y), acc[r][2]);
          acc[r][3] = __ffma2_rn(w2, make_float2(x1.z, x1.w), acc[r][3]);
        }
      }
    }
  }
}

// Generic fallback of a kernel-6 plan (Algorithm 1 row pairs, V = 4 tiles of 128 columns in the
// stage): per pair of rows, the shared columns (one X slice feeding both) then each row's own, in the
// order the TMEM kernel sums them.
template <int RW>
__device__ __forceinline__ void consume_pairs(float2 (&acc)[RW][2], const float* __restrict__ xs,
                                              const uint8_t* __restrict__ ms, int warp, int lane, int hdr_bytes) {
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(ms) + warp * RW;
  const float2* ent = reinterpret_cast<const float2*>(ms + hdr_bytes);  // {column field, weight}
  const float* xl = xs + lane * 4;
  auto xrow = [&](float cf) { return *reinterpret_cast<const float4*>(xl + ((__float_as_uint(cf) & 255u) >> 2) * 128); };
#pragma unroll
  for (int i = 0; i < RW / 2; ++i) {
    const uint32_t ha = hdr[2 * i], hb = hdr[2 * i + 1];
    const int ns = int((ha >> 8) & 0xffu), na = int(ha & 0xffu), nb = int(hb & 0xffu);
    const float2* e = ent + (ha >> 16);
    for (int k = 0; k < ns; ++k, e += 2) {
      const float4 x = xrow(e[0].x);
      fma4(acc[2 * i], e[0].y, x);
      fma4(acc[2 * i + 1], e[1].x, x);
    }
    for (int k = 0; k < na; ++k, ++e) fma4(acc[2 * i], e->y, xrow(e->x));
    for (int k = 0; k < nb; ++k, ++e) fma4(acc[2 * i + 1], e->y, xrow(e->x));
  }
}

// Group kernel, one chunk: the warp owns a 16-row group.  For every column of the group's union in
// this chunk one X row slice load (V floats per lane) feeds the FMAs of every nonzero of the group
// in that column; each nonzero jumps through a 16-entry branch table to a snippet that names its
// row's accumulators statically (group_entry.inc, generated; "statically encoding the
// accumulation position in the vector register name").  Columns ascend, so every row still
// accumulates in ascending column order (bitwise identical to the row kernel).
template <int V, int SB>
__device__ __forceinline__ void consume_group(uint64_t (&acc)[16][V / 2], const float* __restrict__ xs,
                                              const uint8_t* __restrict__ ms, int warp, int lane) {
  const uint4 hd = reinterpret_cast<const uint4*>(ms)[warp];
  const uint32_t* heads = reinterpret_cast<const uint32_t*>(ms) + hd.x;
  const int n = int(hd.y);
  uint32_t wp = smem_u32(ms) + hd.z * 4u;
  const uint32_t xl = smem_u32(xs) + uint32_t(lane) * 16u;
  uint4 h4 = make_uint4(0, 0, 0, 0);
  for (int e = 0; e < n; ++e) {
    const int t = e & 3;
    if (t == 0) h4 = *reinterpret_cast<const uint4*>(heads + e);
    const uint32_t h = t == 0 ? h4.x : t == 1 ? h4.y : t == 2 ? h4.z : h4.w;
    if constexpr (V == 8 && SB == 1) group_entry_v8_sb1(acc, h, xl, wp);
    else if constexpr (V == 8 && SB == 2) group_entry_v8_sb2(acc, h, xl, wp);
    else if constexpr (V == 8) group_entry_v8_sb4(acc, h, xl, wp);
    else if constexpr (SB == 1) group_entry_v4_sb1(acc, h, xl, wp);
    else if constexpr (SB == 2) group_entry_v4_sb2(acc, h, xl, wp);
    else group_entry_v4_sb4(acc, h, xl, wp);
  }
}

// Fused epilogue: y = acc + b[orig]; ReLU; store to Y[orig][n0 + ...] (inverse permutation).
__device__ __forceinline__ float2 as_f2(float2 v) { return v; }
__device__ __forceinline__ float2 as_f2(uint64_t v) {
  return make_float2(__uint_as_float(uint32_t(v)), __uint_as_float(uint32_t(v >> 32)));
}
// accumulator register type: float2 (row kernel, CUDA C++ FFMA2) or its bit pattern (group kernel PTX)
template <int KIND> struct AccSel { using type = float2; };
template <> struct AccSel<2> { using type = uint64_t; };
template <int KIND> using AccT = typename AccSel<KIND>::type;

// A warp's output rows (row_orig: plan memory) and their biases, loaded ahead of the epilogue (the row
// kernel: at its start, so the global-load latency overlaps the K loop).  Bias: caller memory — after
// pdl_wait.
template <int RW> struct RowPre {
  int32_t orow[RW];
  float b[RW];
};
template <int RW>
__device__ __forceinline__ RowPre<RW> row_pre(const KParamsY& p, int panel) {
  RowPre<RW> q;
#pragma unroll
  for (int r = 0; r < RW; ++r) q.orow[r] = p.row_orig[panel * RW + r];
#pragma unroll
  for (int r = 0; r < RW; ++r) q.b[r] = (q.orow[r] >= 0 && p.bias && !p.kws) ? p.bias[q.orow[r]] : 0.f;
  return q;
}

// Stores of one lane's output values of row `row` (columns n .. n + NV − 1) to every destination.
template <int NV, bool VEC>
__device__ __forceinline__ void y_store_row(const KParamsY& p, int32_t row, int64_t n, const float (&v)[NV]) {
  const bool single = p.Y != nullptr;
  for (int d = 0; d < (single ? 1 : p.yo.n); ++d) {
    float* yrow = single ? p.Y + int64_t(row) * p.N : p.yo.y[d] + int64_t(row) * p.yo.ld + p.yo.col0;
    const bool mc = !single && p.yo.mc;
    if (VEC && NV == 4) {
      if (n < p.N) y_st4(yrow + n, v[0], v[1], v[2], v[3], mc);
    } else if (VEC && NV == 2) {
      if (n < p.N) y_st2(yrow + n, v[0], v[1], mc);
    } else {
#pragma unroll
      for (int q = 0; q < NV; ++q)
        if (n + q < p.N) y_st1(yrow + n + q, v[q], mc);
    }
  }
}

// CTA-local split rows (row kernel, p.slotpk set; CTA-uniform): after the K loop every piece's raw
// partial sums go to shared-memory slot L (the stage ring, idle by then), and the warp holding a row's
// first piece adds the row's pieces in piece order, then the bias and the activation — the same
// operations, in the same order, as split_reduce_kernel over the workspace.  Consumer warps only
// (named barrier 1; the producer warp has exited).
// Per slot of p.slotpk: pk = L | cnt << 8 | is_first << 16 (L: the piece's shared-memory slot, a
// row's pieces consecutive) and the row's target Y row.
template <int RW, int V, bool VEC, typename A>
__device__ __forceinline__ void combine_pieces(const A (&acc)[RW][V / 2], const KParamsY& p, float* ps, int panel,
                                               int lane, int64_t n0) {
  constexpr int TN = 32 * V, NV = V == 2 ? 2 : 4;
  int2 pc[RW];  // {pk, target}; pk = 0 for whole rows and empty slots (no piece: nothing to do)
#pragma unroll
  for (int r = 0; r < RW; ++r) pc[r] = p.slotpk[panel * RW + r];
  asm volatile("bar.sync 1, %0;" ::"r"(p.wc * 32) : "memory");  // every warp is done with the ring
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    if (!(pc[r].x & 0x1ff00)) continue;  // not a piece (a piece has cnt ≥ 1)
    float* d = ps + (pc[r].x & 255) * TN + lane * NV;
#pragma unroll
    for (int h = 0; h < (V == 2 ? 1 : V / 4); ++h) {
      if constexpr (V == 2) {
        *reinterpret_cast<float2*>(d) = as_f2(acc[r][0]);
      } else {
        const float2 a0 = as_f2(acc[r][2 * h]), a1 = as_f2(acc[r][2 * h + 1]);
        *reinterpret_cast<float4*>(d + h * 128) = make_float4(a0.x, a0.y, a1.x, a1.y);
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(p.wc * 32) : "memory");
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    if (!((pc[r].x >> 16) & 1)) continue;
    const int L0 = pc[r].x & 255, cnt = (pc[r].x >> 8) & 255;
    const float b = p.bias ? p.bias[pc[r].y] : 0.f;
#pragma unroll
    for (int h = 0; h < (V == 2 ? 1 : V / 4); ++h) {
      const float* s0 = ps + L0 * TN + lane * NV + h * 128;
      float v[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) v[q] = s0[q];
      for (int k = 1; k < cnt; ++k)
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] += s0[k * TN + q];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        if (p.bias) v[q] += b;
        if (p.act == SDNN_ACT_RELU) v[q] = v[q] > 0.f ? v[q] : 0.f;
      }
      y_store_row<NV, VEC>(p, pc[r].y, n0 + h * 128 + lane * NV, v);
    }
  }
}

// pre: the rows and biases loaded ahead (row_pre), or NULL: loaded here — by lanes 0 .. RW − 1 at
// once and shuffled to the warp per row (loads placed between the rows' stores would be serialised
// behind them: two global round trips per row instead of two per warp).
template <int RW, int V, bool VEC, typename A>
__device__ __forceinline__ void epilogue(const A (&acc)[RW][V / 2], const KParamsY& p, const RowPre<RW>* pre,
                                         int panel, int lane, int64_t n0) {
  static_assert(RW <= 32, "one lane per row");
  int32_t orow_l = -1;
  float b_l = 0.f;
  if (!pre) {
    orow_l = lane < RW ? p.row_orig[panel * RW + lane] : -1;
    b_l = (orow_l >= 0 && p.bias && !p.kws) ? p.bias[orow_l] : 0.f;
  }
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int32_t orow = pre ? pre->orow[r] : __shfl_sync(0xffffffffu, orow_l, r);
    const float b = pre ? pre->b[r] : __shfl_sync(0xffffffffu, b_l, r);
    if (orow == -1 || (orow <= -2 && p.slotpk)) continue;  // CTA-local pieces: combine_pieces
    // a piece of a split row (row_orig = −2 − piece): its raw partial sums go to workspace row
    // `piece`; split_reduce_kernel adds the pieces, the bias and the activation
    const bool piece = orow <= -2 || p.kws;  // raw partial sums: a split row's piece or a split-K slice
    if constexpr (V == 2) {
      const int64_t n = n0 + lane * 2;
      const float2 a0 = as_f2(acc[r][0]);
      float v[2] = {a0.x, a0.y};
      if (!piece) {
        v[0] += b;
        v[1] += b;
        if (p.act == SDNN_ACT_RELU) {
          v[0] = v[0] > 0.f ? v[0] : 0.f;
          v[1] = v[1] > 0.f ? v[1] : 0.f;
        }
      }
      const bool single = piece || p.Y;
      for (int d = 0; d < (single ? 1 : p.yo.n); ++d) {
        float* yrow = p.kws    ? p.kws + (int64_t(blockIdx.y) * p.M + orow) * p.N
                      : piece  ? p.ws + int64_t(-2 - orow) * p.N
                      : single ? p.Y + int64_t(orow) * p.N
                               : p.yo.y[d] + int64_t(orow) * p.yo.ld + p.yo.col0;
        const bool mc = !single && !p.kws && p.yo.mc;
        if (VEC && piece) {  // raw partial sums: plain stores, kept in L2 for the reduction kernel
          if (n < p.N) *reinterpret_cast<float2*>(yrow + n) = make_float2(v[0], v[1]);
        } else if (VEC) {
          if (n < p.N) y_st2(yrow + n, v[0], v[1], mc);
        } else {
          if (n < p.N) y_st1(yrow + n, v[0], mc);
          if (n + 1 < p.N) y_st1(yrow + n + 1, v[1], mc);
        }
      }
      continue;
    }
#pragma unroll
    for (int h = 0; h < V / 4; ++h) {
      const int64_t n = n0 + h * 128 + lane * 4;
      const float2 a0 = as_f2(acc[r][2 * h]), a1 = as_f2(acc[r][2 * h + 1]);
      float v[4] = {a0.x, a0.y, a1.x, a1.y};
      if (!piece) {
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] += b;
        if (p.act == SDNN_ACT_RELU) {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = v[q] > 0.f ? v[q] : 0.f;
        }
      }
      // p.Y set: one destination of leading dimension N (sdnn_spmm); else every yo.y[d] (sdnn_spmm_multi)
      const bool single = piece || p.Y;
      for (int d = 0; d < (single ? 1 : p.yo.n); ++d) {
        float* yrow = p.kws    ? p.kws + (int64_t(blockIdx.y) * p.M + orow) * p.N
                      : piece  ? p.ws + int64_t(-2 - orow) * p.N
                      : single ? p.Y + int64_t(orow) * p.N
                               : p.yo.y[d] + int64_t(orow) * p.yo.ld + p.yo.col0;
        const bool mc = !single && !p.kws && p.yo.mc;
        if (VEC && piece) {  // raw partial sums: plain stores, kept in L2 for the reduction kernel
          if (n < p.N) *reinterpret_cast<float4*>(yrow + n) = make_float4(v[0], v[1], v[2], v[3]);
        } else if (VEC) {
          if (n < p.N) y_st4(yrow + n, v[0], v[1], v[2], v[3], mc);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (n + q < p.N) y_st1(yrow + n + q, v[q], mc);
        }
      }
    }
  }
}

// Split rows (row plan): Y[row] = act(Σ_pieces ws[piece] (in piece order) + b[row]).  One thread per
// column; blockIdx.y = split row.  split = {rows[ns], first piece[ns], piece count[ns]}.
__global__ void split_reduce_kernel(const float* __restrict__ ws, const int32_t* __restrict__ split, int32_t ns,
                                    const float* __restrict__ bias, int32_t act, const YOut yo, int64_t N) {
  pdl_trigger();
  pdl_wait();
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  for (int32_t sr = int32_t(blockIdx.y); sr < ns; sr += int32_t(gridDim.y)) {  // gridDim.y ≤ 65535
  const int32_t row = split[sr], first = split[ns + sr], cnt = split[2 * ns + sr];
  float v = ws[int64_t(first) * N + n];
  for (int32_t k = 1; k < cnt; ++k) v += ws[int64_t(first + k) * N + n];
  if (bias) v += bias[row];
  if (act == SDNN_ACT_RELU) v = v > 0.f ? v : 0.f;
#pragma unroll
  for (int d = 0; d < kMaxDst; ++d)  // static indices: yo stays in the parameter bank (no local copy)
    if (d < yo.n) y_st1(yo.y[d] + int64_t(row) * yo.ld + yo.col0 + n, v, yo.mc);
  }
}

// Split-K (row / TMEM / conv kernels): Y[row] = act(Σ_{s < KS} kws[s][row] (slice order) + b[row]).
// One thread per column (C = 1) or per 4 columns (C = 4: N % 4 == 0, 16-byte aligned destinations —
// float4 loads and stores, the same additions in the same order); blockIdx.y = row.
template <int C>
__global__ void splitk_reduce_kernel(const float* __restrict__ kws, int32_t KS, int32_t M, const float* __restrict__ bias,
                                     int32_t act, const YOut yo, int64_t N) {
  pdl_trigger();
  pdl_wait();
  const int64_t n = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * C;
  if (n >= N) return;
  const int64_t slice = int64_t(M) * N;
  for (int32_t row = int32_t(blockIdx.y); row < M; row += int32_t(gridDim.y)) {  // gridDim.y ≤ 65535
    float v[C];
    const float* src = kws + int64_t(row) * N + n;
    if constexpr (C == 4) {
      const float4 a = *reinterpret_cast<const float4*>(src);
      v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
      for (int32_t s = 1; s < KS; ++s) {
        const float4 b = *reinterpret_cast<const float4*>(src + s * slice);
        v[0] += b.x, v[1] += b.y, v[2] += b.z, v[3] += b.w;
      }
    } else {
      v[0] = src[0];
      for (int32_t s = 1; s < KS; ++s) v[0] += src[s * slice];
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (bias) v[c] += bias[row];
      if (act == SDNN_ACT_RELU) v[c] = v[c] > 0.f ? v[c] : 0.f;
    }
#pragma unroll
    for (int d = 0; d < kMaxDst; ++d) {  // static indices: yo stays in the parameter bank (no local copy)
      if (d >= yo.n) continue;
      float* dst = yo.y[d] + int64_t(row) * yo.ld + yo.col0 + n;
      if constexpr (C == 4) y_st4(dst, v[0], v[1], v[2], v[3], yo.mc);
      else y_st1(dst, v[0], yo.mc);
    }
  }
}

// Fast path: TMA producer warp + W_c consumer warps, mbarrier stage ring.
// KIND 1 = row kernel (RW rows per warp), KIND 2 = group kernel (RW = 16).
template <int KIND, int RW, int V, int SB = 0>
__global__ void __launch_bounds__(KIND == 2 ? (kMaxGroupWarps + 1) * 32 : 17 * 32, 1)
    spmm_tma_kernel(const __grid_constant__ CUtensorMap tmap, const KParamsY p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TN = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % p.nrb;
  const int64_t tile = blockIdx.x / p.nrb;
  const int64_t n0 = tile * TN;
  const int S = p.stages;
  uint8_t* xstage = smem;
  uint8_t* mstage = smem + size_t(S) * p.x_stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(mstage + size_t(S) * p.m_stage_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.wc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();

  // split-K (gridDim.y > 1): this CTA's K chunks [j0, j1)
  const int j0 = int(blockIdx.y) * p.nch / int(gridDim.y), j1 = (int(blockIdx.y) + 1) * p.nch / int(gridDim.y);
  if (warp == p.wc) {  // producer
    if (lane == 0) {
      const int64_t* off = p.blk_off + int64_t(rb) * p.nch;
      // the first stages' metadata (plan memory) before the dependency wait, their X tiles after it;
      // the chunk offsets are loaded together (S ≤ 4), then one chunk ahead of their use — a small
      // call's start-up is otherwise a chain of dependent global loads
      const int pre = S < j1 - j0 ? S : j1 - j0;
      int64_t o[5];
#pragma unroll
      for (int t = 0; t < 5; ++t) o[t] = t <= pre ? off[j0 + t] : 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < pre) {
          const uint32_t mbytes = uint32_t(o[t + 1] - o[t]);
          mbar_expect_tx(&full[t], uint32_t(p.x_stage_bytes) + mbytes);
          bulk_load(mstage + size_t(t) * p.m_stage_bytes, p.meta + o[t], mbytes, &full[t]);
        }
      }
      pdl_wait();
      for (int t = 0; t < pre; ++t)
        tma_load_2d(xstage + size_t(t) * p.x_stage_bytes, &tmap, int32_t(n0), (j0 + t) * p.kc, &full[t]);
      int64_t lo = 0, hi = 0;
#pragma unroll
      for (int t = 0; t < 5; ++t)
        if (t == pre) lo = o[t];
      if (j0 + pre < j1) hi = off[j0 + pre + 1];
      int s = pre % S, ph = 0;  // stage and the phase of its empty barrier to wait for
      for (int j = j0 + pre; j < j1; ++j) {
        const int64_t nxt = j + 1 < j1 ? off[j + 2] : 0;
        jitter(p.dbg, uint32_t(j));
        mbar_wait(&empty[s], ph);
        const uint32_t mbytes = uint32_t(hi - lo);
        mbar_expect_tx(&full[s], uint32_t(p.x_stage_bytes) + mbytes);
        tma_load_2d(xstage + size_t(s) * p.x_stage_bytes, &tmap, int32_t(n0), j * p.kc, &full[s]);
        bulk_load(mstage + size_t(s) * p.m_stage_bytes, p.meta + lo, mbytes, &full[s]);
        lo = hi;
        hi = nxt;
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  AccT<KIND> acc[RW][V / 2];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int q = 0; q < V / 2; ++q) acc[r][q] = AccT<KIND>{};
  pdl_wait();  // bias (prefetched now), Y / workspace in the epilogue
  // output rows and biases loaded before the K loop where the registers allow (≤ 16 accumulators; the
  // 8-row / V = 8 tiles would spill), else after it
  constexpr bool PRE = RW * V <= 16;
  RowPre<RW> pre;
  if constexpr (PRE) pre = row_pre<RW>(p, rb * p.wc + warp);

  for (int j = j0, s = 0, ph = 0; j < j1; ++j) {
    mbar_wait(&full[s], ph);
    const float* xs = reinterpret_cast<const float*>(xstage + size_t(s) * p.x_stage_bytes);
    if constexpr (KIND == 2)
      consume_group<V, SB>(acc, xs, mstage + size_t(s) * p.m_stage_bytes, warp, lane);
    else
      consume_chunk<RW, V>(acc, xs, mstage + size_t(s) * p.m_stage_bytes, warp, lane, p.hdr_bytes);
    jitter(p.dbg, uint32_t(j) * 7u + 1u);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  }
  (void)TN;
  epilogue<RW, V, true>(acc, p, PRE ? &pre : nullptr, rb * p.wc + warp, lane, n0);
  if constexpr (KIND == 1)
    if (p.slotpk) combine_pieces<RW, V, true>(acc, p, reinterpret_cast<float*>(xstage), rb * p.wc + warp, lane, n0);
}

// Generic path (N % 4 != 0 or unaligned X/Y): the same consumption, with the stage filled by all
// threads using bounds-checked loads (zero fill) and a block barrier instead of TMA/mbarriers.
template <int KIND, int RW, int V, int SB = 0>
__global__ void __launch_bounds__(KIND == 2 ? kMaxGroupWarps * 32 : (KIND == 4 || KIND == 6) ? kTmemRWarps * 32 : 16 * 32, 1)
    spmm_generic_kernel(const KParamsY p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TN = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % p.nrb;
  const int64_t n0 = int64_t(blockIdx.x / p.nrb) * TN;
  float* xs = reinterpret_cast<float*>(smem);
  uint8_t* ms = smem + p.x_stage_bytes;
  const int64_t* off = p.blk_off + int64_t(rb) * p.nch;
  const int nthr = blockDim.x;

  AccT<KIND> acc[RW][V / 2];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int q = 0; q < V / 2; ++q) acc[r][q] = AccT<KIND>{};

  for (int j = 0; j < p.nch; ++j) {
    __syncthreads();
    const int k0 = j * p.kc;
    for (int idx = threadIdx.x; idx < p.kc * TN; idx += nthr) {
      const int kk = idx / TN, nn = idx % TN;
      const int64_t k = k0 + kk, n = n0 + nn;
      xs[idx] = (k < p.K && n < p.N) ? p.X[k * p.N + n] : 0.f;
    }
    const int32_t mbytes = int32_t(off[j + 1] - off[j]);
    const uint4* src = reinterpret_cast<const uint4*>(p.meta + off[j]);
    for (int idx = threadIdx.x; idx < mbytes / 16; idx += nthr) reinterpret_cast<uint4*>(ms)[idx] = src[idx];
    __syncthreads();
    if constexpr (KIND == 2)
      consume_group<V, SB>(acc, xs, ms, warp, lane);
    else if constexpr (KIND == 6)
      consume_pairs<RW>(acc, xs, ms, warp, lane, p.hdr_bytes);
    else
      consume_chunk<RW, V, (KIND == 4 || KIND == 5 ? KIND - 2 : 0)>(acc, xs, ms, warp, lane, p.hdr_bytes);
  }
  epilogue<RW, V, false>(acc, p, static_cast<const RowPre<RW>*>(nullptr), rb * p.wc + warp, lane, n0);
}


// ------------------------------------------------------------------------------------------------
// Sparse k×k convolution (§3.2.3): the filters are the OC × (IC·FY·FX)
// sparse matrix of a row plan (column k = (ic·FY + fy)·FX + fx), and the dense operand is the
// virtual matrix X_v[k][n] = X[ic][b][oy·s + fy − pad][ox·s + fx − pad] (0 outside the image),
// n = (b·Ho + oy)·Wo + ox, "realized on the fly from the input dense activations with the proper
// offsets".  Same consumption and fused epilogue as the row kernel; the X stage is gathered by every
// thread with 4-byte cp.async (src-size 0 → zero fill for the padding taps), double-buffered so the
// gather of chunk j + 1 overlaps the FMAs of chunk j.  Y is OC × (B·Ho·Wo) = [OC][B][Ho][Wo].
struct ConvGeom {
  int32_t B, IC, H, W, Ho, Wo, FY, FX, pad, stride;
};
// The convolution's virtual operand written out: Xv[k][n] = X[ic][b][oy·s + fy − pad][ox·s + fx − pad]
// (0 outside the image), k = (ic·FY + fy)·FX + fx, n = (b·Ho + oy)·Wo + ox — the K × N matrix the
// TMEM-R SpMM then multiplies (sdnn_conv2d's explicit form for deep, wide layers).  One thread per
// element of a row segment: coalesced stores along n, the loads stride `s` along the image row.
__global__ void im2col_kernel(const float* __restrict__ X, float* __restrict__ Xv, const ConvGeom c, int64_t N) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int32_t k = int32_t(blockIdx.y);
  if (n >= N) return;
  const int32_t fx = k % c.FX, fy = (k / c.FX) % c.FY, ic = k / (c.FX * c.FY);
  const int32_t ox = int32_t(n % c.Wo), oy = int32_t((n / c.Wo) % c.Ho), b = int32_t(n / (int64_t(c.Wo) * c.Ho));
  const int32_t y = oy * c.stride + fy - c.pad, x = ox * c.stride + fx - c.pad;
  float v = 0.f;
  if (y >= 0 && y < c.H && x >= 0 && x < c.W) v = X[((int64_t(ic) * c.B + b) * c.H + y) * c.W + x];
  Xv[int64_t(k) * N + n] = v;
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {  // zero-fill when !valid
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int RW, bool VEC>
__global__ void __launch_bounds__(16 * 32, 1) spmm_conv_kernel(const KParamsY p, const ConvGeom c) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int V = 4, TN = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % p.nrb;
  const int64_t n0 = int64_t(blockIdx.x / p.nrb) * TN;
  // stage addresses from the shared-memory base (pointer arrays would become generic loads)
  auto xs_of = [&](int b) { return reinterpret_cast<float*>(smem + size_t(b) * p.x_stage_bytes); };
  auto ms_of = [&](int b) { return smem + 2 * size_t(p.x_stage_bytes) + size_t(b) * p.m_stage_bytes; };
  const int64_t* off = p.blk_off + int64_t(rb) * p.nch;
  // this thread's column of the stage (blockDim.x is a multiple of TN) and its output pixel
  const int nn = int(threadIdx.x) % TN, kk0 = int(threadIdx.x) / TN, kstep = int(blockDim.x) / TN;
  const int64_t n = n0 + nn;
  const bool col_ok = n < p.N;
  const int HWo = c.Ho * c.Wo, FYX = c.FY * c.FX;
  const int bimg = col_ok ? int(n / HWo) : 0;
  const int rem = col_ok ? int(n - int64_t(bimg) * HWo) : 0;
  const int iy0 = (rem / c.Wo) * c.stride - c.pad, ix0 = (rem % c.Wo) * c.stride - c.pad;
  const float* xb = p.X + int64_t(bimg) * c.H * c.W;  // + ic·B·H·W + iy·W + ix
  const int64_t icstride = int64_t(c.B) * c.H * c.W;
  auto gather = [&](int j, int buf) {
    int k = j * p.kc + kk0;
    int ic = k / FYX, t = k - ic * FYX;
    for (int kk = kk0; kk < p.kc; kk += kstep) {
      const int fy = t / c.FX, fx = t - fy * c.FX;
      const int iy = iy0 + fy, ix = ix0 + fx;
      const bool ok = col_ok && k < p.K && iy >= 0 && iy < c.H && ix >= 0 && ix < c.W;
      const float* src = ok ? xb + ic * icstride + int64_t(iy) * c.W + ix : p.X;
      cp_async4(xs_of(buf) + kk * TN + nn, src, ok);
      k += kstep;
      t += kstep;
      while (t >= FYX) {
        t -= FYX;
        ++ic;
      }
    }
    const int mbytes = int(off[j + 1] - off[j]);
    const uint8_t* msrc = p.meta + off[j];
    for (int i = int(threadIdx.x); i < mbytes / 16; i += int(blockDim.x)) cp_async16(ms_of(buf) + 16 * i, msrc + 16 * i);
    cp_async_commit();
  };
  float2 acc[RW][V / 2];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int q = 0; q < V / 2; ++q) acc[r][q] = make_float2(0.f, 0.f);
  gather(0, 0);
  for (int j = 0; j < p.nch; ++j) {
    if (j + 1 < p.nch) {
      gather(j + 1, (j + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    consume_chunk<RW, V>(acc, xs_of(j & 1), ms_of(j & 1), warp, lane, p.hdr_bytes);
    __syncthreads();
  }
  epilogue<RW, V, VEC>(acc, p, static_cast<const RowPre<RW>*>(nullptr), rb * p.wc + warp, lane, n0);
}

// Patch form (the default): per K chunk the CTA stages the *input* rows its tile needs — the window
// of the zero-padded input P[ic][b·Hp + y + pad][x + pad] (Hp = H + 2·pad, Wp = W + 2·pad) covering
// the tile's output rows and the filter halo, for the chunk's input channels — instead of the FY·FX
// shifted copies of the virtual matrix (≈ 4-9× fewer staged elements, one coalesced row per warp
// step).  X_v[k][n] = patch[tab[k − k0] + pos(n)], tab = (ic − ic_lo)·PS + fy·Wp + fx per chunk
// column, pos(n) = (b·Hp + oy·stride − vr0)·Wp + ox·stride per output pixel.  A lane owns the
// pixels n0 + lane + 32q (q < 4), so each of its four loads per nonzero is a conflict-free
// warp-contiguous read and the epilogue stores are coalesced.
// V16 (W % 4 = 0): each patch row keeps a 4-float left margin so the image row lands 16-byte
// aligned at column 4 and is filled with 16-byte cp.async (a quarter of the copies); margins, pad
// columns and rows outside the image are zeroed once per kernel and never written again.
template <int RW, int PX, bool V16>
// (min 2 resident 512-thread blocks → ≤ 64 registers: 4-warp CTAs then fit 8 per SM instead of 4;
// 256 channels at 28×28: 231 → 180 µs, profiles/r01_conv_regcap.log)
__global__ void __launch_bounds__(16 * 32, 2) spmm_conv2_kernel(const KParamsY p, const ConvGeom c, int32_t PSrows,
                                                               int32_t ICC) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TN = 32 * PX;  // PX pixels per lane: 4, or 2 for small grids (twice the CTAs)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = int(blockDim.x) >> 5;
  const int rb = blockIdx.x % p.nrb;
  const int64_t n0 = int64_t(blockIdx.x / p.nrb) * TN;
  // padded row: Wp columns; in smem a row is RS floats, padded column xp at smem column xp + CO
  const int Hp = c.H + 2 * c.pad, Wp = c.W + 2 * c.pad, FYX = c.FY * c.FX;
  const int CO = V16 ? 4 - c.pad : 0, RS = V16 ? ((4 + c.W + c.pad + 3) & ~3) : Wp, PS = PSrows * RS;
  const int W4 = c.W >> 2;  // V16: 16-byte pieces per image row
  const int HWo = c.Ho * c.Wo;
  const size_t stage = ((size_t(ICC) * PS * 4 + size_t(p.kc) * 4 + 127) & ~size_t(127)) + size_t(p.m_stage_bytes);
  // srcoff[e], e < PS: offset of patch element e (row e / Wp, column e mod Wp) within one input
  // channel, −1 for padding; the same for every channel and chunk of this tile (after both stages)
  int32_t* srcoff = reinterpret_cast<int32_t*>(smem + 2 * stage);
  // stage b: patch floats at smem + b·stage, then the tap table, then the metadata block (addresses
  // recomputed from smem — no pointer arrays, so every access stays an LDS/STS)
  auto patch_of = [&](int b) { return reinterpret_cast<float*>(smem + size_t(b) * stage); };
  auto tab_of = [&](int b) { return reinterpret_cast<int32_t*>(smem + size_t(b) * stage + size_t(ICC) * PS * 4); };
  auto ms_of = [&](int b) { return smem + size_t(b + 1) * stage - p.m_stage_bytes; };
  const int64_t* off = p.blk_off + int64_t(rb) * p.nch;
  // the tile's first virtual input row, and each lane's four pixels
  const int b0 = int(n0 / HWo), oy0 = int((n0 - int64_t(b0) * HWo) / c.Wo);
  const int vr0 = b0 * Hp + oy0 * c.stride;
  int po[PX];
#pragma unroll
  for (int q = 0; q < PX; ++q) {
    const int64_t n = n0 + lane + 32 * q;
    const int b = int(n / HWo), rem = int(n - int64_t(b) * HWo), oy = rem / c.Wo, ox = rem - oy * c.Wo;
    po[q] = n < p.N ? (b * Hp + oy * c.stride - vr0) * RS + ox * c.stride + CO : CO;
  }
  const int64_t icstride = int64_t(c.B) * c.H * c.W;
  if constexpr (V16) {
    // items e < PSrows·W4: row r = e / W4, piece c4; srcoff = element offset of the piece, −1 if the
    // row is outside the image (stays zero)
    for (int e = int(threadIdx.x); e < PSrows * W4; e += int(blockDim.x)) {
      const int r = e / W4, c4 = e - r * W4, vr = vr0 + r, b = vr / Hp, iy = vr - b * Hp - c.pad;
      srcoff[e] = (b < c.B && iy >= 0 && iy < c.H) ? (b * c.H + iy) * c.W + 4 * c4 : -1;
      srcoff[PSrows * W4 + e] = r * RS + 4 + 4 * c4;  // destination float offset within a channel
    }
    float* z = reinterpret_cast<float*>(smem);  // zero both stages' patches (margins, pad, outside rows)
    for (int b2 = 0; b2 < 2; ++b2)
      for (int e = int(threadIdx.x); e < ICC * PS; e += int(blockDim.x))
        reinterpret_cast<float*>(smem + size_t(b2) * stage)[e] = 0.f;
    (void)z;
  } else {
    for (int e = int(threadIdx.x); e < PS; e += int(blockDim.x)) {
      const int r = e / Wp, xp = e - r * Wp, vr = vr0 + r, b = vr / Hp, iy = vr - b * Hp - c.pad, ix = xp - c.pad;
      srcoff[e] = (b < c.B && iy >= 0 && iy < c.H && ix >= 0 && ix < c.W) ? (b * c.H + iy) * c.W + ix : -1;
    }
  }
  __syncthreads();
  auto gather = [&](int j, int buf) {
    const int k0 = j * p.kc, ic_lo = k0 / FYX;
    for (int icl = 0; icl < ICC; ++icl) {  // the chunk's input channels, element-parallel over the patch
      const int ic = ic_lo + icl;
      const float* src = p.X + int64_t(ic < c.IC ? ic : 0) * icstride;
      float* dst = patch_of(buf) + icl * PS;
      if constexpr (V16) {
        for (int e = int(threadIdx.x); e < PSrows * W4; e += int(blockDim.x)) {
          const int so = srcoff[e];
          if (so < 0) continue;  // outside the image: zero since the kernel start
          cp_async16z(dst + srcoff[PSrows * W4 + e], ic < c.IC ? src + so : p.X, ic < c.IC);
        }
      } else {
        for (int e = int(threadIdx.x); e < PS; e += int(blockDim.x)) {
          const int so = srcoff[e];
          const bool ok = so >= 0 && ic < c.IC;
          cp_async4(dst + e, ok ? src + so : p.X, ok);
        }
      }
    }
    for (int cl = int(threadIdx.x); cl < p.kc; cl += int(blockDim.x)) {
      const int k = k0 + cl, ic = k / FYX, t = k - ic * FYX, fy = t / c.FX, fx = t - fy * c.FX;
      tab_of(buf)[cl] = (ic - ic_lo) * PS + fy * RS + fx;
    }
    const int mbytes = int(off[j + 1] - off[j]);
    const uint8_t* msrc = p.meta + off[j];
    for (int i = int(threadIdx.x); i < mbytes / 16; i += int(blockDim.x)) cp_async16(ms_of(buf) + 16 * i, msrc + 16 * i);
    cp_async_commit();
  };
  float2 acc[RW][PX / 2];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int q = 0; q < PX / 2; ++q) acc[r][q] = make_float2(0.f, 0.f);
  // split-K (gridDim.y > 1): this CTA's K chunks [j0, j1); raw partial sums to p.kws
  const int j0 = int(blockIdx.y) * p.nch / int(gridDim.y), j1 = (int(blockIdx.y) + 1) * p.nch / int(gridDim.y);
  gather(j0, 0);
  for (int j = j0; j < j1; ++j) {
    const int bj = (j - j0) & 1;
    if (j + 1 < j1) {
      gather(j + 1, bj ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* xs = patch_of(bj);
    const int32_t* tb = tab_of(bj);
    const uint8_t* msb = ms_of(bj);
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(msb) + warp * RW;
    const float4* ent = reinterpret_cast<const float4*>(msb + p.hdr_bytes);
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const uint32_t h = hdr[r];
      const int cnt = int(h & 0xffffu);
      const float4* e = ent + (h >> 16) / 2;
      for (int i = 0; i < cnt; i += 2) {
        const float4 ee = e[i >> 1];
        {
          const float* xp = xs + tb[__float_as_int(ee.x)];
          const float2 w2 = make_float2(ee.y, ee.y);
#pragma unroll
          for (int q = 0; q < PX / 2; ++q)
            acc[r][q] = __ffma2_rn(w2, make_float2(xp[po[2 * q]], xp[po[2 * q + 1]]), acc[r][q]);
        }
        {  // an odd row segment's partner slot is the zero entry (column 0, weight 0) of the packing
          const float* xp = xs + tb[__float_as_int(ee.z)];
          const float2 w2 = make_float2(ee.w, ee.w);
#pragma unroll
          for (int q = 0; q < PX / 2; ++q)
            acc[r][q] = __ffma2_rn(w2, make_float2(xp[po[2 * q]], xp[po[2 * q + 1]]), acc[r][q]);
        }
      }
    }
    __syncthreads();
  }
  // epilogue: + bias[orig], act, coalesced stores of pixels n0 + lane + 32q
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int32_t orow = p.row_orig[(rb * p.wc + warp) * RW + r];
    if (orow < 0) continue;
    const float bv = (p.bias && !p.kws) ? p.bias[orow] : 0.f;
    float v[PX];
#pragma unroll
    for (int q = 0; q < PX / 2; ++q) {
      v[2 * q] = acc[r][q].x + bv;
      v[2 * q + 1] = acc[r][q].y + bv;
    }
    float* yrow = p.kws ? p.kws + (int64_t(blockIdx.y) * p.M + orow) * p.N : p.Y + int64_t(orow) * p.N;
#pragma unroll
    for (int q = 0; q < PX; ++q) {
      const int64_t n = n0 + lane + 32 * q;
      const float y = (p.act == SDNN_ACT_RELU && !p.kws) ? (v[q] > 0.f ? v[q] : 0.f) : v[q];
      if (n < p.N) {
        if (p.kws) yrow[n] = y;  // split-K slice: kept in L2 for the reduction kernel
        else __stcs(yrow + n, y);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// TMEM kernel (DESIGN.md §6 "TMEM kernel").  The row kernel reads one 4-byte X operand per FMA from
// shared memory, and shared memory delivers 128 B/clk/SM — a 25 % ceiling on the FMA pipe.  Tensor
// memory is read into registers by tcgen05.ld at up to ~357 B/clk/SM (.32x32b.x16) / ~200 B/clk/SM
// (.x4) (tools/microbench/tmem_bw.cu, profiles/r01_tmem_bw.log), so here the X tile lives in TMEM
// and the CUDA cores read their operands from there:
//   * TMEM lane L (0..127) holds columns n0 + 4L .. 4L+3 of N; TMEM column 4·k + v holds
//     X[k0 + k][n0 + 4L + v].  Two halves of 256 columns = two K chunks of 64 (double buffer).
//   * a producer thread streams X[k0:k0+16, n0:n0+512] pieces (TMA, 3-D map so a K row of the tile
//     is 2 KB contiguous) into a 4-slot shared-memory ring and moves each K row into TMEM with one
//     tcgen05.cp.128x128b (lane L ← bytes 16L..16L+15 of the row); tcgen05.commit → mbarriers
//     signal "slot reusable" and "chunk in TMEM";
//   * consumer warp w reads TMEM lane quarter q = w % 4 (hardware rule: warp w%4 owns lanes
//     32q..32q+31), i.e. N columns n0 + 128q + 4·lane + v, for the 16 rows of warp slot w / 4;
//     per nonzero (col, w): tcgen05.ld.32x32b.x4 at TMEM column 4·col → 4 floats → 2 FFMA2;
//   * metadata (row-kernel format, 64 rows per block) arrives by bulk copy; the epilogue is the
//     row kernel's (bias, ReLU, store to the original row).
// Every row still accumulates its nonzeros in ascending column order with fp32 FMA: results are
// bitwise identical to the row kernel's.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float4& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(taddr));
}
// Completes this thread's tcgen05.ld; the loaded registers pass through the asm so that no use of
// them can be scheduled above the wait.
__device__ __forceinline__ void tmem_wait_ld(float4& a) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(a.x), "+f"(a.y), "+f"(a.z), "+f"(a.w) : : "memory");
}
__device__ __forceinline__ void tmem_wait_ld(float4& a, float4& b) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(a.x), "+f"(a.y), "+f"(a.z), "+f"(a.w), "+f"(b.x), "+f"(b.y), "+f"(b.z), "+f"(b.w)
               :
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld(float4& a, float4& b, float4& c, float4& d) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(a.x), "+f"(a.y), "+f"(a.z), "+f"(a.w), "+f"(b.x), "+f"(b.y), "+f"(b.z), "+f"(b.w),
                 "+f"(c.x), "+f"(c.y), "+f"(c.z), "+f"(c.w), "+f"(d.x), "+f"(d.y), "+f"(d.z), "+f"(d.w)
               :
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float4 (&v)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "f"(v[0].x), "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z), "f"(v[1].w),
      "f"(v[2].x), "f"(v[2].y), "f"(v[2].z), "f"(v[2].w), "f"(v[3].x), "f"(v[3].y), "f"(v[3].z), "f"(v[3].w));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}
// Shared-memory matrix descriptor (tcgen05): no swizzle, K-major canonical layout — 8-row × 16-byte
// core matrices, 128 B apart along the 128 rows (SBO); the second 16-byte column 2 KB further (LBO).
__device__ __forceinline__ uint64_t cp_desc(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(2048 >> 4) << 16) | (uint64_t(128 >> 4) << 32) |
         (uint64_t(1) << 46);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kTmemConsumers = 4 * kTmemPanels;  // 16 consumer warps
constexpr int kTmemPieceBytes = 32 * 1024;        // one TMA piece: 8192 / (128·V) K rows × 128·V columns
constexpr int kTmemMetaSlots = 2;
constexpr size_t tmem_smem_bytes(int m_stage_bytes) {
  return size_t(kTmemPieces) * kTmemPieceBytes + size_t(kTmemMetaSlots) * m_stage_bytes + 16 * 8 + 16;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float4& a, float4& b, float4& c, float4& d) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w), "=f"(c.x), "=f"(c.y),
        "=f"(c.z), "=f"(c.w), "=f"(d.x), "=f"(d.y), "=f"(d.z), "=f"(d.w)
      : "r"(taddr));
}
template <int V> struct TmemLd;
template <> struct TmemLd<4> {
  static __device__ __forceinline__ void ld(uint32_t taddr, float4 (&v)[1]) { tmem_ld4(taddr, v[0]); }
};
template <> struct TmemLd<8> {
  static __device__ __forceinline__ void ld(uint32_t taddr, float4 (&v)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[0].z), "=f"(v[0].w), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[1].z),
                   "=f"(v[1].w)
                 : "r"(taddr));
  }
};

// Split-K TMEM launches (gridDim.y slices): this CTA's chunk range [first, first + count), cut at
// even chunks so a chunk's TMEM half (packed into the metadata as 256·(chunk mod 2)) matches the
// half the CTA's own double buffer gives it.  One slice: all chunks.
template <bool SPLIT> __device__ __forceinline__ int2 tmem_chunks(int nch) {
  if constexpr (!SPLIT) {
    return make_int2(0, nch);
  } else {
    const int pairs = (nch + 1) / 2, y = int(blockIdx.y), ny = int(gridDim.y);
    const int a = 2 * (y * pairs / ny), b = min(nch, 2 * ((y + 1) * pairs / ny));
    return make_int2(a, b - a);
  }
}

// Consumer warp of TMEM lane quarter q, warp slot wi: the chunk loop (wait for the chunk's
// metadata and TMEM half, 4 / 2 nonzeros per step: tcgen05.ld → FFMA2) and the fused epilogue.
template <int V, bool MULTI, bool SPLIT = false>
__device__ __forceinline__ void tmem_consume(const TmemParams<MULTI || SPLIT>& p, uint8_t* mring, uint64_t* mfull, uint64_t* mempty,
                                             uint64_t* tfull, uint64_t* tfree, int rb, int64_t n0, int q, int wi,
                                             int lane) {
  constexpr int RW = tmem_rows(V);
  constexpr int MS = kTmemMetaSlots;
  constexpr int G = V / 4;
  constexpr int U = tmem_pad(V);
  const uint32_t tl = uint32_t(q * 32) << 16;  // this warp's TMEM lane quarter (allocation at lane 0, column 0)
  float2 acc[RW][2 * G];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) acc[r][c] = make_float2(0.f, 0.f);
  const int nrel = tmem_chunks<SPLIT>(p.nch).y;
  for (int j = 0; j < nrel; ++j) {
    const int h = j & 1, m = j % MS;
    mbar_wait(&mfull[m], (j / MS) & 1);
    mbar_wait(&tfull[h], (j >> 1) & 1);
    tc_fence_after();
    const uint8_t* ms = mring + size_t(m) * p.m_stage_bytes;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(ms) + wi * RW;
    const float4* ent = reinterpret_cast<const float4*>(ms + p.hdr_bytes);
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const uint32_t hh = hdr[r];
      const int cnt = int(hh & 0xffu);
      const float4* e = ent + (hh >> 16) / 2;
      if (p.dbg & 2) continue;
      int i = 0;
      if constexpr (V == 4) {  // leading aligned 1×4 runs: one x16 load each
        const int nrun = int((hh >> 8) & 0xffu);
        for (; i < 4 * nrun; i += 4) {
          const float4 e0 = e[i >> 1], e1 = e[(i >> 1) + 1];
          float4 xa, xb, xc, xd;
          tmem_ld16(tl + __float_as_uint(e0.x), xa, xb, xc, xd);
          tmem_wait_ld(xa, xb, xc, xd);
          fma4(*reinterpret_cast<float2(*)[2]>(&acc[r][0]), e0.y, xa);
          fma4(*reinterpret_cast<float2(*)[2]>(&acc[r][0]), e0.w, xb);
          fma4(*reinterpret_cast<float2(*)[2]>(&acc[r][0]), e1.y, xc);
          fma4(*reinterpret_cast<float2(*)[2]>(&acc[r][0]), e1.w, xd);
        }
      }
      // steps of U nonzeros (zero-padded to U): U TMEM loads in flight, then the FFMA2s in
      // ascending column order
      for (; i < cnt; i += U) {
        float4 ee[U / 2];
#pragma unroll
        for (int t = 0; t < U / 2; ++t) ee[t] = e[(i >> 1) + t];
        float4 x[U][G];
#if SDNN_DIAG == 1  // diagnostics build: no TMEM loads (operands from the metadata)
#pragma unroll
        for (int t = 0; t < U; ++t)
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float v = (t & 1) ? ee[t >> 1].z : ee[t >> 1].x;
            x[t][g] = make_float4(v, v, v, v);
          }
#else
#pragma unroll
        for (int t = 0; t < U / 2; ++t) {
          TmemLd<V>::ld(tl + __float_as_uint(ee[t].x), x[2 * t]);
          TmemLd<V>::ld(tl + __float_as_uint(ee[t].z), x[2 * t + 1]);
        }
        if constexpr (U == 4 && G == 1) tmem_wait_ld(x[0][0], x[1][0], x[2][0], x[3][0]);
        else tmem_wait_ld(x[0][0], x[0][1], x[1][0], x[1][1]);
#endif
#if SDNN_DIAG == 2  // diagnostics build: no FFMA2 (one FADD per load keeps it live)
#pragma unroll
        for (int t = 0; t < U; ++t) acc[r][0].x += x[t][0].x;
#else
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const float w = (t & 1) ? ee[t >> 1].w : ee[t >> 1].y;
#pragma unroll
          for (int g = 0; g < G; ++g) fma4(*reinterpret_cast<float2(*)[2]>(&acc[r][2 * g]), w, x[t][g]);
        }
#endif
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&tfree[h]);
      mbar_arrive(&mempty[m]);
    }
  }
  // epilogue: row panel rb·4 + wi; lane columns n0 + 128q + 4·lane (+ 512 for the second group)
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int32_t orow = p.row_orig[(rb * kTmemPanels + wi) * RW + r];
    if (orow < 0) continue;
    const float b = (p.bias && !SPLIT) ? p.bias[orow] : 0.f;
    float* yrow = MULTI ? nullptr : p.Y + int64_t(orow) * p.N;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t n = n0 + g * 512 + q * 128 + lane * 4;
      float v[4] = {acc[r][2 * g].x + b, acc[r][2 * g].y + b, acc[r][2 * g + 1].x + b, acc[r][2 * g + 1].y + b};
      if (p.act == SDNN_ACT_RELU && !SPLIT) {
#pragma unroll
        for (int t = 0; t < 4; ++t) v[t] = v[t] > 0.f ? v[t] : 0.f;
      }
      if constexpr (SPLIT) {  // split-K slice: raw partial sums (splitk_reduce_kernel adds bias, act)
        if (n < p.N)
          *reinterpret_cast<float4*>(p.kws + (int64_t(blockIdx.y) * p.M + orow) * p.N + n) =
              make_float4(v[0], v[1], v[2], v[3]);  // L2-resident for the reduction (no streaming hint)
      } else if constexpr (MULTI) {  // sdnn_spmm_multi: every destination, leading dimension ld, offset col0
        if (n < p.N)
          for (int d = 0; d < p.yo.n; ++d)
            y_st4(p.yo.y[d] + int64_t(orow) * p.yo.ld + p.yo.col0 + n, v[0], v[1], v[2], v[3], p.yo.mc);
      } else {
        if (n < p.N) __stcs(reinterpret_cast<float4*>(yrow + n), make_float4(v[0], v[1], v[2], v[3]));
      }
    }
  }
}

// V = 4: TMEM lane L ↔ columns n0 + 4L + {0..3}; V = 8: also n0 + 512 + 4L + {0..3} (TMEM columns
// 8k + 4..7), so both halves of a lane's data come from contiguous 2 KB runs of an X row and the
// epilogue stores two coalesced float4 per row.
// FILL 0: one producer warp moves each TMA piece into TMEM with tcgen05.cp (~46 B/clk/SM at most,
// profiles/r01_tmem_cp.log); FILL 1: four filler warps (one per TMEM lane quarter) read the piece
// with LDS.128 and write TMEM with tcgen05.st.32x32b.x16 (~216 B/clk/SM), filler 0 lane 0 also
// issues the TMA and metadata copies.
template <int FILL> __host__ __device__ constexpr int tmem_side_warps() { return FILL ? 4 : 1; }
// FILL 2: odd pieces of a chunk by tcgen05.cp (issued by filler 0 lane 0), even pieces by the four
// filler warps with tcgen05.st — the two fill paths run side by side.
template <int V, int FILL, bool MULTI = false, bool SPLIT = false>
__global__ void __launch_bounds__((kTmemConsumers + tmem_side_warps<FILL>()) * 32, 1)
    spmm_tmem_kernel(const __grid_constant__ CUtensorMap tmap, const TmemParams<MULTI || SPLIT> p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TN = 128 * V;
  constexpr int KC = tmem_kc(V);
  constexpr int PK = 8192 / TN;  // K rows per 32 KB piece
  constexpr int PPC = KC / PK;   // pieces per K chunk
  constexpr int S = kTmemPieces, MS = kTmemMetaSlots;
  constexpr int G = V / 4;       // float4 groups per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % p.nrb;
  const int64_t n0 = int64_t(blockIdx.x / p.nrb) * TN;
  uint8_t* xring = smem;
  uint8_t* mring = smem + size_t(S) * kTmemPieceBytes;
  uint64_t* slot_full = reinterpret_cast<uint64_t*>(mring + size_t(MS) * p.m_stage_bytes);
  uint64_t* slot_empty = slot_full + S;
  uint64_t* tfull = slot_empty + S;  // [2]: K chunk resident in TMEM half h
  uint64_t* tfree = tfull + 2;       // [2]: every consumer warp is done with TMEM half h
  uint64_t* mfull = tfree + 2;       // [MS]
  uint64_t* mempty = mfull + MS;     // [MS]
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(mempty + MS);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&slot_full[s], 1);
      mbar_init(&slot_empty[s], tmem_side_warps<FILL>());
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], tmem_side_warps<FILL>());
      mbar_init(&tfree[h], kTmemConsumers);
    }
    for (int m = 0; m < MS; ++m) {
      mbar_init(&mfull[m], 1);
      mbar_init(&mempty[m], kTmemConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_s;

  if (FILL >= 1 && warp >= kTmemConsumers) {  // fillers: TMA → smem ring → LDS.128 → tcgen05.st → TMEM half
    const int q = warp & 3;  // warps 16..19 → lane quarters 0..3
    const uint32_t tq = tbase + (uint32_t(q * 32) << 16);
    const bool leader = warp == kTmemConsumers && lane == 0;
    const int2 jr = tmem_chunks<SPLIT>(p.nch);  // this CTA's chunks (all of them unless split-K)
    const int64_t* off = p.blk_off + int64_t(rb) * p.nch + jr.x;
    const int total = jr.y * PPC;
    const int32_t nb = int32_t(n0 / 128);
    auto load_piece = [&](int i) {
      const int s = i % S;
      if (p.dbg & 1) {
        mbar_arrive(&slot_full[s]);
        return;
      }
      mbar_expect_tx(&slot_full[s], kTmemPieceBytes);
      tma_load_3d(xring + size_t(s) * kTmemPieceBytes, &tmap, 0, nb, (jr.x * PPC + i) * PK, &slot_full[s]);
    };
    auto load_meta = [&](int j) {
      const int m = j % MS;
      const uint32_t mbytes = uint32_t(off[j + 1] - off[j]);
      mbar_expect_tx(&mfull[m], mbytes);
      bulk_load(mring + size_t(m) * p.m_stage_bytes, p.meta + off[j], mbytes, &mfull[m]);
    };
    if (leader) {
      for (int i = 0; i < S && i < total; ++i) load_piece(i);
      for (int j = 0; j < MS && j < jr.y; ++j) load_meta(j);  // this slice's chunks only
    }
    for (int j = 0; j < jr.y; ++j) {
      const int h = j & 1;
      if (j >= 2) {  // half h held chunk j−2: wait until every consumer is done with it
        mbar_wait(&tfree[h], ((j >> 1) - 1) & 1);
        tc_fence_after();
        if (leader) {
          mbar_wait(&mempty[j % MS], ((j >> 1) - 1) & 1);
          load_meta(j);
        }
      }
      for (int pc = 0; pc < PPC; ++pc) {
        const int i = j * PPC + pc, s = i % S;
        if (FILL == 2 && (pc & 1)) {  // this piece goes through the tcgen05.cp engine
          if (leader) {
            mbar_wait(&slot_full[s], (i / S) & 1);
            const uint32_t src = smem_u32(xring + size_t(s) * kTmemPieceBytes);
#pragma unroll
            for (int kk = 0; kk < PK; kk += 8 / V)
              tc_cp_128x256b(tbase + uint32_t(h * 256 + (pc * PK + kk) * V), cp_desc(src + uint32_t(kk * TN) * 4));
            tc_commit(&slot_empty[s]);
          } else if (lane == 0) {
            mbar_arrive(&slot_empty[s]);
          }
        } else if (p.dbg & 4) {  // diagnostics: no fill at all (TMEM keeps stale data)
          mbar_wait(&slot_full[s], (i / S) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[s]);
        } else {
          mbar_wait(&slot_full[s], (i / S) & 1);
          const float4* src = reinterpret_cast<const float4*>(xring + size_t(s) * kTmemPieceBytes) + q * 32 + lane;
          // all PK·V/4 LDS.128 of the piece first (latency overlapped), then the tcgen05.st.x16s
          constexpr int NST = PK * V / 16;
          float4 v[NST][4];
#pragma unroll
          for (int u = 0; u < NST; ++u)
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int kk = u * (16 / V);
              v[u][t] = V == 4 ? src[(kk + t) * (TN / 4)] : src[(kk + (t >> 1)) * (TN / 4) + (t & 1) * 128];
            }
#pragma unroll
          for (int u = 0; u < NST; ++u) tmem_st16(tq + uint32_t(h * 256 + (pc * PK + u * (16 / V)) * V), v[u]);
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[s]);
        }
        if (leader && i + S < total) {
          mbar_wait(&slot_empty[s], (i / S) & 1);
          load_piece(i + S);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (FILL == 2 && leader) tc_commit(&tfull[h]);  // also covers this thread's tcgen05.cp of the chunk
      else if (lane == 0) mbar_arrive(&tfull[h]);
    }
  } else if (warp == kTmemConsumers) {  // producer: TMA → smem ring → tcgen05.cp → TMEM half
    if (lane == 0) {
      const int64_t* off = p.blk_off + int64_t(rb) * p.nch;
      const int total = p.nch * PPC;
      const int32_t nb = int32_t(n0 / 128);
      auto load_piece = [&](int i) {
        const int s = i % S;
        mbar_expect_tx(&slot_full[s], kTmemPieceBytes);
        tma_load_3d(xring + size_t(s) * kTmemPieceBytes, &tmap, 0, nb, i * PK, &slot_full[s]);
      };
      auto load_meta = [&](int j) {
        const int m = j % MS;
        const uint32_t mbytes = uint32_t(off[j + 1] - off[j]);
        mbar_expect_tx(&mfull[m], mbytes);
        bulk_load(mring + size_t(m) * p.m_stage_bytes, p.meta + off[j], mbytes, &mfull[m]);
      };
      for (int i = 0; i < S && i < total; ++i) load_piece(i);
      for (int j = 0; j < MS && j < p.nch; ++j) load_meta(j);
      for (int i = 0; i < total; ++i) {
        const int s = i % S, j = i / PPC, h = j & 1, pc = i % PPC;
        if (pc == 0 && j >= 2) {  // half h held chunk j−2: wait until every consumer is done with it
          mbar_wait(&tfree[h], ((j >> 1) - 1) & 1);
          tc_fence_after();
          mbar_wait(&mempty[j % MS], ((j >> 1) - 1) & 1);
          load_meta(j);
        }
        mbar_wait(&slot_full[s], (i / S) & 1);
        const uint32_t src = smem_u32(xring + size_t(s) * kTmemPieceBytes);
        // tcgen05.cp.128x256b: lane L ← 16 B at 16L (SBO 128 B per 8 lanes) and 16 B one LBO =
        // 2 KB further: V = 4 → K rows kk, kk+1 (TMEM columns 4kk..4kk+7); V = 8 → columns n0+4L
        // and n0+512+4L of row kk (TMEM columns 8kk..8kk+7).  ~90 cycles per copy whatever its
        // size (profiles/r01_tmem_cp.log), so the widest shape.
#pragma unroll
        for (int kk = 0; kk < PK; kk += 8 / V)
          tc_cp_128x256b(tbase + uint32_t(h * 256 + (pc * PK + kk) * V), cp_desc(src + uint32_t(kk * TN) * 4));
        tc_commit(&slot_empty[s]);
        if (pc == PPC - 1) tc_commit(&tfull[h]);
        if (i + S < total) {
          mbar_wait(&slot_empty[s], (i / S) & 1);
          load_piece(i + S);
        }
      }
    }
  } else {
    // one code copy for all four lane quarters (four specialised copies exceed the SM's
    // instruction cache: profiles/r01_tmem_fill_diag.log)
    if (tbase != 0) __trap();  // the 512-column allocation starts at lane 0, column 0
    tmem_consume<V, MULTI, SPLIT>(p, mring, mfull, mempty, tfull, tfree, rb, n0, warp & 3, warp >> 2, lane);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// ------------------------------------------------------------------------------------------------
// TMEM kernel, replicated lane quarters (kernel 4, the c5 bench kernel).
//   * N tile TN = 128; every TMEM lane quarter holds the same tile: lane 32q + l ↔ columns
//     n0 + 4l .. 4l+3, TMEM column 4·k + v (+ 256 for the odd K chunks) ↔ X[k0 + k].  Two halves of
//     256 columns double-buffer K chunks of 64 rows.
//   * issuer warp q (lane 0) streams piece q (16 K rows × 128 columns, 8 KB) of every K chunk: TMA into
//     its own two shared-memory slots, then one tcgen05.cp.32x128b.warpx4 per K row, which copies the
//     row's 512 bytes into the same 32 lanes × 16 B of all four lane quarters (the copy engine does
//     the replication: one shared-memory read per X element; the LDS.128 + tcgen05.st fill it replaced
//     read every element four times and cost 12 % of the kernel, profiles/r02_fill_lds_vs_sttm.log,
//     r02_ab_tmemr_cp.log).  Issuer 0 also bulk-copies the per-chunk metadata.  Each X element staged
//     from L2 serves 240 rows (24 warps × 10), 4× the rows of a non-replicated 512-column tile.
//   * consumer warp w (quarter w % 4) owns a 10-row panel; its metadata already holds the TMEM
//     address (lane base | column), so per pair of nonzeros: one LDS.128 (col, w, col, w), two R2UR,
//     two tcgen05.ld.32x32b.x4, four FFMA2 — two pairs per step while ≥ 2 remain; rows are padded to
//     whole pairs only (8 % padding on c5 against 23 % at steps of four).
//   * leading aligned 1×4 runs (block-clustered masks, c4): one tcgen05.ld.x16 per run.
// Every row accumulates in ascending column order with fp32 FMA: bitwise equal to the row kernel.
// ------------------------------------------------------------------------------------------------
constexpr int kTmemRConsumers = kTmemRWarps;  // 24 consumer warps
constexpr int kTmemRPieceBytes = 16 * 128 * 4;  // 8 KB: 16 K rows × 128 columns
constexpr int kTmemRMetaSlots = 2;
constexpr size_t tmemr_smem_bytes(int m_stage_bytes) {
  return size_t(kTmemRPieces) * kTmemRPieceBytes + size_t(kTmemRMetaSlots) * m_stage_bytes + 32 * 8 + 16;
}

// g0: global index of this item's first chunk in the CTA's chunk stream (persistent CTAs run several
// (row block, N tile) items through one pipeline; 0 otherwise) — it fixes the TMEM half, the
// metadata slot and the mbarrier phases of every chunk.
// RUNS: 0 no 1×4 runs in the plan, 1 leading runs then ordinary entries, 2 every entry in a run
template <bool MULTI, bool SPLIT, int RUNS, int RW, bool PAIRS = false>
__device__ __forceinline__ void tmemr_consume(const TmemParams<MULTI || SPLIT>& p, uint8_t* mring, uint64_t* mfull,
                                              uint64_t* mempty, uint64_t* tfull, uint64_t* tfree, int rb, int64_t n0,
                                              int warp, int lane, int g0 = 0) {
  constexpr int MS = kTmemRMetaSlots;
  float2 acc[RW][2];
#pragma unroll
  for (int r = 0; r < RW; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
  const int nrel = tmem_chunks<SPLIT>(p.nch).y;
  for (int j = 0; j < nrel; ++j) {
    const int g = g0 + j;
    const int h = g & 1, m = g % MS;
    mbar_wait(&mfull[m], (g / MS) & 1);
    mbar_wait(&tfull[h], (g >> 1) & 1);
    tc_fence_after();
    const uint8_t* ms = mring + size_t(m) * p.m_stage_bytes;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(ms) + warp * RW;
    // the warp's row segments are contiguous in the block (emit order): one stream pointer for all
    // of them, started at the first row's segment; row headers give the entry counts (prefetched one
    // row ahead)
    uint32_t hn = hdr[0];
    const float4* e = reinterpret_cast<const float4*>(ms + p.hdr_bytes) + (hn >> 17);
#if SDNN_DIAG == 3  // diagnostics build: consumers skip their entry streams (barrier hand-offs only)
    if (true) {
    } else
#endif
    if constexpr (PAIRS) {  // kernel 6: Algorithm 1 row pairs (rows 2i, 2i+1): shared columns, then each row's own
#pragma unroll
      for (int i = 0; i < RW / 2; ++i) {
        const uint32_t ha = hdr[2 * i], hb = hdr[2 * i + 1];
        int ns = int((ha >> 8) & 0xffu);
        for (; ns >= 2; ns -= 2, e += 2) {  // two shared columns {col, w_a, w_b, 0}: one load feeds both rows
          const float4 e0 = e[0], e1 = e[1];
          float4 xa, xb;
          tmem_ld4(__float_as_uint(e0.x), xa);
          tmem_ld4(__float_as_uint(e1.x), xb);
          tmem_wait_ld(xa, xb);
          fma4(acc[2 * i], e0.y, xa);
          fma4(acc[2 * i + 1], e0.z, xa);
          fma4(acc[2 * i], e1.y, xb);
          fma4(acc[2 * i + 1], e1.z, xb);
        }
        if (ns) {
          const float4 e0 = e[0];
          float4 xa;
          tmem_ld4(__float_as_uint(e0.x), xa);
          tmem_wait_ld(xa);
          fma4(acc[2 * i], e0.y, xa);
          fma4(acc[2 * i + 1], e0.z, xa);
          ++e;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {  // the first row's own columns, then the second row's
          int n = int((t ? hb : ha) & 0xffu);
          for (; n >= 4; n -= 4, e += 2) {
            const float4 e0 = e[0], e1 = e[1];
            float4 xa, xb, xc, xd;
            tmem_ld4(__float_as_uint(e0.x), xa);
            tmem_ld4(__float_as_uint(e0.z), xb);
            tmem_ld4(__float_as_uint(e1.x), xc);
            tmem_ld4(__float_as_uint(e1.z), xd);
            tmem_wait_ld(xa, xb, xc, xd);
            fma4(acc[2 * i + t], e0.y, xa);
            fma4(acc[2 * i + t], e0.w, xb);
            fma4(acc[2 * i + t], e1.y, xc);
            fma4(acc[2 * i + t], e1.w, xd);
          }
          if (n) {
            const float4 e0 = e[0];
            float4 xa, xb;
            tmem_ld4(__float_as_uint(e0.x), xa);
            tmem_ld4(__float_as_uint(e0.z), xb);
            tmem_wait_ld(xa, xb);
            fma4(acc[2 * i + t], e0.y, xa);
            fma4(acc[2 * i + t], e0.w, xb);
            ++e;
          }
        }
      }
    } else
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const uint32_t hh = hn;
      if (r + 1 < RW) hn = hdr[r + 1];
      int n = int(hh & 0xffu);  // entries (a whole number of pairs), runs included
      if constexpr (RUNS) {
        for (int nrun = int((hh >> 8) & 0xffu); nrun > 0; --nrun, e += 2, n -= 4) {  // aligned 1×4 runs
          const float4 e0 = e[0], e1 = e[1];
          float4 xa, xb, xc, xd;
          tmem_ld16(__float_as_uint(e0.x), xa, xb, xc, xd);
          tmem_wait_ld(xa, xb, xc, xd);
          fma4(acc[r], e0.y, xa);
          fma4(acc[r], e0.w, xb);
          fma4(acc[r], e1.y, xc);
          fma4(acc[r], e1.w, xd);
        }
      }
      if constexpr (RUNS == 2) continue;  // every entry was in a run (no per-row tail checks)
      for (; n >= 4; n -= 4, e += 2) {  // two pairs: four loads in flight
        const float4 e0 = e[0], e1 = e[1];
        float4 xa, xb, xc, xd;
        tmem_ld4(__float_as_uint(e0.x), xa);
        tmem_ld4(__float_as_uint(e0.z), xb);
        tmem_ld4(__float_as_uint(e1.x), xc);
        tmem_ld4(__float_as_uint(e1.z), xd);
        tmem_wait_ld(xa, xb, xc, xd);
        fma4(acc[r], e0.y, xa);
        fma4(acc[r], e0.w, xb);
        fma4(acc[r], e1.y, xc);
        fma4(acc[r], e1.w, xd);
      }
      if (n) {  // one pair
        const float4 e0 = e[0];
        float4 xa, xb;
        tmem_ld4(__float_as_uint(e0.x), xa);
        tmem_ld4(__float_as_uint(e0.z), xb);
        tmem_wait_ld(xa, xb);
        fma4(acc[r], e0.y, xa);
        fma4(acc[r], e0.w, xb);
        ++e;
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&tfree[h]);
      mbar_arrive(&mempty[m]);
    }
  }
  // epilogue: panel rb·24 + warp; lane columns n0 + 4·lane.  Lane r < RW loads row r's output row and
  // bias (two global round trips for the warp instead of two per row: the loads of one row could not
  // pass the previous row's store), then each row takes them by shuffle.
  pdl_wait();  // bias, Y / workspace
  const int64_t n = n0 + lane * 4;
  const int32_t orow_l = lane < RW ? p.row_orig[(rb * kTmemRConsumers + warp) * RW + lane] : -1;
  const float b_l = (p.bias && !SPLIT && orow_l >= 0) ? p.bias[orow_l] : 0.f;
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int32_t orow = __shfl_sync(0xffffffffu, orow_l, r);
    const float b = __shfl_sync(0xffffffffu, b_l, r);
    if (orow < 0) continue;
    float v[4] = {acc[r][0].x + b, acc[r][0].y + b, acc[r][1].x + b, acc[r][1].y + b};
    if (p.act == SDNN_ACT_RELU && !SPLIT) {
#pragma unroll
      for (int t = 0; t < 4; ++t) v[t] = v[t] > 0.f ? v[t] : 0.f;
    }
    if (n >= p.N) continue;
    if constexpr (SPLIT) {  // split-K slice: raw partial sums (splitk_reduce_kernel adds bias, act)
      // plain store: the slices stay in L2 for splitk_reduce_kernel (a streaming store sent them to DRAM)
      *reinterpret_cast<float4*>(p.kws + (int64_t(blockIdx.y) * p.M + orow) * p.N + n) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (MULTI) {  // sdnn_spmm_multi: every destination, leading dimension ld, offset col0
      for (int d = 0; d < p.yo.n; ++d)
        y_st4(p.yo.y[d] + int64_t(orow) * p.yo.ld + p.yo.col0 + n, v[0], v[1], v[2], v[3], p.yo.mc);
    } else {
      __stcs(reinterpret_cast<float4*>(p.Y + int64_t(orow) * p.N + n), make_float4(v[0], v[1], v[2], v[3]));
    }
  }
}

// PERSIST: one CTA per SM runs the items (row block, N tile) blockIdx.x, blockIdx.x + gridDim.x, …
// through one continuous chunk pipeline — the issuers fetch the next item's chunks while the
// consumers finish the current item and store its Y — for short K ranges, where a CTA's pipeline
// start-up and drain are a large part of its life.
template <bool MULTI = false, bool SPLIT = false, int RUNS = 1, int RW = tmem_rows(4), bool PAIRS = false,
          bool PERSIST = false>
__global__ void __launch_bounds__((kTmemRConsumers + 4) * 32, 1)
    spmm_tmemr_kernel(const __grid_constant__ CUtensorMap tmap, const TmemParams<MULTI || SPLIT> p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int PK = 16;          // K rows per TMA piece
  constexpr int PPC = 64 / PK;    // pieces per K chunk
  constexpr int S = kTmemRPieces, MS = kTmemRMetaSlots;
  constexpr int D = kTmemRPieces / 4;  // K chunks of X in flight in shared memory (4 issuers × D slots)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % p.nrb;
  const int64_t n0 = int64_t(blockIdx.x / p.nrb) * 128;
  uint8_t* xring = smem;
  uint8_t* mring = smem + size_t(S) * kTmemRPieceBytes;
  uint64_t* slot_full = reinterpret_cast<uint64_t*>(mring + size_t(MS) * p.m_stage_bytes);
  uint64_t* slot_empty = slot_full + S;
  uint64_t* tfull = slot_empty + S;  // [2]: K chunk resident in TMEM half h
  uint64_t* tfree = tfull + 2;       // [2]: every consumer warp is done with TMEM half h
  uint64_t* mfull = tfree + 2;       // [MS]
  uint64_t* mempty = mfull + MS;     // [MS]
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(mempty + MS);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&slot_full[s], 1);
      mbar_init(&slot_empty[s], 1);  // the issuer's tcgen05.commit
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 4);  // one tcgen05.commit per issuer
      mbar_init(&tfree[h], kTmemRConsumers);
    }
    for (int m = 0; m < MS; ++m) {
      mbar_init(&mfull[m], 1);
      mbar_init(&mempty[m], kTmemRConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tbase = *tbase_s;

  if (warp >= kTmemRConsumers) {
    // issuers: filler q owns piece q (16 K rows) of every chunk: TMA → its own two smem slots (q, q + 4
    // for even / odd chunks) → 16 × tcgen05.cp.32x128b.warpx4 (one per K row: 512 B of smem into the
    // same 32 lanes × 16 B of all four lane quarters) → commit to the slot's and the half's mbarriers.
    // One smem read per X element instead of four LDS.128 (one per quarter): the LDS fill cost 12 % of
    // the kernel (profiles/r02_fill_lds_vs_sttm.log).
    const int q = warp & 3;
    const int2 jr = tmem_chunks<SPLIT>(p.nch);
    if (lane == 0) {
      // chunk g of this CTA's stream → (row block, N tile, chunk); one item unless PERSIST
      const int items = PERSIST ? (p.nrb * int((p.N + 127) / 128) - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x) : 1;
      const int total = PERSIST ? items * p.nch : jr.y;
      auto where = [&](int g, int& rb_, int64_t& n0_, int& j_) {
        if constexpr (PERSIST) {
          const int u = g / p.nch, id = int(blockIdx.x) + u * int(gridDim.x);
          j_ = g - u * p.nch;
          rb_ = id % p.nrb;
          n0_ = int64_t(id / p.nrb) * 128;
        } else {
          j_ = jr.x + g;
          rb_ = rb;
          n0_ = n0;
        }
      };
      auto load_piece = [&](int g) {
        const int s = q + 4 * (g % D);
        if (p.dbg & 1) {
          mbar_arrive(&slot_full[s]);
          return;
        }
        int rb_, j_;
        int64_t n0_;
        where(g, rb_, n0_, j_);
        mbar_expect_tx(&slot_full[s], kTmemRPieceBytes);
        tma_load_2d(xring + size_t(s) * kTmemRPieceBytes, &tmap, int32_t(n0_), j_ * 64 + q * PK, &slot_full[s]);
      };
      auto load_meta = [&](int g) {
        const int m = g % MS;
        int rb_, j_;
        int64_t n0_;
        where(g, rb_, n0_, j_);
        const int64_t* off = p.blk_off + int64_t(rb_) * p.nch + j_;
        const uint32_t mbytes = uint32_t(off[1] - off[0]);
        mbar_expect_tx(&mfull[m], mbytes);
        bulk_load(mring + size_t(m) * p.m_stage_bytes, p.meta + off[0], mbytes, &mfull[m]);
      };
      // the first chunks' metadata (plan memory) before the dependency wait, X after it; one item:
      // their offsets loaded together (a short K range's start-up is otherwise a chain of loads)
      // one item: later chunks' offsets are read one chunk ahead, before the wait for a free slot
      const int64_t* moff = p.blk_off + int64_t(rb) * p.nch + jr.x;
      int64_t mlo = 0;  // the next metadata block's start offset (one item)
      if (q == 0) {
        if constexpr (!PERSIST) {
          static_assert(MS == 2, "prologue offsets for two metadata slots");
          const int64_t o0 = moff[0], o1 = moff[1], o2 = total > 1 ? moff[2] : 0;
          for (int j = 0; j < MS && j < total; ++j) {
            const int64_t lo = j ? o1 : o0, hi = j ? o2 : o1;
            mbar_expect_tx(&mfull[j], uint32_t(hi - lo));
            bulk_load(mring + size_t(j) * p.m_stage_bytes, p.meta + lo, uint32_t(hi - lo), &mfull[j]);
          }
          mlo = o2;
        } else {
          for (int j = 0; j < MS && j < total; ++j) load_meta(j);
        }
      }
      pdl_wait();
      for (int j = 0; j < D && j < total; ++j) load_piece(j);
      for (int j = 0; j < total; ++j) {
        const int h = j & 1, s = q + 4 * (j % D);
        jitter(p.dbg, uint32_t(j) * 5u + 3u);
        if (j >= 2) {  // half h held chunk j−2: wait until every consumer is done with it
          mbar_wait_sleep(&tfree[h], ((j >> 1) - 1) & 1);
          tc_fence_after();
        }
        if (q == 0 && j >= MS) {
          if constexpr (!PERSIST) {
            const int64_t mhi = moff[j + 1];  // in flight during the wait
            mbar_wait(&mempty[j % MS], ((j / MS) - 1) & 1);
            mbar_expect_tx(&mfull[j % MS], uint32_t(mhi - mlo));
            bulk_load(mring + size_t(j % MS) * p.m_stage_bytes, p.meta + mlo, uint32_t(mhi - mlo), &mfull[j % MS]);
            mlo = mhi;
          } else {
            mbar_wait(&mempty[j % MS], ((j / MS) - 1) & 1);
            load_meta(j);
          }
        }
        mbar_wait(&slot_full[s], (j / D) & 1);
        jitter(p.dbg, uint32_t(j) * 11u + 4u);
        const uint32_t src = smem_u32(xring + size_t(s) * kTmemRPieceBytes);
#if SDNN_DIAG != 4  // diagnostics build 4: no smem → TMEM copies (commits only)
#pragma unroll
        for (int kk = 0; kk < PK; ++kk)
          asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + uint32_t(h * 256 + (q * PK + kk) * 4)),
                       "l"(cp_desc(src + uint32_t(kk) * 512)) : "memory");
#endif
        tc_commit(&slot_empty[s]);
        tc_commit(&tfull[h]);
        if (j + D < total) {  // this slot's next chunk (its copies above must have read it first)
          mbar_wait(&slot_empty[s], (j / D) & 1);
          load_piece(j + D);
        }
      }
    }
  } else {
    if (tbase != 0) __trap();  // the 512-column allocation starts at lane 0, column 0 (addresses are absolute)
    if constexpr (PERSIST) {
      const int W = p.nrb * int((p.N + 127) / 128);
      for (int id = int(blockIdx.x), g0 = 0; id < W; id += int(gridDim.x), g0 += p.nch)
        tmemr_consume<MULTI, SPLIT, RUNS, RW, PAIRS>(p, mring, mfull, mempty, tfull, tfree, id % p.nrb,
                                                     int64_t(id / p.nrb) * 128, warp, lane, g0);
    } else {
      tmemr_consume<MULTI, SPLIT, RUNS, RW, PAIRS>(p, mring, mfull, mempty, tfull, tfree, rb, n0, warp, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
#define SDNN_CUDA_TRY(call)                                                                            \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) return fail(SDNN_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(f);
  });
  return fn;
}

template <int KIND, int RW, int V, int SB = 0>
static cudaError_t set_smem_attrs() {
  cudaError_t e = cudaFuncSetAttribute(spmm_tma_kernel<KIND, RW, V, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBudget + 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(spmm_generic_kernel<KIND, RW, V, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kSmemBudget + 1024);
}

// Resident CTAs per SM for a kernel at a block size and dynamic shared memory (cached: the query
// runs once per distinct configuration).
static int occupancy(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, size_t>, int>> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(fn, smem * 4096 + size_t(threads));
  for (const auto& kv : cache)
    if (kv.first == key) return kv.second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) n = 1;
  cache.emplace_back(key, n);
  return n;
}

// Launch with programmatic stream serialization (see pdl_wait / pdl_trigger): the kernel may be
// scheduled while the previous kernel on the stream drains.  SDNN_PDL=0 launches plainly (A/B runs).
static bool pdl_on() {
  static const bool on = [] {
    const char* e = getenv("SDNN_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
static cudaLaunchConfig_t pdl_cfg(dim3 grid, dim3 block, size_t smem, cudaStream_t st, cudaLaunchAttribute* at) {
  at->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at->val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cfg;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchAttribute at;
  const cudaLaunchConfig_t cfg = pdl_cfg(grid, block, smem, st, &at);
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// The split-K reduction of a call (raw slices kws[0..KS) of M × N each): the float4 form when N % 4 == 0
// and every destination is 16-byte aligned (the split paths' workspace always is).
static cudaError_t launch_splitk_reduce(const float* kws, int32_t KS, int32_t M, const float* bias, int32_t act,
                                        const YOut& yo, int64_t N, cudaStream_t st) {
  const unsigned rows = unsigned(std::min(M, 65535));
  if (N % 4 == 0 && y_aligned16(yo))
    return launch_k(splitk_reduce_kernel<4>, dim3(unsigned((N / 4 + 255) / 256), rows), 256, 0, st, kws, KS, M, bias,
                    act, yo, N);
  return launch_k(splitk_reduce_kernel<1>, dim3(unsigned((N + 255) / 256), rows), 256, 0, st, kws, KS, M, bias, act,
                  yo, N);
}

static sdnn_status launch_codegen(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                                  const YOut& yo, cudaStream_t stream) {
  const Plan& pl = h->plan;
  if (N >= (int64_t(1) << 30)) return fail(SDNN_ERR_UNSUPPORTED, "codegen kernel needs N < 2^30");
  if (yo.n != 1 || yo.ld != N || yo.col0 != 0)
    return fail(SDNN_ERR_UNSUPPORTED, "the codegen kernel writes one dense M×N output");
  float* Y = yo.y[0];
  const int32_t tile = 32 * pl.cg_warps;
  uint32_t ntiles = uint32_t((N + tile - 1) / tile);
  uint64_t px = reinterpret_cast<uint64_t>(X), py = reinterpret_cast<uint64_t>(Y),
           pb = reinterpret_cast<uint64_t>(bias);
  uint32_t ld4 = uint32_t(N * 4), n32 = uint32_t(N), a32 = uint32_t(act);
  void* args[] = {&px, &py, &pb, &ld4, &ld4, &n32, &a32, &ntiles};
  const unsigned grid = unsigned(std::min<int64_t>(h->cg_ctas, ntiles));
  std::lock_guard<std::mutex> lk(h->cg_mu);
  SDNN_CUDA_TRY(cudaEventRecord(h->cg_fork, stream));
  for (size_t p = 0; p < h->cg_funcs.size(); ++p) {
    SDNN_CUDA_TRY(cudaStreamWaitEvent(h->cg_streams[p], h->cg_fork, 0));
    CUresult r = driver().launchKernel(h->cg_funcs[p], grid, 1, 1, unsigned(tile), 1, 1, 0,
                                       reinterpret_cast<CUstream>(h->cg_streams[p]), args, nullptr);
    if (r != CUDA_SUCCESS) {
      const char* es = nullptr;
      driver().getErrorString(r, &es);
      return fail(SDNN_ERR_CUDA, std::string("codegen launch: ") + (es ? es : "?"));
    }
    SDNN_CUDA_TRY(cudaEventRecord(h->cg_join[p], h->cg_streams[p]));
    SDNN_CUDA_TRY(cudaStreamWaitEvent(stream, h->cg_join[p], 0));
  }
  return SDNN_OK;
}

// SDNN_JITTER=1: timing perturbation of the pipelines (tests only; see jitter())
static int32_t jitter_flag() {
  static const int32_t f = [] {
    const char* e = getenv("SDNN_JITTER");
    return (e && atoi(e) > 0) ? 256 : 0;
  }();
  return f;
}

static sdnn_status launch_tmem(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                               const YOut& yo, cudaStream_t stream, int KS = 1, cudaMemPool_t pool = nullptr) {
  const Plan& pl = h->plan;
  const bool rep = pl.kernel == 4 || pl.kernel == 6;  // replicated-quarter kernels (V = 4, TN = 128); else V = 8
  const bool prs = pl.kernel == 6;                      // Algorithm 1 row pairs
  const int V = tmem_v(pl.kernel), TN = tmem_tn(pl.kernel);
  const int64_t ntiles = (N + TN - 1) / TN;
  const int64_t nblocks = ntiles * pl.num_row_blocks;
  if (nblocks > 0x7fffffffLL) return fail(SDNN_ERR_UNSUPPORTED, "N too large for one launch");
  // split-K: slices are cut at even chunks (a chunk's TMEM half is packed into the metadata); every
  // slice keeps at least two chunk pairs, else no split
  if (KS > 1) {
    KS = std::min(KS, ((pl.num_chunks + 1) / 2) / 2);
    if (KS < 2) KS = 1;
  }
  KParamsY p{};
  p.meta = h->d_meta;
  p.blk_off = h->d_blk_off;
  p.row_orig = h->d_row_orig;
  p.X = X;
  p.bias = bias;
  p.yo = yo;
  p.Y = y_plain(yo, N) ? yo.y[0] : nullptr;
  p.N = N;
  p.K = pl.K;
  p.nch = pl.num_chunks;
  p.kc = pl.k_chunk;
  p.wc = pl.cta_panels;
  p.nrb = pl.num_row_blocks;
  p.m_stage_bytes = int32_t(align_up(pl.max_block_bytes, 128));
  p.hdr_bytes = int32_t(align_up(int64_t(pl.panel_rows) * pl.cta_panels * 4, 16));
  p.act = act;
  {
    static const int dbg = [] {
      const char* e = getenv("SDNN_DEBUG_TMEM");
      return e ? atoi(e) : 0;
    }();
    p.dbg = dbg | jitter_flag();
  }
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return fail(SDNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  CUresult cr;
  if (rep) {
    // 2-D view of X {N, K}: one box {128 columns, 16 K rows} = one 8 KB piece, rows contiguous
    const cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(pl.K)};
    const cuuint64_t strides[1] = {cuuint64_t(N) * 4};
    const cuuint32_t box[2] = {128, 16};
    const cuuint32_t estr[2] = {1, 1};
    cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // 3-D view of X: {128 columns, N/128 column blocks, K rows}, so one box {128, V, 8192/TN} lands in
    // shared memory as contiguous TN-column K rows (32 KB).
    const cuuint64_t dims[3] = {128, cuuint64_t(N / 128), cuuint64_t(pl.K)};
    const cuuint64_t strides[2] = {512, cuuint64_t(N) * 4};
    const cuuint32_t box[3] = {128, cuuint32_t(V), cuuint32_t(8192 / TN)};
    const cuuint32_t estr[3] = {1, 1, 1};
    cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (cr != CUDA_SUCCESS) return fail(SDNN_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(cr)));
  const size_t smem = rep ? tmemr_smem_bytes(p.m_stage_bytes) : tmem_smem_bytes(p.m_stage_bytes);
  if (smem > size_t(kSmemBudget) + 1024) return fail(SDNN_ERR_INTERNAL, "TMEM kernel stage does not fit shared memory");
  static const int fill_env = [] {
    const char* e = getenv("SDNN_TMEM_FILL");
    return e ? atoi(e) : -1;
  }();
  const int fill = rep ? 1 : (fill_env >= 0 ? fill_env : pl.tmem_fill);
  const unsigned threads = rep ? unsigned(kTmemRConsumers + 4) * 32 : unsigned(kTmemConsumers + (fill ? 4 : 1)) * 32;
  const unsigned grid = unsigned(nblocks);
  const bool multi = !y_plain(yo, N);
  if (multi && fill != 1) return fail(SDNN_ERR_UNSUPPORTED, "multi-destination TMEM launch needs the filler-warp fill");
  if (KS > 1) {  // split-K slices (raw partial sums) + splitk_reduce_kernel
    if (multi || fill != 1 || !pool) return fail(SDNN_ERR_INTERNAL, "TMEM split-K needs one destination and a pool");
    KParamsY q{};
    static_cast<KParams&>(q) = p;
    float* kws = nullptr;
    SDNN_CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&kws), size_t(KS) * pl.M * size_t(N) * 4, pool, stream));
    q.kws = kws;
    q.M = pl.M;
    const dim3 g2{grid, unsigned(KS)};
    if (prs) launch_k(spmm_tmemr_kernel<false, true, false, tmem_rows(4), true>, g2, threads, smem, stream, tmap, q);
    else if (rep) launch_k(spmm_tmemr_kernel<false, true>, g2, threads, smem, stream, tmap, q);
    else spmm_tmem_kernel<8, 1, false, true><<<g2, threads, smem, stream>>>(tmap, q);
    cudaError_t le = cudaGetLastError();
    if (le == cudaSuccess) {
      launch_splitk_reduce(kws, KS, pl.M, bias, act, yo, N, stream);
      le = cudaGetLastError();
    }
    cudaFreeAsync(kws, stream);
    if (le != cudaSuccess) return fail(SDNN_ERR_CUDA, std::string("TMEM split-K: ") + cudaGetErrorString(le));
    return SDNN_OK;
  }
  // persistent CTAs (one per SM, items round-robin through one chunk pipeline): the next item's first
  // chunks are fetched while the current item drains and stores its Y, and the CTA set-up (TMEM
  // allocation, barriers) is paid once — worth it for short K ranges (≤ 8 chunks) over many items
  // (≥ 4 per SM): c4 2048×512 at 80 / 95 % 197 → 188 µs, 103 → 99 µs; with fewer or longer items the
  // static round-robin loses to the hardware's CTA scheduling (c3 512², c2 3072×768 +5 %, c4 512×2048
  // at 95 % +13 %, c5 −4 %: profiles/r02_persist2_ab.log, r02_persist_ab.log).
  // SDNN_TMEM_PERSIST=0 / 1 forces it off / on.
  static const int persist_env = [] {
    const char* e = getenv("SDNN_TMEM_PERSIST");
    return e ? atoi(e) : -1;
  }();
  // Even chunk counts only (forced or not): a chunk's TMEM half is packed into the metadata as the parity
  // of its index within the K range, while the persistent pipeline alternates halves over the CTA's
  // whole chunk stream — with an odd count every second item would read the other half (found by
  // tests/stress/fuzz.py: K = 2, 64, 192, 300, 448 over >= 4 items per SM gave wrong Y from the CTA's second
  // item on; tests/test_gpu_parity.py::test_short_k_many_items).
  const bool persist_auto = nblocks >= 4 * int64_t(h->sms) && pl.num_chunks <= 8;
  const bool persist = rep && !prs && !multi && pl.num_chunks % 2 == 0 &&
                       (persist_env > 0 || (persist_env < 0 && persist_auto));
  if (persist) {
    const unsigned pg = unsigned(std::min<int64_t>(nblocks, h->sms));
    if (h->tmem_runs_only)
      launch_k(spmm_tmemr_kernel<false, false, 2, tmem_rows(4), false, true>, pg, threads, smem, stream,
               tmap, static_cast<const KParams&>(p));
    else if (h->tmem_runs)
      launch_k(spmm_tmemr_kernel<false, false, true, tmem_rows(4), false, true>, pg, threads, smem, stream, 
          tmap, static_cast<const KParams&>(p));
    else
      launch_k(spmm_tmemr_kernel<false, false, false, tmem_rows(4), false, true>, pg, threads, smem, stream, 
          tmap, static_cast<const KParams&>(p));
    SDNN_CUDA_TRY(cudaGetLastError());
    return SDNN_OK;
  }
  if (prs && multi) launch_k(spmm_tmemr_kernel<true, false, false, tmem_rows(4), true>, grid, threads, smem, stream, tmap, p);
  else if (prs)
    launch_k(spmm_tmemr_kernel<false, false, false, tmem_rows(4), true>, grid, threads, smem, stream, tmap, static_cast<const KParams&>(p));
  else if (rep && multi) launch_k(spmm_tmemr_kernel<true, false>, grid, threads, smem, stream, tmap, p);
  else if (rep && h->tmem_runs_only) launch_k(spmm_tmemr_kernel<false, false, 2>, grid, threads, smem, stream, tmap, static_cast<const KParams&>(p));
  else if (rep && h->tmem_runs) launch_k(spmm_tmemr_kernel<false, false, true>, grid, threads, smem, stream, tmap, static_cast<const KParams&>(p));
  else if (rep) launch_k(spmm_tmemr_kernel<false, false, false>, grid, threads, smem, stream, tmap, static_cast<const KParams&>(p));
  else if (multi) spmm_tmem_kernel<8, 1, true><<<grid, threads, smem, stream>>>(tmap, p);
  else if (fill == 2) spmm_tmem_kernel<8, 2><<<grid, threads, smem, stream>>>(tmap, p);
  else if (fill == 1) spmm_tmem_kernel<8, 1><<<grid, threads, smem, stream>>>(tmap, p);
  else spmm_tmem_kernel<8, 0><<<grid, threads, smem, stream>>>(tmap, p);
  SDNN_CUDA_TRY(cudaGetLastError());
  return SDNN_OK;
}

// The TMEM kernel runs one CTA per SM and pays once the call has at least a third of a wave of
// CTAs (round 2, TMEM-R kernel: 3072×768 at N = 512, 52 CTAs, 38.1 → 32.9 µs against the row plan,
// profiles/r02_tune_rules.log; round 1's kernel needed half a wave).
static bool tmem_worth(const sdnn_handle_s* a, const float* X, int64_t N, const YOut& yo) {
  return a && N % tmem_n_align(a->plan.kernel) == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 && y_aligned16(yo) &&
         3 * int64_t(a->plan.num_row_blocks) * ((N + tmem_tn(a->plan.kernel) - 1) / tmem_tn(a->plan.kernel)) >= a->sms;
}

static sdnn_status launch_main(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                               const YOut& yo, float* ws, cudaStream_t stream, float* kws = nullptr, int KS = 1,
                               bool local = false);
// The TMEM plan of an auto call: the 10-rows-per-warp plan or, where the handle has one, the second
// plan with ~25 % more row blocks — whichever gives the smaller waves × (rows per warp + 1.5) for this
// N (one CTA per SM; the 1.5 rows stand for a CTA's fixed fill and set-up).  Graph-timed with 8 rows
// per warp forced (profiles/r02_tmem_rows_ab.log): c2 3072×768 30.7 → 27.4 µs (104 → 128 CTAs, one
// wave), c3 1024×512 50.3 → 44.9 µs (245 → 294 CTAs, two waves either way); c5 34.3 → 36.5 ms and c4
// 2048×512 at 80 % 174 → 197 µs (more waves) — which the estimate rejects; c3 256×128 at 4 rows per
// warp 7.8 → 7.2 µs (98 → 147 CTAs, profiles/r02_tmem_rows_probe.log).
static sdnn_handle_s* tmem_pick(sdnn_handle_s* h, int64_t N) {
  sdnn_handle_s* a = h->alt;
  sdnn_handle_s* b = h->alt2;
  if (!a || !b) return a;
  const int64_t T = (N + tmem_tn(a->plan.kernel) - 1) / tmem_tn(a->plan.kernel);
  auto est = [&](const sdnn_handle_s* x) {
    const int64_t nrb = x->plan.num_row_blocks;
    const double waves = double((nrb * T + h->sms - 1) / h->sms);
    return waves * (double(x->plan.M) / double(nrb * kTmemRWarps) + 1.5);
  };
  return est(b) < est(a) ? b : a;
}
static int row_tile_v_small(const Plan& pl, int64_t N, int sms);
// Split rows summed inside the row kernel (combine_pieces): the plan's pieces are CTA-local
// (d_slotpk), the call takes the fast path (TMA row kernel), and the block's pieces fit the stage
// ring at the call's N tile (checked again in launch_main against the chosen stage depth).
// SDNN_LOCAL_PIECES=0 keeps the workspace + split_reduce_kernel form (A/B runs).
static bool row_pieces_local(const sdnn_handle_s* h, const float* X, int64_t N, const YOut& yo) {
  static const bool env_off = [] {
    const char* e = getenv("SDNN_LOCAL_PIECES");
    return e && atoi(e) == 0;
  }();
  const Plan& pl = h->plan;
  return !env_off && h->d_slotpk && pl.kernel == 1 && N % 4 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
         y_aligned16(yo) && int64_t(h->pieces_per_cta) <= int64_t(pl.k_chunk);
}

// N-tile width of the row / group kernels for a call: V = 8 floats per lane (TN = 256) when that
// still gives ≥ 2 CTAs per SM worth of work units, else V = 4 (TN = 128).
static int row_tile_v(const Plan& pl, int64_t N) {
  return int64_t(pl.num_row_blocks) * ((N + 255) / 256) < 2 * 148 ? 4 : 8;
}
// Row kernel only: V = 2 (TN = 64, twice the warps and CTAs) when the V = 4 grid is under half a
// wave, or under one wave with CTAs of ≤ 8 warps (profiles/r01_row_small_n.log: 1024², 70 %,
// N = 128: 44 → 26 µs; with 16-warp CTAs a 1.7-wave V = 2 grid lost: 4096², N = 256, 91 → 121 µs).
static int row_tile_v_small(const Plan& pl, int64_t N, int sms) {
  const int v = row_tile_v(pl, N);
  static const int env = [] {  // SDNN_ROW_V=2|4: force the small-N tile choice (experiments)
    const char* e = getenv("SDNN_ROW_V");
    return e ? atoi(e) : 0;
  }();
  if (pl.kernel == 1 && v == 4 && (env == 2 || env == 4)) return env;
  // one 64-column tile: wider tiles would leave lanes idle (r01_row_v.log: 4096², N = 64, 127 → 98 µs)
  if (pl.kernel == 1 && N <= 64) return 2;
  if (pl.kernel != 1 || v != 4) return v;
  const int64_t g4 = int64_t(pl.num_row_blocks) * ((N + 127) / 128);
  return (2 * g4 <= sms || (g4 < sms && pl.cta_panels <= 8)) ? 2 : 4;
}
// Row-plan call whose grid (row blocks × N tiles) is under one wave: the narrow plan (more row
// blocks of 4-row panels) fills the GPU instead (profiles/r01_row_geometry.log: 4096², N = 128:
// 166 → 90 µs; 2048², N = 512: 70 → 50 µs).
// Split-K factor for a row-kernel call (fast path, no split rows): only when the call puts fewer
// than 8 warps on an SM and the K range is long (≥ 32 chunks): KS ≤ 8 slices of ≥ 4 chunks each,
// up to ~16 warps per SM.
// The partial-sum round trip and the reduction kernel cost more than the shorter chains save on
// larger grids (profiles/r01_split_k.log: 768×3072, N = 128: 44 → 27 µs, 512×4096: 55 → 24 µs; an
// earlier looser rule lost on 2048², N = 512, 256 CTAs: 50 → 69 µs).  SDNN_SPLIT_K=n forces n (1 = off) for experiments.
static int splitk_for(const sdnn_handle_s* h, int64_t N, const float* X, const YOut& yo) {
  const Plan& pl = h->plan;
  if (pl.kernel != 1 || !pl.split_row.empty() || pl.no_split_k) return 1;
  if (!(N % 4 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 && y_aligned16(yo))) return 1;
  static const int env = [] {
    const char* e = getenv("SDNN_SPLIT_K");
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return std::max(1, std::min(env, pl.num_chunks));
  // counted on the V = 4 tile (N > 64) that launch_main then takes for split calls: K slices fill
  // the GPU better than V = 2's extra CTAs (r01_row_v.log: 768×3072, N = 256: 54 → 45 µs)
  const int64_t tn = N <= 64 ? 64 : 32 * row_tile_v(pl, N);
  const int64_t ctas = int64_t(pl.num_row_blocks) * ((N + tn - 1) / tn);
  const int64_t warps = ctas * (pl.cta_panels + 1);
  if (warps > 8 * int64_t(h->sms) || pl.num_chunks < 8) return 1;  // only clearly under-filled GPUs
  if (pl.num_chunks < 32) {
    // short K ranges (8-31 chunks): slices of ≥ 2 chunks, a power of two — the serial chunk chain
    // of a small call is its latency (graph-timed, profiles/r01_split_k_small.log: 1024², N = 128,
    // 23 → 15 µs; 512² 90 %, N = 64, 9.7 → 6.9 µs; no gain at 4 chunks, 256²)
    const int64_t ks = std::min<int64_t>({8, pl.num_chunks / 2, 16 * int64_t(h->sms) / warps});
    return ks >= 8 ? 8 : ks >= 4 ? 4 : ks >= 2 ? 2 : 1;
  }
  const int64_t ks = std::min<int64_t>({8, pl.num_chunks / 4, 16 * int64_t(h->sms) / warps});
  return ks >= 2 ? int(ks) : 1;
}
// TMEM plan with split-K: a call on the TMEM fast path whose grid is under 0.9 of a wave runs over
// KS ≤ 8 slices of K (cut at even chunks, ≥ 2 chunk pairs each), KS = ⌊SMs / grid⌋, then the
// slice-ordered reduction — when K has ≥ 16 chunks (≥ 8 for calls of ≥ 1e8 multiply-adds; shorter
// ranges: the unsplit kernel or the row plans), at a single N tile only for long K (≥ 48 chunks; ≥ 32
// with ≥ 20 % nonzeros or when the row plan has split rows and so cannot split K itself), and when the
// split grid reaches a third of a wave (8 CTAs in that last case).  Re-derived for the TMEM-R kernel from sdnn_tune over the
// BASELINE configs and the round-1 shape grid (profiles/r02_tune_rules*.log): 4096² N = 512 146 →
// 96 µs, 768×3072 N = 2048 95 → 67 µs, 512×4096 N = 2048 91 → 48 µs; 768×3072 / 512×4096 at N = 128
// (4 / 3 row blocks) stayed on the row plan's split-K (22.2 / 19.9 → 14.7 / 13.0 µs) until plans with
// split rows stopped splitting K (session 4: see row_cannot_split below).
// SDNN_TMEM_SPLIT_K=0 disables it.
static sdnn_handle_s* narrow_pick(const sdnn_handle_s* h, int64_t N);
static int tmem_split_for(const sdnn_handle_s* h, const float* X, int64_t N, const YOut& yo) {
  const sdnn_handle_s* a = h->alt;
  if (!a || h->plan.no_split_k || !h->ws_pool) return 0;
  if (!y_plain(yo, N)) return 0;
  if (!(N % tmem_n_align(a->plan.kernel) == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 && y_aligned16(yo))) return 0;
  static const int env = [] {
    const char* e = getenv("SDNN_TMEM_SPLIT_K");
    return e ? atoi(e) : -1;
  }();
  if (env == 0) return 0;
  const Plan& ap = a->plan;
  const int64_t TN = tmem_tn(ap.kernel);
  const int64_t grid = int64_t(ap.num_row_blocks) * ((N + TN - 1) / TN);
  // K ranges of 8-15 chunks split too (in two: ≥ 2 chunk pairs per slice) once the call is large enough
  // for the second kernel not to matter (≥ 1e8 multiply-adds): 1059×578 80 % at N = 1152 37.8 → 27 µs,
  // c2 3072×768 at N = 512 27.8 → 24.7 µs (tools/tune_gap.py, profiles/r02_s4_tune_gap.log)
  const int min_chunks = double(ap.nnz) * double(N) >= 1e8 ? 8 : 16;
  if (10 * grid >= 9 * int64_t(h->sms) || ap.num_chunks < min_chunks) return 0;
  const bool dense = 5 * ap.nnz >= int64_t(ap.M) * ap.K;
  // The row plan this call would otherwise take cannot split K when it has split rows (heavy rows of a
  // log-normal pattern: their pieces are summed inside the CTA) — its one CTA per row block then walks
  // the whole K range.  There the TMEM split wins from 32 chunks and from 8 split CTAs on (c2 768×3072
  // at N = 128, the BERT FFN down projection at 128 tokens: row plan 42.1 µs, 8 TMEM slices of 4 row
  // blocks 20.6 µs; 537×3333 and 1068×2578 log-normal at N = 128: 32 → 18 µs, 34 → 21 µs; one row block,
  // 70-97 × 2655: 30-39 → 16-18 µs;
  // profiles/r02_s4_tune_gap.log).
  const sdnn_handle_s* rp = narrow_pick(h, N);
  const bool row_cannot_split = !(rp ? rp : h)->plan.split_row.empty();
  if (N < 2 * TN && ap.num_chunks < (dense || row_cannot_split ? 32 : 48)) return 0;
  const int64_t pairs = (ap.num_chunks + 1) / 2;
  // at most one CTA per SM in total: a second partial wave of split CTAs doubles the time (768×3072,
  // N = 1024: 5 slices of 32 CTAs = 160 CTAs, 55 µs against 39 µs at 4 slices)
  const int64_t ks = std::min<int64_t>({8, pairs / 2, int64_t(h->sms) / grid});
  if (ks < 2) return 0;
  if (3 * grid * ks < h->sms && !(row_cannot_split && ks >= 4 && grid * ks >= 8)) return 0;
  return int(ks);
}
static bool narrow_worth(const sdnn_handle_s* h, int64_t N) {
  if (!h->narrow) return false;
  const int64_t tn = 32 * row_tile_v(h->plan, N);
  return int64_t(h->plan.num_row_blocks) * ((N + tn - 1) / tn) < h->sms;
}
// The narrow plan a call takes: 16-row blocks (5-warp CTAs, TN = 128) when that grid is one to three
// waves, else the ≥ 64-block plan (profiles/r01_tune_grid.log, N = 128 / 256: 4096² 169 → 127 µs at
// 70 % and 72 → 67 µs at 90 %, 3072² 109 → 78 µs and 57 → 42 µs, 2048² at N = 256 75 → 67 µs; the
// 4096², N = 256 grid of 512 CTAs and the 2048², N = 128 grid of 128 lost).
static sdnn_handle_s* narrow_pick(const sdnn_handle_s* h, int64_t N) {
  if (!narrow_worth(h, N)) return nullptr;
  if (h->narrow4) {
    const int64_t g = int64_t(h->narrow4->plan.num_row_blocks) * ((N + 127) / 128);
    // at N ≤ 64 (V = 2 tiles, little work per CTA) only where split-K still applies to it (≤ 8 warps
    // per SM); else the ≥ 64-block plan with split-K (graph-timed A/B, r01_ab_rules.log: 4096² 90 %,
    // N = 64: 58 → 43 µs; 3072², 192 blocks: narrow4 31 µs against 34)
    const int64_t warps = g * (h->narrow4->plan.cta_panels + 1);
    if (g > h->sms && g <= 3 * int64_t(h->sms) && (N > 64 || warps <= 8 * int64_t(h->sms))) return h->narrow4;
  }
  return h->narrow;
}

// Row / group plan of h: split rows (stream-ordered workspace, reduced after the main kernel) and
// split-K (ks_force < 0: automatic, splitk_for; else that many slices), then the kernel.
static sdnn_status launch_row(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                              const YOut& yo, cudaStream_t stream, int ks_force) {
  const Plan& pl = h->plan;
  // split rows (row plan): a stream-ordered workspace for the pieces' partial sums, reduced after
  // the main kernel (no host synchronisation; allocation nodes under CUDA-graph capture)
  float* ws = nullptr;
  int32_t ns = int32_t(pl.split_row.size());
  // CTA-local split rows on the row kernel's fast path: summed in shared memory by the kernel itself
  const bool local = ns > 0 && row_pieces_local(h, X, N, yo);
  if (local) ns = 0;
  if (ns > 0) {
    SDNN_CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ws), pl.piece_row.size() * size_t(N) * 4,
                                          h->ws_pool, stream));
  }
  // split-K (row kernel, small grids): KS CTAs per (row block, N tile), each over a K-chunk range,
  // raw partial sums to a stream-ordered workspace, summed in slice order by splitk_reduce_kernel
  const int KS = !pl.split_row.empty() || pl.no_split_k ? 1 : (ks_force > 0 ? std::min(ks_force, pl.num_chunks) : splitk_for(h, N, X, yo));
  float* kws = nullptr;
  if (KS > 1)
    SDNN_CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&kws), size_t(KS) * pl.M * size_t(N) * 4,
                                          h->ws_pool, stream));
  sdnn_status st = launch_main(h, X, N, bias, act, yo, ws, stream, kws, KS, local);
  if (KS > 1) {
    if (st == SDNN_OK) {
      launch_splitk_reduce(kws, KS, pl.M, bias, act, yo, N, stream);
      const cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) st = fail(SDNN_ERR_CUDA, std::string("splitk_reduce_kernel: ") + cudaGetErrorString(le));
    }
    cudaFreeAsync(kws, stream);
  }
  if (ns > 0) {
    if (st == SDNN_OK) {
      const dim3 grid{unsigned((N + 255) / 256), unsigned(std::min(ns, 65535))};
      launch_k(split_reduce_kernel, grid, 256, 0, stream, ws, h->d_split, ns, bias, act, yo, N);
      const cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) st = fail(SDNN_ERR_CUDA, std::string("split_reduce_kernel: ") + cudaGetErrorString(le));
    }
    cudaFreeAsync(ws, stream);
  }
  return st;
}

// Fast-path call (aligned X / Y, one destination, N % 4 == 0) that sdnn_tune measured for this N.
static bool tuned_for(const sdnn_handle_s* h, const float* X, int64_t N, const YOut& yo, sdnn_handle_s::Tuned* t) {
  if (!y_plain(yo, N) || N % 4 || reinterpret_cast<uintptr_t>(X) % 16 || !y_aligned16(yo))
    return false;
  std::lock_guard<std::mutex> lk(h->tune_mu);
  const auto it = h->tuned.find(N);
  if (it == h->tuned.end()) return false;
  *t = it->second;
  return true;
}
static sdnn_status launch_auto(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                               const YOut& yo, cudaStream_t stream);
static sdnn_status launch_path(sdnn_handle_s* h, const sdnn_handle_s::Tuned& t, const float* X, int64_t N,
                               const float* bias, int32_t act, const YOut& yo, cudaStream_t stream) {
  if (t.path < 0) return launch_auto(h, X, N, bias, act, yo, stream);  // the built-in rules
  if (t.path == 0) {
    sdnn_handle_s* th = h->alt ? h->alt : h;
    return launch_tmem(th, X, N, bias, act, yo, stream, t.ks, h->ws_pool);
  }
  return launch_row(t.path == 3 ? h->narrow4 : t.path == 2 ? h->narrow : h, X, N, bias, act, yo, stream, t.ks);
}

static sdnn_status launch_auto(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                               const YOut& yo, cudaStream_t stream);
static sdnn_status launch(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act, const YOut& yo,
                          cudaStream_t stream) {
  sdnn_handle_s::Tuned t;
  if (tuned_for(h, X, N, yo, &t) && t.path >= 0) return launch_path(h, t, X, N, bias, act, yo, stream);
  return launch_auto(h, X, N, bias, act, yo, stream);
}
// The built-in per-call rules (what an untuned call takes).
static sdnn_status launch_auto(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                               const YOut& yo, cudaStream_t stream) {
  if (const int ks = tmem_split_for(h, X, N, yo); ks > 1)
    return launch_tmem(h->alt, X, N, bias, act, yo, stream, ks, h->ws_pool);
  if (tmem_worth(h->alt, X, N, yo)) return launch_tmem(tmem_pick(h, N), X, N, bias, act, yo, stream);
  if (sdnn_handle_s* nw = narrow_pick(h, N)) return launch(nw, X, N, bias, act, yo, stream);
  const Plan& pl = h->plan;
  if (pl.kernel == 3) return launch_codegen(h, X, N, bias, act, yo, stream);
  if ((pl.kernel == 4 || pl.kernel == 5 || pl.kernel == 6) && N % tmem_n_align(pl.kernel) == 0 &&
      reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
      y_aligned16(yo))
    return launch_tmem(h, X, N, bias, act, yo, stream);
  return launch_row(h, X, N, bias, act, yo, stream, -1);
}

// The row / group / generic kernels of a plan (everything but TMEM and codegen).
static sdnn_status launch_main(sdnn_handle_s* h, const float* X, int64_t N, const float* bias, int32_t act,
                               const YOut& yo, float* ws, cudaStream_t stream, float* kws, int KS, bool local) {
  const Plan& pl = h->plan;
  const int rw = pl.panel_rows, wc = pl.cta_panels;
  // V: widest N tile that still gives >= 2 CTAs per SM worth of work units.
  int V = row_tile_v_small(pl, N, h->sms);
  if (KS > 1 && pl.kernel == 1 && N > 64 && row_tile_v(pl, N) == 4) V = 4;  // split-K calls: see splitk_for
  if (pl.kernel == 4 || pl.kernel == 5 || pl.kernel == 6) V = 4;  // TMEM plan, ragged / unaligned call: generic kernel
  const int TN = 32 * V;
  const int64_t ntiles = (N + TN - 1) / TN;
  const int64_t nblocks = ntiles * pl.num_row_blocks;
  if (nblocks > 0x7fffffffLL) return fail(SDNN_ERR_UNSUPPORTED, "N too large for one launch");

  KParamsY p{};
  p.meta = h->d_meta;
  p.blk_off = h->d_blk_off;
  p.row_orig = h->d_row_orig;
  p.X = X;
  p.bias = bias;
  p.yo = yo;
  p.Y = y_plain(yo, N) ? yo.y[0] : nullptr;
  p.dbg = jitter_flag();
  p.N = N;
  p.K = pl.K;
  p.nch = pl.num_chunks;
  p.kc = pl.k_chunk;
  p.wc = wc;
  p.nrb = pl.num_row_blocks;
  p.x_stage_bytes = int32_t(align_up(int64_t(pl.k_chunk) * TN * 4, 128));
  p.m_stage_bytes = int32_t(align_up(pl.max_block_bytes, 128));
  p.hdr_bytes = int32_t(align_up(int64_t(rw) * wc * 4, 16));
  p.act = act;
  p.ws = ws;
  p.kws = kws;
  p.M = pl.M;
  // one stage holds k_chunk K rows of the N tile: ≥ pieces_per_cta slots of TN floats (row_pieces_local)
  p.slotpk = local ? h->d_slotpk : nullptr;

  const bool fast = (N % 4 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0) && y_aligned16(yo) && pl.kernel < 4;
  if (fast) {
    const int sb = pl.group_sb;
    const void* fn = nullptr;
    if (pl.kernel == 2 && V == 8 && sb == 1) fn = reinterpret_cast<const void*>(spmm_tma_kernel<2, 16, 8, 1>);
    else if (pl.kernel == 2 && V == 8 && sb == 2) fn = reinterpret_cast<const void*>(spmm_tma_kernel<2, 16, 8, 2>);
    else if (pl.kernel == 2 && V == 8) fn = reinterpret_cast<const void*>(spmm_tma_kernel<2, 16, 8, 4>);
    else if (pl.kernel == 2 && sb == 1) fn = reinterpret_cast<const void*>(spmm_tma_kernel<2, 16, 4, 1>);
    else if (pl.kernel == 2 && sb == 2) fn = reinterpret_cast<const void*>(spmm_tma_kernel<2, 16, 4, 2>);
    else if (pl.kernel == 2) fn = reinterpret_cast<const void*>(spmm_tma_kernel<2, 16, 4, 4>);
    else if (rw == 8 && V == 8) fn = reinterpret_cast<const void*>(spmm_tma_kernel<1, 8, 8>);
    else if (rw == 8 && V == 4) fn = reinterpret_cast<const void*>(spmm_tma_kernel<1, 8, 4>);
    else if (rw == 8) fn = reinterpret_cast<const void*>(spmm_tma_kernel<1, 8, 2>);
    else if (rw == 4 && V == 8) fn = reinterpret_cast<const void*>(spmm_tma_kernel<1, 4, 8>);
    else if (V == 4) fn = reinterpret_cast<const void*>(spmm_tma_kernel<1, 4, 4>);
    else fn = reinterpret_cast<const void*>(spmm_tma_kernel<1, 4, 2>);
    const int threads = (wc + 1) * 32;
    auto smem_for = [&](int S) { return size_t(S) * (p.x_stage_bytes + p.m_stage_bytes) + size_t(2 * S) * 8; };
    int S = int(kSmemBudget / (p.x_stage_bytes + p.m_stage_bytes));
    S = std::min(S, std::min(pl.num_chunks, 4));
    if (S < 1) return fail(SDNN_ERR_INTERNAL, "stage does not fit shared memory");
    // Stage depth vs. resident CTAs: a small grid runs faster with fewer stages and more CTAs per
    // SM (profiles/r01_row_stages.log: c2 768² 52 → 30 µs at 2 stages, c3 256×128 22 → 12 µs at 1).
    // Take fewer stages while that cuts the number of waves by ≥ 10 %, and only for grids within
    // two waves; large grids keep the deep pipeline.
    {
      auto waves = [&](int s) {
        const int occ = std::max(1, occupancy(fn, threads, smem_for(s)));
        return double(nblocks) * KS / (double(h->sms) * occ);
      };
      double best = waves(S);
      int best_s = S;
      for (int s = S - 1; s >= 1 && best > 1.0; --s) {
        const double w = waves(s);
        if (w < 0.9 * best) {
          best = w;
          best_s = s;
        }
      }
      if (best <= 2.0) S = best_s;
      static const int s_env = [] {
        const char* e = getenv("SDNN_ROW_STAGES");
        return e ? atoi(e) : 0;
      }();
      if (s_env > 0) S = std::min(S, s_env);
    }
    p.stages = S;
    const size_t smem = smem_for(S);
    PFN_encodeTiled enc = get_encode_fn();
    if (!enc) return fail(SDNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(pl.K)};
    const cuuint64_t strides[1] = {cuuint64_t(N) * 4};
    const cuuint32_t box[2] = {cuuint32_t(TN), cuuint32_t(pl.k_chunk)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SDNN_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(cr)));
    void* args[] = {&tmap, &p};
    cudaLaunchAttribute at;
    const cudaLaunchConfig_t cfg = pdl_cfg(dim3(unsigned(nblocks), unsigned(KS)), dim3(unsigned(threads)), smem, stream, &at);
    SDNN_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  } else {
    if (KS > 1) return fail(SDNN_ERR_INTERNAL, "split-K outside the row kernel's fast path");
    if (p.slotpk) return fail(SDNN_ERR_INTERNAL, "CTA-local split rows outside the row kernel's fast path");
    p.stages = 1;
    const size_t smem = size_t(p.x_stage_bytes) + p.m_stage_bytes;
    const dim3 grid{unsigned(nblocks)}, block{unsigned(wc * 32)};
    const int sb = pl.group_sb;
    if (pl.kernel == 2 && V == 8 && sb == 1) spmm_generic_kernel<2, 16, 8, 1><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 2 && V == 8 && sb == 2) spmm_generic_kernel<2, 16, 8, 2><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 2 && V == 8) spmm_generic_kernel<2, 16, 8, 4><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 2 && sb == 1) spmm_generic_kernel<2, 16, 4, 1><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 2 && sb == 2) spmm_generic_kernel<2, 16, 4, 2><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 2) spmm_generic_kernel<2, 16, 4, 4><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 4) spmm_generic_kernel<4, tmem_rows(4), 4><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 5) spmm_generic_kernel<5, tmem_rows(8), 4><<<grid, block, smem, stream>>>(p);
    else if (pl.kernel == 6) spmm_generic_kernel<6, tmem_rows(4), 4><<<grid, block, smem, stream>>>(p);
    else if (rw == 8 && V == 8) spmm_generic_kernel<1, 8, 8><<<grid, block, smem, stream>>>(p);
    else if (rw == 8 && V == 4) spmm_generic_kernel<1, 8, 4><<<grid, block, smem, stream>>>(p);
    else if (rw == 8) spmm_generic_kernel<1, 8, 2><<<grid, block, smem, stream>>>(p);
    else if (rw == 4 && V == 8) spmm_generic_kernel<1, 4, 8><<<grid, block, smem, stream>>>(p);
    else if (V == 4) spmm_generic_kernel<1, 4, 4><<<grid, block, smem, stream>>>(p);
    else spmm_generic_kernel<1, 4, 2><<<grid, block, smem, stream>>>(p);
  }
  SDNN_CUDA_TRY(cudaGetLastError());
  return SDNN_OK;
}

static bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  if (!a || !b || !an || !bn) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + bn && b0 < a0 + an;
}

static sdnn_status check_device(const sdnn_handle_s* h) {
  int dev = -1;
  SDNN_CUDA_TRY(cudaGetDevice(&dev));
  if (dev != h->device)
    return fail(SDNN_ERR_DEVICE_MISMATCH, "current device " + std::to_string(dev) + " != handle device " +
                                              std::to_string(h->device));
  return SDNN_OK;
}

extern "C" {

static sdnn_status prepare_one(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M,
                               int32_t K, const sdnn_perm_opts* perm_opts, sdnn_handle* out,
                               const std::vector<int32_t>* perm = nullptr, Plan* given = nullptr) {
  if (!out) return fail(SDNN_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  int dev = -1;
  SDNN_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  SDNN_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0)
    return fail(SDNN_ERR_UNSUPPORTED, "libsdnn is built for sm_100a (B200); device is sm_" +
                                          std::to_string(prop.major) + std::to_string(prop.minor));
  sdnn_handle_s* h = new (std::nothrow) sdnn_handle_s;
  if (!h) return fail(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed");
  sdnn_status st = SDNN_OK;
  if (given) h->plan = std::move(*given);  // sdnn_deserialize: a plan prepared earlier
  else st = build_plan(csr_ptr, col_idx, vals, M, K, perm_opts, h->plan, perm);
  if (st != SDNN_OK) {
    delete h;
    return st;
  }
  h->device = dev;
  h->sms = prop.multiProcessorCount;
  static std::once_flag attr_once[64];
  cudaError_t ae = cudaSuccess;
  std::call_once(attr_once[dev & 63], [&] {
    ae = set_smem_attrs<1, 8, 8>();
    if (ae == cudaSuccess) ae = set_smem_attrs<1, 8, 4>();
    if (ae == cudaSuccess) ae = set_smem_attrs<1, 4, 8>();
    if (ae == cudaSuccess) ae = set_smem_attrs<1, 4, 4>();
    if (ae == cudaSuccess) ae = set_smem_attrs<1, 8, 2>();
    if (ae == cudaSuccess) ae = set_smem_attrs<1, 4, 2>();
    if (ae == cudaSuccess) ae = set_smem_attrs<2, 16, 8, 1>();
    if (ae == cudaSuccess) ae = set_smem_attrs<2, 16, 8, 2>();
    if (ae == cudaSuccess) ae = set_smem_attrs<2, 16, 8, 4>();
    if (ae == cudaSuccess) ae = set_smem_attrs<2, 16, 4, 1>();
    if (ae == cudaSuccess) ae = set_smem_attrs<2, 16, 4, 2>();
    if (ae == cudaSuccess) ae = set_smem_attrs<2, 16, 4, 4>();
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_generic_kernel<4, tmem_rows(4), 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_generic_kernel<5, tmem_rows(8), 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_generic_kernel<6, tmem_rows(4), 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, true, tmem_rows(4), false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, false, tmem_rows(4), false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, false, tmem_rows(4), true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<true, false, false, tmem_rows(4), true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, true, false, tmem_rows(4), true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmem_kernel<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, 2, tmem_rows(4), false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);

    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmem_kernel<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmem_kernel<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmem_kernel<8, 1, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmemr_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(spmm_tmem_kernel<8, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBudget + 1024);
  });
  auto cleanup = [&](sdnn_status s, const std::string& m) {
    cudaFree(h->d_meta);
    cudaFree(h->d_blk_off);
    cudaFree(h->d_row_orig);
    cudaFree(h->d_split);
    cudaFree(h->d_slotpk);
    if (h->ws_pool) cudaMemPoolDestroy(h->ws_pool);
    delete h;
    return fail(s, m);
  };
  if (ae != cudaSuccess) return cleanup(SDNN_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(ae));
  Plan& pl = h->plan;
  const size_t mbytes = std::max<size_t>(pl.meta.size(), 16);
  cudaError_t e = cudaMalloc(&h->d_meta, mbytes);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_blk_off, pl.blk_off.size() * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_row_orig, pl.row_orig.size() * 4);
  if (e != cudaSuccess)
    return cleanup(e == cudaErrorMemoryAllocation ? SDNN_ERR_OUT_OF_MEMORY : SDNN_ERR_CUDA,
                   std::string("cudaMalloc: ") + cudaGetErrorString(e));
  if (pl.kernel == 4) {  // any aligned 1×4 runs (header bits 8..15)?  else launches take the run-free consumer;
    // runs only (every segment = its runs: block-clustered masks) → the consumer without tail checks
    h->tmem_runs = false;
    h->tmem_runs_only = true;
    const int64_t rcta = int64_t(pl.panel_rows) * pl.cta_panels;
    for (size_t b = 0; b + 1 < pl.blk_off.size(); ++b)
      for (int64_t sl = 0; sl < rcta; ++sl) {
        uint32_t hw;
        std::memcpy(&hw, pl.meta.data() + pl.blk_off[b] + sl * 4, 4);
        const uint32_t runs = (hw >> 8) & 0xffu, cnt = hw & 0xffu;
        h->tmem_runs |= runs != 0;
        h->tmem_runs_only &= cnt == 4 * runs;
      }
    h->tmem_runs_only &= h->tmem_runs;
  }
  if (!pl.meta.empty()) e = cudaMemcpy(h->d_meta, pl.meta.data(), pl.meta.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(h->d_blk_off, pl.blk_off.data(), pl.blk_off.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(h->d_row_orig, pl.row_orig.data(), pl.row_orig.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !pl.split_row.empty()) {
    std::vector<int32_t> tab(pl.split_row);
    tab.insert(tab.end(), pl.split_first.begin(), pl.split_first.end());
    tab.insert(tab.end(), pl.split_count.begin(), pl.split_count.end());
    e = cudaMalloc(&h->d_split, tab.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_split, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
  }
  // CTA-local split rows (row plans whose pieces of each row share a row block): per slot
  // pk = L | cnt << 8 | is_first << 16 (L = the piece's index among its block's pieces, in piece-id
  // order — a row's pieces are consecutive) and the target row (the first piece sums the group)
  if (e == cudaSuccess && !pl.split_row.empty() && pl.kernel == 1) {
    const int64_t rcta = int64_t(pl.panel_rows) * pl.cta_panels;
    const size_t np = pl.piece_row.size();
    std::vector<int64_t> slot_of(np, -1);
    for (size_t sl = 0; sl < pl.row_orig.size(); ++sl)
      if (pl.row_orig[sl] <= -2 && size_t(-2 - pl.row_orig[sl]) < np) slot_of[size_t(-2 - pl.row_orig[sl])] = int64_t(sl);
    bool local = true;
    std::vector<int32_t> srow(np, -1), cnt(np, 0), firstp(np, 0);
    for (size_t i = 0; i < pl.split_row.size(); ++i)
      for (int32_t k = 0; k < pl.split_count[i]; ++k) {
        const size_t pid = size_t(pl.split_first[i] + k);
        srow[pid] = pl.split_row[i];
        cnt[pid] = pl.split_count[i];
        firstp[pid] = pl.split_first[i];
        if (slot_of[pid] < 0 || slot_of[pid] / rcta != slot_of[size_t(pl.split_first[i])] / rcta) local = false;
      }
    for (size_t pid = 0; pid < np && local; ++pid)
      if (srow[pid] < 0 || cnt[pid] > 255) local = false;
    if (local) {
      std::vector<int2> tab(pl.row_orig.size(), make_int2(0, 0));
      std::vector<int32_t> nblk(size_t(pl.num_row_blocks), 0);
      // L: rank among the block's pieces by id (pieces are visited in id order)
      for (size_t pid = 0; pid < np; ++pid) {
        const int64_t sl = slot_of[pid];
        const int32_t L = nblk[size_t(sl / rcta)]++;
        tab[size_t(sl)] = make_int2(L | (cnt[pid] << 8) | (int32_t(firstp[pid]) == int32_t(pid) ? 1 << 16 : 0), srow[pid]);
      }
      for (int32_t v : nblk) h->pieces_per_cta = std::max(h->pieces_per_cta, v);
      if (h->pieces_per_cta <= 255) {
        e = cudaMalloc(&h->d_slotpk, tab.size() * sizeof(int2));
        if (e == cudaSuccess) e = cudaMemcpy(h->d_slotpk, tab.data(), tab.size() * sizeof(int2), cudaMemcpyHostToDevice);
      }
    }
  }
  // workspace pool of the split-row pieces and the split-K slices (row and TMEM plans)
  if (e == cudaSuccess && pl.kernel != 3) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    e = cudaMemPoolCreate(&h->ws_pool, &props);
    uint64_t keep = ~uint64_t(0);
    if (e == cudaSuccess) e = cudaMemPoolSetAttribute(h->ws_pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (e != cudaSuccess) return cleanup(SDNN_ERR_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  pl.meta_size_uploaded = int64_t(pl.meta.size());
  std::vector<uint8_t>().swap(pl.meta);
  if (pl.kernel == 3) {
    cudaFree(0);  // make the runtime's primary context current for the driver API
    const int32_t threads = int32_t(std::max(1u, std::thread::hardware_concurrency()));
    sdnn_status cs = codegen_build(csr_ptr, col_idx, vals, K, pl.cg_panels, pl.cg_warps, pl.cg_prefetch, h->cg_mods,
                                   h->cg_funcs, threads);
    if (cs != SDNN_OK) {
      std::string m = sdnn_last_error_message();
      sdnn_destroy(h);
      return fail(cs, m);
    }
    const int32_t P = int32_t(pl.cg_panels.size());
    const int32_t slots = prop.multiProcessorCount * (pl.cg_warps * 32 <= 192 ? 2 : 1);
    h->cg_ctas = std::max(1, slots / P);
    h->cg_streams.assign(size_t(P), nullptr);
    h->cg_join.assign(size_t(P), nullptr);
    cudaError_t ce = cudaEventCreateWithFlags(&h->cg_fork, cudaEventDisableTiming);
    for (int32_t p = 0; p < P && ce == cudaSuccess; ++p) {
      ce = cudaStreamCreateWithFlags(&h->cg_streams[p], cudaStreamNonBlocking);
      if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->cg_join[p], cudaEventDisableTiming);
    }
    if (ce != cudaSuccess) {
      sdnn_destroy(h);
      return fail(SDNN_ERR_CUDA, std::string("codegen streams: ") + cudaGetErrorString(ce));
    }
  }
  *out = h;
  return SDNN_OK;
}

sdnn_status sdnn_prepare(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                         const sdnn_perm_opts* perm_opts, sdnn_handle* out) {
  sdnn_status st = prepare_one(csr_ptr, col_idx, vals, M, K, perm_opts, out);
  if (st != SDNN_OK || (perm_opts && perm_opts->kernel != 0)) return st;
  // auto: also the TMEM plan (same permutation, same per-row accumulation order → the two give
  // bitwise-identical results up to the sign of an exact zero)
  sdnn_perm_opts o{};
  o.struct_size = sizeof(o);
  o.permute = perm_opts ? perm_opts->permute : 1;
  o.kernel = 4;
  o.flags = perm_opts ? (perm_opts->flags & SDNN_FLAG_PERMUTED_OUTPUT) : 0u;  // TMEM plans never split rows
  const std::vector<int32_t>* perm = &(*out)->plan.perm;  // Algorithm 1 once per handle
  sdnn_handle alt = nullptr;
  st = prepare_one(csr_ptr, col_idx, vals, M, K, &o, &alt, perm);
  if (st == SDNN_ERR_UNSUPPORTED) {
    alt = nullptr;  // no TMEM plan fits this matrix (metadata blocks beyond shared memory): row plans only
  } else if (st != SDNN_OK) {
    std::string m = sdnn_last_error_message();
    sdnn_destroy(*out);
    *out = nullptr;
    return fail(st, m);
  }
  (*out)->alt = alt;
  // the second TMEM plan: ~25 % more row blocks (at least one), r = ⌈M / (24 · blocks)⌉ rows per warp
  if (alt) {
    const int64_t nrb1 = alt->plan.num_row_blocks, nrb2 = nrb1 + std::max<int64_t>(1, nrb1 / 4);
    const int64_t r = (int64_t(M) + kTmemRWarps * nrb2 - 1) / (kTmemRWarps * nrb2);
    if (r >= 1 && r < tmem_rows(4) && (int64_t(M) + kTmemRWarps * r - 1) / (kTmemRWarps * r) > nrb1) {
      sdnn_perm_opts o2 = o;
      o2.panel_rows_max = int32_t(r);
      sdnn_handle alt2 = nullptr;
      if (prepare_one(csr_ptr, col_idx, vals, M, K, &o2, &alt2, perm) == SDNN_OK) (*out)->alt2 = alt2;
    }
  }
  // and, when the row plan has few row blocks, a row plan of 4-row panels with ≥ 64 row blocks for
  // the calls whose grid would not fill the GPU (launch: narrow_worth)
  const Plan& wide = (*out)->plan;
  if (wide.kernel == 1 && !(perm_opts && (perm_opts->panel_rows_max || perm_opts->cta_panels))) {
    int32_t wc = 16;
    while (wc > 4 && (M + 4 * wc - 1) / (4 * wc) < 64) wc /= 2;
    if ((M + 4 * wc - 1) / (4 * wc) > wide.num_row_blocks) {
      sdnn_perm_opts n = perm_opts ? *perm_opts : sdnn_perm_opts{};
      n.struct_size = sizeof(n);
      if (!perm_opts) n.permute = 1;
      n.kernel = 1;
      n.panel_rows_max = 4;
      n.cta_panels = wc;
      sdnn_handle nar = nullptr;
      st = prepare_one(csr_ptr, col_idx, vals, M, K, &n, &nar, perm);
      if (st != SDNN_OK) {
        std::string m = sdnn_last_error_message();
        sdnn_destroy(*out);
        *out = nullptr;
        return fail(st, m);
      }
      (*out)->narrow = nar;
      if (wc > 4 && (M + 15) / 16 > nar->plan.num_row_blocks) {
        n.cta_panels = 4;
        sdnn_handle nar4 = nullptr;
        st = prepare_one(csr_ptr, col_idx, vals, M, K, &n, &nar4, perm);
        if (st != SDNN_OK) {
          std::string m = sdnn_last_error_message();
          sdnn_destroy(*out);
          *out = nullptr;
          return fail(st, m);
        }
        (*out)->narrow4 = nar4;
      }
    }
  }
  return SDNN_OK;
}

sdnn_status sdnn_destroy(sdnn_handle h) {
  if (!h) return SDNN_OK;
  if (h->alt) sdnn_destroy(h->alt);
  if (h->alt2) sdnn_destroy(h->alt2);
  if (h->narrow) sdnn_destroy(h->narrow);
  if (h->narrow4) sdnn_destroy(h->narrow4);
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != h->device) cudaSetDevice(h->device);
  {
    HostStage& hs = h->hs;
    for (int i = 0; i < 3; ++i) {
      if (hs.s[i]) cudaStreamSynchronize(hs.s[i]);
      for (int b = 0; b < kHostBufs; ++b)
        if (hs.ev[i][b]) cudaEventDestroy(hs.ev[i][b]);
      if (hs.s[i]) cudaStreamDestroy(hs.s[i]);
    }
    for (int b = 0; b < kHostBufs; ++b) {
      cudaFree(hs.x[b]);
      cudaFree(hs.y[b]);
    }
    cudaFree(hs.bias);
  }
  cudaFree(h->d_meta);
  cudaFree(h->d_blk_off);
  cudaFree(h->d_row_orig);
  cudaFree(h->d_split);
  cudaFree(h->d_slotpk);
  if (h->ws_pool) {
    cudaDeviceSynchronize();
    cudaMemPoolDestroy(h->ws_pool);
  }
  for (cudaStream_t st : h->cg_streams)
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t ev : h->cg_join)
    if (ev) cudaEventDestroy(ev);
  if (h->cg_fork) cudaEventDestroy(h->cg_fork);
  for (CUmodule m : h->cg_mods)
    if (m) driver().moduleUnload(m);
  if (cur != h->device && cur >= 0) cudaSetDevice(cur);
  delete h;
  return SDNN_OK;
}

sdnn_status sdnn_spmm(sdnn_handle h, const float* X, int64_t N, const float* bias, int32_t act, float* Y,
                      void* stream) {
  if (!h) return fail(SDNN_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (N < 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "N < 0");
  if (act != SDNN_ACT_NONE && act != SDNN_ACT_RELU) return fail(SDNN_ERR_INVALID_ARGUMENT, "unknown act");
  if (N == 0) return SDNN_OK;
  if (!X || !Y) return fail(SDNN_ERR_INVALID_ARGUMENT, "X or Y is NULL");
  const size_t ybytes = size_t(h->plan.M) * size_t(N) * 4;
  if (overlaps(Y, ybytes, X, size_t(h->plan.K) * size_t(N) * 4) || overlaps(Y, ybytes, bias, size_t(h->plan.M) * 4))
    return fail(SDNN_ERR_INVALID_ARGUMENT, "Y overlaps X or bias");
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  return launch(h, X, N, bias, act, y_single(Y, N), static_cast<cudaStream_t>(stream));
}

sdnn_status sdnn_spmm_multi(sdnn_handle h, const float* X, int64_t N, const float* bias, int32_t act,
                            float* const* Y_dsts, int32_t n_dst, int64_t ldy, int64_t col0, void* stream) {
  if (!h) return fail(SDNN_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (N < 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "N < 0");
  if (act != SDNN_ACT_NONE && act != SDNN_ACT_RELU) return fail(SDNN_ERR_INVALID_ARGUMENT, "unknown act");
  if (!Y_dsts || n_dst < 1 || n_dst > kMaxDst) return fail(SDNN_ERR_INVALID_ARGUMENT, "need 1..8 destinations");
  if (col0 < 0 || ldy < col0 + N) return fail(SDNN_ERR_INVALID_ARGUMENT, "need col0 >= 0 and ldy >= col0 + N");
  if (N == 0) return SDNN_OK;
  if (!X) return fail(SDNN_ERR_INVALID_ARGUMENT, "X is NULL");
  YOut yo{};
  yo.n = n_dst;
  yo.ld = ldy;
  yo.col0 = col0;
  const size_t span = (size_t(h->plan.M - 1) * size_t(ldy) + size_t(col0 + N)) * 4;
  for (int32_t d = 0; d < n_dst; ++d) {
    if (!Y_dsts[d]) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL destination");
    yo.y[d] = Y_dsts[d];
    if (overlaps(Y_dsts[d], span, X, size_t(h->plan.K) * size_t(N) * 4) || overlaps(Y_dsts[d], span, bias, size_t(h->plan.M) * 4))
      return fail(SDNN_ERR_INVALID_ARGUMENT, "a destination overlaps X or bias");
  }
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  return launch(h, X, N, bias, act, yo, static_cast<cudaStream_t>(stream));
}

sdnn_status sdnn_spmm_multicast(sdnn_handle h, const float* X, int64_t N, const float* bias, int32_t act, float* Y_mc,
                                int64_t ldy, int64_t col0, void* stream) {
  if (!h) return fail(SDNN_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (h->plan.kernel == 3) return fail(SDNN_ERR_UNSUPPORTED, "the codegen kernel has no multicast epilogue");
  float* const dst[1] = {Y_mc};
  // validation and launch as sdnn_spmm_multi with one destination, then flag it multicast
  if (N < 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "N < 0");
  if (act != SDNN_ACT_NONE && act != SDNN_ACT_RELU) return fail(SDNN_ERR_INVALID_ARGUMENT, "unknown act");
  if (!Y_mc) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL multicast destination");
  if (col0 < 0 || ldy < col0 + N) return fail(SDNN_ERR_INVALID_ARGUMENT, "need col0 >= 0 and ldy >= col0 + N");
  if (N == 0) return SDNN_OK;
  if (!X) return fail(SDNN_ERR_INVALID_ARGUMENT, "X is NULL");
  YOut yo{};
  yo.n = 1;
  yo.mc = 1;
  yo.ld = ldy;
  yo.col0 = col0;
  yo.y[0] = dst[0];
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  return launch(h, X, N, bias, act, yo, static_cast<cudaStream_t>(stream));
}

static sdnn_status conv2d_impl(sdnn_handle h, const float* X, int32_t B, int32_t IC, int32_t H, int32_t W,
                               int32_t FY, int32_t FX, int32_t pad, int32_t stride, const float* bias, int32_t act,
                               float* Y, void* stream, int px_force, int ks_force);

sdnn_status sdnn_conv2d(sdnn_handle h, const float* X, int32_t B, int32_t IC, int32_t H, int32_t W, int32_t FY,
                        int32_t FX, int32_t pad, int32_t stride, const float* bias, int32_t act, float* Y,
                        void* stream) {
  int px = -1, ks = -1;
  if (h) {
    std::lock_guard<std::mutex> lk(h->tune_mu);
    const auto it = h->conv_tuned.find({B, IC, H, W, FY, FX, pad, stride});
    if (it != h->conv_tuned.end()) {
      px = it->second.first;
      ks = it->second.second;
    }
  }
  return conv2d_impl(h, X, B, IC, H, W, FY, FX, pad, stride, bias, act, Y, stream, px, ks);
}

static sdnn_status conv2d_impl(sdnn_handle h, const float* X, int32_t B, int32_t IC, int32_t H, int32_t W,
                               int32_t FY, int32_t FX, int32_t pad, int32_t stride, const float* bias, int32_t act,
                               float* Y, void* stream, int px_force, int ks_force) {
  if (!h) return fail(SDNN_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (B < 0 || IC < 1 || H < 1 || W < 1 || FY < 1 || FX < 1 || pad < 0 || stride < 1)
    return fail(SDNN_ERR_INVALID_ARGUMENT, "need B >= 0, IC, H, W, FY, FX, stride >= 1 and pad >= 0");
  if (act != SDNN_ACT_NONE && act != SDNN_ACT_RELU) return fail(SDNN_ERR_INVALID_ARGUMENT, "unknown act");
  static const std::pair<int, int> conv_force = [] {  // SDNN_CONV_PX / SDNN_CONV_KS (experiments)
    const char* a = getenv("SDNN_CONV_PX");
    const char* b = getenv("SDNN_CONV_KS");
    return std::make_pair(a ? atoi(a) : 0, b ? atoi(b) : 0);
  }();
  if (px_force <= 0 && (conv_force.first == 2 || conv_force.first == 4)) px_force = conv_force.first;
  if (ks_force <= 0 && conv_force.second > 0) ks_force = conv_force.second;
  if (h->plan.no_split_k && ks_force > 1) ks_force = 1;  // a tuned / forced split never overrides the flag
  const Plan& pl = h->plan;
  if (int64_t(IC) * FY * FX != pl.K)
    return fail(SDNN_ERR_INVALID_ARGUMENT, "handle K = " + std::to_string(pl.K) + " != IC·FY·FX");
  if (pl.kernel != 1 || !pl.split_row.empty())
    return fail(SDNN_ERR_UNSUPPORTED, "sdnn_conv2d needs a row plan without split rows (kernel 0 or 1, "
                                      "SDNN_FLAG_NO_ROW_SPLIT)");
  const int32_t Ho = (H + 2 * pad - FY) / stride + 1, Wo = (W + 2 * pad - FX) / stride + 1;
  if (H + 2 * pad < FY || W + 2 * pad < FX || Ho < 1 || Wo < 1)
    return fail(SDNN_ERR_INVALID_ARGUMENT, "empty output (filter larger than the padded image)");
  const int64_t N = int64_t(B) * Ho * Wo;
  if (N == 0) return SDNN_OK;
  if (!X || !Y) return fail(SDNN_ERR_INVALID_ARGUMENT, "X or Y is NULL");
  if (overlaps(Y, size_t(pl.M) * size_t(N) * 4, X, size_t(IC) * B * H * W * 4) ||
      overlaps(Y, size_t(pl.M) * size_t(N) * 4, bias, size_t(pl.M) * 4))
    return fail(SDNN_ERR_INVALID_ARGUMENT, "Y overlaps X or bias");
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  // explicit form: write the virtual operand Xv (K × N) once, then the TMEM-R SpMM of the handle's
  // TMEM plan.  On the paper's suite (OC ≤ 256, profiles/r02_conv_forms.log) it wins only at 256
  // channels, 14-28 px, 90 % (−8 %, −7 %) and loses up to 1.7× elsewhere: with ≤ 256 filters the
  // 240-row TMEM row blocks run half empty.  So by default only layers with ≥ 480 filters (two full row
  // blocks) and ≥ 8 nonzeros per virtual row take it when the TMEM kernel takes the call;
  // sdnn_conv2d_tune times it as a candidate (px_force = -2), SDNN_CONV_IM2COL=0|1 forces it off / on.
  {
    static const int exp_env = [] {  // SDNN_CONV_IM2COL=0|1 (experiments)
      const char* e = getenv("SDNN_CONV_IM2COL");
      return e ? atoi(e) : -1;
    }();
    const YOut yo1 = y_single(Y, N);
    const bool aligned = N % 4 == 0 && reinterpret_cast<uintptr_t>(Y) % 16 == 0;
    const bool tmem_takes = h->alt && aligned && (tmem_worth(h->alt, reinterpret_cast<const float*>(uintptr_t(256)), N, yo1) ||
                                                  tmem_split_for(h, reinterpret_cast<const float*>(uintptr_t(256)), N, yo1) > 1);
    const bool want = px_force == -2 || (px_force <= 0 && ks_force <= 0 &&
                                         (exp_env >= 0 ? exp_env > 0 : pl.M >= 480 && pl.nnz >= 8 * int64_t(pl.K)));
    if (want && tmem_takes && h->ws_pool) {
      float* xv = nullptr;
      SDNN_CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&xv), size_t(pl.K) * size_t(N) * 4, h->ws_pool,
                                            static_cast<cudaStream_t>(stream)));
      const ConvGeom cg{B, IC, H, W, Ho, Wo, FY, FX, pad, stride};
      im2col_kernel<<<dim3(unsigned((N + 255) / 256), unsigned(pl.K)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
          X, xv, cg, N);
      cudaError_t le = cudaGetLastError();
      sdnn_status st2 = le == cudaSuccess ? SDNN_OK : fail(SDNN_ERR_CUDA, std::string("im2col: ") + cudaGetErrorString(le));
      if (st2 == SDNN_OK) {
        if (const int ks = tmem_split_for(h, xv, N, yo1); ks > 1)
          st2 = launch_tmem(h->alt, xv, N, bias, act, yo1, static_cast<cudaStream_t>(stream), ks, h->ws_pool);
        else
          st2 = launch_tmem(tmem_pick(h, N), xv, N, bias, act, yo1, static_cast<cudaStream_t>(stream));
      }
      cudaFreeAsync(xv, static_cast<cudaStream_t>(stream));
      return st2;
    }
  }
  constexpr int TN = 128;
  const int rw = pl.panel_rows, wc = pl.cta_panels;
  const int64_t nblocks = int64_t(pl.num_row_blocks) * ((N + TN - 1) / TN);
  if (nblocks > 0x7fffffffLL) return fail(SDNN_ERR_UNSUPPORTED, "output too large for one launch");
  KParamsY p{};
  p.meta = h->d_meta;
  p.blk_off = h->d_blk_off;
  p.row_orig = h->d_row_orig;
  p.X = X;
  p.bias = bias;
  p.yo = y_single(Y, N);
  p.Y = Y;
  p.N = N;
  p.K = pl.K;
  p.nch = pl.num_chunks;
  p.kc = pl.k_chunk;
  p.wc = wc;
  p.nrb = pl.num_row_blocks;
  p.x_stage_bytes = int32_t(align_up(int64_t(pl.k_chunk) * TN * 4, 128));
  p.m_stage_bytes = int32_t(align_up(pl.max_block_bytes, 128));
  p.hdr_bytes = int32_t(align_up(int64_t(rw) * wc * 4, 16));
  p.act = act;
  const ConvGeom cg{B, IC, H, W, Ho, Wo, FY, FX, pad, stride};
  // patch form: the largest input window a tile needs (rows of the padded input, all images laid
  // end to end) and the channels a K chunk can touch
  {
    // pixel tile: 4 pixels per lane (128), or 2 (64) when the 128-pixel grid is under one wave and
    // the K range too short for split-K (few input channels: C = 32/64 at 7-28 px, 10-15 % faster;
    // deeper K keeps 128 pixels and splits K instead, profiles/r01_conv_bench.jsonl)
    const int PX = px_force > 0 ? px_force : ((nblocks < h->sms && pl.num_chunks < 16) ? 2 : 4);
    const int64_t TNc = 32 * PX, nb2 = int64_t(pl.num_row_blocks) * ((N + TNc - 1) / TNc);
    const int64_t Hp = int64_t(H) + 2 * pad, HWo = int64_t(Ho) * Wo;
    int64_t rows = 0;
    for (int64_t n0 = 0; n0 < N; n0 += TNc) {
      const int64_t n1 = std::min<int64_t>(n0 + TNc, N) - 1;
      const int64_t b0 = n0 / HWo, oy0 = (n0 - b0 * HWo) / Wo, b1 = n1 / HWo, oy1 = (n1 - b1 * HWo) / Wo;
      rows = std::max<int64_t>(rows, (b1 * Hp + oy1 * stride + FY - 1) - (b0 * Hp + oy0 * stride) + 1);
    }
    // input channels a K chunk touches: kc / (FY·FX) when chunks start on channel boundaries
    // (k_chunk a multiple of FY·FX, e.g. 72 for 3×3), else up to two partial channels more
    const int64_t FYX = int64_t(FY) * FX, ICC = pl.k_chunk % FYX == 0 ? pl.k_chunk / FYX : (pl.k_chunk - 1) / FYX + 2;
    const int64_t Wp = int64_t(W) + 2 * pad;
    const bool v16 = W % 4 == 0 && pad <= 4 && reinterpret_cast<uintptr_t>(X) % 16 == 0;
    const int64_t RS = v16 ? ((4 + int64_t(W) + pad + 3) & ~int64_t(3)) : Wp;
    const size_t stage = align_up(int64_t(ICC * rows * RS * 4 + int64_t(pl.k_chunk) * 4), 128) + size_t(p.m_stage_bytes);
    static const int conv_env = [] {
      const char* e = getenv("SDNN_CONV_GATHER");
      return e ? atoi(e) : 0;
    }();
    const size_t smem2 = 2 * stage + size_t(rows * (v16 ? 2 * (W / 4) : Wp)) * 4;
    if (conv_env == 0 && smem2 <= size_t(kSmemBudget) && rows * Wp < (int64_t(1) << 30)) {
#define SDNN_CONV2(R, X_, V_) reinterpret_cast<const void*>(spmm_conv2_kernel<R, X_, V_>)
      const void* fn2 = rw == 8 ? (PX == 2 ? (v16 ? SDNN_CONV2(8, 2, true) : SDNN_CONV2(8, 2, false))
                                           : (v16 ? SDNN_CONV2(8, 4, true) : SDNN_CONV2(8, 4, false)))
                                : (PX == 2 ? (v16 ? SDNN_CONV2(4, 2, true) : SDNN_CONV2(4, 2, false))
                                           : (v16 ? SDNN_CONV2(4, 4, true) : SDNN_CONV2(4, 4, false)));
#undef SDNN_CONV2
      SDNN_CUDA_TRY(cudaFuncSetAttribute(fn2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
      // split-K as for the row kernel: small images leave the GPU under-filled (few pixel tiles)
      const int64_t warps = nb2 * wc;
      int KS = 1;
      // (a conv chunk stages a whole input patch, so slices of ≥ 2 chunks already pay on a tiny grid:
      // 64 channels at 7×7, 25 → 11 µs, profiles/r01_conv_split.log), up to ~32 warps per SM, a power
      // of two; a 4-chunk K range only on grids under 8 warps per SM (graph-timed conv suite,
      // r01_conv_bench_rules.jsonl: 32 channels at 56 px 24 → 19 µs unsplit; 128 channels at 7 px
      // 19 → 15 µs with 8 slices instead of 4)
      if (ks_force > 0)
        KS = std::min(ks_force, pl.num_chunks);
      else if (!pl.no_split_k && warps <= 12 * int64_t(h->sms) &&
               (pl.num_chunks >= 8 || (pl.num_chunks >= 4 && warps <= 8 * int64_t(h->sms)))) {
        const int64_t ks = std::min<int64_t>({8, pl.num_chunks / 2, 32 * int64_t(h->sms) / warps});
        KS = ks >= 8 ? 8 : ks >= 4 ? 4 : ks >= 2 ? 2 : 1;
      }
      cudaStream_t st_ = static_cast<cudaStream_t>(stream);
      float* kws = nullptr;
      if (KS > 1) SDNN_CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&kws),
                                                        size_t(KS) * pl.M * size_t(N) * 4, h->ws_pool, st_));
      p.kws = kws;
      p.M = pl.M;
      int32_t psr = int32_t(rows), icc = int32_t(ICC);
      void* args2[] = {&p, const_cast<ConvGeom*>(&cg), &psr, &icc};
      cudaError_t le = cudaLaunchKernel(fn2, dim3(unsigned(nb2), unsigned(KS)), dim3(unsigned(wc * 32)), args2,
                                        smem2, st_);
      if (le == cudaSuccess && KS > 1) {
        launch_splitk_reduce(kws, KS, pl.M, bias, act, y_single(Y, N), N, st_);
        le = cudaGetLastError();
      }
      if (KS > 1) cudaFreeAsync(kws, st_);
      if (le != cudaSuccess) return fail(SDNN_ERR_CUDA, std::string("sdnn_conv2d: ") + cudaGetErrorString(le));
      return SDNN_OK;
    }
  }
  // gather form (very wide images, or SDNN_CONV_GATHER=1): the virtual matrix itself is staged
  if (wc < 4) return fail(SDNN_ERR_UNSUPPORTED, "the gather form of sdnn_conv2d needs >= 4 panels per CTA");
  const size_t smem = 2 * size_t(p.x_stage_bytes) + 2 * size_t(p.m_stage_bytes);
  if (smem > size_t(kSmemBudget)) return fail(SDNN_ERR_INTERNAL, "conv stage does not fit shared memory");
  const bool vec = N % 4 == 0 && reinterpret_cast<uintptr_t>(Y) % 16 == 0;
  const void* fn = rw == 8 ? (vec ? reinterpret_cast<const void*>(spmm_conv_kernel<8, true>)
                                  : reinterpret_cast<const void*>(spmm_conv_kernel<8, false>))
                           : (vec ? reinterpret_cast<const void*>(spmm_conv_kernel<4, true>)
                                  : reinterpret_cast<const void*>(spmm_conv_kernel<4, false>));
  SDNN_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  void* args[] = {&p, const_cast<ConvGeom*>(&cg)};
  SDNN_CUDA_TRY(cudaLaunchKernel(fn, dim3(unsigned(nblocks)), dim3(unsigned(wc * 32)), args, smem,
                                 static_cast<cudaStream_t>(stream)));
  return SDNN_OK;
}

sdnn_status sdnn_spmm_host(sdnn_handle h, const float* X_host, int64_t N, const float* bias_host, int32_t act,
                           float* Y_host, int64_t block_cols) {
  if (!h) return fail(SDNN_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (N < 0 || block_cols < 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "N < 0 or block_cols < 0");
  if (act != SDNN_ACT_NONE && act != SDNN_ACT_RELU) return fail(SDNN_ERR_INVALID_ARGUMENT, "unknown act");
  if (N == 0) return SDNN_OK;
  if (!X_host || !Y_host) return fail(SDNN_ERR_INVALID_ARGUMENT, "X or Y is NULL");
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  const int64_t M = h->plan.M, K = h->plan.K;
  int64_t nc = block_cols;
  if (nc == 0) {  // ~128 MiB of X+Y per block, multiple of 512 columns (a TMEM N tile)
    nc = std::max<int64_t>(512, (int64_t(128) << 20) / ((M + K) * 4) / 512 * 512);
  }
  nc = std::min(nc, N);
  // The staging state (streams, events, two X/Y block buffers, bias) lives in the handle and is
  // reused by every call; calls on one handle are serialised on its mutex.
  std::lock_guard<std::mutex> lk(h->host_mu);
  HostStage& hs = h->hs;
  sdnn_status rs = SDNN_OK;
  std::string msg;
  auto ck = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rs == SDNN_OK) {
      rs = e == cudaErrorMemoryAllocation ? SDNN_ERR_OUT_OF_MEMORY : SDNN_ERR_CUDA;
      msg = std::string(what) + ": " + cudaGetErrorString(e);
    }
    return rs == SDNN_OK;
  };
  if (!hs.s[0]) {
    for (int i = 0; i < 3 && rs == SDNN_OK; ++i) {
      ck(cudaStreamCreateWithFlags(&hs.s[i], cudaStreamNonBlocking), "cudaStreamCreate");
      for (int b = 0; b < kHostBufs && rs == SDNN_OK; ++b)
        ck(cudaEventCreateWithFlags(&hs.ev[i][b], cudaEventDisableTiming), "cudaEventCreate");
    }
    if (rs == SDNN_OK) ck(cudaMalloc(reinterpret_cast<void**>(&hs.bias), size_t(M * 4)), "cudaMalloc(bias)");
  }
  if (rs == SDNN_OK && hs.cols < nc) {
    ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    for (int b = 0; b < kHostBufs; ++b) {
      cudaFree(hs.x[b]);
      cudaFree(hs.y[b]);
      hs.x[b] = hs.y[b] = nullptr;
    }
    hs.cols = 0;
    for (int b = 0; b < kHostBufs && rs == SDNN_OK; ++b) {
      ck(cudaMalloc(reinterpret_cast<void**>(&hs.x[b]), size_t(K * nc * 4)), "cudaMalloc(X block)");
      if (rs == SDNN_OK) ck(cudaMalloc(reinterpret_cast<void**>(&hs.y[b]), size_t(M * nc * 4)), "cudaMalloc(Y block)");
    }
    if (rs == SDNN_OK) hs.cols = nc;
  }
  cudaStream_t* s = hs.s;
  const float* bd = nullptr;
  if (rs == SDNN_OK && bias_host) {
    ck(cudaMemcpyAsync(hs.bias, bias_host, size_t(M * 4), cudaMemcpyHostToDevice, s[1]), "cudaMemcpyAsync(bias)");
    bd = hs.bias;
  }
  if (rs == SDNN_OK) {
    // s[0]: H2D copies, s[1]: kernels, s[2]: D2H copies.  ev[0][b]: X block in buffer b ready;
    // ev[1][b]: kernel on buffer b done; ev[2][b]: Y buffer b drained to host.
    for (int b = 0; b < kHostBufs; ++b) {
      ck(cudaEventRecord(hs.ev[1][b], s[1]), "cudaEventRecord");
      ck(cudaEventRecord(hs.ev[2][b], s[1]), "cudaEventRecord");
    }
    int i = 0;
    for (int64_t c0 = 0; c0 < N && rs == SDNN_OK; c0 += nc, ++i) {
      const int b = i % kHostBufs;
      const int64_t w = std::min(nc, N - c0);
      ck(cudaStreamWaitEvent(s[0], hs.ev[1][b], 0), "cudaStreamWaitEvent");
      ck(cudaMemcpy2DAsync(hs.x[b], size_t(w * 4), X_host + c0, size_t(N * 4), size_t(w * 4), size_t(K),
                           cudaMemcpyHostToDevice, s[0]), "cudaMemcpy2DAsync(X)");
      ck(cudaEventRecord(hs.ev[0][b], s[0]), "cudaEventRecord");
      ck(cudaStreamWaitEvent(s[1], hs.ev[0][b], 0), "cudaStreamWaitEvent");
      ck(cudaStreamWaitEvent(s[1], hs.ev[2][b], 0), "cudaStreamWaitEvent");
      if (rs == SDNN_OK) {
        sdnn_status ls = launch(h, hs.x[b], w, bd, act, y_single(hs.y[b], w), s[1]);
        if (ls != SDNN_OK) { rs = ls; msg = sdnn_last_error_message(); }
      }
      ck(cudaEventRecord(hs.ev[1][b], s[1]), "cudaEventRecord");
      ck(cudaStreamWaitEvent(s[2], hs.ev[1][b], 0), "cudaStreamWaitEvent");
      ck(cudaMemcpy2DAsync(Y_host + c0, size_t(N * 4), hs.y[b], size_t(w * 4), size_t(w * 4), size_t(M),
                           cudaMemcpyDeviceToHost, s[2]), "cudaMemcpy2DAsync(Y)");
      ck(cudaEventRecord(hs.ev[2][b], s[2]), "cudaEventRecord");
    }
  }
  for (int i = 0; i < 3; ++i)
    if (s[i]) ck(cudaStreamSynchronize(s[i]), "cudaStreamSynchronize");
  if (rs != SDNN_OK) return fail(rs, msg);
  return SDNN_OK;
}

sdnn_status sdnn_spmm_kernel(sdnn_handle h, int64_t N, const float* X, const float* Y, int32_t* kernel) {
  if (!h || !kernel || N < 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL handle / kernel or N < 0");
  const YOut yo = y_single(const_cast<float*>(Y), N);
  sdnn_handle_s::Tuned t;
  if (tuned_for(h, X, N, yo, &t) && t.path >= 0) {
    *kernel = t.path == 0 ? (h->alt ? h->alt->plan.kernel : h->plan.kernel) : 1;
    return SDNN_OK;
  }
  if (tmem_worth(h->alt, X, N, yo) || tmem_split_for(h, X, N, yo) > 1) {
    *kernel = h->alt->plan.kernel;
    return SDNN_OK;
  }
  if (sdnn_handle_s* nw = narrow_pick(h, N)) return sdnn_spmm_kernel(nw, N, X, Y, kernel);
  const int k = h->plan.kernel;
  const bool tma = N % 4 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 && y_aligned16(yo);
  *kernel = (k == 4 || k == 5 || k == 6) ? (N % tmem_n_align(k) == 0 && tma ? k : -k) : (k == 3 || tma) ? k : -k;
  return SDNN_OK;
}

sdnn_status sdnn_get_permutation(sdnn_handle h, int32_t* out_perm) {
  if (!h || !out_perm) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL handle or out_perm");
  std::memcpy(out_perm, h->plan.perm.data(), h->plan.perm.size() * 4);
  return SDNN_OK;
}

sdnn_status sdnn_get_info(sdnn_handle h, sdnn_info* info) {
  if (!h || !info) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL handle or info");
  if (info->struct_size != sizeof(sdnn_info)) return fail(SDNN_ERR_INVALID_ARGUMENT, "sdnn_info.struct_size mismatch");
  plan_fill_info(h->plan, h->device, info);
  info->meta_bytes = h->plan.meta_size_uploaded;
  info->alt_kernel = h->alt ? h->alt->plan.kernel : 0;
  info->narrow_row_blocks = h->narrow ? h->narrow->plan.num_row_blocks : 0;
  info->narrow4_row_blocks = h->narrow4 ? h->narrow4->plan.num_row_blocks : 0;
  return SDNN_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// Serialization of a prepared handle (the paper's reusable preparation): every plan
// of the handle (main, TMEM, narrow, narrow4) with its packed metadata, so a process can skip
// Algorithm 1 and the packing.  Blob: "SDNNPLAN", u32 version, u32 plan count, then per plan a u32
// role (0 main, 1 TMEM, 2 narrow, 3 narrow4) and its fields in a fixed order (little-endian, sizes as u64).
namespace {
constexpr uint32_t kBlobVersion = 2;  // 2: role 4 = the second TMEM plan
struct BlobW {
  std::vector<uint8_t> b;
  template <class T> void s(const T& v) {
    const uint8_t* q = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), q, q + sizeof(T));
  }
  template <class T> void v(const std::vector<T>& x) {
    s<uint64_t>(x.size());
    const uint8_t* q = reinterpret_cast<const uint8_t*>(x.data());
    b.insert(b.end(), q, q + x.size() * sizeof(T));
  }
};
struct BlobR {
  const uint8_t* p;
  size_t n, off = 0;
  bool ok = true;
  template <class T> void s(T& v) {
    if (!ok || off + sizeof(T) > n) { ok = false; return; }
    std::memcpy(&v, p + off, sizeof(T));
    off += sizeof(T);
  }
  template <class T> void v(std::vector<T>& x) {
    uint64_t m = 0;
    s(m);
    if (!ok || m > (n - off) / sizeof(T)) { ok = false; return; }
    x.resize(size_t(m));
    std::memcpy(x.data(), p + off, size_t(m) * sizeof(T));
    off += size_t(m) * sizeof(T);
  }
};
template <class IO> void plan_fields(IO& io, Plan& p) {
  io.s(p.M); io.s(p.K); io.s(p.nnz); io.s(p.permuted); io.s(p.permuted_output); io.s(p.no_split_k);
  io.s(p.kernel); io.s(p.group_entries); io.s(p.group_sb); io.s(p.group_subblocks); io.s(p.panel_rows);
  io.s(p.cta_panels); io.s(p.num_panels); io.s(p.num_row_blocks); io.s(p.k_chunk); io.s(p.num_chunks);
  io.s(p.max_block_bytes); io.s(p.max_panel_nnz); io.s(p.tmem_fill);
  io.v(p.perm); io.v(p.row_orig); io.v(p.blk_off); io.v(p.meta);
  io.v(p.piece_row); io.v(p.piece_begin); io.v(p.piece_end); io.v(p.split_row); io.v(p.split_first);
  io.v(p.split_count);
}
// A handle's plan with its metadata copied back from the device (the host copy is freed at upload).
sdnn_status plan_with_meta(const sdnn_handle_s* h, Plan& out) {
  out = h->plan;
  out.meta.resize(size_t(h->plan.meta_size_uploaded));
  if (!out.meta.empty()) SDNN_CUDA_TRY(cudaMemcpy(out.meta.data(), h->d_meta, out.meta.size(), cudaMemcpyDeviceToHost));
  return SDNN_OK;
}
// Structural checks of a deserialized plan before it is uploaded and launched.
bool plan_sane(const Plan& p, uint32_t role) {
  if (p.M < 1 || p.K < 1 || p.kernel < 1 || p.kernel > 6 || p.kernel == 3) return false;
  // plan kind per role: 0 main (row / group / TMEM), 1 TMEM alternative, 2-3 narrow row plans, 4 the
  // second TMEM plan of an auto handle (TMEM-R only: tmem_pick compares it with role 1)
  if ((role == 1 && p.kernel != 4 && p.kernel != 5 && p.kernel != 6) || ((role == 2 || role == 3) && p.kernel != 1) ||
      (role == 4 && p.kernel != 4))
    return false;
  if (p.perm.size() != size_t(p.M) || p.num_row_blocks < 1 || p.num_chunks < 1 || p.k_chunk < 1) return false;
  if (p.num_chunks != (p.K + p.k_chunk - 1) / p.k_chunk) return false;
  // panel geometry the kernels are compiled for
  if (p.num_panels != int64_t(p.num_row_blocks) * p.cta_panels) return false;
  if ((p.kernel == 4 || p.kernel == 6) &&
      (p.panel_rows != tmem_rows(4) || p.cta_panels != kTmemRWarps || p.k_chunk != tmem_kc(4)))
    return false;
  if (p.kernel == 5 && (p.panel_rows != tmem_rows(8) || p.cta_panels != kTmemPanels || p.k_chunk != tmem_kc(8)))
    return false;
  if (p.kernel == 1 && ((p.panel_rows != 4 && p.panel_rows != 8) || p.cta_panels < 1 || p.cta_panels > 16)) return false;
  if (p.kernel == 2 && (p.panel_rows != 16 || p.cta_panels < 1 || p.cta_panels > kMaxGroupWarps)) return false;
  if (p.blk_off.size() != size_t(p.num_row_blocks) * size_t(p.num_chunks) + 1) return false;
  if (p.row_orig.size() != size_t(p.num_panels) * size_t(p.panel_rows)) return false;
  if (p.blk_off.front() != 0 || p.blk_off.back() != int64_t(p.meta.size())) return false;
  if (p.max_block_bytes < 16) return false;
  // the stage ring the launch sizes from max_block_bytes must fit shared memory
  const int mstage = int(align_up(p.max_block_bytes, 128));
  if ((p.kernel == 4 || p.kernel == 6) && tmemr_smem_bytes(mstage) > size_t(kSmemBudget) + 1024) return false;
  if (p.kernel == 5 && tmem_smem_bytes(mstage) > size_t(kSmemBudget) + 1024) return false;
  if ((p.kernel == 1 || p.kernel == 2) && int64_t(p.k_chunk) * kMaxTN * 4 + mstage > kSmemBudget) return false;
  for (size_t i = 1; i < p.blk_off.size(); ++i)
    if (p.blk_off[i] < p.blk_off[i - 1] || p.blk_off[i] - p.blk_off[i - 1] > p.max_block_bytes ||
        p.blk_off[i] % 16)
      return false;
  // split rows: piece tables of one length, split ranges inside them, output rows inside Y
  if (p.piece_begin.size() != p.piece_row.size() || p.piece_end.size() != p.piece_row.size()) return false;
  if (p.split_first.size() != p.split_row.size() || p.split_count.size() != p.split_row.size()) return false;
  if (p.kernel != 1 && !p.piece_row.empty()) return false;
  for (size_t i = 0; i < p.split_row.size(); ++i)
    if (p.split_row[i] < 0 || p.split_row[i] >= p.M || p.split_first[i] < 0 || p.split_count[i] < 1 ||
        int64_t(p.split_first[i]) + p.split_count[i] > int64_t(p.piece_row.size()))
      return false;
  for (int32_t r : p.row_orig)
    if (r >= p.M || (r <= -2 && size_t(-2 - int64_t(r)) >= p.piece_row.size())) return false;
  // kernel 6 (row pairs): per slot pair, the shared (16-byte) entries and both own lists inside the
  // block, contiguous, TMEM columns with the warp's lane base
  if (p.kernel == 6) {
    const int64_t rcta = int64_t(p.panel_rows) * p.cta_panels;
    const int64_t hdr = align_up(rcta * 4, 16);
    for (int64_t b = 0; b + 1 < int64_t(p.blk_off.size()); ++b) {
      const int64_t bytes = p.blk_off[b + 1] - p.blk_off[b];
      if (bytes < hdr) return false;
      const uint8_t* blk = p.meta.data() + p.blk_off[b];
      const int64_t nent = (bytes - hdr) / 8;
      for (int64_t sl = 0; sl < rcta; sl += 2) {
        uint32_t ha, hb;
        std::memcpy(&ha, blk + sl * 4, 4);
        std::memcpy(&hb, blk + sl * 4 + 4, 4);
        const int64_t start = ha >> 16, ns = (ha >> 8) & 0xffu, na = ha & 0xffu, b0 = hb >> 16, nb = hb & 0xffu;
        if (start % 2 || na % 2 || nb % 2 || b0 != start + 2 * ns + na || b0 + nb > nent) return false;
        const uint32_t lb = uint32_t(32 * ((sl / p.panel_rows) & 3)) << 16;
        for (int64_t e = start; e < b0 + nb; ++e) {
          if (e < start + 2 * ns && (e - start) % 2) continue;  // second half of a shared entry {w_b, 0}
          uint32_t c;
          std::memcpy(&c, blk + hdr + e * 8, 4);
          if ((c & ~0xffffu) != lb || (c & 0xffffu) >= 512u || (c & 0xffu) % 4u) return false;
        }
      }
    }
    return true;
  }
  // row-format metadata (row / TMEM kernels): every slot's segment inside its block, columns inside
  // the chunk (the kernels index shared / tensor memory with them)
  if (p.kernel != 2) {
    const int64_t rcta = int64_t(p.panel_rows) * p.cta_panels;
    const int64_t hdr = align_up(rcta * 4, 16);
    const int V = (p.kernel == 4 || p.kernel == 5) ? tmem_v(p.kernel) : 0;
    for (int64_t b = 0; b + 1 < int64_t(p.blk_off.size()); ++b) {
      const int64_t bytes = p.blk_off[b + 1] - p.blk_off[b];
      if (bytes < hdr) return false;
      const uint8_t* blk = p.meta.data() + p.blk_off[b];
      const int64_t nent = (bytes - hdr) / 8;
      for (int64_t sl = 0; sl < rcta; ++sl) {
        uint32_t h;
        std::memcpy(&h, blk + sl * 4, 4);
        const int64_t start = h >> 16, cnt = V ? (h & 0xffu) : (h & 0xffffu), runs = V ? (h >> 8) & 0xffu : 0;
        if (start + cnt + (cnt & 1) > nent || 4 * runs > cnt || (V && (start % 2 || cnt % 2))) return false;
        for (int64_t e = start; e < start + cnt; ++e) {
          uint32_t c;
          std::memcpy(&c, blk + hdr + e * 8, 4);
          if (V) {  // TMEM column V·k + 256·half | lane base of the slot's warp (kernel 4)
            const uint32_t lb = p.kernel == 4 ? uint32_t(32 * ((sl / p.panel_rows) & 3)) << 16 : 0u;
            if ((c & ~0xffffu) != lb || (c & 0xffffu) >= 512u || (c & 0xffu) % uint32_t(V)) return false;
          } else if (c >= uint32_t(p.k_chunk)) {
            return false;
          }
        }
      }
    }
  }
  return true;
}
}  // namespace

extern "C" {

sdnn_status sdnn_serialize(sdnn_handle h, void* buf, size_t* size) {
  if (!h || !size) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL handle or size");
  const sdnn_handle_s* parts[5] = {h, h->alt, h->narrow, h->narrow4, h->alt ? h->alt2 : nullptr};
  for (const sdnn_handle_s* q : parts)
    if (q && q->plan.kernel == 3)
      return fail(SDNN_ERR_UNSUPPORTED, "codegen plans are JIT-compiled from the CSR and are not serialized");
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  BlobW w;
  try {
    const char magic[8] = {'S', 'D', 'N', 'N', 'P', 'L', 'A', 'N'};
    w.b.insert(w.b.end(), magic, magic + 8);
    w.s(kBlobVersion);
    uint32_t count = 0;
    for (const sdnn_handle_s* q : parts) count += q ? 1 : 0;
    w.s(count);
    for (uint32_t role = 0; role < 5; ++role) {
      if (!parts[role]) continue;
      Plan pl;
      st = plan_with_meta(parts[role], pl);
      if (st != SDNN_OK) return st;
      w.s(role);
      plan_fields(w, pl);
    }
  } catch (const std::bad_alloc&) {
    return fail(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed");
  }
  if (!buf) {
    *size = w.b.size();
    return SDNN_OK;
  }
  if (*size < w.b.size()) {
    const size_t have = *size;
    *size = w.b.size();
    return fail(SDNN_ERR_INVALID_ARGUMENT, "buffer of " + std::to_string(have) + " bytes < " + std::to_string(w.b.size()));
  }
  std::memcpy(buf, w.b.data(), w.b.size());
  *size = w.b.size();
  return SDNN_OK;
}

sdnn_status sdnn_deserialize(const void* buf, size_t size, sdnn_handle* out) {
  if (!buf || !out) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL buffer or out");
  *out = nullptr;
  BlobR r{static_cast<const uint8_t*>(buf), size};
  if (size < 16 || std::memcmp(buf, "SDNNPLAN", 8) != 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "not an sdnn blob");
  r.off = 8;
  uint32_t ver = 0, count = 0;
  r.s(ver);
  r.s(count);
  if (!r.ok || ver != kBlobVersion) return fail(SDNN_ERR_UNSUPPORTED, "blob version " + std::to_string(ver) + " != " + std::to_string(kBlobVersion));
  if (count < 1 || count > 5) return fail(SDNN_ERR_INVALID_ARGUMENT, "corrupt blob (plan count)");
  sdnn_handle parts[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  auto cleanup = [&](sdnn_status s, const std::string& m) {
    for (auto& q : parts)
      if (q) sdnn_destroy(q);
    return fail(s, m);
  };
  try {
    for (uint32_t i = 0; i < count; ++i) {
      uint32_t role = 5;
      r.s(role);
      Plan pl;
      plan_fields(r, pl);
      if (!r.ok || role > 4 || parts[role] || (role == 3 && !parts[2]) || (role == 4 && !parts[1]) ||
          !plan_sane(pl, role) || (role == 0) != (i == 0) ||
          (role == 4 && (pl.M != parts[1]->plan.M || pl.K != parts[1]->plan.K || parts[1]->plan.kernel != 4)))
        return cleanup(SDNN_ERR_INVALID_ARGUMENT, "corrupt blob (plan " + std::to_string(i) + ")");
      sdnn_status st = prepare_one(nullptr, nullptr, nullptr, pl.M, pl.K, nullptr, &parts[role], nullptr, &pl);
      if (st != SDNN_OK) {
        std::string m = sdnn_last_error_message();
        return cleanup(st, m);
      }
    }
  } catch (const std::bad_alloc&) {
    return cleanup(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed");
  }
  if (r.off != size) return cleanup(SDNN_ERR_INVALID_ARGUMENT, "corrupt blob (trailing bytes)");
  parts[0]->alt = parts[1];
  parts[0]->alt2 = parts[4];
  parts[0]->narrow = parts[2];
  parts[0]->narrow4 = parts[3];
  *out = parts[0];
  return SDNN_OK;
}

}  // extern "C"

extern "C" {

// sdnn_tune: time every applicable path for this N (TMEM plan, row plan, narrow row plans, each with
// split-K 1/2/4/8) on the caller's buffers and keep the fastest for later calls with this N
// (the paper's per-matrix autotuning).  Synchronises the stream.
sdnn_status sdnn_tune(sdnn_handle h, const float* X, int64_t N, float* Y, void* stream, int32_t* path_out,
                      float* us_out) {
  if (!h || !X || !Y || N <= 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL handle / buffer or N <= 0");
  if (h->plan.kernel == 3) return fail(SDNN_ERR_UNSUPPORTED, "codegen handles are not tuned");
  const YOut yo = y_single(Y, N);
  if (N % 4 || reinterpret_cast<uintptr_t>(X) % 16 || !y_aligned16(yo))
    return fail(SDNN_ERR_INVALID_ARGUMENT, "sdnn_tune needs N % 4 == 0 and 16-byte aligned X and Y");
  sdnn_status st = check_device(h);
  if (st != SDNN_OK) return st;
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  std::vector<sdnn_handle_s::Tuned> cands{{-1, 0}};  // the built-in rules first (ties keep them)
  const bool has_tmem = (h->alt || h->plan.kernel == 4 || h->plan.kernel == 5 || h->plan.kernel == 6) &&
                        N % tmem_n_align(h->alt ? h->alt->plan.kernel : h->plan.kernel) == 0;
  const bool row_ok = h->plan.kernel == 1 || h->plan.kernel == 2;
  // TMEM split-K slices are cut at even chunks and keep ≥ 2 chunk pairs each (launch_tmem caps KS):
  // candidates beyond that cap would repeat a smaller KS
  const Plan& tp = h->alt ? h->alt->plan : h->plan;
  const int tmem_ks_max = std::max(1, ((tp.num_chunks + 1) / 2) / 2);
  for (int ks : {1, 2, 4, 8}) {
    if (ks > 1 && h->plan.no_split_k) break;  // SDNN_FLAG_NO_SPLIT_K: never split the K range
    if (has_tmem && (ks == 1 || ks <= tmem_ks_max)) cands.push_back({0, ks});
    if (row_ok) cands.push_back({1, ks});
    if (h->narrow) cands.push_back({2, ks});
    if (h->narrow4) cands.push_back({3, ks});
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  SDNN_CUDA_TRY(cudaEventCreate(&e0));
  SDNN_CUDA_TRY(cudaEventCreate(&e1));
  float best = 0.f;
  sdnn_handle_s::Tuned pick;
  for (const auto& c : cands) {
    if (c.path == 1 && c.ks > 1 && !h->plan.split_row.empty()) continue;  // split rows: no split-K
    st = launch_path(h, c, X, N, nullptr, SDNN_ACT_NONE, yo, sm);          // warm-up
    if (st != SDNN_OK && &c != &cands.front() && cudaPeekAtLastError() == cudaSuccess) {
      st = SDNN_OK;  // a candidate this call cannot launch (e.g. a grid limit): skip it, keep tuning
      continue;
    }
    if (st != SDNN_OK) break;
    cudaEventRecord(e0, sm);
    for (int r = 0; r < 5 && st == SDNN_OK; ++r) st = launch_path(h, c, X, N, nullptr, SDNN_ACT_NONE, yo, sm);
    cudaEventRecord(e1, sm);
    if (st != SDNN_OK) break;
    cudaError_t ce = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e0, e1);
    if (ce != cudaSuccess) {
      st = fail(SDNN_ERR_CUDA, std::string("sdnn_tune: ") + cudaGetErrorString(ce));
      break;
    }
    if (&c == &cands.front() || ms < 0.97f * best) {  // a path must beat the rules by > 3 %
      best = ms;
      pick = c;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != SDNN_OK) return st;
  {
    std::lock_guard<std::mutex> lk(h->tune_mu);
    h->tuned[N] = pick;
  }
  if (path_out) *path_out = pick.path < 0 ? -1 : pick.path * 16 + pick.ks;
  if (us_out) *us_out = best * 1000.f / 5.f;
  return SDNN_OK;
}

}  // extern "C"

extern "C" {

// sdnn_conv2d_tune: time sdnn_conv2d's tile choices for this geometry (the built-in rules, then
// 2 / 4 pixels per lane × 1 / 2 / 4 / 8 K slices) and keep the fastest (> 3 % better than the
// rules) for later calls with the same geometry.  Synchronises the stream.
sdnn_status sdnn_conv2d_tune(sdnn_handle h, const float* X, int32_t B, int32_t IC, int32_t H, int32_t W, int32_t FY,
                             int32_t FX, int32_t pad, int32_t stride, float* Y, void* stream, int32_t* choice_out,
                             float* us_out) {
  if (!h || !X || !Y) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL handle or buffer");
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  std::vector<std::pair<int, int>> cands{{-1, -1}};
  for (int px : {4, 2})
    for (int ks : {1, 2, 4, 8})
      if (ks == 1 || !h->plan.no_split_k) cands.emplace_back(px, ks);  // SDNN_FLAG_NO_SPLIT_K: never split
  if (h->alt) cands.emplace_back(-2, 0);  // the explicit form: virtual operand written out + TMEM-R SpMM
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  SDNN_CUDA_TRY(cudaEventCreate(&e0));
  SDNN_CUDA_TRY(cudaEventCreate(&e1));
  float best = 0.f;
  std::pair<int, int> pick{-1, -1};
  sdnn_status st = SDNN_OK;
  for (size_t i = 0; i < cands.size(); ++i) {
    const auto c = cands[i];
    st = conv2d_impl(h, X, B, IC, H, W, FY, FX, pad, stride, nullptr, SDNN_ACT_NONE, Y, stream, c.first, c.second);
    if (st != SDNN_OK) break;
    cudaEventRecord(e0, sm);
    for (int r = 0; r < 5 && st == SDNN_OK; ++r)
      st = conv2d_impl(h, X, B, IC, H, W, FY, FX, pad, stride, nullptr, SDNN_ACT_NONE, Y, stream, c.first, c.second);
    cudaEventRecord(e1, sm);
    if (st != SDNN_OK) break;
    cudaError_t ce = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e0, e1);
    if (ce != cudaSuccess) {
      st = fail(SDNN_ERR_CUDA, std::string("sdnn_conv2d_tune: ") + cudaGetErrorString(ce));
      break;
    }
    if (i == 0 || ms < 0.97f * best) {
      best = ms;
      pick = c;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != SDNN_OK) return st;
  {
    std::lock_guard<std::mutex> lk(h->tune_mu);
    h->conv_tuned[{B, IC, H, W, FY, FX, pad, stride}] = pick;
  }
  if (choice_out) *choice_out = pick.first == -2 ? -2 : pick.first < 0 ? -1 : pick.first * 16 + pick.second;
  if (us_out) *us_out = best * 1000.f / 5.f;
  return SDNN_OK;
}

}  // extern "C"
