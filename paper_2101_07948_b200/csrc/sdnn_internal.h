// sdnn_internal.h — shared by the product sources of libsdnn only (never by oracle/).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/sdnn.h"

namespace sdnn {

// Thread-local error detail behind sdnn_last_error_message().
void set_error(const std::string& msg);
sdnn_status fail(sdnn_status s, const std::string& msg);

// Host-side result of preparation ("execution-ordered format"):
//   row_orig[num_panels * panel_rows]  original row per panel slot (−1: empty slot)
//   blk_off[num_row_blocks * num_chunks + 1]  byte offsets of the (row block, chunk) blocks in meta
//   meta: per block, a header of R_cta = cta_panels·panel_rows uint32 words
//         (start_entry << 16 | count) padded to 16 B, then 8-byte entries {uint32 col_local, float w}
//         with every row segment starting at an even entry (16-byte aligned pairs).
struct Plan {
  int32_t M = 0, K = 0;
  int64_t nnz = 0;
  int32_t permuted = 0;
  int32_t permuted_output = 0;  // SDNN_FLAG_PERMUTED_OUTPUT: row_orig / split_row hold plan positions
  int32_t no_split_k = 0;       // SDNN_FLAG_NO_SPLIT_K: the row kernel never splits K across CTAs
  int32_t kernel = 1;          // 1 = row kernel, 2 = group kernel
  int64_t group_entries = 0;   // union entries of the group format
  int32_t group_sb = 0;        // group kernel sub-block rows (1, 2 or 4)
  int64_t group_subblocks = 0; // nonzero sub-blocks over all entries
  int32_t panel_rows = 0, cta_panels = 0, num_panels = 0, num_row_blocks = 0;
  int32_t k_chunk = 0, num_chunks = 0;
  int32_t max_block_bytes = 0;
  int64_t max_panel_nnz = 0;
  int64_t meta_size_uploaded = 0;
  std::vector<int32_t> perm;      // order[i] = original row at permuted position i
  std::vector<int32_t> row_orig;
  std::vector<int64_t> blk_off;
  std::vector<uint8_t> meta;
  // codegen kernel (kernel == 3): row panels (original row ids, Algorithm 1 order) baked into code
  std::vector<std::vector<int32_t>> cg_panels;
  int32_t cg_warps = 0, cg_prefetch = 0;
  int32_t tmem_fill = 1;       // TMEM kernels: 1 = filler warps (tcgen05.st), 0 = tcgen05.cp
  // row plan: heavy rows split into pieces (contiguous CSR entry ranges) that the LPT places like
  // rows; a piece's slot has row_orig = −2 − piece id and its partial sums go to a workspace row
  // that split_reduce_kernel adds up (piece order) before the bias and activation.
  std::vector<int32_t> piece_row, piece_begin, piece_end;
  std::vector<int32_t> split_row, split_first, split_count;
};

sdnn_status validate_csr(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K);
// Algorithm 1 with an inverted index; order must hold M entries.
void algorithm1(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K, int32_t* order);
std::string codegen_panel_ptx(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals,
                              const std::vector<int32_t>& rows, int32_t K, int32_t warps, int32_t D,
                              const std::string& name);
}  // namespace sdnn
#include <cuda.h>
namespace sdnn {
// Driver-API entry points, resolved at run time through cudaGetDriverEntryPoint so that libsdnn
// does not link libcuda (the CPU-only container has none; tests load the library there).
struct DriverApi {
  CUresult (*moduleLoadDataEx)(CUmodule*, const void*, unsigned, CUjit_option*, void**) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*moduleUnload)(CUmodule) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                           void**, void**) = nullptr;
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
  CUresult (*ctxGetCurrent)(CUcontext*) = nullptr;
  CUresult (*ctxSetCurrent)(CUcontext) = nullptr;
  bool ok = false;
};
const DriverApi& driver();
sdnn_status codegen_build(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t K,
                          const std::vector<std::vector<int32_t>>& panels, int32_t warps, int32_t D,
                          std::vector<CUmodule>& mods, std::vector<CUfunction>& funcs, int32_t threads);
// perm: a permutation already computed for this matrix (another plan of the same handle), so
// Algorithm 1 runs once per handle; nullptr → computed here (or identity when opts->permute = 0).
sdnn_status build_plan(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                       const sdnn_perm_opts* opts, Plan& plan, const std::vector<int32_t>* perm = nullptr);

// Shared-memory budget used for the X/metadata stage ring (bytes) and the fixed CTA layout.
constexpr int kSmemBudget = 220 * 1024;
constexpr int kMaxTN = 256;  // widest N tile (V = 8 floats per lane)
constexpr int kMaxGroupWarps = 11;  // group kernel: consumer warps per CTA (register budget)
constexpr int kCgMaxRows = 128;     // codegen kernel: accumulators (rows) per panel
constexpr int kCgWarps = 6;         // codegen kernel: warps per CTA (2 CTAs/SM at <= 168 registers)
constexpr int kCgPrefetch = 24;     // codegen kernel: X columns in flight per lane

// TMEM kernels (sdnn_spmm.cu): the X tile lives in tensor memory.
//   kernel 4 ("tmem", V = 4, replicated lane quarters): every TMEM lane quarter holds the same 128
//     columns of N (lane 32q + l ↔ n0 + 4l .. 4l+3; TMEM column 4·k_local + v + 256·half), and the 24
//     consumer warps each own their own tmem_rows(4) = 10-row panel (240 rows per CTA), so the X
//     tile staged once serves 4× the rows of a non-replicated layout (a quarter of the L2 → SM fill
//     traffic) and the TMEM lane base of warp w's quarter (w % 4) is packed into its metadata.
//     Row segments are padded to whole pairs (tmem_pad(4) = 2).
//   kernel 5 ("tmem8", V = 8): lane L ↔ columns n0 + 4L + v and n0 + 512 + 4L + v (N tile 1024),
//     6 warp slots × 5 rows shared by the 4 quarters (30 rows per CTA), segments padded to pairs.
// K chunk = one TMEM half of 256 columns (256 / V K rows), double-buffered.
#ifdef __CUDACC__
#define SDNN_HD __host__ __device__
#else
#define SDNN_HD
#endif
SDNN_HD constexpr int tmem_rows(int V) { return V == 4 ? 10 : 5; }
SDNN_HD constexpr int tmem_kc(int V) { return 256 / V; }
SDNN_HD constexpr int tmem_pad(int V) { return 2; }  // row segments padded to whole pairs
constexpr int kTmemPanels = 6;        // kernel 5: warp slots per lane quarter
constexpr int kTmemRWarps = 24;       // kernel 4: consumer warps (= panels per row block)
constexpr int kTmemPieces = 4;        // kernel 5: smem ring depth (32 KB TMA pieces)
#ifndef SDNN_TMEMR_PIECES
#define SDNN_TMEMR_PIECES 8
#endif
// kernel 4: smem ring depth (8 KB TMA pieces: 16 K rows × 128 columns; 4 per K chunk, one per issuer):
// two K chunks of X in flight; four (16 pieces) measured 0.3-1.5 % slower on every config
// (profiles/r02_ring_depth_ab.log) — the TMEM double buffer, not the TMA latency, paces the fill
constexpr int kTmemRPieces = SDNN_TMEMR_PIECES;
inline int tmem_v(int kernel) { return kernel == 5 ? 8 : 4; }
inline int tmem_tn(int kernel) { return kernel == 5 ? 1024 : 128; }  // N tile of a TMEM plan
// N granularity of a TMEM plan's fast path: kernels 4 / 6 read X through a 2-D tensor map (any
// N % 4 == 0: the last tile's columns past N are zero-filled by TMA and not stored); kernel 5's 3-D
// map needs whole 128-column blocks
inline int tmem_n_align(int kernel) { return kernel == 5 ? 128 : 4; }

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace sdnn
