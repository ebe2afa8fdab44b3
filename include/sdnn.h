/*
 * sdnn.h — C ABI of libsdnn: the SparseDNN hot path (arXiv 2101.07948) on NVIDIA B200 (sm_100a).
 *
 *   Y = act(W·X + b)      W: M×K fp32 unstructured-sparse weight (CSR), X: K×N fp32 dense activation,
 *                         b: fp32[M] bias (optional), act ∈ {NONE, RELU}, Y: M×N fp32.
 *
 * The operation is the paper's SpMM, "sparse matrix -- dense matrix multiplication" (PAPER.md P:62,
 * §2.2), computed by a microkernel that broadcasts each nonzero of the sparse operand and multiplies it
 * with the dense row slice (P:135 fig:spmm, §3.2.2), with the following elementwise layer fused
 * (§3.1).  Work is split into a one-time preparation stage and a per-request execution stage
 * (§2.1, §3): sdnn_prepare performs the weight permutation of Algorithm 1 (§3.1.2)
 * and re-stores the matrix in its own execution-ordered format; sdnn_spmm runs the multiply.
 *
 * Conventions
 *   - Every entry point returns sdnn_status; no C++ exception crosses the boundary.
 *   - "host" pointers are ordinary CPU memory; "device" pointers are CUDA global memory on the
 *     handle's device.  Matrices are row-major and contiguous: X is K×N (row stride N floats),
 *     Y is M×N (row stride N floats).  Indices are int32; sizes of N are int64.
 *   - A failing call leaves outputs untouched where possible and sets a thread-local message
 *     readable with sdnn_last_error_message().
 *   - Numerics: fp32 FMA accumulation on CUDA cores in a fixed order (bitwise reproducible for the
 *     same handle and inputs); accuracy contract |Y − Y_exact| ≤ 1e-4 · (Σ|w||x| + |b|) per element
 *     (BASELINE.json north_star, reading C9).
 */
#ifndef SDNN_H_
#define SDNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDNN_ABI_VERSION 1

#if defined(__GNUC__)
#define SDNN_API __attribute__((visibility("default")))
#else
#define SDNN_API
#endif

typedef enum {
  SDNN_OK = 0,
  SDNN_ERR_INVALID_ARGUMENT = 1, /* NULL where not allowed, negative size, unknown act, aliasing  */
  SDNN_ERR_INVALID_CSR = 2,      /* CSR invariants violated (message names the first bad row)      */
  SDNN_ERR_UNSUPPORTED = 3,      /* valid input this build cannot run (e.g. device is not sm_100)  */
  SDNN_ERR_OUT_OF_MEMORY = 4,    /* host or device allocation failed                              */
  SDNN_ERR_CUDA = 5,             /* a CUDA runtime/driver call or kernel launch failed            */
  SDNN_ERR_DEVICE_MISMATCH = 6,  /* current device differs from the handle's device               */
  SDNN_ERR_INTERNAL = 7
} sdnn_status;

typedef enum { SDNN_ACT_NONE = 0, SDNN_ACT_RELU = 1 } sdnn_act;

/* Preparation options.  Pass NULL for defaults.  struct_size must be sizeof(sdnn_perm_opts). */
typedef struct {
  uint32_t struct_size;
  int32_t permute;          /* 1 (default): Algorithm 1 greedy row reorder; 0: identity   */
  int32_t kernel;           /* 0 = auto: the row kernel's plan (or the group kernel's, by cost model)
                               plus the TMEM-R kernel's plan; each sdnn_spmm call takes the TMEM
                               plan when N % 4 == 0, X/Y are 16-byte aligned and the call has at
                               least a third of a wave of CTAs (or TMEM split-K fills one), else
                               the row plan.
                               1 = row kernel (each nonzero reads its X row slice from shared
                               memory), 2 = group kernel (16-row groups: one X load feeds every
                               nonzero of the group in that column), 3 = codegen (per-panel
                               generated PTX with the weights as FFMA immediates, JIT-compiled
                               during sdnn_prepare), 4 = TMEM-R kernel (a 128-column X
                               tile replicated into all four TMEM lane quarters by tcgen05.cp,
                               24 warps × 10-row panels, operands read by tcgen05.ld), 5 = TMEM
                               kernel with 8 columns per lane (round 1's layout, 5-row panels),
                               6 = TMEM-R with Algorithm 1 row pairs (columns two paired rows share
                               are loaded once; per-row summation order differs from the others).
                               4 and 6 take their fast path when N % 4 == 0 and X/Y are 16-byte
                               aligned, 5 when N % 128 == 0; else a generic kernel on the same plan. */
  int32_t panel_rows_max;   /* row kernel: rows per warp panel, 0 = auto, else 4 or 8 (group: 16);
                               kernel 4: 1..10 = about that many rows per warp (more row blocks of
                               the fixed 24 × 10-slot geometry; 0 = 10).  Auto handles keep a
                               second TMEM plan with ~25 % more row blocks and take it per call
                               where its grid fills the waves better (serialized with the
                               handle, blob role 4)                                              */
  int32_t cta_panels;       /* panels (warps) per CTA row block: 0 = auto, else 1..16                */
  int32_t k_chunk;          /* reduction-dimension tile (split-K tiling): 0 = auto, else 8..128,
                               multiple of 8.  An explicit chunk must fit two pipeline stages (its X
                               tile at the widest N tile, 1 KB per K row, plus its largest metadata
                               block) in 220 KB of shared memory — about 104 at most; beyond that
                               sdnn_prepare returns SDNN_ERR_UNSUPPORTED                            */
  int32_t group_sb;         /* group kernel sub-block rows: 0 = auto (cost model), 1, 2 or 4         */
  uint32_t flags;           /* SDNN_FLAG_NO_ROW_SPLIT | SDNN_FLAG_PERMUTED_OUTPUT | SDNN_FLAG_NO_SPLIT_K */
} sdnn_perm_opts;

/* Read-only description of a prepared handle (or a host plan). */
typedef struct {
  uint32_t struct_size;     /* in: sizeof(sdnn_info)                                                 */
  int32_t M, K;
  int64_t nnz;
  int32_t device;           /* CUDA ordinal, −1 for a host-only plan                                  */
  int32_t permuted;         /* 1 if Algorithm 1 was applied                                           */
  int32_t kernel;           /* the primary plan's kernel: 1 row, 2 group, 3 codegen, 4/5/6 TMEM       */
  int32_t group_entries_per_nnz_x1000; /* group format: union entries per nonzero · 1000            */
  int32_t group_sb;         /* group kernel sub-block rows (0 for the row kernel)                     */
  int32_t group_subblocks_per_nnz_x1000; /* nonzero sub-blocks per nonzero · 1000                    */
  int32_t panel_rows;       /* R_w: rows per warp panel                                               */
  int32_t cta_panels;       /* W_c: panels per CTA                                                    */
  int32_t num_panels;       /* P = num_row_blocks · W_c (trailing panels may be empty)               */
  int32_t num_row_blocks;   /* ⌈M / (R_w·W_c)⌉                                                        */
  int32_t k_chunk;          /* KC                                                                     */
  int32_t num_chunks;       /* ⌈K / KC⌉                                                               */
  int64_t meta_bytes;       /* device bytes of the execution-ordered stream                           */
  int32_t max_block_bytes;  /* largest (row block, chunk) metadata block, bytes                       */
  int32_t alt_kernel;       /* auto handles: kernel of the second (TMEM) plan, else 0                 */
  int64_t max_panel_nnz;
  int32_t num_split_rows;   /* row plan: rows split into pieces (≤ one per warp of ONE row block; the
                               row kernel adds them in shared memory at its end — the generic path
                               through a workspace and a second kernel — in piece order, before the
                               bias: deterministic, but not bitwise equal to the unsplit order)      */
  int32_t num_pieces;       /* total pieces of the split rows                                         */
  int32_t narrow_row_blocks; /* auto handles: row blocks of the narrow row plan (4-row panels) taken by
                               row-plan calls whose grid is under one wave; 0 = none                 */
  int32_t narrow4_row_blocks; /* auto handles: row blocks of the second narrow plan (4-row panels, 4 per
                               CTA) taken instead when its N-tile-128 grid is one to three waves; 0 = none */
} sdnn_info;

/* sdnn_perm_opts.flags */
#define SDNN_FLAG_NO_ROW_SPLIT 1u  /* row plan: never split a row across warps                         */
/* Y rows (and bias entries) in the plan's row order instead of the original order: sdnn_spmm writes
 * Y_perm[i] = act(W[order[i]]·X + b_perm[i]) with order = sdnn_get_permutation and the caller's bias
 * given as b_perm[i] = b[order[i]].  The paper's cross-layer form: the next layer consumes
 * Y_perm after its columns are relabelled the same way (sdnn_csr_permute_columns), so no layer
 * un-permutes.  Not with the codegen kernel (kernel = 3: SDNN_ERR_UNSUPPORTED). */
#define SDNN_FLAG_PERMUTED_OUTPUT 2u
/* Row kernel: never split the K range across CTAs.  By default a row-kernel call whose grid is under
 * two waves runs KS ≤ 8 CTAs per (row block, N tile), each over a range of K chunks, and a second
 * small kernel sums the KS partial results in slice order before bias and activation: deterministic,
 * but not bitwise equal to the unsplit (sequential) summation order. */
#define SDNN_FLAG_NO_SPLIT_K 4u

typedef struct sdnn_handle_s* sdnn_handle; /* opaque; owns its device memory; immutable after prepare */
typedef struct sdnn_plan_s* sdnn_plan;     /* opaque host-only plan (no device needed)               */

/* ------------------------------------------------------------------ preparation (once per weight)
 * sdnn_prepare: validate the CSR (row_ptr[0] = 0, nondecreasing, row_ptr[M] = nnz < 2^31,
 * 0 ≤ col < K, strictly increasing columns per row; explicit zero values are kept as structural
 * nonzeros, reading C6), apply Algorithm 1 (opts->permute), pack the permuted rows into
 * warp panels and the execution-ordered per-(row block, K chunk) metadata stream, and
 * upload it to the CURRENT CUDA device.  All three arrays are HOST pointers, read during the call
 * only.  nnz = 0 is allowed (Y = act(b)).  Synchronous; deterministic (same input → bit-identical
 * device arrays).  Errors: INVALID_ARGUMENT (NULL out, M < 1, K < 1, NULL arrays with nnz > 0,
 * bad opts), INVALID_CSR, UNSUPPORTED (device is not compute capability 10.0), OUT_OF_MEMORY, CUDA. */
SDNN_API sdnn_status sdnn_prepare(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M,
                         int32_t K, const sdnn_perm_opts* perm_opts, sdnn_handle* out);

/* Release a handle.  NULL is a no-op.  The caller must ensure no sdnn_spmm on it is in flight. */
SDNN_API sdnn_status sdnn_destroy(sdnn_handle h);

/* ------------------------------------------------------------------ execution (per request)
 * sdnn_spmm: Y = act(W·X + b) on DEVICE buffers of the handle's device.
 *   X     device, K×N row-major fp32 (exactly the handle's K rows; caller guarantees ≥ K·N floats)
 *   N     ≥ 0 columns; N = 0 returns SDNN_OK without work
 *   bias  device fp32[M] in ORIGINAL row order, or NULL for no bias
 *   act   SDNN_ACT_NONE or SDNN_ACT_RELU
 *   Y     device, M×N row-major fp32, written in ORIGINAL row order (the permutation is invisible);
 *         must not overlap X or bias
 *   stream cudaStream_t (NULL = legacy default stream).  The call enqueues and returns without a
 *         host synchronisation; device faults surface at the caller's next sync.  Kernels are
 *         launched with programmatic dependent launch: a call's grid may start its prologue (barrier
 *         setup, TMEM allocation, plan-metadata copies) while the previous kernel on `stream`
 *         drains, and reads X / bias and writes Y only after that kernel has completed (stream
 *         order is unchanged for the caller).
 * Fast path: X and Y 16-byte aligned and N % 4 == 0 (TMA tiles); otherwise a slower correct path.
 * Errors: INVALID_ARGUMENT (NULL handle/X/Y, N < 0, bad act, Y overlapping X or bias),
 * DEVICE_MISMATCH (current device ≠ handle device), CUDA (launch failure). */
SDNN_API sdnn_status sdnn_spmm(sdnn_handle h, const float* X, int64_t N, const float* bias, int32_t act, float* Y,
                      void* stream);

/* sdnn_spmm_multi: the same operation, Y written to n_dst (1..8) device buffers at once — the fused
 * form of "SpMM, then all-gather of Y" (BASELINE north_star): each destination is an
 * M×ldy row-major buffer (ldy ≥ col0 + N) that receives Y in columns [col0, col0 + N), e.g. every
 * rank's symmetric-memory Y buffer mapped into this device (peer or multicast addresses), with col0
 * the rank's column offset; the epilogue stores each output element to every destination, so the
 * transfer overlaps the kernel.  Visibility on the peers follows the caller's barrier (e.g. the
 * symmetric-memory barrier after the call).  Same errors as sdnn_spmm, plus INVALID_ARGUMENT for
 * n_dst outside 1..8, a NULL destination, col0 < 0 or ldy < col0 + N.  The vector fast paths need
 * ldy, col0 multiples of 4 and 16-byte-aligned destinations; the codegen kernel is UNSUPPORTED. */
SDNN_API sdnn_status sdnn_spmm_multi(sdnn_handle h, const float* X, int64_t N, const float* bias, int32_t act,
                                     float* const* Y_dsts, int32_t n_dst, int64_t ldy, int64_t col0, void* stream);

/* sdnn_spmm_multicast: the fused all-gather through NVLink SHARP multicast: Y_mc is a
 * multicast address — one virtual address bound to every rank's M×ldy row-major Y buffer (e.g.
 * torch symmetric memory's multicast_ptr) — and the epilogue writes each output element once with
 * multimem.st; NVSwitch replicates it into every rank's buffer at columns [col0, col0 + N).  Same
 * argument rules and errors as sdnn_spmm_multi with n_dst = 1; the caller owns the multicast object
 * and orders visibility with its barrier.  Without multicast support use sdnn_spmm_multi with the
 * peers' addresses. */
SDNN_API sdnn_status sdnn_spmm_multicast(sdnn_handle h, const float* X, int64_t N, const float* bias, int32_t act,
                                         float* Y_mc, int64_t ldy, int64_t col0, void* stream);

/* sdnn_spmm_host: the same operation on HOST buffers (X host K×N, bias host fp32[M] or NULL, Y host
 * M×N).  Columns are processed in blocks of `block_cols` (0 = auto), with host→device copy, kernel
 * and device→host copy of successive blocks overlapped on internal streams; pinned (page-locked)
 * host buffers give full PCIe/C2C bandwidth.  Synchronous: returns after Y is complete in host
 * memory.  Uses the current device (must be the handle's).  Errors as sdnn_spmm plus OUT_OF_MEMORY. */
SDNN_API sdnn_status sdnn_spmm_host(sdnn_handle h, const float* X_host, int64_t N, const float* bias_host, int32_t act,
                           float* Y_host, int64_t block_cols);

/* sdnn_conv2d: sparse k×k convolution (§3.2.3, "treated as an SpMM where the sparse
 * matrix is the filters treated as an OC by IC × Fx × Fy matrix ... the dense matrix is a virtual
 * matrix that is realized on the fly from the input dense activations with the proper offsets").
 *   h       a handle prepared from the filters as the CSR of the OC × (IC·FY·FX) matrix, column
 *           (ic·FY + fy)·FX + fx, with a row plan without split rows (kernel 0 or 1 and
 *           SDNN_FLAG_NO_ROW_SPLIT); else SDNN_ERR_UNSUPPORTED.  K must equal IC·FY·FX.
 *   X       DEVICE fp32 [IC][B][H][W] (the C×(B·H·W) activation layout of the 1×1 convs).
 *   Y       DEVICE fp32 [OC][B][Ho][Wo], Ho = (H + 2·pad − FY)/stride + 1 (same for Wo), written in
 *           original output-channel order; bias fp32[OC] or NULL; act as sdnn_spmm.
 *   Y[oc][b][oy][ox] = act(Σ W[oc][ic][fy][fx] · X[ic][b][oy·stride + fy − pad][ox·stride + fx − pad]
 *                          + bias[oc]), taps outside the image contribute 0.
 * Enqueued on `stream`, no host sync.  B = 0 → SDNN_OK, nothing done.  Errors as sdnn_spmm, plus
 * SDNN_ERR_INVALID_ARGUMENT for an empty output or K ≠ IC·FY·FX. */
SDNN_API sdnn_status sdnn_conv2d(sdnn_handle h, const float* X, int32_t B, int32_t IC, int32_t H, int32_t W,
                                 int32_t FY, int32_t FX, int32_t pad, int32_t stride, const float* bias, int32_t act,
                                 float* Y, void* stream);

/* sdnn_serialize / sdnn_deserialize: the prepared handle (every plan it keeps — row, both TMEM plans,
 * narrow — with its execution-ordered metadata) as a self-contained blob, so another process skips
 * Algorithm 1 and the packing (the paper's reusable preparation stage).
 *   sdnn_serialize(h, NULL, &size) stores the blob size; sdnn_serialize(h, buf, &size) writes it to
 *   the HOST buffer (SDNN_ERR_INVALID_ARGUMENT if *size is too small; *size = bytes written).
 *   Codegen handles (kernel 3, JIT-compiled from the CSR) → SDNN_ERR_UNSUPPORTED.
 *   sdnn_deserialize(buf, size, &h) uploads the plans to the current device; a corrupt or
 *   truncated blob → SDNN_ERR_INVALID_ARGUMENT, another format version → SDNN_ERR_UNSUPPORTED.
 *   Only the structure is validated (sizes, offsets, row indices); the packed stream itself is
 *   trusted — load blobs this library wrote.
 * Results of the deserialized handle are bitwise those of the original. */
SDNN_API sdnn_status sdnn_serialize(sdnn_handle h, void* buf, size_t* size);
SDNN_API sdnn_status sdnn_deserialize(const void* buf, size_t size, sdnn_handle* out);

/* sdnn_tune: per-matrix autotuning ("we can perform autotuning on the sparse weight
 * matrix to find the best settings for the microkernel and the tiling factor").  Times every path the
 * handle can take for this N — TMEM plan, row plan, narrow row plans, each with split-K 1/2/4/8 — on
 * the caller's DEVICE buffers X (K×N) and Y (M×N, overwritten), and keeps the fastest for every later
 * fast-path call with this N (N % 4 == 0, 16-byte aligned X / Y, one destination).  Synchronises
 * `stream`.  The built-in per-call rules are a candidate too and are kept unless a path beats them
 * by more than 3 %.  path_out (optional) = −1 (the rules) or 16·path + slices (path 0 TMEM, 1 row,
 * 2 narrow, 3 narrow4); us_out
 * (optional) = its time per call in µs.  Results then follow the chosen path's summation order.
 * Tuning state is per handle, guarded by a mutex, and not serialized.  Codegen handles →
 * SDNN_ERR_UNSUPPORTED; N % 4 ≠ 0 or unaligned buffers → SDNN_ERR_INVALID_ARGUMENT. */
/* sdnn_conv2d_tune: the same for sdnn_conv2d — times its tile choices for this geometry (the built-in
 * rules, then 2 / 4 output pixels per lane × 1 / 2 / 4 / 8 K slices, and — handles with a TMEM plan —
 * the explicit form: the virtual operand written out, then the TMEM-R SpMM) on the caller's DEVICE
 * X / Y (overwritten) and keeps the fastest (> 3 % better than the rules) for later calls with the
 * same {B, IC, H, W, FY, FX, pad, stride}.  choice_out = −1 (rules), −2 (explicit form) or
 * 16·pixels + slices. */
SDNN_API sdnn_status sdnn_conv2d_tune(sdnn_handle h, const float* X, int32_t B, int32_t IC, int32_t H, int32_t W,
                                      int32_t FY, int32_t FX, int32_t pad, int32_t stride, float* Y, void* stream,
                                      int32_t* choice_out, float* us_out);
SDNN_API sdnn_status sdnn_tune(sdnn_handle h, const float* X, int64_t N, float* Y, void* stream, int32_t* path_out,
                               float* us_out);

/* ------------------------------------------------------------------ introspection
 * sdnn_get_permutation: out_perm (HOST, M entries) receives order[i] = original row at permuted
 * position i (Algorithm 1 output, SPEC S:295 convention).  sdnn_get_info fills *info. */
SDNN_API sdnn_status sdnn_get_permutation(sdnn_handle h, int32_t* out_perm);
/* Which kernel sdnn_spmm launches for these arguments (no launch, no device access; X and Y only
 * for their alignment): 1 row, 2 group, 3 codegen, 4/5 TMEM; negative = that plan's generic
 * (non-TMA) fallback kernel, used when N % 4 != 0 (N % 128 != 0 for 4/5) or X/Y are unaligned. */
SDNN_API sdnn_status sdnn_spmm_kernel(sdnn_handle h, int64_t N, const float* X, const float* Y, int32_t* kernel);
SDNN_API sdnn_status sdnn_get_info(sdnn_handle h, sdnn_info* info);

/* ------------------------------------------------------------------ host-only planning (no GPU)
 * sdnn_permutation: Algorithm 1 alone, on host CSR, inverted-index implementation;
 * order[M] (HOST) receives the permutation; ties → lowest original row (readings C2, C3).
 * Validates the CSR like sdnn_prepare. */
SDNN_API sdnn_status sdnn_permutation(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K,
                             int32_t* order);

/* sdnn_csr_permute_columns: the CSR of W·P, P the permutation matrix of `order` (HOST, K entries,
 * order[i] = the original column that moves to position i; a bijection of 0..K−1): every entry
 * (r, c, w) becomes (r, pos(c), w) with order[pos(c)] = c, each row re-sorted by its new columns.
 * out_col_idx / out_vals: HOST, nnz = csr_ptr[M] entries each (row pointers are unchanged).  For
 * the next layer of a chain whose previous layer ran with SDNN_FLAG_PERMUTED_OUTPUT.
 * Errors: SDNN_ERR_INVALID_CSR (as sdnn_prepare), SDNN_ERR_INVALID_ARGUMENT (NULL, not a
 * permutation). */
SDNN_API sdnn_status sdnn_csr_permute_columns(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals,
                                              int32_t M, int32_t K, const int32_t* order, int32_t* out_col_idx,
                                              float* out_vals);

/* sdnn_plan_create: everything sdnn_prepare does except the upload, on host.  sdnn_plan_export
 * copies the plan's arrays into caller HOST buffers sized from sdnn_plan_get_info:
 *   row_orig  int32[num_panels·panel_rows]  original row of each panel slot, −1 for empty slots
 *   blk_off   int64[num_row_blocks·num_chunks + 1] byte offset of each metadata block in `meta`
 *   meta      uint8[meta_bytes]  execution-ordered blocks; see DESIGN.md "Execution-ordered format"
 * Any export pointer may be NULL to skip it.  Used by the packing-invariant tests. */
SDNN_API sdnn_status sdnn_plan_create(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M,
                             int32_t K, const sdnn_perm_opts* perm_opts, sdnn_plan* out);
SDNN_API sdnn_status sdnn_plan_get_info(sdnn_plan p, sdnn_info* info);
SDNN_API sdnn_status sdnn_plan_export(sdnn_plan p, int32_t* row_orig, int64_t* blk_off, uint8_t* meta);
/* Split rows of a row plan (info.num_pieces entries each; NULL arrays are skipped): piece i of original
 * row row[i] covers the CSR entries begin[i], begin[i] + P, begin[i] + 2P, … < end[i], P being the
 * number of pieces of that row (interleaved pieces); slots whose row_orig is −2 − i hold piece i. */
SDNN_API sdnn_status sdnn_plan_export_pieces(sdnn_plan p, int32_t* row, int32_t* begin, int32_t* end);
SDNN_API sdnn_status sdnn_plan_destroy(sdnn_plan p);

/* sdnn_plan_codegen_ptx: the generated PTX of codegen panel `panel` of a plan created with
 * kernel = 3 (the same CSR must be passed again; HOST pointers).  If `out` is NULL only *len (bytes
 * incl. the terminating NUL) is returned; else `out` must hold *len bytes.  For inspection/tests. */
SDNN_API sdnn_status sdnn_plan_codegen_ptx(sdnn_plan p, const int32_t* csr_ptr, const int32_t* col_idx,
                                           const float* vals, int32_t panel, char* out, int64_t* len);

/* ------------------------------------------------------------------ errors / version */
SDNN_API const char* sdnn_status_string(sdnn_status s);
SDNN_API const char* sdnn_last_error_message(void); /* thread-local; "" if none */
SDNN_API int32_t sdnn_abi_version(void);

/* Environment knobs read by libsdnn (diagnostics and experiments only; unset = the product path):
 *   SDNN_TMEM_FILL   kernel 5's fill path: 1 = filler warps with tcgen05.st (default), 0 = one
 *                    producer thread with tcgen05.cp, 2 = both (odd/even pieces); kernels 4 / 6
 *                    always fill with tcgen05.cp.32x128b.warpx4
 *   SDNN_TMEM_PERSIST 1 / 0 = kernel 4 runs one CTA per SM over its (row block, N tile) items
 *                    always / never (default: when K has ≤ 8 chunks and there are ≥ 4 items per SM)
 *   SDNN_JITTER      1 = pseudo-random sleeps at the pipelines' mbarrier hand-offs (protocol tests;
 *                    results unchanged, slower)
 *   SDNN_DEBUG_TMEM  bit mask, TMEM kernels: 1 skip the X loads (TMA), 2 skip the FMA loop, 4 skip the
 *                    smem -> TMEM fill — results are WRONG with any bit set (timing decomposition)
 *   SDNN_ROW_STAGES  upper bound on the row kernel's stage-ring depth
 *   SDNN_SPLIT_K     row kernel: force this many K slices (1 = never split); default: automatic for
 *                    under-filled calls (see SDNN_FLAG_NO_SPLIT_K)
 *   SDNN_CONV_GATHER 1 = sdnn_conv2d stages the virtual matrix itself instead of the input patch
 *   SDNN_ROW_V       2 | 4: row kernel's N-tile width (floats per lane) on calls whose automatic
 *                    choice is between the two (small grids, no split-K)
 *   SDNN_TMEM_SPLIT_K 0 = never split the TMEM plan's K range
 *   SDNN_CONV_PX, SDNN_CONV_KS  sdnn_conv2d: force 2 | 4 output pixels per lane / this many K slices
 *   SDNN_PDL         0 = launch without programmatic dependent launch (A/B runs)
 *   SDNN_LOCAL_PIECES 0 = split rows through the workspace + reduction kernel even where the row
 *                    kernel could add them in shared memory (A/B runs; bitwise the same Y)
 * (and, at build time, -DSDNN_DIAG=1|2: TMEM consumer without tcgen05.ld / without FFMA2). */

#ifdef __cplusplus
}
#endif
#endif /* SDNN_H_ */
