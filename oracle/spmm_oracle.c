/*
 * oracle/spmm_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU definition of what the SparseDNN hot path computes.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * this library.  It shares no code, header or constant with the CUDA product path
 * (paper_2101_07948_b200/), and the product never calls it.
 *
 * Functions
 *   oracle_spmm      Y = act(W·X + b) over CSR W, fp64 accumulation, one rounding to fp32, and the
 *                    per-element error scale S = Σ|w||x| + |b|.
 *                    Definition: SpMM "sparse matrix -- dense matrix multiplication" (PAPER.md P:62,
 *                    §2.2); the microkernel multiplies each nonzero of A with the B row slice and
 *                    accumulates (P:135 fig:spmm caption, §3.2.2); the elementwise layer that
 *                    follows is fused (§3.1); 64-bit-accumulating oracle.
 *                    Readings: C7 act ∈ {NONE, RELU}, ReLU(v) = v > 0 ? v : 0;
 *                    C8 products summed in stored (ascending column) order, then bias added once;
 *                    C9 scale S includes |b|.  Parity pinned: tests/test_oracle.py (P1-P5).
 *   oracle_spmm_omp  The same loop with rows distributed over OpenMP threads (timing variant for
 *                    the cpu_baseline).  Per-row summation order is unchanged, so the result is
 *                    bitwise identical to oracle_spmm (pinned in tests/test_oracle.py).
 *   oracle_alg1      Algorithm 1 "Weight Reordering Algorithm", step by step with dense
 *                    boolean row patterns:  rem = {0..m-1} (reading C1);
 *                    row = argmax_{x∈rem} |nnz(A[x])|;  B[0] = A[row];  for i in 1..m-1:
 *                    row = argmax_{x∈rem} |nnz(B[i-1]) ∩ nnz(A[x])|  (C4), ties → lowest original
 *                    index (C2, C3).  Output order[i] = source row placed at position i.
 *                    Parity pinned: the printed trace {1},{0,1,2},{1,2} → [1,2,0] and a
 *                    pure-Python brute force on random matrices (tests/test_oracle.py P6).
 *
 * Build (by __graft_entry__.build() or tests): gcc -O2 -fopenmp -fPIC -shared (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void oracle_row(const int32_t* row_ptr, const int32_t* col_idx, const float* vals, int64_t N,
                       const float* X, const float* bias, int32_t act, int32_t m, double* acc, double* s,
                       float* Y, double* S) {
  for (int64_t n = 0; n < N; ++n) { acc[n] = 0.0; s[n] = 0.0; }
  for (int32_t p = row_ptr[m]; p < row_ptr[m + 1]; ++p) {
    const int64_t c = col_idx[p];
    const double w = (double)vals[p];
    const float* xr = X + c * N;
    for (int64_t n = 0; n < N; ++n) {
      const double x = (double)xr[n];
      acc[n] += w * x;          /* fp32 x fp32 product is exact in fp64 */
      s[n] += fabs(w) * fabs(x);
    }
  }
  const double b = bias ? (double)bias[m] : 0.0;
  for (int64_t n = 0; n < N; ++n) {
    double v = acc[n] + b;
    if (act == 1) v = (v > 0.0) ? v : 0.0;
    Y[(int64_t)m * N + n] = (float)v;   /* the single round-to-nearest-even */
    if (S) S[(int64_t)m * N + n] = s[n] + fabs(b);
  }
}

/* Returns 0 on success, 1 on allocation failure, 2 on bad act. S may be NULL. */
int oracle_spmm(const int32_t* row_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                const float* X, int64_t N, const float* bias, int32_t act, float* Y, double* S) {
  (void)K;
  if (act != 0 && act != 1) return 2;
  if (N <= 0) return 0;
  double* acc = (double*)malloc(sizeof(double) * (size_t)N);
  double* s = (double*)malloc(sizeof(double) * (size_t)N);
  if (!acc || !s) { free(acc); free(s); return 1; }
  for (int32_t m = 0; m < M; ++m) oracle_row(row_ptr, col_idx, vals, N, X, bias, act, m, acc, s, Y, S);
  free(acc); free(s);
  return 0;
}

/* OpenMP-over-rows timing variant; nthreads <= 0 means the OpenMP default.  Returns threads used. */
int oracle_spmm_omp(const int32_t* row_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                    const float* X, int64_t N, const float* bias, int32_t act, float* Y, double* S,
                    int32_t nthreads) {
  (void)K;
  if (act != 0 && act != 1) return -2;
  if (N <= 0) return 0;
  int used = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  int fail = 0;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * (size_t)N);
    double* s = (double*)malloc(sizeof(double) * (size_t)N);
    if (!acc || !s) {
#pragma omp atomic write
      fail = 1;
    } else {
#pragma omp for schedule(dynamic, 4)
      for (int32_t m = 0; m < M; ++m) oracle_row(row_ptr, col_idx, vals, N, X, bias, act, m, acc, s, Y, S);
    }
#ifdef _OPENMP
#pragma omp single
    used = omp_get_num_threads();
#endif
    free(acc); free(s);
  }
  return fail ? -1 : used;
}

/* Algorithm 1.  order[M] receives the permutation.  Returns 0, or 1 on allocation failure.
 * Row patterns as dense bitsets: O(M*K/8) memory, O(M^2 * K/64) time — slow and obvious, by design. */
int oracle_alg1(const int32_t* row_ptr, const int32_t* col_idx, int32_t M, int32_t K, int32_t* order) {
  if (M <= 0) return 0;
  const size_t W = ((size_t)K + 63) / 64;
  uint64_t* pat = (uint64_t*)calloc((size_t)M * W, sizeof(uint64_t));
  unsigned char* rem = (unsigned char*)malloc((size_t)M);
  if (!pat || !rem) { free(pat); free(rem); return 1; }
  for (int32_t i = 0; i < M; ++i) {                    /* line 3: rem = {0 ... m-1} (reading C1) */
    rem[i] = 1;
    for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
      pat[(size_t)i * W + (size_t)col_idx[p] / 64] |= (uint64_t)1 << (col_idx[p] % 64);
  }
  /* line 4: row = argmax_{x in rem} |nnz(A[x])| ; strict '>' keeps the lowest index on ties (C2) */
  int32_t row = -1; int64_t best = -1;
  for (int32_t x = 0; x < M; ++x) {
    int64_t cnt = 0;
    for (size_t w = 0; w < W; ++w) cnt += __builtin_popcountll(pat[(size_t)x * W + w]);
    if (cnt > best) { best = cnt; row = x; }
  }
  order[0] = row; rem[row] = 0;                       /* lines 5-6: B[0] = A[row]; rem.remove(row) */
  for (int32_t i = 1; i < M; ++i) {                    /* line 7: for i in 1 ... m-1 (reading C1) */
    const uint64_t* prev = pat + (size_t)order[i - 1] * W;        /* nnz(B[i-1]) */
    row = -1; best = -1;
    for (int32_t x = 0; x < M; ++x) {                  /* line 8: argmax_{x in rem} |nnz(B[i-1]) ∩ nnz(A[x])| */
      if (!rem[x]) continue;
      const uint64_t* cand = pat + (size_t)x * W;
      int64_t inter = 0;
      for (size_t w = 0; w < W; ++w) inter += __builtin_popcountll(prev[w] & cand[w]);
      if (inter > best) { best = inter; row = x; }     /* ties, incl. all-zero overlap → lowest x (C2, C3) */
    }
    order[i] = row; rem[row] = 0;                      /* lines 9-10 */
  }
  free(pat); free(rem);
  return 0;
}
