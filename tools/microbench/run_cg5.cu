// Runs a proto_codegen5 cubin: X (K×N) via a TMA tensor map with {64 × KC} boxes.
// usage: run_cg5 file.cubin nnz_per_panel N W KC S R
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#define CKD(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("CU error %s line %d\n", s, __LINE__); exit(1);} } while (0)
int main(int argc, char** argv) {
  cudaFree(0);
  CUmodule mod; CUfunction f;
  CKD(cuModuleLoad(&mod, argv[1]));
  CKD(cuModuleGetFunction(&f, mod, "cg"));
  double nnzp = atof(argv[2]); unsigned N = atoi(argv[3]); int W = atoi(argv[4]); int KC = atoi(argv[5]); int S = atoi(argv[6]);
  const int K = 4096; const int R = argc > 7 ? atoi(argv[7]) : 64;
  float *X, *Y;
  cudaMalloc(&X, size_t(K) * N * 4); cudaMalloc(&Y, size_t(R) * N * 4);
  cudaMemset(X, 0, size_t(K) * N * 4);
  CUtensorMap tm;
  cuuint64_t dims[2] = {N, (cuuint64_t)K}; cuuint64_t str[1] = {cuuint64_t(N) * 4};
  cuuint32_t box[2] = {64, (cuuint32_t)KC}; cuuint32_t es[2] = {1, 1};
  CKD(cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  unsigned ldy4 = N * 4;
  int smem = S * W * KC * 256 + 16 * S;
  CKD(cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem));
  void* args[] = {&tm, &Y, &ldy4, &N};
  unsigned grid = (N + 64 * W - 1) / (64 * W);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int SM; cudaDeviceGetAttribute(&SM, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    CKD(cuLaunchKernel(f, grid, 1, 1, (W + 1) * 32, 1, 1, smem, 0, args, 0));
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = nnzp * double(N);
    printf("cg5 W=%d KC=%d S=%d N=%u: %.3f ms  %.2f TFLOP/s  (%.1f%% of 74.4)  err=%s\n", W, KC, S, N, ms,
           2 * fmas / (ms * 1e-3) / 1e12, 100 * 2 * fmas / (ms * 1e-3) / 74.4e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
