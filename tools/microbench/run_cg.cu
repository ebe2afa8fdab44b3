// Runs a prototype generated-code SpMM cubin (tools/proto_codegen.py) and reports FMA throughput.
// usage: run_cg file.cubin fma_per_panel npan N
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
  double fpp = atof(argv[2]); unsigned npan = atoi(argv[3]); unsigned N = atoi(argv[4]); int v2 = argc > 5 ? atoi(argv[5]) : 0; int thr = argc > 6 ? atoi(argv[6]) : 384;
  const int K = 4096, R = 128;
  float *X, *Y;
  cudaMalloc(&X, size_t(K) * N * 4); cudaMalloc(&Y, size_t(R) * N * 4);
  cudaMemset(X, 0, size_t(K) * N * 4);
  unsigned ldx4 = N * 4, ldy4 = N * 4;
  unsigned ntiles = v2 ? (N + 2 * thr - 1) / (2 * thr) : (N + 383) / 384;
  float* W; cudaMalloc(&W, 1 << 22); cudaMemset(W, 0, 1 << 22);
  void* args1[] = {&X, &Y, &ldx4, &ldy4, &N, &npan};
  void* args2[] = {&X, &Y, &W, &ldx4, &ldy4, &N};
  unsigned never = 0;
  void* args3[] = {&X, &Y, &ldx4, &ldy4, &N, &never};
  void** args = v2 == 3 ? args3 : v2 ? args2 : args1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int SM; cudaDeviceGetAttribute(&SM, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    CKD(cuLaunchKernel(f, ntiles * npan, 1, 1, v2 ? thr : 384, 1, 1, 0, 0, args, 0));
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = fpp * npan * double(N);  // fpp = FMAs per panel per column of N
    printf("cg npan=%u N=%u: %.3f ms  %.2f TFLOP/s  (%.1f%% of 74.4)  FMA/clk/SM@1.965GHz %.1f  err=%s\n", npan, N, ms,
           2 * fmas / (ms * 1e-3) / 1e12, 100 * 2 * fmas / (ms * 1e-3) / 74.4e12,
           fmas / (ms * 1e-3) / 1.965e9 / SM, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
