// Runs a codegen-probe cubin (gen_codegen_ptx.py) through the driver API and reports the
// per-SM FMA rate for 1..P concurrent instruction streams per SM.
// usage: run_probe probe.cubin fma_per_iter maxvar
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
  CKD(cuModuleGetFunction(&f, mod, "probe"));
  double fpi = atof(argv[2]); int maxvar = atoi(argv[3]);
  int SM; cudaDeviceGetAttribute(&SM, cudaDevAttrMultiProcessorCount, 0);
  int smem = 256 * 256;
  CKD(cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem));
  float* o; long long* clk; cudaMalloc(&o, 64); cudaMalloc(&clk, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int cps = 1; cps <= 3; ++cps) {
    for (int nvar = 1; nvar <= maxvar; nvar *= 2) {
      int iters = 10; unsigned nv = nvar;
      void* args[] = {&o, &iters, &clk, &nv};
      int blocks = SM * cps;
      CKD(cuLaunchKernel(f, blocks, 1, 1, 128, 1, 1, smem, 0, args, 0));
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      CKD(cuLaunchKernel(f, blocks, 1, 1, 128, 1, 1, smem, 0, args, 0));
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      double fmas = fpi * iters * 128.0 * blocks;
      printf("probe ctas/SM=%d nvar=%d: %.3f ms  %.2f TFLOP/s  per-SM FMA/clk(block0) %.1f  clk %.0f MHz err=%s\n",
             cps, nvar, ms, 2 * fmas / (ms * 1e-3) / 1e12, fpi * iters * 128.0 * cps / c, c / (ms * 1e3),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
