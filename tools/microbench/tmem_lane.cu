// Does tcgen05.ld.32x32b need the lane-quarter base in the TMEM address, or does a warp always read
// its own quarter?  Fill lane L, column c with L*1000 + c; warp w reads column 5 with lane field
// (a) 32·(w%4) and (b) 0; print what lane 0 of each warp got.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(float* out) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(uint32_t(__cvta_generic_to_shared(&tb))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tb + (uint32_t(warp * 32) << 16);
  for (int c = 0; c < 16; c += 4) {
    float v = float((warp * 32 + lane) * 1000 + c);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + c), "f"(v), "f"(v + 1), "f"(v + 2), "f"(v + 3));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  float a, b;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(a) : "r"(tb + (uint32_t(warp * 32) << 16) + 5));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(b) : "r"(tb + 5));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[threadIdx.x * 2] = a; out[threadIdx.x * 2 + 1] = b;
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  float* d; cudaMalloc(&d, 128 * 2 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(e));
  float h[256]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  for (int w = 0; w < 4; ++w) printf("warp %d lane 0: with lane base %.0f, with lane field 0 %.0f; lane 7: %.0f %.0f\n", w, h[w * 64], h[w * 64 + 1], h[(w * 32 + 7) * 2], h[(w * 32 + 7) * 2 + 1]);
  return 0;
}
