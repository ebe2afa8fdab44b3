// tcgen05.cp.128x256b throughput when several warps issue copies concurrently (one elected thread
// per warp, each with its own mbarrier): does the smem → TMEM copy engine pipeline copies from
// different issuers?  One CTA per SM.  usage: tmem_cp_multi
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) | (uint64_t(1) << 46);
}
__global__ void __launch_bounds__(512, 1) k(int nw, int iters, int B, long long* cyc) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = float(i);
  if (threadIdx.x < 16) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[threadIdx.x])));
  }
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tb = tbase;
  long long t0 = clock64();
  if (warp < nw && lane == 0) {
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      for (int b = 0; b < B; ++b) {
        const uint32_t src = su32(sm) + uint32_t(((warp * B + b) * 4096) & 65535);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + uint32_t(((warp * B + b) * 8) & 511)),
                     "l"(desc(src, 2048, 128)) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
      asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(&bar[warp])), "r"(ph) : "memory");
      ph ^= 1;
    }
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0 && warp < nw) cyc[blockIdx.x * 16 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 16));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  const int iters = 256;
  for (int nw : {1, 2, 4, 8})
    for (int B : {4, 16}) {
      k<<<sms, 512, 65536>>>(nw, 4, B, cyc);
      CK(cudaDeviceSynchronize());
      k<<<sms, 512, 65536>>>(nw, iters, B, cyc);
      CK(cudaDeviceSynchronize());
      long long c[16];
      CK(cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (int w = 0; w < nw; ++w) mx = c[w] > mx ? c[w] : mx;
      printf("issuers %d B=%2d: %6.1f B/clk/SM\n", nw, B, double(iters) * B * 4096 * nw / double(mx));
    }
  return 0;
}
