// tcgen05.cp (shared memory -> TMEM) throughput: one thread issues B copies of a given shape, commits
// to an mbarrier, waits, repeats.  Also tcgen05.st from registers (all 4 lane quarters) as the
// alternative fill path.  One CTA per SM.  usage: tmem_cp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) | (uint64_t(1) << 46);
}

// mode 0: 128x128b (2 KB per cp), mode 1: 128x256b (4 KB per cp), mode 2: tcgen05.st.32x32b.x16 by 4 warps
__global__ void __launch_bounds__(128, 1) cp_kernel(int mode, int iters, int B, long long* cyc) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = float(i);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
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
  if (mode < 2) {
    if (threadIdx.x == 0) {
      uint32_t ph = 0;
      for (int it = 0; it < iters; ++it) {
        for (int b = 0; b < B; ++b) {
          const uint32_t src = su32(sm) + uint32_t((b * 4096) & 65535);
          if (mode == 0)
            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tb + uint32_t((b * 4) & 511)),
                         "l"(desc(src, 2048, 128)) : "memory");
          else
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + uint32_t((b * 8) & 511)),
                         "l"(desc(src, 2048, 128)) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
                su32(&bar)),
            "r"(ph)
            : "memory");
        ph ^= 1;
      }
    }
  } else {
    const uint32_t tl = tb + (uint32_t(warp * 32) << 16);
    float v = float(lane);
    for (int it = 0; it < iters; ++it) {
      for (int b = 0; b < B; ++b) {
        const uint32_t c = uint32_t((b * 16) & 511);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tl + c),
            "f"(v)
            : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  CK(cudaMalloc(&cyc, sizeof(long long) * sms));
  CK(cudaFuncSetAttribute(cp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  const int iters = 256;
  for (int mode = 0; mode < 3; ++mode)
    for (int B : {4, 16, 64}) {
      cp_kernel<<<sms, 128, 65536>>>(mode, 4, B, cyc);
      CK(cudaDeviceSynchronize());
      cp_kernel<<<sms, 128, 65536>>>(mode, iters, B, cyc);
      CK(cudaDeviceSynchronize());
      long long c;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      const double bytes = double(iters) * B * (mode == 0 ? 2048 : mode == 1 ? 4096 : 4 * 32 * 16 * 4);
      printf("%s B=%2d: %.1f B/clk/SM  (%.0f cycles per batch)\n",
             mode == 0 ? "cp.128x128b " : mode == 1 ? "cp.128x256b " : "st.32x32b.x16", B, bytes / double(c),
             double(c) / iters);
    }
  return 0;
}
