// tcgen05.cp.cta_group::1.32x128b.warpx4 throughput (smem 512 B → the same 32 lanes × 16 B in all four TMEM
// lane quarters): the fill a replicated-quarter TMEM tile needs (one copy per X row of 128 columns).
// nw issuing warps (one elected thread each), B copies per tcgen05.commit, one CTA per SM; optional
// concurrent LDTM load (nl warps of tcgen05.ld.32x32b.x4 + FFMA2, as the consumers).  usage: tmem_cp_x4
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) | (uint64_t(1) << 46);
}
__global__ void __launch_bounds__(1024, 1) k(int nw, int nl, int iters, int B, long long* cyc, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = float(i);
  if (threadIdx.x < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[threadIdx.x])));
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
  if (warp < nw) {
    if (lane == 0) {
      uint32_t ph = 0;
      for (int it = 0; it < iters; ++it) {
        for (int b = 0; b < B; ++b) {
          const uint32_t src = su32(sm) + uint32_t(((warp * B + b) * 512) & 65535);
          const uint32_t dst = tb + uint32_t(256 + ((warp * B + b) * 4) % 256);  // columns 256..511
          asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(dst), "l"(desc(src, 128, 128)) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
        asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(su32(&bar[warp])), "r"(ph) : "memory");
        ph ^= 1;
      }
    }
  } else if (warp >= 4 && warp < 4 + nl) {  // consumer-like TMEM reads of columns 0..255
    const uint32_t tq = tb + (uint32_t((warp & 3) * 32) << 16);
    float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
    uint32_t col = uint32_t(warp * 13);
    for (int it = 0; it < iters * 8; ++it) {
      float v[4][4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        col = (col * 5 + 7) & 252;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=f"(v[b][0]), "=f"(v[b][1]), "=f"(v[b][2]), "=f"(v[b][3]) : "r"(tq + col));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        acc0 = __ffma2_rn(make_float2(1.0001f, 1.0001f), make_float2(v[b][0], v[b][1]), acc0);
        acc1 = __ffma2_rn(make_float2(1.0001f, 1.0001f), make_float2(v[b][2], v[b][3]), acc1);
      }
    }
    out[blockIdx.x * 1024 + threadIdx.x] = acc0.x + acc0.y + acc1.x + acc1.y;
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  float* out;
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  const int iters = 256;
  for (int nl : {0, 24})
    for (int nw : {1, 2, 4})
      for (int B : {4, 16, 64}) {
        if (nw * B > 64) continue;
        k<<<sms, 1024, 65536>>>(nw, nl, 4, B, cyc, out);
        CK(cudaDeviceSynchronize());
        k<<<sms, 1024, 65536>>>(nw, nl, iters, B, cyc, out);
        CK(cudaDeviceSynchronize());
        long long c[32];
        CK(cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost));
        long long mx = 0, ml = 0;
        for (int w = 0; w < nw; ++w) mx = c[w] > mx ? c[w] : mx;
        for (int w = 4; w < 4 + nl; ++w) ml = c[w] > ml ? c[w] : ml;
        const double copies = double(iters) * B * nw;
        printf("32x128b.warpx4 issuers %d B=%2d loaders %2d: %6.1f cyc/copy  %6.1f B/clk src  %6.1f B/clk TMEM-write"
               "  | loaders: %6.1f B/clk TMEM-read (%lld cyc)\n",
               nw, B, nl, double(mx) / copies, copies * 512 / double(mx), copies * 2048 / double(mx),
               nl ? double(iters) * 8 * 4 * 512 * nl / double(ml) : 0.0, ml);
      }
  return 0;
}
