// TMEM -> register read bandwidth vs shared-memory (LDS.128) bandwidth as operand paths for CUDA-core
// FFMA (the SpMM operand-delivery question).  One CTA per SM; the first NT warps read
// TMEM (their lane quarter 32·(w%4), warp-uniform pseudo-random columns, tcgen05.ld .32x32b.x{X},
// B loads per tcgen05.wait::ld), the other NL warps read shared memory with LDS.128 (each lane 16 B
// of a warp-uniform pseudo-random 512-byte row: conflict-free).  Per-warp cycles via clock64;
// aggregate = all bytes / slowest warp of block 0.  Are the two paths additive?
// usage: tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int X> struct TL;
#define TLDEF(X, REGS, ...)                                                                         \
  template <> struct TL<X> {                                                                        \
    static __device__ __forceinline__ void ld(uint32_t a, float* v) {                               \
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x" #X ".b32 " REGS ", [%" #X "];" : __VA_ARGS__ : "r"(a)); \
    }                                                                                               \
  };
TLDEF(1, "{%0}", "=f"(v[0]))
TLDEF(2, "{%0,%1}", "=f"(v[0]), "=f"(v[1]))
TLDEF(4, "{%0,%1,%2,%3}", "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]))
TLDEF(8, "{%0,%1,%2,%3,%4,%5,%6,%7}", "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
      "=f"(v[6]), "=f"(v[7]))
TLDEF(16, "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}", "=f"(v[0]), "=f"(v[1]), "=f"(v[2]),
      "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]),
      "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]))

template <int X, int B>
__global__ void __launch_bounds__(768, 1) bw_kernel(int nt, int iters_t, int iters_l, float* out, long long* cyc) {
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float xs[8192];  // 32 KB LDS source: 64 rows x 512 B
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) xs[i] = float(i & 127) * 1e-3f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        uint32_t(__cvta_generic_to_shared(&tbase))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase + (uint32_t((warp & 3) * 32) << 16);
  if (warp < 4) {
    for (int c = 0; c < 512; c += 4) {
      float a = float(lane + c) * 1e-3f;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tb + c), "f"(a), "f"(a),
                   "f"(a), "f"(a));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  float acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.f;
  long long t0 = clock64();
  uint32_t col = uint32_t(warp * 13);
  if (warp < nt) {
    for (int it = 0; it < iters_t; ++it) {
      float v[B][X];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        col = (col * 5 + 7) & (511 - (X - 1));
        TL<X>::ld(tb + col, v[b]);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int q = 0; q < X; ++q) acc[q] = fmaf(v[b][q], 1.0001f, acc[q]);
    }
  } else {
    const float4* x4 = reinterpret_cast<const float4*>(xs) + lane;
    for (int it = 0; it < iters_l; ++it) {
      float4 v[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        col = (col * 5 + 7) & 63;
        v[b] = x4[col * 32];
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        acc[0] = fmaf(v[b].x, 1.0001f, acc[0]);
        acc[1] = fmaf(v[b].y, 1.0001f, acc[1]);
        acc[2] = fmaf(v[b].z, 1.0001f, acc[2]);
        acc[3] = fmaf(v[b].w, 1.0001f, acc[3]);
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += acc[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int X, int B>
int run(int nt, int nl, int iters_t, int iters_l, int sms) {
  const int nw = nt + nl;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  CK(cudaMemset(cyc, 0, sizeof(long long) * sms * 32));
  bw_kernel<X, B><<<sms, nw * 32>>>(nt, 4, 4, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bw_kernel<X, B><<<sms, nw * 32>>>(nt, iters_t, iters_l, out, cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c[32];
  CK(cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost));
  long long ct = 0, cl = 0;
  for (int w = 0; w < nw; ++w) (w < nt ? ct : cl) = std::max(w < nt ? ct : cl, c[w]);
  const double bt = double(nt) * 32 * 4 * X * B * iters_t, bl = double(nl) * 512 * 8 * iters_l;
  const double cmax = double(std::max(ct, cl));
  printf("TMEM x%-2d B=%-2d warps T=%2d L=%2d: T %6.1f B/clk  L %6.1f B/clk  total %6.1f B/clk/SM (cyc T %lld L %lld)  %.3f ms\n",
         X, B, nt, nl, ct ? bt / ct : 0.0, cl ? bl / cl : 0.0, (bt + bl) / cmax, ct, cl, ms);
  cudaFree(out);
  cudaFree(cyc);
  return 0;
}

#include <algorithm>
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int I = 2048;
  // TMEM alone
  for (int nt : {8, 16, 24}) {
    run<2, 8>(nt, 0, I, 0, sms);
    run<4, 8>(nt, 0, I, 0, sms);
    run<8, 4>(nt, 0, I, 0, sms);
    run<8, 8>(nt, 0, I, 0, sms);
    run<16, 2>(nt, 0, I, 0, sms);
    run<16, 4>(nt, 0, I, 0, sms);
  }
  // LDS.128 alone
  for (int nl : {8, 16, 24}) run<4, 8>(0, nl, 0, I, sms);
  // both, concurrently (iteration counts scaled so both halves take similar time)
  run<4, 8>(8, 8, I, I, sms);
  run<8, 4>(8, 8, I, I, sms);
  run<8, 4>(8, 8, I, I / 2, sms);
  run<8, 4>(12, 12, I, I / 2, sms);
  run<16, 2>(12, 12, I, I / 2, sms);
  run<16, 4>(8, 8, I, I, sms);
  return 0;
}
