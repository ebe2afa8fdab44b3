// tcgen05.ld throughput by shape at 512 B per warp-instruction (4 registers per thread):
// 32x32b.x4, 16x64b.x4, 16x128b.x2, 16x256b.x1 — which shape feeds CUDA-core operands fastest?
// One CTA per SM, NW warps, B loads in flight per tcgen05.wait::ld, warp-uniform random columns.
// usage: tmem_shapes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int S> __device__ __forceinline__ void ld4(uint32_t a, float (&v)[4]) {
  if constexpr (S == 0)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
  else if constexpr (S == 1)
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
  else if constexpr (S == 2)
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
  else
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
}

template <int S, int B>
__global__ void __launch_bounds__(768, 1) k(int iters, float* out, long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(uint32_t(__cvta_generic_to_shared(&tbase))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase + (uint32_t((warp & 3) * 32) << 16);
  float acc = 0.f;
  uint32_t col = uint32_t(warp * 13);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[B][4];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      col = (col * 5 + 7) & 0x1f8;  // 8-column aligned
      ld4<S>(tb + col, v[b]);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int b = 0; b < B; ++b) acc += v[b][0] + v[b][1] + v[b][2] + v[b][3];
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int S, int B> int run(const char* name, int nw, float* out, long long* cyc, int sms) {
  const int iters = 2000;
  k<S, B><<<sms, nw * 32>>>(8, out, cyc);
  CK(cudaDeviceSynchronize());
  k<S, B><<<sms, nw * 32>>>(iters, out, cyc);
  CK(cudaDeviceSynchronize());
  long long c[32];
  CK(cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int w = 0; w < nw; ++w) mx = c[w] > mx ? c[w] : mx;
  printf("%-12s warps %2d B=%d: %6.1f B/clk/SM\n", name, nw, B, double(iters) * B * 512 * nw / double(mx));
  return 0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  CK(cudaMalloc(&out, sizeof(float) * sms * 768));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  for (int nw : {8, 16, 24}) {
    run<0, 4>("32x32b.x4", nw, out, cyc, sms);
    run<1, 4>("16x64b.x4", nw, out, cyc, sms);
    run<2, 4>("16x128b.x2", nw, out, cyc, sms);
    run<3, 4>("16x256b.x1", nw, out, cyc, sms);
  }
  return 0;
}
