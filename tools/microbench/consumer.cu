// Consumer-loop microbenchmark for the TMEM SpMM kernel: X pre-filled in tensor
// memory, synthetic execution-ordered metadata (uniform 90 % sparsity, binomial row counts per K
// chunk) resident in shared memory, no fill and no TMA — only the consumer warps' loop
//   LDS (col, w) → R2UR → tcgen05.ld → FFMA2
// so that loop variants (rows per warp, warps, V, padding U, unroll, pairs of rows, register
// budget) can be compared on useful FMA / clk / SM.  NFW idle warps stand in for the filler warps'
// register share.  usage: consumer [chunks]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int X> struct TL;
template <> struct TL<4> {
  static __device__ __forceinline__ void ld(uint32_t a, float (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
  }
};
template <> struct TL<8> {
  static __device__ __forceinline__ void ld(uint32_t a, float (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(a));
  }
};
template <> struct TL<16> {
  static __device__ __forceinline__ void ld(uint32_t a, float (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                   "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                 : "r"(a));
  }
};
template <int N> __device__ __forceinline__ void twait(float (&v)[N]) {
  // pass the registers through so no use is hoisted above the wait
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+f"(v[i]));
}
template <int V> __device__ __forceinline__ void fmaV(float2 (&acc)[V / 2], float w, const float (&x)[V]) {
  const float2 w2 = make_float2(w, w);
#pragma unroll
  for (int g = 0; g < V / 2; ++g) acc[g] = __ffma2_rn(w2, make_float2(x[2 * g], x[2 * g + 1]), acc[g]);
}

// header word: start (float4 units) << 16 | steps; entries: float4 {col, w, col, w}
// MODE 0: per-row step loop, U entries per step (U/2 float4), all loads then FMAs
// MODE 1: as 0, loop unrolled ×2 (2U loads in flight when ≥ 2 steps remain)
// MODE 2: pairs of rows: rows r, r+1 advance together for min(steps) steps, then the rest alone
template <int V, int RW, int U, int NCW, int NFW, int MODE, int UNI>
__global__ void __launch_bounds__((NCW + NFW) * 32, 1)
    cons_kernel(const uint4* __restrict__ meta_g, int blk_u4, int nblk, int chunks, float* out, long long* cyc) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* ms = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < blk_u4 * nblk; i += blockDim.x) ms[i] = meta_g[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase_s;
  if (warp < 4) {
    const uint32_t tq = tb + (uint32_t(warp * 32) << 16);
    for (int c = 0; c < 512; c += 4) {
      float a = float((lane * 7 + c) & 63) * (1.f / 64.f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tq + c), "f"(a), "f"(a + 1.f),
                   "f"(a + 2.f), "f"(a + 3.f));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp < NCW) {
    const int q = warp & 3, wi = warp >> 2;
    uint32_t tl;
    if (UNI) tl = __shfl_sync(0xffffffffu, uint32_t(q * 32) << 16, 0);
    else tl = uint32_t(q * 32) << 16;
    float2 acc[RW][V / 2];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int g = 0; g < V / 2; ++g) acc[r][g] = make_float2(0.f, 0.f);
    for (int j = 0; j < chunks; ++j) {
      const uint4* blk = ms + size_t(j % nblk) * blk_u4;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(blk) + wi * RW;
      const float4* ent = reinterpret_cast<const float4*>(blk);
      auto step = [&](int r, const float4* e) {
        float4 ee[U / 2];
#pragma unroll
        for (int t = 0; t < U / 2; ++t) ee[t] = e[t];
        float x[U][V];
#pragma unroll
        for (int t = 0; t < U / 2; ++t) {
          TL<V>::ld(tb + tl + __float_as_uint(ee[t].x), x[2 * t]);
          TL<V>::ld(tb + tl + __float_as_uint(ee[t].z), x[2 * t + 1]);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int t = 0; t < U; ++t) {
#pragma unroll
          for (int i = 0; i < V; ++i) asm volatile("" : "+f"(x[t][i]));
          fmaV<V>(acc[r], (t & 1) ? ee[t >> 1].w : ee[t >> 1].y, x[t]);
        }
      };
      if constexpr (MODE == 2) {
#pragma unroll
        for (int r = 0; r < RW; r += 2) {
          const uint32_t ha = hdr[r], hb = hdr[r + 1];
          const float4* ea = ent + (ha >> 16);
          const float4* eb = ent + (hb >> 16);
          int na = int(ha & 0xffffu), nb = int(hb & 0xffffu);
          int nm = min(na, nb);
          for (int s = 0; s < nm; ++s) {
            float4 ea4[U / 2], eb4[U / 2];
#pragma unroll
            for (int t = 0; t < U / 2; ++t) { ea4[t] = ea[t]; eb4[t] = eb[t]; }
            float xa[U][V], xb[U][V];
#pragma unroll
            for (int t = 0; t < U / 2; ++t) {
              TL<V>::ld(tb + tl + __float_as_uint(ea4[t].x), xa[2 * t]);
              TL<V>::ld(tb + tl + __float_as_uint(ea4[t].z), xa[2 * t + 1]);
              TL<V>::ld(tb + tl + __float_as_uint(eb4[t].x), xb[2 * t]);
              TL<V>::ld(tb + tl + __float_as_uint(eb4[t].z), xb[2 * t + 1]);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int t = 0; t < U; ++t) {
#pragma unroll
              for (int i = 0; i < V; ++i) asm volatile("" : "+f"(xa[t][i]), "+f"(xb[t][i]));
              fmaV<V>(acc[r], (t & 1) ? ea4[t >> 1].w : ea4[t >> 1].y, xa[t]);
              fmaV<V>(acc[r + 1], (t & 1) ? eb4[t >> 1].w : eb4[t >> 1].y, xb[t]);
            }
            ea += U / 2;
            eb += U / 2;
          }
          for (int s = nm; s < na; ++s, ea += U / 2) step(r, ea);
          for (int s = nm; s < nb; ++s, eb += U / 2) step(r + 1, eb);
        }
      } else {
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          const uint32_t hh = hdr[r];
          const float4* e = ent + (hh >> 16);
          int n = int(hh & 0xffffu);
          if constexpr (MODE == 1) {
            for (; n >= 2; n -= 2, e += U) {
              float4 ee[U];
#pragma unroll
              for (int t = 0; t < U; ++t) ee[t] = e[t];
              float x[2 * U][V];
#pragma unroll
              for (int t = 0; t < U; ++t) {
                TL<V>::ld(tb + tl + __float_as_uint(ee[t].x), x[2 * t]);
                TL<V>::ld(tb + tl + __float_as_uint(ee[t].z), x[2 * t + 1]);
              }
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
              for (int t = 0; t < 2 * U; ++t) {
#pragma unroll
                for (int i = 0; i < V; ++i) asm volatile("" : "+f"(x[t][i]));
                fmaV<V>(acc[r], (t & 1) ? ee[t >> 1].w : ee[t >> 1].y, x[t]);
              }
            }
          }
          for (; n > 0; --n, e += U / 2) step(r, e);
        }
      }
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int g = 0; g < V / 2; ++g) s += acc[r][g].x + acc[r][g].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = warp < NCW ? t1 - t0 : 0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// Synthetic metadata: nblk blocks (block b → TMEM half b & 1), rows = NCW/4·RW, K chunk = 256/V
// rows, each row's nonzeros Bernoulli(density) over the chunk, padded to U with weight 0.
struct Meta {
  std::vector<uint4> words;
  int blk_u4 = 0;
  double useful_nz_per_blk = 0;  // Σ over rows of real nonzeros (per block, averaged)
  double padded_nz_per_blk = 0;
};
static Meta make_meta(int V, int RW, int U, int NCW, int nblk, double density, unsigned seed) {
  const int rows = NCW / 4 * RW, KC = 256 / V;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  std::vector<std::vector<uint32_t>> blocks;
  int maxw = 0;
  Meta m;
  for (int b = 0; b < nblk; ++b) {
    const int hdr_u4 = (rows + 3) / 4;
    std::vector<uint32_t> w(size_t(hdr_u4) * 4, 0u);
    for (int r = 0; r < rows; ++r) {
      std::vector<int> cols;
      for (int k = 0; k < KC; ++k)
        if (uni(rng) < density) cols.push_back(k);
      m.useful_nz_per_blk += cols.size();
      const int steps = int((cols.size() + U - 1) / U);
      m.padded_nz_per_blk += steps * U;
      const uint32_t start_u4 = uint32_t(w.size() / 4);
      w[r] = (start_u4 << 16) | uint32_t(steps);
      for (int s = 0; s < steps * U; ++s) {
        const bool real = s < int(cols.size());
        const int k = real ? cols[s] : (cols.empty() ? 0 : cols.back());
        const uint32_t tcol = uint32_t(V * k + 256 * (b & 1));
        const float wv = real ? 0.01f * float(1 + (s % 7)) : 0.f;
        uint32_t wbits;
        memcpy(&wbits, &wv, 4);
        w.push_back(tcol);
        w.push_back(wbits);
      }
      while (w.size() % 4) w.push_back(0u);
    }
    maxw = std::max(maxw, int(w.size()));
    blocks.push_back(w);
  }
  m.blk_u4 = (maxw + 3) / 4;
  m.words.assign(size_t(m.blk_u4) * nblk, make_uint4(0, 0, 0, 0));
  for (int b = 0; b < nblk; ++b) memcpy(&m.words[size_t(b) * m.blk_u4], blocks[b].data(), blocks[b].size() * 4);
  m.useful_nz_per_blk /= nblk;
  m.padded_nz_per_blk /= nblk;
  return m;
}

template <int V, int RW, int U, int NCW, int NFW, int MODE, int UNI>
static void run(const char* name, int chunks, double density = 0.1) {
  const int nblk = 8;
  Meta m = make_meta(V, RW, U, NCW, nblk, density, 1234);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* mg;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&mg, m.words.size() * sizeof(uint4)));
  CK(cudaMemcpy(mg, m.words.data(), m.words.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  auto kern = cons_kernel<V, RW, U, NCW, NFW, MODE, UNI>;
  const size_t smem = m.words.size() * sizeof(uint4);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  kern<<<sms, (NCW + NFW) * 32, smem>>>(mg, m.blk_u4, nblk, 4, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, (NCW + NFW) * 32, smem>>>(mg, m.blk_u4, nblk, chunks, out, cyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(size_t(sms) * 32);
  CK(cudaMemcpy(c.data(), cyc, c.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  long long cmax = 0;
  for (int w = 0; w < NCW; ++w) cmax = std::max(cmax, c[w]);
  // useful FMAs per CTA: per block Σ nnz × (V columns × 32 lanes) × 4 lane quarters
  const double fma_cta = m.useful_nz_per_blk * V * 32.0 * 4.0 * chunks / 1.0;
  const double fma_per_clk = fma_cta / double(cmax);
  const double tflops = 2.0 * fma_cta * sms / (ms * 1e-3) / 1e12;
  printf("%-34s regs %3d  pad %.2f  useful FMA/clk/SM %6.1f (%5.1f %% of 128)  %7.3f ms  %6.2f TF(eff)\n", name,
         fa.numRegs, m.padded_nz_per_blk / m.useful_nz_per_blk, fma_per_clk, fma_per_clk / 128.0 * 100.0, ms, tflops);
  fflush(stdout);
  CK(cudaFree(mg));
  CK(cudaFree(out));
  CK(cudaFree(cyc));
}


// ---- MODE P: replicated lane quarters (every quarter holds the same X columns; the quarters' warps own
// different rows, lane base baked into the metadata), V = 8, pairs of entries per step, two-deep
// software pipeline (the next pair's loads are issued before this pair's FFMA2s), rows padded to
// whole pairs.  Header word per (warp, row): start_u4 << 16 | pairs.  Each warp stream ends with a
// dummy pair (lookahead target).  NFW filler warps: FB = 0 idle, 1 = emulate the replicated fill
// (every filler reads the whole 32 KB chunk tile with LDS.128 and writes its quarter with
// tcgen05.st.x16), once per consumer chunk, unsynchronised.
template <int N> __device__ __forceinline__ void tld8(uint32_t a, float (&v)[8]) { TL<8>::ld(a, v); }
__device__ __forceinline__ void fma8(float2 (&acc)[4], float w, const float (&x)[8]) {
  const float2 w2 = make_float2(w, w);
#pragma unroll
  for (int g = 0; g < 4; ++g) acc[g] = __ffma2_rn(w2, make_float2(x[2 * g], x[2 * g + 1]), acc[g]);
}
__device__ __forceinline__ void twait_all() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
template <int RW, int NCW, int NFW, int REGC, int REGF, int FB>
__global__ void __launch_bounds__((NCW + NFW) * 32, 1)
    pipe_kernel(const uint4* __restrict__ meta_g, int blk_u4, int nblk, int chunks, float* out, long long* cyc) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* ms = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < blk_u4 * nblk; i += blockDim.x) ms[i] = meta_g[i];
  float4* tile = reinterpret_cast<float4*>(smem + size_t(blk_u4) * nblk * 16);
  if (FB)
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) tile[i] = make_float4(1.f, 2.f, 3.f, float(i & 7));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase_s;
  if (warp < 4) {
    const uint32_t tq = tb + (uint32_t(warp * 32) << 16);
    for (int c = 0; c < 512; c += 4) {
      float a = float((lane * 7 + c) & 63) * (1.f / 64.f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tq + c), "f"(a), "f"(a + 1.f),
                   "f"(a + 2.f), "f"(a + 3.f));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp < NCW) {
    if (REGC) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGC));
    float2 acc[RW][4];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int g = 0; g < 4; ++g) acc[r][g] = make_float2(0.f, 0.f);
    for (int j = 0; j < chunks; ++j) {
      const uint4* blk = ms + size_t(j % nblk) * blk_u4;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(blk) + warp * RW;
      const float4* e = reinterpret_cast<const float4*>(blk) + (hdr[0] >> 16);
      float xa0[8], xa1[8], xb0[8], xb1[8];
      float4 fa = e[0];
      tld8<8>(tb + __float_as_uint(fa.x), xa0);
      tld8<8>(tb + __float_as_uint(fa.z), xa1);
      ++e;
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        int n = int(hdr[r] & 0xffffu);
        for (; n >= 2; n -= 2, e += 2) {
          const float4 fb = e[0];
          twait_all();
#pragma unroll
          for (int i = 0; i < 8; ++i) asm volatile("" : "+f"(xa0[i]), "+f"(xa1[i]));
          tld8<8>(tb + __float_as_uint(fb.x), xb0);
          tld8<8>(tb + __float_as_uint(fb.z), xb1);
          fma8(acc[r], fa.y, xa0);
          fma8(acc[r], fa.w, xa1);
          fa = e[1];
          twait_all();
#pragma unroll
          for (int i = 0; i < 8; ++i) asm volatile("" : "+f"(xb0[i]), "+f"(xb1[i]));
          tld8<8>(tb + __float_as_uint(fa.x), xa0);
          tld8<8>(tb + __float_as_uint(fa.z), xa1);
          fma8(acc[r], fb.y, xb0);
          fma8(acc[r], fb.w, xb1);
        }
        if (n) {  // odd pair count: one pair, then the lookahead lands in B → move it to A
          const float4 fb = e[0];
          twait_all();
#pragma unroll
          for (int i = 0; i < 8; ++i) asm volatile("" : "+f"(xa0[i]), "+f"(xa1[i]));
          tld8<8>(tb + __float_as_uint(fb.x), xb0);
          tld8<8>(tb + __float_as_uint(fb.z), xb1);
          fma8(acc[r], fa.y, xa0);
          fma8(acc[r], fa.w, xa1);
          twait_all();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            asm volatile("" : "+f"(xb0[i]), "+f"(xb1[i]));
            xa0[i] = xb0[i];
            xa1[i] = xb1[i];
          }
          fa = fb;
          ++e;
        }
      }
      twait_all();
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("" : "+f"(xa0[i]), "+f"(xa1[i]));
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int g = 0; g < 4; ++g) s += acc[r][g].x + acc[r][g].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    if (REGF) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGF));
    if (FB) {
      const uint32_t tq = tb + (uint32_t((warp & 3) * 32) << 16);
      for (int j = 0; j < chunks; ++j) {
        // one chunk: 32 K rows × 256 columns = 32 KB; each lane reads 1 KB (64 × LDS.128), writes 16 × x16
#pragma unroll 1
        for (int u = 0; u < 16; ++u) {
          float4 v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) v[t] = tile[(u * 4 + t) * 32 + lane];
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
              "%15, %16};" ::"r"(tq + uint32_t(256 * (j & 1) + 16 * (u & 15))),
              "f"(v[0].x), "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z), "f"(v[1].w),
              "f"(v[2].x), "f"(v[2].y), "f"(v[2].z), "f"(v[2].w), "f"(v[3].x), "f"(v[3].y), "f"(v[3].z), "f"(v[3].w));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// metadata for pipe_kernel: NCW warps × RW rows, K chunk 32 rows (V = 8), Bernoulli(density), rows
// padded to whole pairs, lane base of warp w's quarter (w % 4) baked into every column.
static Meta make_meta_p(int RW, int NCW, int nblk, double density, unsigned seed) {
  const int KC = 32;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  std::vector<std::vector<uint32_t>> blocks;
  int maxw = 0;
  Meta m;
  for (int b = 0; b < nblk; ++b) {
    const int hdr_u4 = (NCW * RW + 3) / 4;
    std::vector<uint32_t> w(size_t(hdr_u4) * 4, 0u);
    for (int wp = 0; wp < NCW; ++wp) {
      const uint32_t lb = uint32_t((wp & 3) * 32) << 16;
      for (int r = 0; r < RW; ++r) {
        std::vector<int> cols;
        for (int k = 0; k < KC; ++k)
          if (uni(rng) < density) cols.push_back(k);
        m.useful_nz_per_blk += cols.size() / 4.0;  // ×4 below counts quarters; here every row is one warp's
        const int pairs = int((cols.size() + 1) / 2);
        m.padded_nz_per_blk += pairs * 2 / 4.0;
        w[wp * RW + r] = (uint32_t(w.size() / 4) << 16) | uint32_t(pairs);
        for (int s = 0; s < pairs * 2; ++s) {
          const bool real = s < int(cols.size());
          const int k = real ? cols[s] : (cols.empty() ? 0 : cols.back());
          const float wv = real ? 0.01f * float(1 + (s % 7)) : 0.f;
          uint32_t wb;
          memcpy(&wb, &wv, 4);
          w.push_back(lb | uint32_t(8 * k + 256 * (b & 1)));
          w.push_back(wb);
        }
      }
      w.push_back(lb);  // dummy lookahead pair
      w.push_back(0u);
      w.push_back(lb);
      w.push_back(0u);
    }
    maxw = std::max(maxw, int(w.size()));
    blocks.push_back(w);
  }
  m.blk_u4 = (maxw + 3) / 4;
  m.words.assign(size_t(m.blk_u4) * nblk, make_uint4(0, 0, 0, 0));
  for (int b = 0; b < nblk; ++b) memcpy(&m.words[size_t(b) * m.blk_u4], blocks[b].data(), blocks[b].size() * 4);
  m.useful_nz_per_blk /= nblk;
  m.padded_nz_per_blk /= nblk;
  return m;
}

template <int RW, int NCW, int NFW, int REGC, int REGF, int FB>
static void run_p(const char* name, int chunks, double density = 0.1) {
  const int nblk = 8;
  Meta m = make_meta_p(RW, NCW, nblk, density, 4321);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* mg;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&mg, m.words.size() * sizeof(uint4)));
  CK(cudaMemcpy(mg, m.words.data(), m.words.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  auto kern = pipe_kernel<RW, NCW, NFW, REGC, REGF, FB>;
  const size_t smem = m.words.size() * sizeof(uint4) + 32768;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  kern<<<sms, (NCW + NFW) * 32, smem>>>(mg, m.blk_u4, nblk, 4, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, (NCW + NFW) * 32, smem>>>(mg, m.blk_u4, nblk, chunks, out, cyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(size_t(sms) * 32);
  CK(cudaMemcpy(c.data(), cyc, c.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  long long cmax = 0, fmax = 0;
  for (int w = 0; w < NCW; ++w) cmax = std::max(cmax, c[w]);
  for (int w = NCW; w < NCW + NFW; ++w) fmax = std::max(fmax, c[w]);
  const double fma_cta = m.useful_nz_per_blk * 8 * 32.0 * 4.0 * chunks;
  const double fma_per_clk = fma_cta / double(std::max(cmax, fmax));
  const double tflops = 2.0 * fma_cta * sms / (ms * 1e-3) / 1e12;
  printf("%-34s regs %3d  pad %.2f  useful FMA/clk/SM %6.1f (%5.1f %% of 128)  cons %lld fill %lld cyc  %7.3f ms  %6.2f TF(eff)\n",
         name, fa.numRegs, m.padded_nz_per_blk / m.useful_nz_per_blk, fma_per_clk, fma_per_clk / 128.0 * 100.0, cmax,
         fmax, ms, tflops);
  fflush(stdout);
  CK(cudaFree(mg));
  CK(cudaFree(out));
  CK(cudaFree(cyc));
}


// ---- MODE R: replicated lane quarters, V = 4 (TN = 128): every warp owns its rows, lane base baked into
// the metadata, rows padded to whole pairs, one contiguous entry stream per warp (row headers: pairs),
// steps of two pairs (4 loads) while ≥ 2 pairs remain, then one pair.
template <int RW, int NCW, int NFW, int FB>
__global__ void __launch_bounds__((NCW + NFW) * 32, 1)
    r_kernel(const uint4* __restrict__ meta_g, int blk_u4, int nblk, int chunks, float* out, long long* cyc) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* ms = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < blk_u4 * nblk; i += blockDim.x) ms[i] = meta_g[i];
  float4* tile = reinterpret_cast<float4*>(smem + size_t(blk_u4) * nblk * 16);
  if (FB)
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) tile[i] = make_float4(1.f, 2.f, 3.f, float(i & 7));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase_s;
  if (warp < 4) {
    const uint32_t tq = tb + (uint32_t(warp * 32) << 16);
    for (int c = 0; c < 512; c += 4) {
      float a = float((lane * 7 + c) & 63) * (1.f / 64.f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tq + c), "f"(a), "f"(a + 1.f),
                   "f"(a + 2.f), "f"(a + 3.f));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp < NCW) {
    float2 acc[RW][2];
#pragma unroll
    for (int r = 0; r < RW; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
    for (int j = 0; j < chunks; ++j) {
      const uint4* blk = ms + size_t(j % nblk) * blk_u4;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(blk) + warp * 16;  // [0] = stream start (float4), [1..RW] = pairs
      const float4* e = reinterpret_cast<const float4*>(blk) + __shfl_sync(0xffffffffu, hdr[0], 0);
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        int n = __shfl_sync(0xffffffffu, int(hdr[1 + r]), 0);
        for (; n >= 2; n -= 2, e += 2) {
          const float4 f0 = e[0], f1 = e[1];
          float x0[4], x1[4], x2[4], x3[4];
          TL<4>::ld(__float_as_uint(f0.x), x0);
          TL<4>::ld(__float_as_uint(f0.z), x1);
          TL<4>::ld(__float_as_uint(f1.x), x2);
          TL<4>::ld(__float_as_uint(f1.z), x3);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 4; ++i) asm volatile("" : "+f"(x0[i]), "+f"(x1[i]), "+f"(x2[i]), "+f"(x3[i]));
          fmaV<4>(acc[r], f0.y, x0);
          fmaV<4>(acc[r], f0.w, x1);
          fmaV<4>(acc[r], f1.y, x2);
          fmaV<4>(acc[r], f1.w, x3);
        }
        if (n) {
          const float4 f0 = e[0];
          float x0[4], x1[4];
          TL<4>::ld(__float_as_uint(f0.x), x0);
          TL<4>::ld(__float_as_uint(f0.z), x1);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 4; ++i) asm volatile("" : "+f"(x0[i]), "+f"(x1[i]));
          fmaV<4>(acc[r], f0.y, x0);
          fmaV<4>(acc[r], f0.w, x1);
          ++e;
        }
      }
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < RW; ++r) s += acc[r][0].x + acc[r][0].y + acc[r][1].x + acc[r][1].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else if (FB) {
    const uint32_t tq = tb + (uint32_t((warp & 3) * 32) << 16);
    const float4* src = tile + lane;
    for (int j = 0; j < chunks; ++j) {
      // one chunk: 64 K rows × 128 columns = 32 KB; each lane reads 1 KB (64 × LDS.128), writes 16 × x16
#pragma unroll 1
      for (int u = 0; u < 16; ++u) {
        float4 v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) v[t] = src[(u * 4 + t) * 32];
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16};" ::"r"(tq + uint32_t(256 * (j & 1) + 16 * u)),
            "f"(v[0].x), "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z), "f"(v[1].w),
            "f"(v[2].x), "f"(v[2].y), "f"(v[2].z), "f"(v[2].w), "f"(v[3].x), "f"(v[3].y), "f"(v[3].z), "f"(v[3].w));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

static Meta make_meta_r(int RW, int NCW, int nblk, double density, unsigned seed) {
  const int KC = 64;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  std::vector<std::vector<uint32_t>> blocks;
  int maxw = 0;
  Meta m;
  for (int b = 0; b < nblk; ++b) {
    std::vector<uint32_t> w(size_t(NCW) * 16, 0u);
    for (int wp = 0; wp < NCW; ++wp) {
      const uint32_t lb = uint32_t((wp & 3) * 32) << 16;
      w[wp * 16] = uint32_t(w.size() / 4);
      for (int r = 0; r < RW; ++r) {
        std::vector<int> cols;
        for (int k = 0; k < KC; ++k)
          if (uni(rng) < density) cols.push_back(k);
        m.useful_nz_per_blk += cols.size() / 4.0;
        const int pairs = int((cols.size() + 1) / 2);
        m.padded_nz_per_blk += pairs * 2 / 4.0;
        w[wp * 16 + 1 + r] = uint32_t(pairs);
        for (int s = 0; s < pairs * 2; ++s) {
          const bool real = s < int(cols.size());
          const int k = real ? cols[s] : (cols.empty() ? 0 : cols.back());
          const float wv = real ? 0.01f * float(1 + (s % 7)) : 0.f;
          uint32_t wb;
          memcpy(&wb, &wv, 4);
          w.push_back(lb | uint32_t(4 * k + 256 * (b & 1)));
          w.push_back(wb);
        }
      }
    }
    maxw = std::max(maxw, int(w.size()));
    blocks.push_back(w);
  }
  m.blk_u4 = (maxw + 3) / 4;
  m.words.assign(size_t(m.blk_u4) * nblk, make_uint4(0, 0, 0, 0));
  for (int b = 0; b < nblk; ++b) memcpy(&m.words[size_t(b) * m.blk_u4], blocks[b].data(), blocks[b].size() * 4);
  m.useful_nz_per_blk /= nblk;
  m.padded_nz_per_blk /= nblk;
  return m;
}

template <int RW, int NCW, int NFW, int FB>
static void run_r(const char* name, int chunks, double density = 0.1) {
  const int nblk = 8;
  Meta m = make_meta_r(RW, NCW, nblk, density, 777);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* mg;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&mg, m.words.size() * sizeof(uint4)));
  CK(cudaMemcpy(mg, m.words.data(), m.words.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  auto kern = r_kernel<RW, NCW, NFW, FB>;
  const size_t smem = m.words.size() * sizeof(uint4) + 32768;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  kern<<<sms, (NCW + NFW) * 32, smem>>>(mg, m.blk_u4, nblk, 4, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, (NCW + NFW) * 32, smem>>>(mg, m.blk_u4, nblk, chunks, out, cyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(size_t(sms) * 32);
  CK(cudaMemcpy(c.data(), cyc, c.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  long long cmax = 0, fmax = 0;
  for (int w = 0; w < NCW; ++w) cmax = std::max(cmax, c[w]);
  for (int w = NCW; w < NCW + NFW; ++w) fmax = std::max(fmax, c[w]);
  const double fma_cta = m.useful_nz_per_blk * 4 * 32.0 * 4.0 * chunks;
  const double fma_per_clk = fma_cta / double(std::max(cmax, fmax));
  const double tflops = 2.0 * fma_cta * sms / (ms * 1e-3) / 1e12;
  printf("%-34s regs %3d  pad %.2f  useful FMA/clk/SM %6.1f (%5.1f %% of 128)  cons %lld fill %lld cyc  %7.3f ms  %6.2f TF(eff)\n",
         name, fa.numRegs, m.padded_nz_per_blk / m.useful_nz_per_blk, fma_per_clk, fma_per_clk / 128.0 * 100.0, cmax,
         fmax, ms, tflops);
  fflush(stdout);
  CK(cudaFree(mg));
  CK(cudaFree(out));
  CK(cudaFree(cyc));
}
int main(int argc, char** argv) {
  const int chunks = argc > 1 ? atoi(argv[1]) : 2048;
  if (argc > 2 && argv[2][0] == 'r') {
    run_r<10, 24, 4, 0>("R V4 RW10 24+4 idle", chunks);
    run_r<10, 24, 4, 1>("R V4 RW10 24+4 fill", chunks);
    run_r<8, 24, 4, 0>("R V4 RW8 24+4 idle", chunks);
    run_r<12, 20, 4, 0>("R V4 RW12 20+4 idle", chunks);
    run_r<12, 20, 4, 1>("R V4 RW12 20+4 fill", chunks);
    run_r<16, 16, 4, 0>("R V4 RW16 16+4 idle", chunks);
    run_r<10, 28, 0, 0>("R V4 RW10 28+0", chunks);
    run_r<10, 24, 4, 0>("R V4 RW10 24+4 d=0.2", chunks, 0.2);
    run_r<10, 24, 4, 0>("R V4 RW10 24+4 d=0.05", chunks, 0.05);
    return 0;
  }
  if (argc > 2) {
    run_p<8, 16, 4, 112, 32, 0>("P V8 RW8 16+4 reg112/32 idle", chunks);
    run_p<8, 16, 4, 112, 32, 1>("P V8 RW8 16+4 reg112/32 fill", chunks);
    run_p<8, 16, 0, 0, 0, 0>("P V8 RW8 16+0", chunks);
    run_p<10, 12, 4, 152, 32, 0>("P V8 RW10 12+4 reg152/32 idle", chunks);
    run_p<12, 12, 4, 152, 32, 0>("P V8 RW12 12+4 reg152/32 idle", chunks);
    run_p<12, 12, 4, 152, 32, 1>("P V8 RW12 12+4 reg152/32 fill", chunks);
    run_p<8, 16, 4, 112, 32, 0>("P V8 RW8 16+4 d=0.2", chunks, 0.2);
    run_p<8, 16, 4, 112, 32, 0>("P V8 RW8 16+4 d=0.05", chunks, 0.05);
    return 0;
  }
  // product today: V4 U4 10 rows × 24 warps + 4 fillers
  run<4, 10, 4, 24, 4, 0, 0>("V4 U4 RW10 24+4 m0", chunks);
  run<4, 10, 4, 24, 4, 0, 1>("V4 U4 RW10 24+4 m0 uni", chunks);
  run<4, 10, 4, 24, 4, 1, 0>("V4 U4 RW10 24+4 unroll2", chunks);
  run<4, 10, 4, 24, 4, 2, 0>("V4 U4 RW10 24+4 pairs", chunks);
  run<4, 10, 2, 24, 4, 0, 0>("V4 U2 RW10 24+4 m0", chunks);
  run<4, 10, 2, 24, 4, 1, 0>("V4 U2 RW10 24+4 unroll2", chunks);
  run<4, 10, 2, 24, 4, 2, 0>("V4 U2 RW10 24+4 pairs", chunks);
  run<4, 8, 4, 24, 4, 0, 0>("V4 U4 RW8 24+4 m0", chunks);
  run<4, 8, 4, 24, 4, 2, 0>("V4 U4 RW8 24+4 pairs", chunks);
  run<4, 12, 4, 20, 4, 0, 0>("V4 U4 RW12 20+4 m0", chunks);
  run<4, 12, 4, 20, 4, 2, 0>("V4 U4 RW12 20+4 pairs", chunks);
  run<4, 20, 4, 12, 4, 0, 0>("V4 U4 RW20 12+4 m0", chunks);
  run<4, 20, 4, 12, 4, 2, 0>("V4 U4 RW20 12+4 pairs", chunks);
  run<4, 10, 4, 24, 0, 0, 0>("V4 U4 RW10 24+0 m0", chunks);
  run<4, 10, 4, 24, 0, 2, 0>("V4 U4 RW10 24+0 pairs", chunks);
  run<8, 5, 2, 24, 4, 0, 0>("V8 U2 RW5 24+4 m0", chunks);
  run<8, 6, 2, 24, 4, 0, 0>("V8 U2 RW6 24+4 m0", chunks);
  run<8, 6, 2, 24, 4, 2, 0>("V8 U2 RW6 24+4 pairs", chunks);
  run<8, 6, 2, 24, 4, 1, 0>("V8 U2 RW6 24+4 unroll2", chunks);
  run<8, 5, 2, 24, 4, 1, 0>("V8 U2 RW5 24+4 unroll2", chunks);
  run<8, 10, 2, 12, 4, 0, 0>("V8 U2 RW10 12+4 m0", chunks);
  run<8, 10, 2, 12, 4, 2, 0>("V8 U2 RW10 12+4 pairs", chunks);
  run<8, 8, 2, 16, 4, 2, 0>("V8 U2 RW8 16+4 pairs", chunks);
  run<8, 4, 2, 32, 0, 2, 0>("V8 U2 RW4 32+0 pairs", chunks);
  run<16, 4, 2, 12, 4, 0, 0>("V16 U2 RW4 12+4 m0", chunks);
  run<16, 4, 2, 12, 4, 2, 0>("V16 U2 RW4 12+4 pairs", chunks);
  run<16, 2, 2, 24, 4, 2, 0>("V16 U2 RW2 24+4 pairs", chunks);
  return 0;
}
