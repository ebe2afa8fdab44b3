// Metadata-format microbenchmark: the TMEM-R consumer step with the metadata read in
// different forms, to separate the two candidate bounds of the consumer loop — the number of
// MIO instructions (LDS + LDTM) per nonzero, or the bytes those loads write into the register file
// (a broadcast LDS.128 writes 32 lanes × 16 B, as many as a tcgen05.ld.32x32b.x4):
//   MODE 0  the product's form: LDS.128 {col, w, col, w} per 2 entries       (0.5 LDS, 256 B / nz)
//   MODE 1  LDS.128 {c0, c1, c2, c3} per 4 entries, weight a constant        (0.25 LDS, 128 B / nz)  [timing only]
//   MODE 2  LDS.128 {w0..w3} + LDS.64 {c0|c1, c2|c3} (16-bit TMEM columns, the
//           warp's lane base added in the kernel) per 4 entries (32 B of smem) (0.5 LDS, 192 B / nz)
//   MODE 4  lane-distributed metadata: one coalesced LDS.64 per 32 entries (lane l keeps entry l), each
//           entry's col and w broadcast through the uniform datapath (SEL + REDUX.OR -> UR): no
//           broadcast load writes the register file                          (1/32 LDS, 8 B / nz)
//   MODE 5  columns as in MODE 4 (REDUX), weights by one broadcast LDS.128 per 4 entries  (128 B / nz) [timing only]
// Rows padded to multiples of 4 entries in every mode; rates are per padded entry.  No fill, no TMA.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void tld4(uint32_t a, float4& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
}
__device__ __forceinline__ void twait(float4& a, float4& b, float4& c, float4& d) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  asm volatile("" : "+f"(a.x), "+f"(a.y), "+f"(a.z), "+f"(a.w), "+f"(b.x), "+f"(b.y), "+f"(b.z), "+f"(b.w));
  asm volatile("" : "+f"(c.x), "+f"(c.y), "+f"(c.z), "+f"(c.w), "+f"(d.x), "+f"(d.y), "+f"(d.z), "+f"(d.w));
}
__device__ __forceinline__ void fma4(float2 (&acc)[2], float w, const float4 x) {
  const float2 w2 = make_float2(w, w);
  acc[0] = __ffma2_rn(w2, make_float2(x.x, x.y), acc[0]);
  acc[1] = __ffma2_rn(w2, make_float2(x.z, x.w), acc[1]);
}

constexpr int RW = 10, NCW = 24, NFW = 4;

// per chunk block: header RW words per warp (groups of 4 entries per row), then per warp a stream
// start (16-byte units) in word [NCW * RW + warp]; streams laid out per mode
// SYNC > 0: the consumer warps meet at a named barrier every SYNC chunks (the product's TMEM halves
// let a warp run at most about one chunk ahead of the slowest: per-chunk load imbalance between
// warps then costs time)
template <int MODE, int SYNC = 0>
__global__ void __launch_bounds__((NCW + NFW) * 32, 1)
    meta_kernel(const uint4* __restrict__ meta_g, int blk_u4, int nblk, int chunks, float* out, long long* cyc) {
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
    const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
    float2 acc[RW][2];
#pragma unroll
    for (int r = 0; r < RW; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
    uint2 ent = make_uint2(0u, 0u);  // MODE 4 / 5: this lane's entry of the current 32-entry window
    int pos = 32;
    for (int j = 0; j < chunks; ++j) {
      if (MODE >= 4) pos = 32;  // a new chunk's stream starts elsewhere: reload the window
      if (SYNC && j % SYNC == 0) asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
      const uint4* blk = ms + size_t(j % nblk) * blk_u4;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(blk) + warp * RW;
      const uint4* e = blk + __shfl_sync(0xffffffffu, reinterpret_cast<const uint32_t*>(blk)[NCW * RW + warp], 0);
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        int n = __shfl_sync(0xffffffffu, int(hdr[r]), 0);  // groups of 4 entries
        for (; n > 0; --n) {
          float4 xa, xb, xc, xd;
          float w0, w1, w2, w3;
          if constexpr (MODE == 0) {
            const float4 e0 = reinterpret_cast<const float4*>(e)[0], e1 = reinterpret_cast<const float4*>(e)[1];
            tld4(__float_as_uint(e0.x), xa);
            tld4(__float_as_uint(e0.z), xb);
            tld4(__float_as_uint(e1.x), xc);
            tld4(__float_as_uint(e1.z), xd);
            w0 = e0.y; w1 = e0.w; w2 = e1.y; w3 = e1.w;
            e += 2;
          } else if constexpr (MODE == 1) {
            const uint4 c = e[0];
            tld4(c.x, xa);
            tld4(c.y, xb);
            tld4(c.z, xc);
            tld4(c.w, xd);
            w0 = 0.011f; w1 = 0.012f; w2 = 0.013f; w3 = 0.014f;
            e += 1;
          } else if constexpr (MODE == 2) {
            const float4 wv = reinterpret_cast<const float4*>(e)[0];
            const uint2 c = reinterpret_cast<const uint2*>(e + 1)[0];
            tld4(lb | (c.x & 0xffffu), xa);
            tld4(lb | (c.x >> 16), xb);
            tld4(lb | (c.y & 0xffffu), xc);
            tld4(lb | (c.y >> 16), xd);
            w0 = wv.x; w1 = wv.y; w2 = wv.z; w3 = wv.w;
            e += 2;
          } else if constexpr (MODE == 4 || MODE == 5) {
            if (pos == 32) {
              ent = reinterpret_cast<const uint2*>(e)[lane];
              pos = 0;
            }
            const uint32_t c0 = __reduce_or_sync(0xffffffffu, lane == pos ? ent.x : 0u);
            const uint32_t c1 = __reduce_or_sync(0xffffffffu, lane == pos + 1 ? ent.x : 0u);
            const uint32_t c2 = __reduce_or_sync(0xffffffffu, lane == pos + 2 ? ent.x : 0u);
            const uint32_t c3 = __reduce_or_sync(0xffffffffu, lane == pos + 3 ? ent.x : 0u);
            tld4(c0, xa);
            tld4(c1, xb);
            tld4(c2, xc);
            tld4(c3, xd);
            if constexpr (MODE == 4) {
              w0 = __uint_as_float(__reduce_or_sync(0xffffffffu, lane == pos ? ent.y : 0u));
              w1 = __uint_as_float(__reduce_or_sync(0xffffffffu, lane == pos + 1 ? ent.y : 0u));
              w2 = __uint_as_float(__reduce_or_sync(0xffffffffu, lane == pos + 2 ? ent.y : 0u));
              w3 = __uint_as_float(__reduce_or_sync(0xffffffffu, lane == pos + 3 ? ent.y : 0u));
            } else {
              const float4 wv = reinterpret_cast<const float4*>(e)[0];
              w0 = wv.x; w1 = wv.y; w2 = wv.z; w3 = wv.w;
            }
            pos += 4;
            e += 2;
          } else {
            const uint32_t* c = reinterpret_cast<const uint32_t*>(e);
            tld4(c[0], xa);
            tld4(c[1], xb);
            tld4(c[2], xc);
            tld4(c[3], xd);
            w0 = 0.011f; w1 = 0.012f; w2 = 0.013f; w3 = 0.014f;
            e += 1;
          }
          twait(xa, xb, xc, xd);
          fma4(acc[r], w0, xa);
          fma4(acc[r], w1, xb);
          fma4(acc[r], w2, xc);
          fma4(acc[r], w3, xd);
        }
      }
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < RW; ++r) s += acc[r][0].x + acc[r][0].y + acc[r][1].x + acc[r][1].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

struct Meta {
  std::vector<uint4> words;
  int blk_u4 = 0;
  double padded = 0, useful = 0;  // entries per block
};
static Meta make_meta(int mode, int nblk, double density, unsigned seed) {
  const int KC = 64;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  std::vector<std::vector<uint32_t>> blocks;
  Meta m;
  size_t maxw = 0;
  const size_t hdr_words = size_t(NCW) * RW + NCW;
  for (int b = 0; b < nblk; ++b) {
    std::vector<uint32_t> w((hdr_words + 3) / 4 * 4, 0u);
    for (int wp = 0; wp < NCW; ++wp) {
      const uint32_t lb = uint32_t((wp & 3) * 32) << 16;
      w[NCW * RW + wp] = uint32_t(w.size() / 4);
      for (int r = 0; r < RW; ++r) {
        std::vector<int> cols;
        for (int k = 0; k < KC; ++k)
          if (uni(rng) < density) cols.push_back(k);
        m.useful += double(cols.size());
        const int groups = int((cols.size() + 3) / 4);
        m.padded += 4.0 * groups;
        w[wp * RW + r] = uint32_t(groups);
        for (int gi = 0; gi < groups; ++gi) {
          uint32_t c[4], wb[4];
          for (int t = 0; t < 4; ++t) {
            const int s = gi * 4 + t;
            const bool real = s < int(cols.size());
            const int k = real ? cols[s] : cols.back();
            const float wv = real ? 0.01f * float(1 + (s % 7)) : 0.f;
            memcpy(&wb[t], &wv, 4);
            c[t] = uint32_t(4 * k + 256 * (b & 1));
          }
          if (mode == 0 || mode == 4 || mode == 5) {
            for (int t = 0; t < 4; ++t) { w.push_back(lb | c[t]); w.push_back(wb[t]); }
          } else if (mode == 1 || mode == 3) {
            for (int t = 0; t < 4; ++t) w.push_back(lb | c[t]);
          } else {
            for (int t = 0; t < 4; ++t) w.push_back(wb[t]);
            w.push_back(c[0] | (c[1] << 16));
            w.push_back(c[2] | (c[3] << 16));
            w.push_back(0u);
            w.push_back(0u);
          }
        }
      }
      while (w.size() % 4) w.push_back(0u);
    }
    maxw = std::max(maxw, w.size());
    blocks.push_back(w);
  }
  m.blk_u4 = int((maxw + 3) / 4);
  m.words.assign(size_t(m.blk_u4) * nblk, make_uint4(0, 0, 0, 0));
  for (int b = 0; b < nblk; ++b) memcpy(&m.words[size_t(b) * m.blk_u4], blocks[b].data(), blocks[b].size() * 4);
  m.padded /= nblk;
  m.useful /= nblk;
  return m;
}

template <int MODE, int SYNC = 0>
static void run(const char* name, int chunks, int nblk = 8) {
  Meta m = make_meta(MODE, nblk, 0.1, 777);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* mg;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&mg, m.words.size() * sizeof(uint4)));
  CK(cudaMemcpy(mg, m.words.data(), m.words.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 32));
  auto kern = meta_kernel<MODE, SYNC>;
  const size_t smem = m.words.size() * sizeof(uint4) + (MODE >= 4 ? 256 : 0);  // MODE 4/5 windows read up to 31 entries past a stream
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
  const double ent = m.padded * chunks;  // padded entries per CTA
  printf("%-48s regs %3d smem %6zu  padded entries/clk/SM %.4f  = %5.1f FMA/clk/SM (%4.1f %% of 128)  ldtm B/clk %5.1f  %7.3f ms\n",
         name, fa.numRegs, smem, ent / double(cmax), ent * 128.0 / double(cmax), ent * 128.0 / double(cmax) / 1.28,
         ent * 512.0 / double(cmax), ms);
  fflush(stdout);
  CK(cudaFree(mg));
  CK(cudaFree(out));
  CK(cudaFree(cyc));
}

int main(int argc, char** argv) {
  const int chunks = argc > 1 ? atoi(argv[1]) : 2048;
  for (int rep = 0; rep < 2; ++rep) {
    run<0>("MODE 0 LDS.128 {c,w,c,w} /2 (product)", chunks);
    run<1>("MODE 1 LDS.128 {c0..c3} /4, const w", chunks);
    run<2>("MODE 2 LDS.128 {w0..w3} + LDS.64 16-bit cols /4", chunks);
    run<4>("MODE 4 lane-distributed LDS.64 /32, REDUX col + w", chunks);
    run<5>("MODE 5 REDUX col, LDS.128 {w0..w3} /4", chunks);
    run<0, 0>("MODE 0, 12 distinct blocks, no sync", chunks, 12);
    run<0, 1>("MODE 0, 12 distinct blocks, barrier every chunk", chunks, 12);
    run<0, 2>("MODE 0, 12 distinct blocks, barrier every 2 chunks", chunks, 12);
  }
  return 0;
}
