// Mixed operand path microbenchmark (round-2 question: is shared memory a second,
// independent operand path next to tensor memory?).  The TMEM-R consumer loop of the bench kernel
//   LDS.128 (col, w, col, w) -> R2UR -> tcgen05.ld.32x32b.x4 -> wait -> FFMA2
// runs on NT warps while NS other warps run the same loop with the X operand read from a 32 KB
// shared-memory tile instead (LDS.128 of the lane's 4 columns of X row k; the metadata column field
// is then the byte offset 512·k).  No fill, no TMA: the consumers' ceiling only.  Shared-memory warps
// get `fs` × the chunks of the TMEM warps so that both kinds run concurrently for most of the time.
// usage: mixed [chunks]
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
__device__ __forceinline__ void tld4(uint32_t a, float (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
}
__device__ __forceinline__ void fma4(float2 (&acc)[2], float w, const float (&x)[4]) {
  const float2 w2 = make_float2(w, w);
  acc[0] = __ffma2_rn(w2, make_float2(x[0], x[1]), acc[0]);
  acc[1] = __ffma2_rn(w2, make_float2(x[2], x[3]), acc[1]);
}
__device__ __forceinline__ void fma4(float2 (&acc)[2], float w, const float4 x) {
  const float2 w2 = make_float2(w, w);
  acc[0] = __ffma2_rn(w2, make_float2(x.x, x.y), acc[0]);
  acc[1] = __ffma2_rn(w2, make_float2(x.z, x.w), acc[1]);
}

// metadata block per chunk: per warp 16 header words ([0] stream start in float4, [1..RW] pairs per
// row), then entry pairs {col, w, col, w}
template <int RW, int NT, int NS, int NFW>
__global__ void __launch_bounds__((NT + NS + NFW) * 32, 1)
    mixed_kernel(const uint4* __restrict__ meta_g, int blk_u4, int nblk, int chunks_t, int chunks_s, float* out,
                 long long* cyc) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* ms = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < blk_u4 * nblk; i += blockDim.x) ms[i] = meta_g[i];
  float4* tile = reinterpret_cast<float4*>(smem + size_t(blk_u4) * nblk * 16);
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
  if (warp < NT + NS) {
    const bool sw = warp >= NT;
    const int chunks = sw ? chunks_s : chunks_t;
    float2 acc[RW][2];
#pragma unroll
    for (int r = 0; r < RW; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
    const char* xl = reinterpret_cast<const char*>(tile) + 16 * lane;
    for (int j = 0; j < chunks; ++j) {
      const uint4* blk = ms + size_t(j % nblk) * blk_u4;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(blk) + warp * 16;
      const float4* e = reinterpret_cast<const float4*>(blk) + __shfl_sync(0xffffffffu, hdr[0], 0);
      if (!sw) {
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          int n = __shfl_sync(0xffffffffu, int(hdr[1 + r]), 0);
          for (; n >= 2; n -= 2, e += 2) {
            const float4 f0 = e[0], f1 = e[1];
            float x0[4], x1[4], x2[4], x3[4];
            tld4(__float_as_uint(f0.x), x0);
            tld4(__float_as_uint(f0.z), x1);
            tld4(__float_as_uint(f1.x), x2);
            tld4(__float_as_uint(f1.z), x3);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 4; ++i) asm volatile("" : "+f"(x0[i]), "+f"(x1[i]), "+f"(x2[i]), "+f"(x3[i]));
            fma4(acc[r], f0.y, x0);
            fma4(acc[r], f0.w, x1);
            fma4(acc[r], f1.y, x2);
            fma4(acc[r], f1.w, x3);
          }
          if (n) {
            const float4 f0 = e[0];
            float x0[4], x1[4];
            tld4(__float_as_uint(f0.x), x0);
            tld4(__float_as_uint(f0.z), x1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 4; ++i) asm volatile("" : "+f"(x0[i]), "+f"(x1[i]));
            fma4(acc[r], f0.y, x0);
            fma4(acc[r], f0.w, x1);
            ++e;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          int n = __shfl_sync(0xffffffffu, int(hdr[1 + r]), 0);
          for (; n >= 2; n -= 2, e += 2) {
            const float4 f0 = e[0], f1 = e[1];
            const float4 x0 = *reinterpret_cast<const float4*>(xl + __float_as_uint(f0.x));
            const float4 x1 = *reinterpret_cast<const float4*>(xl + __float_as_uint(f0.z));
            const float4 x2 = *reinterpret_cast<const float4*>(xl + __float_as_uint(f1.x));
            const float4 x3 = *reinterpret_cast<const float4*>(xl + __float_as_uint(f1.z));
            fma4(acc[r], f0.y, x0);
            fma4(acc[r], f0.w, x1);
            fma4(acc[r], f1.y, x2);
            fma4(acc[r], f1.w, x3);
          }
          if (n) {
            const float4 f0 = e[0];
            const float4 x0 = *reinterpret_cast<const float4*>(xl + __float_as_uint(f0.x));
            const float4 x1 = *reinterpret_cast<const float4*>(xl + __float_as_uint(f0.z));
            fma4(acc[r], f0.y, x0);
            fma4(acc[r], f0.w, x1);
            ++e;
          }
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
  if (lane == 0) cyc[blockIdx.x * 64 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

struct Meta {
  std::vector<uint4> words;
  int blk_u4 = 0;
  double nz_t = 0, nz_s = 0;  // useful nonzeros per block, TMEM warps / smem warps
};
static Meta make_meta(int RW, int NT, int NS, int nblk, double density, unsigned seed) {
  const int KC = 64;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  std::vector<std::vector<uint32_t>> blocks;
  int maxw = 0;
  Meta m;
  const int NW = NT + NS;
  for (int b = 0; b < nblk; ++b) {
    std::vector<uint32_t> w(size_t(NW) * 16, 0u);
    for (int wp = 0; wp < NW; ++wp) {
      const bool sw = wp >= NT;
      const uint32_t lb = uint32_t((wp & 3) * 32) << 16;
      w[wp * 16] = uint32_t(w.size() / 4);
      for (int r = 0; r < RW; ++r) {
        std::vector<int> cols;
        for (int k = 0; k < KC; ++k)
          if (uni(rng) < density) cols.push_back(k);
        (sw ? m.nz_s : m.nz_t) += double(cols.size());
        const int pairs = int((cols.size() + 1) / 2);
        w[wp * 16 + 1 + r] = uint32_t(pairs);
        for (int s = 0; s < pairs * 2; ++s) {
          const bool real = s < int(cols.size());
          const int k = real ? cols[s] : (cols.empty() ? 0 : cols.back());
          const float wv = real ? 0.01f * float(1 + (s % 7)) : 0.f;
          uint32_t wb;
          memcpy(&wb, &wv, 4);
          w.push_back(sw ? uint32_t(512 * k) : (lb | uint32_t(4 * k + 256 * (b & 1))));
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
  m.nz_t /= nblk;
  m.nz_s /= nblk;
  return m;
}

template <int RW, int NT, int NS, int NFW>
static void run(const char* name, int chunks, double fs) {
  const int nblk = 8;
  Meta m = make_meta(RW, NT, NS, nblk, 0.1, 777);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* mg;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&mg, m.words.size() * sizeof(uint4)));
  CK(cudaMemcpy(mg, m.words.data(), m.words.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, sizeof(float) * sms * 2048));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 64));
  CK(cudaMemset(cyc, 0, sizeof(long long) * sms * 64));
  auto kern = mixed_kernel<RW, NT, NS, NFW>;
  const size_t smem = m.words.size() * sizeof(uint4) + 32768;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  const int ct = chunks, cs = int(chunks * fs + 0.5);
  const int threads = (NT + NS + NFW) * 32;
  kern<<<sms, threads, smem>>>(mg, m.blk_u4, nblk, 4, 4, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, threads, smem>>>(mg, m.blk_u4, nblk, ct, cs, out, cyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(size_t(sms) * 64);
  CK(cudaMemcpy(c.data(), cyc, c.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  long long ct_max = 0, cs_max = 0;
  for (int w = 0; w < NT; ++w) ct_max = std::max(ct_max, c[w]);
  for (int w = NT; w < NT + NS; ++w) cs_max = std::max(cs_max, c[w]);
  // useful FMAs per CTA: nonzeros × 128 columns
  const double fma_t = m.nz_t * 128.0 * ct, fma_s = m.nz_s * 128.0 * cs;
  const double cmax = double(std::max(ct_max, cs_max));
  const double tflops = 2.0 * (fma_t + fma_s) * sms / (ms * 1e-3) / 1e12;
  printf("%-26s fs %.2f regs %3d  FMA/clk/SM total %6.1f (%5.1f %%)  tmem-warps %6.1f smem-warps %6.1f  cyc t %lld s %lld  %7.3f ms %6.2f TF\n",
         name, fs, fa.numRegs, (fma_t + fma_s) / cmax, (fma_t + fma_s) / cmax / 128.0 * 100.0,
         ct_max ? fma_t / double(ct_max) : 0.0, cs_max ? fma_s / double(cs_max) : 0.0, ct_max, cs_max, ms, tflops);
  fflush(stdout);
  CK(cudaFree(mg));
  CK(cudaFree(out));
  CK(cudaFree(cyc));
}

int main(int argc, char** argv) {
  const int chunks = argc > 1 ? atoi(argv[1]) : 2048;
  run<10, 24, 0, 4>("T24 S0", chunks, 0.0);
  run<10, 0, 24, 4>("T0 S24", chunks, 1.0);
  for (double fs : {0.3, 0.5, 0.7, 1.0}) run<10, 20, 4, 4>("T20 S4", chunks, fs);
  for (double fs : {0.3, 0.5, 0.7, 1.0}) run<10, 18, 6, 4>("T18 S6", chunks, fs);
  for (double fs : {0.3, 0.5, 0.7}) run<10, 16, 8, 4>("T16 S8", chunks, fs);
  for (double fs : {0.3, 0.5, 0.7}) run<10, 24, 4, 0>("T24 S4 (28 warps)", chunks, fs);
  for (double fs : {0.3, 0.5, 0.7}) run<10, 24, 8, 0>("T24 S8 (32 warps)", chunks, fs);
  return 0;
}
