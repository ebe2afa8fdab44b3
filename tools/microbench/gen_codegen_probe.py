"""Generate a probe for the per-matrix specialised ("codegen") microkernel idea.

Each variant is straight-line code for one R-row panel over U union columns: per column one
LDS.64 of X (V = 2 floats per lane) and, for each nonzero of that column in the panel, two FFMAs
with the weight as an immediate into statically named accumulators ("statically encoding
the accumulation position in the vector register name").  Warps pick variant = warp % P, so P
distinct instruction streams run concurrently on every SM.  This measures instruction-fetch cost
of nnz-sized code on the B200, which decides whether f1 is viable.
"""
import random
import sys

R, V = 64, 2
U = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
DENS = 0.1
XCOLS = 256  # smem holds 256 columns x 64 floats = 64 KB

rng = random.Random(0)
out = []
out.append("#include <cstdio>\n#include <cuda_runtime.h>\n")
out.append("extern \"C\" __global__ void __launch_bounds__(128, 1) probe(float* out, int iters, long long* clk, int nvar) {")
out.append("  extern __shared__ float2 xs[];")
out.append("  for (int i = threadIdx.x; i < %d * 32; i += blockDim.x) xs[i] = make_float2(i * 1e-3f, 1.f);" % XCOLS)
out.append("  __syncthreads();")
out.append("  int lane = threadIdx.x & 31; int var = (threadIdx.x >> 5) % nvar;")
for r in range(R):
    out.append("  float a%d_0 = 0.f, a%d_1 = 0.f;" % (r, r))
out.append("  long long t0 = clock64();")
out.append("  for (int it = 0; it < iters; ++it) {")
nfma = 0
for p in range(P):
    out.append("  %sif (var == %d) {" % ("" if p == 0 else "else ", p))
    for c in range(U):
        rows = [r for r in range(R) if rng.random() < DENS]
        if not rows:
            continue
        out.append("    { float2 x = xs[%d * 32 + lane];" % (c % XCOLS))
        for r in rows:
            w = rng.gauss(0, 0.05)
            out.append("      a%d_0 = fmaf(x.x, %.9ef, a%d_0); a%d_1 = fmaf(x.y, %.9ef, a%d_1);" % (r, w, r, r, w, r))
            if p == 0:
                nfma += 2
        out.append("    }")
    out.append("  }")
out.append("  }")
out.append("  long long t1 = clock64();")
out.append("  float s = 0.f;")
for r in range(R):
    out.append("  s += a%d_0 + a%d_1;" % (r, r))
out.append("  if (s == 12345.f) out[0] = s;")
out.append("  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;")
out.append("}")
out.append("""
int main(int argc, char** argv) {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int SM = p.multiProcessorCount;
  float* o; long long* clk; cudaMalloc(&o, 64); cudaMalloc(&clk, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, %d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double fma_per_thread_iter = %d.0;
  for (int nvar = 1; nvar <= %d; nvar *= 2) {
    for (int threads : {128}) {
      int blocks = SM; int iters = 20;
      probe<<<blocks, threads, %d>>>(o, 2, clk, nvar);
      cudaDeviceSynchronize();
      cudaEventRecord(e0); probe<<<blocks, threads, %d>>>(o, iters, clk, nvar); cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      double fmas = fma_per_thread_iter * iters * threads * blocks;
      printf("codegen probe U=%d R=%d nvar=%%d threads=%%d: %%.3f ms  %%.2f TFLOP/s  per-SM FMA/clk %%.1f  (err %%s)\\n",
             nvar, threads, ms, 2 * fmas / (ms * 1e-3) / 1e12, fma_per_thread_iter * iters * threads / c,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
""" % (XCOLS * 256, nfma, P, XCOLS * 256, XCOLS * 256, U, R))
open(sys.argv[3] if len(sys.argv) > 3 else "codegen_probe.cu", "w").write("\n".join(out))
print("fma per thread per iter:", nfma)
