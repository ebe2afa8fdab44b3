// sdnn_codegen.cpp — the per-matrix sparse code generator (§3.2.2), B200 form.
//
// The paper generates, for each sparse weight, x86 code whose register names statically encode the
// accumulation position and whose value order follows the traversal, and emits the
// assembly itself to bypass the compiler.  Here the preparation stage emits PTX, one kernel
// per row panel of R rows, and JIT-compiles it for sm_100a:
//   * each lane owns one column n of Y; the R accumulators of the panel are registers a<r>;
//   * for every column k of the panel's union, in ascending order, the lane loads X[k][n] (issued
//     D columns ahead, straight from L2: no reuse inside the SM to stage for) and issues one
//     `fma.rn.f32 a<r>, x, <w as immediate>, a<r>` per nonzero (r, k) — SASS `FFMA R, R, imm, R`,
//     full rate (128/clk/SM, profiles/r01_microbench.log);
//   * epilogue: + bias[orig row], ReLU, store to the ORIGINAL row (row ids are immediates);
//   * CTAs are persistent: each panel kernel gets a few CTAs that sweep the N tiles in the same
//     order as every other panel's CTAs, and all panel kernels run concurrently (one stream each),
//     so the X tile being read is shared in L2 by all panels (X is read from HBM ~once).
// Measured design point (tools/proto_codegen.py + tools/microbench/run_cg.cu): the
// kernel is instruction-fetch bound (≈1.5 instructions/clk/SM for streaming code); FFMA-immediate
// code with R ≈ 128 keeps X traffic at 4 B per R/10 FMAs, well under the L2 bandwidth.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sdnn_internal.h"

namespace sdnn {

static void appendf(std::string& s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static void appendf(std::string& s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  const int n = vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (n < int(sizeof buf)) {
    s.append(buf, size_t(n));
  } else {
    std::string big(size_t(n) + 1, '\0');
    va_start(ap, fmt);
    vsnprintf(&big[0], big.size(), fmt, ap);
    va_end(ap);
    s.append(big.data(), size_t(n));
  }
}

const DriverApi& driver() {
  static DriverApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
    };
    bool ok = true;
    ok &= get("cuModuleLoadDataEx", reinterpret_cast<void**>(&api.moduleLoadDataEx));
    ok &= get("cuModuleGetFunction", reinterpret_cast<void**>(&api.moduleGetFunction));
    ok &= get("cuModuleUnload", reinterpret_cast<void**>(&api.moduleUnload));
    ok &= get("cuLaunchKernel", reinterpret_cast<void**>(&api.launchKernel));
    ok &= get("cuGetErrorString", reinterpret_cast<void**>(&api.getErrorString));
    ok &= get("cuCtxGetCurrent", reinterpret_cast<void**>(&api.ctxGetCurrent));
    ok &= get("cuCtxSetCurrent", reinterpret_cast<void**>(&api.ctxSetCurrent));
    api.ok = ok;
  });
  return api;
}

static uint32_t f32_bits(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  return u;
}

// PTX for one panel.  rows[i] = original row id of accumulator i (−1 never occurs here).
std::string codegen_panel_ptx(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals,
                              const std::vector<int32_t>& rows, int32_t K, int32_t warps, int32_t D,
                              const std::string& name) {
  const int32_t R = int32_t(rows.size());
  // union columns with their (accumulator, weight) lists, ascending column order
  std::vector<int32_t> cnt(K, 0);
  for (int32_t i = 0; i < R; ++i)
    for (int32_t p = csr_ptr[rows[i]]; p < csr_ptr[rows[i] + 1]; ++p) cnt[col_idx[p]]++;
  std::vector<int32_t> start(K + 1, 0);
  for (int32_t c = 0; c < K; ++c) start[c + 1] = start[c] + cnt[c];
  std::vector<int32_t> acc_of(start[K]);
  std::vector<float> w_of(start[K]);
  {
    std::vector<int32_t> fill(start.begin(), start.end() - 1);
    for (int32_t i = 0; i < R; ++i)
      for (int32_t p = csr_ptr[rows[i]]; p < csr_ptr[rows[i] + 1]; ++p) {
        const int32_t c = col_idx[p];
        acc_of[fill[c]] = i;
        w_of[fill[c]] = vals[p];
        fill[c]++;
      }
  }
  std::vector<int32_t> ucols;
  for (int32_t c = 0; c < K; ++c)
    if (cnt[c]) ucols.push_back(c);
  const int32_t U = int32_t(ucols.size());
  const int32_t Dx = std::max<int32_t>(1, std::min<int32_t>(D, U));
  const int32_t TILE = 32 * warps;

  std::string s;
  s.reserve(size_t(start[K]) * 48 + size_t(U) * 96 + size_t(R) * 160 + 4096);
  s += ".version 8.8\n.target sm_100a\n.address_size 64\n\n";
  appendf(s,
          ".visible .entry %s(.param .u64 pX, .param .u64 pY, .param .u64 pB, .param .u32 ldx4, .param .u32 ldy4,"
          " .param .u32 N, .param .u32 act, .param .u32 ntiles)\n",
          name.c_str());
  appendf(s, ".maxntid %d, 1, 1\n.minnctapersm %d\n{\n", TILE, TILE <= 192 ? 2 : 1);
  appendf(s, "  .reg .f32 a<%d>; .reg .f32 x<%d>; .reg .f32 v, b;\n", std::max(R, 1), Dx);
  s += "  .reg .b64 px0, px, py0, py, pb, pc, t64;\n  .reg .b32 r<16>;\n  .reg .pred p<8>;\n";
  s += "  ld.param.u64 px0, [pX]; ld.param.u64 py0, [pY]; ld.param.u64 pb, [pB];\n";
  s += "  ld.param.u32 r0, [ldx4]; ld.param.u32 r1, [ldy4]; ld.param.u32 r2, [N]; ld.param.u32 r3, [act];\n";
  s += "  ld.param.u32 r4, [ntiles];\n";
  s += "  setp.ne.u64 p2, pb, 0; setp.eq.u32 p3, r3, 1;\n";  // p2: has bias, p3: relu
  s += "  mov.u32 r5, %ctaid.x; mov.u32 r6, %nctaid.x; mov.u32 r7, %tid.x; sub.u32 r9, r2, 1;\n";
  s += "TILE:\n  setp.ge.u32 p0, r5, r4; @p0 bra DONE;\n";
  appendf(s, "  mad.lo.u32 r8, r5, %d, r7;\n", TILE);       // n
  s += "  min.u32 r10, r8, r9;\n";                          // clamped column for loads
  s += "  mul.wide.u32 t64, r10, 4; add.u64 px, px0, t64;\n";
  for (int32_t i = 0; i < R; ++i) appendf(s, "  mov.f32 a%d, 0f00000000;\n", i);
  auto load = [&](int32_t u, int32_t reg) {
    appendf(s, "  mad.wide.u32 pc, r0, %d, px; ld.global.nc.L1::no_allocate.f32 x%d, [pc];\n", ucols[u], reg);
  };
  for (int32_t u = 0; u < std::min(Dx, U); ++u) load(u, u);
  for (int32_t u = 0; u < U; ++u) {
    const int32_t c = ucols[u], xr = u % Dx;
    for (int32_t q = start[c]; q < start[c + 1]; ++q)
      appendf(s, "  fma.rn.f32 a%d, x%d, 0f%08X, a%d;\n", acc_of[q], xr, f32_bits(w_of[q]), acc_of[q]);
    if (u + Dx < U) load(u + Dx, xr);
  }
  // epilogue: y = a + b[orig]; ReLU (v > 0 ? v : 0); store to Y[orig][n] if n < N
  s += "  setp.ge.u32 p1, r8, r2; @p1 bra NEXT;\n";
  s += "  mul.wide.u32 t64, r8, 4; add.u64 py, py0, t64;\n";
  for (int32_t i = 0; i < R; ++i) {
    const int32_t o = rows[i];
    appendf(s, "  mov.f32 v, a%d; @p2 ld.global.nc.f32 b, [pb+%lld]; @p2 add.f32 v, v, b;\n", i, (long long)o * 4);
    s += "  setp.gt.f32 p4, v, 0f00000000; @p3 selp.f32 v, v, 0f00000000, p4;\n";
    appendf(s, "  mad.wide.u32 pc, r1, %d, py; st.global.f32 [pc], v;\n", o);
  }
  s += "NEXT:\n  add.u32 r5, r5, r6; bra TILE;\nDONE:\n  ret;\n}\n";
  return s;
}

// JIT one module (driver API, ptxas optimisation level 1: streaming straight-line code gains
// nothing from -O3 scheduling and -O3 spills the accumulators).
static CUresult jit_module(const std::string& ptx, CUmodule* mod, std::string* log) {
  char err[4096] = {0};
  CUjit_option opts[] = {CU_JIT_OPTIMIZATION_LEVEL, CU_JIT_ERROR_LOG_BUFFER, CU_JIT_ERROR_LOG_BUFFER_SIZE_BYTES};
  void* vals[] = {reinterpret_cast<void*>(uintptr_t(1)), err, reinterpret_cast<void*>(uintptr_t(sizeof err))};
  CUresult r = driver().moduleLoadDataEx(mod, ptx.c_str(), 3, opts, vals);
  if (r != CUDA_SUCCESS && log) *log = err;
  return r;
}

sdnn_status codegen_build(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t K,
                          const std::vector<std::vector<int32_t>>& panels, int32_t warps, int32_t D,
                          std::vector<CUmodule>& mods, std::vector<CUfunction>& funcs, int32_t threads) {
  const size_t P = panels.size();
  mods.assign(P, nullptr);
  funcs.assign(P, nullptr);
  const DriverApi& d = driver();
  if (!d.ok) return fail(SDNN_ERR_CUDA, "CUDA driver entry points unavailable");
  CUcontext ctx = nullptr;
  if (d.ctxGetCurrent(&ctx) != CUDA_SUCCESS || !ctx) return fail(SDNN_ERR_CUDA, "no current CUDA context");
  std::vector<CUresult> res(P, CUDA_SUCCESS);
  std::vector<std::string> logs(P);
  const int32_t T = std::max<int32_t>(1, std::min<int32_t>(threads, int32_t(P)));
  std::vector<std::thread> pool;
  for (int32_t t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      d.ctxSetCurrent(ctx);
      for (size_t p = size_t(t); p < P; p += size_t(T)) {
        const std::string name = "sdnn_cg_p" + std::to_string(p);
        const std::string ptx = codegen_panel_ptx(csr_ptr, col_idx, vals, panels[p], K, warps, D, name);
        res[p] = jit_module(ptx, &mods[p], &logs[p]);
        if (res[p] == CUDA_SUCCESS) res[p] = d.moduleGetFunction(&funcs[p], mods[p], name.c_str());
      }
    });
  }
  for (auto& th : pool) th.join();
  for (size_t p = 0; p < P; ++p) {
    if (res[p] != CUDA_SUCCESS) {
      const char* es = nullptr;
      d.getErrorString(res[p], &es);
      for (CUmodule m : mods)
        if (m) d.moduleUnload(m);
      mods.clear();
      funcs.clear();
      return fail(res[p] == CUDA_ERROR_OUT_OF_MEMORY ? SDNN_ERR_OUT_OF_MEMORY : SDNN_ERR_CUDA,
                  "codegen JIT of panel " + std::to_string(p) + " failed: " + (es ? es : "?") + " " + logs[p]);
    }
  }
  return SDNN_OK;
}

}  // namespace sdnn
