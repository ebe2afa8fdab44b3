// sdnn_prepare.cpp — host side of the preparation stage (§2.1, §3):
// CSR validation, Algorithm 1 weight permutation (§3.1.2), and packing into the
// execution-ordered format the kernel reads sequentially (§3.2.2).  No CUDA here; the
// upload lives in sdnn_spmm.cu.  Independent of oracle/ (shares no code with it).
#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "sdnn_internal.h"

namespace sdnn {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
sdnn_status fail(sdnn_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

sdnn_status validate_csr(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K) {
  if (M < 1 || K < 1) return fail(SDNN_ERR_INVALID_ARGUMENT, "M and K must be >= 1");
  if (!csr_ptr) return fail(SDNN_ERR_INVALID_ARGUMENT, "csr_ptr is NULL");
  if (csr_ptr[0] != 0) return fail(SDNN_ERR_INVALID_CSR, "csr_ptr[0] != 0");
  for (int32_t m = 0; m < M; ++m)
    if (csr_ptr[m + 1] < csr_ptr[m])
      return fail(SDNN_ERR_INVALID_CSR, "csr_ptr decreases at row " + std::to_string(m));
  const int64_t nnz = csr_ptr[M];
  if (nnz > 0 && !col_idx) return fail(SDNN_ERR_INVALID_ARGUMENT, "col_idx is NULL with nnz > 0");
  for (int32_t m = 0; m < M; ++m) {
    int32_t prev = -1;
    for (int32_t p = csr_ptr[m]; p < csr_ptr[m + 1]; ++p) {
      const int32_t c = col_idx[p];
      if (c < 0 || c >= K)
        return fail(SDNN_ERR_INVALID_CSR, "column index out of range in row " + std::to_string(m));
      if (c <= prev)
        return fail(SDNN_ERR_INVALID_CSR,
                    "columns not strictly increasing (unsorted or duplicate) in row " + std::to_string(m));
      prev = c;
    }
  }
  return SDNN_OK;
}

// Algorithm 1.  line 4: the first row is the one with most nonzeros; line 8: each next
// row maximises |nnz(B[i-1]) ∩ nnz(A[x])| over the remaining rows.  Ties → lowest original index
// (readings C2/C3).  Inverted index: per step, every row sharing a column with the previous row gets
// +1 per shared column, then one argmax scan over the remaining rows — O(Σ_c colnnz(c)^2 + M^2).
void algorithm1(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K, int32_t* order) {
  std::vector<int32_t> col_ptr(K + 1, 0), col_rows(csr_ptr[M]);
  for (int32_t p = 0; p < csr_ptr[M]; ++p) col_ptr[col_idx[p] + 1]++;
  for (int32_t c = 0; c < K; ++c) col_ptr[c + 1] += col_ptr[c];
  {
    std::vector<int32_t> fill(col_ptr.begin(), col_ptr.end() - 1);
    for (int32_t m = 0; m < M; ++m)
      for (int32_t p = csr_ptr[m]; p < csr_ptr[m + 1]; ++p) col_rows[fill[col_idx[p]]++] = m;
  }
  std::vector<uint8_t> rem(M, 1);
  std::vector<int32_t> cnt(M, 0);
  int32_t row = 0;
  for (int32_t x = 1; x < M; ++x)
    if (csr_ptr[x + 1] - csr_ptr[x] > csr_ptr[row + 1] - csr_ptr[row]) row = x;
  order[0] = row;
  rem[row] = 0;
  for (int32_t i = 1; i < M; ++i) {
    const int32_t prev = order[i - 1];
    for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) {
      const int32_t c = col_idx[p];
      for (int32_t q = col_ptr[c]; q < col_ptr[c + 1]; ++q) cnt[col_rows[q]]++;
    }
    int32_t best = -1, arg = -1;
    for (int32_t x = 0; x < M; ++x)
      if (rem[x] && cnt[x] > best) { best = cnt[x]; arg = x; }
    for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) {
      const int32_t c = col_idx[p];
      for (int32_t q = col_ptr[c]; q < col_ptr[c + 1]; ++q) cnt[col_rows[q]] = 0;
    }
    order[i] = arg;
    rem[arg] = 0;
  }
}

// Bytes of the (row block, chunk) metadata block for a given KC, over all blocks; returns max.
static int64_t max_block_bytes_for(const int32_t* csr_ptr, const int32_t* col_idx, const std::vector<int32_t>& perm,
                                   int32_t M, int32_t K, int32_t rcta, int32_t kc) {
  const int32_t nch = (K + kc - 1) / kc;
  const int64_t hdr = align_up(int64_t(rcta) * 4, 16);
  std::vector<int64_t> ent(nch);
  int64_t mx = hdr;
  for (int32_t b0 = 0; b0 < M; b0 += rcta) {
    std::fill(ent.begin(), ent.end(), 0);
    for (int32_t s = 0; s < rcta && b0 + s < M; ++s) {
      const int32_t r = perm[b0 + s];
      int32_t cur = -1, c_in = 0;
      for (int32_t p = csr_ptr[r]; p < csr_ptr[r + 1]; ++p) {
        const int32_t j = col_idx[p] / kc;
        if (j != cur) {
          if (cur >= 0) ent[cur] += align_up(c_in, 2);
          cur = j;
          c_in = 0;
        }
        ++c_in;
      }
      if (cur >= 0) ent[cur] += align_up(c_in, 2);
    }
    for (int32_t j = 0; j < nch; ++j) mx = std::max(mx, hdr + ent[j] * 8);
  }
  return align_up(mx, 16);
}

sdnn_status build_plan(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                       const sdnn_perm_opts* opts, Plan& plan) {
  sdnn_perm_opts o{};
  o.struct_size = sizeof(o);
  o.permute = 1;
  if (opts) {
    if (opts->struct_size != sizeof(sdnn_perm_opts))
      return fail(SDNN_ERR_INVALID_ARGUMENT, "sdnn_perm_opts.struct_size mismatch");
    o = *opts;
    if (o.flags != 0) return fail(SDNN_ERR_INVALID_ARGUMENT, "sdnn_perm_opts.flags must be 0");
    if (o.permute != 0 && o.permute != 1) return fail(SDNN_ERR_INVALID_ARGUMENT, "permute must be 0 or 1");
    if (o.panel_rows_max != 0 && o.panel_rows_max != 4 && o.panel_rows_max != 8)
      return fail(SDNN_ERR_INVALID_ARGUMENT, "panel_rows_max must be 0, 4 or 8");
    if (o.cta_panels < 0 || o.cta_panels > 16) return fail(SDNN_ERR_INVALID_ARGUMENT, "cta_panels must be 0..16");
    if (o.k_chunk != 0 && (o.k_chunk < 8 || o.k_chunk > 128 || o.k_chunk % 8))
      return fail(SDNN_ERR_INVALID_ARGUMENT, "k_chunk must be 0 or a multiple of 8 in [8, 128]");
  }
  sdnn_status st = validate_csr(csr_ptr, col_idx, M, K);
  if (st != SDNN_OK) return st;
  const int64_t nnz = csr_ptr[M];
  if (nnz > 0 && !vals) return fail(SDNN_ERR_INVALID_ARGUMENT, "vals is NULL with nnz > 0");

  try {
    plan = Plan{};
    plan.M = M;
    plan.K = K;
    plan.nnz = nnz;
    plan.permuted = o.permute;
    plan.perm.resize(M);
    if (o.permute)
      algorithm1(csr_ptr, col_idx, M, K, plan.perm.data());
    else
      for (int32_t i = 0; i < M; ++i) plan.perm[i] = i;

    // Launch geometry: R_w rows per warp panel, W_c panels per CTA.
    const int32_t rw = o.panel_rows_max ? o.panel_rows_max : (M >= 2048 ? 8 : 4);
    int32_t wc = o.cta_panels;
    if (!wc) {
      wc = 16;
      while (wc > 4 && (M + rw * wc - 1) / (rw * wc) < 32) wc /= 2;
    }
    const int32_t rcta = rw * wc;
    plan.panel_rows = rw;
    plan.cta_panels = wc;
    plan.num_row_blocks = (M + rcta - 1) / rcta;
    plan.num_panels = plan.num_row_blocks * wc;

    // K chunk (split-K tiling along the reduction dimension): the largest KC whose stage
    // (X tile at the widest N tile + metadata block) fits three times in the shared-memory budget.
    int32_t kc = o.k_chunk, stages = 0;
    int64_t mb = 0;
    const int32_t cands[] = {64, 32, 16, 8};
    if (kc) {
      mb = max_block_bytes_for(csr_ptr, col_idx, plan.perm, M, K, rcta, kc);
      stages = int32_t(kSmemBudget / (int64_t(kc) * kMaxTN * 4 + align_up(mb, 128)));
      if (stages < 2) return fail(SDNN_ERR_UNSUPPORTED, "k_chunk too large for the shared-memory budget");
    } else {
      for (int32_t c : cands) {
        const int64_t m = max_block_bytes_for(csr_ptr, col_idx, plan.perm, M, K, rcta, c);
        const int32_t s = int32_t(kSmemBudget / (int64_t(c) * kMaxTN * 4 + align_up(m, 128)));
        if (s >= 3 || (c == 8 && s >= 2)) { kc = c; mb = m; stages = s; break; }
      }
      if (!kc) return fail(SDNN_ERR_UNSUPPORTED, "no K chunk fits the shared-memory budget");
    }
    (void)stages;
    plan.k_chunk = kc;
    plan.num_chunks = (K + kc - 1) / kc;
    plan.max_block_bytes = int32_t(mb);

    // row_orig
    plan.row_orig.assign(size_t(plan.num_panels) * rw, -1);
    for (int32_t p = 0; p < M; ++p) plan.row_orig[p] = plan.perm[p];
    for (int32_t pn = 0; pn < plan.num_panels; ++pn) {
      int64_t s = 0;
      for (int32_t r = 0; r < rw; ++r) {
        const int32_t orow = plan.row_orig[size_t(pn) * rw + r];
        if (orow >= 0) s += csr_ptr[orow + 1] - csr_ptr[orow];
      }
      plan.max_panel_nnz = std::max(plan.max_panel_nnz, s);
    }

    // Execution-ordered metadata: blocks ordered [row block][chunk], rows in slot order,
    // each row's entries in ascending column order (the order the kernel accumulates them).
    const int32_t nch = plan.num_chunks;
    const int64_t hdr = align_up(int64_t(rcta) * 4, 16);
    plan.blk_off.assign(size_t(plan.num_row_blocks) * nch + 1, 0);
    // first pass: sizes
    std::vector<int32_t> rowpos(rcta);
    std::vector<std::vector<int32_t>> seg_cnt(rcta, std::vector<int32_t>(nch));
    int64_t total = 0;
    std::vector<int64_t> sizes(size_t(plan.num_row_blocks) * nch);
    for (int32_t b = 0; b < plan.num_row_blocks; ++b) {
      std::vector<int64_t> ent(nch, 0);
      for (int32_t s = 0; s < rcta; ++s) {
        const int32_t orow = plan.row_orig[size_t(b) * rcta + s];
        if (orow < 0) continue;
        std::vector<int32_t> c_in(nch, 0);
        for (int32_t p = csr_ptr[orow]; p < csr_ptr[orow + 1]; ++p) c_in[col_idx[p] / kc]++;
        for (int32_t j = 0; j < nch; ++j) ent[j] += align_up(c_in[j], 2);
      }
      for (int32_t j = 0; j < nch; ++j) {
        sizes[size_t(b) * nch + j] = align_up(hdr + ent[j] * 8, 16);
        total += sizes[size_t(b) * nch + j];
      }
    }
    for (size_t i = 0; i < sizes.size(); ++i) plan.blk_off[i + 1] = plan.blk_off[i] + sizes[i];
    plan.meta.assign(size_t(total), 0);
    // second pass: fill
    for (int32_t b = 0; b < plan.num_row_blocks; ++b) {
      for (int32_t s = 0; s < rcta; ++s) {
        const int32_t orow = plan.row_orig[size_t(b) * rcta + s];
        rowpos[s] = orow >= 0 ? csr_ptr[orow] : 0;
      }
      for (int32_t j = 0; j < nch; ++j) {
        uint8_t* blk = plan.meta.data() + plan.blk_off[size_t(b) * nch + j];
        uint32_t* h = reinterpret_cast<uint32_t*>(blk);
        uint8_t* ent = blk + hdr;
        int32_t e = 0;
        const int32_t lim = (j + 1) * kc;
        for (int32_t s = 0; s < rcta; ++s) {
          const int32_t orow = plan.row_orig[size_t(b) * rcta + s];
          int32_t c = 0;
          if (orow >= 0) {
            int32_t& p = rowpos[s];
            while (p < csr_ptr[orow + 1] && col_idx[p] < lim) {
              const uint32_t cl = uint32_t(col_idx[p] - j * kc);
              std::memcpy(ent + size_t(e + c) * 8, &cl, 4);
              std::memcpy(ent + size_t(e + c) * 8 + 4, &vals[p], 4);
              ++c;
              ++p;
            }
          }
          h[s] = (uint32_t(e) << 16) | uint32_t(c);
          e += int32_t(align_up(c, 2));
        }
      }
    }
  } catch (const std::bad_alloc&) {
    return fail(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed during planning");
  }
  return SDNN_OK;
}

}  // namespace sdnn

using namespace sdnn;

struct sdnn_plan_s {
  Plan plan;
};

static void fill_info(const Plan& p, int32_t device, sdnn_info* info) {
  info->M = p.M;
  info->K = p.K;
  info->nnz = p.nnz;
  info->device = device;
  info->permuted = p.permuted;
  info->panel_rows = p.panel_rows;
  info->cta_panels = p.cta_panels;
  info->num_panels = p.num_panels;
  info->num_row_blocks = p.num_row_blocks;
  info->k_chunk = p.k_chunk;
  info->num_chunks = p.num_chunks;
  info->meta_bytes = int64_t(p.meta.size());
  info->max_block_bytes = p.max_block_bytes;
  info->reserved0 = 0;
  info->max_panel_nnz = p.max_panel_nnz;
}

namespace sdnn {
void plan_fill_info(const Plan& p, int32_t device, sdnn_info* info) { fill_info(p, device, info); }
}  // namespace sdnn

extern "C" {

const char* sdnn_status_string(sdnn_status s) {
  switch (s) {
    case SDNN_OK: return "SDNN_OK";
    case SDNN_ERR_INVALID_ARGUMENT: return "SDNN_ERR_INVALID_ARGUMENT";
    case SDNN_ERR_INVALID_CSR: return "SDNN_ERR_INVALID_CSR";
    case SDNN_ERR_UNSUPPORTED: return "SDNN_ERR_UNSUPPORTED";
    case SDNN_ERR_OUT_OF_MEMORY: return "SDNN_ERR_OUT_OF_MEMORY";
    case SDNN_ERR_CUDA: return "SDNN_ERR_CUDA";
    case SDNN_ERR_DEVICE_MISMATCH: return "SDNN_ERR_DEVICE_MISMATCH";
    case SDNN_ERR_INTERNAL: return "SDNN_ERR_INTERNAL";
  }
  return "SDNN_UNKNOWN_STATUS";
}

const char* sdnn_last_error_message(void) { return g_err.c_str(); }
int32_t sdnn_abi_version(void) { return SDNN_ABI_VERSION; }

sdnn_status sdnn_permutation(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K, int32_t* order) {
  if (!order) return fail(SDNN_ERR_INVALID_ARGUMENT, "order is NULL");
  sdnn_status st = validate_csr(csr_ptr, col_idx, M, K);
  if (st != SDNN_OK) return st;
  try {
    algorithm1(csr_ptr, col_idx, M, K, order);
  } catch (const std::bad_alloc&) {
    return fail(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed");
  }
  return SDNN_OK;
}

sdnn_status sdnn_plan_create(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                             const sdnn_perm_opts* perm_opts, sdnn_plan* out) {
  if (!out) return fail(SDNN_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  sdnn_plan p = new (std::nothrow) sdnn_plan_s;
  if (!p) return fail(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed");
  sdnn_status st = build_plan(csr_ptr, col_idx, vals, M, K, perm_opts, p->plan);
  if (st != SDNN_OK) {
    delete p;
    return st;
  }
  *out = p;
  return SDNN_OK;
}

sdnn_status sdnn_plan_get_info(sdnn_plan p, sdnn_info* info) {
  if (!p || !info) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL plan or info");
  if (info->struct_size != sizeof(sdnn_info)) return fail(SDNN_ERR_INVALID_ARGUMENT, "sdnn_info.struct_size mismatch");
  fill_info(p->plan, -1, info);
  return SDNN_OK;
}

sdnn_status sdnn_plan_export(sdnn_plan p, int32_t* row_orig, int64_t* blk_off, uint8_t* meta) {
  if (!p) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL plan");
  const Plan& pl = p->plan;
  if (row_orig) std::memcpy(row_orig, pl.row_orig.data(), pl.row_orig.size() * 4);
  if (blk_off) std::memcpy(blk_off, pl.blk_off.data(), pl.blk_off.size() * 8);
  if (meta && !pl.meta.empty()) std::memcpy(meta, pl.meta.data(), pl.meta.size());
  return SDNN_OK;
}

sdnn_status sdnn_plan_destroy(sdnn_plan p) {
  delete p;
  return SDNN_OK;
}

}  // extern "C"
