// sdnn_prepare.cpp — host side of the preparation stage (§2.1, §3):
// CSR validation, Algorithm 1 weight permutation (§3.1.2), and packing into the
// execution-ordered format the kernel reads sequentially (§3.2.2).  No CUDA here; the
// upload lives in sdnn_spmm.cu.  Independent of oracle/ (shares no code with it).
#include <algorithm>
#include <array>
#include <cstdlib>
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
// +1 per shared column.  Two ways to take the argmax, chosen per step by the number T of list entries
// the previous row's columns hold (both give the argmax scan's order, row for row):
//  * T ≥ M/2 (dense patterns, c5): plain increment / reset loops and one scan over the remaining rows;
//  * T < M/2 (tall sparse matrices): only the touched rows can have a positive overlap, so the argmax
//    runs over them (lowest index among equals) and, when no remaining row is touched, the answer is the
//    lowest remaining index (a moving pointer) — no M² term: 100 000 rows of ~4 nonzeros take 5 s
//    instead of 33 s.
// Placed rows leave the column lists when a list is walked in the second mode, and everywhere each time
// the number of remaining rows has halved (O(nnz·log M) in total).
void algorithm1(const int32_t* csr_ptr, const int32_t* col_idx, int32_t M, int32_t K, int32_t* order) {
  std::vector<int32_t> col_ptr(K + 1, 0), col_rows(csr_ptr[M]);
  for (int32_t p = 0; p < csr_ptr[M]; ++p) col_ptr[col_idx[p] + 1]++;
  for (int32_t c = 0; c < K; ++c) col_ptr[c + 1] += col_ptr[c];
  std::vector<int32_t> col_end(col_ptr.begin(), col_ptr.end() - 1);  // live end of each column's list
  for (int32_t m = 0; m < M; ++m)
    for (int32_t p = csr_ptr[m]; p < csr_ptr[m + 1]; ++p) col_rows[col_end[col_idx[p]]++] = m;
  std::vector<uint8_t> rem(M, 1);
  std::vector<int32_t> cnt(M, 0);
  int32_t row = 0;
  for (int32_t x = 1; x < M; ++x)
    if (csr_ptr[x + 1] - csr_ptr[x] > csr_ptr[row + 1] - csr_ptr[row]) row = x;
  order[0] = row;
  rem[row] = 0;
  int32_t lo = 0;              // lowest remaining row index
  int32_t next_compact = M / 2;  // remaining rows at which every list is compacted next
  for (int32_t i = 1; i < M; ++i) {
    const int32_t prev = order[i - 1];
    if (M - i <= next_compact && next_compact > 0) {
      for (int32_t c = 0; c < K; ++c) {
        int32_t w = col_ptr[c];
        for (int32_t q = col_ptr[c]; q < col_end[c]; ++q)
          if (rem[col_rows[q]]) col_rows[w++] = col_rows[q];
        col_end[c] = w;
      }
      next_compact /= 2;
    }
    while (!rem[lo]) ++lo;
    int64_t T = 0;
    for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) T += col_end[col_idx[p]] - col_ptr[col_idx[p]];
    int32_t best = -1, arg = -1;
    if (2 * T >= M) {
      for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) {
        const int32_t c = col_idx[p];
        for (int32_t q = col_ptr[c]; q < col_end[c]; ++q) cnt[col_rows[q]]++;
      }
      for (int32_t x = lo; x < M; ++x)
        if (rem[x] && cnt[x] > best) { best = cnt[x]; arg = x; }
      for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) {
        const int32_t c = col_idx[p];
        for (int32_t q = col_ptr[c]; q < col_end[c]; ++q) cnt[col_rows[q]] = 0;
      }
    } else {
      for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) {
        const int32_t c = col_idx[p];
        int32_t w = col_ptr[c];
        for (int32_t q = col_ptr[c]; q < col_end[c]; ++q) {
          const int32_t r = col_rows[q];
          if (!rem[r]) continue;  // placed since this list was last compacted: drop it
          col_rows[w++] = r;
          cnt[r]++;
        }
        col_end[c] = w;
      }
      best = 0;
      for (int32_t p = csr_ptr[prev]; p < csr_ptr[prev + 1]; ++p) {
        const int32_t c = col_idx[p];
        for (int32_t q = col_ptr[c]; q < col_end[c]; ++q) {
          const int32_t r = col_rows[q], n = cnt[r];  // 0 on a row's later visits: never a candidate
          if (n > best || (n == best && n > 0 && r < arg)) { best = n; arg = r; }
          cnt[r] = 0;
        }
      }
      if (arg < 0) arg = lo;  // no remaining row shares a column with the previous one
    }
    order[i] = arg;
    rem[arg] = 0;
  }
}

// ------------------------------------------------------------------------------------------------
// Execution-ordered format: one metadata block per (row block, K chunk), in the order the
// kernel consumes them.  Two layouts:
//  row kernel   header: R_cta uint32 words (start_entry << 16 | count), padded to 16 B; then 8-byte
//               entries {uint32 col_local, float w}, each row segment starting at an even entry.
//  group kernel header: W_c × 16 B {head_off_words, n_entries, w_off_words, 0}; per warp the
//               entry heads (uint32: col_local | sub-block mask << 16; 16/SB sub-blocks of SB
//               rows) padded to 16 B; then per warp the weights: for each entry, for each nonzero
//               sub-block in ascending order, SB weights (0 for rows without a nonzero), 16-B aligned.
// Emitter: walks blocks in order; with `out` == nullptr it only computes the block sizes.
// ------------------------------------------------------------------------------------------------
struct Geometry {
  int32_t kernel, rw, wc, kc, nch, nrb, sb;
  int32_t tmem = 0;  // TMEM kernel variant of the row format (see emit_blocks)
  bool runs = true;  // TMEM V = 4: encode leading aligned 1×4 runs (block-clustered masks only)
  bool pairs = false;  // kernel 6: Algorithm 1 row pairs, shared columns loaded once (emit_blocks)
};
struct EmitStats {
  int64_t entries = 0;    // row kernel: padded entries; group kernel: union entries
  int64_t subblocks = 0;  // group kernel: nonzero sub-blocks over all entries
};

struct Pieces {  // split rows of a row plan (see Plan::piece_*)
  std::vector<int32_t> row, begin, end, stride;
};

static void emit_blocks(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals,
                        const std::vector<int32_t>& row_orig, const Geometry& g, std::vector<int64_t>& sizes,
                        uint8_t* out, const std::vector<int64_t>* offs, EmitStats* stats,
                        const Pieces* pieces = nullptr) {
  // CSR entry range of a slot: a whole row, a piece of a split row (row_orig = −2 − piece), or empty
  struct Range {
    int32_t begin, end, stride;
  };
  auto range_of = [&](int32_t orow) -> Range {
    if (orow >= 0) return {csr_ptr[orow], csr_ptr[orow + 1], 1};
    if (orow <= -2 && pieces) {
      const size_t i = size_t(-2 - orow);
      return {pieces->begin[i], pieces->end[i], pieces->stride[i]};
    }
    return {0, 0, 1};
  };
  const int32_t rcta = g.rw * g.wc;
  sizes.assign(size_t(g.nrb) * g.nch, 0);
  std::vector<int32_t> cur(rcta);
  int64_t ent_total = 0, sb_total = 0;
  // group scratch
  std::vector<uint16_t> mask(g.kc);
  std::vector<float> wv(size_t(g.kc) * 16);
  for (int32_t b = 0; b < g.nrb; ++b) {
    std::vector<int32_t> stop(rcta), step(rcta);
    for (int32_t s = 0; s < rcta; ++s) {
      const Range rg = range_of(row_orig[size_t(b) * rcta + s]);
      cur[s] = rg.begin;
      stop[s] = rg.end;
      step[s] = rg.stride;
    }
    for (int32_t j = 0; j < g.nch; ++j) {
      const int32_t lo = j * g.kc, hi = lo + g.kc;
      uint8_t* blk = out ? out + (*offs)[size_t(b) * g.nch + j] : nullptr;
      int64_t bytes = 0;
      if (g.pairs) {
        // kernel 6 (TMEM, Algorithm 1 row pairs): per pair of slots (2i, 2i+1) of a warp, the chunk's
        // entries of its two rows split three ways, each ascending: shared columns (16 bytes:
        // {TMEM column, w_a, w_b, 0}, one load feeding both rows), then the first row's other
        // columns and then the second row's ({TMEM column, w} pairs of 8 bytes, each list padded to
        // whole pairs with weight-0 entries).  Headers: slot 2i = start << 16 | shared << 8 | a-only
        // count, slot 2i+1 = start of its list << 16 | b-only count (entries of 8 bytes).
        const int64_t hdr = align_up(int64_t(rcta) * 4, 16);
        const uint32_t half = uint32_t(j & 1) * 256u;
        int32_t e = 0;
        std::vector<std::pair<int32_t, float>> ra, rb;
        for (int32_t s = 0; s < rcta; s += 2) {
          const uint32_t lane_base = uint32_t(32 * ((s / g.rw) & 3)) << 16;
          for (int32_t t = 0; t < 2; ++t) {
            auto& lst = t ? rb : ra;
            lst.clear();
            const int32_t orow = row_orig[size_t(b) * rcta + s + t];
            if (orow < 0) continue;
            int32_t& q = cur[s + t];
            while (q < stop[s + t] && col_idx[q] < hi) {
              lst.push_back({col_idx[q] - lo, vals ? vals[q] : 0.f});
              ++q;
            }
          }
          std::vector<std::array<float, 2>> sh;
          std::vector<int32_t> shc;
          std::vector<std::pair<int32_t, float>> ao, bo;
          size_t ia = 0, ib = 0;
          while (ia < ra.size() || ib < rb.size()) {
            if (ib == rb.size() || (ia < ra.size() && ra[ia].first < rb[ib].first)) ao.push_back(ra[ia++]);
            else if (ia == ra.size() || rb[ib].first < ra[ia].first) bo.push_back(rb[ib++]);
            else {
              shc.push_back(ra[ia].first);
              sh.push_back({ra[ia].second, rb[ib].second});
              ++ia, ++ib;
            }
          }
          const int32_t na = int32_t(align_up(int64_t(ao.size()), 2)), nb = int32_t(align_up(int64_t(bo.size()), 2));
          const int32_t ns = int32_t(sh.size());
          if (blk) {
            auto put = [&](int32_t at, uint32_t cl, float w) {
              std::memcpy(blk + hdr + size_t(at) * 8, &cl, 4);
              std::memcpy(blk + hdr + size_t(at) * 8 + 4, &w, 4);
            };
            for (int32_t i = 0; i < ns; ++i) {  // {column, w_a} {w_b, 0}
              const uint32_t cl = (uint32_t(shc[i]) * 4u + half) | lane_base;
              std::memcpy(blk + hdr + size_t(e + 2 * i) * 8, &cl, 4);
              std::memcpy(blk + hdr + size_t(e + 2 * i) * 8 + 4, &sh[i][0], 4);
              std::memcpy(blk + hdr + size_t(e + 2 * i + 1) * 8, &sh[i][1], 4);
            }
            const int32_t a0 = e + 2 * ns, b0 = a0 + na;
            for (int32_t i = 0; i < na; ++i)
              i < int32_t(ao.size()) ? put(a0 + i, (uint32_t(ao[i].first) * 4u + half) | lane_base, ao[i].second)
                                     : put(a0 + i, half | lane_base, 0.f);
            for (int32_t i = 0; i < nb; ++i)
              i < int32_t(bo.size()) ? put(b0 + i, (uint32_t(bo[i].first) * 4u + half) | lane_base, bo[i].second)
                                     : put(b0 + i, half | lane_base, 0.f);
            reinterpret_cast<uint32_t*>(blk)[s] = (uint32_t(e) << 16) | (uint32_t(ns) << 8) | uint32_t(na);
            reinterpret_cast<uint32_t*>(blk)[s + 1] = (uint32_t(b0) << 16) | uint32_t(nb);
          }
          e += 2 * ns + na + nb;
        }
        ent_total += e;
        bytes = align_up(hdr + int64_t(e) * 8, 16);
      } else if (g.kernel == 1) {
        // TMEM variant (g.tmem = V): the column field is the TMEM column offset of X[col] in the
        // chunk's TMEM half (V·col_local + 256·(j mod 2)) — for kernel 4 (g.wc = 24, replicated lane
        // quarters) with the TMEM lane base of the slot's warp, (32·(warp mod 4)) << 16, added — and
        // every row segment is padded to whole pairs of entries with zero weights (the count in the
        // header includes the padding) so the kernel loads entries two at a time; the padding adds
        // 0·X (X finite).
        // V = 4 also counts leading runs: while a row segment starts with aligned 1×4 runs (four
        // nonzeros at columns k..k+3, k % 4 == 0 — the blocks of a block-clustered mask), their
        // number goes into header bits 8..15 so the kernel fetches each run's four X row slices with
        // one tcgen05.ld.x16 in a loop of its own; later runs are ordinary entries (ascending column
        // order is kept).  The count field is then bits 0..7 (a segment has at most 64 + 3 entries).
        const int64_t hdr = align_up(int64_t(rcta) * 4, 16);
        const uint32_t half = uint32_t(j & 1) * 256u;
        int32_t e = 0;
        for (int32_t s = 0; s < rcta; ++s) {
          const int32_t orow = row_orig[size_t(b) * rcta + s];
          // kernel 4: TMEM lane base of the quarter of warp s / rw
          const uint32_t lane_base = (g.tmem == 4 && g.wc == kTmemRWarps) ? uint32_t(32 * ((s / g.rw) & 3)) << 16 : 0u;
          int32_t c = 0, runs = 0;
          bool leading = true;
          auto put = [&](uint32_t cl, float w) {
            if (blk) {
              std::memcpy(blk + hdr + size_t(e + c) * 8, &cl, 4);
              std::memcpy(blk + hdr + size_t(e + c) * 8 + 4, &w, 4);
            }
            ++c;
          };
          if (orow != -1) {
            int32_t& p = cur[s];
            const int32_t end = stop[s];
            const int32_t stp = step[s];
            while (p < end && col_idx[p] < hi) {
              const int32_t col = col_idx[p];
              if (stp == 1 && g.tmem == 4 && g.runs && leading && col % 4 == 0 && p + 3 < end && col_idx[p + 3] == col + 3 &&
                  col + 3 < hi) {
                for (int32_t t = 0; t < 4; ++t) put((uint32_t(col + t - lo) * 4u + half) | lane_base, vals[p + t]);
                p += 4;
                ++runs;
                continue;
              }
              leading = false;
              put(g.tmem ? (uint32_t(col - lo) * uint32_t(g.tmem) + half) | lane_base : uint32_t(col - lo), vals[p]);
              p += stp;
            }
          }
          const int32_t cpad = g.tmem ? int32_t(align_up(c, tmem_pad(g.tmem))) : c;
          while (c < cpad) put(half | lane_base, 0.f);
          if (blk) reinterpret_cast<uint32_t*>(blk)[s] = (uint32_t(e) << 16) | (uint32_t(runs) << 8) | uint32_t(cpad);
          e += int32_t(align_up(cpad, 2));
        }
        ent_total += e;
        bytes = align_up(hdr + int64_t(e) * 8, 16);
      } else {
        // group kernel: per warp (16-row group) the union of its rows' columns in this chunk
        const int64_t hdr = int64_t(g.wc) * 16;
        int64_t head_words = 0, w_words = 0;
        std::vector<std::vector<uint32_t>> wh(g.wc);
        std::vector<std::vector<float>> ww(g.wc);
        for (int32_t w = 0; w < g.wc; ++w) {
          std::fill(mask.begin(), mask.end(), 0);
          for (int32_t r = 0; r < 16; ++r) {
            const int32_t s = w * 16 + r;
            const int32_t orow = row_orig[size_t(b) * rcta + s];
            if (orow < 0) continue;
            int32_t& p = cur[s];
            while (p < csr_ptr[orow + 1] && col_idx[p] < hi) {
              const int32_t cl = col_idx[p] - lo;
              mask[cl] |= uint16_t(1u << r);
              wv[size_t(cl) * 16 + r] = vals ? vals[p] : 0.f;
              ++p;
            }
          }
          for (int32_t cl = 0; cl < g.kc; ++cl) {
            if (!mask[cl]) continue;
            const uint32_t m = mask[cl];
            uint32_t sbm = 0;
            for (int32_t sb = 0; sb < 16 / g.sb; ++sb) {
              const uint32_t part = (m >> (sb * g.sb)) & ((1u << g.sb) - 1u);
              if (!part) continue;
              sbm |= 1u << sb;
              for (int32_t i = 0; i < g.sb; ++i)  // SB weights, zero for rows without a nonzero
                ww[w].push_back(part >> i & 1u ? wv[size_t(cl) * 16 + sb * g.sb + i] : 0.f);
              ++sb_total;
            }
            wh[w].push_back(uint32_t(cl) | (sbm << 16));
          }
          head_words += align_up(int64_t(wh[w].size()), 4);
          w_words += align_up(int64_t(ww[w].size()), 4);
          ent_total += int64_t(wh[w].size());
        }
        bytes = align_up(hdr + head_words * 4 + w_words * 4, 16);
        if (blk) {
          uint32_t* h32 = reinterpret_cast<uint32_t*>(blk);
          int64_t hpos = hdr / 4, wpos = hdr / 4 + head_words;
          for (int32_t w = 0; w < g.wc; ++w) {
            h32[w * 4 + 0] = uint32_t(hpos);
            h32[w * 4 + 1] = uint32_t(wh[w].size());
            h32[w * 4 + 2] = uint32_t(wpos);
            h32[w * 4 + 3] = 0;
            std::memcpy(h32 + hpos, wh[w].data(), wh[w].size() * 4);
            hpos += align_up(int64_t(wh[w].size()), 4);
            std::memcpy(h32 + wpos, ww[w].data(), ww[w].size() * 4);
            wpos += align_up(int64_t(ww[w].size()), 4);  // 16-byte aligned vector weight loads
          }
        }
      }
      sizes[size_t(b) * g.nch + j] = bytes;
    }
  }
  if (stats) {
    stats->entries = ent_total;
    stats->subblocks = sb_total;
  }
}

static int64_t max_of(const std::vector<int64_t>& v) {
  int64_t m = 0;
  for (int64_t x : v) m = std::max(m, x);
  return m;
}

// X stage bytes at the widest N tile + metadata stage; S stages must fit the smem budget.
static int32_t stages_for(int32_t kc, int64_t max_block) {
  return int32_t(kSmemBudget / (int64_t(kc) * kMaxTN * 4 + align_up(max_block, 128)));
}

sdnn_status build_plan(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M, int32_t K,
                       const sdnn_perm_opts* opts, Plan& plan, const std::vector<int32_t>* perm) {
  sdnn_perm_opts o{};
  o.struct_size = sizeof(o);
  o.permute = 1;
  if (opts) {
    if (opts->struct_size != sizeof(sdnn_perm_opts))
      return fail(SDNN_ERR_INVALID_ARGUMENT, "sdnn_perm_opts.struct_size mismatch");
    o = *opts;
    if (o.flags & ~(SDNN_FLAG_NO_ROW_SPLIT | SDNN_FLAG_PERMUTED_OUTPUT | SDNN_FLAG_NO_SPLIT_K))
      return fail(SDNN_ERR_INVALID_ARGUMENT, "unknown sdnn_perm_opts.flags bits");
    if ((o.flags & SDNN_FLAG_PERMUTED_OUTPUT) && o.kernel == 3)
      return fail(SDNN_ERR_UNSUPPORTED, "SDNN_FLAG_PERMUTED_OUTPUT is not available with the codegen kernel");
    if (o.permute != 0 && o.permute != 1) return fail(SDNN_ERR_INVALID_ARGUMENT, "permute must be 0 or 1");
    if (o.kernel < 0 || o.kernel > 6) return fail(SDNN_ERR_INVALID_ARGUMENT, "kernel must be 0..6");
    if (o.kernel == 4 || o.kernel == 5 || o.kernel == 6) {
      // kernel 4 alone takes panel_rows_max = 1..10: about that many rows per warp (more row blocks)
      const bool rows_ok = o.panel_rows_max == 0 || (o.kernel == 4 && o.panel_rows_max >= 1 && o.panel_rows_max <= tmem_rows(4));
      if (!rows_ok || o.cta_panels != 0 || (o.k_chunk != 0 && o.k_chunk != tmem_kc(tmem_v(o.kernel))) ||
          o.group_sb != 0)
        return fail(SDNN_ERR_INVALID_ARGUMENT,
                    "the TMEM kernels have a fixed geometry (tiling options 0; kernel 4: panel_rows_max 1..10)");
    } else if (o.kernel == 3) {
      if (o.panel_rows_max < 0 || o.panel_rows_max > kCgMaxRows)
        return fail(SDNN_ERR_INVALID_ARGUMENT, "panel_rows_max must be 0..128 with the codegen kernel");
    } else if (o.panel_rows_max != 0 && o.panel_rows_max != 4 && o.panel_rows_max != 8 &&
               !(o.panel_rows_max == 16 && o.kernel == 2)) {
      return fail(SDNN_ERR_INVALID_ARGUMENT, "panel_rows_max must be 0, 4 or 8 (16 with the group kernel)");
    }
    if (o.cta_panels < 0 || o.cta_panels > 16) return fail(SDNN_ERR_INVALID_ARGUMENT, "cta_panels must be 0..16");
    if (o.kernel == 2 && o.cta_panels > kMaxGroupWarps)
      return fail(SDNN_ERR_INVALID_ARGUMENT, "cta_panels must be <= 11 with the group kernel");
    if (o.group_sb != 0 && o.group_sb != 1 && o.group_sb != 2 && o.group_sb != 4)
      return fail(SDNN_ERR_INVALID_ARGUMENT, "group_sb must be 0, 1, 2 or 4");
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
    plan.no_split_k = (o.flags & SDNN_FLAG_NO_SPLIT_K) ? 1 : 0;
    plan.perm.resize(M);
    if (o.permute && perm && perm->size() == size_t(M))
      plan.perm = *perm;
    else if (o.permute)
      algorithm1(csr_ptr, col_idx, M, K, plan.perm.data());
    else
      for (int32_t i = 0; i < M; ++i) plan.perm[i] = i;

    if (o.kernel == 3) {
      // Codegen kernel (sdnn_codegen.cpp): consecutive rows of the Algorithm 1 order form a panel,
      // so rows with similar patterns share one X load per union column.  Panel count P:
      // the smallest divisor of the CTA slots (2 per SM on 148 SMs = 296) with ceil(M / P) <= 128,
      // so every panel gets the same number of persistent CTAs and all panels sweep N in lockstep.
      const int32_t rmax = o.panel_rows_max ? o.panel_rows_max : kCgMaxRows;
      const int32_t need = (M + rmax - 1) / rmax;
      const int32_t slots = 296;
      int32_t P = need;
      for (int32_t d = need; d <= slots; ++d)
        if (slots % d == 0) { P = d; break; }
      if (P > M) P = M;
      plan.kernel = 3;
      plan.cg_warps = kCgWarps;
      plan.cg_prefetch = kCgPrefetch;
      plan.cg_panels.assign(P, {});
      const int32_t rows_per = (M + P - 1) / P;
      for (int32_t i = 0; i < M; ++i) plan.cg_panels[i / rows_per].push_back(plan.perm[i]);
      while (!plan.cg_panels.empty() && plan.cg_panels.back().empty()) plan.cg_panels.pop_back();
      plan.panel_rows = rows_per;
      plan.cta_panels = 1;
      plan.num_panels = int32_t(plan.cg_panels.size());
      plan.num_row_blocks = plan.num_panels;
      plan.row_orig.assign(size_t(plan.num_panels) * rows_per, -1);
      for (int32_t pn = 0; pn < plan.num_panels; ++pn) {
        int64_t s = 0;
        for (size_t r = 0; r < plan.cg_panels[pn].size(); ++r) {
          plan.row_orig[size_t(pn) * rows_per + r] = plan.cg_panels[pn][r];
          s += csr_ptr[plan.cg_panels[pn][r] + 1] - csr_ptr[plan.cg_panels[pn][r]];
        }
        plan.max_panel_nnz = std::max(plan.max_panel_nnz, s);
      }
      plan.k_chunk = K;
      plan.num_chunks = 1;
      plan.blk_off.assign(size_t(plan.num_row_blocks) + 1, 0);
      return SDNN_OK;
    }

    // Candidate geometries: the row kernel (R_w rows per warp) and the group kernel (16 rows per
    // warp).  Launch geometry: W_c warps per CTA, enough row blocks to fill
    // the machine for the typical N.
    auto make_geo = [&](int32_t kernel, int32_t sb) {
      Geometry g{};
      if (kernel == 4 || kernel == 5 || kernel == 6) {
        // TMEM kernels (sdnn_spmm.cu): row-kernel format, tmem_rows(V)-row warp panels; kernel 4: 24
        // panels per CTA row block (one per consumer warp, replicated lane quarters), kernel 5: 6
        // (one per warp slot, shared by the 4 lane quarters); K chunk = one TMEM half.
        g.kernel = 1;
        g.tmem = tmem_v(kernel);
        g.rw = tmem_rows(g.tmem);
        // runs pay only on block-clustered masks: encode them when ≥ 1/4 of the nonzeros sit in aligned
        // 1×4 groups (a uniform 90 % mask has ~0.1 % by chance — then the kernel takes its run-free loop)
        if (g.pairs) {
          g.runs = false;  // kernel 6: no x16 run loads (a run's four entries are ordinary entries)
        } else if (g.tmem == 4) {
          int64_t in_runs = 0;
          for (int32_t r = 0; r < M; ++r)
            for (int32_t q = csr_ptr[r]; q + 3 < csr_ptr[r + 1]; ++q)
              if (col_idx[q] % 4 == 0 && col_idx[q + 3] == col_idx[q] + 3) in_runs += 4;
          g.runs = 4 * in_runs >= nnz;
        }
        // (rows per warp: 10 measured against 9 and 8 on c5 — 41.8 / 43.4 / 48.1 ms,
        // profiles/r02_tmemr_rows_per_warp.log: fewer rows per CTA cost more than the freed registers gain)
        g.wc = (kernel == 4 || kernel == 6) ? kTmemRWarps : kTmemPanels;
        g.pairs = kernel == 6;
        g.nrb = (M + g.rw * g.wc - 1) / (g.rw * g.wc);
        // kernel 4 with panel_rows_max = r < 10: row blocks for ~r rows per warp (the panels' slots
        // partly empty) — more, lighter CTAs for calls whose grid would fill its last wave badly
        if (kernel == 4 && o.panel_rows_max > 0 && o.panel_rows_max < g.rw)
          g.nrb = std::max(g.nrb, int32_t((int64_t(M) + int64_t(o.panel_rows_max) * g.wc - 1) /
                                          (int64_t(o.panel_rows_max) * g.wc)));
        return g;
      }
      g.kernel = kernel;
      g.sb = sb;
      g.rw = kernel == 2 ? 16 : (o.panel_rows_max ? o.panel_rows_max : (M >= 2048 ? 8 : 4));
      int32_t wc = o.cta_panels;
      if (!wc) {
        wc = kernel == 2 ? kMaxGroupWarps : 16;
        while (wc > 4 && (M + g.rw * wc - 1) / (g.rw * wc) < (kernel == 2 ? 16 : 32)) wc = kernel == 2 ? wc - 1 : wc / 2;
      }
      g.wc = wc;
      g.nrb = (M + g.rw * wc - 1) / (g.rw * wc);
      return g;
    };
    // Row → (CTA, warp, slot) assignment.  Group kernel: the Algorithm 1 order itself, so rows
    // with similar patterns share a 16-row group.  Row kernel: every nonzero costs the
    // same wherever its row sits, so rows are dealt to warps by nnz instead — longest-processing-
    // time first onto the least-loaded warp with a free slot — which keeps the heavy rows of a
    // skewed (log-normal) matrix from piling into one warp.  Within a warp the rows keep their
    // Algorithm 1 order.
    //
    // Heavy rows (row plan only; not with SDNN_FLAG_NO_ROW_SPLIT): a row with more nonzeros than the
    // mean load of a warp, T = ⌈nnz / warps⌉ (at least 64), would make its warp the critical path of
    // the whole launch (log-normal rows: up to K nonzeros) — and, since the warps of a CTA advance
    // through the K chunks together, of every chunk.  It is dealt out in P = ⌈nnz_row / T⌉
    // interleaved pieces (piece q: entries q, q + P, … of the row, ascending columns) so each piece
    // has ~1/P of every chunk, and the pieces are placed by the LPT like rows.
    Pieces pcs;
    auto row_orig_for = [&](Geometry& g, Pieces* out) {
      if (out) *out = Pieces{};
      if (g.kernel == 2) {
        std::vector<int32_t> ro(size_t(g.nrb) * g.wc * g.rw, -1);
        for (int32_t p = 0; p < M; ++p) ro[p] = plan.perm[p];
        return ro;
      }
      std::vector<int32_t> pos(M);
      for (int32_t i = 0; i < M; ++i) pos[plan.perm[i]] = i;
      auto nz = [&](int32_t r) { return csr_ptr[r + 1] - csr_ptr[r]; };
      if (g.pairs) {
        // kernel 6: rows go in pairs of consecutive Algorithm 1 positions (perm[2i], perm[2i+1]) —
        // the rows with the most common columns — so a shared column is loaded once for
        // both; pairs are dealt to warps by the LPT (weight = both rows' nonzeros), rw / 2 per warp,
        // and keep their Algorithm 1 order inside a warp
        const int32_t np = (M + 1) / 2, cap = g.rw / 2;
        g.nrb = std::max(g.nrb, int32_t((int64_t(np) + int64_t(cap) * g.wc - 1) / (int64_t(cap) * g.wc)));
        const int32_t nw = g.nrb * g.wc;
        std::vector<std::pair<int64_t, int32_t>> items;
        items.reserve(size_t(np));
        for (int32_t i = 0; i < np; ++i)
          items.push_back({nz(plan.perm[2 * i]) + (2 * i + 1 < M ? nz(plan.perm[2 * i + 1]) : 0), i});
        std::stable_sort(items.begin(), items.end(),
                         [](const std::pair<int64_t, int32_t>& a, const std::pair<int64_t, int32_t>& b) {
                           return a.first > b.first;
                         });
        std::vector<std::pair<int64_t, int32_t>> heap;
        for (int32_t w = 0; w < nw; ++w) heap.push_back({0, w});
        auto cmp = [](const std::pair<int64_t, int32_t>& a, const std::pair<int64_t, int32_t>& b) { return a > b; };
        std::vector<std::vector<int32_t>> prs(nw);
        for (const auto& it : items) {
          std::pop_heap(heap.begin(), heap.end(), cmp);
          auto [load, w] = heap.back();
          heap.pop_back();
          prs[w].push_back(it.second);
          if (int32_t(prs[w].size()) < cap) {
            heap.push_back({load + it.first + 1, w});
            std::push_heap(heap.begin(), heap.end(), cmp);
          }
        }
        std::vector<int32_t> ro(size_t(nw) * g.rw, -1);
        for (int32_t w = 0; w < nw; ++w) {
          std::sort(prs[w].begin(), prs[w].end());
          for (size_t j = 0; j < prs[w].size(); ++j) {
            const int32_t i = prs[w][j];
            ro[size_t(w) * g.rw + 2 * j] = plan.perm[2 * i];
            if (2 * i + 1 < M) ro[size_t(w) * g.rw + 2 * j + 1] = plan.perm[2 * i + 1];
          }
        }
        return ro;
      }
      // items: whole rows (id = row) and pieces (id = −2 − piece); weight = nonzeros
      std::vector<std::pair<int64_t, int32_t>> items;
      items.reserve(size_t(M));
      const bool split = out && g.kernel == 1 && g.tmem == 0 && !(o.flags & SDNN_FLAG_NO_ROW_SPLIT);
      const int32_t nw0 = g.nrb * g.wc;
      const int64_t T = std::max<int64_t>(64, (nnz + nw0 - 1) / std::max(nw0, 1));
      // split rows: [first piece, piece count) per heavy row, heaviest first
      std::vector<std::pair<int64_t, std::pair<int32_t, int32_t>>> groups;
      for (int32_t r = 0; r < M; ++r) {
        const int64_t n = nz(r);
        if (split && n > T) {
          // at most one piece per warp of a CTA: the pieces of a row share a row block, so the row
          // kernel adds them in shared memory at its end (no workspace, no reduction kernel)
          const int32_t P = int32_t(std::min<int64_t>((n + T - 1) / T, g.wc));
          groups.push_back({n, {int32_t(out->row.size()), P}});
          for (int32_t q = 0; q < P; ++q) {  // piece q: entries q, q + P, q + 2P, … of the row
            items.push_back({(n - q + P - 1) / P, -2 - int32_t(out->row.size())});
            out->row.push_back(r);
            out->begin.push_back(csr_ptr[r] + q);
            out->end.push_back(csr_ptr[r + 1]);
            out->stride.push_back(P);
          }
        } else {
          items.push_back({n, r});
        }
      }
      auto orig_of = [&](int32_t id) { return id >= 0 ? id : out->row[size_t(-2 - id)]; };
      // pieces need slots: more row blocks if the rows already fill them
      const int64_t per_block = int64_t(g.rw) * g.wc;
      g.nrb = int32_t(std::max<int64_t>(g.nrb, (int64_t(items.size()) + per_block - 1) / per_block));
      const int32_t nw = g.nrb * g.wc;
      std::vector<int32_t> ro(size_t(nw) * g.rw, -1);
      std::stable_sort(items.begin(), items.end(),
                       [&](const std::pair<int64_t, int32_t>& a, const std::pair<int64_t, int32_t>& b) {
                         return a.first > b.first;
                       });
      std::vector<int32_t> fill(nw, 0);
      std::vector<int64_t> load(nw, 0);
      std::vector<std::vector<int32_t>> rows(nw);
      // 1. the split rows' pieces, heaviest row first: the row block whose least-loaded free warps
      //    take the pieces with the smallest resulting maximum load (lowest block on ties), one piece
      //    per warp.  Bounded work (groups × warps); beyond it, or if no block has room, the pieces
      //    go through the LPT below like rows (anywhere: workspace + reduction kernel instead).
      bool local = !groups.empty() && int64_t(groups.size()) * g.nrb * g.wc <= 8000000;
      std::stable_sort(groups.begin(), groups.end(),
                       [](const auto& a, const auto& b) { return a.first > b.first; });
      std::vector<char> placed(out ? out->row.size() : 0, 0);
      for (size_t gi = 0; local && gi < groups.size(); ++gi) {
        const int32_t first = groups[gi].second.first, P = groups[gi].second.second;
        std::vector<int64_t> wt(P);
        for (int32_t q = 0; q < P; ++q) {
          const int64_t n = (out->end[size_t(first + q)] - out->begin[size_t(first + q)] + P - 1) / P;
          wt[size_t(q)] = n;
        }
        int32_t best_b = -1;
        int64_t best_c = 0;
        std::vector<int32_t> best_w, cand;
        for (int32_t b = 0; b < g.nrb; ++b) {
          cand.clear();
          for (int32_t w = b * g.wc; w < (b + 1) * g.wc; ++w)
            if (fill[w] < g.rw) cand.push_back(w);
          if (int32_t(cand.size()) < P) continue;
          std::stable_sort(cand.begin(), cand.end(), [&](int32_t x, int32_t y) { return load[x] < load[y]; });
          int64_t c = 0;
          for (int32_t q = 0; q < P; ++q) c = std::max(c, load[cand[size_t(q)]] + wt[size_t(q)] + 1);
          if (best_b < 0 || c < best_c) {
            best_b = b;
            best_c = c;
            best_w.assign(cand.begin(), cand.begin() + P);
          }
        }
        if (best_b < 0) {
          local = false;
          break;
        }
        for (int32_t q = 0; q < P; ++q) {
          const int32_t w = best_w[size_t(q)];
          rows[w].push_back(-2 - (first + q));
          load[w] += wt[size_t(q)] + 1;
          ++fill[w];
          placed[size_t(first + q)] = 1;
        }
      }
      if (!local) {  // undo: every item through the LPT
        std::fill(fill.begin(), fill.end(), 0);
        std::fill(load.begin(), load.end(), 0);
        for (auto& v : rows) v.clear();
        std::fill(placed.begin(), placed.end(), 0);
      }
      // 2. LPT: min-heap of (load, warp); warps with full slots leave the heap
      std::vector<std::pair<int64_t, int32_t>> heap;
      heap.reserve(nw);
      for (int32_t w = 0; w < nw; ++w)
        if (fill[w] < g.rw) heap.push_back({load[w], w});
      auto cmp = [](const std::pair<int64_t, int32_t>& a, const std::pair<int64_t, int32_t>& b) { return a > b; };
      std::make_heap(heap.begin(), heap.end(), cmp);
      for (const auto& it : items) {
        if (it.second <= -2 && placed[size_t(-2 - it.second)]) continue;
        std::pop_heap(heap.begin(), heap.end(), cmp);
        auto [ld, w] = heap.back();
        heap.pop_back();
        rows[w].push_back(it.second);
        if (++fill[w] < g.rw) {
          heap.push_back({ld + it.first + 1, w});
          std::push_heap(heap.begin(), heap.end(), cmp);
        }
      }
      for (int32_t w = 0; w < nw; ++w) {
        std::sort(rows[w].begin(), rows[w].end(), [&](int32_t a, int32_t b) {
          const int32_t pa = pos[orig_of(a)], pb = pos[orig_of(b)];
          return pa != pb ? pa < pb : a > b;  // pieces of one row: in piece order (ids −2, −3, …)
        });
        for (size_t i = 0; i < rows[w].size(); ++i) ro[size_t(w) * g.rw + i] = rows[w][i];
      }
      return ro;
    };
    // K chunk (split-K tiling along the reduction dimension): the largest KC whose stage
    // (X tile at the widest N tile + metadata block) fits three times in the shared-memory budget.
    auto choose_kc = [&](Geometry& g, const std::vector<int32_t>& ro, EmitStats* entries) -> bool {
      std::vector<int64_t> sizes;
      const int32_t cands[] = {64, 32, 16, 8};
      for (int32_t c : cands) {
        if (o.k_chunk && c != o.k_chunk) continue;
        g.kc = c;
        g.nch = (K + c - 1) / c;
        emit_blocks(csr_ptr, col_idx, vals, ro, g, sizes, nullptr, nullptr, entries, &pcs);
        if (g.tmem == 4)  // kernels 4 / 6: 8 KB TMA pieces × kTmemRPieces + two metadata slots
          return int64_t(kTmemRPieces) * 8192 + 2 * align_up(max_of(sizes), 128) + 1024 <= kSmemBudget;
        const int32_t s = stages_for(c, max_of(sizes));
        if (s >= 3 || (s >= 2 && (o.k_chunk || c == 8))) return true;
      }
      if (o.k_chunk) {  // explicit KC not in the candidate list
        g.kc = o.k_chunk;
        g.nch = (K + g.kc - 1) / g.kc;
        emit_blocks(csr_ptr, col_idx, vals, ro, g, sizes, nullptr, nullptr, entries, &pcs);
        return stages_for(g.kc, max_of(sizes)) >= 2;
      }
      return false;
    };

    // Cost model (SM cycles per warp-level unit of work at V = 8 floats per lane; DESIGN.md
    // "Kernel choice"): shared-memory wavefronts at 128 B/clk (≈85 % attainable), FMA pipe at 128
    // lanes/clk, issue at 4 warp-instructions/clk.  Row kernel per nonzero: 8 X wavefronts + 0.5
    // entry.  Group kernel per union entry: 8 X wavefronts + 0.25 head + 1 per nonzero sub-block
    // (weights), 2·SB FMA cycles per nonzero sub-block, issue ≈ (2·16/SB + nsb·(2 + 4·SB) + 8) / 4.
    auto cost = [&](const Geometry& g, const EmitStats& st) {
      if (g.kernel == 1) return 8.5 / 0.85 * double(nnz);
      const double E = double(st.entries), S = double(st.subblocks);
      const double lds = (8.25 * E + S) / 0.85, fma = 2.0 * g.sb * S / 0.95;
      const double issue = (2.0 * (16 / g.sb) * E + S * (2 + 4 * g.sb) + 8 * E) / 4.0;
      return std::max(lds, std::max(fma, issue));
    };
    Geometry g{};
    std::vector<int32_t> ro;
    EmitStats stats;
    {
      std::vector<Geometry> cands;
      if (o.kernel == 4 || o.kernel == 5 || o.kernel == 6) {
        o.k_chunk = tmem_kc(tmem_v(o.kernel));
        cands.push_back(make_geo(o.kernel, 0));
      } else if (o.kernel != 2) {
        cands.push_back(make_geo(1, 0));
      }
      if (o.kernel == 2)
        for (int32_t sb : {1, 2, 4})
          if (!o.group_sb || o.group_sb == sb) cands.push_back(make_geo(2, sb));
      double best = 0;
      bool found = false;
      Pieces best_pcs;
      for (Geometry c : cands) {
        std::vector<int32_t> r = row_orig_for(c, &pcs);
        EmitStats st;
        bool fits = choose_kc(c, r, &st);
        // kernel 4 (240 rows per CTA): a dense matrix's metadata block can outgrow its shared-memory
        // slot — spread the rows over more row blocks (fewer rows per warp) until it fits
        while (!fits && c.tmem == 4 && int64_t(c.nrb) * c.wc < M) {
          c.nrb = int32_t(std::min<int64_t>(int64_t(c.nrb) * 2, (M + c.wc - 1) / c.wc));
          r = row_orig_for(c, &pcs);
          fits = choose_kc(c, r, &st);
        }
        if (!fits) continue;
        const double cc = cost(c, st);
        if (!found || cc < best) { best = cc; g = c; ro.swap(r); stats = st; found = true; best_pcs = pcs; }
      }
      pcs = best_pcs;
      if (!found) return fail(SDNN_ERR_UNSUPPORTED, "no K chunk fits the shared-memory budget");
    }
    plan.kernel = (o.kernel == 4 || o.kernel == 5 || o.kernel == 6) ? o.kernel : g.kernel;
    plan.panel_rows = g.rw;
    plan.cta_panels = g.wc;
    plan.num_row_blocks = g.nrb;
    plan.num_panels = g.nrb * g.wc;
    plan.k_chunk = g.kc;
    plan.num_chunks = g.nch;
    plan.row_orig.swap(ro);
    for (int32_t pn = 0; pn < plan.num_panels; ++pn) {
      int64_t s = 0;
      for (int32_t r = 0; r < g.rw; ++r) {
        const int32_t orow = plan.row_orig[size_t(pn) * g.rw + r];
        if (orow >= 0) s += csr_ptr[orow + 1] - csr_ptr[orow];
        if (orow <= -2) {
          const size_t i = size_t(-2 - orow);
          s += (pcs.end[i] - pcs.begin[i] + pcs.stride[i] - 1) / pcs.stride[i];
        }
      }
      plan.max_panel_nnz = std::max(plan.max_panel_nnz, s);
    }
    // split-row table for the reduction kernel (pieces of a row have consecutive ids)
    plan.piece_row = pcs.row;
    plan.piece_begin = pcs.begin;
    plan.piece_end = pcs.end;
    for (size_t i = 0; i < pcs.row.size(); ++i) {
      if (i == 0 || pcs.row[i] != pcs.row[i - 1]) {
        plan.split_row.push_back(pcs.row[i]);
        plan.split_first.push_back(int32_t(i));
        plan.split_count.push_back(0);
      }
      plan.split_count.back()++;
    }
    std::vector<int64_t> sizes;
    emit_blocks(csr_ptr, col_idx, vals, plan.row_orig, g, sizes, nullptr, nullptr, &stats, &pcs);
    plan.group_entries = g.kernel == 2 ? stats.entries : 0;
    plan.group_sb = g.kernel == 2 ? g.sb : 0;
    plan.group_subblocks = g.kernel == 2 ? stats.subblocks : 0;
    plan.max_block_bytes = int32_t(max_of(sizes));
    plan.blk_off.assign(sizes.size() + 1, 0);
    for (size_t i = 0; i < sizes.size(); ++i) plan.blk_off[i + 1] = plan.blk_off[i] + sizes[i];
    // zero-filled: the partner slot of an odd row segment stays (column 0, weight 0.0), which the
    // row kernel and the conv kernels read unconditionally as an entry pair
    plan.meta.assign(size_t(plan.blk_off.back()), 0);
    emit_blocks(csr_ptr, col_idx, vals, plan.row_orig, g, sizes, plan.meta.data(), &plan.blk_off, nullptr, &pcs);
    if (o.flags & SDNN_FLAG_PERMUTED_OUTPUT) {
      // output rows (and bias entries) by plan position instead of original row; the
      // metadata above was emitted from the original rows' CSR entries, so this comes last
      std::vector<int32_t> pos(static_cast<size_t>(M));
      for (int32_t i = 0; i < M; ++i) pos[size_t(plan.perm[i])] = i;
      for (auto& r : plan.row_orig)
        if (r >= 0) r = pos[size_t(r)];
      for (auto& r : plan.split_row) r = pos[size_t(r)];
      plan.permuted_output = 1;
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
  info->kernel = p.kernel;
  info->group_entries_per_nnz_x1000 = p.nnz ? int32_t(1000 * p.group_entries / p.nnz) : 0;
  info->group_sb = p.group_sb;
  info->group_subblocks_per_nnz_x1000 = p.nnz ? int32_t(1000 * p.group_subblocks / p.nnz) : 0;
  info->panel_rows = p.panel_rows;
  info->cta_panels = p.cta_panels;
  info->num_panels = p.num_panels;
  info->num_row_blocks = p.num_row_blocks;
  info->k_chunk = p.k_chunk;
  info->num_chunks = p.num_chunks;
  info->meta_bytes = int64_t(p.meta.size());
  info->max_block_bytes = p.max_block_bytes;
  info->alt_kernel = 0;
  info->max_panel_nnz = p.max_panel_nnz;
  info->num_split_rows = int32_t(p.split_row.size());
  info->num_pieces = int32_t(p.piece_row.size());
  info->narrow_row_blocks = 0;
  info->narrow4_row_blocks = 0;
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

sdnn_status sdnn_csr_permute_columns(const int32_t* csr_ptr, const int32_t* col_idx, const float* vals, int32_t M,
                                     int32_t K, const int32_t* order, int32_t* out_col_idx, float* out_vals) {
  if (!order || !out_col_idx || !out_vals) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL order or output");
  sdnn_status st = validate_csr(csr_ptr, col_idx, M, K);
  if (st != SDNN_OK) return st;
  if (csr_ptr[M] > 0 && !vals) return fail(SDNN_ERR_INVALID_ARGUMENT, "vals is NULL with nnz > 0");
  try {
    std::vector<int32_t> pos(size_t(K), -1);
    for (int32_t i = 0; i < K; ++i) {
      const int32_t c = order[i];
      if (c < 0 || c >= K || pos[size_t(c)] != -1) return fail(SDNN_ERR_INVALID_ARGUMENT, "order is not a permutation of 0..K-1");
      pos[size_t(c)] = i;
    }
    std::vector<std::pair<int32_t, float>> row;
    for (int32_t r = 0; r < M; ++r) {
      row.clear();
      for (int32_t p = csr_ptr[r]; p < csr_ptr[r + 1]; ++p) row.emplace_back(pos[size_t(col_idx[p])], vals[p]);
      std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (size_t i = 0; i < row.size(); ++i) {
        out_col_idx[csr_ptr[r] + int32_t(i)] = row[i].first;
        out_vals[csr_ptr[r] + int32_t(i)] = row[i].second;
      }
    }
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

sdnn_status sdnn_plan_export_pieces(sdnn_plan p, int32_t* row, int32_t* begin, int32_t* end) {
  if (!p) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL plan");
  const Plan& pl = p->plan;
  const size_t n = pl.piece_row.size() * 4;
  if (row && n) std::memcpy(row, pl.piece_row.data(), n);
  if (begin && n) std::memcpy(begin, pl.piece_begin.data(), n);
  if (end && n) std::memcpy(end, pl.piece_end.data(), n);
  return SDNN_OK;
}

sdnn_status sdnn_plan_codegen_ptx(sdnn_plan p, const int32_t* csr_ptr, const int32_t* col_idx, const float* vals,
                                  int32_t panel, char* out, int64_t* len) {
  if (!p || !len || !csr_ptr) return fail(SDNN_ERR_INVALID_ARGUMENT, "NULL plan, csr_ptr or len");
  const Plan& pl = p->plan;
  if (pl.kernel != 3) return fail(SDNN_ERR_INVALID_ARGUMENT, "plan was not created with kernel = 3");
  if (panel < 0 || panel >= int32_t(pl.cg_panels.size())) return fail(SDNN_ERR_INVALID_ARGUMENT, "panel out of range");
  try {
    const std::string ptx = codegen_panel_ptx(csr_ptr, col_idx, vals, pl.cg_panels[panel], pl.K, pl.cg_warps,
                                              pl.cg_prefetch, "sdnn_cg_p" + std::to_string(panel));
    if (out) {
      if (*len < int64_t(ptx.size()) + 1) return fail(SDNN_ERR_INVALID_ARGUMENT, "buffer too small");
      std::memcpy(out, ptx.c_str(), ptx.size() + 1);
    }
    *len = int64_t(ptx.size()) + 1;
  } catch (const std::bad_alloc&) {
    return fail(SDNN_ERR_OUT_OF_MEMORY, "host allocation failed");
  }
  return SDNN_OK;
}

sdnn_status sdnn_plan_destroy(sdnn_plan p) {
  delete p;
  return SDNN_OK;
}

}  // extern "C"
