// N1 — profile-table staging (host side).
//
// Restates PolicyIndex.__init__ (policy.py:118-134) for the three exhaustive regimes of every
// grid at once and merges them into ONE rank structure, so that the per-timestep kernel does a
// single threshold search per cap and reads all 3 policies' decisions from it:
//
//   * entries are sorted by (power_w, mtl, bs)                               policy.py:129
//   * regime slices: batching = mtl == batching_mtl, multi-tenant =
//     bs == multi_tenant_bs, combination = all                               policy.py:100-107
//   * prefix-best with _prefer (higher ips, then lower (power, mtl, bs))     policy.py:90-97,131-134
//   * feasible_count = bisect_right(powers, cap) = #regime entries <= cap    policy.py:139
//
// For every cap, all three regimes' (selection, feasible_count) depend only on how many
// COMBINATION entries have power <= cap, i.e. on the grid bin of the cap among the grid's
// distinct power thresholds. fp32 caps use thresholds rounded UP to fp32, which admits exactly
// the same entries as the fp64 comparison (power <= cap  <=>  roundup32(power) <= cap for an
// fp32 cap). Grids are merged by taking the union of their thresholds ("union bins"); each grid
// maps union bin -> grid bin through umap.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <map>
#include <set>
#include <utility>

#include "cs_internal.h"

namespace cs {
namespace {

uint32_t f32_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
uint64_t f64_bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

// Smallest fp32 >= d (d finite, > 0). Round-up (not round-to-nearest) keeps the comparison
// exact: for any fp32 cap c, d <= c  <=>  roundup32(d) <= c.
float roundup_f32(double d) {
  float f = (float)d;
  if ((double)f < d) f = std::nextafter(f, INFINITY);
  return f;
}

struct Entry {
  int32_t mtl, bs;
  double thr, pw;
  int32_t idx;
  uint64_t key;  // threshold bits in the cap dtype
};

// _prefer (policy.py:90-97): true when a is preferred over b.
bool prefer(const Entry& a, const Entry& b) {
  if (a.thr != b.thr) return a.thr > b.thr;
  if (a.pw != b.pw) return a.pw < b.pw;
  if (a.mtl != b.mtl) return a.mtl < b.mtl;
  return a.bs <= b.bs;
}

bool in_regime(int p, const Entry& e, int32_t bmtl, int32_t mbs) {
  if (p == CS_BATCHING) return e.mtl == bmtl;
  if (p == CS_MULTI_TENANT) return e.bs == mbs;
  return true;
}

// ---- LUT builder -------------------------------------------------------------------------
struct LutBuilder {
  const std::vector<uint64_t>& T;
  bool f32;
  const std::vector<uint64_t>* vio = nullptr;  // fp32: violation floors per union bin
  std::vector<uint32_t> sub;  // sub-table entries (appended after level 1)
  uint32_t n_sub = 0;
  uint32_t unsafe = 0;        // fp32 leaves whose selections are not proven to fit their caps
  uint32_t sub0 = 0;          // fp32: first sub-table entry (= level-1 size): redirects hold byte offsets
  bool too_big = false;       // fp32: a sub-table beyond the 25-bit byte offset of a redirect

  LutBuilder(const std::vector<uint64_t>& t, bool is_f32, const std::vector<uint64_t>* v = nullptr, uint32_t s0 = 0)
      : T(t), f32(is_f32), vio(v), sub0(s0) {}

  // Bit 0 of an fp32 leaf (free: K is a multiple of 4) flags a leaf for which some cap of its
  // range could select a config drawing more than the cap. Proof per leaf: every cap of the
  // bucket is >= `start` and maps to bin `b0`; caps >= `t1` (the bucket's threshold) map to b0+1.
  uint32_t flag(uint64_t start, uint32_t b0, bool has_t1, uint64_t t1) {
    if (!vio) return 0u;
    bool ok = (*vio)[b0] <= start;
    if (has_t1) ok = ok && (*vio)[b0 + 1] <= t1;
    if (!ok) ++unsafe;
    return ok ? 0u : 1u;
  }

  uint32_t lb(uint64_t v) const { return (uint32_t)(std::lower_bound(T.begin(), T.end(), v) - T.begin()); }

  // Entry for the half-open bit range [start, start + 2^s) (start aligned to 2^s), or the
  // single value `start` when s == 0. Encodings: see cs_internal.h.
  uint32_t make(uint64_t start, uint32_t s) {
    uint64_t end = (s >= 63) ? ~0ull : start + (1ull << s);
    uint32_t base = lb(start);
    uint32_t stop = (s >= 63) ? (uint32_t)T.size() : lb(end);
    uint32_t n = stop - base;
    if (f32) {  // leaves hold E - (start << 2) (cs_internal.h): the kernel adds (cap << 2)
      const uint32_t off = (uint32_t)start << 2;
      if (n == 0) return ((base << 16) | flag(start, base, false, 0)) - off;
      if (n == 1 && s <= kMaxShift32) {
        const uint32_t tl = (uint32_t)(T[base] - start);
        if (tl == 0) return (((base + 1) << 16) | flag(start, base + 1, false, 0)) - off;  // threshold on the start
        return ((base << 16) | ((0x4000u - tl) << 2) | flag(start, base, true, T[base])) - off;
      }
    } else {  // fp64: bit 14 marks a leaf not proven violation-free (the kernel ORs it)
      if (n == 0) return (base << 16) | (flag(start, base, false, 0) << 14);
      if (n == 1) return (base << 16) | 1u | (flag(start, base, true, T[base]) << 14);
    }
    uint32_t ns = s >= 4 ? s - 4 : 0;
    uint32_t id = n_sub++;
    size_t off = sub.size();
    sub.resize(off + kSubFan);
    for (uint32_t i = 0; i < (uint32_t)kSubFan; ++i) {
      uint32_t ent;
      if (s >= 4) {
        ent = make(start + ((uint64_t)i << ns), ns);
      } else {
        uint64_t v = (start & ~15ull) | i;
        if (v >= start && v < end) ent = make(v, 0);
        else ent = (lb(v) << 16) - (f32 ? (uint32_t)v << 2 : 0u);  // unreachable slot (never indexed)
      }
      sub[off + i] = ent;
    }
    if (f32) {  // the sub-table's byte offset in the LUT, so the kernel forms its address with adds
      const uint64_t off = ((uint64_t)sub0 + (uint64_t)id * kSubFan) * 4u;
      if (off >= (1ull << 25)) too_big = true;
      return ((uint32_t)off << 7) | (ns << 2) | kRedirect32;
    }
    return (id << 16) | kRedirect | ns;
  }
};

// Level-1 shift search + build for one LUT size (budgets in 32-bit entries).
std::string build_lut(const Tables& t, const std::vector<uint64_t>& T, bool f32, uint32_t level1_max,
                      uint32_t total_budget, Tables::Lut& out) {
  // fp32: level-1 buckets k = (bits >> S1) - KBASE with an empty guard bucket below the first
  // threshold and one above the last (the kernel clamps k, not the cap). fp64: clamp the cap.
  const uint32_t width = f32 ? 32 : 64;
  auto range = [&](uint32_t s, uint64_t* kb, uint64_t* nb) -> bool {
    if (f32) {
      // s >= 1 keeps ((int32)bits >> s) - KBASE free of int32 overflow for sign-bit patterns
      if (s == 0 || (T.front() >> s) == 0) return false;  // and leaves room for the guard bucket
      *kb = (T.front() >> s) - 1;
      *nb = (T.back() >> s) - *kb + 2;
    } else {
      *kb = (uint64_t)t.lo >> s;
      *nb = ((uint64_t)t.hi >> s) - *kb + 1;
    }
    return true;
  };
  // The finest level 1 whose LUT fits the budget; when none does (many grids: thousands of
  // thresholds), the finest one within 12 % of the smallest LUT — a coarse level 1 of similar
  // size sends nearly every cap through 2-3 sub-table levels (C3: shift 17 vs 12, 1.38x slower).
  uint32_t best_s = width - 2;
  size_t best_total = ~(size_t)0;
  bool fits = false;
  std::vector<std::pair<uint32_t, size_t>> cand;  // (shift, total) of the valid shifts
  // (fp32 shifts start at 6: the kernel's first sub-table step shifts the cap by S1 - 6 >= 0)
  for (uint32_t s = f32 ? 6u : 0u; s + 1 < width; ++s) {
    if (f32 && s > kMaxShift32) break;
    uint64_t kb, nb;
    // fp32 buckets stop at shift 14 (the leaf's K): thresholds spread over more than ~16 octaves
    // take a longer level 1 at shift 14 instead of a coarser one
    if (!range(s, &kb, &nb) || (nb > level1_max && !(f32 && s == kMaxShift32 && cand.empty()))) continue;
    LutBuilder lbld(T, f32, nullptr, (uint32_t)nb);
    for (uint64_t k = 0; k < nb; ++k) lbld.make((kb + k) << s, s);
    const size_t total = nb + lbld.sub.size();
    if (f32 && lbld.n_sub > kMaxSub32) continue;
    cand.emplace_back(s, total);
    if (total < best_total) best_total = total, best_s = s;
    if (total <= total_budget) {
      best_s = s;
      fits = true;
      break;
    }
  }
  if (!fits)
    for (const auto& c : cand)
      if ((double)c.second <= 1.12 * (double)best_total) {
        best_s = c.first;
        break;
      }
  if (const char* e = std::getenv("CS_LUT_FORCE_SHIFT")) best_s = (uint32_t)std::atoi(e);  // tuning only
  const uint32_t s = best_s;
  uint64_t kb, nb;
  if (!range(s, &kb, &nb)) return "power thresholds too small for the fp32 LUT (need bits > 2^S1)";
  LutBuilder lbld(T, f32, &t.vio, (uint32_t)nb);
  out.kbase = kb;
  std::vector<uint32_t> level1(nb);
  for (uint64_t k = 0; k < nb; ++k) level1[k] = lbld.make((kb + k) << s, s);
  if (f32 && (lbld.n_sub > kMaxSub32 || lbld.too_big)) return "threshold LUT needs more than 32768 sub-tables";
  if (lbld.n_sub > 65535) return "threshold LUT needs more than 65535 sub-tables";
  out.shift1 = s;
  out.n_level1 = (uint32_t)nb;
  out.n_sub = lbld.n_sub;
  out.n_unsafe = lbld.unsafe;
  out.lut = std::move(level1);
  out.lut.insert(out.lut.end(), lbld.sub.begin(), lbld.sub.end());
  return std::string();
}

}  // namespace

std::string build_tables(const cs_grid_desc* grids, int32_t n_grids, int32_t cap_dtype, int32_t batching_mtl,
                         int32_t mt_bs, Tables& out) {
  if (cap_dtype != CS_CAP_F32 && cap_dtype != CS_CAP_F64) return "cap_dtype must be CS_CAP_F32 or CS_CAP_F64";
  if (n_grids < 1 || grids == nullptr) return "need at least one grid";
  const bool f32 = cap_dtype == CS_CAP_F32;
  Tables& t = out;
  t.cap_dtype = cap_dtype;
  t.M = n_grids;
  t.batching_mtl = batching_mtl;
  t.mt_bs = mt_bs;

  std::vector<std::vector<Entry>> sorted(n_grids);
  std::vector<std::vector<uint64_t>> gthr(n_grids);
  std::set<uint64_t> uni;
  t.e_off.assign(1, 0);
  for (int g = 0; g < n_grids; ++g) {
    const cs_grid_desc& d = grids[g];
    if (d.n_entries < 1) return "grid " + std::to_string(g) + " has no entries";
    if (!d.mtl || !d.bs || !d.throughput_ips || !d.power_w) return "null grid array";
    std::vector<Entry>& es = sorted[g];
    es.resize(d.n_entries);
    std::set<std::pair<int32_t, int32_t>> seen;
    for (int i = 0; i < d.n_entries; ++i) {
      Entry& e = es[i];
      e.mtl = d.mtl[i];
      e.bs = d.bs[i];
      e.thr = d.throughput_ips[i];
      e.pw = d.power_w[i];
      e.idx = i;
      if (e.mtl < 1 || e.bs < 1) return "mtl and bs must be >= 1";
      if (!(std::isfinite(e.thr) && e.thr > 0)) return "throughput must be positive";
      if (!(std::isfinite(e.pw) && e.pw > 0)) return "power must be positive";
      if (!seen.insert({e.mtl, e.bs}).second) return "duplicate config in grid " + std::to_string(g);
      e.key = f32 ? (uint64_t)f32_bits(roundup_f32(e.pw)) : f64_bits(e.pw);
      t.e_mtl.push_back(e.mtl);
      t.e_bs.push_back(e.bs);
      t.e_thr.push_back(e.thr);
      t.e_pw.push_back(e.pw);
    }
    t.e_off.push_back((int32_t)t.e_mtl.size());
    // policy.py:129 — strict total order since (mtl, bs) is unique
    std::sort(es.begin(), es.end(), [](const Entry& a, const Entry& b) {
      if (a.pw != b.pw) return a.pw < b.pw;
      if (a.mtl != b.mtl) return a.mtl < b.mtl;
      return a.bs < b.bs;
    });
    for (const Entry& e : es) {
      if (gthr[g].empty() || gthr[g].back() != e.key) gthr[g].push_back(e.key);
      uni.insert(e.key);
    }
    t.idle_pw.push_back(std::isnan(d.idle_power_w) ? 0.0 : d.idle_power_w);
  }
  t.thresholds.assign(uni.begin(), uni.end());
  const int64_t D = (int64_t)t.thresholds.size();
  if (D + 1 > 65536) return "more than 65535 distinct power thresholds across grids";
  t.U = (int32_t)(D + 1);
  t.maxB = 0;
  t.grid_bins.resize(n_grids);
  for (int g = 0; g < n_grids; ++g) {
    t.grid_bins[g] = (int32_t)gthr[g].size() + 1;
    t.maxB = std::max(t.maxB, t.grid_bins[g]);
  }
  const int32_t maxB = t.maxB;
  t.sel.assign((size_t)n_grids * 3 * maxB, -1);
  t.cnt.assign((size_t)n_grids * 3 * maxB, 0);
  t.sthr.assign((size_t)n_grids * 3 * maxB, 0.0);
  t.spw.assign((size_t)n_grids * 3 * maxB, 0.0);
  t.umap.assign((size_t)n_grids * t.U, 0);
  t.sig.assign((size_t)n_grids * t.U, 0);
  t.vio.assign((size_t)t.U, 0);

  for (int g = 0; g < n_grids; ++g) {
    const std::vector<Entry>& es = sorted[g];
    const int B = t.grid_bins[g];
    // walk the combination order once, recording every regime's prefix best/count at the end
    // of each distinct threshold (= at each grid bin boundary)
    int best[3] = {-1, -1, -1};
    int64_t cnt[3] = {0, 0, 0};
    size_t i = 0;
    for (int b = 1; b < B; ++b) {
      const uint64_t th = gthr[g][b - 1];
      for (; i < es.size() && es[i].key <= th; ++i) {
        for (int p = 0; p < 3; ++p) {
          if (!in_regime(p, es[i], batching_mtl, mt_bs)) continue;
          ++cnt[p];
          if (best[p] < 0 || !prefer(es[best[p]], es[i])) best[p] = (int)i;
        }
      }
      for (int p = 0; p < 3; ++p) {
        size_t o = ((size_t)g * 3 + p) * maxB + b;
        t.cnt[o] = cnt[p];
        if (best[p] >= 0) {
          const Entry& e = es[best[p]];
          t.sel[o] = e.idx;
          t.sthr[o] = e.thr;
          t.spw[o] = e.pw;
        }
      }
    }
    // union bin -> grid bin, and segment ids (a policy switches configs between two steps iff
    // their segment ids differ: prefix-best never returns to an earlier entry)
    int32_t seg[3] = {0, 0, 0};
    std::vector<uint64_t> gsig(B, 0);
    for (int b = 1; b < B; ++b) {
      for (int p = 0; p < 3; ++p) {
        size_t o = ((size_t)g * 3 + p) * maxB;
        if (t.sel[o + b] != t.sel[o + b - 1]) ++seg[p];
      }
      gsig[b] = (uint64_t)seg[0] | ((uint64_t)seg[1] << 16) | ((uint64_t)seg[2] << 32);
    }
    size_t j = 0;
    for (int u = 0; u < t.U; ++u) {
      if (u > 0) {
        const uint64_t th = t.thresholds[u - 1];
        while (j < gthr[g].size() && gthr[g][j] <= th) ++j;
      }
      uint16_t gb = (uint16_t)j;
      t.umap[(size_t)g * t.U + u] = gb;
      t.sig[(size_t)g * t.U + u] = gsig[gb];
      // violation floor: the largest selected power among this grid's 3 policies
      for (int p = 0; p < 3; ++p) {
        size_t o = ((size_t)g * 3 + p) * maxB + gb;
        if (t.sel[o] < 0) continue;
        uint64_t k = f32 ? (uint64_t)f32_bits(roundup_f32(t.spw[o])) : f64_bits(t.spw[o]);
        t.vio[u] = std::max(t.vio[u], k);
      }
    }
  }

  // ---- sampling selector tables (policy.py:191-273): the combination order (= the sorted
  // feasible list, policy.py:246), the combination count per grid bin, and each entry's
  // present-entry neighbourhood (policy.py:200-215: mtl -/+ 1 at the same bs, then the nearest
  // present bs to bs/2 and bs*2 at the same mtl, ties to the smaller bs).
  t.csort.clear();
  t.nbr.clear();
  t.ccnt.assign((size_t)n_grids * maxB, 0);
  for (int g = 0; g < n_grids; ++g) {
    for (const Entry& e : sorted[g]) t.csort.push_back(e.idx);
    for (int b = 0; b < maxB; ++b) t.ccnt[(size_t)g * maxB + b] = (int32_t)t.cnt[((size_t)g * 3 + 2) * maxB + b];
    const cs_grid_desc& d = grids[g];
    std::map<std::pair<int32_t, int32_t>, int32_t> at;
    std::map<int32_t, std::vector<int32_t>> bs_at;
    for (int i = 0; i < d.n_entries; ++i) {
      at[{d.mtl[i], d.bs[i]}] = i;
      bs_at[d.mtl[i]].push_back(d.bs[i]);
    }
    auto find = [&](int32_t m, int32_t b) {
      auto it = at.find({m, b});
      return it == at.end() ? -1 : it->second;
    };
    for (int i = 0; i < d.n_entries; ++i) {
      int32_t nb[4] = {-1, -1, -1, -1};
      int k = 0;
      for (int32_t m : {d.mtl[i] - 1, d.mtl[i] + 1}) {
        const int e = m >= 1 ? find(m, d.bs[i]) : -1;
        if (e >= 0) nb[k++] = e;
      }
      for (double target : {(double)d.bs[i] / 2.0, (double)d.bs[i] * 2.0}) {
        int32_t best = -1;
        double bd = 0.0;
        for (int32_t b : bs_at[d.mtl[i]]) {
          if (b == d.bs[i]) continue;
          const double dist = std::fabs((double)b - target);
          if (best < 0 || dist < bd || (dist == bd && b < best)) best = b, bd = dist;
        }
        if (best < 0) continue;
        const int e = find(d.mtl[i], best);
        if (e >= 0 && std::find(nb, nb + k, e) == nb + k) nb[k++] = e;
      }
      t.nbr.insert(t.nbr.end(), nb, nb + 4);
    }
  }

  // ---- selection segments: maximal runs of union bins sharing a selection, per (grid, policy).
  // The epilogue sums count x value once per segment instead of once per bin.
  t.seg_off.assign(1, 0);
  for (int g = 0; g < n_grids; ++g) {
    for (int p = 0; p < 3; ++p) {
      int u = 0;
      while (u < t.U) {
        const uint64_t sid = (t.sig[(size_t)g * t.U + u] >> (16 * p)) & 0xFFFFull;
        int v = u;
        while (v + 1 < t.U && ((t.sig[(size_t)g * t.U + v + 1] >> (16 * p)) & 0xFFFFull) == sid) ++v;
        t.seg.insert(t.seg.end(), {u, v, (int32_t)t.umap[(size_t)g * t.U + u], 0});
        u = v + 1;
      }
      t.seg_off.push_back((int32_t)(t.seg.size() / 4));
    }
  }

  // ---- LUT over the union thresholds ----
  // Two sizes: the default LUT (every kernel) and, when a finer level 1 exists, a big one that
  // eval_kernel takes whenever it fits in shared memory without costing resident warps (fewer
  // multi-threshold buckets -> fewer warps on the redirect path).
  const std::vector<uint64_t>& T = t.thresholds;
  t.lo = (int64_t)T.front() - 1;
  t.hi = (int64_t)T.back();
  uint32_t l1max = 8192;
  if (const char* e = std::getenv("CS_LUT_LEVEL1_MAX")) l1max = (uint32_t)std::atoi(e);  // tuning only
  std::string err = build_lut(t, T, f32, l1max, l1max + l1max / 2, t.lut_main);
  if (!err.empty()) return err;
  if (f32) {
    err = build_lut(t, T, f32, 20480, 24576, t.lut_big);
    if (!err.empty() || t.lut_big.shift1 >= t.lut_main.shift1) t.lut_big = Tables::Lut{};
    // (many grids: with thousands of thresholds the default and big budgets take the same coarse
    // level 1; a 36k-entry LUT fits next to 8-warp groups once their trace histograms go straight
    // to global memory — C3 5.86 -> 5.50 ms at shift 11)
    const uint32_t cur = t.lut_big.lut.empty() ? t.lut_main.shift1 : t.lut_big.shift1;
    err = build_lut(t, T, f32, 20480, 36864, t.lut_huge);
    if (!err.empty() || t.lut_huge.shift1 >= cur) t.lut_huge = Tables::Lut{};
  }
  if (f32 && t.U > 0xFFF0) return "more than 65519 distinct power thresholds across grids";
  t.kbase = t.lut_main.kbase;
  t.shift1 = t.lut_main.shift1;
  t.n_level1 = t.lut_main.n_level1;
  t.n_sub = t.lut_main.n_sub;
  t.n_unsafe = t.lut_main.n_unsafe;
  t.lut = t.lut_main.lut;
  return std::string();
}

}  // namespace cs
