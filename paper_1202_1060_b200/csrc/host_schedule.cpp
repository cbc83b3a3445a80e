// host_schedule.cpp -- CN-group schedules and their derived tables.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>

#include "host.hpp"
#include "rng.cuh"

namespace ldpcb {

// Flattens the groups and derives, per group, the sorted set of VNs whose
// messages the sub-iteration refreshes (decoder.hpp:115-120): the B200
// kernels read these tables instead of sorting on the fly.
ScheduleData schedule_from_groups(const CodeData& c, Kind kind, const Rows& groups) {
  if (groups.empty()) throw std::invalid_argument("schedule needs at least one group");
  ScheduleData s;
  s.kind = kind;
  s.G = static_cast<int>(groups.size());
  s.grp_off.assign(1, 0);
  s.touch_off.assign(1, 0);
  std::vector<char> mark(c.n, 0);
  std::vector<int32_t> vns;
  for (const auto& g : groups) {
    vns.clear();
    for (int r : g) {
      if (r < 0 || r >= c.m) throw std::invalid_argument("group CN index out of range");
      s.grp_cns.push_back(r);
      s.edge_updates_per_iter += c.row_off[r + 1] - c.row_off[r];
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e)
        if (!mark[c.cols[e]]) {
          mark[c.cols[e]] = 1;
          vns.push_back(c.cols[e]);
        }
    }
    std::sort(vns.begin(), vns.end());
    for (int v : vns) mark[v] = 0;
    s.touch_vns.insert(s.touch_vns.end(), vns.begin(), vns.end());
    s.grp_off.push_back(static_cast<int32_t>(s.grp_cns.size()));
    s.touch_off.push_back(static_cast<int32_t>(s.touch_vns.size()));
    s.touched_per_iter += static_cast<int64_t>(vns.size());
    s.max_group = std::max(s.max_group, static_cast<int>(g.size()));
    s.max_touched = std::max(s.max_touched, static_cast<int>(vns.size()));
  }
  s.group_size = s.max_group;
  return s;
}

ScheduleData flooding_schedule(const CodeData& c) {
  Rows g(1, std::vector<int>(c.m));
  for (int r = 0; r < c.m; ++r) g[0][r] = r;
  return schedule_from_groups(c, Kind::flooding, g);
}

// The reference's random grouping (schedule.hpp:54-115): a shuffled pool;
// with r == 0 a balanced partition, otherwise the sequential construction
// where group g reuses k = round(N_G r) CNs of (group g-1 minus group g-2).
Rows random_groups(int M, int G, double overlap, uint64_t seed_value) {
  Stream rng(seed_value);
  std::vector<int> pool(M);
  for (int i = 0; i < M; ++i) pool[i] = i;
  rng.permute(pool.data(), static_cast<uint64_t>(M));
  Rows groups(G);
  if (overlap == 0.0) {
    const int base = M / G, extra = M % G;
    size_t at = 0;
    for (int g = 0; g < G; ++g) {
      const int sz = base + (g < extra ? 1 : 0);
      groups[g].assign(pool.begin() + at, pool.begin() + at + sz);
      at += sz;
    }
    return groups;
  }
  const double denom = G - (G - 1) * overlap;
  const int nominal = static_cast<int>(std::ceil(M / denom));
  const int k = static_cast<int>(std::llround(nominal * overlap));
  if (G > 1 && 2 * k > nominal)
    throw std::invalid_argument("infeasible (G, r): overlap " + std::to_string(k) + " exceeds the fresh half of N_G=" +
                                std::to_string(nominal));
  size_t at = 0;
  auto fresh = [&](int want) {
    const int got = std::min<int>(want, static_cast<int>(pool.size() - at));
    std::vector<int> out(pool.begin() + at, pool.begin() + at + got);
    at += got;
    return out;
  };
  groups[0] = fresh(nominal);
  if (static_cast<int>(groups[0].size()) < std::min(nominal, M))
    throw std::invalid_argument("infeasible (G, r): first group cannot be filled");
  for (int g = 1; g < G; ++g) {
    std::vector<int> cand;
    if (g == 1) {
      cand = groups[0];
    } else {
      const auto& pp = groups[g - 2];
      for (int cn : groups[g - 1])
        if (std::find(pp.begin(), pp.end(), cn) == pp.end()) cand.push_back(cn);
    }
    rng.permute(cand.data(), cand.size());
    const int take = std::min<int>(k, static_cast<int>(cand.size()));
    groups[g].assign(cand.begin(), cand.begin() + take);
    int want = nominal - take;
    if (g == G - 1) want = static_cast<int>(pool.size() - at);
    auto f = fresh(want);
    if (g < G - 1 && static_cast<int>(f.size()) < want)
      throw std::invalid_argument("infeasible (G, r): fresh pool exhausted at group " + std::to_string(g + 1));
    groups[g].insert(groups[g].end(), f.begin(), f.end());
    if (groups[g].empty()) throw std::invalid_argument("infeasible (G, r): empty group " + std::to_string(g + 1));
  }
  if (at != pool.size()) throw std::invalid_argument("infeasible (G, r): groups do not cover all CNs");
  return groups;
}

// make_disjoint_schedule / make_nondisjoint_schedule (schedule.hpp:136-171)
// with the stored grouping only (the per-iteration regroup stream is not
// part of the uploaded-once device schedule).
ScheduleData reference_random_schedule(const CodeData& c, Kind kind, int G, double overlap, uint64_t seed) {
  if (G < 1 || G > c.m) throw std::invalid_argument("need 1 <= G <= M");
  if (kind == Kind::disjoint) overlap = 0.0;
  if (!(overlap >= 0.0) || overlap >= 1.0) throw std::invalid_argument("need 0 <= r < 1");
  ScheduleData s = schedule_from_groups(c, kind, random_groups(c.m, G, overlap, stream_seed(seed, 1)));
  s.overlap = overlap;
  s.seed = seed;
  if (kind == Kind::disjoint)
    s.group_size = (c.m + G - 1) / G;
  else
    s.group_size = static_cast<int>(std::ceil(c.m / (G - (G - 1) * overlap)));
  return s;
}

ScheduleData per_frame_schedule(const CodeData& c, Kind kind, int G, double overlap, uint64_t schedule_seed,
                                bool regroup) {
  if (kind == Kind::flooding) return flooding_schedule(c);
  ScheduleData s = reference_random_schedule(c, kind, G, overlap, stream_seed(schedule_seed, 0));
  s.seed = schedule_seed;
  s.per_frame = true;
  s.regroup = regroup;
  if (s.overlap != 0.0) {
    const double denom = G - (G - 1) * s.overlap;
    s.nominal = static_cast<int>(std::ceil(c.m / denom));
    s.k_overlap = static_cast<int>(std::llround(s.nominal * s.overlap));
  }
  return s;
}

// Fixed windows: group g = CNs (g*stride + j) mod M for j < window, in that
// order (BASELINE: 8 windows of 84 at stride 63 on M=504; 45 x 960 at 720).
ScheduleData window_schedule(const CodeData& c, Kind kind, int G, int window, int stride) {
  if (G < 1 || window < 1 || stride < 0 || window > c.m)
    throw std::invalid_argument("need G >= 1, 1 <= window <= M, stride >= 0");
  Rows groups(G, std::vector<int>(window));
  for (int g = 0; g < G; ++g)
    for (int j = 0; j < window; ++j)
      groups[g][j] = static_cast<int>((static_cast<long long>(g) * stride + j) % c.m);
  ScheduleData s = schedule_from_groups(c, kind, groups);
  s.group_size = window;
  s.overlap = window > stride ? static_cast<double>(window - stride) / window : 0.0;
  return s;
}

// Complexity-fair cap floor(M I / (M + (G-1) N_G r)) (schedule.hpp:206-210)
int iteration_budget(const ScheduleData& s, int n_checks, int i_max) {
  if (s.kind != Kind::nondisjoint || s.overlap == 0.0) return i_max;
  const double extra = (s.G - 1) * static_cast<double>(s.group_size) * s.overlap;
  return static_cast<int>(std::floor(static_cast<double>(n_checks) * i_max / (n_checks + extra)));
}

namespace {

// Shared-memory bank colouring. A warp of the resident kernel (two frames
// per CTA) works on 16 consecutive items of a list per half-warp, and each
// instruction gathers or scatters one 64-bit frame-interleaved element per
// item: elements whose index is equal mod 16 fall in the same banks and
// serialise. The annealers below reorder what is free to reorder so that,
// per (16-item block, column), few items share a colour:
//  * the edges of each CN (boxplus is symmetric): columns are the record
//    positions, colour = VN mod 16, for the gathers of P and, separately, the
//    in-place stores of single-touch posteriors;
//  * the items of VN-record lists (fix-ups, exact totals): columns are L/P of
//    the VN and each c2v slot, colour = slot mod 16.
// Cost = sum over cells of the largest colour count (duplicates counted, a
// slight overestimate). Deterministic (fixed seeds, fixed move counts).
constexpr int kBankBlock = 16, kColours = 16;

struct ColourCells {
  int cols;
  std::vector<uint8_t> cnt;  // [cell][colour]
  std::vector<int> best;     // [cell]
  ColourCells(int cells, int cols_) : cols(cols_), cnt(static_cast<size_t>(cells) * kColours, 0), best(cells, 0) {}
  int max_of(int cell) const {
    int m = 0;
    for (int k = 0; k < kColours; ++k) m = std::max<int>(m, cnt[cell * kColours + k]);
    return m;
  }
};

// Layout chosen by the annealer below: the record order of every CN's edges
// and the shared-memory colour of every VN.
struct BankLayout {
  std::vector<int> perm;    // perm[off + p] = original edge index (relative to the row) at record position p
  std::vector<int> colour;  // colour[v] = shared-memory position of VN v mod 16
};

// Joint annealing of (1) the edge order inside each CN (boxplus is
// symmetric) and (2) the colour of each VN: its position in the P / L arrays
// is colour + 16 * rank, so colour classes keep the sizes of v mod 16 and
// the positions stay a permutation of [0, n). Moves swap two edges of a CN
// or the colours of two VNs.
BankLayout bank_layout(const CodeData& c, const std::vector<std::vector<int>>& group_cns,
                       const std::vector<std::vector<char>>& single) {
  BankLayout L;
  L.perm.resize(c.E);
  L.colour.resize(c.n);
  for (int r = 0; r < c.m; ++r)
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) L.perm[e] = e - c.row_off[r];
  for (int v = 0; v < c.n; ++v) L.colour[v] = v % kColours;
  if (c.n > 32768 || c.m < 2) return L;
  std::vector<int>& perm = L.perm;
  std::vector<int>& col = L.colour;
  const int D = c.max_cdeg;
  // (group, block) of every CN occurrence
  struct Occ {
    int cell0;  // first cell of its block: cells [cell0, cell0 + 2D) = D gather + D store columns
    int group;
  };
  std::vector<std::vector<Occ>> occ(c.m);
  int nblocks = 0;
  for (int g = 0; g < static_cast<int>(group_cns.size()); ++g)
    for (int j = 0; j < static_cast<int>(group_cns[g].size()); ++j) {
      if (j % kBankBlock == 0) ++nblocks;
      occ[group_cns[g][j]].push_back({(nblocks - 1) * 2 * D, g});
    }
  const int ncells = nblocks * 2 * D;
  // per cell: colour counts, a histogram of those counts and their maximum,
  // so every increment / decrement updates the total cost in O(1)
  constexpr int H = kBankBlock * 4 + 1;
  std::vector<uint8_t> cnt(static_cast<size_t>(ncells) * kColours, 0);
  std::vector<uint16_t> hist(static_cast<size_t>(ncells) * H, 0);
  std::vector<uint8_t> mx(ncells, 0);
  for (int i = 0; i < ncells; ++i) hist[static_cast<size_t>(i) * H] = kColours;
  long long total = 0;
  auto bump = [&](int cell, int k, int sign) {
    uint8_t& x = cnt[static_cast<size_t>(cell) * kColours + k];
    uint16_t* h = &hist[static_cast<size_t>(cell) * H];
    --h[x];
    x = static_cast<uint8_t>(x + sign);
    ++h[x];
    if (sign > 0 && x > mx[cell]) {
      mx[cell] = x;
      ++total;
    } else if (sign < 0 && h[mx[cell]] == 0) {
      --mx[cell];
      --total;
    }
  };
  // position of edge e inside its row's record (inverse of perm)
  std::vector<int> rpos(c.E), row_of(c.E);
  for (int r = 0; r < c.m; ++r)
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) {
      rpos[c.row_off[r] + perm[e]] = e - c.row_off[r];
      row_of[e] = r;
    }
  auto vn_at = [&](int r, int p) { return c.cols[c.row_off[r] + perm[c.row_off[r] + p]]; };
  auto add = [&](int r, int p, int v, int sign) {
    const int k = col[v];
    for (const Occ& o : occ[r]) {
      bump(o.cell0 + p, k, sign);
      if (single[o.group][v]) bump(o.cell0 + D + p, k, sign);
    }
  };
  for (int r = 0; r < c.m; ++r)
    for (int p = 0; p < c.row_off[r + 1] - c.row_off[r]; ++p) add(r, p, vn_at(r, p), +1);
  const long long c0 = total;
  const BankLayout initial = L;  // structured codes (QC) may start out conflict-free
  Stream rng(0x6c64706362616e6bull);
  static const long long scale = [] {
    const char* e = std::getenv("LDPCB_BANK_ITERS");  // moves per CN; tuning / A-B only
    return e ? std::atoll(e) : 4000ll;
  }();
  const long long iters = std::min<long long>(20000000, scale * c.m);
  auto swap_edges = [&](int r, int p1, int p2) {
    const int v1 = vn_at(r, p1), v2 = vn_at(r, p2);
    add(r, p1, v1, -1);
    add(r, p2, v2, -1);
    std::swap(perm[c.row_off[r] + p1], perm[c.row_off[r] + p2]);
    rpos[c.row_off[r] + perm[c.row_off[r] + p1]] = p1;
    rpos[c.row_off[r] + perm[c.row_off[r] + p2]] = p2;
    add(r, p1, v2, +1);
    add(r, p2, v1, +1);
  };
  auto vn_add = [&](int v, int sign) {
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {
      const int e = c.var_edges[j];
      add(row_of[e], rpos[e], v, sign);
    }
  };
  auto swap_colours = [&](int v1, int v2) {
    vn_add(v1, -1);
    vn_add(v2, -1);
    std::swap(col[v1], col[v2]);
    vn_add(v1, +1);
    vn_add(v2, +1);
  };
  long long best_total = total;
  BankLayout best = L;
  for (long long it = 0; it < iters; ++it) {
    const double T = 1.0 * (1.0 - static_cast<double>(it) / iters) + 0.02;
    const long long before = total;
    if (rng.below(2) == 0) {  // swap two edges of a CN
      const int r = static_cast<int>(rng.below(c.m));
      const int deg = c.row_off[r + 1] - c.row_off[r];
      if (deg < 2 || occ[r].empty() || occ[r].size() > 16) continue;
      const int p1 = static_cast<int>(rng.below(deg));
      int p2 = static_cast<int>(rng.below(deg - 1));
      if (p2 >= p1) ++p2;
      swap_edges(r, p1, p2);
      const long long d = total - before;
      if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_edges(r, p1, p2);
    } else {  // swap the colours of two VNs
      const int v1 = static_cast<int>(rng.below(c.n)), v2 = static_cast<int>(rng.below(c.n));
      if (col[v1] == col[v2]) continue;
      swap_colours(v1, v2);
      const long long d = total - before;
      if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_colours(v1, v2);
    }
    if (total < best_total && it > iters / 2) {
      best_total = total;
      best = L;
    }
  }
  if (total > best_total) {
    L = best;
    total = best_total;
  }
  if (std::getenv("LDPCB_BANK_DEBUG"))
    std::fprintf(stderr, "bank_layout: %d cells, cost %.3f -> %.3f per cell (%lld moves)\n", ncells,
                 static_cast<double>(c0) / ncells, static_cast<double>(total) / ncells, iters);
  return total <= c0 ? L : initial;
}

void bank_order_vns(std::vector<int>& vns, int begin, int end, const CodeData& c, const std::vector<int>& edge_slot,
                    const std::vector<int>& vcol, uint64_t seed) {
  const int count = end - begin;
  if (count <= kBankBlock || c.n > 32768) return;
  const int cols = 1 + c.max_vdeg;
  auto colour = [&](int v, int q) {  // q = 0: L/P of v, else the (q-1)-th c2v slot (-1: none)
    if (q == 0) return vcol[v];
    const int j = c.var_off[v] + q - 1;
    return j < c.var_off[v + 1] ? edge_slot[c.var_edges[j]] % kColours : -1;
  };
  const int nblocks = (count + kBankBlock - 1) / kBankBlock;
  ColourCells cc(nblocks * cols, cols);
  auto add = [&](int i, int sign) {
    const int v = vns[begin + i], b = i / kBankBlock;
    for (int q = 0; q < cols; ++q) {
      const int k = colour(v, q);
      if (k >= 0) cc.cnt[(b * cols + q) * kColours + k] += sign;
    }
  };
  for (int i = 0; i < count; ++i) add(i, +1);
  long long total = 0;
  for (int i = 0; i < nblocks * cols; ++i) total += (i % cols == 0 ? 2 : 1) * (cc.best[i] = cc.max_of(i));
  const long long c0 = total;
  const std::vector<int> initial(vns.begin() + begin, vns.begin() + end);
  Stream rng(seed);
  const long long iters = 100ll * count;
  std::vector<int> fresh(2 * cols);
  for (long long it = 0; it < iters; ++it) {
    const double T = 2.0 * (1.0 - static_cast<double>(it) / iters) + 0.02;
    const int i1 = static_cast<int>(rng.below(count)), i2 = static_cast<int>(rng.below(count));
    const int b1 = i1 / kBankBlock, b2 = i2 / kBankBlock;
    if (b1 == b2) continue;
    int old = 0;
    for (int q = 0; q < cols; ++q) old += (q == 0 ? 2 : 1) * (cc.best[b1 * cols + q] + cc.best[b2 * cols + q]);
    add(i1, -1);
    add(i2, -1);
    std::swap(vns[begin + i1], vns[begin + i2]);
    add(i1, +1);
    add(i2, +1);
    int now = 0;
    for (int q = 0; q < cols; ++q) {
      fresh[2 * q] = cc.max_of(b1 * cols + q);
      fresh[2 * q + 1] = cc.max_of(b2 * cols + q);
      now += (q == 0 ? 2 : 1) * (fresh[2 * q] + fresh[2 * q + 1]);  // L load + P store
    }
    const int d = now - old;
    if (d <= 0 || rng.unit() < std::exp(-d / T)) {
      for (int q = 0; q < cols; ++q) {
        cc.best[b1 * cols + q] = fresh[2 * q];
        cc.best[b2 * cols + q] = fresh[2 * q + 1];
      }
      total += d;
    } else {
      add(i1, -1);
      add(i2, -1);
      std::swap(vns[begin + i1], vns[begin + i2]);
      add(i1, +1);
      add(i2, +1);
    }
  }
  if (std::getenv("LDPCB_BANK_DEBUG"))
    std::fprintf(stderr, "bank_order_vns: %d items, cost %.3f -> %.3f per block\n", count,
                 static_cast<double>(c0) / nblocks, static_cast<double>(total) / nblocks);
  if (total > c0) std::copy(initial.begin(), initial.end(), vns.begin() + begin);
}

}  // namespace

KernelTables kernel_tables(const CodeData& c, const ScheduleData& s, int cs, bool regular_rows) {
  const bool packed = cs == 4 && regular_rows && c.max_cdeg <= 6 && c.n < 65536;  // common.cuh CnRecord
  if ((!packed && cs < 2 + c.max_cdeg) || cs % 4) throw std::invalid_argument("bad CN record stride");
  KernelTables t;
  t.cs = cs;
  t.vs4 = (1 + c.max_vdeg + 3) / 4;
  t.slot_stride = regular_rows ? (c.max_cdeg | 1) : 0;
  // irregular rows: CN r's slots start at slot_base[r], each CN holding an
  // odd number of slots (deg | 1), so consecutive CNs of one degree in a
  // warp hit distinct shared-memory banks (an even degree d would repeat
  // every 32 / gcd(2d, 32) CNs: 8-way conflicts for d = 8)
  std::vector<long long> slot_base(c.m + 1, 0);
  for (int r = 0; r < c.m; ++r) slot_base[r + 1] = slot_base[r] + ((c.row_off[r + 1] - c.row_off[r]) | 1);
  const long long slots = (t.slot_stride ? static_cast<long long>(c.m) * t.slot_stride : slot_base[c.m]) + 1;
  if (slots >= (1ll << 30)) throw std::invalid_argument("code too large for 32-bit edge records");
  t.n_slots = static_cast<int>(slots);
  const int zero = t.n_slots - 1;
  // groups without repeated CNs, and the VNs each group touches once
  std::vector<std::vector<int>> group_cns(s.G);
  std::vector<std::vector<char>> single(s.G);
  {
    std::vector<char> in_group(c.m, 0);
    std::vector<int> touches(c.n, 0);
    for (int g = 0; g < s.G; ++g) {
      auto& cns = group_cns[g];
      for (int i = s.grp_off[g]; i < s.grp_off[g + 1]; ++i) {
        const int r = s.grp_cns[i];
        if (in_group[r]) continue;
        in_group[r] = 1;
        cns.push_back(r);
      }
      for (int r : cns) {
        in_group[r] = 0;
        for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) ++touches[c.cols[e]];
      }
      single[g].assign(c.n, 0);
      for (int r : cns)
        for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) single[g][c.cols[e]] = touches[c.cols[e]] == 1;
      for (int r : cns)
        for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) touches[c.cols[e]] = 0;
    }
  }
  // record position of every edge (bank colouring), then its c2v slot
  const BankLayout lay = bank_layout(c, group_cns, single);
  const std::vector<int>& perm = lay.perm;
  // shared-memory position of every VN: colour + 16 * rank inside its colour
  t.vn_pos.resize(c.n);
  {
    std::vector<int> rank(kColours, 0);
    for (int v = 0; v < c.n; ++v) t.vn_pos[v] = lay.colour[v] + kColours * rank[lay.colour[v]]++;
  }
  const std::vector<int32_t>& vp = t.vn_pos;
  std::vector<int> pos(c.E);
  for (int r = 0; r < c.m; ++r)
    for (int p = 0; p < c.row_off[r + 1] - c.row_off[r]; ++p) pos[c.row_off[r] + perm[c.row_off[r] + p]] = p;
  t.edge_slot.resize(c.E);
  for (int r = 0; r < c.m; ++r)
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e)
      t.edge_slot[e] = static_cast<int>(t.slot_stride ? r * t.slot_stride + pos[e] : slot_base[r] + pos[e]);
  auto put_vn = [&](std::vector<int32_t>& out, int v) {
    out.push_back(vp[v]);
    int w = 1;
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j, ++w) out.push_back(t.edge_slot[c.var_edges[j]]);
    for (; w < 4 * t.vs4; ++w) out.push_back(zero);
  };
  // CN record [slot of position 0, single-touch mask by position, VNs by position]
  auto put_cn = [&](std::vector<int32_t>& out, int r, const std::vector<char>* one) {
    const int off = c.row_off[r], deg = c.row_off[r + 1] - off;
    uint32_t mask = 0;
    if (one)
      for (int p = 0; p < deg; ++p)
        if ((*one)[c.cols[off + perm[off + p]]]) mask |= 1u << p;
    const int slot = static_cast<int>(t.slot_stride ? r * t.slot_stride : slot_base[r]);
    if (packed) {  // {slot | mask << 24, v0 | v1 << 16, v2 | v3 << 16, v4 | v5 << 16}
      uint32_t w[4] = {static_cast<uint32_t>(slot) | (mask << 24), 0, 0, 0};
      for (int p = 0; p < deg; ++p)
        w[1 + p / 2] |= static_cast<uint32_t>(vp[c.cols[off + perm[off + p]]]) << (16 * (p & 1));
      for (uint32_t x : w) out.push_back(static_cast<int32_t>(x));
      return mask;
    }
    out.push_back(slot);
    out.push_back(static_cast<int32_t>(mask));
    for (int p = 0; p < deg; ++p) out.push_back(vp[c.cols[off + perm[off + p]]]);
    for (int k = 2 + deg; k < t.cs; ++k) out.push_back(-1);
    return mask;
  };
  // VN records (fix-ups, exact totals) grouped by VN degree, each run in
  // bank-coloured order: a warp's VNs then have one degree and its record
  // walk stops at the same padded row (decoder.cu vn_sum). Regular codes: one run.
  auto order_by_degree = [&](std::vector<int>& vns, uint64_t seed) {
    auto deg = [&](int v) { return c.var_off[v + 1] - c.var_off[v]; };
    std::stable_sort(vns.begin(), vns.end(), [&](int a, int b) { return deg(a) < deg(b); });
    for (int b = 0, e; b < static_cast<int>(vns.size()); b = e) {
      for (e = b + 1; e < static_cast<int>(vns.size()) && deg(vns[e]) == deg(vns[b]);) ++e;
      bank_order_vns(vns, b, e, c, t.edge_slot, lay.colour,
                     b == 0 ? seed : seed + static_cast<uint64_t>(deg(vns[b])) * 0x9e37ull);
    }
  };
  // 16-bit fix-up records: one 16-byte row holds a VN of degree <= 7
  if (t.vs4 > 1 && t.n_slots <= 65536 && c.n <= 65536) t.vs16 = (1 + c.max_vdeg + 7) / 8;
  auto put_vn16 = [&](std::vector<int32_t>& out, int v) {
    std::vector<uint32_t> f(8 * t.vs16, static_cast<uint32_t>(zero));
    f[0] = static_cast<uint32_t>(vp[v]);
    int w = 1;
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j, ++w) f[w] = static_cast<uint32_t>(t.edge_slot[c.var_edges[j]]);
    for (size_t i = 0; i < f.size(); i += 2) out.push_back(static_cast<int32_t>(f[i] | (f[i + 1] << 16)));
  };
  t.cn_off.assign(1, 0);
  t.fix_off.assign(1, 0);
  std::vector<int> touches(c.n, 0);
  std::vector<int> shared_vns;
  std::vector<char> processed(c.m, 0), touched(c.n, 0);  // fresh-frame bookkeeping (host.hpp)
  for (int g = 0; g < s.G; ++g) {
    const auto& cns = group_cns[g];
    for (int r : cns) t.recompute |= put_cn(t.cn_rec, r, &single[g]) != 0;
    for (int r : cns) {  // against the state before this group (Jacobi)
      const int off = c.row_off[r], deg = c.row_off[r + 1] - off;
      uint32_t f = processed[r] ? 0u : 1u << 31;
      for (int p = 0; p < deg && p < 31; ++p)
        if (!touched[c.cols[off + perm[off + p]]]) f |= 1u << p;
      t.cn_fresh.push_back(f);
    }
    for (int r : cns) {
      processed[r] = 1;
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) touched[c.cols[e]] = 1;
    }
    for (int r : cns)
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) ++touches[c.cols[e]];
    shared_vns.clear();
    for (int r : cns)
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) {
        const int v = c.cols[e];
        if (touches[v] >= 2) {
          shared_vns.push_back(v);
          touches[v] = -touches[v];  // list once
        }
      }
    for (int r : cns)
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) touches[c.cols[e]] = 0;
    std::sort(shared_vns.begin(), shared_vns.end());
    if (c.max_vdeg < 16) order_by_degree(shared_vns, 0x66697875ull + g);
    for (int v : shared_vns) put_vn(t.fix_rec, v);
    for (int v : shared_vns) {  // slot fields of CNs processed by the end of this group
      uint32_t f = 0;
      for (int j = c.var_off[v]; j < c.var_off[v + 1] && j - c.var_off[v] < 32; ++j)
        if (processed[c.var_cns[j]]) f |= 1u << (j - c.var_off[v]);
      t.fix_fresh.push_back(f);
    }
    if (t.vs16)
      for (int v : shared_vns) put_vn16(t.fix_rec16, v);
    t.cn_off.push_back(t.cn_off.back() + static_cast<int>(cns.size()));
    t.fix_off.push_back(t.fix_off.back() + static_cast<int>(shared_vns.size()));
    t.max_cn_items = std::max(t.max_cn_items, static_cast<int>(cns.size()));
    t.max_fix_items = std::max(t.max_fix_items, static_cast<int>(shared_vns.size()));
  }
  t.covers = c.max_vdeg <= 31 && c.max_cdeg <= 31 &&
             std::all_of(processed.begin(), processed.end(), [](char x) { return x != 0; }) &&
             std::all_of(touched.begin(), touched.end(), [](char x) { return x != 0; });
  // all_vn_rec is indexed by shared-memory position (the per-frame kernel
  // looks records up by the positions in its CN records)
  std::vector<int> all(c.n);
  for (int v = 0; v < c.n; ++v) all[vp[v]] = v;
  for (int v : all) put_vn(t.all_vn_rec, v);
  if (c.max_vdeg < 16) order_by_degree(all, 0x616c6cull);
  for (int v : all) put_vn(t.tot_vn_rec, v);
  if (t.vs16)
    for (int v : all) put_vn16(t.tot_rec16, v);
  for (int r = 0; r < c.m; ++r) put_cn(t.all_rec, r, nullptr);
  return t;
}

// VNs adjacent to both consecutive groups (schedule.hpp:175-201)
std::vector<int> measure_cocsg(const CodeData& c, const ScheduleData& s) {
  std::vector<int> out;
  std::vector<char> prev(c.n), seen(c.n);
  for (int t = 1; t < s.G; ++t) {
    std::fill(prev.begin(), prev.end(), 0);
    std::fill(seen.begin(), seen.end(), 0);
    for (int i = s.grp_off[t - 1]; i < s.grp_off[t]; ++i) {
      const int r = s.grp_cns[i];
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) prev[c.cols[e]] = 1;
    }
    int cnt = 0;
    for (int i = s.grp_off[t]; i < s.grp_off[t + 1]; ++i) {
      const int r = s.grp_cns[i];
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) {
        const int v = c.cols[e];
        if (prev[v] && !seen[v]) {
          seen[v] = 1;
          ++cnt;
        }
      }
    }
    out.push_back(cnt);
  }
  return out;
}

}  // namespace ldpcb
