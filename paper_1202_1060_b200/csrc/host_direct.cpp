// host_direct.cpp -- tables of the direct (posterior-free) resident kernel
// (direct.cu): cell assignment with shared-memory bank colouring and the
// per-group CN records. See host.hpp DirectTables for the formats.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "host.hpp"
#include "rng.cuh"

namespace ldpcb {

namespace {

constexpr int kColours = 16;  // 8-byte cells: a half-warp's 64-bit accesses cover the 32 banks once
constexpr int kLanes = 16;

// Colouring problem: every "set" lists the cells one shared-memory instruction
// of one half-warp touches; its cost is the largest number of cells sharing
// a colour (the wavefronts that instruction needs). Cells of one kind (c2v /
// L) swap colours, so each colour class keeps its size and the final cell
// id colour + 16 * rank stays a permutation of the kind's range.
struct SetCounts {
  std::vector<uint8_t> cnt;    // [set][colour]
  std::vector<uint16_t> hist;  // [set][count] -> colours with that count
  std::vector<uint8_t> mx;
  long long total = 0;  // sum over sets of the largest colour count: the wavefronts issued
  long long pairs = 0;  // sum over sets and colours of cnt (cnt - 1) / 2: the smooth annealing objective
  static constexpr int H = kLanes + 1;
  int add_set() {
    const int id = static_cast<int>(mx.size());
    mx.push_back(0);
    cnt.resize(cnt.size() + kColours, 0);
    hist.resize(hist.size() + H, 0);
    hist[static_cast<size_t>(id) * H] = kColours;
    return id;
  }
  void bump(int set, int k, int sign) {
    uint8_t& x = cnt[static_cast<size_t>(set) * kColours + k];
    uint16_t* h = &hist[static_cast<size_t>(set) * H];
    --h[x];
    pairs += sign > 0 ? x : -(x - 1);
    x = static_cast<uint8_t>(x + sign);
    ++h[x];
    if (sign > 0 && x > mx[set]) {
      mx[set] = x;
      ++total;
    } else if (sign < 0 && h[mx[set]] == 0) {
      --mx[set];
      --total;
    }
  }
};

}  // namespace

DirectTables direct_tables(const CodeData& c, const ScheduleData& s, int ng) {
  DirectTables t;
  t.ng = ng;
  if (s.per_frame || c.max_vdeg > 3 || c.max_cdeg != 6 || ng < 1 || ng > 3) return t;
  for (int r = 0; r < c.m; ++r)
    if (c.row_off[r + 1] - c.row_off[r] != 6) return t;
  const int E = c.E, n = c.n;
  const int l_base = (E + 15) / 16 * 16;
  const int cells = (l_base + (n + 15) / 16 * 16 + 1 + 15) / 16 * 16;
  if (cells * 8 > 65536) return t;
  // groups without repeated CNs (a second update of a CN inside a group would
  // read the same pre-group messages and write the same values)
  std::vector<std::vector<int>> group_cns(s.G);
  {
    std::vector<char> in_group(c.m, 0);
    for (int g = 0; g < s.G; ++g) {
      for (int i = s.grp_off[g]; i < s.grp_off[g + 1]; ++i) {
        const int r = s.grp_cns[i];
        if (in_group[r]) continue;
        in_group[r] = 1;
        group_cns[g].push_back(r);
      }
      for (int r : group_cns[g]) in_group[r] = 0;
      t.max_items = std::max(t.max_items, static_cast<int>(group_cns[g].size()));
    }
  }
  // the other two edges of every edge's VN, ascending CN order (-1: none)
  std::vector<int> oth_a(E, -1), oth_b(E, -1);
  for (int v = 0; v < n; ++v)
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {
      int* slot[2] = {&oth_a[c.var_edges[j]], &oth_b[c.var_edges[j]]};
      int w = 0;
      for (int i = c.var_off[v]; i < c.var_off[v + 1]; ++i)
        if (i != j) *slot[w++] = c.var_edges[i];
    }
  // ---- bank colouring: cells [0, E) = c2v of edge e, [E, E + n) = L of VN v.
  // The sets of a CN occurrence (a half-warp window of a group) are
  // set0 + 4 * position + {0 own c2v, 1 L, 2 first other c2v, 3 second}; the
  // record position of every edge inside its CN is free as well (boxplus is
  // symmetric), so moves swap the colours of two cells of a kind or the
  // positions of two edges of a CN.
  std::vector<int> colour(E + n), pos(E), row_of(E);
  for (int e = 0; e < E; ++e) colour[e] = e % kColours;
  for (int v = 0; v < n; ++v) colour[E + v] = v % kColours;
  for (int r = 0; r < c.m; ++r)
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) pos[e] = e - c.row_off[r], row_of[e] = r;
  SetCounts sc;
  std::vector<std::vector<int>> occ(c.m);  // CN -> set0 of each occurrence
  for (int g = 0; g < s.G; ++g) {
    const int cn = static_cast<int>(group_cns[g].size());
    for (int i0 = 0; i0 < ng * cn; i0 += kLanes) {  // one half-warp of CN items
      int set0 = -1;
      for (int q = 0; q < 24; ++q) {
        const int id = sc.add_set();
        if (q == 0) set0 = id;
      }
      for (int i = i0; i < std::min(ng * cn, i0 + kLanes); ++i) occ[group_cns[g][i % cn]].push_back(set0);
    }
  }
  // the four accesses of edge e's record position, in every occurrence of its CN
  auto edge_access = [&](int e, int sign) {
    const int v = c.cols[e];
    for (int set0 : occ[row_of[e]]) {
      const int b = set0 + 4 * pos[e];
      sc.bump(b, colour[e], sign);
      sc.bump(b + 1, colour[E + v], sign);
      if (oth_a[e] >= 0) sc.bump(b + 2, colour[oth_a[e]], sign);
      if (oth_b[e] >= 0) sc.bump(b + 3, colour[oth_b[e]], sign);
    }
  };
  // every set membership of one cell
  auto cell_access = [&](int x, int sign) {
    if (x >= E) {  // L cell: read by every edge of the VN
      const int v = x - E;
      for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {
        const int e = c.var_edges[j];
        for (int set0 : occ[row_of[e]]) sc.bump(set0 + 4 * pos[e] + 1, colour[x], sign);
      }
      return;
    }
    for (int set0 : occ[row_of[x]]) sc.bump(set0 + 4 * pos[x], colour[x], sign);  // own
    const int v = c.cols[x];
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {  // read by the VN's other edges
      const int e = c.var_edges[j];
      if (e == x) continue;
      const int q = oth_a[e] == x ? 2 : 3;
      for (int set0 : occ[row_of[e]]) sc.bump(set0 + 4 * pos[e] + q, colour[x], sign);
    }
  };
  for (int e = 0; e < E; ++e) edge_access(e, +1);
  const long long cost0 = sc.total;
  const int nsets = static_cast<int>(sc.mx.size());
  if (E + n <= 32768 && nsets > 0) {
    Stream rng(0x6469726563746c79ull);
    static const long long scale = [] {
      const char* e = std::getenv("LDPCB_BANK_ITERS");  // moves per CN; tuning / A-B only
      return e ? std::atoll(e) : 4000ll;
    }();
    const long long iters = std::min<long long>(20000000, scale * c.m);
    std::vector<int> best_colour = colour, best_pos = pos;
    long long best_total = sc.total;
    auto swap_colours = [&](int x, int y) {
      cell_access(x, -1);
      cell_access(y, -1);
      std::swap(colour[x], colour[y]);
      cell_access(x, +1);
      cell_access(y, +1);
    };
    auto swap_positions = [&](int e1, int e2) {
      edge_access(e1, -1);
      edge_access(e2, -1);
      std::swap(pos[e1], pos[e2]);
      edge_access(e1, +1);
      edge_access(e2, +1);
    };
    // annealed on the colliding pairs (the wavefront count itself is a
    // plateau landscape: it only moves when a set's maximum does) plus the
    // wavefronts; the best wavefront count seen is kept
    for (long long it = 0; it < iters; ++it) {
      const double T = 0.6 * (1.0 - static_cast<double>(it) / iters) + 0.05;
      const long long before = sc.pairs + sc.total;
      const int kind = static_cast<int>(rng.below(8));
      if (kind < 3) {  // positions of two edges of a CN
        const int r = static_cast<int>(rng.below(c.m));
        if (occ[r].empty()) continue;
        const int k1 = static_cast<int>(rng.below(6));
        int k2 = static_cast<int>(rng.below(5));
        if (k2 >= k1) ++k2;
        const int e1 = c.row_off[r] + k1, e2 = c.row_off[r] + k2;
        swap_positions(e1, e2);
        const long long d = sc.pairs + sc.total - before;
        if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_positions(e1, e2);
      } else {
        const bool lcell = kind == 7;
        const int lo = lcell ? E : 0, cnt = lcell ? n : E;
        const int x = lo + static_cast<int>(rng.below(cnt)), y = lo + static_cast<int>(rng.below(cnt));
        if (colour[x] == colour[y]) continue;
        swap_colours(x, y);
        const long long d = sc.pairs + sc.total - before;
        if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_colours(x, y);
      }
      if (sc.total < best_total && it > iters / 2) {
        best_total = sc.total;
        best_colour = colour;
        best_pos = pos;
      }
    }
    if (sc.total > best_total) colour = best_colour, pos = best_pos;
    if (std::getenv("LDPCB_BANK_DEBUG"))
      std::fprintf(stderr, "direct_tables: %d sets, cost %.3f -> %.3f per set (%lld moves)\n", nsets,
                   static_cast<double>(cost0) / nsets, static_cast<double>(std::min(sc.total, best_total)) / nsets,
                   iters);
  }
  // edge at record position k of CN r
  std::vector<int> at(E);
  for (int e = 0; e < E; ++e) at[c.row_off[row_of[e]] + pos[e]] = e;
  // cell ids: colour + 16 * rank inside the colour class of the kind
  std::vector<int> cell(E + n);
  {
    std::vector<int> rank(kColours, 0);
    for (int e = 0; e < E; ++e) cell[e] = colour[e] + kColours * rank[colour[e]]++;
    std::fill(rank.begin(), rank.end(), 0);
    t.vn_pos.resize(n);
    for (int v = 0; v < n; ++v) {
      t.vn_pos[v] = colour[E + v] + kColours * rank[colour[E + v]]++;
      cell[E + v] = l_base + t.vn_pos[v];
    }
  }
  const int zero = cells - 1;
  auto off = [&](int cell_id) { return static_cast<uint32_t>(cell_id) * 8u; };
  auto c2v_off = [&](int e) { return off(e >= 0 ? cell[e] : zero); };
  auto put_edge = [&](std::vector<int32_t>& out, int e) {
    out.push_back(static_cast<int32_t>(c2v_off(e) | (off(cell[E + c.cols[e]]) << 16)));
    out.push_back(static_cast<int32_t>(c2v_off(oth_a[e]) | (c2v_off(oth_b[e]) << 16)));
  };
  t.cn_off.assign(1, 0);
  for (int g = 0; g < s.G; ++g) {
    for (int r : group_cns[g])
      for (int k = 0; k < 6; ++k) put_edge(t.cn_rec, at[c.row_off[r] + k]);
    t.cn_off.push_back(t.cn_off.back() + static_cast<int>(group_cns[g].size()));
  }
  for (int e = 0; e < E; ++e) put_edge(t.edge_rec, e);
  t.vn_rec.assign(2 * static_cast<size_t>(n), 0);
  for (int v = 0; v < n; ++v) {
    uint32_t f[3] = {off(zero), off(zero), off(zero)};
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) f[j - c.var_off[v]] = c2v_off(c.var_edges[j]);
    t.vn_rec[2 * t.vn_pos[v]] = static_cast<int32_t>(f[0] | (f[1] << 16));
    t.vn_rec[2 * t.vn_pos[v] + 1] = static_cast<int32_t>(f[2]);
  }
  for (int r = 0; r < c.m; ++r) {
    uint32_t w[4] = {0, 0, 0, 0};
    for (int k = 0; k < 6; ++k) w[k / 2] |= static_cast<uint32_t>(t.vn_pos[c.cols[c.row_off[r] + k]]) << (16 * (k & 1));
    for (uint32_t x : w) t.all_cn.push_back(static_cast<int32_t>(x));
  }
  t.cells = cells;
  t.l_base = l_base;
  t.ok = true;
  return t;
}

}  // namespace ldpcb
