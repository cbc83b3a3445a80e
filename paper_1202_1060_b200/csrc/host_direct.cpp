// host_direct.cpp -- tables of the direct (posterior-free) resident kernel
// (direct.cu): holder assignment, cell assignment with shared-memory bank
// colouring and the per-group CN records. See host.hpp DirectTables.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>

#include "host.hpp"
#include "rng.cuh"

namespace ldpcb {

namespace {

// A cell holds fv frames (4 fv bytes): one wavefront serves 128 bytes, i.e.
// 32 / fv lanes, and the cells it touches fall in 32 / fv bank groups
// ("colours"): 16 for two frames per cell, 8 for four.
constexpr int kMaxColours = 16;
constexpr int kSetsPerWindow = 20;  // 6 own stores, 2 x 3 holder reads, 4 x 2 other reads

// first read set of record position p (relative to the window's set0)
inline int read_base(int p) { return p < 2 ? 6 + 3 * p : 12 + 2 * (p - 2); }

// Colouring problem: every "set" lists the cells one shared-memory instruction
// of one wavefront touches; its cost is the largest number of cells sharing
// a colour (the wavefronts that instruction needs). Cells of one kind (c2v /
// L) swap colours, so each colour class keeps its size and the final cell
// id colour + colours * rank stays a permutation of the kind's range.
struct SetCounts {
  int kColours;
  int H;
  explicit SetCounts(int colours) : kColours(colours), H(colours + 1) {}
  std::vector<uint8_t> cnt;    // [set][colour]
  std::vector<uint16_t> hist;  // [set][count] -> colours with that count
  std::vector<uint8_t> mx;
  long long total = 0;  // sum over sets of the largest colour count: the wavefronts issued
  long long pairs = 0;  // sum over sets and colours of cnt (cnt - 1) / 2: the smooth annealing objective
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

// One holder edge per VN such that every CN holds exactly two: a perfect
// matching of the VNs to two slots per CN in the (3,6)-biregular graph (it
// always exists), found with augmenting paths. hold[v] = the chosen edge id;
// empty when no such matching exists.
std::vector<int> holder_edges(const CodeData& c) {
  std::vector<int> hold(c.n, -1);
  std::vector<int> slot_vn(2 * static_cast<size_t>(c.m), -1);
  std::vector<char> vis(2 * static_cast<size_t>(c.m));
  std::function<bool(int)> augment = [&](int v) {
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j)
      for (int t = 0; t < 2; ++t) {
        const int sl = 2 * c.var_cns[j] + t;
        if (vis[sl]) continue;
        vis[sl] = 1;
        if (slot_vn[sl] < 0 || augment(slot_vn[sl])) {
          slot_vn[sl] = v;
          hold[v] = c.var_edges[j];
          return true;
        }
      }
    return false;
  };
  for (int v = 0; v < c.n; ++v) {
    std::fill(vis.begin(), vis.end(), 0);
    if (!augment(v)) return {};
  }
  for (int v : slot_vn)
    if (v < 0) return {};
  return hold;
}

}  // namespace

DirectTables direct_tables(const CodeData& c, const ScheduleData& s, int fv) {
  DirectTables t;
  t.fv = fv;
  if (s.per_frame || c.max_vdeg != 3 || c.max_cdeg != 6 || (fv != 2 && fv != 4)) return t;
  if (s.G > 96 || s.grp_cns.size() > 65535) return t;  // kernels.cuh DevGraph::d_goff
  const int kColours = 32 / fv, kLanes = 32 / fv;
  const uint32_t cell_bytes = 4u * static_cast<uint32_t>(fv);
  for (int r = 0; r < c.m; ++r)
    if (c.row_off[r + 1] - c.row_off[r] != 6) return t;
  for (int v = 0; v < c.n; ++v)
    if (c.var_off[v + 1] - c.var_off[v] != 3) return t;
  const int E = c.E, n = c.n;
  // One group of more CNs than a CTA has threads (flooding): its CN items run in several
  // rounds, so the Jacobi order needs the old messages kept while new ones are written:
  // two copies of the edge cells, read one / write the other, swapped every iteration.
  const bool flood = s.G == 1 && s.grp_off[1] - s.grp_off[0] > 96;
  const int e_cells = (E + 15) / 16 * 16;
  const int l_base = flood ? 2 * e_cells : e_cells;
  const int cells = l_base + (n + 15) / 16 * 16;
  if (static_cast<long long>(cells) * cell_bytes > 65536) return t;
  t.buf_cells = flood ? e_cells : 0;
  const std::vector<int> hold = holder_edges(c);
  if (hold.empty()) return t;
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
  // Cells [0, E): edge e (a holder edge's cell carries c2v + L); [E, E + n): L of VN v.
  // rd[3 e + q]: the cells edge e reads. Holder edge: v2c = (rd0 + rd1) + rd2 with
  // rd0 / rd1 the VN's two other edges (free order: one exact addition) and rd2 = L.
  // Other edges: v2c = rd0 + rd1, the holder's cell and the third edge's.
  std::vector<int> rd(3 * static_cast<size_t>(E), -1), row_of(E), pos(E);
  std::vector<char> is_holder(E, 0);
  for (int v = 0; v < n; ++v) is_holder[hold[v]] = 1;
  for (int v = 0; v < n; ++v)
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {
      const int e = c.var_edges[j];
      int w = 0;
      for (int i = c.var_off[v]; i < c.var_off[v + 1]; ++i)
        if (i != j) rd[3 * e + w++] = c.var_edges[i];
      if (is_holder[e]) rd[3 * e + 2] = E + v;
    }
  // record positions: the two holder edges of a CN first
  for (int r = 0; r < c.m; ++r) {
    int ph = 0, po = 2;
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) {
      row_of[e] = r;
      pos[e] = is_holder[e] ? ph++ : po++;
    }
  }
  auto slot_of = [&](int e, int x) { return rd[3 * e] == x ? 0 : (rd[3 * e + 1] == x ? 1 : 2); };
  // ---- bank colouring. The sets of a CN occurrence (the CN items one
  // wavefront serves in one group) are set0 + position for the own store and
  // set0 + read_base(position) + q for the reads. Free: the colour of every
  // cell, the record position of an edge inside its class (boxplus is
  // symmetric) and the order of the first two reads of an edge.
  std::vector<int> colour(E + n);
  for (int e = 0; e < E; ++e) colour[e] = e % kColours;
  for (int v = 0; v < n; ++v) colour[E + v] = v % kColours;
  SetCounts sc(kColours);
  std::vector<std::vector<int>> occ(c.m);  // CN -> set0 of each occurrence
  std::vector<std::vector<int>> win_cns;   // window -> its CNs
  for (int g = 0; g < s.G; ++g) {
    const int cn = static_cast<int>(group_cns[g].size());
    for (int i0 = 0; i0 < cn; i0 += kLanes) {
      int set0 = -1;
      for (int q = 0; q < kSetsPerWindow; ++q) {
        const int id = sc.add_set();
        if (q == 0) set0 = id;
      }
      win_cns.emplace_back();
      for (int i = i0; i < std::min(cn, i0 + kLanes); ++i) {
        occ[group_cns[g][i]].push_back(set0);
        win_cns.back().push_back(group_cns[g][i]);
      }
    }
  }
  // the accesses of edge e's record position, in every occurrence of its CN
  auto edge_access = [&](int e, int sign) {
    for (int set0 : occ[row_of[e]]) {
      sc.bump(set0 + pos[e], colour[e], sign);
      const int b = set0 + read_base(pos[e]);
      for (int q = 0; q < 3; ++q)
        if (rd[3 * e + q] >= 0) sc.bump(b + q, colour[rd[3 * e + q]], sign);
    }
  };
  // every set membership of one cell
  auto cell_access = [&](int x, int sign) {
    if (x >= E) {  // L cell: read by the VN's holder edge
      const int e = hold[x - E];
      for (int set0 : occ[row_of[e]]) sc.bump(set0 + read_base(pos[e]) + 2, colour[x], sign);
      return;
    }
    for (int set0 : occ[row_of[x]]) sc.bump(set0 + pos[x], colour[x], sign);  // own
    const int v = c.cols[x];
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {  // read by the VN's other edges
      const int e = c.var_edges[j];
      if (e == x) continue;
      const int q = slot_of(e, x);
      for (int set0 : occ[row_of[e]]) sc.bump(set0 + read_base(pos[e]) + q, colour[x], sign);
    }
  };
  for (int e = 0; e < E; ++e) edge_access(e, +1);
  const long long cost0 = sc.total;
  const int nsets = static_cast<int>(sc.mx.size());
  t.wavefronts = nsets ? static_cast<double>(cost0) / nsets : 1.0;
  std::vector<int> at(E);  // edge at record position k of CN r
  for (int e = 0; e < E; ++e) at[c.row_off[row_of[e]] + pos[e]] = e;
  if (E + n <= 32768 && nsets > 0) {
    Stream rng(0x6469726563746c79ull);
    static const long long scale = [] {
      const char* e = std::getenv("LDPCB_BANK_ITERS");  // moves per CN; tuning / A-B only
      return e ? std::atoll(e) : 4000ll;
    }();
    const long long iters = std::min<long long>(40000000, scale * c.m);
    std::vector<int> best_colour = colour, best_pos = pos, best_rd = rd;
    long long best_total = sc.total;
    // a cell of the most loaded colour of a random conflicting set (-1: the set drawn has no conflict)
    auto conflicting_cell = [&]() {
      const int set = static_cast<int>(rng.below(nsets));
      if (sc.mx[set] < 2) return -1;
      const int rel = set % kSetsPerWindow;
      int k, q;  // record position and access (0 own, 1.. reads)
      if (rel < 6)
        k = rel, q = 0;
      else if (rel < 12)
        k = (rel - 6) / 3, q = 1 + (rel - 6) % 3;
      else
        k = 2 + (rel - 12) / 2, q = 1 + (rel - 12) % 2;
      int pick = -1, seen = 0;
      for (int r : win_cns[set / kSetsPerWindow]) {
        const int e = at[c.row_off[r] + k];
        const int x = q == 0 ? e : rd[3 * e + q - 1];
        if (x < 0 || sc.cnt[static_cast<size_t>(set) * kColours + colour[x]] != sc.mx[set]) continue;
        if (rng.below(++seen) == 0) pick = x;
      }
      return pick;
    };
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
      at[c.row_off[row_of[e1]] + pos[e1]] = e1;
      at[c.row_off[row_of[e2]] + pos[e2]] = e2;
      edge_access(e1, +1);
      edge_access(e2, +1);
    };
    // annealed on the colliding pairs (the wavefront count itself is a
    // plateau landscape: it only moves when a set's maximum does) plus the
    // wavefronts; the best wavefront count seen is kept
    for (long long it = 0; it < iters; ++it) {
      const double T = 0.6 * (1.0 - static_cast<double>(it) / iters) + 0.05;
      const long long before = sc.pairs + sc.total;
      const int kind = static_cast<int>(rng.below(10));
      if (kind >= 8) {  // the first two reads of an edge
        const int e = static_cast<int>(rng.below(E));
        if (occ[row_of[e]].empty()) continue;
        auto swap_slots = [&]() {
          edge_access(e, -1);
          std::swap(rd[3 * e], rd[3 * e + 1]);
          edge_access(e, +1);
        };
        swap_slots();
        const long long d = sc.pairs + sc.total - before;
        if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_slots();
      } else if (kind < 3) {  // positions of two edges of a CN, inside their class
        const int r = static_cast<int>(rng.below(c.m));
        if (occ[r].empty()) continue;
        int k1, k2;
        if (rng.below(3) == 0) {
          k1 = 0, k2 = 1;
        } else {
          k1 = 2 + static_cast<int>(rng.below(4));
          k2 = 2 + static_cast<int>(rng.below(3));
          if (k2 >= k1) ++k2;
        }
        const int e1 = at[c.row_off[r] + k1], e2 = at[c.row_off[r] + k2];
        swap_positions(e1, e2);
        const long long d = sc.pairs + sc.total - before;
        if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_positions(e1, e2);
      } else {
        // half of the colour moves start from a cell that conflicts
        int x = kind < 6 ? conflicting_cell() : -1;
        const bool lcell = x >= 0 ? x >= E : kind == 7;
        const int lo = lcell ? E : 0, cnt = lcell ? n : E;
        if (x < 0) x = lo + static_cast<int>(rng.below(cnt));
        const int y = lo + static_cast<int>(rng.below(cnt));
        if (colour[x] == colour[y]) continue;
        swap_colours(x, y);
        const long long d = sc.pairs + sc.total - before;
        if (d > 0 && rng.unit() >= std::exp(-d / T)) swap_colours(x, y);
      }
      if (sc.total < best_total && it > iters / 2) {
        best_total = sc.total;
        best_colour = colour;
        best_pos = pos;
        best_rd = rd;
      }
    }
    if (sc.total > best_total) colour = best_colour, pos = best_pos, rd = best_rd;
    t.wavefronts = static_cast<double>(std::min(sc.total, best_total)) / nsets;
    if (std::getenv("LDPCB_BANK_DEBUG"))
      std::fprintf(stderr, "direct_tables: %d sets, cost %.3f -> %.3f per set (%lld moves)\n", nsets,
                   static_cast<double>(cost0) / nsets, static_cast<double>(std::min(sc.total, best_total)) / nsets,
                   iters);
    for (int e = 0; e < E; ++e) at[c.row_off[row_of[e]] + pos[e]] = e;
  }
  // cell ids: colour + colours * rank inside the colour class of the kind
  std::vector<int> cell(E + n);
  {
    std::vector<int> rank(kMaxColours, 0);
    for (int e = 0; e < E; ++e) cell[e] = colour[e] + kColours * rank[colour[e]]++;
    std::fill(rank.begin(), rank.end(), 0);
    t.vn_pos.resize(n);
    for (int v = 0; v < n; ++v) {
      t.vn_pos[v] = colour[E + v] + kColours * rank[colour[E + v]]++;
      cell[E + v] = l_base + t.vn_pos[v];
    }
  }
  auto off = [&](int x) { return static_cast<uint32_t>(cell[x]) * cell_bytes; };
  // CN record: ten 16-bit-pair words in a 12-int stride (host.hpp)
  auto put_cn = [&](std::vector<int32_t>& out, int r) {
    std::vector<uint32_t> f;
    for (int k = 0; k < 2; ++k) {
      const int e = at[c.row_off[r] + k];
      f.insert(f.end(), {off(e), off(rd[3 * e]), off(rd[3 * e + 1]), off(rd[3 * e + 2])});
    }
    for (int k = 2; k < 6; ++k) {
      const int e = at[c.row_off[r] + k];
      f.insert(f.end(), {off(e), off(rd[3 * e]), off(rd[3 * e + 1])});
    }
    f.resize(24, 0u);
    for (size_t i = 0; i < f.size(); i += 2) out.push_back(static_cast<int32_t>(f[i] | (f[i + 1] << 16)));
  };
  t.cn_off.assign(1, 0);
  for (int g = 0; g < s.G; ++g) {
    for (int r : group_cns[g]) put_cn(t.cn_rec, r);
    t.cn_off.push_back(t.cn_off.back() + static_cast<int>(group_cns[g].size()));
  }
  // per CN-major edge id: own | (holder ? L : 0xffff) << 16, rd0 | rd1 << 16
  for (int e = 0; e < E; ++e) {
    t.edge_rec.push_back(static_cast<int32_t>(off(e) | ((is_holder[e] ? off(rd[3 * e + 2]) : 0xffffu) << 16)));
    t.edge_rec.push_back(static_cast<int32_t>(off(rd[3 * e]) | (off(rd[3 * e + 1]) << 16)));
  }
  // per VN position: holder cell | second << 16, third (the other two edges in ascending CN order)
  t.vn_rec.assign(2 * static_cast<size_t>(n), 0);
  t.vn_hold.resize(n);
  for (int v = 0; v < n; ++v) {
    uint32_t f[2] = {0, 0};
    int w = 0;
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j)
      if (c.var_edges[j] != hold[v]) f[w++] = off(c.var_edges[j]);
    t.vn_rec[2 * t.vn_pos[v]] = static_cast<int32_t>(off(hold[v]) | (f[0] << 16));
    t.vn_rec[2 * t.vn_pos[v] + 1] = static_cast<int32_t>(f[1]);
    t.vn_hold[v] = static_cast<int32_t>(off(hold[v]));
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
