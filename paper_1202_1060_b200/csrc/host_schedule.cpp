// host_schedule.cpp -- CN-group schedules and their derived tables.
#include <algorithm>
#include <cmath>

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

KernelTables kernel_tables(const CodeData& c, const ScheduleData& s, int cs, bool regular_rows) {
  if (cs < 2 + c.max_cdeg || cs % 4) throw std::invalid_argument("bad CN record stride");
  KernelTables t;
  t.cs = cs;
  t.vs4 = (1 + c.max_vdeg + 3) / 4;
  t.slot_stride = regular_rows ? (c.max_cdeg | 1) : 0;
  const long long slots = (t.slot_stride ? static_cast<long long>(c.m) * t.slot_stride : c.E) + 1;
  if (slots >= (1ll << 30)) throw std::invalid_argument("code too large for 32-bit edge records");
  t.n_slots = static_cast<int>(slots);
  const int zero = t.n_slots - 1;
  t.edge_slot.resize(c.E);
  for (int r = 0; r < c.m; ++r)
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e)
      t.edge_slot[e] = t.slot_stride ? r * t.slot_stride + (e - c.row_off[r]) : e;
  auto put_vn = [&](std::vector<int32_t>& out, int v) {
    out.push_back(v);
    int w = 1;
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j, ++w) out.push_back(t.edge_slot[c.var_edges[j]]);
    for (; w < 4 * t.vs4; ++w) out.push_back(zero);
  };
  auto put_cn = [&](std::vector<int32_t>& out, int r, uint32_t mask) {
    const int off = c.row_off[r], deg = c.row_off[r + 1] - off;
    out.push_back(t.edge_slot[off]);
    out.push_back(static_cast<int32_t>(mask));
    for (int k = 0; k < deg; ++k) out.push_back(c.cols[off + k]);
    for (int k = 2 + deg; k < t.cs; ++k) out.push_back(-1);
  };
  t.cn_off.assign(1, 0);
  t.fix_off.assign(1, 0);
  std::vector<char> in_group(c.m, 0);
  std::vector<int> touches(c.n, 0);
  std::vector<int> cns, shared_vns;
  for (int g = 0; g < s.G; ++g) {
    cns.clear();
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
    for (int r : cns) {
      uint32_t mask = 0;
      for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e)
        if (touches[c.cols[e]] == 1) mask |= 1u << (e - c.row_off[r]);
      t.recompute |= mask != 0;
      put_cn(t.cn_rec, r, mask);
    }
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
    for (int v : shared_vns) put_vn(t.fix_rec, v);
    t.cn_off.push_back(t.cn_off.back() + static_cast<int>(cns.size()));
    t.fix_off.push_back(t.fix_off.back() + static_cast<int>(shared_vns.size()));
    t.max_cn_items = std::max(t.max_cn_items, static_cast<int>(cns.size()));
    t.max_fix_items = std::max(t.max_fix_items, static_cast<int>(shared_vns.size()));
  }
  for (int v = 0; v < c.n; ++v) put_vn(t.all_vn_rec, v);
  for (int r = 0; r < c.m; ++r) put_cn(t.all_rec, r, 0);
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
