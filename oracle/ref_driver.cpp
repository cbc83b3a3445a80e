// ref_driver.cpp -- CPU ORACLE (test infrastructure only).
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/ldpc/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libldpc_ref.so. It only composes the reference's public inline
// functions (the same composition the reference's own tests use:
// tests/acceptance.cpp:142-146, tests/test_decoder.cpp:129-147); it contains
// no decoder arithmetic of its own. Used to pin oracle/ldpc_oracle.c, to make
// golden fixtures (tests/golden/make_golden.py) and as bench.py's
// `--impl reference` CPU arm. Never linked by the product.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "ldpc/channel.hpp"
#include "ldpc/decoder.hpp"
#include "ldpc/rng.hpp"
#include "ldpc/schedule.hpp"
#include "ldpc/sim.hpp"
#include "ldpc/tanner.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

std::vector<std::vector<int>> rows_from_csr(int m, const int32_t* off, const int32_t* cols) {
  std::vector<std::vector<int>> rows(m);
  for (int r = 0; r < m; ++r) rows[r].assign(cols + off[r], cols + off[r + 1]);
  return rows;
}

ldpc::GroupSchedule make_sched(int kind, int n_groups, const int32_t* grp_off, const int32_t* grp_cns,
                               double overlap, uint64_t seed, int regroup) {
  ldpc::GroupSchedule s;
  s.kind = static_cast<ldpc::ScheduleKind>(kind);
  s.n_groups = n_groups;
  s.overlap_ratio = overlap;
  s.seed = seed;
  s.regroup_each_iteration = regroup != 0;
  s.groups = rows_from_csr(n_groups, grp_off, grp_cns);
  int gs = 0;
  for (const auto& g : s.groups) gs = std::max(gs, static_cast<int>(g.size()));
  s.group_size = gs;
  return s;
}

int export_groups(const std::vector<std::vector<int>>& groups, int32_t* grp_off, int32_t* grp_cns, int cap) {
  int w = 0;
  grp_off[0] = 0;
  for (std::size_t g = 0; g < groups.size(); ++g) {
    if (w + static_cast<int>(groups[g].size()) > cap) {
      g_err = "slot buffer too small";
      return -1;
    }
    for (int cn : groups[g]) grp_cns[w++] = cn;
    grp_off[g + 1] = w;
  }
  return w;
}

// decode with full state access: init_state + run_subiteration + the totals
// loop of decoder.hpp:162-167 (acceptance.cpp:142-146 composes the same way).
void decode_composed(const ldpc::TannerGraph& g, const ldpc::GroupSchedule& s, std::span<const double> llr,
                     int max_iters, bool early_stop, uint8_t* bits, int32_t* iterations, uint8_t* converged,
                     double* posterior, int32_t* trace) {
  ldpc::DecoderState st = ldpc::init_state(g, llr);
  if (trace)
    for (int i = 0; i < max_iters; ++i) trace[i] = -1;
  std::vector<std::vector<int>> regrouped;
  const std::vector<std::vector<int>>* groups = &s.groups;
  int iters = 0;
  bool conv = false;
  for (int iter = 1; iter <= max_iters; ++iter) {
    if (iter > 1 && s.regroup_each_iteration && s.kind != ldpc::ScheduleKind::flooding) {
      regrouped = ldpc::schedule_groups_for(s, g.n_checks, static_cast<std::uint64_t>(iter));
      groups = &regrouped;
    }
    for (const auto& group : *groups) ldpc::run_subiteration(st, g, group);
    for (int n = 0; n < g.n_vars; ++n) {
      double total = st.channel_llr[n];
      for (int eid : g.var_edge_ids[n]) total += st.c2v[eid];
      st.total_llr[n] = total;
      st.hard_decision[n] = total >= 0.0 ? 0 : 1;
    }
    const int w = ldpc::syndrome_weight(g, st.hard_decision);
    if (trace) trace[iter - 1] = w;
    iters = iter;
    conv = w == 0;
    if (conv && early_stop) break;
  }
  if (bits) std::memcpy(bits, st.hard_decision.data(), g.n_vars);
  if (iterations) *iterations = early_stop ? iters : max_iters;
  if (converged) *converged = conv;
  if (posterior) std::memcpy(posterior, st.total_llr.data(), sizeof(double) * g.n_vars);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_graph_create(int n, int m, const int32_t* off, const int32_t* cols) {
  try {
    return new ldpc::TannerGraph(ldpc::build_from_check_lists(n, rows_from_csr(m, off, cols)));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_graph_destroy(void* g) { delete static_cast<ldpc::TannerGraph*>(g); }

// var_off[n+1], var_cns[E], var_edges[E]
void ref_graph_var_view(void* gp, int32_t* var_off, int32_t* var_cns, int32_t* var_edges) {
  const auto& g = *static_cast<ldpc::TannerGraph*>(gp);
  int w = 0;
  var_off[0] = 0;
  for (int n = 0; n < g.n_vars; ++n) {
    for (std::size_t j = 0; j < g.var_adj[n].size(); ++j) {
      var_cns[w] = g.var_adj[n][j];
      var_edges[w] = g.var_edge_ids[n][j];
      ++w;
    }
    var_off[n + 1] = w;
  }
}

int ref_random_regular(int n, int dv, int dc, uint64_t seed, int32_t* cols_out) {
  try {
    const auto g = ldpc::random_regular_graph(n, dv, dc, seed);
    int w = 0;
    for (const auto& row : g.check_adj)
      for (int v : row) cols_out[w++] = v;
    return g.n_checks;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Parses alist text; returns E (and fills n, m, row_off[m+1], cols[E] when
// the caps suffice) or -1 with the AlistError message (kind and line).
int ref_parse_alist(const char* text, int* n, int* m, int32_t* row_off, int32_t* cols, int cap_m, int cap_e,
                    int* err_kind, int* err_line) {
  try {
    const auto g = ldpc::parse_alist(text);
    *n = g.n_vars;
    *m = g.n_checks;
    if (g.n_checks <= cap_m && g.n_edges <= cap_e) {
      for (int r = 0; r <= g.n_checks; ++r) row_off[r] = g.check_edge_offset[r];
      int w = 0;
      for (const auto& row : g.check_adj)
        for (int v : row) cols[w++] = v;
    }
    return g.n_edges;
  } catch (const ldpc::AlistError& e) {
    if (err_kind) *err_kind = static_cast<int>(e.kind());
    if (err_line) *err_line = e.line();
    return fail(e);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// serialize_alist into buf; returns the length (buf filled when cap suffices)
long ref_serialize_alist(void* gp, char* buf, long cap) {
  const std::string s = ldpc::serialize_alist(*static_cast<ldpc::TannerGraph*>(gp));
  if (static_cast<long>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<long>(s.size());
}

double ref_sigma2_from_ebn0(double ebn0_db, double rate) {
  try {
    return ldpc::sigma2_from_ebn0(ebn0_db, rate);
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

int ref_transmit_all_zero(double sigma2, uint64_t seed, int n, uint64_t frame_id, double* llr) {
  try {
    ldpc::ChannelConfig cfg;
    cfg.sigma2 = sigma2;
    cfg.seed = seed;
    const auto v = ldpc::transmit_all_zero(cfg, n, frame_id);
    std::memcpy(llr, v.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return ldpc::mix_seed(seed, stream); }

// Draws `count` values from Rng(seed): kind 0 = next_u64, 1 = next_unit,
// 2 = next_gaussian, 3 = next_below(bound) (as doubles for 1/2, u64 otherwise)
void ref_rng_draw(uint64_t seed, int kind, uint64_t bound, int count, uint64_t* out_u64, double* out_f64) {
  ldpc::Rng rng(seed);
  for (int i = 0; i < count; ++i) {
    switch (kind) {
      case 0: out_u64[i] = rng.next_u64(); break;
      case 1: out_f64[i] = rng.next_unit(); break;
      case 2: out_f64[i] = rng.next_gaussian(); break;
      default: out_u64[i] = rng.next_below(bound); break;
    }
  }
}

// make_{disjoint,nondisjoint}_schedule (schedule.hpp:136-171); returns slots
int ref_make_schedule(void* gp, int kind, int n_groups, double overlap, uint64_t seed, int32_t* grp_off,
                      int32_t* grp_cns, int cap, int* group_size) {
  try {
    const auto& g = *static_cast<ldpc::TannerGraph*>(gp);
    ldpc::GroupSchedule s;
    if (kind == 0)
      s = ldpc::make_flooding_schedule(g);
    else if (kind == 1)
      s = ldpc::make_disjoint_schedule(g, n_groups, seed);
    else
      s = ldpc::make_nondisjoint_schedule(g, n_groups, overlap, seed);
    if (group_size) *group_size = s.group_size;
    return export_groups(s.groups, grp_off, grp_cns, cap);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_iteration_budget(int n_checks, int i_max, int kind, int n_groups, int group_size, double overlap) {
  ldpc::GroupSchedule s;
  s.kind = static_cast<ldpc::ScheduleKind>(kind);
  s.n_groups = n_groups;
  s.group_size = group_size;
  s.overlap_ratio = overlap;
  return ldpc::iteration_budget(n_checks, i_max, s);
}

// measure_cocsg (schedule.hpp:175-201): counts[G-1]; returns G-1
int ref_measure_cocsg(void* gp, int n_groups, const int32_t* grp_off, const int32_t* grp_cns, int32_t* counts) {
  const auto s = make_sched(2, n_groups, grp_off, grp_cns, 0.0, 0, 0);
  const auto rep = ldpc::measure_cocsg(*static_cast<ldpc::TannerGraph*>(gp), s);
  for (std::size_t i = 0; i < rep.transition_counts.size(); ++i) counts[i] = rep.transition_counts[i];
  return static_cast<int>(rep.transition_counts.size());
}

// check_update (decoder.hpp:59-87) on a single CN of the given degree
void ref_check_update(int degree, const double* v2c, double* c2v) {
  std::vector<std::vector<int>> row(1);
  for (int k = 0; k < degree; ++k) row[0].push_back(k);
  const auto g = ldpc::build_from_check_lists(degree, row);
  ldpc::DecoderState st = ldpc::init_state(g, std::vector<double>(degree, 0.0));
  for (int k = 0; k < degree; ++k) st.v2c[g.edge_id(0, k)] = v2c[k];
  ldpc::check_update(st, g, 0);
  for (int k = 0; k < degree; ++k) c2v[k] = st.c2v[g.edge_id(0, k)];
}

// ldpc::decode itself (decoder.hpp:143-181): early stop always on
int ref_decode(void* gp, int kind, int n_groups, const int32_t* grp_off, const int32_t* grp_cns, double overlap,
               uint64_t seed, int regroup, const double* llr, int max_iters, uint8_t* bits, int32_t* iterations,
               uint8_t* converged, int32_t* trace, int64_t* cn_updates) {
  try {
    const auto& g = *static_cast<ldpc::TannerGraph*>(gp);
    const auto s = make_sched(kind, n_groups, grp_off, grp_cns, overlap, seed, regroup);
    const auto out = ldpc::decode(g, s, std::span<const double>(llr, g.n_vars), max_iters);
    if (bits) std::memcpy(bits, out.bits.data(), g.n_vars);
    if (iterations) *iterations = out.iterations;
    if (converged) *converged = out.converged;
    if (trace) {
      for (int i = 0; i < max_iters; ++i)
        trace[i] = i < static_cast<int>(out.syndrome_weight_trace.size()) ? out.syndrome_weight_trace[i] : -1;
    }
    if (cn_updates) *cn_updates = out.cn_updates;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_decode_composed(void* gp, int kind, int n_groups, const int32_t* grp_off, const int32_t* grp_cns,
                        double overlap, uint64_t seed, int regroup, const double* llr, int max_iters, int early_stop,
                        uint8_t* bits, int32_t* iterations, uint8_t* converged, double* posterior, int32_t* trace) {
  try {
    const auto& g = *static_cast<ldpc::TannerGraph*>(gp);
    if (max_iters < 1) throw std::invalid_argument("max_iters must be >= 1");
    const auto s = make_sched(kind, n_groups, grp_off, grp_cns, overlap, seed, regroup);
    decode_composed(g, s, std::span<const double>(llr, g.n_vars), max_iters, early_stop != 0, bits, iterations,
                    converged, posterior, trace);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// init_state + n_subiters x run_subiteration cycling through the groups
int ref_run_subiterations(void* gp, int n_groups, const int32_t* grp_off, const int32_t* grp_cns, const double* llr,
                          int n_subiters, double* c2v, double* v2c) {
  try {
    const auto& g = *static_cast<ldpc::TannerGraph*>(gp);
    const auto s = make_sched(2, n_groups, grp_off, grp_cns, 0.0, 0, 0);
    ldpc::DecoderState st = ldpc::init_state(g, std::span<const double>(llr, g.n_vars));
    for (int t = 0; t < n_subiters; ++t) ldpc::run_subiteration(st, g, s.groups[t % n_groups]);
    if (c2v) std::memcpy(c2v, st.c2v.data(), sizeof(double) * g.n_edges);
    if (v2c) std::memcpy(v2c, st.v2c.data(), sizeof(double) * g.n_edges);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Frame-parallel batch decode on `threads` std::threads pulling frame ids from
// an atomic counter, as the reference harness does (sim.hpp:136-150). fp32
// LLRs are promoted to double. early_stop=1 calls ldpc::decode.
int ref_decode_batch_f32(void* gp, int kind, int n_groups, const int32_t* grp_off, const int32_t* grp_cns,
                         const float* llr, int64_t frames, int max_iters, int early_stop, int threads, uint8_t* bits,
                         int32_t* iterations, uint8_t* converged, float* posterior) {
  try {
    const auto& g = *static_cast<ldpc::TannerGraph*>(gp);
    const auto s = make_sched(kind, n_groups, grp_off, grp_cns, 0.0, 0, 0);
    std::atomic<int64_t> next(0);
    std::atomic<int> rc(0);
    auto worker = [&]() {
      std::vector<double> in(g.n_vars), post(g.n_vars);
      for (;;) {
        const int64_t f = next.fetch_add(1);
        if (f >= frames) return;
        for (int v = 0; v < g.n_vars; ++v) in[v] = static_cast<double>(llr[f * g.n_vars + v]);
        int32_t it = 0;
        uint8_t cv = 0;
        uint8_t* b = bits ? bits + f * g.n_vars : nullptr;
        if (early_stop && !posterior) {
          const auto out = ldpc::decode(g, s, in, max_iters);
          if (b) std::memcpy(b, out.bits.data(), g.n_vars);
          it = out.iterations;
          cv = out.converged;
        } else {
          decode_composed(g, s, in, max_iters, early_stop != 0, b, &it, &cv, posterior ? post.data() : nullptr,
                          nullptr);
          if (posterior)
            for (int v = 0; v < g.n_vars; ++v) posterior[f * g.n_vars + v] = static_cast<float>(post[v]);
        }
        if (iterations) iterations[f] = it;
        if (converged) converged[f] = cv;
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    return rc.load();
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// transmit_all_zero for frames [frame0, frame0+frames), rounded to fp32
int ref_transmit_batch_f32(double sigma2, uint64_t seed, int n, uint64_t frame0, int64_t frames, float* llr,
                           int threads) {
  ldpc::ChannelConfig cfg;
  cfg.sigma2 = sigma2;
  cfg.seed = seed;
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    for (;;) {
      const int64_t f = next.fetch_add(1);
      if (f >= frames) return;
      const auto v = ldpc::transmit_all_zero(cfg, n, frame0 + static_cast<uint64_t>(f));
      for (int i = 0; i < n; ++i) llr[f * n + i] = static_cast<float>(v[i]);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  return 0;
}

// ldpc::run_sweep (sim.hpp:96-186) on an explicit graph. out has 11 doubles
// per point: frames, bit_errors, frame_errors, converged_frames, ber, fer,
// mean_iters_converged, mean_iters_all, iter_limit, wall_seconds, ebn0_db.
int ref_run_sweep(void* gp, int kind, int n_groups, double overlap, int regroup, const double* ebn0, int n_points,
                  int i_max, int budgeted, long max_frames, int min_frame_errors, uint64_t channel_seed,
                  uint64_t schedule_seed, int workers, double* out) {
  try {
    ldpc::SimConfig cfg;
    cfg.kind = static_cast<ldpc::ScheduleKind>(kind);
    cfg.n_groups = n_groups;
    cfg.overlap = overlap;
    cfg.regroup_each_iteration = regroup != 0;
    cfg.ebn0_db.assign(ebn0, ebn0 + n_points);
    cfg.i_max = i_max;
    cfg.budgeted = budgeted != 0;
    cfg.max_frames = max_frames;
    cfg.min_frame_errors = min_frame_errors;
    cfg.channel_seed = channel_seed;
    cfg.schedule_seed = schedule_seed;
    cfg.workers = workers;
    const auto res = ldpc::run_sweep(cfg, *static_cast<ldpc::TannerGraph*>(gp));
    for (std::size_t i = 0; i < res.size(); ++i) {
      const auto& r = res[i];
      double* o = out + 11 * i;
      o[0] = r.frames;
      o[1] = static_cast<double>(r.bit_errors);
      o[2] = r.frame_errors;
      o[3] = r.converged_frames;
      o[4] = r.ber;
      o[5] = r.fer;
      o[6] = r.mean_iters_converged;
      o[7] = r.mean_iters_all;
      o[8] = r.iter_limit;
      o[9] = r.wall_seconds;
      o[10] = r.ebn0_db;
    }
    return static_cast<int>(res.size());
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
