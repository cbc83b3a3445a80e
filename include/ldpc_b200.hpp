// ldpc_b200.hpp -- C++ host API of the B200 decoder, mirroring the reference's
// header-only API (arxiv/paper_1202_1060 proj/include/ldpc/*.hpp) over the C
// ABI of ldpc_b200.h. Same names, argument meaning and error behaviour:
//
//   ldpc::TannerGraph, build_from_check_lists,   -> ldpc_b200::TannerGraph
//     random_regular_graph, parse_alist,            (tanner.hpp:21-37, 79-114,
//     serialize_alist                                172-317, 356-393)
//   ldpc::GroupSchedule, make_*_schedule,          -> ldpc_b200::GroupSchedule
//     iteration_budget, measure_cocsg               (schedule.hpp:32-210)
//   ldpc::sigma2_from_ebn0                         -> ldpc_b200::sigma2_from_ebn0
//   ldpc::DecodeOutcome, ldpc::decode               -> ldpc_b200::decode
//     (decoder.hpp:31-37, 143-181)
//   run_sweep's frame loop + aggregation            -> ldpc_b200::simulate
//     (sim.hpp:111-124, 162-181)
//
// Preconditions throw std::invalid_argument exactly where the reference does
// (max_iters < 1, LLR length != n, infeasible (G, r), malformed graphs);
// alist errors throw ldpc_b200::AlistError with the reference's kind and
// line. Decoding runs on the current CUDA device; link with -lldpc_b200.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "ldpc_b200.h"

namespace ldpc_b200 {

enum class AlistErrorKind {
  malformed_header,
  bad_token,
  degree_error,
  length_mismatch,
  index_out_of_range,
  duplicate_entry,
  edge_count_mismatch,
  transpose_mismatch,
  trailing_content,
  truncated,
};

class AlistError : public std::runtime_error {
 public:
  AlistError(AlistErrorKind kind, int line, const std::string& what)
      : std::runtime_error(what), kind_(kind), line_(line) {}
  AlistErrorKind kind() const { return kind_; }
  int line() const { return line_; }

 private:
  AlistErrorKind kind_;
  int line_;
};

namespace detail {
inline void check(int status) {
  if (status == LDPCB_OK) return;
  const std::string msg = ldpcb_last_error();
  if (status == LDPCB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

enum class ScheduleKind { flooding = LDPCB_FLOODING, disjoint = LDPCB_DISJOINT, nondisjoint = LDPCB_NONDISJOINT };

inline const char* to_string(ScheduleKind kind) {
  switch (kind) {
    case ScheduleKind::flooding: return "bp";
    case ScheduleKind::disjoint: return "gsbp";
    case ScheduleKind::nondisjoint: return "ndgsbp";
  }
  return "?";
}

class TannerGraph {
 public:
  int n_vars = 0, n_checks = 0, n_edges = 0;

  static TannerGraph from_handle(ldpcb_code h) {
    TannerGraph g;
    g.h_ = std::shared_ptr<ldpcb_code_s>(h, ldpcb_code_destroy);
    int32_t n, m, e, dc, dv;
    detail::check(ldpcb_code_dims(h, &n, &m, &e, &dc, &dv));
    g.n_vars = n;
    g.n_checks = m;
    g.n_edges = e;
    return g;
  }
  ldpcb_code handle() const { return h_.get(); }

  // CN-major adjacency, like TannerGraph::check_adj / check_edge_offset
  std::vector<std::vector<int>> check_adj() const {
    std::vector<int32_t> off(n_checks + 1), cols(n_edges);
    detail::check(ldpcb_code_export(handle(), off.data(), cols.data(), nullptr, nullptr, nullptr));
    std::vector<std::vector<int>> rows(n_checks);
    for (int r = 0; r < n_checks; ++r) rows[r].assign(cols.begin() + off[r], cols.begin() + off[r + 1]);
    return rows;
  }
  int check_degree(int m) const { return static_cast<int>(check_adj()[m].size()); }
  int64_t count_4cycles() const {
    int64_t c = 0;
    detail::check(ldpcb_code_count_4cycles(handle(), &c));
    return c;
  }
  bool operator==(const TannerGraph& o) const {
    return n_vars == o.n_vars && n_checks == o.n_checks && check_adj() == o.check_adj();
  }

 private:
  std::shared_ptr<ldpcb_code_s> h_;
};

inline TannerGraph build_from_check_lists(int n_vars, const std::vector<std::vector<int>>& check_lists) {
  std::vector<int32_t> off(1, 0), cols;
  for (const auto& row : check_lists) {
    cols.insert(cols.end(), row.begin(), row.end());
    off.push_back(static_cast<int32_t>(cols.size()));
  }
  if (cols.empty()) cols.push_back(0);
  ldpcb_code h = nullptr;
  detail::check(ldpcb_code_from_check_lists(n_vars, static_cast<int>(check_lists.size()), off.data(), cols.data(), &h));
  return TannerGraph::from_handle(h);
}

inline TannerGraph random_regular_graph(int n_vars, int d_v, int d_c, std::uint64_t seed) {
  ldpcb_code h = nullptr;
  detail::check(ldpcb_code_random_regular(n_vars, d_v, d_c, seed, &h));
  return TannerGraph::from_handle(h);
}

inline TannerGraph random_regular_graph_girth6(int n_vars, int d_v, int d_c, std::uint64_t seed) {
  ldpcb_code h = nullptr;
  detail::check(ldpcb_code_random_regular_girth6(n_vars, d_v, d_c, seed, &h));
  return TannerGraph::from_handle(h);
}

inline TannerGraph parse_alist(std::string_view text) {
  ldpcb_code h = nullptr;
  int kind = -1, line = 0;
  const std::string s(text);
  const int st = ldpcb_code_parse_alist(s.c_str(), &h, &kind, &line);
  if (st == LDPCB_EALIST) throw AlistError(static_cast<AlistErrorKind>(kind), line, ldpcb_last_error());
  detail::check(st);
  return TannerGraph::from_handle(h);
}

inline std::string serialize_alist(const TannerGraph& g) {
  int64_t len = 0;
  detail::check(ldpcb_code_serialize_alist(g.handle(), nullptr, 0, &len));
  std::string out(static_cast<size_t>(len) + 1, '\0');
  detail::check(ldpcb_code_serialize_alist(g.handle(), out.data(), len + 1, &len));
  out.resize(static_cast<size_t>(len));
  return out;
}

class GroupSchedule {
 public:
  ScheduleKind kind = ScheduleKind::flooding;
  int n_groups = 1;
  double overlap_ratio = 0.0;
  int group_size = 0;
  bool regroup_each_iteration = false;  // device schedules are fixed per decode
  std::vector<std::vector<int>> groups;

  static GroupSchedule from_handle(ldpcb_schedule h) {
    GroupSchedule s;
    s.h_ = std::shared_ptr<ldpcb_schedule_s>(h, ldpcb_schedule_destroy);
    int32_t kind, G, slots, gs;
    int64_t eu, tu;
    detail::check(ldpcb_schedule_dims(h, &kind, &G, &slots, &gs, &s.overlap_ratio, &eu, &tu));
    s.kind = static_cast<ScheduleKind>(kind);
    s.n_groups = G;
    s.group_size = gs;
    std::vector<int32_t> off(G + 1), cns(slots > 0 ? slots : 1);
    detail::check(ldpcb_schedule_export(h, off.data(), cns.data()));
    s.groups.resize(G);
    for (int g = 0; g < G; ++g) s.groups[g].assign(cns.begin() + off[g], cns.begin() + off[g + 1]);
    return s;
  }
  ldpcb_schedule handle() const { return h_.get(); }

 private:
  std::shared_ptr<ldpcb_schedule_s> h_;
};

inline GroupSchedule make_flooding_schedule(const TannerGraph& g) {
  ldpcb_schedule h = nullptr;
  detail::check(ldpcb_schedule_flooding(g.handle(), &h));
  return GroupSchedule::from_handle(h);
}

inline GroupSchedule make_disjoint_schedule(const TannerGraph& g, int n_groups, std::uint64_t seed) {
  ldpcb_schedule h = nullptr;
  detail::check(ldpcb_schedule_disjoint(g.handle(), n_groups, seed, &h));
  return GroupSchedule::from_handle(h);
}

inline GroupSchedule make_nondisjoint_schedule(const TannerGraph& g, int n_groups, double overlap,
                                               std::uint64_t seed) {
  ldpcb_schedule h = nullptr;
  detail::check(ldpcb_schedule_nondisjoint(g.handle(), n_groups, overlap, seed, &h));
  return GroupSchedule::from_handle(h);
}

// run_sweep's grouping (sim.hpp:113-117): each frame draws its own groups
// from mix_seed(schedule_seed, frame_id), redrawn every iteration when
// regroup_each_iteration (decoder.hpp:153-156); generated on the device.
inline GroupSchedule make_per_frame_schedule(const TannerGraph& g, ScheduleKind kind, int n_groups, double overlap,
                                             std::uint64_t schedule_seed, bool regroup_each_iteration = true) {
  ldpcb_schedule h = nullptr;
  detail::check(ldpcb_schedule_per_frame(g.handle(), static_cast<int>(kind), n_groups, overlap, schedule_seed,
                                         regroup_each_iteration ? 1 : 0, &h));
  return GroupSchedule::from_handle(h);
}

inline GroupSchedule make_window_schedule(const TannerGraph& g, int n_groups, int window, int stride) {
  ldpcb_schedule h = nullptr;
  const int kind = window > stride ? LDPCB_NONDISJOINT : LDPCB_DISJOINT;
  detail::check(ldpcb_schedule_windows(g.handle(), kind, n_groups, window, stride, &h));
  return GroupSchedule::from_handle(h);
}

inline GroupSchedule schedule_from_groups(const TannerGraph& g, ScheduleKind kind,
                                          const std::vector<std::vector<int>>& groups) {
  std::vector<int32_t> off(1, 0), cns;
  for (const auto& grp : groups) {
    cns.insert(cns.end(), grp.begin(), grp.end());
    off.push_back(static_cast<int32_t>(cns.size()));
  }
  if (cns.empty()) cns.push_back(0);
  ldpcb_schedule h = nullptr;
  detail::check(ldpcb_schedule_from_groups(g.handle(), static_cast<int>(kind), static_cast<int>(groups.size()),
                                           off.data(), cns.data(), &h));
  return GroupSchedule::from_handle(h);
}

inline int iteration_budget(const GroupSchedule& s, int i_max) {
  int32_t b = 0;
  detail::check(ldpcb_schedule_iteration_budget(s.handle(), i_max, &b));
  return b;
}

inline double sigma2_from_ebn0(double ebn0_db, double rate) {
  double s2 = 0.0;
  detail::check(ldpcb_sigma2_from_ebn0(ebn0_db, rate, &s2));
  return s2;
}

struct DecodeOutcome {
  std::vector<std::uint8_t> bits;
  bool converged = false;
  int iterations = 0;
  std::vector<int> syndrome_weight_trace;  // unsatisfied checks per iteration
  long long cn_updates = 0;
};

// decode() with the reference signature (decoder.hpp:143-144); the LLRs are
// rounded to fp32 on the way to the device.
inline DecodeOutcome decode(const TannerGraph& g, const GroupSchedule& s, std::span<const double> channel_llr,
                            int max_iters) {
  if (max_iters < 1) throw std::invalid_argument("max_iters must be >= 1");
  if (static_cast<int>(channel_llr.size()) != g.n_vars)
    throw std::invalid_argument("channel LLR length does not match the code length");
  std::vector<float> x(channel_llr.begin(), channel_llr.end());
  DecodeOutcome out;
  out.bits.resize(g.n_vars);
  std::vector<int32_t> trace(max_iters);
  int32_t it = 0;
  uint8_t cv = 0;
  detail::check(ldpcb_decode_host(g.handle(), s.handle(), 1, x.data(), max_iters, 1, out.bits.data(), 0, &it, &cv,
                                  nullptr, trace.data(), nullptr));
  out.converged = cv != 0;
  out.iterations = it;
  out.syndrome_weight_trace.assign(trace.begin(), trace.begin() + it);
  long long slots = 0;
  for (const auto& grp : s.groups) slots += static_cast<long long>(grp.size());
  out.cn_updates = slots * it;
  return out;
}

// Batched decode of frames x n fp32 LLRs from host memory.
struct BatchOutcome {
  std::vector<std::uint8_t> bits;  // frames x n
  std::vector<int32_t> iterations;
  std::vector<std::uint8_t> converged;
  std::array<int64_t, 6> counters{};  // frames, bit_errors, frame_errors, converged, iter_sum, iter_sum_converged
};

inline BatchOutcome decode_batch(const TannerGraph& g, const GroupSchedule& s, std::span<const float> llr,
                                 int max_iters, bool early_stop = true) {
  if (llr.size() % static_cast<size_t>(g.n_vars))
    throw std::invalid_argument("channel LLR length does not match the code length");
  const int64_t frames = static_cast<int64_t>(llr.size() / g.n_vars);
  BatchOutcome out;
  out.bits.resize(llr.size());
  out.iterations.resize(frames);
  out.converged.resize(frames);
  detail::check(ldpcb_decode_host(g.handle(), s.handle(), frames, llr.data(), max_iters, early_stop ? 1 : 0,
                                  out.bits.data(), 0, out.iterations.data(), out.converged.data(), nullptr, nullptr,
                                  out.counters.data()));
  return out;
}

// Monte-Carlo frames [frame_begin, frame_begin+frames) with the device channel
// (run_frame + aggregation, sim.hpp:111-124, 162-181).
inline std::array<int64_t, 6> simulate(const TannerGraph& g, const GroupSchedule& s, double ebn0_db,
                                       std::uint64_t channel_seed, int64_t frame_begin, int64_t frames,
                                       int max_iters, bool early_stop = true) {
  const double rate = static_cast<double>(g.n_vars - g.n_checks) / g.n_vars;  // sim.hpp:103
  std::array<int64_t, 6> c{};
  detail::check(ldpcb_simulate_host(g.handle(), s.handle(), sigma2_from_ebn0(ebn0_db, rate), channel_seed,
                                    frame_begin, frames, max_iters, early_stop ? 1 : 0, c.data()));
  return c;
}

// simulate over several GPUs (ldpcb_simulate_multi): one host thread per
// entry of `devices`, contiguous frame-id ranges, counters summed
inline std::array<int64_t, 6> simulate(const TannerGraph& g, const GroupSchedule& s, double ebn0_db,
                                       std::uint64_t channel_seed, int64_t frame_begin, int64_t frames,
                                       int max_iters, bool early_stop, const std::vector<int>& devices) {
  const double rate = static_cast<double>(g.n_vars - g.n_checks) / g.n_vars;  // sim.hpp:103
  std::array<int64_t, 6> c{};
  detail::check(ldpcb_simulate_multi(g.handle(), s.handle(), devices.data(), static_cast<int>(devices.size()),
                                     sigma2_from_ebn0(ebn0_db, rate), channel_seed, frame_begin, frames, max_iters,
                                     early_stop ? 1 : 0, c.data()));
  return c;
}

// SimResult (sim.hpp:44-56)
struct SimResult {
  double ebn0_db = 0.0;
  long frames = 0;
  long long bit_errors = 0;
  long frame_errors = 0;
  long converged_frames = 0;
  double ber = 0.0;
  double fer = 0.0;
  double mean_iters_converged = 0.0;
  double mean_iters_all = 0.0;
  int iter_limit = 0;
  double wall_seconds = 0.0;
};

// run_sweep (sim.hpp:96-186) on the calling thread's GPU: frames 0,1,... per
// point until the smallest prefix holding min_frame_errors frame errors, or
// max_frames. Pass make_per_frame_schedule for the harness's own grouping.
// With a non-empty `devices` list every wave is split over those GPUs
// (ldpcb_run_sweep_multi); the result is the same for any device list.
inline std::vector<SimResult> run_sweep(const TannerGraph& g, const GroupSchedule& s,
                                        const std::vector<double>& ebn0_db, int iter_limit, long max_frames,
                                        int min_frame_errors, std::uint64_t channel_seed = 1,
                                        const std::vector<int>& devices = {}) {
  std::vector<double> raw(11 * ebn0_db.size());
  if (devices.empty())
    detail::check(ldpcb_run_sweep_host(g.handle(), s.handle(), ebn0_db.data(), static_cast<int>(ebn0_db.size()),
                                       iter_limit, max_frames, min_frame_errors, channel_seed, 0, raw.data()));
  else
    detail::check(ldpcb_run_sweep_multi(g.handle(), s.handle(), devices.data(), static_cast<int>(devices.size()),
                                        ebn0_db.data(), static_cast<int>(ebn0_db.size()), iter_limit, max_frames,
                                        min_frame_errors, channel_seed, 0, raw.data()));
  std::vector<SimResult> out(ebn0_db.size());
  for (std::size_t i = 0; i < out.size(); ++i) {
    const double* o = raw.data() + 11 * i;
    auto& r = out[i];
    r.frames = static_cast<long>(o[0]);
    r.bit_errors = static_cast<long long>(o[1]);
    r.frame_errors = static_cast<long>(o[2]);
    r.converged_frames = static_cast<long>(o[3]);
    r.ber = o[4];
    r.fer = o[5];
    r.mean_iters_converged = o[6];
    r.mean_iters_all = o[7];
    r.iter_limit = static_cast<int>(o[8]);
    r.wall_seconds = o[9];
    r.ebn0_db = o[10];
  }
  return out;
}

}  // namespace ldpc_b200
