// C++ host API tests (include/ldpc_b200.hpp), written like the reference's
// own Catch2 suites (proj/tests/test_tanner.cpp, test_schedule.cpp,
// test_channel.cpp, test_decoder.cpp) but self-contained. `test_api` runs the
// host-only cases; `test_api gpu` adds the decoding cases.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "ldpc_b200.hpp"

using namespace ldpc_b200;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++failures;                                                        \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                      \
  do {                                                                   \
    bool thrown = false;                                                 \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (const type&) {                                              \
      thrown = true;                                                     \
    }                                                                    \
    if (!thrown) {                                                       \
      std::printf("FAIL %s:%d: %s did not throw\n", __FILE__, __LINE__, #expr); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static TannerGraph fig1() { return build_from_check_lists(8, {{0, 1, 2}, {1, 3, 4}, {3, 5, 6}, {5, 7}}); }

static void host_cases() {
  // tanner.hpp: construction, determinism, alist round trip and errors
  const TannerGraph g = fig1();
  CHECK(g.n_vars == 8 && g.n_checks == 4 && g.n_edges == 11);
  CHECK_THROWS_AS(build_from_check_lists(4, {{0, 1}, {2}}), std::invalid_argument);
  CHECK_THROWS_AS(build_from_check_lists(4, {{0, 0}, {1, 2}}), std::invalid_argument);
  const TannerGraph r = random_regular_graph(504, 3, 6, 1);
  CHECK(r.n_checks == 252);
  for (const auto& row : r.check_adj()) CHECK(row.size() == 6);
  CHECK(random_regular_graph(60, 3, 6, 42) == random_regular_graph(60, 3, 6, 42));
  CHECK(!(random_regular_graph(60, 3, 6, 42) == random_regular_graph(60, 3, 6, 43)));
  CHECK_THROWS_AS(random_regular_graph(5, 3, 6, 1), std::invalid_argument);
  CHECK(parse_alist(serialize_alist(r)) == r);
  CHECK(parse_alist(serialize_alist(g)) == g);
  try {
    parse_alist("8\n2 3\n");
    CHECK(false);
  } catch (const AlistError& e) {
    CHECK(e.kind() == AlistErrorKind::malformed_header && e.line() == 1);
  }
  const TannerGraph c1 = random_regular_graph_girth6(1008, 3, 6, 1);
  CHECK(c1.count_4cycles() == 0);

  // schedule.hpp: the paper's overlapped construction and its budget
  const TannerGraph s504 = random_regular_graph(504, 3, 6, 3);
  const GroupSchedule nd = make_nondisjoint_schedule(s504, 12, 0.4, 123);
  CHECK(nd.group_size == 34 && nd.groups.size() == 12 && nd.groups[11].size() == 32);
  CHECK(iteration_budget(nd, 1000) == 627);
  const GroupSchedule gs = make_disjoint_schedule(s504, 12, 17);
  for (const auto& grp : gs.groups) CHECK(grp.size() == 21);
  CHECK_THROWS_AS(make_nondisjoint_schedule(s504, 12, 1.0, 1), std::invalid_argument);
  const GroupSchedule w = make_window_schedule(c1, 8, 84, 63);
  CHECK(w.kind == ScheduleKind::nondisjoint && w.groups.size() == 8 && w.groups[7][83] == (441 + 83) % 504);

  // channel.hpp
  CHECK(std::abs(sigma2_from_ebn0(0.0, 0.5) - 1.0) < 1e-12);
  CHECK(std::abs(sigma2_from_ebn0(1.163, 0.5) - 0.76506) < 1e-4);
  CHECK_THROWS_AS(sigma2_from_ebn0(1.0, 0.0), std::invalid_argument);
}

static void gpu_cases() {
  // decoder.hpp: noiseless input converges in one iteration (test_decoder.cpp:149-156)
  const TannerGraph g = random_regular_graph(60, 3, 6, 21);
  const auto out = decode(g, make_flooding_schedule(g), std::vector<double>(60, 1e9), 10);
  CHECK(out.converged && out.iterations == 1);
  for (auto b : out.bits) CHECK(b == 0);
  // a saturated codeword is a fixed point (:158-168)
  const TannerGraph f = fig1();
  const std::vector<std::uint8_t> word{1, 1, 0, 1, 0, 1, 0, 1};
  std::vector<double> llr(8);
  for (int n = 0; n < 8; ++n) llr[n] = word[n] ? -30.0 : 30.0;
  const auto fp = decode(f, make_flooding_schedule(f), llr, 5);
  CHECK(fp.converged && fp.iterations == 1 && fp.bits == word);
  CHECK(fp.syndrome_weight_trace.size() == 1 && fp.syndrome_weight_trace[0] == 0);
  // preconditions (decoder.hpp:40-41, 145)
  CHECK_THROWS_AS(decode(g, make_flooding_schedule(g), std::vector<double>(59, 0.0), 10), std::invalid_argument);
  CHECK_THROWS_AS(decode(g, make_flooding_schedule(g), std::vector<double>(60, 0.0), 0), std::invalid_argument);

  // batch vs single-frame decode, counters, converged => zero syndrome
  const TannerGraph c1 = random_regular_graph_girth6(1008, 3, 6, 1);
  const GroupSchedule nd = make_window_schedule(c1, 8, 84, 63);
  std::mt19937_64 rng(5);
  std::normal_distribution<double> z(0.0, 1.0);
  const double s2 = sigma2_from_ebn0(1.5, 0.5);
  const int frames = 64;
  std::vector<float> x(frames * 1008);
  for (auto& v : x) v = static_cast<float>(2.0 / s2 * (1.0 + std::sqrt(s2) * z(rng)));
  const auto batch = decode_batch(c1, nd, x, 20);
  CHECK(batch.counters[0] == frames);
  const auto rows = c1.check_adj();
  long long bit_errors = 0;
  for (int fr = 0; fr < frames; ++fr) {
    std::vector<double> one(x.begin() + fr * 1008, x.begin() + (fr + 1) * 1008);
    const auto single = decode(c1, nd, one, 20);
    CHECK(single.iterations == batch.iterations[fr]);
    CHECK(std::memcmp(single.bits.data(), batch.bits.data() + fr * 1008, 1008) == 0);
    if (single.converged) {
      for (const auto& row : rows) {
        int p = 0;
        for (int v : row) p ^= single.bits[v];
        CHECK(p == 0);
      }
    }
    for (auto b : single.bits) bit_errors += b;
  }
  CHECK(batch.counters[1] == bit_errors);
  const auto sim = simulate(c1, nd, 2.0, 1, 0, 1000, 20);
  CHECK(sim[0] == 1000 && sim[2] <= sim[0] && sim[4] >= sim[0]);
  std::printf("simulate 1000 frames @2.0 dB: frame errors %lld, mean iterations %.3f\n",
              static_cast<long long>(sim[2]), static_cast<double>(sim[4]) / sim[0]);

  // run_sweep with the harness's per-frame regrouping (sim.hpp:96-186)
  const GroupSchedule pf = make_per_frame_schedule(c1, ScheduleKind::nondisjoint, 8, 0.25, 2, true);
  const auto res = run_sweep(c1, pf, {1.5, 2.0}, 20, 100000, 25);
  CHECK(res.size() == 2 && res[0].ebn0_db == 1.5 && res[1].ebn0_db == 2.0);
  for (const auto& r : res) {
    CHECK(r.frame_errors == 25 && r.frames < 100000 && r.iter_limit == 20);
    CHECK(r.fer == static_cast<double>(r.frame_errors) / r.frames);
  }
  CHECK(res[1].frames > res[0].frames);
  CHECK_THROWS_AS(run_sweep(c1, pf, {}, 20, 10, 1), std::invalid_argument);

  // several GPUs through the boundary (the north-star split, sim.hpp:96-186
  // driven from C++): device 0 listed twice = two workers with contiguous
  // frame ranges; counters and sweep records equal the one-device results
  const auto sim2 = simulate(c1, nd, 2.0, 1, 0, 1000, 20, true, {0, 0});
  CHECK(sim2 == sim);
  const auto res2 = run_sweep(c1, pf, {1.5, 2.0}, 20, 100000, 25, 1, {0, 0, 0});
  CHECK(res2.size() == res.size());
  for (std::size_t i = 0; i < res.size() && i < res2.size(); ++i) {
    CHECK(res2[i].frames == res[i].frames && res2[i].bit_errors == res[i].bit_errors);
    CHECK(res2[i].frame_errors == res[i].frame_errors && res2[i].converged_frames == res[i].converged_frames);
    CHECK(res2[i].mean_iters_all == res[i].mean_iters_all);
  }
  CHECK_THROWS_AS(simulate(c1, nd, 2.0, 1, 0, 10, 20, true, {}), std::invalid_argument);
  CHECK_THROWS_AS(simulate(c1, nd, 2.0, 1, 0, 10, 20, true, {0, 4096}), std::invalid_argument);
  CHECK_THROWS_AS(make_per_frame_schedule(c1, ScheduleKind::nondisjoint, 8, 0.9, 2), std::invalid_argument);
}

int main(int argc, char** argv) {
  try {
    host_cases();
    if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) gpu_cases();
  } catch (const std::exception& e) {
    std::printf("FAIL: uncaught %s\n", e.what());
    ++failures;
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
