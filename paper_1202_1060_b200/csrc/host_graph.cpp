// host_graph.cpp -- code construction, validation and alist I/O.
#include <algorithm>
#include <numeric>

#include "host.hpp"
#include "rng.cuh"

namespace ldpcb {

// Validation and CSR/CSC layout (tanner.hpp:79-114): indices in range, no
// repeated VN in a CN, CN degree >= 2, VN degree >= 1; VN view ascending.
CodeData build_code(int n_vars, const Rows& rows) {
  if (n_vars < 1 || rows.empty()) throw std::invalid_argument("graph must have at least one VN and one CN");
  CodeData c;
  c.n = n_vars;
  c.m = static_cast<int>(rows.size());
  c.row_off.assign(c.m + 1, 0);
  std::vector<char> mark(n_vars, 0);
  for (int r = 0; r < c.m; ++r) {
    const auto& row = rows[r];
    if (row.size() < 2) throw std::invalid_argument("check node " + std::to_string(r) + " has degree < 2");
    for (int v : row) {
      if (v < 0 || v >= n_vars) throw std::invalid_argument("VN index out of range in check node " + std::to_string(r));
      if (mark[v]) throw std::invalid_argument("duplicate VN in check node " + std::to_string(r));
      mark[v] = 1;
    }
    for (int v : row) mark[v] = 0;
    c.row_off[r + 1] = c.row_off[r] + static_cast<int>(row.size());
    c.max_cdeg = std::max(c.max_cdeg, static_cast<int>(row.size()));
  }
  c.E = c.row_off[c.m];
  c.cols.reserve(c.E);
  for (const auto& row : rows) c.cols.insert(c.cols.end(), row.begin(), row.end());

  c.var_off.assign(n_vars + 1, 0);
  for (int v : c.cols) ++c.var_off[v + 1];
  for (int v = 0; v < n_vars; ++v) {
    if (c.var_off[v + 1] == 0) throw std::invalid_argument("isolated VN " + std::to_string(v));
    c.max_vdeg = std::max(c.max_vdeg, c.var_off[v + 1]);
    c.var_off[v + 1] += c.var_off[v];
  }
  c.var_cns.resize(c.E);
  c.var_edges.resize(c.E);
  std::vector<int32_t> cursor(c.var_off.begin(), c.var_off.end() - 1);
  for (int r = 0; r < c.m; ++r)
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) {
      const int v = c.cols[e];
      c.var_cns[cursor[v]] = r;
      c.var_edges[cursor[v]] = e;
      ++cursor[v];
    }
  return c;
}

Rows rows_of(const CodeData& c) {
  Rows rows(c.m);
  for (int r = 0; r < c.m; ++r) rows[r].assign(c.cols.begin() + c.row_off[r], c.cols.begin() + c.row_off[r + 1]);
  return rows;
}

// Socket permutation with whole-draw rejection (tanner.hpp:356-393): socket s
// belongs to VN s / dv; CN r takes sockets [r*dc, (r+1)*dc); a draw with a
// repeated VN in any CN is discarded and the permutation shuffled again.
Rows regular_rows(int n_vars, int dv, int dc, uint64_t seed) {
  if (n_vars < 1 || dv < 1 || dc < 2) throw std::invalid_argument("need n_vars >= 1, d_v >= 1, d_c >= 2");
  const long long sockets = static_cast<long long>(n_vars) * dv;
  if (sockets % dc) throw std::invalid_argument("socket count " + std::to_string(sockets) + " is not divisible by d_c");
  const int m = static_cast<int>(sockets / dc);
  Stream rng(seed);
  std::vector<int> perm(sockets);
  std::iota(perm.begin(), perm.end(), 0);
  std::vector<char> mark(n_vars, 0);
  for (int attempt = 0; attempt < 20000; ++attempt) {
    rng.permute(perm.data(), static_cast<uint64_t>(sockets));
    bool ok = true;
    for (int r = 0; r < m && ok; ++r) {
      const int* s = perm.data() + static_cast<long long>(r) * dc;
      for (int k = 0; k < dc; ++k) {
        const int v = s[k] / dv;
        if (mark[v]) {
          ok = false;
          break;
        }
        mark[v] = 1;
      }
      for (int k = 0; k < dc; ++k) mark[s[k] / dv] = 0;
    }
    if (!ok) continue;
    Rows rows(m, std::vector<int>(dc));
    for (int r = 0; r < m; ++r)
      for (int k = 0; k < dc; ++k) rows[r][k] = perm[static_cast<long long>(r) * dc + k] / dv;
    return rows;
  }
  throw std::runtime_error("could not draw a duplicate-free regular graph after 20000 attempts");
}

namespace {

// Mutable bipartite view used by the repair passes below.
struct Wiring {
  Rows& rows;
  std::vector<std::vector<int>> cns_of;  // VN -> CNs (unordered)
  std::vector<int> edge_row, edge_slot;  // flat edge index -> (row, slot)
  std::vector<int> hits;                 // scratch, per CN

  Wiring(int n_vars, Rows& r) : rows(r), cns_of(n_vars), hits(r.size(), 0) {
    for (int i = 0; i < static_cast<int>(rows.size()); ++i)
      for (int k = 0; k < static_cast<int>(rows[i].size()); ++k) {
        cns_of[rows[i][k]].push_back(i);
        edge_row.push_back(i);
        edge_slot.push_back(k);
      }
  }

  bool row_holds(int r, int v) const { return std::find(rows[r].begin(), rows[r].end(), v) != rows[r].end(); }

  // Does CN r share two VNs with another CN (a length-4 cycle through r)?
  bool row_in_4cycle(int r) {
    bool found = false;
    std::vector<int> touched;
    for (int v : rows[r])
      for (int c : cns_of[v]) {
        if (c == r) continue;
        if (hits[c]++ == 0) touched.push_back(c);
        if (hits[c] >= 2) found = true;
      }
    for (int c : touched) hits[c] = 0;
    return found;
  }

  // First slot of r whose VN closes a 4-cycle, or -1.
  int cycle_slot(int r) {
    std::vector<int> touched;
    int bad_cn = -1;
    for (int v : rows[r])
      for (int c : cns_of[v]) {
        if (c == r) continue;
        if (hits[c]++ == 0) touched.push_back(c);
        if (hits[c] >= 2 && bad_cn < 0) bad_cn = c;
      }
    for (int c : touched) hits[c] = 0;
    if (bad_cn < 0) return -1;
    for (int k = 0; k < static_cast<int>(rows[r].size()); ++k)
      if (row_holds(bad_cn, rows[r][k])) return k;
    return -1;
  }

  void relink(int v, int from, int to) {
    auto& l = cns_of[v];
    *std::find(l.begin(), l.end(), from) = to;
  }

  // Exchange the VNs on edges (r1,k1) and (r2,k2).
  void swap_edges(int r1, int k1, int r2, int k2) {
    const int v1 = rows[r1][k1], v2 = rows[r2][k2];
    rows[r1][k1] = v2;
    rows[r2][k2] = v1;
    relink(v1, r1, r2);
    relink(v2, r2, r1);
  }
};

}  // namespace

// Deterministic 4-cycle breaking: every CN on a 4-cycle exchanges the VN on
// one offending edge with the VN on a uniformly drawn edge elsewhere; the
// exchange is kept only if it creates no repeated VN and leaves both CNs off
// every 4-cycle. Degrees of all VNs and CNs are unchanged.
void break_4cycles(int n_vars, Rows& rows, uint64_t seed) {
  Wiring w(n_vars, rows);
  const uint64_t E = w.edge_row.size();
  Stream rng(stream_seed(seed, 0x4c44504334ull));
  for (int pass = 0; pass < 400; ++pass) {
    std::vector<int> bad;
    for (int r = 0; r < static_cast<int>(rows.size()); ++r)
      if (w.row_in_4cycle(r)) bad.push_back(r);
    if (bad.empty()) return;
    for (int r : bad) {
      const int k = w.cycle_slot(r);
      if (k < 0) continue;
      for (int attempt = 0; attempt < 2000; ++attempt) {
        const uint64_t e = rng.below(E);
        const int r2 = w.edge_row[e], k2 = w.edge_slot[e];
        if (r2 == r) continue;
        const int v1 = rows[r][k], v2 = rows[r2][k2];
        if (v1 == v2 || w.row_holds(r, v2) || w.row_holds(r2, v1)) continue;
        w.swap_edges(r, k, r2, k2);
        if (!w.row_in_4cycle(r) && !w.row_in_4cycle(r2)) break;
        w.swap_edges(r, k, r2, k2);  // undo
      }
    }
  }
  throw std::runtime_error("could not remove all 4-cycles");
}

// Base matrix J x K: each entry is empty with probability p_empty, otherwise
// a circulant shift drawn uniformly from [0, z); columns (then rows) short of
// the minimum degree receive extra entries at random positions. Check
// (r, i) connects VN c*z + (i + shift) mod z for every present entry, columns
// ascending.
Rows qc_rows(int J, int K, int z, double p_empty, int min_col_degree, uint64_t seed) {
  if (J < 1 || K < 1 || z < 1) throw std::invalid_argument("QC base matrix needs J, K, Z >= 1");
  if (!(p_empty >= 0.0 && p_empty < 1.0)) throw std::invalid_argument("p_empty must be in [0, 1)");
  if (min_col_degree > J || K < 2) throw std::invalid_argument("infeasible QC degree constraints");
  Stream rng(seed);
  std::vector<int> base(static_cast<size_t>(J) * K, -1);
  for (int r = 0; r < J; ++r)
    for (int c = 0; c < K; ++c)
      if (rng.unit() > p_empty) base[r * K + c] = static_cast<int>(rng.below(z));
  auto col_deg = [&](int c) {
    int d = 0;
    for (int r = 0; r < J; ++r) d += base[r * K + c] >= 0;
    return d;
  };
  auto row_deg = [&](int r) {
    int d = 0;
    for (int c = 0; c < K; ++c) d += base[r * K + c] >= 0;
    return d;
  };
  for (int c = 0; c < K; ++c)
    while (col_deg(c) < min_col_degree) {
      const int r = static_cast<int>(rng.below(J));
      if (base[r * K + c] < 0) base[r * K + c] = static_cast<int>(rng.below(z));
    }
  for (int r = 0; r < J; ++r)
    while (row_deg(r) < 2) {
      const int c = static_cast<int>(rng.below(K));
      if (base[r * K + c] < 0) base[r * K + c] = static_cast<int>(rng.below(z));
    }
  Rows rows(static_cast<size_t>(J) * z);
  for (int r = 0; r < J; ++r)
    for (int i = 0; i < z; ++i) {
      auto& row = rows[static_cast<size_t>(r) * z + i];
      for (int c = 0; c < K; ++c) {
        const int s = base[r * K + c];
        if (s >= 0) row.push_back(c * z + (i + s) % z);
      }
    }
  return rows;
}

// VN degrees assigned in class order (first counts[0] VNs get degrees[0],
// ...); sockets permuted once; CN r takes sockets [r*dc, (r+1)*dc); repeated
// VNs inside a CN are repaired by exchanges with uniformly drawn edges.
Rows irregular_rows(int n_vars, const std::vector<int>& degrees, const std::vector<int>& counts, int dc,
                    uint64_t seed) {
  if (degrees.size() != counts.size() || degrees.empty()) throw std::invalid_argument("degree classes mismatch");
  if (dc < 2) throw std::invalid_argument("need d_c >= 2");
  long long total = 0, sockets = 0;
  for (size_t i = 0; i < degrees.size(); ++i) {
    if (degrees[i] < 1 || counts[i] < 0) throw std::invalid_argument("bad degree class");
    total += counts[i];
    sockets += static_cast<long long>(degrees[i]) * counts[i];
  }
  if (total != n_vars) throw std::invalid_argument("degree class counts must sum to n_vars");
  if (sockets % dc) throw std::invalid_argument("socket count is not divisible by d_c");
  std::vector<int> sock;
  sock.reserve(sockets);
  int v = 0;
  for (size_t i = 0; i < degrees.size(); ++i)
    for (int j = 0; j < counts[i]; ++j, ++v)
      for (int d = 0; d < degrees[i]; ++d) sock.push_back(v);
  Stream rng(seed);
  rng.permute(sock.data(), sock.size());
  const int m = static_cast<int>(sockets / dc);
  Rows rows(m, std::vector<int>(dc));
  for (int r = 0; r < m; ++r)
    for (int k = 0; k < dc; ++k) rows[r][k] = sock[static_cast<size_t>(r) * dc + k];

  Wiring w(n_vars, rows);
  Stream fix(stream_seed(seed, 0x445550ull));
  for (int r = 0; r < m; ++r) {
    for (int k = 0; k < dc; ++k) {
      auto repeated = [&]() {
        for (int j = 0; j < dc; ++j)
          if (j != k && rows[r][j] == rows[r][k]) return true;
        return false;
      };
      int guard = 0;
      while (repeated()) {
        if (++guard > 100000) throw std::runtime_error("could not repair repeated edges");
        const uint64_t e = fix.below(sockets);
        const int r2 = w.edge_row[e], k2 = w.edge_slot[e];
        if (r2 == r) continue;
        const int v1 = rows[r][k], v2 = rows[r2][k2];
        if (w.row_holds(r, v2) || w.row_holds(r2, v1)) continue;
        w.swap_edges(r, k, r2, k2);
      }
    }
  }
  return rows;
}

int64_t count_4cycles(const CodeData& c) {
  int64_t total = 0;
  std::vector<int> hits(c.m, 0);
  std::vector<int> touched;
  for (int r = 0; r < c.m; ++r) {
    touched.clear();
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) {
      const int v = c.cols[e];
      for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) {
        const int r2 = c.var_cns[j];
        if (r2 <= r) continue;
        if (hits[r2]++ == 0) touched.push_back(r2);
      }
    }
    for (int r2 : touched) {
      total += static_cast<int64_t>(hits[r2]) * (hits[r2] - 1) / 2;
      hits[r2] = 0;
    }
  }
  return total;
}

// ---------------------------------------------------------------- alist ----

namespace {

struct Line {
  int no = 0;
  std::vector<long long> vals;
};

std::vector<Line> tokenize(std::string_view text) {
  std::vector<Line> out;
  size_t pos = 0;
  int no = 0;
  while (pos <= text.size()) {
    size_t end = text.find('\n', pos);
    const std::string_view s = text.substr(pos, end == std::string_view::npos ? std::string_view::npos : end - pos);
    ++no;
    Line ln;
    ln.no = no;
    auto blank = [](char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; };
    size_t i = 0;
    while (i < s.size()) {
      while (i < s.size() && blank(s[i])) ++i;
      if (i == s.size()) break;
      bool neg = false;
      if (s[i] == '-') {
        neg = true;
        ++i;
      }
      if (i == s.size() || s[i] < '0' || s[i] > '9') throw AlistFailure(AlistKind::bad_token, no, "non-numeric token");
      long long x = 0;
      while (i < s.size() && s[i] >= '0' && s[i] <= '9') {
        x = x * 10 + (s[i] - '0');
        if (x > (1ll << 40)) throw AlistFailure(AlistKind::bad_token, no, "token out of range");
        ++i;
      }
      if (i < s.size() && !blank(s[i])) throw AlistFailure(AlistKind::bad_token, no, "non-numeric token");
      ln.vals.push_back(neg ? -x : x);
    }
    if (!ln.vals.empty()) out.push_back(std::move(ln));
    if (end == std::string_view::npos) break;
    pos = end + 1;
  }
  return out;
}

}  // namespace

// Same grammar, checks and error kinds/lines as tanner.hpp:163-282.
CodeData parse_alist(std::string_view text) {
  const auto lines = tokenize(text);
  size_t cur = 0;
  auto next = [&](const char* what) -> const Line& {
    if (cur >= lines.size())
      throw AlistFailure(AlistKind::truncated, lines.empty() ? 1 : lines.back().no,
                         std::string("unexpected end of input, expected ") + what);
    return lines[cur++];
  };
  const Line& hdr = next("N M header");
  if (hdr.vals.size() != 2 || hdr.vals[0] < 1 || hdr.vals[1] < 1)
    throw AlistFailure(AlistKind::malformed_header, hdr.no, "expected two positive integers N M");
  const int n = static_cast<int>(hdr.vals[0]), m = static_cast<int>(hdr.vals[1]);
  const Line& mx = next("max degree header");
  if (mx.vals.size() != 2 || mx.vals[0] < 1 || mx.vals[1] < 1)
    throw AlistFailure(AlistKind::malformed_header, mx.no, "expected two positive maximum degrees");
  const int max_col = static_cast<int>(mx.vals[0]), max_row = static_cast<int>(mx.vals[1]);

  auto degrees = [&](int count, int cap, bool col) {
    std::vector<int> d;
    while (static_cast<int>(d.size()) < count) {
      const Line& ln = next(col ? "column degrees" : "row degrees");
      for (long long x : ln.vals) {
        if (static_cast<int>(d.size()) == count)
          throw AlistFailure(AlistKind::length_mismatch, ln.no, "too many degree entries");
        if (x < 1)
          throw AlistFailure(AlistKind::degree_error, ln.no, col ? "degree-0 column (isolated VN)" : "row degree below 1");
        if (!col && x < 2) throw AlistFailure(AlistKind::degree_error, ln.no, "check node of degree < 2");
        if (x > cap) throw AlistFailure(AlistKind::degree_error, ln.no, "degree exceeds declared maximum");
        d.push_back(static_cast<int>(x));
      }
    }
    return d;
  };
  const auto cdeg = degrees(n, max_col, true);
  const int rdeg_line = cur < lines.size() ? lines[cur].no : 0;
  const auto rdeg = degrees(m, max_row, false);
  const long long ce = std::accumulate(cdeg.begin(), cdeg.end(), 0ll);
  const long long re = std::accumulate(rdeg.begin(), rdeg.end(), 0ll);
  if (ce != re)
    throw AlistFailure(AlistKind::edge_count_mismatch, rdeg_line,
                       "column degrees sum to " + std::to_string(ce) + " but row degrees sum to " + std::to_string(re));

  auto list = [&](int want, int cap, int bound, const char* what, int* line_no) {
    const Line& ln = next(what);
    if (static_cast<int>(ln.vals.size()) > cap)
      throw AlistFailure(AlistKind::length_mismatch, ln.no, "more entries than the declared maximum degree");
    std::vector<int> out;
    for (long long x : ln.vals) {
      if (x == 0) continue;
      if (x < 0 || x > bound)
        throw AlistFailure(AlistKind::index_out_of_range, ln.no, "index " + std::to_string(x) + " out of range");
      out.push_back(static_cast<int>(x) - 1);
    }
    if (static_cast<int>(out.size()) != want)
      throw AlistFailure(AlistKind::length_mismatch, ln.no,
                         "list has " + std::to_string(out.size()) + " entries, declared degree is " +
                             std::to_string(want));
    std::vector<char> seen(bound, 0);
    for (int x : out) {
      if (seen[x]) throw AlistFailure(AlistKind::duplicate_entry, ln.no, "duplicate index in list");
      seen[x] = 1;
    }
    if (line_no) *line_no = ln.no;
    return out;
  };
  Rows col_lists(n), row_lists(m);
  std::vector<int> row_line(m);
  for (int v = 0; v < n; ++v) col_lists[v] = list(cdeg[v], max_col, m, "column neighbor list", nullptr);
  for (int r = 0; r < m; ++r) row_lists[r] = list(rdeg[r], max_row, n, "row neighbor list", &row_line[r]);
  if (cur != lines.size())
    throw AlistFailure(AlistKind::trailing_content, lines[cur].no, "trailing content after row lists");

  Rows induced(m);
  for (int v = 0; v < n; ++v)
    for (int r : col_lists[v]) induced[r].push_back(v);
  for (int r = 0; r < m; ++r) {
    auto a = row_lists[r];
    std::sort(a.begin(), a.end());
    std::sort(induced[r].begin(), induced[r].end());
    if (a != induced[r])
      throw AlistFailure(AlistKind::transpose_mismatch, row_line[r],
                         "row list of check " + std::to_string(r + 1) + " does not match the column lists");
  }
  try {
    return build_code(n, row_lists);
  } catch (const std::invalid_argument& e) {
    throw AlistFailure(AlistKind::degree_error, 1, e.what());
  }
}

// Zero-padded alist (tanner.hpp:286-317); parse_alist(serialize_alist(c))
// reproduces c.
std::string serialize_alist(const CodeData& c) {
  if (c.n < 1 || c.m < 1) throw std::invalid_argument("cannot serialize an empty graph");
  std::string s;
  auto put = [&s](const std::vector<int>& xs) {
    for (size_t i = 0; i < xs.size(); ++i) {
      if (i) s += ' ';
      s += std::to_string(xs[i]);
    }
    s += '\n';
  };
  put({c.n, c.m});
  put({c.max_vdeg, c.max_cdeg});
  std::vector<int> d(c.n);
  for (int v = 0; v < c.n; ++v) d[v] = c.var_off[v + 1] - c.var_off[v];
  put(d);
  d.assign(c.m, 0);
  for (int r = 0; r < c.m; ++r) d[r] = c.row_off[r + 1] - c.row_off[r];
  put(d);
  for (int v = 0; v < c.n; ++v) {
    std::vector<int> l(c.max_vdeg, 0);
    for (int j = c.var_off[v]; j < c.var_off[v + 1]; ++j) l[j - c.var_off[v]] = c.var_cns[j] + 1;
    put(l);
  }
  for (int r = 0; r < c.m; ++r) {
    std::vector<int> l(c.max_cdeg, 0);
    for (int e = c.row_off[r]; e < c.row_off[r + 1]; ++e) l[e - c.row_off[r]] = c.cols[e] + 1;
    put(l);
  }
  return s;
}

}  // namespace ldpcb
