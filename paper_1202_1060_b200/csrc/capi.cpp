// capi.cpp -- the extern "C" boundary (include/ldpc_b200.h): handles,
// validation, error mapping, device uploads and stream orchestration.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <exception>

#include "host.hpp"
#include "kernels.cuh"
#include "rng.cuh"
#include "ldpc_b200.h"

namespace {

thread_local std::string g_last_error;

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
void cuda_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

template <class F>
int guard(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const ldpcb::AlistFailure& e) {
    g_last_error = e.what();
    return LDPCB_EALIST;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return LDPCB_EINVAL;
  } catch (const CudaFailure& e) {
    g_last_error = e.what();
    return LDPCB_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LDPCB_ERUNTIME;
  }
}

template <class T>
T* upload(const std::vector<T>& v) {
  T* d = nullptr;
  const size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  cuda_check(cudaMalloc(&d, bytes), "cudaMalloc");
  if (!v.empty()) cuda_check(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy");
  return d;
}

void free_on(int dev, std::vector<void*>& ptrs) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  cudaSetDevice(dev);
  for (void* p : ptrs) cudaFree(p);
  cudaSetDevice(cur);
  ptrs.clear();
}

struct CodeImpl {
  ldpcb::CodeData host;
  bool cregular = true, vregular = true;
  std::mutex mu;
  struct Dev {
    int32_t* cols;
    std::vector<void*> ptrs;
  };
  std::map<int, Dev> dev;

  explicit CodeImpl(ldpcb::CodeData c) : host(std::move(c)) {
    for (int r = 0; r < host.m; ++r) cregular &= (host.row_off[r + 1] - host.row_off[r]) == host.max_cdeg;
    for (int v = 0; v < host.n; ++v) vregular &= (host.var_off[v + 1] - host.var_off[v]) == host.max_vdeg;
  }
  ~CodeImpl() {
    for (auto& kv : dev) free_on(kv.first, kv.second.ptrs);
  }
  const Dev& device() {
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find(d);
    if (it != dev.end()) return it->second;
    Dev x;
    x.cols = upload(host.cols);
    x.ptrs = {x.cols};
    // a pageable cudaMemcpy may return before its DMA lands, and decodes run
    // on non-blocking streams that do not order after the legacy stream
    cuda_check(cudaDeviceSynchronize(), "table upload");
    return dev.emplace(d, std::move(x)).first->second;
  }
};

struct SchedImpl {
  std::shared_ptr<CodeImpl> code;
  ldpcb::ScheduleData host;
  ldpcb::KernelTables tables;
  ldpcb::DirectTables direct;
  std::mutex mu;
  struct Dev {
    int32_t *cn_off, *cn_rec, *fix_off, *fix_rec, *fix_rec16, *tot_rec16, *all_vn_rec, *tot_vn_rec, *all_rec, *edge_slot, *vn_pos;
    uint32_t *cn_fresh, *fix_fresh;
    int32_t *d_cn_rec = nullptr, *d_vn_rec = nullptr, *d_all_cn = nullptr, *d_edge_rec = nullptr,
            *d_vn_pos = nullptr, *d_vn_hold = nullptr;
    std::vector<void*> ptrs;
  };
  std::map<int, Dev> dev;

  ~SchedImpl() {
    for (auto& kv : dev) free_on(kv.first, kv.second.ptrs);
  }
  const Dev& device() {
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find(d);
    if (it != dev.end()) return it->second;
    Dev x;
    x.cn_off = upload(tables.cn_off);
    x.cn_rec = upload(tables.cn_rec);
    x.fix_off = upload(tables.fix_off);
    x.fix_rec = upload(tables.fix_rec);
    x.fix_rec16 = upload(tables.fix_rec16);
    x.tot_rec16 = upload(tables.tot_rec16);
    x.all_vn_rec = upload(tables.all_vn_rec);
    x.tot_vn_rec = upload(tables.tot_vn_rec);
    x.all_rec = upload(tables.all_rec);
    x.edge_slot = upload(tables.edge_slot);
    x.vn_pos = upload(tables.vn_pos);
    x.cn_fresh = upload(tables.cn_fresh);
    x.fix_fresh = upload(tables.fix_fresh);
    x.ptrs = {x.cn_off,     x.cn_rec,     x.fix_off, x.fix_rec,   x.fix_rec16, x.tot_rec16,
              x.all_vn_rec, x.tot_vn_rec, x.all_rec, x.edge_slot, x.vn_pos,  x.cn_fresh, x.fix_fresh};
    if (direct.ok) {
      x.d_cn_rec = upload(direct.cn_rec);
      x.d_vn_rec = upload(direct.vn_rec);
      x.d_all_cn = upload(direct.all_cn);
      x.d_edge_rec = upload(direct.edge_rec);
      x.d_vn_pos = upload(direct.vn_pos);
      x.d_vn_hold = upload(direct.vn_hold);
      x.ptrs.push_back(x.d_vn_hold);
      for (void* q : {static_cast<void*>(x.d_cn_rec), static_cast<void*>(x.d_vn_rec),
                      static_cast<void*>(x.d_all_cn), static_cast<void*>(x.d_edge_rec), static_cast<void*>(x.d_vn_pos)})
        x.ptrs.push_back(q);
    }
    // The record tables are immutable once uploaded: the streamed kernels
    // read them before griddepcontrol.wait (stream.cu). Wait for the DMA of
    // the pageable copies here, since decodes run on non-blocking streams
    // that are not ordered after the legacy stream.
    cuda_check(cudaDeviceSynchronize(), "table upload");
    return dev.emplace(d, std::move(x)).first->second;
  }
};

}  // namespace

struct ldpcb_code_s {
  std::shared_ptr<CodeImpl> impl;
};
struct ldpcb_schedule_s {
  std::shared_ptr<SchedImpl> impl;
};

namespace {

void need(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

int make_code(ldpcb::CodeData c, ldpcb_code* out) {
  need(out != nullptr, "null output handle");
  *out = new ldpcb_code_s{std::make_shared<CodeImpl>(std::move(c))};
  return LDPCB_OK;
}

int make_sched(const std::shared_ptr<CodeImpl>& code, ldpcb::ScheduleData s, ldpcb_schedule* out) {
  need(out != nullptr, "null output handle");
  auto impl = std::make_shared<SchedImpl>();
  impl->code = code;
  impl->host = std::move(s);
  const int bucket = ldpcb::cn_bucket(code->host.max_cdeg, code->cregular);
  if (bucket > 0) {
    // packed 16-byte CN records (common.cuh CnRecord) where the fields fit
    const auto& h = code->host;
    // (the resident kernel requires them for these buckets; such codes always have n < 65536)
    const bool packed = (bucket == 3 || bucket == 6) && h.n < 65536 && static_cast<long long>(h.m) * 7 + 1 < (1 << 24);
    impl->tables = ldpcb::kernel_tables(h, impl->host, packed ? 4 : ldpcb::cn_record_stride(bucket), code->cregular);
    // the posterior-free kernel's tables (direct.cu) where the code and the groups qualify;
    // LDPCB_DIRECT_FV = frames per thread (2 or 4; A/B)
    if (ldpcb::direct_enabled()) {
      const char* e = std::getenv("LDPCB_DIRECT_FV");
      impl->direct = ldpcb::direct_tables(h, impl->host, e ? std::atoi(e) : 2);
    }
  }
  *out = new ldpcb_schedule_s{impl};
  return LDPCB_OK;
}

// Keep freed stream-ordered allocations in the device's default pool instead
// of returning them to the driver at every synchronisation: the host entry
// points allocate multi-GB chunk state per call.
void retain_pool_memory() {
  static std::mutex mu;
  static std::map<int, bool> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

// Host-buffer entry points work on two non-blocking streams per (host
// thread, device) that live as long as the thread: stream-ordered pool
// allocations freed on them are reused by the next call without fresh
// physical mappings (a new stream per call made every multi-GB chunk
// allocation map new memory and serialised the copy/decode pipeline).
struct HostStreams {
  std::map<int, std::array<cudaStream_t, 2>> by_dev;
  ~HostStreams() {
    for (auto& kv : by_dev)
      for (cudaStream_t st : kv.second) cudaStreamDestroy(st);  // errors ignored at teardown
  }
  cudaStream_t get(int k) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    auto it = by_dev.find(dev);
    if (it == by_dev.end()) {
      std::array<cudaStream_t, 2> st{};
      for (auto& x : st) cuda_check(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
      it = by_dev.emplace(dev, st).first;
    }
    return it->second[k];
  }
};
cudaStream_t host_stream(int k) {
  thread_local HostStreams streams;
  return streams.get(k);
}

void check_pair(ldpcb_code code, ldpcb_schedule s) {
  need(code && s, "null handle");
  need(s->impl->code.get() == code->impl.get(), "schedule was built for a different code");
}

ldpcb::DevGraph dev_graph(ldpcb_code code, ldpcb_schedule s) {
  check_pair(code, s);
  retain_pool_memory();
  const auto& c = code->impl->device();
  const auto& d = s->impl->device();
  const auto& h = code->impl->host;
  ldpcb::DevGraph g;
  g.n = h.n;
  g.m = h.m;
  g.E = h.E;
  g.G = s->impl->host.G;
  g.max_cdeg = h.max_cdeg;
  g.max_vdeg = h.max_vdeg;
  g.cregular = code->impl->cregular;
  g.vregular = code->impl->vregular;
  const auto& t = s->impl->tables;
  if (t.cs == 0) throw std::runtime_error("check-node degree above 32 is not supported by the resident kernel");
  g.cs = t.cs;
  g.vs4 = t.vs4;
  g.n_slots = t.n_slots;
  g.recompute = t.recompute;
  g.max_cn_items = t.max_cn_items;
  g.max_fix_items = t.max_fix_items;
  g.cols = c.cols;
  g.edge_slot = d.edge_slot;
  g.vn_pos = d.vn_pos;
  g.cn_off = d.cn_off;
  g.cn_rec = d.cn_rec;
  g.fix_off = d.fix_off;
  g.fix_rec = d.fix_rec;
  g.fix_rec16 = t.vs16 && !std::getenv("LDPCB_NO_FIX16") ? d.fix_rec16 : nullptr;
  g.vs16 = g.fix_rec16 ? t.vs16 : 0;
  g.tot_rec16 = g.vs16 ? d.tot_rec16 : nullptr;
  g.all_vn_rec = d.all_vn_rec;
  g.tot_vn_rec = d.tot_vn_rec;
  g.all_rec = d.all_rec;
  g.cn_fresh = d.cn_fresh;
  g.fix_fresh = d.fix_fresh;
  g.covers = t.covers;
  const auto& dt = s->impl->direct;
  if (dt.ok) {
    g.d_fv = dt.fv;
    g.d_cells = dt.cells;
    g.d_l_base = dt.l_base;
    g.d_buf_cells = dt.buf_cells;
    g.d_max_items = dt.max_items;
    for (size_t i = 0; i < dt.cn_off.size(); ++i) g.d_goff[i] = static_cast<uint16_t>(dt.cn_off[i]);
    g.d_cn_rec = d.d_cn_rec;
    g.d_vn_rec = d.d_vn_rec;
    g.d_all_cn = d.d_all_cn;
    g.d_edge_rec = d.d_edge_rec;
    g.d_vn_pos = d.d_vn_pos;
    g.d_vn_hold = d.d_vn_hold;
  }
  const auto& sh = s->impl->host;
  g.per_frame = sh.per_frame;
  g.regroup = sh.regroup;
  g.balanced = sh.overlap == 0.0;
  g.nominal = sh.nominal;
  g.k_overlap = sh.k_overlap;
  g.list_slots = static_cast<int>(sh.grp_cns.size());
  g.schedule_seed = sh.seed;
  g.h_cn_off = t.cn_off.data();
  g.h_fix_off = t.fix_off.data();
  return g;
}

ldpcb::Rows rows_from_csr(int m, const int32_t* off, const int32_t* cols) {
  need(off != nullptr && cols != nullptr, "null CSR arrays");
  need(off[0] == 0, "row offsets must start at 0");
  ldpcb::Rows rows(m);
  for (int r = 0; r < m; ++r) {
    need(off[r + 1] >= off[r], "row offsets must be non-decreasing");
    rows[r].assign(cols + off[r], cols + off[r + 1]);
  }
  return rows;
}

void launch(int err, const char* what) { cuda_check(err, what); }



}  // namespace

extern "C" {

const char* ldpcb_last_error(void) { return g_last_error.c_str(); }
int ldpcb_abi_version(void) { return 1; }

int ldpcb_code_from_check_lists(int n_vars, int n_checks, const int32_t* row_off, const int32_t* cols,
                                ldpcb_code* out) {
  return guard([&] {
    need(n_checks >= 1 && n_vars >= 1, "graph must have at least one VN and one CN");
    return make_code(ldpcb::build_code(n_vars, rows_from_csr(n_checks, row_off, cols)), out);
  });
}

int ldpcb_code_random_regular(int n_vars, int dv, int dc, uint64_t seed, ldpcb_code* out) {
  return guard([&] { return make_code(ldpcb::build_code(n_vars, ldpcb::regular_rows(n_vars, dv, dc, seed)), out); });
}

int ldpcb_code_random_regular_girth6(int n_vars, int dv, int dc, uint64_t seed, ldpcb_code* out) {
  return guard([&] {
    auto rows = ldpcb::regular_rows(n_vars, dv, dc, seed);
    ldpcb::break_4cycles(n_vars, rows, seed);
    return make_code(ldpcb::build_code(n_vars, rows), out);
  });
}

int ldpcb_code_qc(int base_rows, int base_cols, int z, double p_empty, int min_col_degree, uint64_t seed,
                  ldpcb_code* out) {
  return guard([&] {
    auto rows = ldpcb::qc_rows(base_rows, base_cols, z, p_empty, min_col_degree, seed);
    return make_code(ldpcb::build_code(base_cols * z, rows), out);
  });
}

int ldpcb_code_irregular(int n_vars, int n_classes, const int32_t* vn_degrees, const int32_t* vn_counts, int dc,
                         uint64_t seed, ldpcb_code* out) {
  return guard([&] {
    need(n_classes >= 1 && vn_degrees && vn_counts, "need at least one degree class");
    std::vector<int> d(vn_degrees, vn_degrees + n_classes), c(vn_counts, vn_counts + n_classes);
    return make_code(ldpcb::build_code(n_vars, ldpcb::irregular_rows(n_vars, d, c, dc, seed)), out);
  });
}

int ldpcb_code_parse_alist(const char* text, ldpcb_code* out, int* err_kind, int* err_line) {
  return guard([&] {
    need(text != nullptr, "null text");
    try {
      return make_code(ldpcb::parse_alist(text), out);
    } catch (const ldpcb::AlistFailure& e) {
      if (err_kind) *err_kind = static_cast<int>(e.kind);
      if (err_line) *err_line = e.line;
      throw;
    }
  });
}

int ldpcb_code_serialize_alist(ldpcb_code code, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    need(code != nullptr, "null handle");
    const std::string s = ldpcb::serialize_alist(code->impl->host);
    if (len) *len = static_cast<int64_t>(s.size());
    if (buf && cap > static_cast<int64_t>(s.size())) std::memcpy(buf, s.c_str(), s.size() + 1);
    return LDPCB_OK;
  });
}

int ldpcb_code_dims(ldpcb_code code, int32_t* n_vars, int32_t* n_checks, int32_t* n_edges, int32_t* max_cdeg,
                    int32_t* max_vdeg) {
  return guard([&] {
    need(code != nullptr, "null handle");
    const auto& h = code->impl->host;
    if (n_vars) *n_vars = h.n;
    if (n_checks) *n_checks = h.m;
    if (n_edges) *n_edges = h.E;
    if (max_cdeg) *max_cdeg = h.max_cdeg;
    if (max_vdeg) *max_vdeg = h.max_vdeg;
    return LDPCB_OK;
  });
}

int ldpcb_code_export(ldpcb_code code, int32_t* row_off, int32_t* cols, int32_t* var_off, int32_t* var_cns,
                      int32_t* var_edges) {
  return guard([&] {
    need(code != nullptr, "null handle");
    const auto& h = code->impl->host;
    auto put = [](int32_t* dst, const std::vector<int32_t>& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(int32_t));
    };
    put(row_off, h.row_off);
    put(cols, h.cols);
    put(var_off, h.var_off);
    put(var_cns, h.var_cns);
    put(var_edges, h.var_edges);
    return LDPCB_OK;
  });
}

int ldpcb_code_count_4cycles(ldpcb_code code, int64_t* count) {
  return guard([&] {
    need(code != nullptr && count != nullptr, "null argument");
    *count = ldpcb::count_4cycles(code->impl->host);
    return LDPCB_OK;
  });
}

void ldpcb_code_destroy(ldpcb_code code) { delete code; }

int ldpcb_schedule_from_groups(ldpcb_code code, int kind, int n_groups, const int32_t* grp_off,
                               const int32_t* grp_cns, ldpcb_schedule* out) {
  return guard([&] {
    need(code != nullptr, "null handle");
    need(kind >= 0 && kind <= 2, "unknown schedule kind");
    need(n_groups >= 1, "schedule needs at least one group");
    auto groups = rows_from_csr(n_groups, grp_off, grp_cns);
    return make_sched(code->impl,
                      ldpcb::schedule_from_groups(code->impl->host, static_cast<ldpcb::Kind>(kind), groups), out);
  });
}

int ldpcb_schedule_flooding(ldpcb_code code, ldpcb_schedule* out) {
  return guard([&] {
    need(code != nullptr, "null handle");
    return make_sched(code->impl, ldpcb::flooding_schedule(code->impl->host), out);
  });
}

int ldpcb_schedule_disjoint(ldpcb_code code, int n_groups, uint64_t seed, ldpcb_schedule* out) {
  return guard([&] {
    need(code != nullptr, "null handle");
    return make_sched(code->impl,
                      ldpcb::reference_random_schedule(code->impl->host, ldpcb::Kind::disjoint, n_groups, 0.0, seed),
                      out);
  });
}

int ldpcb_schedule_nondisjoint(ldpcb_code code, int n_groups, double overlap, uint64_t seed, ldpcb_schedule* out) {
  return guard([&] {
    need(code != nullptr, "null handle");
    return make_sched(
        code->impl,
        ldpcb::reference_random_schedule(code->impl->host, ldpcb::Kind::nondisjoint, n_groups, overlap, seed), out);
  });
}

int ldpcb_schedule_per_frame(ldpcb_code code, int kind, int n_groups, double overlap, uint64_t schedule_seed,
                             int regroup_each_iteration, ldpcb_schedule* out) {
  return guard([&] {
    need(code != nullptr, "null handle");
    need(kind >= 0 && kind <= 2, "unknown schedule kind");
    need(code->impl->host.m < 65536, "per-frame groupings support up to 65535 checks");
    return make_sched(code->impl,
                      ldpcb::per_frame_schedule(code->impl->host, static_cast<ldpcb::Kind>(kind), n_groups, overlap,
                                                schedule_seed, regroup_each_iteration != 0),
                      out);
  });
}

int ldpcb_schedule_windows(ldpcb_code code, int kind, int n_groups, int window, int stride, ldpcb_schedule* out) {
  return guard([&] {
    need(code != nullptr, "null handle");
    need(kind >= 0 && kind <= 2, "unknown schedule kind");
    return make_sched(code->impl,
                      ldpcb::window_schedule(code->impl->host, static_cast<ldpcb::Kind>(kind), n_groups, window,
                                             stride),
                      out);
  });
}

int ldpcb_schedule_dims(ldpcb_schedule s, int32_t* kind, int32_t* n_groups, int32_t* n_slots, int32_t* group_size,
                        double* overlap, int64_t* edge_updates_per_iter, int64_t* touched_per_iter) {
  return guard([&] {
    need(s != nullptr, "null handle");
    const auto& h = s->impl->host;
    if (kind) *kind = static_cast<int32_t>(h.kind);
    if (n_groups) *n_groups = h.G;
    if (n_slots) *n_slots = static_cast<int32_t>(h.grp_cns.size());
    if (group_size) *group_size = h.group_size;
    if (overlap) *overlap = h.overlap;
    if (edge_updates_per_iter) *edge_updates_per_iter = h.edge_updates_per_iter;
    if (touched_per_iter) *touched_per_iter = h.touched_per_iter;
    return LDPCB_OK;
  });
}

int ldpcb_schedule_export(ldpcb_schedule s, int32_t* grp_off, int32_t* grp_cns) {
  return guard([&] {
    need(s != nullptr, "null handle");
    const auto& h = s->impl->host;
    if (grp_off) std::memcpy(grp_off, h.grp_off.data(), h.grp_off.size() * sizeof(int32_t));
    if (grp_cns) std::memcpy(grp_cns, h.grp_cns.data(), h.grp_cns.size() * sizeof(int32_t));
    return LDPCB_OK;
  });
}

int ldpcb_schedule_iteration_budget(ldpcb_schedule s, int i_max, int32_t* budget) {
  return guard([&] {
    need(s != nullptr && budget != nullptr, "null argument");
    *budget = ldpcb::iteration_budget(s->impl->host, s->impl->code->host.m, i_max);
    return LDPCB_OK;
  });
}

int ldpcb_schedule_cocsg(ldpcb_schedule s, int32_t* counts) {
  return guard([&] {
    need(s != nullptr && counts != nullptr, "null argument");
    const auto v = ldpcb::measure_cocsg(s->impl->code->host, s->impl->host);
    std::copy(v.begin(), v.end(), counts);
    return LDPCB_OK;
  });
}

void ldpcb_schedule_destroy(ldpcb_schedule s) { delete s; }

int ldpcb_sigma2_from_ebn0(double ebn0_db, double rate, double* sigma2) {
  return guard([&] {
    need(rate > 0.0 && rate <= 1.0, "code rate must be in (0, 1]");
    need(sigma2 != nullptr, "null output");
    *sigma2 = ldpcb::awgn_sigma2(ebn0_db, rate);
    return LDPCB_OK;
  });
}

int ldpcb_channel_llr_device(int n, double sigma2, uint64_t seed, int64_t frame0, int64_t frames, float* d_llr,
                             void* stream) {
  return guard([&] {
    need(n >= 1, "frame length must be >= 1");
    need(frames >= 0 && (frames == 0 || d_llr != nullptr), "bad frame buffer");
    need(sigma2 > 0.0, "sigma2 must be positive");
    launch(ldpcb::launch_channel(n, sigma2, seed, frame0, frames, d_llr, stream), "channel kernel");
    return LDPCB_OK;
  });
}

int ldpcb_channel_stream_state(uint64_t seed, uint64_t frame, uint64_t draws, uint64_t* state) {
  return guard([&] {
    need(state != nullptr, "null state buffer");
    ldpcb::Stream st(ldpcb::stream_seed(seed, frame));
    ldpcb::stream_jump(st, ldpcb::stream_jump_poly(draws));
    state[0] = st.w0;
    state[1] = st.w1;
    state[2] = st.w2;
    state[3] = st.w3;
    return LDPCB_OK;
  });
}

int ldpcb_decode_device(ldpcb_code code, ldpcb_schedule s, int64_t frames, const float* d_llr, int max_iters,
                        int early_stop, uint8_t* d_bits, int bits_packed, int32_t* d_iterations, uint8_t* d_converged,
                        float* d_posterior, int32_t* d_trace, int64_t* d_counters, void* stream) {
  return guard([&] {
    check_pair(code, s);
    need(max_iters >= 1, "max_iters must be >= 1");
    need(frames >= 0, "frames must be >= 0");
    need(frames == 0 || d_llr != nullptr, "null LLR buffer");
    const auto g = dev_graph(code, s);
    ldpcb::DecodeArgs a;
    a.frames = frames;
    a.llr = d_llr;
    a.max_iters = max_iters;
    a.early_stop = early_stop != 0;
    a.bits = d_bits;
    a.bits_packed = bits_packed != 0;
    a.iterations = d_iterations;
    a.converged = d_converged;
    a.posterior = d_posterior;
    a.trace = d_trace;
    a.counters = reinterpret_cast<unsigned long long*>(d_counters);
    ldpcb::Plan p;
    const int err = ldpcb::launch_decode(g, a, stream, &p);
    if (p.kernel == 0) throw std::runtime_error("no decoder plan for this code (check degree or memory)");
    launch(err, "decode kernel");
    return LDPCB_OK;
  });
}

int ldpcb_decode_host(ldpcb_code code, ldpcb_schedule s, int64_t frames, const float* llr, int max_iters,
                      int early_stop, uint8_t* bits, int bits_packed, int32_t* iterations, uint8_t* converged,
                      float* posterior, int32_t* trace, int64_t* counters) {
  return guard([&] {
    check_pair(code, s);
    need(max_iters >= 1, "max_iters must be >= 1");
    need(frames >= 0, "frames must be >= 0");
    need(frames == 0 || llr != nullptr, "null LLR buffer");
    if (frames == 0) return LDPCB_OK;
    const auto g = dev_graph(code, s);
    const int n = g.n;
    const int64_t nb = bits_packed ? (n + 7) / 8 : n;
    const ldpcb::Plan p0 = ldpcb::plan_decode(g, frames, early_stop != 0);
    if (p0.kernel == 0) throw std::runtime_error("no decoder plan for this code (check degree or memory)");
    // chunks of ~32 MB of LLRs, a multiple of the frames per CTA; for the
    // streamed kernel two half-size decode chunks so copies overlap decoding
    int64_t chunk = p0.kernel == 2 ? std::max<int64_t>(4, (p0.fpc / 2 + 3) / 4 * 4)
                                   : std::max<int64_t>(p0.fpc, (int64_t{32} << 20) / (4 * n));
    chunk = std::min<int64_t>(chunk, frames);
    if (p0.kernel != 2) chunk = (chunk + p0.fpc - 1) / p0.fpc * p0.fpc;  // whole CTAs (streamed: fpc = chunk)
    constexpr int kSlots = 2;
    struct Buf {
      float* llr = nullptr;
      uint8_t* bits = nullptr;
      int32_t* it = nullptr;
      uint8_t* cv = nullptr;
      float* post = nullptr;
      int32_t* trace = nullptr;
      int64_t* cnt = nullptr;
    };
    // Owns the per-slot device buffers: on every exit (an error thrown by a
    // copy or a launch included) the buffers are released on their streams
    // and both streams drained, so nothing stays queued against host memory
    // the caller may free once this call returns.
    struct Slots {
      cudaStream_t st[kSlots] = {};
      Buf buf[kSlots];
      ~Slots() {
        for (int k = 0; k < kSlots; ++k) {
          if (!st[k]) continue;
          void* ptrs[] = {buf[k].llr, buf[k].bits, buf[k].it, buf[k].cv, buf[k].post, buf[k].trace, buf[k].cnt};
          for (void* q : ptrs)
            if (q) cudaFreeAsync(q, st[k]);  // errors ignored: best effort on the unwind path
          cudaStreamSynchronize(st[k]);
        }
      }
    } slots;
    cudaStream_t* st = slots.st;
    Buf* buf = slots.buf;
    for (int k = 0; k < kSlots; ++k) {
      st[k] = host_stream(k);
      cuda_check(cudaMallocAsync(&buf[k].llr, chunk * n * sizeof(float), st[k]), "cudaMallocAsync");
      if (bits) cuda_check(cudaMallocAsync(&buf[k].bits, chunk * nb, st[k]), "cudaMallocAsync");
      if (iterations) cuda_check(cudaMallocAsync(&buf[k].it, chunk * sizeof(int32_t), st[k]), "cudaMallocAsync");
      if (converged) cuda_check(cudaMallocAsync(&buf[k].cv, chunk, st[k]), "cudaMallocAsync");
      if (posterior) cuda_check(cudaMallocAsync(&buf[k].post, chunk * n * sizeof(float), st[k]), "cudaMallocAsync");
      if (trace)
        cuda_check(cudaMallocAsync(&buf[k].trace, chunk * max_iters * sizeof(int32_t), st[k]), "cudaMallocAsync");
      if (counters) {
        cuda_check(cudaMallocAsync(&buf[k].cnt, 6 * sizeof(int64_t), st[k]), "cudaMallocAsync");
        cuda_check(cudaMemsetAsync(buf[k].cnt, 0, 6 * sizeof(int64_t), st[k]), "cudaMemsetAsync");
      }
    }
    // Streamed decodes: a call takes (first chunk's copy) + (all decodes), the later copies
    // hide behind decodes. A quarter-size first chunk starts the device four times sooner
    // (C5 n = 64800, 32768 frames: 38 ms of exposed copy become 10).
    const int64_t first = (p0.kernel == 2 && frames > chunk) ? std::max<int64_t>(1024, chunk / 4 / 4 * 4) : chunk;
    int64_t slot = 0;
    for (int64_t c0 = 0, cnt = 0; c0 < frames; c0 += cnt, ++slot) {
      const int k = static_cast<int>(slot % kSlots);
      cnt = std::min(slot == 0 ? std::min(first, chunk) : chunk, frames - c0);
      cuda_check(cudaMemcpyAsync(buf[k].llr, llr + c0 * n, cnt * n * sizeof(float), cudaMemcpyHostToDevice, st[k]),
                 "H2D");
      ldpcb::DecodeArgs a;
      a.frame0 = c0;
      a.frames = cnt;
      a.llr = buf[k].llr;
      a.max_iters = max_iters;
      a.early_stop = early_stop != 0;
      a.bits = buf[k].bits;
      a.bits_packed = bits_packed != 0;
      a.iterations = buf[k].it;
      a.converged = buf[k].cv;
      a.posterior = buf[k].post;
      a.trace = buf[k].trace;
      a.counters = reinterpret_cast<unsigned long long*>(buf[k].cnt);
      launch(ldpcb::launch_decode(g, a, st[k], nullptr), "decode kernel");
      if (trace)
        cuda_check(cudaMemcpyAsync(trace + c0 * max_iters, buf[k].trace, cnt * max_iters * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost, st[k]),
                   "D2H");
      if (bits) cuda_check(cudaMemcpyAsync(bits + c0 * nb, buf[k].bits, cnt * nb, cudaMemcpyDeviceToHost, st[k]), "D2H");
      if (iterations)
        cuda_check(cudaMemcpyAsync(iterations + c0, buf[k].it, cnt * sizeof(int32_t), cudaMemcpyDeviceToHost, st[k]),
                   "D2H");
      if (converged) cuda_check(cudaMemcpyAsync(converged + c0, buf[k].cv, cnt, cudaMemcpyDeviceToHost, st[k]), "D2H");
      if (posterior)
        cuda_check(cudaMemcpyAsync(posterior + c0 * n, buf[k].post, cnt * n * sizeof(float), cudaMemcpyDeviceToHost,
                                   st[k]),
                   "D2H");
    }
    int64_t total[6] = {0, 0, 0, 0, 0, 0};
    for (int k = 0; k < kSlots; ++k) {
      if (counters) {
        int64_t h[6];
        cuda_check(cudaMemcpyAsync(h, buf[k].cnt, sizeof h, cudaMemcpyDeviceToHost, st[k]), "D2H");
        cuda_check(cudaStreamSynchronize(st[k]), "sync");
        for (int i = 0; i < 6; ++i) total[i] += h[i];
      }
      cuda_check(cudaStreamSynchronize(st[k]), "sync");
    }
    if (counters)
      for (int i = 0; i < 6; ++i) counters[i] += total[i];
    return LDPCB_OK;
  });
}

namespace {
// Channel + decode of frames [frame_begin, frame_begin+frames) in chunks
// (sim.hpp:111-124); optional per-frame outcomes and accumulated counters.
void simulate_frames(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed, int64_t frame_begin,
                     int64_t frames, int max_iters, int early_stop, int32_t* d_bit_errors, int32_t* d_iterations,
                     uint8_t* d_converged, int64_t* d_counters, void* stream) {
  check_pair(code, s);
  need(max_iters >= 1, "max_iters must be >= 1");
  need(frames >= 0 && frame_begin >= 0, "bad frame range");
  need(sigma2 > 0.0, "sigma2 must be positive");
  if (frames == 0) return;
  const auto g = dev_graph(code, s);
  const ldpcb::Plan p0 = ldpcb::plan_decode(g, frames, early_stop != 0);
  if (p0.kernel == 0) throw std::runtime_error("no decoder plan for this code (check degree or memory)");
  auto st = static_cast<cudaStream_t>(stream);
  int64_t chunk = std::max<int64_t>(p0.fpc, (int64_t{256} << 20) / (4 * g.n));
  if (p0.kernel == 2 && early_stop) {
    // streamed early stop: frames flow through the frame queue's lanes inside one decode
    // call, so a chunk holds many lane refills (65536 frames where a sixth of the free
    // memory holds their LLRs; the lanes' state takes as much again)
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
    const int64_t fit = static_cast<int64_t>(free_b / 6 / (4ull * g.n));
    chunk = std::max(chunk, std::min<int64_t>(65536, fit));
  }
  chunk = std::min<int64_t>(chunk, frames);
  float* scratch = nullptr;
  cuda_check(cudaMallocAsync(&scratch, chunk * g.n * sizeof(float), st), "cudaMallocAsync");
  for (int64_t c0 = 0; c0 < frames; c0 += chunk) {
    const int64_t cnt = std::min(chunk, frames - c0);
    launch(ldpcb::launch_channel(g.n, sigma2, channel_seed, frame_begin + c0, cnt, scratch, stream), "channel");
    ldpcb::DecodeArgs a;
    a.frame0 = frame_begin + c0;
    a.frames = cnt;
    a.llr = scratch;
    a.max_iters = max_iters;
    a.early_stop = early_stop != 0;
    a.counters = reinterpret_cast<unsigned long long*>(d_counters);
    if (d_bit_errors) a.bit_errors = d_bit_errors + c0;
    if (d_iterations) a.iterations = d_iterations + c0;
    if (d_converged) a.converged = d_converged + c0;
    launch(ldpcb::launch_decode(g, a, stream, nullptr), "decode kernel");
  }
  cuda_check(cudaFreeAsync(scratch, st), "cudaFreeAsync");
}
}  // namespace

int ldpcb_simulate_device(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed, int64_t frame_begin,
                          int64_t frames, int max_iters, int early_stop, int64_t* d_counters, void* stream) {
  return guard([&] {
    need(d_counters != nullptr, "null counters");
    simulate_frames(code, s, sigma2, channel_seed, frame_begin, frames, max_iters, early_stop, nullptr, nullptr,
                    nullptr, d_counters, stream);
    return LDPCB_OK;
  });
}

int ldpcb_simulate_frames_device(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed,
                                 int64_t frame_begin, int64_t frames, int max_iters, int early_stop,
                                 int32_t* d_bit_errors, int32_t* d_iterations, uint8_t* d_converged,
                                 int64_t* d_counters, void* stream) {
  return guard([&] {
    need(d_bit_errors || d_iterations || d_converged || d_counters, "no outputs");
    simulate_frames(code, s, sigma2, channel_seed, frame_begin, frames, max_iters, early_stop, d_bit_errors,
                    d_iterations, d_converged, d_counters, stream);
    return LDPCB_OK;
  });
}

}  // extern "C"

namespace {

// Runs fn(i) for i < n_devices, one host thread per entry of `devices`, each
// bound to its device (the reference's worker pool, sim.hpp:136-150, with a
// GPU per worker). The first failure is rethrown on the calling thread with
// its own exception type, after every worker has finished.
template <class F>
void on_devices(const int* devices, int n_devices, F&& fn) {
  need(devices != nullptr && n_devices >= 1, "need at least one device");
  int count = 0;
  cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  for (int i = 0; i < n_devices; ++i) need(devices[i] >= 0 && devices[i] < count, "device index out of range");
  std::vector<std::exception_ptr> errs(n_devices);
  std::vector<std::thread> pool;
  pool.reserve(n_devices);
  for (int i = 0; i < n_devices; ++i)
    pool.emplace_back([&, i] {
      try {
        cuda_check(cudaSetDevice(devices[i]), "cudaSetDevice");
        fn(i);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// run_sweep (sim.hpp:96-186) on one or more GPUs: waves of frames, each wave
// split into contiguous frame-id ranges over the devices (sim.py shard), the
// per-frame outcomes copied back in frame order, and the point stops at the
// smallest frame index whose prefix holds min_frame_errors frame errors (or
// at max_frames). Frames are keyed by id, so the result depends neither on
// the wave size nor on the number of devices, as in the reference.
void run_sweep_impl(ldpcb_code code, ldpcb_schedule s, const int* devices, int n_devices, const double* ebn0_db,
                    int n_points, int iter_limit, int64_t max_frames, int min_frame_errors, uint64_t channel_seed,
                    int64_t wave_frames, double* out) {
  check_pair(code, s);
  need(ebn0_db != nullptr && n_points >= 1, "need at least one Eb/N0 point");
  need(min_frame_errors >= 1, "min_frame_errors must be >= 1");
  need(max_frames >= 1, "max_frames must be >= 1");
  need(iter_limit >= 1, "max_iters must be >= 1");
  need(out != nullptr, "null output");
  const auto& h = code->impl->host;
  const double rate = static_cast<double>(h.n - h.m) / h.n;
  int64_t cap = wave_frames > 0 ? wave_frames : (int64_t{1} << 20) * n_devices;
  cap = std::min(cap, max_frames);
  std::vector<int32_t> be(cap), it(cap);
  std::vector<uint8_t> cv(cap);
  // one wave on every device: worker i decodes [begin + cnt*i/D, begin + cnt*(i+1)/D)
  auto wave_on_devices = [&](double sigma2, int64_t begin, int64_t cnt) {
    on_devices(devices, n_devices, [&](int i) {
      const int64_t lo = cnt * i / n_devices, len = cnt * (i + 1) / n_devices - lo;
      if (len == 0) return;
      cudaStream_t st = host_stream(0);
      int32_t *d_be = nullptr, *d_it = nullptr;
      uint8_t* d_cv = nullptr;
      auto cleanup = [&] {
        if (d_be) cudaFreeAsync(d_be, st);
        if (d_it) cudaFreeAsync(d_it, st);
        if (d_cv) cudaFreeAsync(d_cv, st);
        cudaStreamSynchronize(st);
      };
      try {
        cuda_check(cudaMallocAsync(&d_be, len * 4, st), "cudaMallocAsync");
        cuda_check(cudaMallocAsync(&d_it, len * 4, st), "cudaMallocAsync");
        cuda_check(cudaMallocAsync(&d_cv, len, st), "cudaMallocAsync");
        simulate_frames(code, s, sigma2, channel_seed, begin + lo, len, iter_limit, 1, d_be, d_it, d_cv, nullptr, st);
        cuda_check(cudaMemcpyAsync(be.data() + lo, d_be, len * 4, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(it.data() + lo, d_it, len * 4, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(cv.data() + lo, d_cv, len, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
      } catch (...) {
        cleanup();
        throw;
      }
      cleanup();
    });
  };
  for (int pt = 0; pt < n_points; ++pt) {
    const auto t0 = std::chrono::steady_clock::now();
    const double sigma2 = ldpcb::awgn_sigma2(ebn0_db[pt], rate);
    int64_t produced = 0, stop = -1, fe_total = 0, conv = 0;
    long long bit_errors = 0, iter_sum = 0, iter_conv = 0;
    // the first wave is small so that high-FER points stop early
    int64_t wave = std::min<int64_t>(cap, 4096);
    while (stop < 0) {
      const int64_t cnt = std::min(wave, max_frames - produced);
      wave_on_devices(sigma2, produced, cnt);
      for (int64_t i = 0; i < cnt; ++i) {  // prefix scan (sim.hpp:150-158) + aggregation (:162-181)
        bit_errors += be[i];
        fe_total += be[i] > 0;
        conv += cv[i];
        iter_sum += it[i];
        iter_conv += cv[i] ? it[i] : 0;
        if (fe_total >= min_frame_errors) {
          stop = produced + i;
          break;
        }
      }
      produced += cnt;
      if (stop < 0 && produced >= max_frames) stop = max_frames - 1;
      wave = std::min(cap, 2 * wave);
    }
    const double frames = static_cast<double>(stop + 1);
    double* o = out + 11 * pt;
    o[0] = frames;
    o[1] = static_cast<double>(bit_errors);
    o[2] = static_cast<double>(fe_total);
    o[3] = static_cast<double>(conv);
    o[4] = static_cast<double>(bit_errors) / (frames * h.n);
    o[5] = static_cast<double>(fe_total) / frames;
    o[6] = conv > 0 ? static_cast<double>(iter_conv) / conv : 0.0;
    o[7] = static_cast<double>(iter_sum) / frames;
    o[8] = iter_limit;
    o[9] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    o[10] = ebn0_db[pt];
  }
}

}  // namespace

extern "C" {

int ldpcb_run_sweep_host(ldpcb_code code, ldpcb_schedule s, const double* ebn0_db, int n_points, int iter_limit,
                         int64_t max_frames, int min_frame_errors, uint64_t channel_seed, int64_t wave_frames,
                         double* out) {
  return guard([&] {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    run_sweep_impl(code, s, &dev, 1, ebn0_db, n_points, iter_limit, max_frames, min_frame_errors, channel_seed,
                   wave_frames, out);
    return LDPCB_OK;
  });
}

int ldpcb_run_sweep_multi(ldpcb_code code, ldpcb_schedule s, const int* devices, int n_devices,
                          const double* ebn0_db, int n_points, int iter_limit, int64_t max_frames,
                          int min_frame_errors, uint64_t channel_seed, int64_t wave_frames, double* out) {
  return guard([&] {
    run_sweep_impl(code, s, devices, n_devices, ebn0_db, n_points, iter_limit, max_frames, min_frame_errors,
                   channel_seed, wave_frames, out);
    return LDPCB_OK;
  });
}

int ldpcb_simulate_multi(ldpcb_code code, ldpcb_schedule s, const int* devices, int n_devices, double sigma2,
                         uint64_t channel_seed, int64_t frame_begin, int64_t frames, int max_iters, int early_stop,
                         int64_t* counters) {
  return guard([&] {
    check_pair(code, s);
    need(counters != nullptr, "null counters");
    need(frames >= 0 && frame_begin >= 0, "bad frame range");
    need(devices != nullptr && n_devices >= 1, "need at least one device");
    // per-worker counters, summed on the host once every worker is done (the
    // in-process counterpart of the NCCL allreduce of sim.py / bench.py)
    std::vector<std::array<int64_t, 6>> part(n_devices);
    on_devices(devices, n_devices, [&](int i) {
      part[i].fill(0);
      const int64_t lo = frames * i / n_devices, len = frames * (i + 1) / n_devices - lo;
      if (len == 0) return;
      if (ldpcb_simulate_host(code, s, sigma2, channel_seed, frame_begin + lo, len, max_iters, early_stop,
                              part[i].data()) != LDPCB_OK)
        throw std::runtime_error("device " + std::to_string(devices[i]) + ": " + g_last_error);
    });
    for (const auto& c : part)
      for (int k = 0; k < 6; ++k) counters[k] += c[k];
    return LDPCB_OK;
  });
}

int ldpcb_simulate_host(ldpcb_code code, ldpcb_schedule s, double sigma2, uint64_t channel_seed, int64_t frame_begin,
                        int64_t frames, int max_iters, int early_stop, int64_t* counters) {
  return guard([&] {
    check_pair(code, s);
    need(counters != nullptr, "null counters");
    cudaStream_t st = host_stream(0);
    int64_t* d = nullptr;
    int rc = LDPCB_OK;
    try {
      cuda_check(cudaMallocAsync(&d, 6 * sizeof(int64_t), st), "cudaMallocAsync");
      cuda_check(cudaMemsetAsync(d, 0, 6 * sizeof(int64_t), st), "cudaMemsetAsync");
      rc = ldpcb_simulate_device(code, s, sigma2, channel_seed, frame_begin, frames, max_iters, early_stop, d, st);
      if (rc == LDPCB_OK) {
        int64_t h[6];
        cuda_check(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
        for (int i = 0; i < 6; ++i) counters[i] += h[i];
      }
    } catch (...) {
      if (d) cudaFreeAsync(d, st);
      cudaStreamSynchronize(st);
      throw;
    }
    const std::string err = g_last_error;  // keep the inner message
    cudaFreeAsync(d, st);
    cudaStreamSynchronize(st);
    g_last_error = err;
    return rc;
  });
}

int ldpcb_check_update_device(int degree, int64_t rows, const float* d_v2c, float* d_c2v, void* stream) {
  return guard([&] {
    need(degree >= 2 && degree <= 32, "degree must be in [2, 32]");
    need(rows >= 0, "rows must be >= 0");
    launch(ldpcb::launch_check_update(degree, rows, d_v2c, d_c2v, stream), "check_update kernel");
    return LDPCB_OK;
  });
}

int ldpcb_schedule_per_frame_groups_device(ldpcb_code code, ldpcb_schedule s, int64_t frame0, int64_t frames,
                                           int iteration, uint16_t* d_cns, void* stream) {
  return guard([&] {
    check_pair(code, s);
    need(s->impl->host.per_frame, "not a per-frame schedule");
    need(iteration >= 1, "iteration must be >= 1");
    need(frames >= 0 && d_cns != nullptr, "bad output");
    const auto g = dev_graph(code, s);
    launch(ldpcb::launch_gen_groups(g, frame0, frames, iteration - 1, 1, d_cns, stream), "group generator");
    return LDPCB_OK;
  });
}

int ldpcb_run_subiterations_device(ldpcb_code code, ldpcb_schedule s, int64_t frames, const float* d_llr,
                                   int n_subiters, float* d_c2v, float* d_v2c, void* stream) {
  return guard([&] {
    check_pair(code, s);
    need(n_subiters >= 1, "n_subiters must be >= 1");
    const auto g = dev_graph(code, s);
    ldpcb::DecodeArgs a;
    a.frames = frames;
    a.llr = d_llr;
    a.max_iters = n_subiters / g.G + 1;
    a.early_stop = 0;
    a.max_subiters = n_subiters;
    a.c2v_out = d_c2v;
    a.v2c_out = d_v2c;
    ldpcb::Plan p;
    const int err = ldpcb::launch_decode(g, a, stream, &p);
    if (p.kernel == 0) throw std::runtime_error("no decoder plan for this code (check degree or memory)");
    launch(err, "decode kernel");
    return LDPCB_OK;
  });
}

int ldpcb_decode_plan(ldpcb_code code, ldpcb_schedule s, int64_t frames, int32_t* kernel, int32_t* fpc,
                      int32_t* threads, int32_t* smem_bytes, int32_t* degree_bucket) {
  return guard([&] {
    const auto g = dev_graph(code, s);
    const auto p = ldpcb::plan_decode(g, frames);
    if (kernel) *kernel = p.kernel == 1 ? 10 + p.fv : (p.kernel == 3 ? 20 + p.fv : p.kernel);
    if (fpc) *fpc = p.fpc;
    if (threads) *threads = p.threads;
    if (smem_bytes) *smem_bytes = p.smem;
    if (degree_bucket) *degree_bucket = p.degree_bucket;
    return LDPCB_OK;
  });
}

int ldpcb_schedule_direct_layout(ldpcb_schedule s, int32_t* frames_per_thread, int32_t* cells, int32_t* l_base,
                                 int32_t* buffer_cells, int32_t* n_items, double* wavefronts_per_access) {
  return guard([&] {
    need(s != nullptr, "null handle");
    const auto& t = s->impl->direct;
    if (frames_per_thread) *frames_per_thread = t.ok ? t.fv : 0;
    if (cells) *cells = t.ok ? t.cells : 0;
    if (l_base) *l_base = t.ok ? t.l_base : 0;
    if (buffer_cells) *buffer_cells = t.ok ? t.buf_cells : 0;
    if (n_items) *n_items = t.ok ? t.cn_off.back() : 0;
    if (wavefronts_per_access) *wavefronts_per_access = t.ok ? t.wavefronts : 0.0;
    return LDPCB_OK;
  });
}

int ldpcb_schedule_direct_export(ldpcb_schedule s, int32_t* cn_off, int32_t* cn_rec, int32_t* vn_rec,
                                 int32_t* vn_hold, int32_t* vn_pos, int32_t* edge_rec) {
  return guard([&] {
    need(s != nullptr, "null handle");
    const auto& t = s->impl->direct;
    need(t.ok, "the posterior-free kernel does not apply to this schedule");
    auto put = [](int32_t* out, const std::vector<int32_t>& v) {
      if (out) std::copy(v.begin(), v.end(), out);
    };
    put(cn_off, t.cn_off);
    put(cn_rec, t.cn_rec);
    put(vn_rec, t.vn_rec);
    put(vn_hold, t.vn_hold);
    put(vn_pos, t.vn_pos);
    put(edge_rec, t.edge_rec);
    return LDPCB_OK;
  });
}

int ldpcb_set_tuning(int frames_per_cta, int threads) {
  return guard([&] {
    need(frames_per_cta == 0 || frames_per_cta == 1 || frames_per_cta == 2 || frames_per_cta == 4 ||
             frames_per_cta == 8 || frames_per_cta == 16,
         "frames_per_cta must be 0 (auto) or a power of two <= 16");
    need(threads == 0 || (threads >= 32 && threads <= 512 && threads % 32 == 0),
         "threads must be 0 (auto) or a multiple of 32 in [32, 512]");
    ldpcb::set_tuning(frames_per_cta, threads);
    return LDPCB_OK;
  });
}

int64_t ldpcb_kernel_launches(void) { return ldpcb::kernel_launch_count(); }

int ldpcb_set_frames_per_thread(int fv) {
  return guard([&] {
    need(fv >= 0 && fv <= 2, "frames per thread must be 0 (auto), 1 or 2");
    ldpcb::set_frames_per_thread(fv);
    return LDPCB_OK;
  });
}

int ldpcb_set_kernel(int kernel) {
  return guard([&] {
    need(kernel >= 0 && kernel <= 3, "kernel must be 0 (auto), 1 (resident, posterior-based), 2 (streamed) or 3 (direct)");
    ldpcb::set_force_kernel(kernel);
    return LDPCB_OK;
  });
}

int ldpcb_set_lazy_totals(int on) {
  return guard([&] {
    ldpcb::set_lazy_totals(on != 0);
    return LDPCB_OK;
  });
}

}  // extern "C"
