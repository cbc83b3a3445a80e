// kernels.cuh -- shared declarations between the C-ABI layer and the CUDA
// kernels of the B200 decoder.
#pragma once
#include <cstdint>

namespace ldpcb {

// Device-resident copy of a code + schedule (uploaded once per device).
struct DevGraph {
  int n = 0, m = 0, E = 0, G = 0;
  int max_cdeg = 0, max_vdeg = 0;
  bool cregular = false;  // every CN has degree max_cdeg
  bool vregular = false;  // every VN has degree max_vdeg
  int cs = 0;   // CN record stride (ints), multiple of 4
  int vs4 = 0;  // VN record stride (int4 units)
  int n_slots = 0;         // c2v slots per frame, incl. the zero slot
  bool recompute = false;  // exact-totals pass needed each iteration
  int max_cn_items = 0, max_fix_items = 0;
  const int32_t* cols = nullptr;        // CSR columns (state dumps)
  const int32_t* edge_slot = nullptr;   // edge id -> c2v slot (state dumps)
  const int32_t* vn_pos = nullptr;      // [n] VN id -> position in the per-VN state arrays
  const int32_t* cn_off = nullptr;      // [G+1] CN record offsets per group
  const int32_t* cn_rec = nullptr;      // see host.hpp KernelTables
  const int32_t* fix_off = nullptr;     // [G+1]
  const int32_t* fix_rec = nullptr;
  const int32_t* fix_rec16 = nullptr;   // 16-bit fix-up records (vs16 > 0), resident kernels
  const int32_t* tot_rec16 = nullptr;   // 16-bit totals records (vs16 > 0), resident kernels
  int vs16 = 0;
  const int32_t* all_vn_rec = nullptr;  // [n] VN records, indexed by VN
  const int32_t* tot_vn_rec = nullptr;  // [n] VN records in bank-coloured order
  const int32_t* all_rec = nullptr;     // [m] CN records, syndrome
  // fresh-frame bits of the streamed frame queue (host.hpp KernelTables)
  const uint32_t* cn_fresh = nullptr;   // per cn_rec record
  const uint32_t* fix_fresh = nullptr;  // per fix_rec record
  bool covers = false;
  // direct (posterior-free) kernel tables (host.hpp DirectTables); d_fv = 0: none
  int d_fv = 0, d_cells = 0, d_l_base = 0, d_max_items = 0, d_buf_cells = 0;
  // first CN record of every group, a kernel parameter (constant bank): group
  // ranges then cost a uniform constant load, no vector register
  static constexpr int kDirectMaxGroups = 96;
  uint16_t d_goff[kDirectMaxGroups + 1] = {};
  const int32_t* d_cn_rec = nullptr;
  const int32_t* d_vn_rec = nullptr;
  const int32_t* d_all_cn = nullptr;
  const int32_t* d_edge_rec = nullptr;
  const int32_t* d_vn_pos = nullptr;
  const int32_t* d_vn_hold = nullptr;
  // per-frame random grouping (host.hpp ScheduleData::per_frame)
  bool per_frame = false, regroup = false, balanced = false;
  int nominal = 0, k_overlap = 0, list_slots = 0;
  uint64_t schedule_seed = 0;
  // host copies of the per-group offsets (owned by the schedule handle)
  const int32_t* h_cn_off = nullptr;
  const int32_t* h_fix_off = nullptr;
};

// One decode launch (all pointers are device pointers; outputs nullable).
struct DecodeArgs {
  int64_t frames = 0;
  const float* llr = nullptr;  // [frames][n]
  int max_iters = 1;
  int early_stop = 1;
  int max_subiters = 0;  // >0: stop after this many sub-iterations and dump state
  int lazy_totals = 0;   // 1: exact totals only in iterations that test the syndrome
  int64_t frame0 = 0;    // frame id of frame 0 (per-frame schedule streams)
  const uint16_t* lists = nullptr;  // per-frame group lists [frames][n_lists][list_slots]
  int n_lists = 0, list_slots = 0;
  uint8_t* bits = nullptr;
  int bits_packed = 0;
  int32_t* iterations = nullptr;
  uint8_t* converged = nullptr;
  int32_t* bit_errors = nullptr;  // per-frame hard-decision weight (all-zero codeword errors)
  float* posterior = nullptr;
  int32_t* trace = nullptr;  // [frames][max_iters]
  unsigned long long* counters = nullptr;  // 6 x int64, accumulated
  float* c2v_out = nullptr;  // [frames][E] (debug dump)
  float* v2c_out = nullptr;  // [frames][E]
};

// Degree bucket of the CN kernel instantiation (exact for regular rows).
inline int cn_bucket(int max_cdeg, bool cregular) {
  if (cregular && (max_cdeg == 3 || max_cdeg == 6)) return max_cdeg;
  if (max_cdeg <= 8) return 8;
  if (max_cdeg <= 16) return 16;
  if (max_cdeg <= 32) return 32;
  return 0;
}
inline int cn_record_stride(int bucket) { return (2 + bucket + 3) / 4 * 4; }

struct Plan {
  int kernel = 0;  // 1 = SMEM-resident frame-interleaved, 2 = HBM-streamed, 3 = SMEM-resident direct (direct.cu)
  int fpc = 0;     // frames per CTA
  int fv = 1;      // frames per thread (resident kernel)
  int threads = 0;
  int smem = 0;    // dynamic shared memory bytes
  int degree_bucket = 0;
  int64_t ctas = 0;
};

// early_stop: the decode stops frames at a zero syndrome (changes the
// preferred frames per CTA); plan queries without a decode use false
Plan plan_decode(const DevGraph& g, int64_t frames, bool early_stop = false);
// returns cudaError_t as int
// per-frame group lists (gen_groups_kernel): out[(f * n_lists + l) * list_slots + j]
// = slot j of the ordered groups of frame frame0+f at iteration list0+l+1
int launch_gen_groups(const DevGraph& g, int64_t frame0, int64_t frames, int list0, int n_lists, uint16_t* out,
                      void* stream);
int launch_decode(const DevGraph& g, const DecodeArgs& a, void* stream, Plan* used);
int launch_channel(int n, double sigma2, uint64_t seed, int64_t frame0, int64_t frames, float* llr, void* stream);
int launch_check_update(int degree, int64_t rows, const float* v2c, float* c2v, void* stream);

void set_tuning(int fpc, int threads);
void set_frames_per_thread(int fv);
void set_force_kernel(int kernel);  // 0 auto, 1 resident (posterior-based), 2 streamed, 3 direct
// posterior-free resident kernel (direct.cu): (3,6)-type codes, groups of at most one CN item per thread
Plan plan_direct(const DevGraph& g, int64_t frames);
int launch_direct(const DevGraph& g, const DecodeArgs& a, void* stream, Plan* used);
bool direct_enabled();
void note_launches(int n);
// HBM-streamed decoder (stream.cu): frames whose state does not fit one SM
int launch_stream(const DevGraph& g, const DecodeArgs& a, void* stream, Plan* used);
Plan plan_stream(const DevGraph& g, int64_t frames);
void set_lazy_totals(int on);
int lazy_totals();
int64_t kernel_launch_count();

}  // namespace ldpcb
