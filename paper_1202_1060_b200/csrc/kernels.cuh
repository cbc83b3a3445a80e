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
  const int32_t* row_off = nullptr;
  const int32_t* cols = nullptr;
  const int32_t* var_off = nullptr;
  const int32_t* var_edges = nullptr;
  const int32_t* grp_off = nullptr;
  const int32_t* grp_cns = nullptr;
  const int32_t* touch_off = nullptr;
  const int32_t* touch_vns = nullptr;
};

// One decode launch (all pointers are device pointers; outputs nullable).
struct DecodeArgs {
  int64_t frames = 0;
  const float* llr = nullptr;  // [frames][n]
  int max_iters = 1;
  int early_stop = 1;
  int max_subiters = 0;  // >0: stop after this many sub-iterations and dump state
  uint8_t* bits = nullptr;
  int bits_packed = 0;
  int32_t* iterations = nullptr;
  uint8_t* converged = nullptr;
  float* posterior = nullptr;
  int32_t* trace = nullptr;  // [frames][max_iters]
  unsigned long long* counters = nullptr;  // 6 x int64, accumulated
  float* c2v_out = nullptr;  // [frames][E] (debug dump)
  float* v2c_out = nullptr;  // [frames][E]
};

struct Plan {
  int kernel = 0;  // 1 = SMEM-resident frame-interleaved
  int fpc = 0;     // frames per CTA
  int threads = 0;
  int smem = 0;    // dynamic shared memory bytes
  int degree_bucket = 0;
  int64_t ctas = 0;
};

Plan plan_decode(const DevGraph& g, int64_t frames);
// returns cudaError_t as int
int launch_decode(const DevGraph& g, const DecodeArgs& a, void* stream, Plan* used);
int launch_channel(int n, double sigma2, uint64_t seed, int64_t frame0, int64_t frames, float* llr, void* stream);
int launch_check_update(int degree, int64_t rows, const float* v2c, float* c2v, void* stream);

void set_tuning(int fpc, int threads);
int64_t kernel_launch_count();

}  // namespace ldpcb
