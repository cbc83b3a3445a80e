// decoder.cu -- B200 (sm_100a) batched group-shuffled sum-product decoder.
//
// Kernel "resident": a CTA decodes FPC frames whose whole state lives in
// shared memory, laid out frame-interleaved (index * FPC + frame) so that the
// FPC lanes working on one CN / VN read the same graph entries (L1
// broadcast) and consecutive shared-memory banks.
//
// Per sub-iteration (decoder.hpp:112-127):
//   CN phase  every (CN of the group, frame): v2c = clamp(P_n - c2v_e)
//             (the posterior form of var_update, decoder.hpp:91-105), the
//             boxplus exclusion outputs, clamp, write c2v        (decoder.hpp:59-87)
//   barrier   (Jacobi inside a group: all CNs read pre-group state)
//   VN phase  every (touched VN, frame): P_n = L_n + sum c2v over the VN's
//             edges in ascending-CN order (= total_llr, decoder.hpp:162-165)
//   barrier
// Per iteration: hard decision (P < 0), syndrome weight, early stop
// (decoder.hpp:166-177). Epilogue: bits, iterations, converged flag,
// posteriors, Monte-Carlo counters (sim.hpp:119-123, 162-181).
//
// Boxplus arithmetic. A message of magnitude x maps to z = exp(-x) in (0,1]
// (z = tanh(phi(x)/2)); boxplus of two messages is z1 (+) z2 =
// (z1 + z2)/(1 + z1 z2), kept projective as (N, D) so no division and no
// subtraction ever happens:  (N1,D1) (+) (N2,D2) = (N1 D2 + N2 D1, D1 D2 + N1 N2).
// Exclusion outputs come from prefix/suffix products, and the output
// magnitude is ln(D/N) = ln2 * (lg2 D - lg2 N). Cost: 1 ex2 + 2 lg2 (MUFU)
// per edge and ~5 FMA. Exactly-zero inputs follow decoder.hpp:77-83: every
// other output of that CN is exactly 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>

#include "kernels.cuh"
#include "rng.cuh"

namespace ldpcb {
namespace {

constexpr float kClamp = 30.0f;  // decoder.hpp:18
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;

std::atomic<int64_t> g_launches{0};
std::atomic<int> g_tune_fpc{0}, g_tune_threads{0};

__device__ __forceinline__ float mufu_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float clamp_llr(float x) { return fminf(fmaxf(x, -kClamp), kClamp); }

// Exclusion boxplus over one CN. x[k] are the clamped incoming v2c for
// k < deg (EXACT: deg == D); store(k, c2v_k) receives every output.
template <int D, bool EXACT, class Store>
__device__ __forceinline__ void boxplus_row(const float (&x)[D], int deg, Store&& store) {
  float z[D];
  unsigned sg = 0, zr = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (EXACT || k < deg) {
      sg |= static_cast<unsigned>(x[k] < 0.f) << k;
      zr |= static_cast<unsigned>(x[k] == 0.f) << k;
      z[k] = mufu_ex2(fabsf(x[k]) * -kLog2e);
    } else {
      z[k] = 0.f;  // boxplus identity (N, D) = (0, 1)
    }
  }
  const unsigned par = __popc(sg) & 1u;
  auto emit = [&](int k, float num, float den) {
    if (EXACT || k < deg) {
      float mag = fminf((mufu_lg2(den) - mufu_lg2(num)) * kLn2, kClamp);
      if (zr & ~(1u << k)) mag = 0.f;
      const unsigned s = par ^ ((sg >> k) & 1u);
      store(k, s ? -mag : mag);
    }
  };
  // prefix products p[k] = z0 (+) ... (+) zk, k <= D-2
  float pn[D > 1 ? D - 1 : 1], pd[D > 1 ? D - 1 : 1];
  pn[0] = z[0];
  pd[0] = 1.f;
#pragma unroll
  for (int k = 1; k < D - 1; ++k) {
    pn[k] = fmaf(z[k], pd[k - 1], pn[k - 1]);
    pd[k] = fmaf(z[k], pn[k - 1], pd[k - 1]);
  }
  emit(D - 1, pn[D - 2], pd[D - 2]);
  float sn = z[D - 1], sd = 1.f;  // suffix s[k+1]
#pragma unroll
  for (int k = D - 2; k >= 1; --k) {
    emit(k, fmaf(pn[k - 1], sd, sn * pd[k - 1]), fmaf(pd[k - 1], sd, pn[k - 1] * sn));
    const float tn = fmaf(z[k], sd, sn);
    const float td = fmaf(z[k], sn, sd);
    sn = tn;
    sd = td;
  }
  emit(0, sn, sd);
}

struct Shared {
  float* c2v;  // [(E+1)][FPC]; slot E stays zero (pads short VN records)
  float* P;    // [n][FPC] posterior (channel + all c2v), unclamped
  float* L;    // [n][FPC] clamped channel LLR
  int* done;   // [FPC]
  int* weight;
  int* iters;
  int* conv;
  int* berr;
};

// One CN record (host.hpp KernelTables) -> the clamped incoming messages
// v2c = clamp(P_v - c2v_e) (posterior form of var_update, decoder.hpp:91-105).
template <int D, bool EXACT>
struct CnRecord {
  static constexpr int kInts = (2 + D + 3) / 4 * 4;
  int r[kInts];
  __device__ __forceinline__ explicit CnRecord(const int32_t* __restrict__ p) {
    const int4* q = reinterpret_cast<const int4*>(p);
#pragma unroll
    for (int i = 0; i < kInts / 4; ++i) {
      const int4 t = __ldg(q + i);
      r[4 * i] = t.x;
      r[4 * i + 1] = t.y;
      r[4 * i + 2] = t.z;
      r[4 * i + 3] = t.w;
    }
  }
  __device__ __forceinline__ int off() const { return r[0]; }
  __device__ __forceinline__ int deg() const { return EXACT ? D : r[1]; }
  __device__ __forceinline__ int var(int k) const { return r[2 + k]; }
};

template <int D, bool EXACT, int FPC>
__device__ __forceinline__ void cn_update(const Shared& s, const int32_t* __restrict__ rec, unsigned f) {
  const CnRecord<D, EXACT> cr(rec);
  const int off = cr.off(), deg = cr.deg();
  float x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    x[k] = 0.f;
    if (EXACT || k < deg) x[k] = clamp_llr(s.P[cr.var(k) * FPC + f] - s.c2v[(off + k) * FPC + f]);
  }
  boxplus_row<D, EXACT>(x, deg, [&](int k, float c) { s.c2v[(off + k) * FPC + f] = c; });
}

// P_v = L_v + sum of c2v over the VN's edges in ascending-CN order (the
// totals of decoder.hpp:162-165; refreshes every v2c of v at once).
template <int FPC, int VS>
__device__ __forceinline__ void vn_refresh(const Shared& s, const int4* __restrict__ rec, int vs4, unsigned f) {
  int4 t = __ldg(rec);
  const int v = t.x;
  float acc = s.L[v * FPC + f];
  acc += s.c2v[t.y * FPC + f];
  acc += s.c2v[t.z * FPC + f];
  acc += s.c2v[t.w * FPC + f];
  const int nq = VS > 0 ? VS : vs4;
#pragma unroll
  for (int q = 1; q < nq; ++q) {
    t = __ldg(rec + q);
    acc += s.c2v[t.x * FPC + f];
    acc += s.c2v[t.y * FPC + f];
    acc += s.c2v[t.z * FPC + f];
    acc += s.c2v[t.w * FPC + f];
  }
  s.P[v * FPC + f] = acc;
}

template <int D, bool EXACT, int FPC>
__device__ __forceinline__ unsigned parity(const Shared& s, const int32_t* __restrict__ rec, unsigned f) {
  const CnRecord<D, EXACT> cr(rec);
  unsigned p = 0;
#pragma unroll
  for (int k = 0; k < D; ++k)
    if (EXACT || k < cr.deg()) p ^= static_cast<unsigned>(s.P[cr.var(k) * FPC + f] < 0.f);
  return p;
}

constexpr int max_threads_for(int D) { return D <= 8 ? 1024 : 512; }

template <int D, bool EXACT, int FPC, int VS>
__global__ void __launch_bounds__(max_threads_for(D)) decode_resident(const DevGraph g, const DecodeArgs a) {
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_active;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = g.n, E = g.E, cs = g.cs;
  Shared s;
  s.c2v = smem;
  s.P = s.c2v + static_cast<size_t>(E + 1) * FPC;
  s.L = s.P + static_cast<size_t>(n) * FPC;
  s.done = reinterpret_cast<int*>(s.L + static_cast<size_t>(n) * FPC);
  s.weight = s.done + FPC;
  s.iters = s.weight + FPC;
  s.conv = s.iters + FPC;
  s.berr = s.conv + FPC;

  const int64_t f0 = static_cast<int64_t>(blockIdx.x) * FPC;
  const int nf = static_cast<int>(min(static_cast<int64_t>(FPC), a.frames - f0));

  // ---- prologue: init_state (decoder.hpp:39-52) in posterior form
  const float* llr = a.llr + f0 * n;
  for (int i = tid; i < nf * n; i += nt) {
    const int f = i / n, v = i - f * n;
    const float x = clamp_llr(__ldg(llr + i));
    s.L[v * FPC + f] = x;
    s.P[v * FPC + f] = x;
  }
  {
    const int total = (E + 1) * FPC;
    float4* c4 = reinterpret_cast<float4*>(s.c2v);
    for (int i = tid; i < total / 4; i += nt) c4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = total / 4 * 4 + tid; i < total; i += nt) s.c2v[i] = 0.f;
  }
  if (tid < FPC) {
    s.done[tid] = tid >= nf;
    s.weight[tid] = 0;
    s.iters[tid] = 0;
    s.conv[tid] = 0;
    s.berr[tid] = 0;
  }
  if (a.trace)
    for (int i = tid; i < nf * a.max_iters; i += nt) a.trace[f0 * a.max_iters + i] = -1;
  __syncthreads();

  const bool dump = a.max_subiters > 0;
  int sub = 0;
  for (int iter = 1; iter <= a.max_iters; ++iter) {
    for (int grp = 0; grp < g.G; ++grp) {
      if (dump && sub == a.max_subiters) goto finish;
      ++sub;
      // CN phase: every (CN of the group, frame) item; Jacobi within the group
      const int c0 = __ldg(g.cn_off + grp);
      const unsigned cnt = static_cast<unsigned>(__ldg(g.cn_off + grp + 1) - c0) * FPC;
      for (unsigned it = tid; it < cnt; it += nt) {
        const unsigned f = it % FPC;
        if (s.done[f]) continue;
        cn_update<D, EXACT, FPC>(s, g.cn_rec + static_cast<size_t>(c0 + it / FPC) * cs, f);
      }
      __syncthreads();
      // VN phase: every (touched VN, frame) item
      const int t0 = __ldg(g.vn_off + grp);
      const unsigned tcnt = static_cast<unsigned>(__ldg(g.vn_off + grp + 1) - t0) * FPC;
      const int4* vrec = reinterpret_cast<const int4*>(g.vn_rec);
      for (unsigned it = tid; it < tcnt; it += nt) {
        const unsigned f = it % FPC;
        if (s.done[f]) continue;
        vn_refresh<FPC, VS>(s, vrec + static_cast<size_t>(t0 + it / FPC) * g.vs4, g.vs4, f);
      }
      __syncthreads();
    }
    if (dump) continue;
    if (!(a.early_stop || a.trace || iter == a.max_iters)) continue;
    // ---- hard decision + syndrome weight (decoder.hpp:166-171)
    {
      const unsigned cnt = static_cast<unsigned>(g.m) * FPC;
      for (unsigned it = tid; it < cnt; it += nt) {
        const unsigned f = it % FPC;
        if (s.done[f]) continue;
        if (parity<D, EXACT, FPC>(s, g.all_rec + static_cast<size_t>(it / FPC) * cs, f)) atomicAdd(&s.weight[f], 1);
      }
    }
    __syncthreads();
    if (tid == 0) {
      int active = 0;
      for (int f = 0; f < nf; ++f) {
        if (s.done[f]) continue;
        const int w = s.weight[f];
        if (a.trace) a.trace[(f0 + f) * a.max_iters + iter - 1] = w;
        s.iters[f] = iter;
        s.conv[f] = w == 0;
        s.weight[f] = 0;
        if (w == 0 && a.early_stop)
          s.done[f] = 1;  // decoder.hpp:173-177
        else
          ++active;
      }
      s_active = active;
    }
    __syncthreads();
    if (s_active == 0) break;
  }
finish:
  __syncthreads();
  if (dump) {
    for (int i = tid; i < nf * E; i += nt) {
      const int f = i / E, e = i - f * E;
      const float c = s.c2v[e * FPC + f];
      if (a.c2v_out) a.c2v_out[f0 * E + i] = c;
      if (a.v2c_out) a.v2c_out[f0 * E + i] = clamp_llr(s.P[__ldg(g.cols + e) * FPC + f] - c);
    }
    return;
  }
  // ---- epilogue: hard decisions, error counts
  if (a.bits && a.bits_packed) {
    const int nb = (n + 7) >> 3;
    for (int i = tid; i < nb * FPC; i += nt) {
      const int f = i % FPC, b = i / FPC;
      if (f >= nf) continue;
      unsigned byte = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int v = b * 8 + j;
        if (v < n && s.P[v * FPC + f] < 0.f) byte |= 1u << j;
      }
      a.bits[(f0 + f) * nb + b] = static_cast<uint8_t>(byte);
      if (byte) atomicAdd(&s.berr[f], __popc(byte));
    }
  } else if (a.bits || a.counters) {
    for (int i = tid; i < nf * n; i += nt) {
      const int f = i / n, v = i - f * n;
      const int bit = s.P[v * FPC + f] < 0.f;  // tie -> 0 (decoder.hpp:166)
      if (a.bits) a.bits[f0 * n + i] = static_cast<uint8_t>(bit);
      if (bit) atomicAdd(&s.berr[f], 1);
    }
  }
  if (a.posterior)
    for (int i = tid; i < nf * n; i += nt) {
      const int f = i / n, v = i - f * n;
      a.posterior[f0 * n + i] = s.P[v * FPC + f];
    }
  if (tid < nf) {
    const int it = a.early_stop ? s.iters[tid] : a.max_iters;
    if (a.iterations) a.iterations[f0 + tid] = it;
    if (a.converged) a.converged[f0 + tid] = static_cast<uint8_t>(s.conv[tid]);
  }
  __syncthreads();
  if (tid == 0 && a.counters) {
    unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
    for (int f = 0; f < nf; ++f) {
      const int it = a.early_stop ? s.iters[f] : a.max_iters;
      c[0] += 1;
      c[1] += s.berr[f];
      c[2] += s.berr[f] > 0;
      c[3] += s.conv[f];
      c[4] += it;
      c[5] += s.conv[f] ? it : 0;
    }
    for (int i = 0; i < 6; ++i) atomicAdd(a.counters + i, c[i]);
  }
}

// ---- channel: transmit_all_zero (channel.hpp:38-46), fp64 then fp32
__global__ void channel_kernel(int n, double sigma, double scale, uint64_t seed, int64_t frame0, int64_t frames,
                               float* __restrict__ llr) {
  const int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= frames) return;
  Stream rng(stream_seed(seed, static_cast<uint64_t>(frame0 + f)));
  float* out = llr + f * n;
  for (int i = 0; i < n; ++i) out[i] = static_cast<float>(scale * (1.0 + sigma * rng.normal()));
}

// ---- one CN per thread on explicit inputs (check_update KATs)
template <int D, bool EXACT>
__global__ void check_update_kernel(int deg, int64_t rows, const float* __restrict__ v2c, float* __restrict__ c2v) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = (EXACT || k < deg) ? clamp_llr(v2c[r * deg + k]) : 0.f;
  boxplus_row<D, EXACT>(x, deg, [&](int k, float c) { c2v[r * deg + k] = c; });
}

using KernelFn = void (*)(const DevGraph, const DecodeArgs);

template <int D, bool EXACT, int VS>
KernelFn pick_fpc(int fpc) {
  switch (fpc) {
    case 1: return decode_resident<D, EXACT, 1, VS>;
    case 2: return decode_resident<D, EXACT, 2, VS>;
    case 4: return decode_resident<D, EXACT, 4, VS>;
    case 8: return decode_resident<D, EXACT, 8, VS>;
    case 16: return decode_resident<D, EXACT, 16, VS>;
    default: return nullptr;
  }
}

KernelFn pick_kernel(const DevGraph& g, int fpc, int* bucket) {
  *bucket = cn_bucket(g.max_cdeg, g.cregular);
  switch (*bucket) {
    case 6: return g.vs4 == 1 ? pick_fpc<6, true, 1>(fpc) : pick_fpc<6, true, 0>(fpc);
    case 3: return pick_fpc<3, true, 0>(fpc);
    case 8: return pick_fpc<8, false, 0>(fpc);
    case 16: return pick_fpc<16, false, 0>(fpc);
    case 32: return pick_fpc<32, false, 0>(fpc);
    default: return nullptr;
  }
}

size_t frame_bytes(const DevGraph& g) { return 4ull * (static_cast<size_t>(g.E) + 1 + 2ull * g.n); }

int device_smem_optin() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 227 * 1024;
  cache[dev] = v;
  return v;
}

}  // namespace

void set_tuning(int fpc, int threads) {
  g_tune_fpc = fpc;
  g_tune_threads = threads;
}

int64_t kernel_launch_count() { return g_launches.load(); }

Plan plan_decode(const DevGraph& g, int64_t frames) {
  Plan p;
  const size_t limit = static_cast<size_t>(device_smem_optin()) - 1024;
  const size_t per = frame_bytes(g);
  auto bytes = [&](int f) { return f * per + 20 * f + 16; };
  int fpc = g_tune_fpc.load();
  if (fpc <= 0) {
    fpc = 8;
    while (fpc > 1 && bytes(fpc) > limit) fpc /= 2;
  }
  if (bytes(fpc) > limit) return p;  // does not fit: no resident plan
  int bucket = 0;
  if (!pick_kernel(g, fpc, &bucket)) return p;
  const int max_nt = bucket <= 8 ? 1024 : 512;
  int nt = g_tune_threads.load();
  if (nt <= 0) {
    // one CN item per thread for the largest group, in whole warps
    nt = (fpc * g.max_cn_items + 31) / 32 * 32;
    nt = std::max(128, std::min(nt, max_nt));
  }
  p.kernel = 1;
  p.fpc = fpc;
  p.threads = std::min(nt, max_nt);
  p.smem = static_cast<int>(bytes(fpc));
  p.degree_bucket = bucket;
  p.ctas = (frames + fpc - 1) / fpc;
  return p;
}

int launch_decode(const DevGraph& g, const DecodeArgs& a, void* stream, Plan* used) {
  const Plan p = plan_decode(g, a.frames);
  if (used) *used = p;
  if (p.kernel == 0) return static_cast<int>(cudaErrorInvalidConfiguration);
  if (a.frames <= 0) return 0;
  int bucket = 0;
  KernelFn fn = pick_kernel(g, p.fpc, &bucket);
  cudaError_t err = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
  if (err != cudaSuccess) return static_cast<int>(err);
  // grid.x limit is 2^31-1, far above any batch
  fn<<<static_cast<unsigned>(p.ctas), p.threads, p.smem, static_cast<cudaStream_t>(stream)>>>(g, a);
  ++g_launches;
  return static_cast<int>(cudaGetLastError());
}

int launch_channel(int n, double sigma2, uint64_t seed, int64_t frame0, int64_t frames, float* llr, void* stream) {
  if (frames <= 0) return 0;
  const double sigma = std::sqrt(sigma2);  // channel.hpp:41-42
  const double scale = 2.0 / sigma2;
  const int tpb = 128;
  const int64_t blocks = (frames + tpb - 1) / tpb;
  channel_kernel<<<static_cast<unsigned>(blocks), tpb, 0, static_cast<cudaStream_t>(stream)>>>(
      n, sigma, scale, seed, frame0, frames, llr);
  ++g_launches;
  return static_cast<int>(cudaGetLastError());
}

int launch_check_update(int degree, int64_t rows, const float* v2c, float* c2v, void* stream) {
  if (rows <= 0) return 0;
  const int tpb = 128;
  const unsigned blocks = static_cast<unsigned>((rows + tpb - 1) / tpb);
  auto st = static_cast<cudaStream_t>(stream);
  if (degree == 6)
    check_update_kernel<6, true><<<blocks, tpb, 0, st>>>(degree, rows, v2c, c2v);
  else if (degree <= 8)
    check_update_kernel<8, false><<<blocks, tpb, 0, st>>>(degree, rows, v2c, c2v);
  else if (degree <= 16)
    check_update_kernel<16, false><<<blocks, tpb, 0, st>>>(degree, rows, v2c, c2v);
  else if (degree <= 32)
    check_update_kernel<32, false><<<blocks, tpb, 0, st>>>(degree, rows, v2c, c2v);
  else
    return static_cast<int>(cudaErrorInvalidValue);
  ++g_launches;
  return static_cast<int>(cudaGetLastError());
}

}  // namespace ldpcb
