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
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "host.hpp"
#include "kernels.cuh"
#include "rng.cuh"

namespace ldpcb {
namespace {

using namespace dev;

std::atomic<int64_t> g_launches{0};
std::atomic<int> g_tune_fpc{0}, g_tune_threads{0}, g_tune_fv{0}, g_lazy_totals{1}, g_force_kernel{0};

// Frame-interleaved shared memory: element i of a per-slot or per-VN array of
// frame f lives at [i * FPC + f]. A thread serves FV adjacent frames (one
// 32-bit or 64-bit shared access per element), so graph records, index math
// and loop overhead are shared by FV frames and FV boxplus chains interleave.
//   c2v : [n_slots] check-to-variable messages (last slot stays zero)
//   P   : [n]       posterior = channel + all c2v (unclamped)
//   L   : [n]       clamped channel LLR
// v2c is never stored: v2c = clamp(P_v - c2v_e), the posterior form of
// var_update (decoder.hpp:91-105). A VN touched by only this CN of the group
// (mask bit) gets its posterior updated in place, P += c2v_new - c2v_old:
// no other CN of the group reads it, so the Jacobi order of
// decoder.hpp:107-113 is kept.
template <int FV>
struct FVec {
  float v[FV];
};

template <int FV>
__device__ __forceinline__ FVec<FV> lds(const float* p) {
  FVec<FV> r;
  if constexpr (FV == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    r.v[0] = t.x;
    r.v[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < FV; ++i) r.v[i] = p[i];
  }
  return r;
}

template <int FV>
__device__ __forceinline__ void sts(float* p, const FVec<FV>& x) {
  if constexpr (FV == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(x.v[0], x.v[1]);
  } else {
#pragma unroll
    for (int i = 0; i < FV; ++i) p[i] = x.v[i];
  }
}

// Keeps the consumers of a prefetched value below this point: the compiler
// otherwise hoists address arithmetic on a record loaded one phase ahead up
// to the load and stalls on it.
__device__ __forceinline__ void pin(int4& t) { asm volatile("" : "+r"(t.x), "+r"(t.y), "+r"(t.z), "+r"(t.w)); }
template <int N>
__device__ __forceinline__ void pin(int (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}
template <int D, bool EXACT>
__device__ __forceinline__ void pin_rec(CnRecord<D, EXACT>& c) { pin(c.r); }
template <int D>
__device__ __forceinline__ void pin_rec(CnRecordPacked<D>& c) { pin(c.w); }

// live: bit i set when frame i of this thread's vector is still decoding
template <int D, bool EXACT, int FPC, int FV, bool ALL_LIVE, class Rec>
__device__ __forceinline__ void cn_update(float* __restrict__ c2v, float* __restrict__ P, const Rec& cr,
                                          unsigned live) {
  const int base = cr.slot();
  const unsigned mask = cr.mask();
  const int deg = cr.deg();
  if constexpr (FV == 1) {
    // one frame: v2c in registers only; every output is stored as the
    // boxplus emits it (keeps wide rows, D = 16 / 32, within the register file)
    if (!ALL_LIVE && !(live & 1u)) return;
    auto row = [&](auto width) {
      constexpr int W = decltype(width)::value;
      float x[W];
#pragma unroll
      for (int k = 0; k < W; ++k) x[k] = cr.has(k) ? P[cr.var(k) * FPC] - c2v[(base + k) * FPC] : 0.f;
      boxplus_row<W, EXACT && W == D>(x, deg, [&](int k, float c) {
        c2v[(base + k) * FPC] = c;
        // in-place posterior: P + (c - old) = v2c + c (v2c = P - old, unclamped)
        if (mask & (1u << k)) P[cr.var(k) * FPC] = x[k] + c;
      });
    };
    // a row of exactly W edges: no padding positions, no per-position predicates
    auto row_exact = [&](auto width) {
      constexpr int W = decltype(width)::value;
      float x[W];
#pragma unroll
      for (int k = 0; k < W; ++k) x[k] = P[cr.var(k) * FPC] - c2v[(base + k) * FPC];
      boxplus_row<W, true>(x, W, [&](int k, float c) {
        c2v[(base + k) * FPC] = c;
        if (mask & (1u << k)) P[cr.var(k) * FPC] = x[k] + c;
      });
    };
    // wide buckets: rows of degree <= 8 (most QC block rows; warps are
    // homogeneous because a group lists whole block rows) take code of their
    // exact width (padding with the boxplus identity (0, 1) is exact, so the
    // outputs are those of the 8-wide code), degree-3..8 rows without padding
    if constexpr (!EXACT && D > 8) {
      switch (deg) {
        case 3: row_exact(std::integral_constant<int, 3>{}); return;
        case 4: row_exact(std::integral_constant<int, 4>{}); return;
        case 5: row_exact(std::integral_constant<int, 5>{}); return;
        case 6: row_exact(std::integral_constant<int, 6>{}); return;
        case 7: row_exact(std::integral_constant<int, 7>{}); return;
        case 8: row_exact(std::integral_constant<int, 8>{}); return;
        default:
          if (deg <= 8) {
            row(std::integral_constant<int, 8>{});
            return;
          }
      }
    }
    row(std::integral_constant<int, D>{});
    return;
  }
  FVec<FV> pv[D], old[D], out[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (cr.has(k)) {
      pv[k] = lds<FV>(P + cr.var(k) * FPC);
      old[k] = lds<FV>(c2v + (base + k) * FPC);
    } else {
#pragma unroll
      for (int i = 0; i < FV; ++i) pv[k].v[i] = old[k].v[i] = 0.f;
    }
  }
  if constexpr (FV == 2) {  // both frames per packed fp32 instruction
    f32x2 x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = sub2(pack2(pv[k].v[0], pv[k].v[1]), pack2(old[k].v[0], old[k].v[1]));
    boxplus_row_x2<D, EXACT>(x, deg, [&](int k, f32x2 c) {
      const f32x2 p = add2(x[k], c);  // in-place posterior: v2c + c
      if (ALL_LIVE || (live & 1u)) {
        out[k].v[0] = lo2(c);
        pv[k].v[0] = lo2(p);
      } else {
        out[k].v[0] = old[k].v[0];
      }
      if (ALL_LIVE || (live & 2u)) {
        out[k].v[1] = hi2(c);
        pv[k].v[1] = hi2(p);
      } else {
        out[k].v[1] = old[k].v[1];
      }
    });
  } else {
#pragma unroll
    for (int i = 0; i < FV; ++i) {
      float x[D];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = pv[k].v[i] - old[k].v[i];
      boxplus_row<D, EXACT>(x, deg, [&](int k, float c) {
        out[k].v[i] = (ALL_LIVE || (live & (1u << i))) ? c : old[k].v[i];
        // in-place posterior: P + (c - old) = v2c + c (v2c = P - old, unclamped)
        pv[k].v[i] = (ALL_LIVE || (live & (1u << i))) ? x[k] + c : pv[k].v[i];
      });
    }
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (!cr.has(k)) continue;
    sts<FV>(c2v + (base + k) * FPC, out[k]);
    if (mask & (1u << k)) sts<FV>(P + cr.var(k) * FPC, pv[k]);
  }
}

// P_v = L_v + sum of c2v over the VN's edges in ascending-CN order: the
// totals of decoder.hpp:162-165 (and every v2c of v refreshed at once).
// Records are padded with the zero slot after the VN's last edge: padding is
// skipped and the record walk stops at the first row that ends in padding
// (fix-up and totals records are grouped by VN degree, so warps stop together).
template <int FPC, int FV, int VS>
__device__ __forceinline__ void vn_sum(const float* __restrict__ c2v, float* __restrict__ P,
                                       const float* __restrict__ L, const int4* __restrict__ rec, int vs4, int4 t,
                                       int zero) {
  const int v = t.x;
  FVec<FV> acc = lds<FV>(L + v * FPC);
  auto add = [&](int slot) {
    if (VS <= 0 && slot == zero) return;
    const FVec<FV> c = lds<FV>(c2v + slot * FPC);
    if constexpr (FV == 2) {
      const f32x2 t = add2(pack2(acc.v[0], acc.v[1]), pack2(c.v[0], c.v[1]));
      acc.v[0] = lo2(t);
      acc.v[1] = hi2(t);
    } else {
#pragma unroll
      for (int i = 0; i < FV; ++i) acc.v[i] += c.v[i];
    }
  };
  add(t.y);
  add(t.z);
  add(t.w);
  const int nq = VS > 0 ? VS : vs4;
#pragma unroll
  for (int q = 1; q < nq; ++q) {
    if (VS <= 0 && t.w == zero) break;
    t = __ldg(rec + q);
    add(t.x);
    add(t.y);
    add(t.z);
    add(t.w);
  }
  sts<FV>(P + v * FPC, acc);
}

// Two independent VN records per step so their loads overlap.
template <int FPC, int FV, int VS>
__device__ __forceinline__ void vn_sum_range(const float* __restrict__ c2v, float* __restrict__ P,
                                             const float* __restrict__ L, const int4* __restrict__ rec, int vs4,
                                             int j0, int count, int jstep, int zero) {
  int j = j0;
  for (; j + jstep < count; j += 2 * jstep) {
    const int4 a = __ldg(rec + j * vs4), b = __ldg(rec + (j + jstep) * vs4);
    vn_sum<FPC, FV, VS>(c2v, P, L, rec + j * vs4, vs4, a, zero);
    vn_sum<FPC, FV, VS>(c2v, P, L, rec + (j + jstep) * vs4, vs4, b, zero);
  }
  if (j < count) vn_sum<FPC, FV, VS>(c2v, P, L, rec + j * vs4, vs4, __ldg(rec + j * vs4), zero);
}

// The same re-sum from a 16-bit record (host.hpp KernelTables::fix_rec16):
// eight fields per 16-byte row, so one row serves a VN of degree <= 7.
template <int FPC, int FV>
__device__ __forceinline__ void vn_sum16(const float* __restrict__ c2v, float* __restrict__ P,
                                         const float* __restrict__ L, const int4* __restrict__ rec, int vs16, int4 t,
                                         int zero) {
  const int v = t.x & 0xffff;
  FVec<FV> acc = lds<FV>(L + v * FPC);
  auto add = [&](int slot) {
    if (slot == zero) return;
    const FVec<FV> c = lds<FV>(c2v + slot * FPC);
#pragma unroll
    for (int i = 0; i < FV; ++i) acc.v[i] += c.v[i];
  };
  auto add2w = [&](int w) {
    add(w & 0xffff);
    add(static_cast<int>(static_cast<unsigned>(w) >> 16));
  };
  add(static_cast<int>(static_cast<unsigned>(t.x) >> 16));
  add2w(t.y);
  add2w(t.z);
  add2w(t.w);
  for (int q = 1; q < vs16 && static_cast<int>(static_cast<unsigned>(t.w) >> 16) != zero; ++q) {
    t = __ldg(rec + q);
    add2w(t.x);
    add2w(t.y);
    add2w(t.z);
    add2w(t.w);
  }
  sts<FV>(P + v * FPC, acc);
}
template <int FPC, int FV>
__device__ __forceinline__ void vn_sum16_range(const float* __restrict__ c2v, float* __restrict__ P,
                                               const float* __restrict__ L, const int4* __restrict__ rec, int vs16,
                                               int j0, int count, int jstep, int zero) {
  int j = j0;
  for (; j + jstep < count; j += 2 * jstep) {
    const int4 a = __ldg(rec + j * vs16), b = __ldg(rec + (j + jstep) * vs16);
    vn_sum16<FPC, FV>(c2v, P, L, rec + j * vs16, vs16, a, zero);
    vn_sum16<FPC, FV>(c2v, P, L, rec + (j + jstep) * vs16, vs16, b, zero);
  }
  if (j < count) vn_sum16<FPC, FV>(c2v, P, L, rec + j * vs16, vs16, __ldg(rec + j * vs16), zero);
}

// parity bit of each frame of the vector
template <int D, bool EXACT, int FPC, int FV>
__device__ __forceinline__ unsigned parity(const float* __restrict__ P, const int32_t* __restrict__ rec, int cs) {
  const ResidentRecord<D, EXACT> cr(rec, cs);
  unsigned p = 0;
#pragma unroll
  for (int k = 0; k < D; ++k)
    if (cr.has(k)) {
      const FVec<FV> x = lds<FV>(P + cr.var(k) * FPC);
#pragma unroll
      for (int i = 0; i < FV; ++i) p ^= static_cast<unsigned>(x.v[i] < 0.f) << i;
    }
  return p;
}

// One sub-iteration of a per-frame grouping (RND): group grp of the frame's
// staged list `lst` (decoder.hpp:112-127). CN phase from the per-CN records,
// barrier, then every VN of the group re-summed exactly, barrier. The
// thread's first CN record was requested one group ahead (group 0: now,
// after the iteration's lists were staged); the next group's is requested here.
template <int D, bool EXACT, int FPC, int FV, int VS, class Rec>
__device__ __forceinline__ void rnd_group(const DevGraph& g, int CS, int vs4, float* __restrict__ c2v,
                                          float* __restrict__ P, const float* __restrict__ L, const int4* s_go,
                                          const uint16_t* lst0, int grp, int j0, int jstep, unsigned live,
                                          Rec& next_cn) {
  const int4* const all_vn = reinterpret_cast<const int4*>(g.all_vn_rec);  // indexed by VN position
  const int c0 = s_go[grp].x, cn = s_go[grp].y - c0;
  const uint16_t* lst = lst0 + c0;
  Rec cur = next_cn;
  if (grp == 0 && j0 < cn) cur.load(g.all_rec + lst[j0] * CS, CS);
  if (grp + 1 < g.G) {
    const int c1 = s_go[grp + 1].x;
    if (j0 < s_go[grp + 1].y - c1) next_cn.load(g.all_rec + lst0[c1 + j0] * CS, CS);
  }
  if (live && j0 < cn) {
    cn_update<D, EXACT, FPC, FV, true>(c2v, P, cur, live);
    for (int j = j0 + jstep; j < cn; j += jstep)
      cn_update<D, EXACT, FPC, FV, true>(c2v, P, Rec(g.all_rec + lst[j] * CS, CS), live);
  }
  // VN records of the first CN's edges, requested before the barrier
  constexpr int KT = D <= 8 ? D : 1;
  int4 t0[KT];
  if constexpr (D <= 8)
    if (live && j0 < cn)
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (cur.has(k)) t0[k] = __ldg(all_vn + cur.var(k) * vs4);
  __syncthreads();
  // every VN of the group re-summed from its record (a VN shared by several
  // CNs is written several times with the same value): each thread re-sums
  // the VNs of the CNs it updated, their VN records requested before any is used
  auto resum = [&](const Rec& r) {
#pragma unroll
    for (int k0 = 0; k0 < D; k0 += 4) {
      int4 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u < D && r.has(k0 + u)) t[u] = __ldg(all_vn + r.var(k0 + u) * vs4);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u < D && r.has(k0 + u)) vn_sum<FPC, FV, VS>(c2v, P, L, all_vn + r.var(k0 + u) * vs4, vs4, t[u], g.n_slots - 1);
    }
  };
  if (live && j0 < cn) {
    if constexpr (D <= 8) {
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (cur.has(k)) vn_sum<FPC, FV, VS>(c2v, P, L, all_vn + cur.var(k) * vs4, vs4, t0[k], g.n_slots - 1);
    } else {
      resum(cur);
    }
    for (int j = j0 + jstep; j < cn; j += jstep) resum(Rec(g.all_rec + lst[j] * CS, CS));
  }
  __syncthreads();
}

#ifndef LDPCB_WIDE_THREADS
#define LDPCB_WIDE_THREADS 256
#endif
constexpr int kWideThreads = LDPCB_WIDE_THREADS;  // 16-wide bucket, one frame per thread
constexpr int max_threads_for(int D, int FV) {
  return FV == 2 ? 256 : (D <= 8 ? 512 : (D <= 16 ? kWideThreads : 128));
}

#ifdef LDPCB_PHASE_TIMING
// Debug build only (scripts/phase_timing.py): CTA-level cycle counts of the
// phases of decode_resident, taken by thread 0 between barriers: [CN phase,
// fix-up phase, iteration end, whole kernel, group phases, CTAs].
__device__ unsigned long long g_phase_cycles[8];
#define PT_MARK(var) long long var = clock64()
#else
#define PT_MARK(var)
#endif

// RND: per-frame random grouping (host.hpp ScheduleData::per_frame). Each
// frame's ordered CN groups come from a generated list (gen_groups_kernel);
// the CN records are the per-CN ones (no in-place posterior updates) and
// after every CN phase each edge of the group re-sums its VN exactly.
template <int D, bool EXACT, int FPC, int FV, int VS, bool RND = false>
__global__ void __launch_bounds__(max_threads_for(D, FV), D <= 16 ? 2 : 1) decode_resident(const DevGraph g,
                                                                                          const DecodeArgs a) {
  static_assert(!RND || FV == 1, "per-frame groupings need one frame per thread");
  const int CS = g.cs;  // CN record stride (ints): packed 4 or CnRecord::kInts
  constexpr int NG = FPC / FV;  // frame vectors per CTA
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_active;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = g.n, m = g.m, S = g.n_slots;
  const int vs4 = VS > 0 ? VS : g.vs4;
  const int fg = tid % NG, j0 = tid / NG, jstep = nt / NG;
  const int fb = fg * FV;  // first frame of this thread's vector
  float* const c2v = smem + fb;
  float* const P = smem + S * FPC + fb;
  float* const L = P + n * FPC;
  int* const s_done = reinterpret_cast<int*>(smem + (S + 2 * n) * FPC);
  int* const s_weight = s_done + FPC;
  int* const s_iters = s_weight + FPC;
  int* const s_conv = s_iters + FPC;
  int* const s_berr = s_conv + FPC;
  // staged group tables: s_go[g] = {first CN item, end, first fix-up item, end}
  int4* const s_go = reinterpret_cast<int4*>(smem + (((S + 2 * n) * FPC + 5 * FPC + 3) & ~3));
  uint16_t* const s_list = reinterpret_cast<uint16_t*>(s_go + g.G);  // RND: [FPC][slots]
  const int slots = a.list_slots;
  const int4* const tot_vn = reinterpret_cast<const int4*>(g.tot_vn_rec);  // bank-coloured order
  const int4* const fix_vn = reinterpret_cast<const int4*>(g.fix_rec);
  const int4* const fix16 = reinterpret_cast<const int4*>(g.fix_rec16);
  const int vs16 = VS > 0 ? 0 : g.vs16;  // 16-bit fix-up records (multi-row VN records only)
  const int4* const tot16 = reinterpret_cast<const int4*>(g.tot_rec16);

  const int64_t f0 = static_cast<int64_t>(blockIdx.x) * FPC;
  const int nf = static_cast<int>(min(static_cast<int64_t>(FPC), a.frames - f0));
#ifdef LDPCB_PHASE_TIMING
  const long long pt_entry = clock64();
#endif

  // ---- prologue: init_state (decoder.hpp:39-52) in posterior form, log2 units
  {
    const float* llr = a.llr + f0 * n;
    auto put = [&](int i, float raw) {  // element i of the CTA's frames -> P and L
      const int ff = i / n, v = __ldg(g.vn_pos + (i - ff * n));
      const float x = clamp_llr(raw) * kLog2e;
      smem[(S + v) * FPC + ff] = x;
      smem[(S + n + v) * FPC + ff] = x;
    };
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(a.llr) & 15) == 0) {
      // 16-byte loads, four per thread in flight before any is used
      constexpr int U = 4;
      const float4* l4 = reinterpret_cast<const float4*>(llr);
      const int nv = nf * n / 4;
      for (int b0 = tid; b0 < nv; b0 += U * nt) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (b0 + u * nt < nv) x[u] = ldg_stream(l4 + b0 + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (b0 + u * nt < nv) {
            const int i = 4 * (b0 + u * nt);
            put(i, x[u].x);
            put(i + 1, x[u].y);
            put(i + 2, x[u].z);
            put(i + 3, x[u].w);
          }
      }
    } else {
      for (int i = tid; i < nf * n; i += nt) put(i, __ldg(llr + i));
    }
    for (int i = nf * n + tid; i < FPC * n; i += nt) {  // padding frames: saturated zero codeword
      const int ff = i / n, v = i - ff * n;
      smem[(S + v) * FPC + ff] = kClampB;
      smem[(S + n + v) * FPC + ff] = kClampB;
    }
    const int total = S * FPC;
    float4* c4 = reinterpret_cast<float4*>(smem);
    for (int i = tid; i < total / 4; i += nt) c4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = total / 4 * 4 + tid; i < total; i += nt) smem[i] = 0.f;
  }
  if (tid < FPC) {
    s_done[tid] = tid >= nf;
    s_weight[tid] = 0;
    s_iters[tid] = 0;
    s_conv[tid] = 0;
    s_berr[tid] = 0;
  }
  for (int i = tid; i < g.G; i += nt) {
    s_go[i] = make_int4(__ldg(g.cn_off + i), __ldg(g.cn_off + i + 1), __ldg(g.fix_off + i), __ldg(g.fix_off + i + 1));
  }
  if (a.trace)
    for (int i = tid; i < nf * a.max_iters; i += nt) a.trace[f0 * a.max_iters + i] = -1;
  __syncthreads();
  auto live_bits = [&](int first) {
    unsigned b = 0;
#pragma unroll
    for (int i = 0; i < FV; ++i) b |= static_cast<unsigned>(!s_done[first + i]) << i;
    return b;
  };
  unsigned live = live_bits(fb);
  // records are prefetched one phase ahead: the first CN item of the next
  // group and the first fix-up item of the current one
  using Rec = ResidentRecord<D, EXACT>;
  Rec next_cn;
  if (!RND && j0 < s_go[0].y - s_go[0].x) next_cn.load(g.cn_rec + static_cast<size_t>(s_go[0].x + j0) * CS, CS);
  // the current group's offsets, in registers; the next group's are read one
  // group ahead so no shared-memory read sits on the critical path
  int4 go = s_go[0];

  const bool dump = a.max_subiters > 0;
  int sub = 0;
#ifdef LDPCB_PHASE_TIMING
  unsigned long long pt_cn = 0, pt_fix = 0, pt_end = 0, pt_groups = 0;
  const long long pt_start = clock64();
  long long pt_loop_end = 0;
#endif
  for (int iter = 1; iter <= a.max_iters; ++iter) {
    if constexpr (RND) {
      if (iter == 1 || a.n_lists > 1) {  // this iteration's groups (decoder.hpp:153-156)
        const int li = a.n_lists > 1 ? iter - 1 : 0;
        // padding frames get CN 0 everywhere: their record loads (issued
        // whether or not the frame is live) must stay in bounds
        for (int i = tid; i < FPC * slots; i += nt) {
          const int ff = i / slots, j = i - ff * slots;
          s_list[i] = ff < nf ? a.lists[((f0 + ff) * a.n_lists + li) * slots + j] : 0;
        }
        __syncthreads();
      }
    }
    for (int grp = 0; grp < g.G; ++grp) {
      if (dump && sub == a.max_subiters) goto finish;
      ++sub;
      // CN phase: every (CN of the group, frame vector); Jacobi within the group
      if constexpr (RND) {
        rnd_group<D, EXACT, FPC, FV, VS>(g, CS, vs4, c2v, P, L, s_go, s_list + fb * slots, grp, j0, jstep, live,
                                         next_cn);
        continue;
      }
      PT_MARK(pt_a);
      const int c0 = go.x, cn = go.y - go.x;
      const int x0 = go.z, xn = go.w - go.z;
      const int4 ngo = s_go[grp + 1 < g.G ? grp + 1 : 0];  // one broadcast read, one group ahead
      int4 fix_first = make_int4(0, 0, 0, 0);
      if (j0 < xn)
        fix_first = vs16 ? __ldg(fix16 + static_cast<size_t>(x0 + j0) * vs16)
                         : __ldg(fix_vn + static_cast<size_t>(x0 + j0) * vs4);
      // this thread's first record was loaded one group ago; the next group's
      // is requested now, a whole CN + fix-up phase before it is needed (the
      // records come from L2: shared memory leaves little L1)
      const Rec cur = next_cn;
      if (j0 < ngo.y - ngo.x) next_cn.load(g.cn_rec + static_cast<size_t>(ngo.x + j0) * CS, CS);
      if (live && j0 < cn) {
        const int32_t* rec = g.cn_rec + static_cast<size_t>(c0) * CS;
        if (live == (1u << FV) - 1) {
          cn_update<D, EXACT, FPC, FV, true>(c2v, P, cur, live);
          for (int j = j0 + jstep; j < cn; j += jstep)
            cn_update<D, EXACT, FPC, FV, true>(c2v, P, Rec(rec + j * CS, CS), live);
        } else {
          cn_update<D, EXACT, FPC, FV, false>(c2v, P, cur, live);
          for (int j = j0 + jstep; j < cn; j += jstep)
            cn_update<D, EXACT, FPC, FV, false>(c2v, P, Rec(rec + j * CS, CS), live);
        }
      }
#ifndef LDPCB_EXP_NOSYNC1
      __syncthreads();
#endif
      PT_MARK(pt_b);
      pin(fix_first);
      // VNs shared by two or more CNs of the group: exact re-sum (a stopped
      // frame re-sums to the value it already holds)
#ifdef LDPCB_EXP_NOFIX  // timing experiment only: wrong results
      if (false) {
#else
      if (xn > 0) {
#endif
        if (live && j0 < xn) {
          if (vs16) {
            const int4* rec = fix16 + static_cast<size_t>(x0) * vs16;
            vn_sum16<FPC, FV>(c2v, P, L, rec + j0 * vs16, vs16, fix_first, S - 1);
            vn_sum16_range<FPC, FV>(c2v, P, L, rec, vs16, j0 + jstep, xn, jstep, S - 1);
          } else {
            const int4* rec = fix_vn + static_cast<size_t>(x0) * vs4;
            vn_sum<FPC, FV, VS>(c2v, P, L, rec + j0 * vs4, vs4, fix_first, S - 1);
            vn_sum_range<FPC, FV, VS>(c2v, P, L, rec, vs4, j0 + jstep, xn, jstep, S - 1);
          }
        }
        __syncthreads();
      }
      pin_rec(next_cn);
      go = ngo;
#ifdef LDPCB_PHASE_TIMING
      const long long pt_c = clock64();
      pt_cn += pt_b - pt_a;
      pt_fix += pt_c - pt_b;
      ++pt_groups;
#endif
    }
    if (dump) continue;
    PT_MARK(pt_d);
    const bool check = a.early_stop || a.trace || iter == a.max_iters;
    // ---- exact totals (decoder.hpp:162-165): removes the rounding of the
    // in-place posterior updates before hard decisions are taken
    if (!RND && g.recompute && (check || !a.lazy_totals)) {
      if (live) {
        if (vs16)
          vn_sum16_range<FPC, FV>(c2v, P, L, tot16, vs16, j0, n, jstep, S - 1);
        else
          vn_sum_range<FPC, FV, VS>(c2v, P, L, tot_vn, vs4, j0, n, jstep, S - 1);
      }
      __syncthreads();
    }
    if (!check) continue;
    // ---- hard decision + syndrome weight (decoder.hpp:166-171)
    if (live) {
      int w[FV] = {};
      for (int j = j0; j < m; j += jstep) {
        const unsigned p = parity<D, EXACT, FPC, FV>(P, g.all_rec + j * CS, CS);
#pragma unroll
        for (int i = 0; i < FV; ++i) w[i] += (p >> i) & 1u;
      }
#pragma unroll
      for (int i = 0; i < FV; ++i)
        if (w[i]) atomicAdd(&s_weight[fb + i], w[i]);
    }
    __syncthreads();
    if (tid == 0) {
      int active = 0;
      for (int ff = 0; ff < nf; ++ff) {
        if (s_done[ff]) continue;
        const int w = s_weight[ff];
        if (a.trace) a.trace[(f0 + ff) * a.max_iters + iter - 1] = w;
        s_iters[ff] = iter;
        s_conv[ff] = w == 0;
        s_weight[ff] = 0;
        if (w == 0 && a.early_stop)
          s_done[ff] = 1;  // decoder.hpp:173-177
        else
          ++active;
      }
      s_active = active;
    }
    __syncthreads();
#ifdef LDPCB_PHASE_TIMING
    pt_end += clock64() - pt_d;
#endif
    live = live_bits(fb);
    if (s_active == 0) break;
  }
#ifdef LDPCB_PHASE_TIMING
  if (tid == 0) {
    atomicAdd(&g_phase_cycles[0], pt_cn);
    atomicAdd(&g_phase_cycles[1], pt_fix);
    atomicAdd(&g_phase_cycles[2], pt_end);
    atomicAdd(&g_phase_cycles[3], static_cast<unsigned long long>(clock64() - pt_start));
    atomicAdd(&g_phase_cycles[4], pt_groups);
    atomicAdd(&g_phase_cycles[5], 1ull);
    atomicAdd(&g_phase_cycles[6], static_cast<unsigned long long>(pt_start - pt_entry));
  }
  pt_loop_end = clock64();
#endif
finish:
  __syncthreads();
  if (dump) {
    if (!RND && g.recompute) vn_sum_range<FPC, FV, VS>(c2v, P, L, tot_vn, vs4, j0, n, jstep, S - 1);
    __syncthreads();
    const int E = g.E;
#pragma unroll
    for (int i = 0; i < FV; ++i) {
      if (fb + i >= nf) continue;
      for (int e = j0; e < E; e += jstep) {
        const float c = c2v[__ldg(g.edge_slot + e) * FPC + i];
        if (a.c2v_out) a.c2v_out[(f0 + fb + i) * E + e] = c * kLn2;
        if (a.v2c_out)
          a.v2c_out[(f0 + fb + i) * E + e] = clamp_bits(P[__ldg(g.vn_pos + __ldg(g.cols + e)) * FPC + i] - c) * kLn2;
      }
    }
    return;
  }
  // ---- epilogue: hard decisions (tie -> 0, decoder.hpp:166), error counts
#pragma unroll
  for (int i = 0; i < FV; ++i) {
    const int f = fb + i;
    if (f >= nf) continue;
    int errs = 0;
    if (a.bits && a.bits_packed) {
      const int nb = (n + 7) >> 3;
      uint8_t* out = a.bits + (f0 + f) * nb;
      for (int b = j0; b < nb; b += jstep) {
        unsigned byte = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int v = b * 8 + j;
          if (v < n && P[__ldg(g.vn_pos + v) * FPC + i] < 0.f) byte |= 1u << j;
        }
        out[b] = static_cast<uint8_t>(byte);
        errs += __popc(byte);
      }
    } else if (a.bits || a.counters || a.bit_errors) {
      for (int v = j0; v < n; v += jstep) {
        const int bit = P[__ldg(g.vn_pos + v) * FPC + i] < 0.f;
        if (a.bits) a.bits[(f0 + f) * n + v] = static_cast<uint8_t>(bit);
        errs += bit;
      }
    }
    if (errs) atomicAdd(&s_berr[f], errs);
    if (a.posterior)
      for (int v = j0; v < n; v += jstep) a.posterior[(f0 + f) * n + v] = P[__ldg(g.vn_pos + v) * FPC + i] * kLn2;
  }
  if (tid < nf) {
    const int it = a.early_stop ? s_iters[tid] : a.max_iters;
    if (a.iterations) a.iterations[f0 + tid] = it;
    if (a.converged) a.converged[f0 + tid] = static_cast<uint8_t>(s_conv[tid]);
  }
  __syncthreads();
  if (a.bit_errors && tid < nf) a.bit_errors[f0 + tid] = s_berr[tid];
  if (tid == 0 && a.counters) {
    unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
    for (int ff = 0; ff < nf; ++ff) {
      const int it = a.early_stop ? s_iters[ff] : a.max_iters;
      c[0] += 1;
      c[1] += s_berr[ff];
      c[2] += s_berr[ff] > 0;
      c[3] += s_conv[ff];
      c[4] += it;
      c[5] += s_conv[ff] ? it : 0;
    }
    for (int i = 0; i < 6; ++i) atomicAdd(a.counters + i, c[i]);
  }
#ifdef LDPCB_PHASE_TIMING
  if (tid == 0 && !dump) atomicAdd(&g_phase_cycles[7], static_cast<unsigned long long>(clock64() - pt_loop_end));
#endif
}

// ---- early-stop decoding from a frame queue (persistent CTAs)
// With early stop a CTA of the kernel above runs until its slowest frame
// stops, and every CTA pays its own prologue. Here a persistent CTA keeps FPC
// frame slots busy: at an iteration boundary (where every frame is at group
// 0 of the same cyclic schedule) a slot whose frame stopped writes that
// frame's outputs and takes the next frame id from a global counter. Each
// frame's arithmetic is the same as in decode_resident (slots are
// independent lanes), so outputs are bit-identical; frames finish in any
// order.
// RND: per-frame groupings, each slot staging its own frame's list for the
// slot's own iteration (lists indexed by the frame's id, as in decode_resident).
template <int D, bool EXACT, int FPC, int FV, int VS, bool RND = false>
__global__ void __launch_bounds__(max_threads_for(D, FV), D <= 16 ? 2 : 1) decode_queue(const DevGraph g,
                                                                                       const DecodeArgs a,
                                                                                       unsigned long long* queue) {
  static_assert(!RND || FV == 1, "per-frame groupings need one frame per thread");
  const int CS = g.cs;
  constexpr int NG = FPC / FV;
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_active, s_retiring;
  __shared__ long long s_frame[FPC];
  __shared__ unsigned long long s_cnt[6];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = g.n, m = g.m, S = g.n_slots;
  const int vs4 = VS > 0 ? VS : g.vs4;
  const int fg = tid % NG, j0 = tid / NG, jstep = nt / NG;
  const int fb = fg * FV;
  float* const c2v = smem + fb;
  float* const P = smem + S * FPC + fb;
  float* const L = P + n * FPC;
  float* const P0 = smem + S * FPC;  // slot-indexed views
  float* const L0 = P0 + n * FPC;
  int* const s_done = reinterpret_cast<int*>(smem + (S + 2 * n) * FPC);
  int* const s_weight = s_done + FPC;
  int* const s_iters = s_weight + FPC;
  int* const s_conv = s_iters + FPC;
  int* const s_berr = s_conv + FPC;
  int4* const s_go = reinterpret_cast<int4*>(smem + (((S + 2 * n) * FPC + 5 * FPC + 3) & ~3));
  uint16_t* const s_list = reinterpret_cast<uint16_t*>(s_go + g.G);  // RND: [FPC][slots]
  const int slots = a.list_slots;
  const int4* const tot_vn = reinterpret_cast<const int4*>(g.tot_vn_rec);
  const int4* const fix_vn = reinterpret_cast<const int4*>(g.fix_rec);
  const int4* const fix16 = reinterpret_cast<const int4*>(g.fix_rec16);
  const int vs16 = VS > 0 ? 0 : g.vs16;  // 16-bit fix-up records (multi-row VN records only)
  const int4* const tot16 = reinterpret_cast<const int4*>(g.tot_rec16);
  const int nb = (n + 7) >> 3;

  // init_state (decoder.hpp:39-52) of slot ff for frame f (f < 0: idle slot)
  auto load_slot = [&](int ff, long long f) {
    if (f >= 0) {
      const float* llr = a.llr + f * n;
      if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(a.llr) & 15) == 0) {
        const float4* l4 = reinterpret_cast<const float4*>(llr);
        for (int b = tid; b < n / 4; b += nt) {
          const float4 x = ldg_stream(l4 + b);
          const float r[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int v = __ldg(g.vn_pos + 4 * b + u);
            const float y = clamp_llr(r[u]) * kLog2e;
            P0[v * FPC + ff] = y;
            L0[v * FPC + ff] = y;
          }
        }
      } else {
        for (int i = tid; i < n; i += nt) {
          const int v = __ldg(g.vn_pos + i);
          const float y = clamp_llr(__ldg(llr + i)) * kLog2e;
          P0[v * FPC + ff] = y;
          L0[v * FPC + ff] = y;
        }
      }
      if (a.trace)
        for (int i = tid; i < a.max_iters; i += nt) a.trace[f * a.max_iters + i] = -1;
    } else {
      for (int i = tid; i < n; i += nt) P0[i * FPC + ff] = L0[i * FPC + ff] = kClampB;
    }
    for (int i = tid; i < S; i += nt) smem[i * FPC + ff] = 0.f;
  };
  auto pull = [&]() -> long long {
    const unsigned long long f = atomicAdd(queue, 1ull);
    return f < static_cast<unsigned long long>(a.frames) ? static_cast<long long>(f) : -1ll;
  };

  if (tid < FPC) {
    s_frame[tid] = pull();
    s_done[tid] = s_frame[tid] < 0;
    s_weight[tid] = s_iters[tid] = s_conv[tid] = s_berr[tid] = 0;
  }
  if (tid < 6) s_cnt[tid] = 0ull;
  for (int i = tid; i < g.G; i += nt)
    s_go[i] = make_int4(__ldg(g.cn_off + i), __ldg(g.cn_off + i + 1), __ldg(g.fix_off + i), __ldg(g.fix_off + i + 1));
  __syncthreads();
  for (int ff = 0; ff < FPC; ++ff) load_slot(ff, s_frame[ff]);
  __syncthreads();
  auto live_bits = [&]() {
    unsigned b = 0;
#pragma unroll
    for (int i = 0; i < FV; ++i) b |= static_cast<unsigned>(!s_done[fb + i]) << i;
    return b;
  };
  unsigned live = live_bits();
  using Rec = ResidentRecord<D, EXACT>;
  Rec next_cn;
  if (!RND && j0 < s_go[0].y - s_go[0].x) next_cn.load(g.cn_rec + static_cast<size_t>(s_go[0].x + j0) * CS, CS);
  int4 go = s_go[0];

  for (;;) {
    if constexpr (RND) {
      // each busy slot's groups for its own next iteration (decoder.hpp:153-156)
      for (int i = tid; i < FPC * slots; i += nt) {
        const int ff = i / slots;
        if (s_done[ff]) {  // idle slot: CN 0 keeps its (unused) record loads in bounds
          s_list[i] = 0;
          continue;
        }
        const int li = a.n_lists > 1 ? s_iters[ff] : 0;
        s_list[i] = a.lists[(s_frame[ff] * a.n_lists + li) * slots + (i - ff * slots)];
      }
      __syncthreads();
    }
    // one iteration for every busy slot (decoder.hpp:157-160), as in decode_resident
    for (int grp = 0; grp < g.G; ++grp) {
      if constexpr (RND) {
        rnd_group<D, EXACT, FPC, FV, VS>(g, CS, vs4, c2v, P, L, s_go, s_list + fb * slots, grp, j0, jstep, live,
                                         next_cn);
        continue;
      }
      const int c0 = go.x, cn = go.y - go.x;
      const int x0 = go.z, xn = go.w - go.z;
      const int4 ngo = s_go[grp + 1 < g.G ? grp + 1 : 0];
      int4 fix_first = make_int4(0, 0, 0, 0);
      if (j0 < xn)
        fix_first = vs16 ? __ldg(fix16 + static_cast<size_t>(x0 + j0) * vs16)
                         : __ldg(fix_vn + static_cast<size_t>(x0 + j0) * vs4);
      const Rec cur = next_cn;
      if (j0 < ngo.y - ngo.x) next_cn.load(g.cn_rec + static_cast<size_t>(ngo.x + j0) * CS, CS);
      if (live && j0 < cn) {
        const int32_t* rec = g.cn_rec + static_cast<size_t>(c0) * CS;
        if (live == (1u << FV) - 1) {
          cn_update<D, EXACT, FPC, FV, true>(c2v, P, cur, live);
          for (int j = j0 + jstep; j < cn; j += jstep)
            cn_update<D, EXACT, FPC, FV, true>(c2v, P, Rec(rec + j * CS, CS), live);
        } else {
          cn_update<D, EXACT, FPC, FV, false>(c2v, P, cur, live);
          for (int j = j0 + jstep; j < cn; j += jstep)
            cn_update<D, EXACT, FPC, FV, false>(c2v, P, Rec(rec + j * CS, CS), live);
        }
      }
      __syncthreads();
      pin(fix_first);
      if (xn > 0) {
        if (live && j0 < xn) {
          if (vs16) {
            const int4* rec = fix16 + static_cast<size_t>(x0) * vs16;
            vn_sum16<FPC, FV>(c2v, P, L, rec + j0 * vs16, vs16, fix_first, S - 1);
            vn_sum16_range<FPC, FV>(c2v, P, L, rec, vs16, j0 + jstep, xn, jstep, S - 1);
          } else {
            const int4* rec = fix_vn + static_cast<size_t>(x0) * vs4;
            vn_sum<FPC, FV, VS>(c2v, P, L, rec + j0 * vs4, vs4, fix_first, S - 1);
            vn_sum_range<FPC, FV, VS>(c2v, P, L, rec, vs4, j0 + jstep, xn, jstep, S - 1);
          }
        }
        __syncthreads();
      }
      pin_rec(next_cn);
      go = ngo;
    }
    // exact totals, hard decisions, syndrome weights (decoder.hpp:162-171)
    if (!RND && g.recompute) {
      if (live) {
        if (vs16)
          vn_sum16_range<FPC, FV>(c2v, P, L, tot16, vs16, j0, n, jstep, S - 1);
        else
          vn_sum_range<FPC, FV, VS>(c2v, P, L, tot_vn, vs4, j0, n, jstep, S - 1);
      }
      __syncthreads();
    }
    if (live) {
      int w[FV] = {};
      for (int j = j0; j < m; j += jstep) {
        const unsigned p = parity<D, EXACT, FPC, FV>(P, g.all_rec + j * CS, CS);
#pragma unroll
        for (int i = 0; i < FV; ++i) w[i] += (p >> i) & 1u;
      }
#pragma unroll
      for (int i = 0; i < FV; ++i)
        if (w[i]) atomicAdd(&s_weight[fb + i], w[i]);
    }
    __syncthreads();
    if (tid == 0) {
      int retiring = 0;
      for (int ff = 0; ff < FPC; ++ff) {
        if (s_done[ff]) continue;
        const int w = s_weight[ff], it = ++s_iters[ff];
        s_weight[ff] = 0;
        if (a.trace) a.trace[s_frame[ff] * a.max_iters + it - 1] = w;
        s_conv[ff] = w == 0;
        if ((w == 0 && a.early_stop) || it == a.max_iters) {  // decoder.hpp:173-177
          s_done[ff] = 2;                                       // retiring
          ++retiring;
        }
      }
      s_retiring = retiring;
    }
    __syncthreads();
    if (s_retiring == 0) continue;
    // outputs of the frames that stopped (sim.hpp:119-123), then refill
    for (int ff = 0; ff < FPC; ++ff) {
      if (s_done[ff] != 2) continue;
      const long long f = s_frame[ff];
      int errs = 0;
      if (a.bits && a.bits_packed) {
        for (int b = tid; b < nb; b += nt) {
          unsigned byte = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int v = b * 8 + j;
            if (v < n && P0[__ldg(g.vn_pos + v) * FPC + ff] < 0.f) byte |= 1u << j;
          }
          a.bits[f * nb + b] = static_cast<uint8_t>(byte);
          errs += __popc(byte);
        }
      } else if (a.bits || a.counters || a.bit_errors) {
        for (int v = tid; v < n; v += nt) {
          const int bit = P0[__ldg(g.vn_pos + v) * FPC + ff] < 0.f;
          if (a.bits) a.bits[f * n + v] = static_cast<uint8_t>(bit);
          errs += bit;
        }
      }
      if (errs) atomicAdd(&s_berr[ff], errs);
      if (a.posterior)
        for (int v = tid; v < n; v += nt) a.posterior[f * n + v] = P0[__ldg(g.vn_pos + v) * FPC + ff] * kLn2;
    }
    __syncthreads();
    if (tid == 0) {
      for (int ff = 0; ff < FPC; ++ff) {
        if (s_done[ff] != 2) continue;
        const long long f = s_frame[ff];
        const int it = s_iters[ff];
        if (a.iterations) a.iterations[f] = it;
        if (a.converged) a.converged[f] = static_cast<uint8_t>(s_conv[ff]);
        if (a.bit_errors) a.bit_errors[f] = s_berr[ff];
        s_cnt[0] += 1;
        s_cnt[1] += s_berr[ff];
        s_cnt[2] += s_berr[ff] > 0;
        s_cnt[3] += s_conv[ff];
        s_cnt[4] += it;
        s_cnt[5] += s_conv[ff] ? it : 0;
        s_frame[ff] = pull();
        s_done[ff] = s_frame[ff] < 0 ? 1 : 3;  // 3: refilled this round
        s_iters[ff] = s_conv[ff] = s_berr[ff] = 0;
      }
      int active = 0;
      for (int ff = 0; ff < FPC; ++ff) active += s_done[ff] != 1;
      s_active = active;
    }
    __syncthreads();
    for (int ff = 0; ff < FPC; ++ff)
      if (s_done[ff] == 3) load_slot(ff, s_frame[ff]);
    __syncthreads();
    if (tid < FPC && s_done[tid] == 3) s_done[tid] = 0;
    __syncthreads();
    live = live_bits();
    if (s_active == 0) break;
  }
  if (tid == 0 && a.counters)
    for (int i = 0; i < 6; ++i)
      if (s_cnt[i]) atomicAdd(a.counters + i, s_cnt[i]);
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

// Segment-parallel channel for long frames: thread (frame, segment s)
// starts its frame's stream advanced by s * L draws (polys[s - 1] = x^(s L)
// mod p, host_rng.cpp) and produces normals [s L, s L + L). L is even, so a
// segment starts on a Box-Muller pair and each normal pairs the same two
// draws as the sequential stream (cos first, sin cached): identical LLRs.
__global__ void channel_seg_kernel(int n, int L, int S, double sigma, double scale, uint64_t seed, int64_t frame0,
                                   int64_t frames, const uint64_t* __restrict__ polys, float* __restrict__ llr) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= frames * S) return;
  const int64_t f = t / S;
  const int s = static_cast<int>(t - f * S);
  Stream rng(stream_seed(seed, static_cast<uint64_t>(frame0 + f)));
  if (s > 0) {  // jump(): xor of the states at the set coefficients
    const uint64_t* poly = polys + 4 * (s - 1);
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int w = 0; w < 4; ++w) {
      const uint64_t word = __ldg(poly + w);
      for (int b = 0; b < 64; ++b) {
        if ((word >> b) & 1u) {
          a0 ^= rng.w0;
          a1 ^= rng.w1;
          a2 ^= rng.w2;
          a3 ^= rng.w3;
        }
        rng.u64();
      }
    }
    rng.w0 = a0;
    rng.w1 = a1;
    rng.w2 = a2;
    rng.w3 = a3;
  }
  const int i0 = s * L, i1 = min(n, i0 + L);
  float* out = llr + f * n;
  for (int i = i0; i < i1; i += 2) {  // Stream::normal(), both halves of a pair
    const double a = rng.unit();
    const double b = rng.unit();
    const double r = sqrt(-2.0 * log(a));
    const double th = 6.283185307179586476925286766559 * b;
    out[i] = static_cast<float>(scale * (1.0 + sigma * (r * cos(th))));
    if (i + 1 < i1) out[i + 1] = static_cast<float>(scale * (1.0 + sigma * (r * sin(th))));
  }
}

// ---- one CN per thread on explicit inputs (check_update KATs)
template <int D, bool EXACT>
__global__ void check_update_kernel(int deg, int64_t rows, const float* __restrict__ v2c, float* __restrict__ c2v) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = (EXACT || k < deg) ? v2c[r * deg + k] * kLog2e : 0.f;
  boxplus_row<D, EXACT>(x, deg, [&](int k, float c) { c2v[r * deg + k] = c * kLn2; });
}

// generate_groups (schedule.hpp:54-115) for (frame, list) pairs on the device:
// list l of frame f uses Rng(mix_seed(mix_seed(schedule_seed, f), list0+l+1)),
// the stream run_sweep / decode draw from (sim.hpp:113-117, decoder.hpp:153-156).
// One thread per list. The pool and the candidate copy live in shared
// memory (uint16); the candidates of group g are exactly the fresh part of
// group g-1 (a carried CN came from group g-2), so no membership array is
// needed. next_below's two 64-bit remainders use per-CTA reciprocals.
struct Below {
  const unsigned long long* recip;  // recip[n] = floor((2^64-1) / n)
  // x mod n for n < 2^16: the Barrett quotient is low by at most 2, so the
  // remainder is < 3n < 2^32 and only the low words of x - q n are needed
  __device__ __forceinline__ uint32_t mod(uint64_t x, uint32_t n) const {
    uint32_t r = static_cast<uint32_t>(x) - static_cast<uint32_t>(__umul64hi(x, recip[n])) * n;
    r = r >= n ? r - n : r;
    return r >= n ? r - n : r;
  }
  // Stream::below (rng.hpp:67-73): rejection below lim = (2^64 - n) mod n,
  // which is < n <= 65535, so it is only computed for such tiny draws
  __device__ __forceinline__ uint32_t draw(Stream& rng, uint32_t n) const {
    for (;;) {
      const uint64_t x = rng.u64();
      if (x > 0xffffull) return mod(x, n);
      if (x >= mod(0ull - n, n)) return mod(x, n);
    }
  }
  __device__ __forceinline__ void permute(Stream& rng, uint16_t* a, int n) const {  // rng.hpp:75-82
    for (int i = n; i > 1; --i) {
      const uint32_t j = draw(rng, static_cast<uint32_t>(i));
      const uint16_t t = a[i - 1];
      a[i - 1] = a[j];
      a[j] = t;
    }
  }
};

__global__ void gen_groups_kernel(int M, int G, int balanced, int nominal, int k, uint64_t schedule_seed,
                                  int64_t frame0, int64_t frames, int list0, int n_lists, int slots,
                                  uint16_t* __restrict__ out) {
  extern __shared__ unsigned long long gsm64[];
  unsigned long long* recip = gsm64;  // [M + 1]
  for (int i = threadIdx.x; i <= M; i += blockDim.x) recip[i] = i > 1 ? ~0ull / static_cast<unsigned>(i) : 0ull;
  const int per = M | 1;  // uint16 per thread (odd: spread banks)
  uint16_t* pool = reinterpret_cast<uint16_t*>(gsm64 + M + 1) + threadIdx.x * per;
  __syncthreads();
  const Below bl{recip};
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= frames * n_lists) return;
  const int64_t f = item / n_lists;
  const int l = static_cast<int>(item - f * n_lists);
  uint16_t* o = out + item * slots;
  Stream rng(stream_seed(stream_seed(schedule_seed, static_cast<uint64_t>(frame0 + f)),
                         static_cast<uint64_t>(list0 + l + 1)));
  for (int i = 0; i < M; ++i) pool[i] = static_cast<uint16_t>(i);
  bl.permute(rng, pool, M);
  if (balanced) {  // disjoint: consecutive slices of the shuffled pool
    for (int i = 0; i < M; ++i) o[i] = pool[i];
    return;
  }
  int next = min(nominal, M), w = next;
  for (int i = 0; i < next; ++i) o[i] = pool[i];
  int fresh_start = 0, fresh_len = next;  // fresh part of the previous group
  for (int grp = 1; grp < G; ++grp) {
    // the candidates are permuted in place: that pool range is never read again
    uint16_t* cand = pool + fresh_start;
    bl.permute(rng, cand, fresh_len);
    const int take = min(k, fresh_len);
    for (int i = 0; i < take; ++i) o[w++] = cand[i];
    const int want = grp == G - 1 ? M - next : nominal - take;
    const int got = min(want, M - next);
    for (int i = 0; i < got; ++i) o[w++] = pool[next + i];
    fresh_start = next;
    fresh_len = got;
    next += got;
  }
}

using KernelFn = void (*)(const DevGraph, const DecodeArgs);

template <int D, bool EXACT, int VS>
KernelFn pick_fpc(int fpc, int fv) {
  if constexpr (D <= 8) {
    if (fv == 2) switch (fpc) {
      case 2: return decode_resident<D, EXACT, 2, 2, VS>;
      case 4: return decode_resident<D, EXACT, 4, 2, VS>;
      case 8: return decode_resident<D, EXACT, 8, 2, VS>;
      default: return nullptr;
    }
  }
  if (fv != 1) return nullptr;
  switch (fpc) {
    case 1: return decode_resident<D, EXACT, 1, 1, VS>;
    case 2: return decode_resident<D, EXACT, 2, 1, VS>;
    case 4: return decode_resident<D, EXACT, 4, 1, VS>;
    case 8: return decode_resident<D, EXACT, 8, 1, VS>;
    case 16: return decode_resident<D, EXACT, 16, 1, VS>;
    default: return nullptr;
  }
}

using QueueFn = void (*)(const DevGraph, const DecodeArgs, unsigned long long*);

// frame-queue kernels for the early-stop plans (frames per CTA <= 2)
template <int D, bool EXACT, int VS>
QueueFn pick_queue_fpc(int fpc, int fv) {
  if constexpr (D <= 8) {
    if (fv == 2) return fpc == 2 ? decode_queue<D, EXACT, 2, 2, VS> : nullptr;
  }
  if (fv != 1) return nullptr;
  switch (fpc) {
    case 1: return decode_queue<D, EXACT, 1, 1, VS>;
    case 2: return decode_queue<D, EXACT, 2, 1, VS>;
    default: return nullptr;
  }
}

template <int D, bool EXACT, int VS>
QueueFn pick_queue_rnd(int fpc) {
  switch (fpc) {
    case 1: return decode_queue<D, EXACT, 1, 1, VS, true>;
    case 2: return decode_queue<D, EXACT, 2, 1, VS, true>;
    default: return nullptr;
  }
}

QueueFn pick_queue(const DevGraph& g, int fpc, int fv) {
  if (g.per_frame) {
    if (fv != 1) return nullptr;
    switch (cn_bucket(g.max_cdeg, g.cregular)) {
      case 6: return g.vs4 == 1 ? pick_queue_rnd<6, true, 1>(fpc) : pick_queue_rnd<6, true, 0>(fpc);
      case 3: return pick_queue_rnd<3, true, 0>(fpc);
      case 8: return pick_queue_rnd<8, false, 0>(fpc);
      case 16: return pick_queue_rnd<16, false, 0>(fpc);
      default: return nullptr;
    }
  }
  switch (cn_bucket(g.max_cdeg, g.cregular)) {
    case 6: return g.vs4 == 1 ? pick_queue_fpc<6, true, 1>(fpc, fv) : pick_queue_fpc<6, true, 0>(fpc, fv);
    case 3: return pick_queue_fpc<3, true, 0>(fpc, fv);
    case 8: return pick_queue_fpc<8, false, 0>(fpc, fv);
    case 16: return pick_queue_fpc<16, false, 0>(fpc, fv);
    case 32: return pick_queue_fpc<32, false, 0>(fpc, fv);
    default: return nullptr;
  }
}

template <int D, bool EXACT, int VS>
KernelFn pick_rnd(int fpc) {
  switch (fpc) {
    case 1: return decode_resident<D, EXACT, 1, 1, VS, true>;
    case 2: return decode_resident<D, EXACT, 2, 1, VS, true>;
    case 4: return decode_resident<D, EXACT, 4, 1, VS, true>;
    default: return nullptr;
  }
}

KernelFn pick_kernel(const DevGraph& g, int fpc, int fv, int* bucket) {
  *bucket = cn_bucket(g.max_cdeg, g.cregular);
  if (g.per_frame) {
    if (fv != 1) return nullptr;
    switch (*bucket) {
      case 6: return g.vs4 == 1 ? pick_rnd<6, true, 1>(fpc) : pick_rnd<6, true, 0>(fpc);
      case 3: return pick_rnd<3, true, 0>(fpc);
      case 8: return pick_rnd<8, false, 0>(fpc);
      case 16: return pick_rnd<16, false, 0>(fpc);
      default: return nullptr;
    }
  }
  switch (*bucket) {
    case 6: return g.vs4 == 1 ? pick_fpc<6, true, 1>(fpc, fv) : pick_fpc<6, true, 0>(fpc, fv);
    case 3: return pick_fpc<3, true, 0>(fpc, fv);
    case 8: return pick_fpc<8, false, 0>(fpc, fv);
    case 16: return pick_fpc<16, false, 0>(fpc, fv);
    case 32: return pick_fpc<32, false, 0>(fpc, fv);
    default: return nullptr;
  }
}

size_t frame_bytes(const DevGraph& g) { return 4ull * (static_cast<size_t>(g.n_slots) + 2ull * g.n); }

int device_smem_per_sm() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess) v = 228 * 1024;
  return v;
}

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
void set_frames_per_thread(int fv) { g_tune_fv = fv; }

int64_t kernel_launch_count() { return g_launches.load(); }
void note_launches(int n) { g_launches += n; }
void set_force_kernel(int kernel) { g_force_kernel = kernel; }

void set_lazy_totals(int on) { g_lazy_totals = on; }

// early-stop decodes from a frame queue (decode_queue) when the batch holds
// at least four waves of CTAs; LDPCB_FRAME_QUEUE=0 never, =2 for any batch
// (A/B and tests)
static int frame_queue_mode() {
  const char* e = std::getenv("LDPCB_FRAME_QUEUE");
  return e ? std::atoi(e) : 1;
}
int lazy_totals() { return g_lazy_totals.load(); }

Plan plan_resident(const DevGraph& g, int64_t frames, bool early_stop);

int launch_gen_groups(const DevGraph& g, int64_t frame0, int64_t frames, int list0, int n_lists, uint16_t* out,
                      void* stream) {
  if (!g.per_frame) return static_cast<int>(cudaErrorInvalidValue);
  if (frames <= 0 || n_lists <= 0) return 0;
  const int per = 2 * (g.m | 1);    // scratch bytes per thread (the pool)
  const int fixed = 8 * (g.m + 1);  // reciprocal table
  const int room = device_smem_optin() - 1024 - fixed;
  if (per > room) return static_cast<int>(cudaErrorInvalidConfiguration);
  // one list per thread: the most lists resident per SM (each is a
  // latency-bound sequential shuffle), the larger CTA on ties
  int tpb = 1, best = 0;
  for (int t : {32, 64, 96, 128, 192, 256}) {
    if (t * per > room) break;
    const int lists = t * (device_smem_per_sm() / (fixed + t * per + 1024));
    if (lists >= best) best = lists, tpb = t;
  }
  if (best == 0) tpb = std::max(1, std::min(128, room / per));
  if (const char* e = std::getenv("LDPCB_GEN_TPB")) tpb = std::max(1, std::min(room / per, std::atoi(e)));
  const int bytes = fixed + tpb * per;
  cudaError_t err = cudaFuncSetAttribute(reinterpret_cast<const void*>(gen_groups_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err != cudaSuccess) return static_cast<int>(err);
  const int64_t items = frames * n_lists;
  gen_groups_kernel<<<static_cast<unsigned>((items + tpb - 1) / tpb), tpb, bytes,
                      static_cast<cudaStream_t>(stream)>>>(g.m, g.G, g.balanced, g.nominal, g.k_overlap,
                                                           g.schedule_seed, frame0, frames, list0, n_lists,
                                                           g.list_slots, out);
  ++g_launches;
  return static_cast<int>(cudaGetLastError());
}

Plan plan_decode(const DevGraph& g, int64_t frames, bool early_stop) {
  if (g.per_frame) return plan_resident(g, frames, early_stop);  // per-frame groups: resident kernel only
  // the posterior-free kernel (direct.cu) wherever its tables exist and no
  // explicit resident tuning was requested; kernel 3 forces it
  const int force = g_force_kernel.load();
  if (force == 3 ||
      (force == 0 && g.d_fv > 0 && g_tune_fpc.load() == 0 && g_tune_threads.load() == 0 && g_tune_fv.load() == 0)) {
    const Plan d = plan_direct(g, frames);
    if (d.kernel == 3 || force == 3) return d;
  }
  if (g_force_kernel.load() == 2) return plan_stream(g, frames);
  Plan p = plan_resident(g, frames, early_stop);
  if (p.kernel == 0 && g_force_kernel.load() != 1) p = plan_stream(g, frames);
  return p;
}

// Registers per thread of a kernel instantiation (cached per function).
int kernel_regs(KernelFn fn) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(reinterpret_cast<const void*>(fn));
  if (it != cache.end()) return it->second;
  cudaFuncAttributes at{};
  const int r = cudaFuncGetAttributes(&at, reinterpret_cast<const void*>(fn)) == cudaSuccess ? at.numRegs : 128;
  cache[reinterpret_cast<const void*>(fn)] = r;
  return r;
}

Plan plan_resident(const DevGraph& g, int64_t frames, bool early_stop) {
  Plan p;
  const size_t limit = static_cast<size_t>(device_smem_optin()) - 1024;
  const size_t per = frame_bytes(g);
  const size_t list_bytes = g.per_frame ? 2ull * g.list_slots : 0;  // per frame
  auto bytes = [&](int f) { return f * (per + list_bytes) + 20 * f + 16 * g.G + 32; };
  const int bucket0 = cn_bucket(g.max_cdeg, g.cregular);
  auto fv_for = [&](int fpc) {
    const int fv = g_tune_fv.load();
    if (fv > 0) return fv;
    return (fpc >= 2 && fpc % 2 == 0 && bucket0 <= 8 && !g.per_frame) ? 2 : 1;
  };
  auto max_threads = [&](int fv) { return max_threads_for(bucket0 <= 8 ? 8 : (bucket0 <= 16 ? 16 : 32), fv); };
  // one CN item per frame vector for the largest group, in whole warps where
  // that stays a multiple of the frame vectors per CTA
  auto threads_for = [&](int fpc, int fv) {
    const int ng = fpc / fv;
    int nt = (ng * g.max_cn_items + 31) / 32 * 32;
    nt = std::max(64, std::min(nt, max_threads(fv)));
    return nt / ng * ng;
  };
  int fpc = g_tune_fpc.load();
  if (fpc <= 0) {
    // the candidate with the most useful CN lanes per SM: resident CTAs
    // (shared memory and registers) x frames per CTA x the fraction of the
    // CTA's threads that hold a CN item of the largest group
    const size_t sm_bytes = static_cast<size_t>(device_smem_per_sm());
    double best = 0.0;
    for (int c : {1, 2, 4, 8, 16}) {
      if (bytes(c) > limit) continue;
      // with early stop a CTA runs until its slowest frame converges: more
      // than two frames per CTA idle their stopped lanes (measured slower)
      if (early_stop && c > 2) continue;
      if (g.per_frame && c > 4) continue;
      const int fv = fv_for(c);
      int bk = 0;
      const KernelFn fn = pick_kernel(g, c, fv, &bk);
      if (!fn) continue;
      const int nt = threads_for(c, fv);
      const int ng = c / fv;
      const int regs = (kernel_regs(fn) * 32 + 255) / 256 * 256;  // per warp, allocation granularity
      const int warps = (nt + 31) / 32;
      const int by_regs = 65536 / (regs * warps);
      const int by_smem = static_cast<int>(sm_bytes / (bytes(c) + 1024));
      const int ctas = std::min({by_regs, by_smem, 32});
      if (ctas <= 0) continue;
      const double util = std::min(1.0, static_cast<double>(ng) * g.max_cn_items / (32.0 * warps));
      const double score = ctas * c * util * (fv == 2 ? 2.0 : 1.0);  // two frames per instruction
      if (score > best * 1.0001) {
        best = score;
        fpc = c;
      }
    }
    if (fpc <= 0) fpc = 1;
    // per-frame groupings with early stop: two frames per CTA taken from the
    // frame queue beat one frame per CTA at more CTAs per SM (C1, G = 8,
    // r = 0.25, <= 20 it: 6.68e6 -> 7.38e6 frames/s; regrouping 3.02e6 -> 3.14e6)
    if (g.per_frame && early_stop && frame_queue_mode() > 0 && fpc == 1 && bytes(2) <= limit) fpc = 2;
  }
  if (bytes(fpc) > limit) return p;  // does not fit: no resident plan
  int bucket = 0;
  const int fv = fv_for(fpc);
  if (!pick_kernel(g, fpc, fv, &bucket)) return p;
  const int ng = fpc / fv;  // frame vectors per CTA
  int nt = g_tune_threads.load();
  if (nt <= 0) nt = threads_for(fpc, fv);
  if (nt % ng || nt > max_threads(fv)) return p;
  p.kernel = 1;
  p.fpc = fpc;
  p.fv = fv;
  p.threads = nt;
  p.smem = static_cast<int>(bytes(fpc));
  p.degree_bucket = bucket;
  p.ctas = (frames + fpc - 1) / fpc;
  return p;
}

int launch_decode(const DevGraph& g, const DecodeArgs& a_in, void* stream, Plan* used) {
  DecodeArgs a = a_in;
  a.lazy_totals = g_lazy_totals.load();
  const Plan p = plan_decode(g, a.frames, a.early_stop != 0);
  if (p.kernel == 2) return launch_stream(g, a, stream, used);
  if (p.kernel == 3) return launch_direct(g, a, stream, used);
  if (used) *used = p;
  if (p.kernel == 0) return static_cast<int>(cudaErrorInvalidConfiguration);
  if (a.frames <= 0) return 0;
  int bucket = 0;
  KernelFn fn = pick_kernel(g, p.fpc, p.fv, &bucket);
  cudaError_t err = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
  if (err != cudaSuccess) return static_cast<int>(err);
  auto st = static_cast<cudaStream_t>(stream);
  // early stop: persistent CTAs take frames from a queue (decode_queue) when
  // the batch (or a per-frame chunk) is at least four waves
  QueueFn qf = nullptr;
  int64_t resident = 0;  // CTAs resident on the device
  if (a.early_stop && a.max_subiters == 0 && frame_queue_mode() > 0) {
    qf = pick_queue(g, p.fpc, p.fv);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    if (!qf || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaFuncSetAttribute(reinterpret_cast<const void*>(qf), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             p.smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qf, p.threads, p.smem) != cudaSuccess || per_sm <= 0)
      qf = nullptr;
    resident = static_cast<int64_t>(sms) * per_sm;
  }
  auto use_queue = [&](int64_t ctas) { return qf && (ctas >= 4 * resident || frame_queue_mode() == 2); };
  auto launch_queue = [&](const DecodeArgs& b, int64_t ctas) {
    unsigned long long* queue = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&queue), sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    qf<<<static_cast<unsigned>(std::min(ctas, resident)), p.threads, p.smem, st>>>(g, b, queue);
    ++g_launches;
    e = cudaGetLastError();
    cudaFreeAsync(queue, st);
    return e;
  };
  if (!g.per_frame && use_queue(p.ctas)) return static_cast<int>(launch_queue(a, p.ctas));
  if (!g.per_frame) {
    // grid.x limit is 2^31-1, far above any batch
    fn<<<static_cast<unsigned>(p.ctas), p.threads, p.smem, st>>>(g, a);
    ++g_launches;
    return static_cast<int>(cudaGetLastError());
  }
  // per-frame (and per-iteration) groups, sim.hpp:113-117: generate the
  // lists for a chunk of frames (<= 512 MB of uint16 lists), then decode it
  a.n_lists = g.regroup ? a.max_iters : 1;
  a.list_slots = g.list_slots;
  const int64_t per_frame_bytes = 2ll * a.n_lists * g.list_slots;
  int64_t chunk = std::max<int64_t>(p.fpc, (512ll << 20) / per_frame_bytes / p.fpc * p.fpc);
  chunk = std::min(chunk, a.frames);
  uint16_t* lists = nullptr;
  err = cudaMallocAsync(reinterpret_cast<void**>(&lists), per_frame_bytes * chunk, st);
  if (err != cudaSuccess) return static_cast<int>(err);
  const int n = g.n, nb = (g.n + 7) / 8;
  for (int64_t c0 = 0; c0 < a.frames && err == cudaSuccess; c0 += chunk) {
    const int64_t cnt = std::min(chunk, a.frames - c0);
    DecodeArgs b = a;
    b.frames = cnt;
    b.frame0 = a.frame0 + c0;
    b.llr = a.llr + c0 * n;
    if (a.bits) b.bits = a.bits + c0 * (a.bits_packed ? nb : n);
    if (a.iterations) b.iterations = a.iterations + c0;
    if (a.converged) b.converged = a.converged + c0;
    if (a.bit_errors) b.bit_errors = a.bit_errors + c0;
    if (a.posterior) b.posterior = a.posterior + c0 * n;
    if (a.trace) b.trace = a.trace + c0 * a.max_iters;
    if (a.c2v_out) b.c2v_out = a.c2v_out + c0 * g.E;
    if (a.v2c_out) b.v2c_out = a.v2c_out + c0 * g.E;
    b.lists = lists;
    err = static_cast<cudaError_t>(launch_gen_groups(g, b.frame0, cnt, 0, a.n_lists, lists, st));
    if (err != cudaSuccess) break;
    const int64_t ctas = (cnt + p.fpc - 1) / p.fpc;
    if (use_queue(ctas)) {
      err = launch_queue(b, ctas);
      continue;
    }
    fn<<<static_cast<unsigned>(ctas), p.threads, p.smem, st>>>(g, b);
    ++g_launches;
    err = cudaGetLastError();
  }
  cudaFreeAsync(lists, st);
  return static_cast<int>(err);
}

#ifdef LDPCB_PHASE_TIMING
extern "C" int ldpcb_debug_phase_cycles(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  }
  return static_cast<int>(cudaDeviceSynchronize());
}
#endif

// Jump polynomials x^(s L) mod p for s = 1 .. S-1, uploaded once per
// (device, L, S) and kept for the process lifetime (a few KB each).
const uint64_t* channel_polys(int L, int S) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, uint64_t*> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, L, S);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<uint64_t> h(4ull * (S - 1));
  for (int s = 1; s < S; ++s) {
    const auto p = stream_jump_poly(static_cast<uint64_t>(s) * L);
    std::copy(p.begin(), p.end(), h.begin() + 4 * (s - 1));
  }
  uint64_t* d = nullptr;
  if (cudaMalloc(&d, h.size() * 8) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  cache[key] = d;
  return d;
}

int launch_channel(int n, double sigma2, uint64_t seed, int64_t frame0, int64_t frames, float* llr, void* stream) {
  if (frames <= 0) return 0;
  const double sigma = std::sqrt(sigma2);  // channel.hpp:41-42
  const double scale = 2.0 / sigma2;
  // Long frames in small batches: split each frame's stream into S segments
  // (jump-ahead) so that about 1024 threads per SM generate noise.
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t want = static_cast<int64_t>(sms) * 1024;
  int S = static_cast<int>(std::min<int64_t>((want + frames - 1) / frames, n / 256));
  if (S >= 2) {
    const int L = ((n + S - 1) / S + 1) & ~1;  // even segment length
    S = (n + L - 1) / L;
    const uint64_t* polys = channel_polys(L, S);
    if (!polys) return static_cast<int>(cudaErrorMemoryAllocation);
    const int tpb = 128;
    const int64_t blocks = (frames * S + tpb - 1) / tpb;
    channel_seg_kernel<<<static_cast<unsigned>(blocks), tpb, 0, static_cast<cudaStream_t>(stream)>>>(
        n, L, S, sigma, scale, seed, frame0, frames, polys, llr);
    ++g_launches;
    return static_cast<int>(cudaGetLastError());
  }
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
