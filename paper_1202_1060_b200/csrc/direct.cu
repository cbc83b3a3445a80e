// direct.cu -- posterior-free SMEM-resident decoder for check-regular
// degree-6 codes whose VNs have degree <= 3 (BASELINE configs 1, 2, 5: the
// (3,6) n=1008 code) under schedules whose groups fit one CN item per thread.
//
// State of the FV frames a CTA decodes (host.hpp DirectTables): one array of
// cells of FV floats (one per frame) -- a cell per edge and an L cell per VN
// (clamped channel LLR, log2 units). Every VN has one holder edge whose cell
// stores c2v + L; every CN holds exactly two. A CN item of group g
// (decoder.hpp:112-127) forms the v2c of its six edges (var_update,
// decoder.hpp:91-105) as
//     holder edge   v2c = (c2v_x + c2v_y) + L          three reads
//     other edges   v2c = (c2v_h + L) + c2v_o          two reads
// runs the exclusion boxplus (check_update, decoder.hpp:59-87; common.cuh) and
// overwrites its own six cells (c2v, or c2v + L for the two it holds): 14
// reads and 6 writes of shared memory per CN. There is no posterior array:
// nothing is updated in place, no fix-up re-sum and no exact-totals pass
// exist, and every v2c is exact to two fp32 additions. Posteriors are formed
// only where the reference forms them: for the hard decision / syndrome test
// (decoder.hpp:162-171) and the outputs.
//
// A thread serves all FV frames of its CN: one 16-byte (FV = 4) or 8-byte
// shared-memory access per cell, every add / mul / fma as packed fp32 on frame
// pairs (common.cuh boxplus_row_x2), and with FV = 4 two independent boxplus
// chains per thread, which fills the fixed-latency gaps a single chain leaves
// and halves the per-frame cost of records, addresses and barriers.
//
// Jacobi inside a group: a CN of the group may read a cell that another CN of
// the same group overwrites (a VN shared by both), so one barrier separates
// the loads of a group from its stores and a second one the stores from the
// next group's loads. A group is one CN item per thread (the launch plan
// guarantees it), so no item of a group can start after another has stored.
//
// Persistent CTAs take frames from a queue (one atomicAdd per frame): at an
// iteration boundary a slot whose frame stopped (zero syndrome with early
// stop, or max_iters) writes its outputs and is refilled; slots are
// independent lanes, so outputs do not depend on the slot a frame used.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "kernels.cuh"

namespace ldpcb {
namespace {

using namespace dev;

#ifndef LDPCB_DIRECT_MINB
#define LDPCB_DIRECT_MINB 5  // A/B: -DLDPCB_DIRECT_MINB=6
#endif
constexpr int kDirectThreads = 96;  // C1 NDGSBP: 84 CN items per group
constexpr int kFloodThreads = 256;  // flooding: 504 CN items per iteration in two rounds; two CTAs per SM at 128 registers
                                    // (18 warps per SM would cap the kernel at 96 registers: 88 bytes of spills)

// The CTA's dynamic shared memory: the cell array, then the hard-decision
// bytes. Every device function addresses it
// through this symbol (a pointer parameter would lose the shared-window base
// and cost an address add per access).
extern __shared__ __align__(16) char dsm[];

// Resident CTAs per SM the register budget is sized for. Shared memory fits
// six 2-frame CTAs (33 KB), but six 96-thread CTAs are 18 warps, five on
// some SM sub-partition, which caps the kernel at 96 registers: ptxas then
// re-issues FMNMX + EX2 for two of a CN item's six inputs where their z is
// needed again (40 MUFU per item instead of 36) and spills 16 bytes. Sized
// for five CTAs (15 warps, 112 registers, no re-issue, no spill) the C5 step
// takes 98.96 ms against 102.85 (64-thread launches, GSBP, still run six
// CTAs per SM). Three 4-frame CTAs (66 KB) with four frames per thread. A seventh 2-frame
// CTA was tried (all control state moved to global memory so that the
// kernel's shared memory is exactly the 32256-byte state): the 16 K registers
// of an SM sub-partition hold five 96-register warps, so 21 warps per SM need
// 80 registers per thread, and that build (64 bytes of spills) ran 4 % slower
// than six CTAs (108.3 against 104.1 ms per 2^21 frames).
template <int FV>
constexpr int direct_min_blocks() {
  return FV == 2 ? LDPCB_DIRECT_MINB : 3;
}

// one cell: FV frames as FV / 2 packed pairs
template <int FV>
struct Cell {
  f32x2 p[FV / 2];
};
template <int FV>
__device__ __forceinline__ Cell<FV> ld_cell(const char* base, uint32_t off) {
  Cell<FV> r;
  if constexpr (FV == 4) {
    const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(base + off);
    r.p[0] = t.x;
    r.p[1] = t.y;
  } else {
    r.p[0] = *reinterpret_cast<const f32x2*>(base + off);
  }
  return r;
}
template <int FV>
__device__ __forceinline__ void st_cell(char* base, uint32_t off, const Cell<FV>& c) {
  if constexpr (FV == 4)
    *reinterpret_cast<ulonglong2*>(base + off) = make_ulonglong2(c.p[0], c.p[1]);
  else
    *reinterpret_cast<f32x2*>(base + off) = c.p[0];
}
template <int FV>
__device__ __forceinline__ Cell<FV> add_cell(const Cell<FV>& a, const Cell<FV>& b) {
  Cell<FV> r;
#pragma unroll
  for (int i = 0; i < FV / 2; ++i) r.p[i] = add2(a.p[i], b.p[i]);
  return r;
}
// bit i = sign of frame i (tie -> 0, decoder.hpp:166)
template <int FV>
__device__ __forceinline__ unsigned sign_bits(const Cell<FV>& t) {
  unsigned b = 0;
#pragma unroll
  for (int i = 0; i < FV / 2; ++i)
    b |= ((lo2(t.p[i]) < 0.f ? 1u : 0u) | (hi2(t.p[i]) < 0.f ? 2u : 0u)) << (2 * i);
  return b;
}

// the ten words of a CN record (host.hpp DirectTables), prefetched into
// registers one group ahead
struct DRec {
  int4 a, b;
  int2 c;
  __device__ __forceinline__ void load(const int32_t* __restrict__ p) {
    const int4* q = reinterpret_cast<const int4*>(p);
    a = __ldg(q);
    b = __ldg(q + 1);
    c = __ldg(reinterpret_cast<const int2*>(q + 2));
  }
  // keeps the consumers of the prefetched record below this point
  __device__ __forceinline__ void pin() {
    asm volatile("" : "+r"(a.x), "+r"(a.y), "+r"(a.z), "+r"(a.w));
    asm volatile("" : "+r"(b.x), "+r"(b.y), "+r"(b.z), "+r"(b.w));
    asm volatile("" : "+r"(c.x), "+r"(c.y));
  }
};

__device__ __forceinline__ uint32_t lo16(int w) { return static_cast<uint32_t>(w) & 0xffffu; }
__device__ __forceinline__ uint32_t hi16(int w) { return static_cast<uint32_t>(w) >> 16; }

// One sub-iteration (decoder.hpp:112-127): the thread's CN item of group grp.
// cn: the CNs of this group; next_rec: the thread's record for this group
// (requested one group ahead). On return they describe the next group.
template <int FV>
__device__ __forceinline__ void direct_group(const DevGraph& g, int tid, int grp, int& cn, int2& nx, DRec& next_rec) {
  const int G = g.G;
  const bool has = tid < cn;
  Cell<FV> x[6], lh[2];
  uint32_t own[6];
  const DRec cur = next_rec;
  // the next group's record, requested a whole group before use (nx = its first
  // record and CN count, read from the constant bank a group ago)
  if (tid < nx.y) next_rec.load(g.d_cn_rec + static_cast<size_t>(nx.x + tid) * 12);
  const int ncn = nx.y;
  if (has) {
    const int4 ra = cur.a, rb = cur.b;
    const int2 rc = cur.c;
    const int w[10] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w, rc.x, rc.y};
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // the two edges this CN holds: (c2v_x + c2v_y) + L
      own[k] = lo16(w[2 * k]);
      const Cell<FV> cx = ld_cell<FV>(dsm, hi16(w[2 * k]));
      const Cell<FV> cy = ld_cell<FV>(dsm, lo16(w[2 * k + 1]));
      lh[k] = ld_cell<FV>(dsm, hi16(w[2 * k + 1]));
      x[k] = add_cell<FV>(add_cell<FV>(cx, cy), lh[k]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // (c2v_h + L) + c2v_o: the holder's cell and the third edge's
      auto field = [&](int i) { return (i & 1) ? hi16(w[4 + i / 2]) : lo16(w[4 + i / 2]); };
      own[2 + j] = field(3 * j);
      x[2 + j] = add_cell<FV>(ld_cell<FV>(dsm, field(3 * j + 1)), ld_cell<FV>(dsm, field(3 * j + 2)));
    }
  }
  int gg = grp + 2;
  gg -= gg >= G ? G : 0;
  gg -= gg >= G ? G : 0;
  nx = make_int2(g.d_goff[gg], g.d_goff[gg + 1] - g.d_goff[gg]);
  __syncthreads();  // every load of the group precedes every store
  if (has) {
    if constexpr (FV == 2) {  // every output stored as the boxplus emits it
      f32x2 xi[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) xi[k] = x[k].p[0];
      boxplus_row_x2<6, true>(xi, 6, [&](int k, f32x2 c) {
        *reinterpret_cast<f32x2*>(dsm + own[k]) = k < 2 ? add2(c, lh[k].p[0]) : c;
      });
    } else {
      Cell<FV> out[6];
#pragma unroll
      for (int i = 0; i < FV / 2; ++i) {
        f32x2 xi[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) xi[k] = x[k].p[i];
        boxplus_row_x2<6, true>(xi, 6, [&](int k, f32x2 c) { out[k].p[i] = c; });
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) st_cell<FV>(dsm, own[k], k < 2 ? add_cell<FV>(out[k], lh[k]) : out[k]);
    }
  }
  __syncthreads();
  next_rec.pin();
  cn = ncn;
}

// One flooding iteration (a single group of more CNs than threads): every
// thread runs its CN items round after round, reading the edge cells at byte
// offset rd and writing those at wr (the two copies, swapped by the caller
// every iteration), so no item can read a message of this iteration and no
// barrier is needed inside the iteration (Jacobi, decoder.hpp:107-113).
template <int FV>
__device__ __forceinline__ void direct_flood_iteration(const DevGraph& g, int tid, int nt, uint32_t rd, uint32_t wr) {
  const int cn = g.d_goff[1] - g.d_goff[0];
  DRec next_rec;
  if (tid < cn) next_rec.load(g.d_cn_rec + static_cast<size_t>(tid) * 12);
  for (int j = tid; j < cn; j += nt) {
    const DRec cur = next_rec;
    if (j + nt < cn) next_rec.load(g.d_cn_rec + static_cast<size_t>(j + nt) * 12);
    const int w[10] = {cur.a.x, cur.a.y, cur.a.z, cur.a.w, cur.b.x, cur.b.y, cur.b.z, cur.b.w, cur.c.x, cur.c.y};
    Cell<FV> x[6], lh[2];
    uint32_t own[6];
    const char* const src = dsm + rd;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      own[k] = lo16(w[2 * k]);
      const Cell<FV> cx = ld_cell<FV>(src, hi16(w[2 * k]));
      const Cell<FV> cy = ld_cell<FV>(src, lo16(w[2 * k + 1]));
      lh[k] = ld_cell<FV>(dsm, hi16(w[2 * k + 1]));
      x[k] = add_cell<FV>(add_cell<FV>(cx, cy), lh[k]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      auto field = [&](int i) { return (i & 1) ? hi16(w[4 + i / 2]) : lo16(w[4 + i / 2]); };
      own[2 + q] = field(3 * q);
      x[2 + q] = add_cell<FV>(ld_cell<FV>(src, field(3 * q + 1)), ld_cell<FV>(src, field(3 * q + 2)));
    }
    static_assert(FV == 2, "flooding runs two frames per thread");
    f32x2 xi[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) xi[k] = x[k].p[0];
    boxplus_row_x2<6, true>(xi, 6, [&](int k, f32x2 c) {
      *reinterpret_cast<f32x2*>(dsm + wr + own[k]) = k < 2 ? add2(c, lh[k].p[0]) : c;
    });
    next_rec.pin();
  }
}

// Per-CTA control state (shared memory): slot ff holds frame `frame[ff]`
// (-1: none); done: 0 decoding, 1 idle, 2 retiring, 3 refilled this round.
template <int FV>
struct DirectCtl {
  long long frame[FV];
  int done[FV], weight[FV], iters[FV], conv[FV], berr[FV];
  unsigned long long cnt[6];
  int active, retiring;
};

__device__ __forceinline__ long long direct_pull(unsigned long long* queue, int64_t frames) {
  const unsigned long long f = atomicAdd(queue, 1ull);
  return f < static_cast<unsigned long long>(frames) ? static_cast<long long>(f) : -1ll;
}

// init_state (decoder.hpp:39-52) of the slots in `mask`: every cell 0
// (c2v = 0), then L = clamp(llr) (kClampB for an idle slot) into the L cells
// and the holder cells (0 + L). All global loads of a batch of elements are
// issued before any is used. The iteration-boundary functions are kept out
// of line: the sub-iteration loop then owns the whole register budget.
template <int FV, bool FLOOD>
__device__ __forceinline__ void direct_load_slots(const DevGraph& g, const DecodeArgs& a, const DirectCtl<FV>* ctl,
                                                  unsigned mask) {
  constexpr int CB = 4 * FV;
  const int tid = threadIdx.x, nt = blockDim.x, n = g.n;
  const uint32_t l_off = static_cast<uint32_t>(g.d_l_base) * CB;
  if (mask == (1u << FV) - 1) {
    Cell<FV> z;
#pragma unroll
    for (int i = 0; i < FV / 2; ++i) z.p[i] = 0ull;
    for (int i = tid; i < g.d_l_base; i += nt) st_cell<FV>(dsm, i * CB, z);
  } else {
#pragma unroll
    for (int ff = 0; ff < FV; ++ff)
      if (mask & (1u << ff))
        for (int i = tid; i < g.d_l_base; i += nt) *reinterpret_cast<float*>(dsm + 4 * ff + i * CB) = 0.f;
  }
  __syncthreads();
  const bool vec = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(a.llr) & 15) == 0;
  constexpr int U = 3;
#pragma unroll
  for (int ff = 0; ff < FV; ++ff) {
    if (!(mask & (1u << ff))) continue;
    char* const sb = dsm + 4 * ff;
    const long long f = ctl->frame[ff];
    auto put = [&](int pos, int hold, float raw) {
      const float y = f >= 0 ? clamp_llr(raw) * kLog2e : kClampB;
      *reinterpret_cast<float*>(sb + l_off + pos * CB) = y;
      *reinterpret_cast<float*>(sb + hold) = y;
      if constexpr (FLOOD)  // both copies of the edge cells
        *reinterpret_cast<float*>(sb + hold + static_cast<uint32_t>(g.d_buf_cells) * CB) = y;
    };
    if (f >= 0 && vec) {
      const float4* l4 = reinterpret_cast<const float4*>(a.llr + f * n);
      const int4* p4 = reinterpret_cast<const int4*>(g.d_vn_pos);
      const int4* h4 = reinterpret_cast<const int4*>(g.d_vn_hold);
      for (int b0 = tid; b0 < n / 4; b0 += U * nt) {
        float4 x[U];
        int4 p[U], h[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (b0 + u * nt < n / 4)
            x[u] = ldg_stream(l4 + b0 + u * nt), p[u] = __ldg(p4 + b0 + u * nt), h[u] = __ldg(h4 + b0 + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (b0 + u * nt < n / 4) {
            put(p[u].x, h[u].x, x[u].x);
            put(p[u].y, h[u].y, x[u].y);
            put(p[u].z, h[u].z, x[u].z);
            put(p[u].w, h[u].w, x[u].w);
          }
      }
    } else {
      const float* llr = a.llr + (f >= 0 ? f : 0) * n;
      for (int i = tid; i < n; i += nt)
        put(__ldg(g.d_vn_pos + i), __ldg(g.d_vn_hold + i), f >= 0 ? __ldg(llr + i) : 0.f);
    }
    if (f >= 0 && a.trace)
      for (int i = tid; i < a.max_iters; i += nt) a.trace[f * a.max_iters + i] = -1;
  }
  __syncthreads();
}

// End of an iteration that tests the syndrome: hard decisions, syndrome
// weights, per-frame bookkeeping (decoder.hpp:162-177), outputs of the frames
// that stopped (sim.hpp:119-123) and their refill from the queue.
// it_cta: iterations since the CTA's slots were last refilled together (fixed
// iteration counts). Returns 0: carry on, 1: slots were refilled, 2: no slot
// is busy and the queue is empty.
template <int FV, bool FLOOD>
__device__ __forceinline__ int direct_iteration_end(const DevGraph& g, const DecodeArgs& a,
                                                    unsigned long long* queue, DirectCtl<FV>* ctl, int it_cta,
                                                    uint32_t rd_flood) {  // byte offset of the current edge cells
  const uint32_t rd = FLOOD ? rd_flood : 0u;
  constexpr int CB = 4 * FV;
  const int tid = threadIdx.x, nt = blockDim.x, n = g.n, m = g.m;
  // hard-decision bytes [n], bit i = frame i: byte offset hd in the CTA's shared memory. Everything below
  // addresses dsm[integer offset], which compiles to LDS [R + uniform base] as in the sub-iteration loop
  // (a derived pointer costs a generic-to-shared conversion and an address add per access).
  const uint32_t hd = static_cast<uint32_t>(g.d_cells) * CB;
  const uint8_t* const s_hd = reinterpret_cast<const uint8_t*>(dsm) + hd;
  const int nb = (n + 7) >> 3;
  const bool check = a.early_stop || a.trace;
  // hard decisions (tie -> 0) from the totals ((c2v_h + L) + c2v) + c2v, one sign bit per frame
  int w[FV] = {};
  if constexpr (FLOOD) {
    // flooding (256 threads, the current copy at a run-time offset) keeps the pointer form: the
    // integer-offset loops below ran its early-stop decodes 5 % slower (1.68e7 against 1.77e7 frames/s)
    uint8_t* const hb = reinterpret_cast<uint8_t*>(dsm + hd);
    for (int pos = tid; pos < n; pos += nt) {
      const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_vn_rec) + pos);
      Cell<FV> t = add_cell<FV>(ld_cell<FV>(dsm + rd, lo16(r.x)), ld_cell<FV>(dsm + rd, hi16(r.x)));
      t = add_cell<FV>(t, ld_cell<FV>(dsm + rd, lo16(r.y)));
      hb[pos] = static_cast<uint8_t>(sign_bits<FV>(t));
    }
    __syncthreads();
    for (int r = tid; r < m; r += nt) {  // syndrome weight (decoder.hpp:129-137)
      const int4 q = __ldg(reinterpret_cast<const int4*>(g.d_all_cn) + r);
      const unsigned x = hb[lo16(q.x)] ^ hb[hi16(q.x)] ^ hb[lo16(q.y)] ^ hb[hi16(q.y)] ^ hb[lo16(q.z)] ^ hb[hi16(q.z)];
#pragma unroll
      for (int i = 0; i < FV; ++i) w[i] += (x >> i) & 1u;
    }
  } else {
#pragma unroll 2
    for (int pos = tid; pos < n; pos += nt) {
      const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_vn_rec) + pos);
      Cell<FV> t = add_cell<FV>(ld_cell<FV>(dsm, lo16(r.x)), ld_cell<FV>(dsm, hi16(r.x)));
      t = add_cell<FV>(t, ld_cell<FV>(dsm, lo16(r.y)));
      dsm[hd + pos] = static_cast<char>(sign_bits<FV>(t));
    }
    __syncthreads();
#pragma unroll 2
    for (int r = tid; r < m; r += nt) {  // syndrome weight (decoder.hpp:129-137)
      const int4 q = __ldg(reinterpret_cast<const int4*>(g.d_all_cn) + r);
      auto b = [&](uint32_t v) { return static_cast<unsigned>(static_cast<uint8_t>(dsm[hd + v])); };
      const unsigned x = b(lo16(q.x)) ^ b(hi16(q.x)) ^ b(lo16(q.y)) ^ b(hi16(q.y)) ^ b(lo16(q.z)) ^ b(hi16(q.z));
#pragma unroll
      for (int i = 0; i < FV; ++i) w[i] += (x >> i) & 1u;
    }
  }
  {
#pragma unroll
    for (int i = 0; i < FV; ++i)
      if (w[i]) atomicAdd(&ctl->weight[i], w[i]);
  }
  __syncthreads();
  if (tid == 0) {
    int retiring = 0, active = 0;
    for (int ff = 0; ff < FV; ++ff) {
      if (!ctl->done[ff]) {
        const int w = ctl->weight[ff];
        const int it = check ? ++ctl->iters[ff] : (ctl->iters[ff] = it_cta);
        if (a.trace) a.trace[ctl->frame[ff] * a.max_iters + it - 1] = w;
        ctl->conv[ff] = w == 0;
        if ((w == 0 && a.early_stop) || it >= a.max_iters) {  // decoder.hpp:173-177
          ctl->done[ff] = 2;
          ++retiring;
        }
      }
      ctl->weight[ff] = 0;
      active += ctl->done[ff] != 1;
    }
    ctl->retiring = retiring;
    ctl->active = active;
  }
  __syncthreads();
  if (ctl->retiring == 0) return ctl->active == 0 ? 2 : 0;
  for (int ff = 0; ff < FV; ++ff) {
    if (ctl->done[ff] != 2) continue;
    const long long f = ctl->frame[ff];
    int errs = 0;
    if (a.bits && a.bits_packed) {
      for (int b = tid; b < nb; b += nt) {
        unsigned byte = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int v = b * 8 + q;
          if (v < n) byte |= ((s_hd[__ldg(g.d_vn_pos + v)] >> ff) & 1u) << q;
        }
        a.bits[f * nb + b] = static_cast<uint8_t>(byte);
        errs += __popc(byte);
      }
    } else if (a.bits || a.counters || a.bit_errors) {
      for (int v = tid; v < n; v += nt) {
        const int bit = (s_hd[__ldg(g.d_vn_pos + v)] >> ff) & 1;
        if (a.bits) a.bits[f * n + v] = static_cast<uint8_t>(bit);
        errs += bit;
      }
    }
    if (errs) atomicAdd(&ctl->berr[ff], errs);
    if (a.posterior) {
      const char* const sb = dsm + rd + 4 * ff;
      for (int v = tid; v < n; v += nt) {
        const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_vn_rec) + __ldg(g.d_vn_pos + v));
        float t = *reinterpret_cast<const float*>(sb + lo16(r.x)) + *reinterpret_cast<const float*>(sb + hi16(r.x));
        t += *reinterpret_cast<const float*>(sb + lo16(r.y));
        a.posterior[f * n + v] = t * kLn2;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int active = 0;
    for (int ff = 0; ff < FV; ++ff) {
      if (ctl->done[ff] == 2) {
        const long long f = ctl->frame[ff];
        const int it = a.early_stop ? ctl->iters[ff] : a.max_iters;
        if (a.iterations) a.iterations[f] = it;
        if (a.converged) a.converged[f] = static_cast<uint8_t>(ctl->conv[ff]);
        if (a.bit_errors) a.bit_errors[f] = ctl->berr[ff];
        ctl->cnt[0] += 1;
        ctl->cnt[1] += ctl->berr[ff];
        ctl->cnt[2] += ctl->berr[ff] > 0;
        ctl->cnt[3] += ctl->conv[ff];
        ctl->cnt[4] += it;
        ctl->cnt[5] += ctl->conv[ff] ? it : 0;
        ctl->frame[ff] = direct_pull(queue, a.frames);
        ctl->done[ff] = ctl->frame[ff] < 0 ? 1 : 3;
        ctl->iters[ff] = ctl->conv[ff] = ctl->berr[ff] = 0;
      }
      active += ctl->done[ff] != 1;
    }
    ctl->active = active;
  }
  __syncthreads();
  if (ctl->active == 0) return 2;
  unsigned mask = 0;
#pragma unroll
  for (int ff = 0; ff < FV; ++ff) mask |= (ctl->done[ff] == 3 ? 1u : 0u) << ff;
  direct_load_slots<FV, FLOOD>(g, a, ctl, mask);
  if (tid < FV && ctl->done[tid] == 3) ctl->done[tid] = 0;
  __syncthreads();
  return 1;
}

// State after a.max_subiters sub-iterations: c2v and v2c per CN-major edge id.
template <int FV>
__device__ __forceinline__ void direct_dump(const DevGraph& g, const DecodeArgs& a, const DirectCtl<FV>* ctl,
                                            uint32_t rd = 0) {  // rd: byte offset of the current edge cells
  const int tid = threadIdx.x, nt = blockDim.x, E = g.E;
  for (int ff = 0; ff < FV; ++ff) {
    const long long f = ctl->frame[ff];
    if (f < 0) continue;
    const char* const sb = dsm + 4 * ff;
    for (int e = tid; e < E; e += nt) {
      const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_edge_rec) + e);
      const bool holder = hi16(r.x) != 0xffffu;
      const float l = holder ? *reinterpret_cast<const float*>(sb + hi16(r.x)) : 0.f;
      // a holder cell stores c2v + L (exact while c2v = 0)
      if (a.c2v_out) a.c2v_out[f * E + e] = (*reinterpret_cast<const float*>(sb + rd + lo16(r.x)) - l) * kLn2;
      if (a.v2c_out) {
        float t = *reinterpret_cast<const float*>(sb + rd + lo16(r.y)) +
                  *reinterpret_cast<const float*>(sb + rd + hi16(r.y));
        if (holder) t += l;
        a.v2c_out[f * E + e] = clamp_bits(t) * kLn2;
      }
    }
  }
}

// FLOOD: one group in rounds over two copies of the edge cells (direct_flood_iteration)
template <int FV, bool FLOOD>
__global__ void __launch_bounds__(FLOOD ? kFloodThreads : kDirectThreads, FLOOD ? 2 : direct_min_blocks<FV>())
    decode_direct(const DevGraph g, const DecodeArgs a, unsigned long long* queue) {
  constexpr int CB = 4 * FV;  // cell bytes
  __shared__ DirectCtl<FV> ctl;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid < FV) {
    ctl.frame[tid] = direct_pull(queue, a.frames);
    ctl.done[tid] = ctl.frame[tid] < 0;
    ctl.weight[tid] = ctl.iters[tid] = ctl.conv[tid] = ctl.berr[tid] = 0;
  }
  if (tid < 6) ctl.cnt[tid] = 0ull;
  {  // padding cells stay zero
    float4* z = reinterpret_cast<float4*>(dsm);
    for (int i = tid; i < g.d_cells * CB / 16; i += nt) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  {
    bool any = false;
#pragma unroll
    for (int ff = 0; ff < FV; ++ff) any |= ctl.frame[ff] >= 0;
    if (!any) return;  // the queue was empty when this CTA started
  }
  direct_load_slots<FV, FLOOD>(g, a, &ctl, (1u << FV) - 1);

  // the thread's CN record one group ahead
  int cn = g.d_goff[1] - g.d_goff[0];
  DRec next_rec;
  if (tid < cn) next_rec.load(g.d_cn_rec + static_cast<size_t>(g.d_goff[0] + tid) * 12);
  const int g1 = g.G > 1 ? 1 : 0;
  int2 nx = make_int2(g.d_goff[g1], g.d_goff[g1 + 1] - g.d_goff[g1]);  // the group after the first
  const bool check = a.early_stop || a.trace;
  const int G = g.G;

  if constexpr (FLOOD) {
    const uint32_t buf = static_cast<uint32_t>(g.d_buf_cells) * CB;
    uint32_t rd = 0;  // the copy of the edge cells that holds the current messages
    if (a.max_subiters > 0) {  // state dump: a sub-iteration is an iteration
      for (int sub = 0; sub < a.max_subiters; ++sub) {
        direct_flood_iteration<FV>(g, tid, nt, rd, buf - rd);
        __syncthreads();
        rd = buf - rd;
      }
      direct_dump<FV>(g, a, &ctl, rd);
      return;
    }
    for (int it_cta = 1;; ++it_cta) {
      direct_flood_iteration<FV>(g, tid, nt, rd, buf - rd);
      __syncthreads();
      rd = buf - rd;
      if (!check && it_cta < a.max_iters) continue;
      const int r = direct_iteration_end<FV, true>(g, a, queue, &ctl, it_cta, rd);
      if (r == 2) break;
      if (r == 1) it_cta = 0;
    }
  } else {
    if (a.max_subiters > 0) {  // state dump
      for (int sub = 0, grp = 0; sub < a.max_subiters; ++sub, grp = grp + 1 < G ? grp + 1 : 0)
        direct_group<FV>(g, tid, grp, cn, nx, next_rec);
      direct_dump<FV>(g, a, &ctl);
      return;
    }
    for (int it_cta = 1;; ++it_cta) {
      // one iteration for every slot (decoder.hpp:157-160)
      for (int grp = 0; grp < G; ++grp) direct_group<FV>(g, tid, grp, cn, nx, next_rec);
      if (!check && it_cta < a.max_iters) continue;
      const int r = direct_iteration_end<FV, false>(g, a, queue, &ctl, it_cta, 0u);
      if (r == 2) break;
      if (r == 1) it_cta = 0;
    }
  }
  if (tid == 0 && a.counters)
    for (int i = 0; i < 6; ++i)
      if (ctl.cnt[i]) atomicAdd(a.counters + i, ctl.cnt[i]);
}

using DirectFn = void (*)(const DevGraph, const DecodeArgs, unsigned long long*);

DirectFn pick_direct(int fv, bool flood) {
  if (flood) return fv == 2 ? decode_direct<2, true> : nullptr;
  return fv == 4 ? decode_direct<4, false> : (fv == 2 ? decode_direct<2, false> : nullptr);
}

}  // namespace

// LDPCB_DIRECT=0 keeps every decode on the posterior-based kernels (A/B)
bool direct_enabled() {
  const char* e = std::getenv("LDPCB_DIRECT");
  return !e || std::atoi(e) != 0;
}

Plan plan_direct(const DevGraph& g, int64_t frames) {
  Plan p;
  const int fv = g.d_fv;
  if ((fv != 2 && fv != 4) || !g.d_cn_rec || g.per_frame) return p;
  const bool flood = g.d_buf_cells > 0;
  if (flood && fv != 2) return p;
  if (!flood && g.d_max_items > kDirectThreads) return p;  // one CN item per thread
  size_t bytes = static_cast<size_t>(g.d_cells) * 4 * fv + ((g.n + 15) & ~15);
  if (const char* e = std::getenv("LDPCB_DIRECT_PAD")) bytes += std::atoi(e);  // occupancy experiments
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) optin = 227 * 1024;
  if (bytes + 512 > static_cast<size_t>(optin)) return p;
  p.kernel = 3;
  p.fpc = fv;
  p.fv = fv;
  p.threads = flood ? kFloodThreads : std::max(64, std::min(kDirectThreads, (g.d_max_items + 31) / 32 * 32));
  p.smem = static_cast<int>(bytes);
  p.degree_bucket = 6;
  p.ctas = (frames + p.fpc - 1) / p.fpc;
  return p;
}

int launch_direct(const DevGraph& g, const DecodeArgs& a, void* stream, Plan* used) {
  const Plan p = plan_direct(g, a.frames);
  if (used) *used = p;
  if (p.kernel != 3) return static_cast<int>(cudaErrorInvalidConfiguration);
  if (a.frames <= 0) return 0;
  DirectFn fn = pick_direct(g.d_fv, g.d_buf_cells > 0);
  cudaError_t err =
      cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
  if (err != cudaSuccess) return static_cast<int>(err);
  // resident CTAs per device (cached per kernel, configuration and device)
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> cache;
  int dev = 0, resident = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(reinterpret_cast<const void*>(fn), p.threads, p.smem, dev);
    auto it = cache.find(key);
    if (it == cache.end()) {
      int sms = 0, per_sm = 0;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, p.threads, p.smem) != cudaSuccess || per_sm <= 0)
        return static_cast<int>(cudaErrorInvalidConfiguration);
      it = cache.emplace(key, sms * per_sm).first;
    }
    resident = it->second;
  }
  auto st = static_cast<cudaStream_t>(stream);
  // state dumps stop every CTA after its first frames: one CTA per FV frames
  const int64_t ctas = a.max_subiters > 0 ? p.ctas : std::min<int64_t>(p.ctas, resident);
  unsigned long long* queue = nullptr;
  err = cudaMallocAsync(reinterpret_cast<void**>(&queue), sizeof(unsigned long long), st);
  if (err == cudaSuccess) err = cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return static_cast<int>(err);
  fn<<<static_cast<unsigned>(ctas), p.threads, p.smem, st>>>(g, a, queue);
  note_launches(1);
  err = cudaGetLastError();
  cudaFreeAsync(queue, st);
  return static_cast<int>(err);
}

}  // namespace ldpcb
