// stream.cu -- HBM-streamed decoder for frames whose state does not fit one
// SM's shared memory (BASELINE configs 4 and 5: n = 64800, 1.3 MB per frame).
//
// A chunk of B frames (B a multiple of 4) is decoded together. Its state
// lives in HBM frame-interleaved, element (i, frame) at i * B + frame:
//   c2v [n_slots][B]   P [n][B]   L [n][B]   (log2 units, as in decoder.cu)
// Each thread serves one (CN or VN record, quad of 4 consecutive frames), so
// every state access is a 16-byte vector load and a warp reads 512
// contiguous bytes. Per sub-iteration of group g (decoder.hpp:112-127):
//   stream_cn<g>      CN updates of the group, in-place posterior update of
//                     VNs touched by one CN of the group (Jacobi-safe)
//   stream_vnsum<g>   exact re-sum of VNs shared by two or more of its CNs
// and per syndrome test: exact totals, syndrome weights, per-frame
// bookkeeping (decoder.hpp:162-177). Kernel boundaries are the barriers.
// HBM roofline: ~16 B per CN-edge update (c2v read+write, posterior
// read+write), SURVEY.md 8(d) roofline A.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace ldpcb {
namespace {

using namespace dev;

// Lane states (done[]): bit 0 set = the lane is not decoding. Chunk mode
// uses 0 / 1; the frame queue adds 2 = decoding the first iteration of a
// frame it was refilled with ("fresh", host.hpp KernelTables::cn_fresh) and
// 3 = retiring (stopped this iteration, outputs pending), 5 = waiting (outputs
// written, to be refilled at the next refill iteration).
enum LaneState : int { kLive = 0, kIdle = 1, kFresh = 2, kRetiring = 3, kWaiting = 5 };

struct ChunkState {
  int64_t B = 0;     // layout stride (frames), multiple of 4
  int nb = 0;        // frames of this chunk that are real
  int zero_slot = 0; // the always-zero c2v slot that pads VN records
  float* c2v = nullptr;
  float* P = nullptr;
  float* L = nullptr;
  int* done = nullptr;    // [B]
  int* weight = nullptr;  // [B]
  int* iters = nullptr;   // [B]
  int* conv = nullptr;    // [B]
  int* berr = nullptr;    // [B]
  // frame queue (launch_stream_queue)
  int64_t* frame = nullptr;           // [B] frame id held by each lane, -1 idle
  unsigned* sw = nullptr;             // [n][B/32] hard-decision sign words
  unsigned* fail = nullptr;           // [B/32] lanes failing some parity check (no-trace syndrome test), or null
  int* list = nullptr;                // [B] lanes retiring this iteration
  int* wlist = nullptr;               // [B] lanes waiting for a refill
  int* ctl = nullptr;                 // [0] retiring lanes, [1] lanes decoding, [2] waiting lanes
  unsigned long long* next = nullptr; // next frame id to hand out
};

// Programmatic dependent launch (per-group kernels): a CTA lets the next
// kernel of the stream start launching at once, and waits for the previous
// kernel to complete (and its writes to be visible) before touching state.
// The next kernel's CTAs are placed as this kernel's last wave drains, which
// hides the launch gap between ~900 dependent launches per chunk.
__device__ __forceinline__ void pdl_launch_next() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_launch_next();
  pdl_wait();
}

// V consecutive frames per thread: one V*4-byte vector access per element
template <int V>
struct Vec {
  float v[V];
};
template <int V>
__device__ __forceinline__ Vec<V> ldv(const float* p) {
  Vec<V> r;
  if constexpr (V == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
  } else if constexpr (V == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    r.v[0] = t.x, r.v[1] = t.y;
  } else {
    r.v[0] = *p;
  }
  return r;
}
template <int V>
__device__ __forceinline__ void stv(float* p, const Vec<V>& x) {
  if constexpr (V == 4)
    *reinterpret_cast<float4*>(p) = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
  else if constexpr (V == 2)
    *reinterpret_cast<float2*>(p) = make_float2(x.v[0], x.v[1]);
  else
    *p = x.v[0];
}
// lane states of the thread's V frames
template <int V>
struct States {
  int d[V];
};
template <int V>
__device__ __forceinline__ States<V> load_states(const ChunkState& s, int64_t q) {
  States<V> r;
  if constexpr (V == 4) {
    const int4 d = *reinterpret_cast<const int4*>(s.done + 4 * q);
    r.d[0] = d.x, r.d[1] = d.y, r.d[2] = d.z, r.d[3] = d.w;
  } else if constexpr (V == 2) {
    const int2 d = *reinterpret_cast<const int2*>(s.done + 2 * q);
    r.d[0] = d.x, r.d[1] = d.y;
  } else {
    r.d[0] = s.done[q];
  }
  return r;
}
// bit i set: frame i of the vector is not decoding
template <int V>
__device__ __forceinline__ unsigned done_bits(const States<V>& st) {
  unsigned b = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) b |= static_cast<unsigned>(st.d[i] & 1) << i;
  return b;
}
// bit i set: frame i is in the first iteration of a refilled frame
template <int V>
__device__ __forceinline__ unsigned fresh_bits(const States<V>& st) {
  unsigned b = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) b |= static_cast<unsigned>(st.d[i] == kFresh) << i;
  return b;
}
template <int V>
__device__ __forceinline__ unsigned done_bits(const ChunkState& s, int64_t q) {
  return done_bits<V>(load_states<V>(s, q));
}

// L = P = clamp(llr) in log2 units, transposed [nb][n] -> [n][B] through a
// 32 x 32 shared-memory tile; padding frames (>= nb) are marked done.
__global__ void stream_init(int n, const int32_t* __restrict__ pos, const float* __restrict__ llr, ChunkState s) {
  __shared__ float tile[32][33];
  const int v0 = blockIdx.x * 32, f0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int f = f0 + r, v = v0 + threadIdx.x;
    tile[r][threadIdx.x] = (f < s.nb && v < n) ? clamp_llr(llr[static_cast<int64_t>(f) * n + v]) * kLog2e : kClampB;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int v = v0 + r, f = f0 + threadIdx.x;
    if (v < n && f < s.B) {
      const float x = tile[threadIdx.x][r];
      const int64_t row = __ldg(pos + v);
      s.L[row * s.B + f] = x;
      s.P[row * s.B + f] = x;
    }
  }
  if (blockIdx.x == 0 && threadIdx.y == 0) {
    const int f = f0 + threadIdx.x;
    if (f < s.B) {
      s.done[f] = f >= s.nb;
      s.weight[f] = 0;
      s.iters[f] = 0;
      s.conv[f] = 0;
      s.berr[f] = 0;
    }
  }
}

// CN phase of one group over (record, V-frame vector) items. fresh (frame
// queue only, else null): per-record bits of KernelTables::cn_fresh for lanes
// in the first iteration of a refilled frame (old c2v = 0, P = L at a VN's
// first touch), which is what a zeroed c2v and P = L would give.
// FRESH = false compiles none of the fresh-frame code (the fixed-iteration
// and chunked early-stop paths: 106 registers, two CTAs per SM; with it 147).
// Two CTAs per SM: the fresh-frame variant is held to 128 registers as well
// (92 bytes of spills; at its natural 146 registers one CTA per SM fits and
// the frame queue's CN launches took 190 us instead of 145).
template <int D, bool EXACT, int V, bool FRESH>
__global__ void __launch_bounds__(256, (D <= 6 && V == 4) ? 2 : 1) stream_cn(const int32_t* __restrict__ recs, int CS, int count, ChunkState s,
                                                 const uint32_t* __restrict__ fresh) {
  pdl_launch_next();
  const int64_t QB = s.B / V;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= count * QB) return;
  const int j = static_cast<int>(item / QB);
  const int64_t q = item - j * QB;
  // the CN record is a constant table: requested before waiting for the
  // previous kernel, so its latency overlaps that kernel's drain
  const CnRecord<D, EXACT> cr(recs + static_cast<int64_t>(j) * CS, CS);
  pdl_wait();
  const States<V> st = load_states<V>(s, q);
  const unsigned dn = done_bits<V>(st);
  if (dn == (1u << V) - 1) return;
  unsigned fr = 0u;
  uint32_t fbits = 0u;
  if constexpr (FRESH) {
    fr = fresh_bits<V>(st);
    fbits = fr ? __ldg(fresh + j) : 0u;
  }
  const int base = cr.slot();
  const unsigned mask = cr.mask();
  const int deg = cr.deg();
  Vec<V> pv[D], old[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (cr.has(k)) {
      pv[k] = ldv<V>(s.P + static_cast<int64_t>(cr.var(k)) * s.B + V * q);
      old[k] = ldv<V>(s.c2v + static_cast<int64_t>(base + k) * s.B + V * q);
      if (FRESH && fr && (fbits & (1u << k))) {  // first touch of this VN in a fresh frame: P = L
        const Vec<V> l = ldv<V>(s.L + static_cast<int64_t>(cr.var(k)) * s.B + V * q);
#pragma unroll
        for (int i = 0; i < V; ++i)
          if (fr & (1u << i)) pv[k].v[i] = l.v[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) pv[k].v[i] = old[k].v[i] = 0.f;
    }
  }
  Vec<V> out[D];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const bool zero_old = FRESH && (fr & (1u << i)) && (fbits >> 31);  // first processing of this CN
    float x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = pv[k].v[i] - (zero_old ? 0.f : old[k].v[i]);
    boxplus_row<D, EXACT>(x, deg, [&](int k, float c) { out[k].v[i] = c; });
  }
  if constexpr (!FRESH) {
    // frames that already stopped (decoder.hpp:173-177) keep their state
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (dn & (1u << i))
#pragma unroll
        for (int k = 0; k < D; ++k) out[k].v[i] = old[k].v[i];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (!cr.has(k)) continue;
      stv<V>(s.c2v + static_cast<int64_t>(base + k) * s.B + V * q, out[k]);
      if (mask & (1u << k)) {
        Vec<V> p;
#pragma unroll
        for (int i = 0; i < V; ++i) p.v[i] = (pv[k].v[i] - old[k].v[i]) + out[k].v[i];
        stv<V>(s.P + static_cast<int64_t>(cr.var(k)) * s.B + V * q, p);
      }
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (!cr.has(k)) continue;
    Vec<V> o, p;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const bool zero_old = (fr & (1u << i)) && (fbits >> 31);
      // frames that already stopped (decoder.hpp:173-177) keep their state
      const bool live = !(dn & (1u << i));
      o.v[i] = live ? out[k].v[i] : old[k].v[i];
      p.v[i] = live ? (pv[k].v[i] - (zero_old ? 0.f : old[k].v[i])) + out[k].v[i] : pv[k].v[i];
    }
    stv<V>(s.c2v + static_cast<int64_t>(base + k) * s.B + V * q, o);
    if (mask & (1u << k)) stv<V>(s.P + static_cast<int64_t>(cr.var(k)) * s.B + V * q, p);
  }
}

// ---- stream_cn with TMA staging (regular rows of degree 3 / 6, four frames
// per thread, chunk layouts whose quad count is a multiple of the CTA size).
// A CTA serves one CN record and kTmaQuads consecutive frame quads: the D
// posterior rows and D c2v rows it needs are 2 D contiguous 4 KB segments of
// the [index][B] state, fetched by 2 D bulk copies (cp.async.bulk, the 1-D
// TMA) that one thread issues against an mbarrier -- no per-thread address
// arithmetic and no registers holding loads in flight, so three CTAs fit an
// SM (144 KB of state in flight against 96 KB for the LDG.128 kernel). Every
// thread then works on its quad in shared memory (packed fp32 on frame
// pairs, bit-identical to the scalar boxplus), writes the new c2v and the
// in-place posteriors over the staged rows, and one thread sends the rows
// back with bulk stores. Same values as stream_cn<D, true, 4, false>.
constexpr int kTmaQuads = 256;                 // quads (threads) per CTA
constexpr int kTmaRowBytes = kTmaQuads * 16;   // one staged row segment

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kTmaQuads, 3) stream_cn_tma(const int32_t* __restrict__ recs, int count, ChunkState s) {
  extern __shared__ __align__(128) char tsm[];  // [2 D][kTmaQuads] float4: posterior rows, then c2v rows
  __shared__ __align__(8) unsigned long long bar_storage;
  pdl_launch_next();
  const int tid = threadIdx.x;
  const int64_t QB = s.B / 4;
  const int64_t tiles_per_rec = QB / kTmaQuads;
  const int j = static_cast<int>(blockIdx.x / tiles_per_rec);
  const int64_t q0 = (blockIdx.x - j * tiles_per_rec) * kTmaQuads;
  if (j >= count) return;
  // the CN record is a constant table: requested before waiting for the previous kernel
  const CnRecordPacked<D> cr(recs + static_cast<int64_t>(j) * 4, 4);
  const uint32_t bar = smem_u32(&bar_storage);
  const uint32_t base = smem_u32(tsm);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  const int slot0 = cr.slot();
  const unsigned mask = cr.mask();
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * D * kTmaRowBytes)
                 : "memory");
#pragma unroll
    for (int k = 0; k < D; ++k) {
      bulk_load(base + k * kTmaRowBytes, s.P + static_cast<int64_t>(cr.var(k)) * s.B + 4 * q0, kTmaRowBytes, bar);
      bulk_load(base + (D + k) * kTmaRowBytes, s.c2v + static_cast<int64_t>(slot0 + k) * s.B + 4 * q0,
                kTmaRowBytes, bar);
    }
  }
  const unsigned dn = done_bits<4>(s, q0 + tid);  // overlaps the copies
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LDPCB_TMA_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@p bra LDPCB_TMA_DONE;\n"
      "bra LDPCB_TMA_WAIT;\n"
      "LDPCB_TMA_DONE:\n"
      "}\n" ::"r"(bar)
      : "memory");
  char* const mine = tsm + tid * 16;
  if (dn != 0xfu) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // the quad as two frame pairs
      f32x2 x[D];
#pragma unroll
      for (int k = 0; k < D; ++k)
        x[k] = sub2(*reinterpret_cast<const f32x2*>(mine + k * kTmaRowBytes + 8 * h),
                    *reinterpret_cast<const f32x2*>(mine + (D + k) * kTmaRowBytes + 8 * h));
      const bool live0 = !(dn & (1u << (2 * h))), live1 = !(dn & (2u << (2 * h)));
      boxplus_row_x2<D, true>(x, D, [&](int k, f32x2 c) {
        f32x2* const cp = reinterpret_cast<f32x2*>(mine + (D + k) * kTmaRowBytes + 8 * h);
        f32x2* const pp = reinterpret_cast<f32x2*>(mine + k * kTmaRowBytes + 8 * h);
        const f32x2 p = add2(x[k], c);  // in-place posterior: v2c + c
        if (live0 && live1) {
          *cp = c;
          if (mask & (1u << k)) *pp = p;
        } else {  // a frame that already stopped (decoder.hpp:173-177) keeps its state
          const f32x2 oc = *cp, op = *pp;
          *cp = pack2(live0 ? lo2(c) : lo2(oc), live1 ? hi2(c) : hi2(oc));
          if (mask & (1u << k)) *pp = pack2(live0 ? lo2(p) : lo2(op), live1 ? hi2(p) : hi2(op));
        }
      });
    }
  }
  // generic-proxy writes above -> async-proxy reads of the bulk stores
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      bulk_store(s.c2v + static_cast<int64_t>(slot0 + k) * s.B + 4 * q0, base + (D + k) * kTmaRowBytes, kTmaRowBytes);
      if (mask & (1u << k))
        bulk_store(s.P + static_cast<int64_t>(cr.var(k)) * s.B + 4 * q0, base + k * kTmaRowBytes, kTmaRowBytes);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes complete before the CTA (and the grid) ends
  }
}

// P_v = L_v + sum of c2v over the VN's edges, ascending CN order (the totals
// of decoder.hpp:162-165), over (VN record, V-frame vector) items.
// Records are padded with the zero slot after the VN's last edge; the loop
// stops there (a warp serves one VN, so the exit is warp-uniform).
template <int V, bool FRESH>
__global__ void __launch_bounds__(256) stream_vnsum(const int4* __restrict__ recs, int vs4, int count, ChunkState s,
                                                    int skip_done, const uint32_t* __restrict__ fresh) {
  pdl_launch_next();
  const int64_t QB = s.B / V;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= count * QB) return;
  const int j = static_cast<int>(item / QB);
  const int64_t q = item - j * QB;
  const int4* rec = recs + static_cast<int64_t>(j) * vs4;
  int4 t = __ldg(rec);  // constant table: requested before the wait
  pdl_wait();
  const States<V> st = load_states<V>(s, q);
  if (skip_done && done_bits<V>(st) == (1u << V) - 1) return;
  // fresh lanes (frame queue): slot fields of CNs not processed yet in the
  // frame's first iteration hold the previous frame's c2v and count as 0
  unsigned fr = 0u;
  uint32_t valid = ~0u;
  if constexpr (FRESH) {
    fr = fresh_bits<V>(st);
    valid = fr ? __ldg(fresh + j) : ~0u;
  }
  const int v = t.x;
  Vec<V> acc = ldv<V>(s.L + static_cast<int64_t>(v) * s.B + V * q);
  int field = 0;
  auto add = [&](int slot) {
    const Vec<V> c = ldv<V>(s.c2v + static_cast<int64_t>(slot) * s.B + V * q);
    const bool stale = FRESH && !((valid >> field) & 1u);
#pragma unroll
    for (int i = 0; i < V; ++i) acc.v[i] += (stale && (fr & (1u << i))) ? 0.f : c.v[i];
  };
  const int zero = s.zero_slot;
  auto add_nz = [&](int slot) {
    if (slot != zero) add(slot);
    ++field;
  };
  add_nz(t.y);
  add_nz(t.z);
  add_nz(t.w);
  for (int r = 1; r < vs4 && t.w != zero; ++r) {
    t = __ldg(rec + r);
    add_nz(t.x);
    add_nz(t.y);
    add_nz(t.z);
    add_nz(t.w);
  }
  stv<V>(s.P + static_cast<int64_t>(v) * s.B + V * q, acc);
}

// Syndrome weight per frame (decoder.hpp:129-137) over (CN, V-frame vector) items.
template <int D, bool EXACT, int V>
__global__ void __launch_bounds__(256) stream_syndrome(const int32_t* __restrict__ recs, int CS, int m, ChunkState s) {
  pdl_enter();
  const int64_t QB = s.B / V;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= m * QB) return;
  const int r = static_cast<int>(item / QB);
  const int64_t q = item - r * QB;
  if (done_bits<V>(s, q) == (1u << V) - 1) return;
  const CnRecord<D, EXACT> cr(recs + static_cast<int64_t>(r) * CS, CS);
  unsigned p = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (!cr.has(k)) continue;
    const Vec<V> x = ldv<V>(s.P + static_cast<int64_t>(cr.var(k)) * s.B + V * q);
#pragma unroll
    for (int i = 0; i < V; ++i) p ^= static_cast<unsigned>(x.v[i] < 0.f) << i;
  }
#pragma unroll
  for (int i = 0; i < V; ++i)
    if (p & (1u << i)) atomicAdd(s.weight + V * q + i, 1);
}

// Per-frame bookkeeping after a syndrome test (decoder.hpp:170-177).
__global__ void stream_iter_end(ChunkState s, int iter, int early_stop, int32_t* trace, int max_iters,
                                int64_t frame0) {
  pdl_enter();
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= s.nb || s.done[f]) return;
  const int w = s.weight[f];
  if (trace) trace[(frame0 + f) * max_iters + iter - 1] = w;
  s.iters[f] = iter;
  s.conv[f] = w == 0;
  s.weight[f] = 0;
  if (w == 0 && early_stop) s.done[f] = 1;
}

// Hard decisions (tie -> 0): packed or byte bits, per-frame error counts and
// optional posteriors, transposed [n][B] -> [frames][...] through shared
// memory. Block (32, 8): tile of 32 frames x 256 VNs.
__global__ void stream_bits(int n, const int32_t* __restrict__ pos, ChunkState s, uint8_t* bits, int packed, float* posterior,
                            int64_t frame0) {
  __shared__ unsigned char tile[32][33];
  __shared__ float ptile[32][33];
  const int f0 = blockIdx.y * 32, b0 = blockIdx.x * 32;  // 32 bytes = 256 VNs
  const int nbytes = (n + 7) / 8;
  int errs = 0;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int b = b0 + r, f = f0 + threadIdx.x;
    unsigned byte = 0;
    if (f < s.nb && b < nbytes)
      for (int j = 0; j < 8; ++j) {
        const int v = 8 * b + j;
        if (v < n && s.P[static_cast<int64_t>(__ldg(pos + v)) * s.B + f] < 0.f) byte |= 1u << j;
      }
    tile[threadIdx.x][r] = static_cast<unsigned char>(byte);
    errs += __popc(byte);
  }
  if (errs) atomicAdd(s.berr + f0 + threadIdx.x, errs);
  __syncthreads();
  if (bits) {
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int f = f0 + r;
      if (f >= s.nb) continue;
      const int b = b0 + threadIdx.x;
      if (b >= nbytes) continue;
      const unsigned byte = tile[r][threadIdx.x];
      if (packed) {
        bits[(frame0 + f) * nbytes + b] = static_cast<uint8_t>(byte);
      } else {
        for (int j = 0; j < 8; ++j)
          if (8 * b + j < n) bits[(frame0 + f) * n + 8 * b + j] = static_cast<uint8_t>((byte >> j) & 1u);
      }
    }
  }
  if (posterior) {
    for (int chunk = 0; chunk < 8; ++chunk) {  // 8 sub-tiles of 32 VNs
      const int vb = 8 * b0 + 32 * chunk;
      __syncthreads();
      for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int v = vb + r, f = f0 + threadIdx.x;
        ptile[r][threadIdx.x] = (v < n && f < s.B) ? s.P[static_cast<int64_t>(__ldg(pos + v)) * s.B + f] * kLn2 : 0.f;
      }
      __syncthreads();
      for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int f = f0 + r, v = vb + threadIdx.x;
        if (f < s.nb && v < n) posterior[(frame0 + f) * n + v] = ptile[threadIdx.x][r];
      }
    }
  }
}

__global__ void stream_final(ChunkState s, const DecodeArgs a, int64_t frame0) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  if (f < s.nb) {
    const int it = a.early_stop ? s.iters[f] : a.max_iters;
    if (a.iterations) a.iterations[frame0 + f] = it;
    if (a.converged) a.converged[frame0 + f] = static_cast<uint8_t>(s.conv[f]);
    if (a.bit_errors) a.bit_errors[frame0 + f] = s.berr[f];
    c[0] = 1;
    c[1] = s.berr[f];
    c[2] = s.berr[f] > 0;
    c[3] = s.conv[f];
    c[4] = it;
    c[5] = s.conv[f] ? it : 0;
  }
  if (!a.counters) return;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    unsigned long long v = c[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(a.counters + i, v);
  }
}

// c2v / v2c dumps in CN-major edge order (run_subiterations)
__global__ void stream_dump(const DevGraph g, ChunkState s, float* c2v_out, float* v2c_out, int64_t frame0) {
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= static_cast<int64_t>(g.E) * s.nb) return;
  const int f = static_cast<int>(item % s.nb);
  const int e = static_cast<int>(item / s.nb);
  const float c = s.c2v[static_cast<int64_t>(__ldg(g.edge_slot + e)) * s.B + f];
  if (c2v_out) c2v_out[(frame0 + f) * g.E + e] = c * kLn2;
  if (v2c_out)
    v2c_out[(frame0 + f) * g.E + e] = clamp_bits(s.P[static_cast<int64_t>(__ldg(g.vn_pos + __ldg(g.cols + e))) * s.B + f] - c) * kLn2;
}

// ---- frame queue (early stop): lanes retire and refill at iteration ends
//
// A lane whose frame stops (zero syndrome, decoder.hpp:173-177) or reaches
// max_iters writes that frame's outputs and takes the next frame id from a
// counter, as the reference's pool pulls the next frame (sim.hpp:136-150).
// Only the new frame's channel LLRs are written (L); its stale c2v and
// posteriors are masked by the fresh bits during its first iteration.
// Posteriors are kept in place between syndrome tests (no all-VN re-sum per
// iteration): the hard decision of a posterior within kNearZero of 0 is taken
// from its exact re-sum (P = L + sum c2v, decoder.hpp:162-166). An in-place
// update P += c_new - c_old rounds at most ulp(43 * 2) = 7.6e-6 (messages are
// clamped to 43.3 in log2 units), so 60 updates (30 iterations, two touches
// each) stay below 5e-4: decisions outside kNearZero equal those of exact totals.
constexpr float kNearZero = 2e-3f;  // log2 units

// P = L + c2v over a VN record (the fix-up / totals arithmetic), one lane
__device__ __forceinline__ float exact_posterior(const ChunkState& s, const int4* __restrict__ rec, int vs4,
                                                 int64_t lane) {
  int4 t = __ldg(rec);
  float acc = s.L[static_cast<int64_t>(t.x) * s.B + lane];
  const int zero = s.zero_slot;
  auto add = [&](int slot) {
    if (slot != zero) acc += s.c2v[static_cast<int64_t>(slot) * s.B + lane];
  };
  add(t.y);
  add(t.z);
  add(t.w);
  for (int r = 1; r < vs4 && t.w != zero; ++r) {
    t = __ldg(rec + r);
    add(t.x);
    add(t.y);
    add(t.z);
    add(t.w);
  }
  return acc;
}

// Hard-decision sign words: sw[p][B/32], word 4W + i bit b = sign of lane
// 4 (32 W + b) + i, one warp per (VN position, 128 lanes). B % 128 == 0.
constexpr int kSignRows = 4;  // VN positions per thread: their posterior loads are in flight together
__global__ void __launch_bounds__(256) stream_signs(const int4* __restrict__ all_vn, int vs4, int n, ChunkState s) {
  pdl_launch_next();
  const int64_t QB = s.B / 4;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int blocks = (n + kSignRows - 1) / kSignRows;
  pdl_wait();
  // the parity-failure words of this iteration's syndrome test start empty (stream_syndrome_or)
  if (s.fail && item < s.B / 32) s.fail[item] = 0u;
  if (item >= blocks * QB) return;  // whole warps (QB is a multiple of 32)
  const int p0 = static_cast<int>(item / QB) * kSignRows;
  const int64_t q = item - (p0 / kSignRows) * QB;
  const States<4> st = load_states<4>(s, q);
  const unsigned dn = done_bits<4>(st);
  Vec<4> xs[kSignRows];
#pragma unroll
  for (int r = 0; r < kSignRows; ++r)
    if (dn != 0xfu && p0 + r < n) xs[r] = ldv<4>(s.P + static_cast<int64_t>(p0 + r) * s.B + 4 * q);
#pragma unroll
  for (int r = 0; r < kSignRows; ++r) {
    const int p = p0 + r;
    if (p >= n) break;  // warp-uniform
    Vec<4>& x = xs[r];
    unsigned neg = 0;
    bool near = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) near |= !(dn & (1u << i)) && fabsf(x.v[i]) < kNearZero;
    if (near) {  // rare: the exact totals of the quad (16-byte loads, as stream_vnsum)
      const int4* rec = all_vn + static_cast<int64_t>(p) * vs4;
      int4 t = __ldg(rec);
      Vec<4> acc = ldv<4>(s.L + static_cast<int64_t>(t.x) * s.B + 4 * q);
      const int zero = s.zero_slot;
      auto add = [&](int slot) {
        if (slot == zero) return;
        const Vec<4> c = ldv<4>(s.c2v + static_cast<int64_t>(slot) * s.B + 4 * q);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc.v[i] += c.v[i];
      };
      add(t.y);
      add(t.z);
      add(t.w);
      for (int rr = 1; rr < vs4 && t.w != zero; ++rr) {
        t = __ldg(rec + rr);
        add(t.x);
        add(t.y);
        add(t.z);
        add(t.w);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (fabsf(x.v[i]) < kNearZero) x.v[i] = acc.v[i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (!(dn & (1u << i))) neg |= static_cast<unsigned>(x.v[i] < 0.f) << i;  // tie -> 0 (decoder.hpp:166)
    uint4 w;
    w.x = __ballot_sync(0xffffffffu, neg & 1u);
    w.y = __ballot_sync(0xffffffffu, neg & 2u);
    w.z = __ballot_sync(0xffffffffu, neg & 4u);
    w.w = __ballot_sync(0xffffffffu, neg & 8u);
    if ((threadIdx.x & 31) == 0)
      *reinterpret_cast<uint4*>(s.sw + static_cast<int64_t>(p) * (s.B / 32) + 4 * (q / 32)) = w;
  }
}

// Which lanes fail some parity check (decoder.hpp:129-137, 173): all an early
// stop without a trace needs. One thread per (32 CNs, 128 lanes): the CN's
// parity over 128 lanes is the XOR of its VNs' sign words (one uint4 each),
// ORed over the thread's CNs and then into fail[] (cleared by stream_signs).
// stream_q_iter_end reads a lane's bit as its syndrome weight (0 / 1).
constexpr int kOrRows = 32;
template <int D, bool EXACT>
__global__ void __launch_bounds__(256) stream_syndrome_or(const int32_t* __restrict__ recs, int CS, int m,
                                                          ChunkState s) {
  pdl_launch_next();
  const int cols = static_cast<int>(s.B / 128);  // uint4 columns of the sign words
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int blk = static_cast<int>(item / cols), col = static_cast<int>(item - static_cast<int64_t>(blk) * cols);
  pdl_wait();
  if (item == 0) s.ctl[0] = 0;  // the retire list of this iteration starts empty
  if (blk * kOrRows >= m) return;
  uint4 acc = make_uint4(0u, 0u, 0u, 0u);
  const int r1 = min(m, (blk + 1) * kOrRows);
  for (int r = blk * kOrRows; r < r1; ++r) {
    const CnRecord<D, EXACT> cr(recs + static_cast<int64_t>(r) * CS, CS);
    uint4 par = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (!cr.has(k)) continue;
      const uint4 w = __ldcg(reinterpret_cast<const uint4*>(s.sw + static_cast<int64_t>(cr.var(k)) * (s.B / 32)) + col);
      par.x ^= w.x, par.y ^= w.y, par.z ^= w.z, par.w ^= w.w;
    }
    acc.x |= par.x, acc.y |= par.y, acc.z |= par.z, acc.w |= par.w;
  }
  unsigned* f = s.fail + 4 * col;
  if (acc.x) atomicOr(f, acc.x);
  if (acc.y) atomicOr(f + 1, acc.y);
  if (acc.z) atomicOr(f + 2, acc.z);
  if (acc.w) atomicOr(f + 3, acc.w);
}

// Syndrome weight per lane (decoder.hpp:129-137) from the sign words.
template <int D, bool EXACT>
__global__ void __launch_bounds__(256) stream_syndrome_sw(const int32_t* __restrict__ recs, int CS, int m,
                                                          ChunkState s) {
  pdl_launch_next();
  const int64_t QB = s.B / 4;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = static_cast<int>(item / QB);
  const CnRecord<D, EXACT> cr(recs + static_cast<int64_t>(r < m ? r : 0) * CS, CS);
  pdl_wait();
  if (item == 0) s.ctl[0] = 0;  // the retire list of this iteration starts empty
  if (item >= m * QB) return;
  const int64_t q = item - r * QB;
  if (done_bits<4>(s, q) == 0xfu) return;
  const int b = static_cast<int>(q & 31);
  const int64_t w0 = 4 * (q / 32);
  unsigned par = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (!cr.has(k)) continue;
    const uint4 w = *reinterpret_cast<const uint4*>(s.sw + static_cast<int64_t>(cr.var(k)) * (s.B / 32) + w0);
    par ^= ((w.x >> b) & 1u) | ((w.y >> b) & 1u) << 1 | ((w.z >> b) & 1u) << 2 | ((w.w >> b) & 1u) << 3;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (par & (1u << i)) atomicAdd(s.weight + 4 * q + i, 1);
}

// Lanes [0, nb) hold frames [0, nb); the others idle.
__global__ void stream_q_setup(ChunkState s, int64_t frames) {
  const int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f < s.B) s.frame[f] = f < s.nb ? f : -1;
  if (f == 0) {
    *s.next = static_cast<unsigned long long>(s.nb);
    s.ctl[0] = 0;
    s.ctl[1] = s.nb;
    s.ctl[2] = 0;
  }
}

// Per-lane bookkeeping after the syndrome test (decoder.hpp:166-177).
// reset_wait: the previous iteration refilled every waiting lane.
__global__ void stream_q_iter_end(ChunkState s, int early_stop, int32_t* trace, int max_iters, int reset_wait) {
  pdl_enter();
  const int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f == 0 && reset_wait) s.ctl[2] = 0;
  if (f >= s.B || (s.done[f] & 1)) return;
  // lane f = 4 (32 W + b) + i is bit b of word 4 W + i (the sign-word layout)
  const int w = s.fail ? static_cast<int>((s.fail[4 * (f / 128) + (f & 3)] >> ((f >> 2) & 31)) & 1u) : s.weight[f];
  s.weight[f] = 0;
  const int it = ++s.iters[f];
  if (trace) trace[s.frame[f] * max_iters + it - 1] = w;
  s.conv[f] = w == 0;
  if ((w == 0 && early_stop) || it == max_iters) {
    s.done[f] = kRetiring;
    s.list[atomicAdd(s.ctl, 1)] = static_cast<int>(f);
  } else {
    s.done[f] = kLive;  // a fresh lane's first iteration is over
  }
}

// A lane takes the next frame of the batch (or goes idle): init_state
// (decoder.hpp:39-52) of the new frame writes L only (fresh bits).
__device__ __forceinline__ void stream_q_refill(const DevGraph& g, const ChunkState& s, const float* __restrict__ llr,
                                                int64_t frames, int64_t f, long long* s_new) {
  const int n = g.n;
  if (threadIdx.x == 0) {
    const unsigned long long nf = atomicAdd(s.next, 1ull);
    *s_new = nf < static_cast<unsigned long long>(frames) ? static_cast<long long>(nf) : -1ll;
    s.frame[f] = *s_new;
  }
  __syncthreads();
  const long long nf = *s_new;
  if (nf >= 0) {
    const float* row = llr + nf * n;
    constexpr int U = 4;  // loads of four rounds in flight before the scattered stores
    for (int v0 = threadIdx.x; v0 < n; v0 += U * blockDim.x) {
      int p[U];
      float x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = min(v0 + u * static_cast<int>(blockDim.x), n - 1);
        p[u] = __ldg(g.vn_pos + v);
        x[u] = __ldg(row + v);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v0 + u * static_cast<int>(blockDim.x) < n)
          s.L[static_cast<int64_t>(p[u]) * s.B + f] = clamp_llr(x[u]) * kLog2e;
    }
  }
  if (threadIdx.x == 0) {
    s.iters[f] = 0;
    s.conv[f] = 0;
    s.weight[f] = 0;
    if (nf >= 0) {
      s.done[f] = kFresh;
    } else {
      s.done[f] = kIdle;
      atomicSub(s.ctl + 1, 1);
    }
  }
  __syncthreads();
}

// Outputs of the retiring lanes (sim.hpp:119-123); one block per retiring
// lane at a time. refill: the lanes that stopped now or in earlier iterations
// (the waiting list) take the next frames; otherwise a stopped lane waits, so
// that the iterations in between run the kernels without fresh-frame code.
__global__ void __launch_bounds__(256) stream_q_retire(const DevGraph g, ChunkState s, const DecodeArgs a,
                                                        const float* __restrict__ llr, int64_t frames, int refill) {
  pdl_enter();
  __shared__ int s_errs;
  __shared__ long long s_new;
  const int n = g.n, nbytes = (n + 7) / 8;
  const int count = s.ctl[0], waiting = refill ? s.ctl[2] : 0;
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  for (int e = blockIdx.x; e < count; e += gridDim.x) {
    const int64_t f = s.list[e];
    const int64_t fr = s.frame[f];
    const int64_t w0 = 4 * (f / 128) + (f & 3);  // sign word of lane f, bit (f / 4) % 32
    const int bit = static_cast<int>((f >> 2) & 31);
    if (threadIdx.x == 0) s_errs = 0;
    __syncthreads();
    int errs = 0;
    for (int b = threadIdx.x; b < nbytes; b += blockDim.x) {
      // the eight positions, then the eight sign words, requested together (one at a time this
      // loop was sixteen dependent L2 / DRAM latencies per byte)
      int p[8];
      unsigned w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) p[j] = __ldg(g.vn_pos + min(8 * b + j, n - 1));
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = __ldcg(s.sw + static_cast<int64_t>(p[j]) * (s.B / 32) + w0);
      unsigned byte = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * b + j < n) byte |= ((w[j] >> bit) & 1u) << j;
      if (a.bits) {
        if (a.bits_packed) {
          a.bits[fr * nbytes + b] = static_cast<uint8_t>(byte);
        } else {
          for (int j = 0; j < 8 && 8 * b + j < n; ++j) a.bits[fr * n + 8 * b + j] = static_cast<uint8_t>((byte >> j) & 1u);
        }
      }
      errs += __popc(byte);
    }
    if (a.posterior)  // exact totals (decoder.hpp:162-165) of the stopped frame
      for (int v = threadIdx.x; v < n; v += blockDim.x) {
        const int p = __ldg(g.vn_pos + v);
        a.posterior[fr * n + v] =
            exact_posterior(s, reinterpret_cast<const int4*>(g.all_vn_rec) + static_cast<int64_t>(p) * g.vs4, g.vs4, f) *
            kLn2;
      }
    if (errs) atomicAdd(&s_errs, errs);
    __syncthreads();  // every read of this lane's state is done before the refill
    if (threadIdx.x == 0) {
      const int it = s.iters[f], cv = s.conv[f], be = s_errs;
      if (a.iterations) a.iterations[fr] = it;
      if (a.converged) a.converged[fr] = static_cast<uint8_t>(cv);
      if (a.bit_errors) a.bit_errors[fr] = be;
      c[0] += 1;
      c[1] += be;
      c[2] += be > 0;
      c[3] += cv;
      c[4] += it;
      c[5] += cv ? it : 0;
      if (!refill) {
        s.done[f] = kWaiting;
        s.wlist[atomicAdd(s.ctl + 2, 1)] = static_cast<int>(f);
      }
    }
    if (refill) stream_q_refill(g, s, llr, frames, f, &s_new);
  }
  for (int e = blockIdx.x; e < waiting; e += gridDim.x) stream_q_refill(g, s, llr, frames, s.wlist[e], &s_new);
  if (threadIdx.x == 0 && a.counters)
    for (int i = 0; i < 6; ++i)
      if (c[i]) atomicAdd(a.counters + i, c[i]);
}

struct StreamKernels {
  void (*cn)(const int32_t*, int, int, ChunkState, const uint32_t*);
  void (*syn)(const int32_t*, int, int, ChunkState);
  void (*vnsum)(const int4*, int, int, ChunkState, int, const uint32_t*);
  void (*syn_sw)(const int32_t*, int, int, ChunkState);  // frame queue (V = 4)
  // frame queue: the same kernels with the fresh-frame code compiled in
  void (*cn_fresh)(const int32_t*, int, int, ChunkState, const uint32_t*);
  void (*vnsum_fresh)(const int4*, int, int, ChunkState, int, const uint32_t*);
  // TMA-staged CN kernel (regular rows of degree 3 / 6, four frames per thread), or null
  void (*cn_tma)(const int32_t*, int, ChunkState);
  int tma_smem;
  void (*syn_or)(const int32_t*, int, int, ChunkState);  // frame queue without a trace
};

template <int D, bool EXACT, int V>
StreamKernels pick_dv() {
  StreamKernels k{stream_cn<D, EXACT, V, false>, stream_syndrome<D, EXACT, V>, stream_vnsum<V, false>,
                  stream_syndrome_sw<D, EXACT>,  stream_cn<D, EXACT, V, true>, stream_vnsum<V, true>,
                  nullptr,                       0,
                  stream_syndrome_or<D, EXACT>};
  if constexpr (EXACT && D <= 6 && V == 4) {
    k.cn_tma = stream_cn_tma<D>;
    k.tma_smem = 2 * D * kTmaRowBytes;
  }
  return k;
}

template <int V>
StreamKernels pick_v(const DevGraph& g) {
  switch (cn_bucket(g.max_cdeg, g.cregular)) {
    case 3: return pick_dv<3, true, V>();
    case 6: return pick_dv<6, true, V>();
    case 8: return pick_dv<8, false, V>();
    case 16: return pick_dv<16, false, V>();
    default: return {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr};
  }
}

// frames per thread: 4 by default (16-byte accesses); LDPCB_STREAM_V = 1 / 2
// (A/B: more threads per launch for small chunks)
int stream_lanes() {
  const char* e = std::getenv("LDPCB_STREAM_V");
  const int v = e ? std::atoi(e) : 4;
  return (v == 1 || v == 2) ? v : 4;
}

StreamKernels pick(const DevGraph& g) {
  switch (stream_lanes()) {
    case 1: return pick_v<1>(g);
    case 2: return pick_v<2>(g);
    default: return pick_v<4>(g);
  }
}

size_t chunk_bytes_per_frame(const DevGraph& g) {
  return 4ull * (static_cast<size_t>(g.n_slots) + 2ull * g.n) + 20;
}

unsigned blocks_for(int64_t items, int tpb) { return static_cast<unsigned>((items + tpb - 1) / tpb); }

// LDPCB_STREAM_PDL=0 launches the per-group kernels without the programmatic
// dependency attribute (A/B); griddepcontrol is then a no-op.
bool stream_pdl() {
  const char* e = std::getenv("LDPCB_STREAM_PDL");
  return !e || std::atoi(e) != 0;
}

// LDPCB_STREAM_TMA=1 selects the TMA-staged CN kernel (bit-identical outputs;
// measured 1 % slower than the LDG.128 kernel on C5 n = 64800: 65.3 against 64.6 ms per step)
bool stream_tma() {
  const char* e = std::getenv("LDPCB_STREAM_TMA");
  return e && std::atoi(e) != 0;
}

template <class... KArgs, class... Args>
cudaError_t launch_pdl_smem(void (*k)(KArgs...), unsigned blocks, int tpb, int smem, cudaStream_t st, bool pdl,
                            Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(tpb);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), unsigned blocks, int tpb, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(tpb);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace

Plan plan_stream(const DevGraph& g, int64_t frames) {
  Plan p;
  if (!pick(g).cn) return p;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 16ull << 30;
  const size_t budget = std::min<size_t>(free_b / 3, 24ull << 30);
  int64_t B = static_cast<int64_t>(budget / chunk_bytes_per_frame(g)) / 128 * 128;
  B = std::min<int64_t>(B, 16384);
  if (const char* e = std::getenv("LDPCB_STREAM_CHUNK")) B = std::min<int64_t>(B, std::max(4, std::atoi(e)) / 4 * 4);
  const int64_t need = (std::max<int64_t>(frames, 1) + 3) / 4 * 4;
  B = std::min(B, need);
  if (B < 4) return p;
  p.kernel = 2;
  p.fpc = static_cast<int>(B);  // frames per chunk
  p.threads = 256;
  p.smem = 0;
  p.degree_bucket = cn_bucket(g.max_cdeg, g.cregular);
  p.ctas = (frames + B - 1) / B;  // chunks
  return p;
}

namespace {

// One sequence of chunks on one stream.
int launch_stream_one(const DevGraph& g, const DecodeArgs& a, cudaStream_t st, const Plan& p) {
  const StreamKernels K = pick(g);
  const int64_t B = p.fpc;
  ChunkState s;
  s.B = B;
  s.zero_slot = g.n_slots - 1;
  const size_t state_bytes = 4ull * (static_cast<size_t>(g.n_slots) + 2ull * g.n) * B;
  char* mem = nullptr;
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&mem), state_bytes + 5 * 4 * B + 256, st);
  if (err != cudaSuccess) return static_cast<int>(err);
  s.c2v = reinterpret_cast<float*>(mem);
  s.P = s.c2v + static_cast<size_t>(g.n_slots) * B;
  s.L = s.P + static_cast<size_t>(g.n) * B;
  s.done = reinterpret_cast<int*>(s.L + static_cast<size_t>(g.n) * B);
  s.weight = s.done + B;
  s.iters = s.weight + B;
  s.conv = s.iters + B;
  s.berr = s.conv + B;
  const int tpb = 256;
  const int64_t QB = B / stream_lanes();
  const bool dump = a.max_subiters > 0;
  const bool pdl = stream_pdl();
  // TMA-staged CN kernel: packed regular-row records, whole CTAs of quads
  bool use_tma = K.cn_tma && g.cs == 4 && stream_lanes() == 4 && QB % kTmaQuads == 0 && stream_tma();
  if (use_tma && cudaFuncSetAttribute(reinterpret_cast<const void*>(K.cn_tma),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, K.tma_smem) != cudaSuccess)
    use_tma = false;
  int launches = 0;
  for (int64_t f0 = 0; f0 < a.frames && err == cudaSuccess; f0 += B) {
    s.nb = static_cast<int>(std::min<int64_t>(B, a.frames - f0));
    err = cudaMemsetAsync(s.c2v, 0, 4ull * g.n_slots * B, st);
    if (err != cudaSuccess) break;
    stream_init<<<dim3((g.n + 31) / 32, static_cast<unsigned>((B + 31) / 32)), dim3(32, 8), 0, st>>>(
        g.n, g.vn_pos, a.llr + f0 * g.n, s);
    ++launches;
    if (a.trace) {
      err = cudaMemsetAsync(a.trace + f0 * a.max_iters, 0xff, 4ull * s.nb * a.max_iters, st);
      if (err != cudaSuccess) break;
    }
    int sub = 0;
    bool stop = false;
    for (int iter = 1; iter <= a.max_iters && !stop && err == cudaSuccess; ++iter) {
      for (int grp = 0; grp < g.G; ++grp) {
        if (dump && sub == a.max_subiters) {
          stop = true;
          break;
        }
        ++sub;
        const int c0 = g.h_cn_off[grp], cn = g.h_cn_off[grp + 1] - c0;
        if (cn > 0 && use_tma) {
          err = launch_pdl_smem(K.cn_tma, static_cast<unsigned>(cn * (QB / kTmaQuads)), kTmaQuads, K.tma_smem, st,
                                pdl, g.cn_rec + static_cast<size_t>(c0) * g.cs, cn, s);
          ++launches;
        } else if (cn > 0) {
          err = launch_pdl(K.cn, blocks_for(cn * QB, tpb), tpb, st, pdl, g.cn_rec + static_cast<size_t>(c0) * g.cs,
                           g.cs, cn, s, static_cast<const uint32_t*>(nullptr));
          ++launches;
        }
        const int x0 = g.h_fix_off[grp], xn = g.h_fix_off[grp + 1] - x0;
        if (xn > 0 && err == cudaSuccess) {
          err = launch_pdl(K.vnsum, blocks_for(xn * QB, tpb), tpb, st, pdl,
                           reinterpret_cast<const int4*>(g.fix_rec) + static_cast<size_t>(x0) * g.vs4, g.vs4, xn,
                           s, 1, static_cast<const uint32_t*>(nullptr));
          ++launches;
        }
        if (err != cudaSuccess) {
          stop = true;
          break;
        }
      }
      if (stop || dump) continue;
      const bool check = a.early_stop || a.trace || iter == a.max_iters;
      if (g.recompute && (check || !a.lazy_totals)) {
        err = launch_pdl(K.vnsum, blocks_for(g.n * QB, tpb), tpb, st, pdl,
                         reinterpret_cast<const int4*>(g.all_vn_rec), g.vs4, g.n, s, 1,
                         static_cast<const uint32_t*>(nullptr));
        ++launches;
      }
      if (!check || err != cudaSuccess) continue;
      err = launch_pdl(K.syn, blocks_for(g.m * QB, tpb), tpb, st, pdl, g.all_rec, g.cs, g.m, s);
      if (err == cudaSuccess)
        err = launch_pdl(stream_iter_end, blocks_for(s.nb, tpb), tpb, st, pdl, s, iter, a.early_stop, a.trace,
                         a.max_iters, f0);
      launches += 2;
    }
    if (dump) {
      if (g.recompute)
        K.vnsum<<<blocks_for(g.n * QB, tpb), tpb, 0, st>>>(reinterpret_cast<const int4*>(g.all_vn_rec), g.vs4, g.n,
                                                           s, 0, nullptr);
      stream_dump<<<blocks_for(static_cast<int64_t>(g.E) * s.nb, tpb), tpb, 0, st>>>(g, s, a.c2v_out, a.v2c_out,
                                                                                      f0);
      launches += 2;
    } else {
      const int nbytes = (g.n + 7) / 8;
      stream_bits<<<dim3((nbytes + 31) / 32, static_cast<unsigned>((B + 31) / 32)), dim3(32, 8), 0, st>>>(
          g.n, g.vn_pos, s, a.bits, a.bits_packed, a.posterior, f0);
      stream_final<<<blocks_for(s.nb, tpb), tpb, 0, st>>>(s, a, f0);
      launches += 2;
    }
    if (err == cudaSuccess) err = cudaGetLastError();
  }
  note_launches(launches);
  cudaFreeAsync(mem, st);
  return static_cast<int>(err);
}

// LDPCB_STREAM_QUEUE=0 decodes early-stop batches chunk by chunk (every
// chunk runs until its slowest frame stops; A/B and tests)
bool stream_queue_enabled() {
  const char* e = std::getenv("LDPCB_STREAM_QUEUE");
  return !e || std::atoi(e) != 0;
}

// iterations between refills of the frame queue's lanes
int stream_refill_every() {
  const char* e = std::getenv("LDPCB_STREAM_REFILL");
  const int v = e ? std::atoi(e) : 4;
  return v < 1 ? 1 : v;
}

// Early stop from a frame queue: B lanes (a multiple of 128) decode until
// every frame of the batch has stopped. Per iteration: the groups' CN and
// fix-up kernels, then sign words, syndrome weights, per-lane bookkeeping,
// and retire + refill. The host reads the number of decoding lanes one
// iteration behind, so the device never waits for the host.
int launch_stream_queue(const DevGraph& g, const DecodeArgs& a, cudaStream_t st, int64_t B0) {
  const StreamKernels K = pick_v<4>(g);
  // lanes: a sixteenth of the batch (so that lanes are refilled many times
  // and the tail, where the last frames run on alone, stays short: 8 % of a
  // 65536-frame batch on 8192 lanes, 4 % on 4096) between 2048 and 8192
  // (kernel efficiency); LDPCB_STREAM_CHUNK caps it
  const int64_t want = std::min<int64_t>(std::max<int64_t>((a.frames / 16 + 127) / 128 * 128, 2048), 8192);
  const int64_t B = (std::min<int64_t>(std::min(B0, want), a.frames) + 127) / 128 * 128;
  ChunkState s;
  s.B = B;
  s.nb = static_cast<int>(std::min<int64_t>(B, a.frames));
  s.zero_slot = g.n_slots - 1;
  const size_t state = 4ull * (static_cast<size_t>(g.n_slots) + 2ull * g.n) * B;
  const size_t lanes = 5 * 4 * B + 8 * B + 4 * B + 4 * B + 64;
  const size_t signs = 4ull * g.n * (B / 32);
  char* mem = nullptr;
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&mem), state + lanes + signs + 4 * (B / 32) + 16, st);
  if (err != cudaSuccess) return static_cast<int>(err);
  s.c2v = reinterpret_cast<float*>(mem);
  s.P = s.c2v + static_cast<size_t>(g.n_slots) * B;
  s.L = s.P + static_cast<size_t>(g.n) * B;
  s.done = reinterpret_cast<int*>(s.L + static_cast<size_t>(g.n) * B);
  s.weight = s.done + B;
  s.iters = s.weight + B;
  s.conv = s.iters + B;
  s.berr = s.conv + B;
  s.frame = reinterpret_cast<int64_t*>(s.berr + B);
  s.list = reinterpret_cast<int*>(s.frame + B);
  s.wlist = s.list + B;
  s.ctl = s.wlist + B;
  s.next = reinterpret_cast<unsigned long long*>(s.ctl + 8);
  s.sw = reinterpret_cast<unsigned*>(mem + state + lanes);
  // without a trace only "does any check fail" is needed per lane (stream_syndrome_or)
  if (!a.trace && K.syn_or) s.fail = reinterpret_cast<unsigned*>(mem + state + lanes + signs);
  // the host's view of the decoding-lane count, one slot per parity of the iteration
  thread_local int* host_live = nullptr;
  if (!host_live && cudaMallocHost(reinterpret_cast<void**>(&host_live), 2 * sizeof(int)) != cudaSuccess) {
    host_live = nullptr;
    cudaFreeAsync(mem, st);
    return static_cast<int>(cudaErrorMemoryAllocation);
  }
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (auto& e : ev)
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  const int tpb = 256;
  const int64_t QB = B / 4;
  const bool pdl = stream_pdl();
  int launches = 0;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (err == cudaSuccess) err = cudaMemsetAsync(s.c2v, 0, 4ull * g.n_slots * B, st);
  if (err == cudaSuccess && a.trace) err = cudaMemsetAsync(a.trace, 0xff, 4ull * a.frames * a.max_iters, st);
  if (err == cudaSuccess) {
    stream_init<<<dim3((g.n + 31) / 32, static_cast<unsigned>((B + 31) / 32)), dim3(32, 8), 0, st>>>(g.n, g.vn_pos,
                                                                                                     a.llr, s);
    stream_q_setup<<<blocks_for(B, tpb), tpb, 0, st>>>(s, a.frames);
    launches += 2;
    err = cudaGetLastError();
  }
  const auto* fix4 = reinterpret_cast<const int4*>(g.fix_rec);
  // Lanes are refilled every `every`-th iteration (LDPCB_STREAM_REFILL, default 4): only the iteration
  // after a refill holds fresh lanes and needs the kernels with the fresh-frame code.
  const int every = stream_refill_every();
  bool refilled = false;  // the previous iteration ended with a refill
  for (int64_t it = 0; err == cudaSuccess; ++it) {
    const bool fresh = refilled;
    for (int grp = 0; grp < g.G && err == cudaSuccess; ++grp) {
      const int c0 = g.h_cn_off[grp], cn = g.h_cn_off[grp + 1] - c0;
      if (cn > 0) {
        err = launch_pdl(fresh ? K.cn_fresh : K.cn, blocks_for(cn * QB, tpb), tpb, st, pdl,
                         g.cn_rec + static_cast<size_t>(c0) * g.cs, g.cs, cn, s,
                         fresh ? g.cn_fresh + c0 : static_cast<const uint32_t*>(nullptr));
        ++launches;
      }
      const int x0 = g.h_fix_off[grp], xn = g.h_fix_off[grp + 1] - x0;
      if (xn > 0 && err == cudaSuccess) {
        err = launch_pdl(fresh ? K.vnsum_fresh : K.vnsum, blocks_for(xn * QB, tpb), tpb, st, pdl,
                         fix4 + static_cast<size_t>(x0) * g.vs4, g.vs4, xn, s, 1,
                         fresh ? g.fix_fresh + x0 : static_cast<const uint32_t*>(nullptr));
        ++launches;
      }
    }
    if (err != cudaSuccess) break;
    err = launch_pdl(stream_signs, blocks_for((g.n + kSignRows - 1) / kSignRows * QB, tpb), tpb, st, pdl,
                     reinterpret_cast<const int4*>(g.all_vn_rec), g.vs4, g.n, s);
    if (err == cudaSuccess && s.fail)
      err = launch_pdl(K.syn_or, blocks_for(static_cast<int64_t>((g.m + kOrRows - 1) / kOrRows) * (B / 128), tpb), tpb,
                       st, pdl, g.all_rec, g.cs, g.m, s);
    else if (err == cudaSuccess)
      err = launch_pdl(K.syn_sw, blocks_for(g.m * QB, tpb), tpb, st, pdl, g.all_rec, g.cs, g.m, s);
    if (err == cudaSuccess)
      err = launch_pdl(stream_q_iter_end, blocks_for(B, tpb), tpb, st, pdl, s, a.early_stop, a.trace, a.max_iters,
                       refilled ? 1 : 0);
    refilled = (it + 1) % every == 0;
    if (err == cudaSuccess)
      err = launch_pdl(stream_q_retire, static_cast<unsigned>(4 * sms), tpb, st, pdl, g, s, a, a.llr, a.frames,
                       refilled ? 1 : 0);
    launches += 4;
    const int k = static_cast<int>(it & 1);
    if (err == cudaSuccess) err = cudaMemcpyAsync(host_live + k, s.ctl + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaEventRecord(ev[k], st);
    if (err != cudaSuccess || it == 0) continue;
    // the previous iteration's count: zero means this iteration found every
    // lane idle (its kernels exit at once) and the batch is done
    err = cudaEventSynchronize(ev[k ^ 1]);
    if (err == cudaSuccess && host_live[k ^ 1] == 0) break;
  }
  note_launches(launches);
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  cudaFreeAsync(mem, st);
  return static_cast<int>(err);
}

}  // namespace

int launch_stream(const DevGraph& g, const DecodeArgs& a, void* stream_v, Plan* used) {
  const Plan p = plan_stream(g, a.frames);
  if (used) *used = p;
  if (p.kernel == 0) return static_cast<int>(cudaErrorInvalidConfiguration);
  if (a.frames <= 0) return 0;
  // early stop: frames stream through the lanes (frame queue) when the tables
  // allow it (every CN grouped, every VN touched, stride-4 lanes)
  if (a.early_stop && a.max_subiters == 0 && g.covers && g.cn_fresh && g.fix_fresh && stream_lanes() == 4 &&
      stream_queue_enabled())
    return launch_stream_queue(g, a, static_cast<cudaStream_t>(stream_v), p.fpc);
  return launch_stream_one(g, a, static_cast<cudaStream_t>(stream_v), p);
}

}  // namespace ldpcb
