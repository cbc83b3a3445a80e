// direct.cu -- posterior-free SMEM-resident decoder for check-regular
// degree-6 codes whose VNs have degree <= 3 (BASELINE configs 1, 2, 5: the
// (3,6) n=1008 code) under schedules whose groups fit one CN item per thread.
//
// State per frame pair (two frames per 8-byte cell, host.hpp DirectTables):
// one c2v cell per edge, one L cell per VN (clamped channel LLR, log2 units).
// A CN item of group g (decoder.hpp:112-127) forms, for each of its six VNs,
//     v2c_k = L_v + c2v_a + c2v_b        (var_update, decoder.hpp:91-105)
// from the OTHER two edges of v, runs the exclusion boxplus (check_update,
// decoder.hpp:59-87; common.cuh) and overwrites its own six c2v cells. There
// is no posterior array: nothing is updated in place, no fix-up re-sum and no
// exact-totals pass exist, and every v2c is exact to two fp32 additions.
// Posteriors are formed only where the reference forms them: for the hard
// decision / syndrome test (decoder.hpp:162-171) and the outputs.
//
// Jacobi inside a group: a CN of the group may read a cell that another CN of
// the same group overwrites (a VN shared by both). Every thread therefore
// arrives on an mbarrier once its own loads have returned and waits on it
// right before its first store -- by then (hundreds of cycles of boxplus
// later) all loads of the group have long been issued, so the wait costs
// nothing -- and one __syncthreads per group orders the stores before the
// next group's loads. A group is one CN item per thread (the launch plan
// guarantees it), so no item of a group can start after another has stored.
//
// Persistent CTAs take frames from a queue (one atomicAdd per frame): at an
// iteration boundary a slot whose frame stopped (zero syndrome with early
// stop, or max_iters) writes its outputs and is refilled; slots are
// independent lanes, so outputs do not depend on the slot a frame used.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "kernels.cuh"

namespace ldpcb {
namespace {

using namespace dev;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// `tie` is a value the wait must follow in program order (the first boxplus
// output): without it the compiler hoists the wait above the arithmetic.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, f32x2& tie) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LDPCB_WAIT:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "@p bra LDPCB_DONE;\n"
      "bra LDPCB_WAIT;\n"
      "LDPCB_DONE:\n"
      "}\n"
      : "+l"(tie)
      : "r"(bar), "r"(parity)
      : "memory");
}

template <int NG>
struct DirectCfg {
  static constexpr int kMaxThreads = NG == 1 ? 96 : (NG == 2 ? 192 : 256);
  static constexpr int kMinBlocks = NG == 1 ? 6 : (NG == 2 ? 3 : 2);
};

// the twelve words of a CN record (host.hpp DirectTables)
struct DRec {
  int4 a, b, c;
  __device__ __forceinline__ void load(const int32_t* __restrict__ p) {
    const int4* q = reinterpret_cast<const int4*>(p);
    a = __ldg(q);
    b = __ldg(q + 1);
    c = __ldg(q + 2);
  }
  __device__ __forceinline__ void pin() {
    asm volatile("" : "+r"(a.x), "+r"(a.y), "+r"(a.z), "+r"(a.w));
    asm volatile("" : "+r"(b.x), "+r"(b.y), "+r"(b.z), "+r"(b.w));
    asm volatile("" : "+r"(c.x), "+r"(c.y), "+r"(c.z), "+r"(c.w));
  }
};

__device__ __forceinline__ f32x2 ldc(const char* base, uint32_t off) {
  return *reinterpret_cast<const f32x2*>(base + off);
}
__device__ __forceinline__ uint32_t lo16(int w) { return static_cast<uint32_t>(w) & 0xffffu; }
__device__ __forceinline__ uint32_t hi16(int w) { return static_cast<uint32_t>(w) >> 16; }

// SPLIT: the split arrive / wait barrier described above; otherwise a plain
// __syncthreads between the loads and the boxplus (A/B).
template <int NG, bool SPLIT>
__global__ void __launch_bounds__(DirectCfg<NG>::kMaxThreads, DirectCfg<NG>::kMinBlocks)
    decode_direct(const DevGraph g, const DecodeArgs a, unsigned long long* queue) {
  constexpr int FPC = 2 * NG;
  extern __shared__ __align__(16) char dsm[];
  __shared__ long long s_frame[FPC];
  __shared__ int s_done[FPC], s_weight[FPC], s_iters[FPC], s_conv[FPC], s_berr[FPC];
  __shared__ unsigned long long s_cnt[6];
  __shared__ __align__(8) unsigned long long s_bar;
  __shared__ int s_active, s_retiring;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = g.n, m = g.m, E = g.E;
  const uint32_t pair_bytes = static_cast<uint32_t>(g.d_cells) * 8u;
  const uint32_t l_off = static_cast<uint32_t>(g.d_l_base) * 8u;
  const int npad = (n + 15) & ~15;
  uint8_t* const s_hd = reinterpret_cast<uint8_t*>(dsm + NG * pair_bytes);  // [NG][npad] sign bits, bit h = frame h
  int2* const s_go = reinterpret_cast<int2*>(dsm + NG * pair_bytes + ((NG * npad + 15) & ~15));
  const int nb = (n + 7) >> 3;
  const uint32_t bar = smem_addr(&s_bar);
  const bool check = a.early_stop || a.trace;
  const bool dump = a.max_subiters > 0;

  // slot ff = frame half h = ff & 1 of pair ff >> 1
  auto slot_base = [&](int ff) { return dsm + (ff >> 1) * pair_bytes + (ff & 1) * 4; };
  // init_state (decoder.hpp:39-52): L = clamp(llr), every c2v = 0 (f < 0: idle slot)
  auto load_slot = [&](int ff, long long f) {
    char* const sb = slot_base(ff);
    if (f >= 0) {
      const float* llr = a.llr + f * n;
      if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(a.llr) & 15) == 0) {
        const float4* l4 = reinterpret_cast<const float4*>(llr);
        for (int b = tid; b < n / 4; b += nt) {
          const float4 x = __ldg(l4 + b);
          const int4 p = __ldg(reinterpret_cast<const int4*>(g.d_vn_pos) + b);
          *reinterpret_cast<float*>(sb + l_off + p.x * 8) = clamp_llr(x.x) * kLog2e;
          *reinterpret_cast<float*>(sb + l_off + p.y * 8) = clamp_llr(x.y) * kLog2e;
          *reinterpret_cast<float*>(sb + l_off + p.z * 8) = clamp_llr(x.z) * kLog2e;
          *reinterpret_cast<float*>(sb + l_off + p.w * 8) = clamp_llr(x.w) * kLog2e;
        }
      } else {
        for (int i = tid; i < n; i += nt)
          *reinterpret_cast<float*>(sb + l_off + __ldg(g.d_vn_pos + i) * 8) = clamp_llr(__ldg(llr + i)) * kLog2e;
      }
      if (a.trace)
        for (int i = tid; i < a.max_iters; i += nt) a.trace[f * a.max_iters + i] = -1;
    } else {
      for (int i = tid; i < n; i += nt) *reinterpret_cast<float*>(sb + l_off + i * 8) = kClampB;
    }
    for (int i = tid; i < g.d_l_base; i += nt) *reinterpret_cast<float*>(sb + i * 8) = 0.f;
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
  if (tid == 0) mbar_init(bar, nt);
  for (int i = tid; i < g.G; i += nt) s_go[i] = make_int2(__ldg(g.d_cn_off + i), __ldg(g.d_cn_off + i + 1));
  {  // every cell zero (the zero cell and the padding cells stay zero)
    float4* z = reinterpret_cast<float4*>(dsm);
    for (int i = tid; i < static_cast<int>(NG * pair_bytes / 16); i += nt) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  {
    bool any = false;
    for (int ff = 0; ff < FPC; ++ff) any |= s_frame[ff] >= 0;
    if (!any) return;  // the queue was empty when this CTA started
  }
  for (int ff = 0; ff < FPC; ++ff) load_slot(ff, s_frame[ff]);
  __syncthreads();

  // this thread's item of a group with cn CNs: pair p = tid / cn, CN j = tid % cn
  auto item_of = [&](int cn, int& p, int& j) {
    p = 0;
    j = tid;
    if constexpr (NG >= 2)
      if (j >= cn) j -= cn, p = 1;
    if constexpr (NG >= 3)
      if (j >= cn) j -= cn, p = 2;
    return j < cn;
  };
  DRec next_rec;
  int2 go = s_go[0];
  {
    int p, j;
    if (item_of(go.y - go.x, p, j)) next_rec.load(g.d_cn_rec + static_cast<size_t>(go.x + j) * 12);
  }
  uint32_t parity = 0;
  int it_cta = 0, sub = 0;

  for (;;) {
    // one iteration for every slot (decoder.hpp:157-160)
    for (int grp = 0; grp < g.G; ++grp) {
      if (dump && sub == a.max_subiters) goto dump_state;
      ++sub;
      const int cn = go.y - go.x;
      const int2 ngo = s_go[grp + 1 < g.G ? grp + 1 : 0];
      int p, j;
      const bool has = item_of(cn, p, j);
      const char* const pb = dsm + p * pair_bytes;
      const DRec cur = next_rec;
      {  // the next group's record, a whole group before it is needed
        int pn, jn;
        if (item_of(ngo.y - ngo.x, pn, jn)) next_rec.load(g.d_cn_rec + static_cast<size_t>(ngo.x + jn) * 12);
      }
      f32x2 x[6];
      uint32_t own[6];
      if (has) {
        const int w[12] = {cur.a.x, cur.a.y, cur.a.z, cur.a.w, cur.b.x, cur.b.y,
                           cur.b.z, cur.b.w, cur.c.x, cur.c.y, cur.c.z, cur.c.w};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          own[k] = lo16(w[2 * k]);
          const f32x2 l = ldc(pb, hi16(w[2 * k]));
          const f32x2 ca = ldc(pb, lo16(w[2 * k + 1]));
          const f32x2 cb = ldc(pb, hi16(w[2 * k + 1]));
          x[k] = add2(add2(l, ca), cb);
        }
      }
      if constexpr (SPLIT) {
        mbar_arrive(bar);  // release: ordered after this thread's loads above
      } else {
        __syncthreads();
      }
      if (has) {
        boxplus_row_x2<6, true>(x, 6, [&](int k, f32x2 c) {
          if constexpr (SPLIT)
            if (k == 5) mbar_wait(bar, parity, c);  // the first output: every load of the group is done
          *reinterpret_cast<f32x2*>(const_cast<char*>(pb) + own[k]) = c;
        });
      }
      parity ^= 1u;
      __syncthreads();
      next_rec.pin();
      go = ngo;
    }
    if (dump) continue;
    ++it_cta;
    if (!check && it_cta < a.max_iters) continue;
    // ---- hard decisions (tie -> 0) from the totals L + sum c2v in ascending
    // CN order (decoder.hpp:162-166), one sign bit per frame in s_hd
    for (int i = tid; i < NG * n; i += nt) {
      const int p = NG == 1 ? 0 : i / n, pos = i - p * n;
      const char* const pb = dsm + p * pair_bytes;
      const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_vn_rec) + pos);
      f32x2 t = ldc(pb, l_off + pos * 8);
      t = add2(t, ldc(pb, lo16(r.x)));
      t = add2(t, ldc(pb, hi16(r.x)));
      t = add2(t, ldc(pb, lo16(r.y)));
      s_hd[p * npad + pos] = static_cast<uint8_t>((lo2(t) < 0.f ? 1u : 0u) | (hi2(t) < 0.f ? 2u : 0u));
    }
    __syncthreads();
    // ---- syndrome weight (decoder.hpp:129-137)
#pragma unroll
    for (int p = 0; p < NG; ++p) {
      int w0 = 0, w1 = 0;
      const uint8_t* hd = s_hd + p * npad;
      for (int r = tid; r < m; r += nt) {
        const int4 q = __ldg(reinterpret_cast<const int4*>(g.d_all_cn) + r);
        const unsigned x = hd[lo16(q.x)] ^ hd[hi16(q.x)] ^ hd[lo16(q.y)] ^ hd[hi16(q.y)] ^ hd[lo16(q.z)] ^ hd[hi16(q.z)];
        w0 += x & 1u;
        w1 += (x >> 1) & 1u;
      }
      if (w0) atomicAdd(&s_weight[2 * p], w0);
      if (w1) atomicAdd(&s_weight[2 * p + 1], w1);
    }
    __syncthreads();
    if (tid == 0) {
      int retiring = 0;
      for (int ff = 0; ff < FPC; ++ff) {
        if (s_done[ff]) continue;
        const int w = s_weight[ff];
        const int it = check ? ++s_iters[ff] : (s_iters[ff] = it_cta);
        if (a.trace) a.trace[s_frame[ff] * a.max_iters + it - 1] = w;
        s_conv[ff] = w == 0;
        if ((w == 0 && a.early_stop) || it >= a.max_iters) {  // decoder.hpp:173-177
          s_done[ff] = 2;                                       // retiring
          ++retiring;
        }
      }
      int active = 0;
      for (int ff = 0; ff < FPC; ++ff) {
        s_weight[ff] = 0;
        active += s_done[ff] != 1;
      }
      s_retiring = retiring;
      s_active = active;
    }
    __syncthreads();
    if (s_retiring == 0) {
      if (s_active == 0) break;
      continue;
    }
    // ---- outputs of the frames that stopped (sim.hpp:119-123), then refill
    for (int ff = 0; ff < FPC; ++ff) {
      if (s_done[ff] != 2) continue;
      const long long f = s_frame[ff];
      const uint8_t* hd = s_hd + (ff >> 1) * npad;
      const int h = ff & 1;
      int errs = 0;
      if (a.bits && a.bits_packed) {
        for (int b = tid; b < nb; b += nt) {
          unsigned byte = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int v = b * 8 + q;
            if (v < n) byte |= ((hd[__ldg(g.d_vn_pos + v)] >> h) & 1u) << q;
          }
          a.bits[f * nb + b] = static_cast<uint8_t>(byte);
          errs += __popc(byte);
        }
      } else if (a.bits || a.counters || a.bit_errors) {
        for (int v = tid; v < n; v += nt) {
          const int bit = (hd[__ldg(g.d_vn_pos + v)] >> h) & 1;
          if (a.bits) a.bits[f * n + v] = static_cast<uint8_t>(bit);
          errs += bit;
        }
      }
      if (errs) atomicAdd(&s_berr[ff], errs);
      if (a.posterior) {
        const char* const sb = slot_base(ff);
        for (int v = tid; v < n; v += nt) {
          const int pos = __ldg(g.d_vn_pos + v);
          const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_vn_rec) + pos);
          float t = *reinterpret_cast<const float*>(sb + l_off + pos * 8);
          t += *reinterpret_cast<const float*>(sb + lo16(r.x));
          t += *reinterpret_cast<const float*>(sb + hi16(r.x));
          t += *reinterpret_cast<const float*>(sb + lo16(r.y));
          a.posterior[f * n + v] = t * kLn2;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      for (int ff = 0; ff < FPC; ++ff) {
        if (s_done[ff] != 2) continue;
        const long long f = s_frame[ff];
        const int it = s_iters[ff];
        if (a.iterations) a.iterations[f] = a.early_stop ? it : a.max_iters;
        if (a.converged) a.converged[f] = static_cast<uint8_t>(s_conv[ff]);
        if (a.bit_errors) a.bit_errors[f] = s_berr[ff];
        s_cnt[0] += 1;
        s_cnt[1] += s_berr[ff];
        s_cnt[2] += s_berr[ff] > 0;
        s_cnt[3] += s_conv[ff];
        s_cnt[4] += a.early_stop ? it : a.max_iters;
        s_cnt[5] += s_conv[ff] ? (a.early_stop ? it : a.max_iters) : 0;
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
    it_cta = 0;
    if (s_active == 0) break;
    __syncthreads();
  }
  if (tid == 0 && a.counters)
    for (int i = 0; i < 6; ++i)
      if (s_cnt[i]) atomicAdd(a.counters + i, s_cnt[i]);
  return;

dump_state:
  // state after max_subiters sub-iterations: c2v and v2c per CN-major edge id
  __syncthreads();
  for (int ff = 0; ff < FPC; ++ff) {
    const long long f = s_frame[ff];
    if (f < 0) continue;
    const char* const sb = slot_base(ff);
    for (int e = tid; e < E; e += nt) {
      const int2 r = __ldg(reinterpret_cast<const int2*>(g.d_edge_rec) + e);
      if (a.c2v_out) a.c2v_out[f * E + e] = *reinterpret_cast<const float*>(sb + lo16(r.x)) * kLn2;
      if (a.v2c_out) {
        float t = *reinterpret_cast<const float*>(sb + hi16(r.x));
        t += *reinterpret_cast<const float*>(sb + lo16(r.y));
        t += *reinterpret_cast<const float*>(sb + hi16(r.y));
        a.v2c_out[f * E + e] = clamp_bits(t) * kLn2;
      }
    }
  }
}

using DirectFn = void (*)(const DevGraph, const DecodeArgs, unsigned long long*);

// LDPCB_DIRECT_SPLIT=1 selects the split arrive / wait barrier (A/B: measured
// 2 % slower than the plain barrier on C1 NDGSBP, 106.9 against 104.5 ms)
bool split_barrier() {
  const char* e = std::getenv("LDPCB_DIRECT_SPLIT");
  return e && std::atoi(e) != 0;
}

DirectFn pick_direct(int ng) {
  const bool sp = split_barrier();
  switch (ng) {
    case 1: return sp ? decode_direct<1, true> : decode_direct<1, false>;
    case 2: return sp ? decode_direct<2, true> : decode_direct<2, false>;
    case 3: return sp ? decode_direct<3, true> : decode_direct<3, false>;
    default: return nullptr;
  }
}

int max_threads_direct(int ng) { return ng == 1 ? 96 : (ng == 2 ? 192 : 256); }

}  // namespace

// LDPCB_DIRECT=0 keeps every decode on the posterior-based kernels (A/B)
bool direct_enabled() {
  const char* e = std::getenv("LDPCB_DIRECT");
  return !e || std::atoi(e) != 0;
}

Plan plan_direct(const DevGraph& g, int64_t frames) {
  Plan p;
  const int ng = g.d_ng;
  if (ng < 1 || ng > 3 || !g.d_cn_rec || g.per_frame) return p;
  if (static_cast<long long>(ng) * g.d_max_items > max_threads_direct(ng)) return p;  // one CN item per thread
  const int npad = (g.n + 15) & ~15;
  const size_t bytes = static_cast<size_t>(ng) * g.d_cells * 8 + ((ng * npad + 15) & ~15) + 8ull * g.G + 16;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) optin = 227 * 1024;
  if (bytes + 512 > static_cast<size_t>(optin)) return p;
  p.kernel = 3;
  p.fpc = 2 * ng;
  p.fv = 2;
  p.threads = std::max(64, std::min(max_threads_direct(ng), (ng * g.d_max_items + 31) / 32 * 32));
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
  DirectFn fn = pick_direct(g.d_ng);
  cudaError_t err =
      cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
  if (err != cudaSuccess) return static_cast<int>(err);
  // resident CTAs per device (cached per kernel, configuration and device)
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> cache;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(reinterpret_cast<const void*>(fn), p.threads, p.smem, dev);
    auto it = cache.find(key);
    if (it == cache.end()) {
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, p.threads, p.smem) != cudaSuccess || per_sm <= 0)
        return static_cast<int>(cudaErrorInvalidConfiguration);
      it = cache.emplace(key, sms * per_sm).first;
    }
    per_sm = it->second;  // CTAs per device
  }
  auto st = static_cast<cudaStream_t>(stream);
  // state dumps stop every CTA after its first frames: one CTA per FPC frames
  const int64_t ctas = a.max_subiters > 0 ? p.ctas : std::min<int64_t>(p.ctas, per_sm);
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
