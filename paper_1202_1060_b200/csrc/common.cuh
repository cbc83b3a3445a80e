// common.cuh -- boxplus arithmetic and table records shared by the resident
// (shared-memory) and streamed (HBM) decoder kernels.
#pragma once
#include <type_traits>
#include <cstdint>

namespace ldpcb {
namespace dev {

constexpr float kClamp = 30.0f;  // decoder.hpp:18
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;
// Inside the kernels messages are kept in log2 units (LLR * log2 e), so the
// boxplus needs no scaling around ex2 / lg2; the clamp scales with them.
constexpr float kClampB = 43.280851226668897f;  // 30 * log2(e)


#ifndef LDPCB_EXP_NOMUFU
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
#else  // timing experiment only (scripts/exp_builds.sh): wrong results
__device__ __forceinline__ float mufu_ex2(float x) { return fmaf(x, 0.01f, 1.0f); }
__device__ __forceinline__ float mufu_lg2(float x) { return fmaf(x, 0.5f, -0.5f); }
#endif

__device__ __forceinline__ float clamp_llr(float x) { return fminf(fmaxf(x, -kClamp), kClamp); }
__device__ __forceinline__ float clamp_bits(float x) { return fminf(fmaxf(x, -kClampB), kClampB); }

// Exclusion boxplus over one CN, in log2 units. x[k] are the incoming v2c
// for k < deg (EXACT: deg == D); |v2c| is clamped to 30 nats here
// (decoder.hpp:125) and the sign travels in the IEEE sign bit.
// store(k, c2v_k) receives every output, clamped to 30 nats (decoder.hpp:74).
//
// Exactly-zero inputs: ex2(-0) = 1 exactly, and every combine below is
// symmetric under N <-> D of an operand equal to (a, a), so any output whose
// exclusion set holds a zero ends with N == D bit-for-bit and a magnitude of
// exactly 0 (decoder.hpp:77-83) without per-edge bookkeeping.
template <int D, bool EXACT, class Store>
__device__ __forceinline__ void boxplus_row(const float (&x)[D], int deg, Store&& store) {
  float z[D];
  unsigned sg = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (EXACT || k < deg) {
      sg ^= __float_as_uint(x[k]);
      z[k] = mufu_ex2(-fminf(fabsf(x[k]), kClampB));
    } else {
      z[k] = 0.f;  // boxplus identity (N, D) = (0, 1)
    }
  }
  // |out| = lg2 D - lg2 N: the boxplus of clamped inputs cannot exceed the
  // clamp, so no output clamp is applied (rounding may add < 1e-5 to a
  // saturated message); the magnitude's sign bit is replaced by the parity of
  // the other inputs' signs in one bit-select.
  auto emit = [&](int k, float num, float den) {
    if (EXACT || k < deg) {
      const unsigned d = __float_as_uint(mufu_lg2(den) - mufu_lg2(num));
      const unsigned t = sg ^ __float_as_uint(x[k]);
      store(k, __uint_as_float((d & 0x7fffffffu) | (t & 0x80000000u)));
    }
  };
  // prefix p[k] = z0 (+) ... (+) zk for k <= D-2: (N, D) <- (N + z D, D + z N)
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
  if (D >= 3) {  // first middle output, suffix = (z[D-1], 1): same rounding pattern without the * 1
    constexpr int k = D >= 3 ? D - 2 : 1;
    emit(k, __fadd_rn(pn[k - 1], __fmul_rn(sn, pd[k - 1])), __fadd_rn(pd[k - 1], __fmul_rn(pn[k - 1], sn)));
    const float tn = z[k] + sn;
    const float td = fmaf(z[k], sn, 1.f);
    sn = tn;
    sd = td;
  }
#pragma unroll
  for (int k = D - 3; k >= 2; --k) {
    // out_k = p[k-1] (+) s[k+1], rounded symmetrically (see above)
    emit(k, __fadd_rn(__fmul_rn(pn[k - 1], sd), __fmul_rn(sn, pd[k - 1])),
         __fadd_rn(__fmul_rn(pd[k - 1], sd), __fmul_rn(pn[k - 1], sn)));
    const float tn = fmaf(z[k], sd, sn);
    const float td = fmaf(z[k], sn, sd);
    sn = tn;
    sd = td;
  }
  if (D >= 4) {  // out_1 = z0 (+) s[2]: prefix p[0] = (z0, 1), same rounding pattern without the * 1
    emit(1, __fadd_rn(__fmul_rn(pn[0], sd), sn), __fadd_rn(sd, __fmul_rn(pn[0], sn)));
    const float tn = fmaf(z[1], sd, sn);
    const float td = fmaf(z[1], sn, sd);
    sn = tn;
    sd = td;
  }
  emit(0, sn, sd);
}

// ---- two frames per instruction: sm_100 packed fp32 (FADD2 / FMUL2 / FFMA2)
// The same arithmetic as boxplus_row on a pair of frames held as one 64-bit
// register pair, so every add / mul / fma issues once for both frames (each
// lane rounds exactly like the scalar instruction: results are bit-identical).
using f32x2 = unsigned long long;
__device__ __forceinline__ f32x2 pack2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo2(f32x2 t) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(t));
  return a;
}
__device__ __forceinline__ float hi2(f32x2 t) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(t));
  return b;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// a * b rounded once, as fma(a, b, -0) with the -0 pair read from constant
// memory: ptxas contracts mul.rn.f32x2 (and an fma with a literal -0 addend)
// into a following add.rn.f32x2, unlike the scalar .rn forms, which would
// break the symmetric rounding boxplus relies on; an fma whose addend it
// cannot see is never fused.
static __constant__ unsigned long long c_negzero2 = 0x8000000080000000ull;
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c_negzero2));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// boxplus_row for two frames at once: x[k] packs frame 0 (low) and frame 1
// (high); store(k, c2v_k) receives packed outputs. Same operation order and
// rounding as boxplus_row, lane by lane.
template <int D, bool EXACT, class Store>
__device__ __forceinline__ void boxplus_row_x2(const f32x2 (&x)[D], int deg, Store&& store) {
  f32x2 z[D];
  unsigned sa = 0, sb = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (EXACT || k < deg) {
      const float a = lo2(x[k]), b = hi2(x[k]);
      sa ^= __float_as_uint(a);
      sb ^= __float_as_uint(b);
      z[k] = pack2(mufu_ex2(-fminf(fabsf(a), kClampB)), mufu_ex2(-fminf(fabsf(b), kClampB)));
    } else {
      z[k] = 0ull;  // (0.f, 0.f): boxplus identity (N, D) = (0, 1)
    }
  }
  const f32x2 one = pack2(1.f, 1.f);
  auto emit = [&](int k, f32x2 num, f32x2 den) {
    if (EXACT || k < deg) {
      const f32x2 dd = sub2(pack2(mufu_lg2(lo2(den)), mufu_lg2(hi2(den))), pack2(mufu_lg2(lo2(num)), mufu_lg2(hi2(num))));
      const unsigned ta = sa ^ __float_as_uint(lo2(x[k])), tb = sb ^ __float_as_uint(hi2(x[k]));
      store(k, pack2(__uint_as_float((__float_as_uint(lo2(dd)) & 0x7fffffffu) | (ta & 0x80000000u)),
                     __uint_as_float((__float_as_uint(hi2(dd)) & 0x7fffffffu) | (tb & 0x80000000u))));
    }
  };
  f32x2 pn[D > 1 ? D - 1 : 1], pd[D > 1 ? D - 1 : 1];
  pn[0] = z[0];
  pd[0] = one;
#pragma unroll
  for (int k = 1; k < D - 1; ++k) {
    pn[k] = fma2(z[k], pd[k - 1], pn[k - 1]);
    pd[k] = fma2(z[k], pn[k - 1], pd[k - 1]);
  }
  emit(D - 1, pn[D - 2], pd[D - 2]);
  f32x2 sn = z[D - 1], sd = one;
  if (D >= 3) {
    constexpr int k = D >= 3 ? D - 2 : 1;
    emit(k, add2(pn[k - 1], mul2(sn, pd[k - 1])), add2(pd[k - 1], mul2(pn[k - 1], sn)));
    const f32x2 tn = add2(z[k], sn);
    const f32x2 td = fma2(z[k], sn, one);
    sn = tn;
    sd = td;
  }
#pragma unroll
  for (int k = D - 3; k >= 2; --k) {
    emit(k, add2(mul2(pn[k - 1], sd), mul2(sn, pd[k - 1])), add2(mul2(pd[k - 1], sd), mul2(pn[k - 1], sn)));
    const f32x2 tn = fma2(z[k], sd, sn);
    const f32x2 td = fma2(z[k], sn, sd);
    sn = tn;
    sd = td;
  }
  if (D >= 4) {
    emit(1, add2(mul2(pn[0], sd), sn), add2(sd, mul2(pn[0], sn)));
    const f32x2 tn = fma2(z[1], sd, sn);
    const f32x2 td = fma2(z[1], sn, sd);
    sn = tn;
    sd = td;
  }
  emit(0, sn, sd);
}

// channel LLRs are read once: keep them out of L1, where the record tables live
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// One CN record (host.hpp KernelTables): [slot of edge 0, single-touch
// mask, v_0 ... v_{D-1}] (v = -1 past the degree), kInts ints. Regular rows
// of degree 3 or 6 on codes with n < 65536 use the packed 16-byte form
// (record stride cs = 4): {slot | mask << 24, v0 | v1 << 16, v2 | v3 << 16,
// v4 | v5 << 16}, one 128-bit load instead of two.
template <int D, bool EXACT>
struct CnRecord {
  static constexpr int kInts = (2 + D + 3) / 4 * 4;
  static constexpr bool kPackable = EXACT && D <= 6;
  int r[kInts];
  CnRecord() = default;
  __device__ __forceinline__ CnRecord(const int32_t* __restrict__ p, int cs) { load(p, cs); }
  __device__ __forceinline__ void load(const int32_t* __restrict__ p, int cs) {
    const int4* q = reinterpret_cast<const int4*>(p);
    if (kPackable && cs == 4) {
      const int4 t = __ldg(q);
      r[0] = t.x & 0xffffff;
      r[1] = static_cast<int>(static_cast<unsigned>(t.x) >> 24);
      const int w[3] = {t.y, t.z, t.w};
#pragma unroll
      for (int k = 0; k < D; ++k)
        r[2 + k] = static_cast<int>((static_cast<unsigned>(w[k >> 1]) >> (16 * (k & 1))) & 0xffffu);
      return;
    }
#pragma unroll
    for (int i = 0; i < kInts / 4; ++i) {
      const int4 t = __ldg(q + i);
      r[4 * i] = t.x;
      r[4 * i + 1] = t.y;
      r[4 * i + 2] = t.z;
      r[4 * i + 3] = t.w;
    }
  }
  __device__ __forceinline__ int slot() const { return r[0]; }
  __device__ __forceinline__ unsigned mask() const { return static_cast<unsigned>(r[1]); }
  __device__ __forceinline__ int var(int k) const { return r[2 + k]; }
  __device__ __forceinline__ bool has(int k) const { return EXACT || r[2 + k] >= 0; }
  __device__ __forceinline__ int deg() const {
    if (EXACT) return D;
    int d = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) d += r[2 + k] >= 0;
    return d;
  }
};


// The packed record kept as loaded and decoded field by field at use: a
// record prefetched a phase ahead then costs nothing until it is used.
template <int D>
struct CnRecordPacked {
  static_assert(D <= 6, "packed records hold at most six 16-bit VN indices");
  int4 w;
  CnRecordPacked() = default;
  __device__ __forceinline__ CnRecordPacked(const int32_t* __restrict__ p, int) { load(p, 4); }
  __device__ __forceinline__ void load(const int32_t* __restrict__ p, int) { w = __ldg(reinterpret_cast<const int4*>(p)); }
  __device__ __forceinline__ int slot() const { return w.x & 0xffffff; }
  __device__ __forceinline__ unsigned mask() const { return static_cast<unsigned>(w.x) >> 24; }
  __device__ __forceinline__ int var(int k) const {
    const unsigned x = static_cast<unsigned>(k < 2 ? w.y : (k < 4 ? w.z : w.w));
    return static_cast<int>((x >> (16 * (k & 1))) & 0xffffu);
  }
  __device__ __forceinline__ bool has(int) const { return true; }
  __device__ __forceinline__ int deg() const { return D; }
};

// Record type of the resident kernel: packed for regular rows of degree <= 6
// (the host packs them whenever n < 65536, always true for a resident code).
template <int D, bool EXACT>
using ResidentRecord = typename std::conditional<EXACT && D <= 6, CnRecordPacked<D>, CnRecord<D, EXACT>>::type;

}  // namespace dev
}  // namespace ldpcb
