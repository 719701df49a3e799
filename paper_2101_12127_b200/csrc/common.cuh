// common.cuh -- device-side contracts shared by every sm_100a kernel.
//
// The integer contracts are the reference's (bit-identical):
//   SplitMix64Next / MixSeeds / Pcg32  -- /root/reference/proj/include/
//                                         datapipe/random.hpp:24-74
// plus an O(log k) LCG jump-ahead so many lanes can draw one PCG stream in
// parallel, and Philox4x32-10 for this build's crop/flip randomness (the
// reference defines no image UDFs).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dpk {

constexpr uint64_t kPcgMult = 6364136223846793005ULL;
constexpr uint64_t kPcgInc = 1442695040888963407ULL;  // random.hpp:72

__host__ __device__ __forceinline__ uint64_t splitmix64_next(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix_seeds(uint64_t a, uint64_t b) {
  uint64_t s = a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2));
  return splitmix64_next(s);
}

// PCG-XSH-RR output function of the pre-advance state (random.hpp:48-54).
__host__ __device__ __forceinline__ uint32_t pcg_output(uint64_t old) {
  uint32_t xorshifted = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((-rot) & 31u));
}

__host__ __device__ __forceinline__ uint64_t pcg_step(uint64_t s) {
  return s * kPcgMult + kPcgInc;
}

// State after Pcg32(seed) construction (random.hpp:41-46).
__host__ __device__ __forceinline__ uint64_t pcg_seeded_state(uint64_t seed) {
  uint64_t s = pcg_step(0);
  s += seed;
  return pcg_step(s);
}

// Affine map of k LCG steps: s_k = mult * s + plus (Brown, "Random number
// generation with arbitrary strides", 1994).
struct LcgJump {
  uint64_t mult, plus;
};

__host__ __device__ __forceinline__ LcgJump lcg_jump(uint64_t k) {
  uint64_t acc_mult = 1, acc_plus = 0;
  uint64_t cur_mult = kPcgMult, cur_plus = kPcgInc;
  while (k) {
    if (k & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    k >>= 1;
  }
  return {acc_mult, acc_plus};
}

__host__ __device__ __forceinline__ uint64_t lcg_apply(LcgJump j, uint64_t s) {
  return j.mult * s + j.plus;
}

// Philox4x32-10 (Salmon et al., SC'11).
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1,
                                                       uint32_t c2, uint32_t c3,
                                                       uint32_t k0, uint32_t k1,
                                                       uint32_t out[4]) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
#endif
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Crop offsets and flip bit for element `id` (key = udf seed, ctr = id).
struct CropParams {
  int oy, ox, flip;
};

__host__ __device__ __forceinline__ CropParams crop_params(uint64_t seed, int64_t id,
                                                           int in_h, int in_w,
                                                           int crop_h, int crop_w) {
  uint32_t r[4];
  uint64_t uid = static_cast<uint64_t>(id);
  philox4x32_10(static_cast<uint32_t>(uid), static_cast<uint32_t>(uid >> 32), 0u, 0u,
                static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), r);
  CropParams p;
  p.oy = static_cast<int>(r[0] % static_cast<uint32_t>(in_h - crop_h + 1));
  p.ox = static_cast<int>(r[1] % static_cast<uint32_t>(in_w - crop_w + 1));
  p.flip = static_cast<int>(r[2] & 1u);
  return p;
}

// Per-channel normalize constants; `rcp` = RN(1 / std) for the exact
// division sequence below.
struct NormConsts {
  float mean[3];
  float stdv[3];
  float rcp[3];
  // The packed-pair ops (f32x2 below) take their 1 / -1 / -0 / -2^23 from
  // here, kernel parameters ptxas cannot constant-fold (see PkK).
  float one = 1.0f, neg_one = -1.0f, neg_zero = -0.0f, neg_magic = -8388608.0f;
};

#ifdef __CUDACC__
// (v - mean) / std rounded exactly as IEEE fp32 division: one rounded
// subtract, then the Markstein correction q' = RN(q + RN(d - q*s) * r) from
// q = RN(d * r), r = RN(1/s).  Proven equal to IEEE division for EVERY fp32
// v in [+0, 255] and the three normalize channels by exhaustive enumeration
// (tools/prove_fast_div.c, run by tests/test_oracle.py), which covers uint8
// pixels (K3) and every bilinear blend of them (K4).
__device__ __forceinline__ float normalize_fast(float v, float mean, float s, float r) {
  float d = __fsub_rn(v, mean);
  float q = __fmul_rn(d, r);
  float rem = __fmaf_rn(-q, s, d);
  return __fmaf_rn(rem, r, q);
}

// ---- packed fp32 pairs (sm_100 FFMA2: two lanes of fp32 per issue slot) ----
// Every op is ONE fma.rn.f32x2 with a single rounding, so each lane equals
// the scalar __f*_rn op bit for bit:  a+b = fma(a, 1, b),  a-b = fma(b, -1,
// a),  a*b = fma(a, b, -0).  ptxas treats the f32x2 forms as contractable
// even with --fmad=false and explicit .rn: it folds fma(x, 1, y) to FADD2 and
// fma(x, y, -0) to FMUL2 and then fuses FMUL2 + FADD2 into one FFMA2 (seen in
// the SASS), which changes the rounding.  So the constants 1 / -1 / -0 come
// from kernel parameters (NormConsts) that ptxas cannot fold: every op stays
// a real FFMA2 and nothing fuses.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 up2(f32x2 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 splat2(float v) { return pk2(v, v); }
struct PkK {  // opaque packed constants, built from NormConsts in registers
  f32x2 one, neg_one, neg_zero, neg_magic;
  __device__ explicit PkK(const NormConsts& n)
      : one(splat2(n.one)), neg_one(splat2(n.neg_one)), neg_zero(splat2(n.neg_zero)), neg_magic(splat2(n.neg_magic)) {}
  PkK() = default;
  __device__ f32x2 add(f32x2 a, f32x2 b) const { return fma2(a, one, b); }
  __device__ f32x2 sub(f32x2 a, f32x2 b) const { return fma2(b, neg_one, a); }
  __device__ f32x2 mul(f32x2 a, f32x2 b) const { return fma2(a, b, neg_zero); }
  // two uint8 -> exact fp32 (the 2^23 magic-number conversion of u8_to_f32)
  __device__ f32x2 u8x2(uint32_t a, uint32_t b) const {
    return fma2(pk2(__uint_as_float(0x4B000000u | a), __uint_as_float(0x4B000000u | b)), one, neg_magic);
  }
  // normalize_fast on a pair; nsd = -std per lane
  __device__ f32x2 normalize(f32x2 v, f32x2 mean, f32x2 nsd, f32x2 r) const {
    const f32x2 d = sub(v, mean);
    const f32x2 q = mul(d, r);
    return fma2(fma2(q, nsd, d), r, q);
  }
  // p + w * (q - p), each op rounded (lerp_rn) on a pair
  __device__ f32x2 lerp(f32x2 p, f32x2 q, f32x2 w) const { return add(p, mul(w, sub(q, p))); }
  // lerp_rn of two uint8 taps given as magic floats p' = 2^23 + p, q' = 2^23 + q:
  // q' - p' == q - p exactly (|q - p| <= 255), so only p is converted -- the
  // same three rounded ops as lerp(u8x2(p), u8x2(q), w), one FFMA2 fewer.
  __device__ f32x2 lerp_u8(f32x2 p_raw, f32x2 q_raw, f32x2 w) const {
    return add(fma2(p_raw, one, neg_magic), mul(w, sub(q_raw, p_raw)));
  }
  static __device__ f32x2 raw_u8x2(uint32_t a, uint32_t b) {
    return pk2(__uint_as_float(0x4B000000u | a), __uint_as_float(0x4B000000u | b));
  }
};

__device__ __forceinline__ void st_cs_f4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// One warp streams two token rows at once (kLoads loads per lane per row in
// flight before the stores): row a/b copies len tokens, then pads with `pad`
// up to lm (lm = len: no padding; len = lm = 0: no row).  Two independent
// rows per warp double the bytes in flight of the short (~1 KB) rows.
template <int kLoads>
__device__ __forceinline__ void stream_row_pair(const int32_t* __restrict__ src_a, int len_a, int lm_a,
                                                int32_t* __restrict__ dst_a, const int32_t* __restrict__ src_b,
                                                int len_b, int lm_b, int32_t* __restrict__ dst_b, int32_t pad,
                                                int lane) {
  const int lm = lm_a > lm_b ? lm_a : lm_b;
  for (int c = lane; c < lm; c += 32 * kLoads) {
    int32_t va[kLoads], vb[kLoads];
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int k = c + 32 * u;
      va[u] = k < len_a ? __ldcs(src_a + k) : pad;
      vb[u] = k < len_b ? __ldcs(src_b + k) : pad;
    }
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int k = c + 32 * u;
      if (k < lm_a) __stcs(dst_a + k, va[u]);
      if (k < lm_b) __stcs(dst_b + k, vb[u]);
    }
  }
}

__device__ __forceinline__ uint4 ld_nc_na_u4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
#endif

}  // namespace dpk

#ifdef __CUDACC__
namespace dpk {

// ---- TMA bulk copies + mbarriers (sm_90+ PTX; SASS UBLKCP / SYNCS) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DP_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// L2 evict-first policy for read-once streams.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Global -> shared bulk copy (TMA engine), completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Exact uint8 -> fp32 without the conversion pipe: 2^23 + x, minus 2^23.
__device__ __forceinline__ float u8_to_f32(uint32_t x) {
  return __fsub_rn(__uint_as_float(0x4B000000u | x), 8388608.0f);
}

}  // namespace dpk
#endif
