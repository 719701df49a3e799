// k_roll.cu -- K10: bilinear-resize image map chains + Batch over a PERIODIC
// column map, with the horizontal blends rolled in registers.
//
// Replaces, for the resize chains of the device UDF library, the reference's
// per-element MapFn sequence and batch assembly (MapAndBatchIterator,
// /root/reference/proj/src/runtime.cpp:1467-1721; a chain map(f).map(g) is
// g(f(e)), optimizer.cpp:165-188):
//     [crop A (random + flip | center)] -> resize -> [crop B] -> [one pixel op]
// e.g. RandomResizedCrop (crop 160 + flip -> resize 224 -> normalize), ResNet
// eval (resize 256 -> center crop 224 -> normalize), and K4's resize 320 ->
// 224 -> normalize.  Every output value is the sequential chain's value
// (oracle/chain.c): top = p00 + wx (p01 - p00), bot = p10 + wx (p11 - p10),
// v = top + wy (bot - top), then the op -- each fp32 op rounded once.
//
// Why a new kernel: K9 recomputes both horizontal blends of every output
// value (2 source rows per output row), and K4 does too; an upscale (160 ->
// 224) reads each source row for ~2.8 output rows, a downscale (320 -> 224)
// for ~1.4.  Here a warp walks a RUN of consecutive output rows of one
// column stripe, so the horizontal blend of each (source row, output column)
// is computed once and kept in registers (two rows, ping-pong, no moves);
// each output row is then one vertical lerp + the op per value.
//
// Any other ratio runs the general form (PI = 0): each lane's 8 pixels keep
// their two taps as runtime byte offsets (one shared-memory byte load per
// tap) and the clamped weights themselves.
//
// Horizontal taps are periodic (instantiated window : mid ratios 10:7, 8:7,
// 5:7, 5:4, 9:7, 12:7, 6:7, 4:7, 3:2, 2:1): win_w = PI * G, mid_w = PO * G and every
// mid column x = PO p + c reads window columns PI p + T(c) and + 1 (the host
// checks every column against the device tap formula; the right-edge clamp
// x1 == x0 gets weight 0, which gives p00 exactly as the clamped blend does).
// One lane owns one period p: it loads the period's source window of a
// staged row as 32-bit words, funnel-shifts them to the window's byte
// offset, and picks the taps with PRMT at compile-time positions as exact
// 2^23 + byte floats (a flipped crop A mirrors the positions: a second
// compile-time pattern).  The row leaves through a per-warp shared buffer as
// coalesced 16-byte streaming stores (crop B / its flip only move where a
// lane's pixels land in that buffer).
//
// Pipeline: persistent, one CTA per SM; one producer warp plans 32 items
// (image, band of output rows) at a time (gather index, Philox crop draws)
// and issues cp.async.bulk copies of the band's source rows into a ring of
// mbarrier stages; W consumer warps split a band into runs x stripes and
// release stages through "empty" mbarriers (no CTA barrier in the loop).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "fastdiv.hpp"
#include "roll.hpp"
#include "status.hpp"

namespace dpk {
namespace {

#ifndef DP_ROLL_WARPS
#define DP_ROLL_WARPS 11  // consumer warps: + the producer = 3 warps per SM sub-partition (<= 168 registers)
#endif
constexpr int kRollMaxWarps = DP_ROLL_WARPS;
constexpr int kRollMaxStages = 8;
constexpr int kRollMaxStripes = 4;
constexpr size_t kRollSmemMax = 224 * 1024;

struct RollIds {
  int64_t base, stride, block;
  __device__ __forceinline__ int64_t of(int64_t r) const {
    if (block == 1) return base + r * stride;
    const int64_t q = r / block;
    return (q * stride + base) * block + (r - q * block);
  }
};

// window rows of mid row m; wy = 0 on the bottom clamp (y1 == y0), where
// top + 0 * (anything finite - top) == top == the clamped blend
struct RollTap {
  int y0, y1;
  float wy;
};

struct RollArgs {
  const uint8_t* images;
  const int64_t* order;
  int64_t first, rows, num_images;
  int64_t* out_ids;
  float* out;
  int in_h, in_w, win_h, win_w, mid_h, mid_w, out_h, out_w;
  int pre_mode, pre_flip, post_mode, post_flip;
  uint64_t pre_seed, post_seed;
  float scale_y, scale_x;  // window / mid, rounded once (chain_coord)
  int band_rows, bands, runs, stripes, cons_warps;
  int stripe_px[kRollMaxStripes + 1];  // stripe s: output pixels [stripe_px[s], stripe_px[s + 1]), multiples of 4
  int stage_stride, stage_bytes, stages;
  int taps_offset, buf_offset, buf_floats;  // smem layout after the stages
  float op_a[3], op_b[3], op_r[3];           // the pixel op: normalize (mean, std, RN(1/std)) or affine (a, b)
  float op2_a[3], op2_b[3];                  // a second pixel op (affine, or normalize with IEEE division)
  NormConsts nc;                             // opaque 1 / -1 / -0 / -2^23 for the packed ops
  RollIds ids;
};

struct RollMeta {
  int64_t id, j;
  int band, nrows, wy_lo, adj, f0, ox1, f1, oy1;
};

struct RollPlan {
  int64_t id, j, row;
  int band, nrows, wy_lo, nsrc, src_row, col0, bytes_row, adj, f0, ox1, f1, oy1;
};

__device__ __forceinline__ RollPlan shfl_plan(const RollPlan& p, int src) {
  RollPlan o;
  o.id = __shfl_sync(0xffffffffu, p.id, src);
  o.j = __shfl_sync(0xffffffffu, p.j, src);
  o.row = __shfl_sync(0xffffffffu, p.row, src);
  o.band = __shfl_sync(0xffffffffu, p.band, src);
  o.nrows = __shfl_sync(0xffffffffu, p.nrows, src);
  o.wy_lo = __shfl_sync(0xffffffffu, p.wy_lo, src);
  o.nsrc = __shfl_sync(0xffffffffu, p.nsrc, src);
  o.src_row = __shfl_sync(0xffffffffu, p.src_row, src);
  o.col0 = __shfl_sync(0xffffffffu, p.col0, src);
  o.bytes_row = __shfl_sync(0xffffffffu, p.bytes_row, src);
  o.adj = __shfl_sync(0xffffffffu, p.adj, src);
  o.f0 = __shfl_sync(0xffffffffu, p.f0, src);
  o.ox1 = __shfl_sync(0xffffffffu, p.ox1, src);
  o.f1 = __shfl_sync(0xffffffffu, p.f1, src);
  o.oy1 = __shfl_sync(0xffffffffu, p.oy1, src);
  return o;
}

// Half-pixel-centre source coordinate (oracle/chain.c chain_coord; the scale
// in / out rounded once on the host).
__device__ __forceinline__ void roll_coord(int d, int in, float scale, int& i0, int& i1, float& w) {
  float s = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(d), 0.5f), scale), 0.5f);
  if (s < 0.0f) s = 0.0f;
  int a = static_cast<int>(s);
  if (a > in - 1) a = in - 1;
  i0 = a;
  i1 = a + 1 < in ? a + 1 : in - 1;
  w = __fsub_rn(s, static_cast<float>(a));
}

__device__ __forceinline__ void roll_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Pixel ops: 0 none, 1 normalize with the proven two-FMA division
// (fastdiv.hpp), 2 affine x * a + b, 3 normalize with IEEE division.
template <int PO, int PI, int kOp>
struct Roll {
  // left tap of pixel c of period p: window column PI p + T(c), floor
  // division (T(0) = -1 when upscaling: the left-edge clamp, weight 1)
  __host__ __device__ static constexpr int T(int c) {
    return ((2 * c + 1) * PI - PO) >= 0 ? ((2 * c + 1) * PI - PO) / (2 * PO)
                                        : -((PO - (2 * c + 1) * PI + 2 * PO - 1) / (2 * PO));
  }
  static constexpr int kF = 3 * PO;                          // floats per period
  // Packed pairs: a pair is one channel of two neighbouring pixels, so
  // every op constant is a per-channel scalar the FFMA2 broadcasts and the
  // tap weights are one pair per pixel pair (an odd period leaves one
  // half-used pair per channel).
  static constexpr int kNPP = (PO + 1) / 2;  // pixel pairs
  static constexpr int kP = 3 * kNPP;
  static constexpr int kW = kNPP;  // weight pairs
  static constexpr int kSpan = 3 * (T(PO - 1) + 2 - T(0));  // window bytes of a period
  static constexpr int kNW = (kSpan + 3) / 4;       // shifted words used
  static constexpr int kNWL = (kSpan + 3 + 3) / 4;  // words loaded (any byte offset)
  // tap byte (left / right) of value e in the shifted window; kFlip: the
  // window mirrored (crop A's flip), pixel order reversed, channels kept
  template <bool kFlip>
  __host__ __device__ static constexpr int L(int e) {
    return kFlip ? 3 * (T(PO - 1) + 1 - T(e / 3)) + e % 3 : 3 * (T(e / 3) - T(0)) + e % 3;
  }
  template <bool kFlip>
  __host__ __device__ static constexpr int R(int e) {
    return kFlip ? L<kFlip>(e) - 3 : L<kFlip>(e) + 3;
  }
  // values (e0, e1) of pair i (e1 == e0: a half-used pair) and its weight pair
  __host__ __device__ static constexpr int e0(int i) { return 6 * (i % kNPP) + i / kNPP; }
  __host__ __device__ static constexpr int e1(int i) { return 2 * (i % kNPP) + 1 < PO ? e0(i) + 3 : e0(i); }
  __host__ __device__ static constexpr int wi(int i) { return i % kNPP; }
  // the pair and half holding value e = 3 * pixel + channel
  __host__ __device__ static constexpr int pair_of(int e) { return (e % 3) * kNPP + (e / 3) / 2; }
  __host__ __device__ static constexpr bool hi_of(int e) { return (e / 3) % 2 == 1; }

  // PI == 0: a general column map -- every pixel's two taps are runtime
  // byte offsets into the staged row (one byte load each), the weights the
  // clamped ones of chain_coord (no periodic form needed)
  static constexpr bool kGen = PI == 0;

  // (the right tap is the next window column, 3 bytes on -- or 3 back when
  // crop A flips; a right-edge clamp carries weight 0 instead)
  template <bool kFlip>
  static __device__ __forceinline__ void hrow_gen(const uint8_t* row, const int (&offl)[PO], f32x2 (&H)[kP],
                                                  const f32x2 (&wx2)[kW], const PkK& k) {
    constexpr int kR = kFlip ? -3 : 3;
#pragma unroll
    for (int i = 0; i < kP; ++i) {
      const int c0 = e0(i) / 3, c1 = e1(i) / 3, ch = e0(i) % 3;
      const f32x2 pl = pk2(__uint_as_float(0x4B000000u | row[offl[c0] + ch]),
                           __uint_as_float(0x4B000000u | row[offl[c1] + ch]));
      const f32x2 pr = pk2(__uint_as_float(0x4B000000u | row[offl[c0] + ch + kR]),
                           __uint_as_float(0x4B000000u | row[offl[c1] + ch + kR]));
      H[i] = k.lerp_u8(pl, pr, wx2[wi(i)]);
    }
  }

  static __device__ __forceinline__ uint32_t pick(const uint32_t* w, int b) {
    return __byte_perm(w[b >> 2], 0x4B000000u, 0x7440u | static_cast<uint32_t>(b & 3));
  }
  static __device__ __forceinline__ f32x2 raw2(const uint32_t* w, int b0, int b1) {
    return pk2(__uint_as_float(pick(w, b0)), __uint_as_float(pick(w, b1)));
  }

  // horizontal blends of one staged row for this lane's period
  template <bool kFlip>
  static __device__ __forceinline__ void hrow(const uint8_t* row, int b, f32x2 (&H)[kP], const f32x2 (&wx2)[kW],
                                              const PkK& k) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(row + (b & ~3));
    const int sh = (b & 3) * 8;
    uint32_t W[kNWL + 1];
#pragma unroll
    for (int i = 0; i < kNWL; ++i) W[i] = src[i];
    W[kNWL] = 0;
    uint32_t w[kNW];
#pragma unroll
    for (int i = 0; i < kNW; ++i) w[i] = __funnelshift_r(W[i], W[i + 1], sh);
#pragma unroll
    for (int i = 0; i < kP; ++i)
      H[i] = k.lerp_u8(raw2(w, L<kFlip>(e0(i)), L<kFlip>(e1(i))), raw2(w, R<kFlip>(e0(i)), R<kFlip>(e1(i))),
                       wx2[wi(i)]);
  }
};

// One consumer warp's state: its stripe and run, the op constants, and the
// lane geometry (period, tap weights, output positions), a function of crop
// B's (offset, flip), recomputed when they change.
template <int PO, int PI, int kOp>
struct RollWarp {
  using RO = Roll<PO, PI, kOp>;
  static constexpr int kP = RO::kP, kF = RO::kF, kW = RO::kW;
  int lane, stripe, run, px_lo, px_hi, n4;
  float* buf;
  PkK k;
  float sa[3], sb[3], sr_[3];  // op constants per channel (normalize: mean, -std, RN(1 / std))
  int g_ox1, g_f1;
  int p, pos[PO], vec_base;
  int xl[RO::kGen ? PO : 1];  // general map: the window column of each pixel's left tap
  bool vec;
  f32x2 wx2[kW];

  __device__ void init(const RollArgs& a, uint8_t* smem, int warp, int lane_) {
    lane = lane_;
    stripe = warp % a.stripes;
    run = warp / a.stripes;
    px_lo = a.stripe_px[stripe];
    px_hi = a.stripe_px[stripe + 1];
    n4 = 3 * (px_hi - px_lo) / 4;
    buf = reinterpret_cast<float*>(smem + a.buf_offset) + static_cast<size_t>(warp) * (a.buf_floats + 128);
    k = PkK(a.nc);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sa[c] = a.op_a[c];
      sb[c] = (kOp & 3) == 1 ? -a.op_b[c] : a.op_b[c];
      sr_[c] = a.op_r[c];
    }
    g_ox1 = g_f1 = -1;
    p = vec_base = 0;
    vec = false;
  }

  __device__ void geometry(const RollArgs& a, const RollMeta& m) {
    g_ox1 = m.ox1;
    g_f1 = m.f1;
    // mid columns of this stripe, the lane's period and where its pixels land
    const int m_lo = m.f1 ? m.ox1 + a.out_w - px_hi : m.ox1 + px_lo;
    const int m_hi = m.f1 ? m.ox1 + a.out_w - px_lo : m.ox1 + px_hi;
    p = m_lo / PO + lane;
    const bool active = p * PO < m_hi;
    if (!active) p = m_lo / PO;  // a valid period (reads stay in the stage); writes nothing
#pragma unroll
    for (int c = 0; c < PO; ++c) {
      const int mc = p * PO + c - m.ox1;  // output pixel before crop B's flip
      const int x = (m.f1 ? a.out_w - 1 - mc : mc) - px_lo;
      // invalid pixels go to this lane's trash slot past the row (no predicated stores)
      pos[c] = active && mc >= 0 && mc < a.out_w && x >= 0 && x < px_hi - px_lo ? 3 * x : a.buf_floats + 4 * lane;
    }
    // float4 stores straight from the pairs when every lane's pixels are
    // all in the stripe or all out, in order (no crop-B flip) and 16-byte aligned
    const int x0 = p * PO - m.ox1 - px_lo;
    const bool whole = !active || (x0 >= 0 && x0 + PO <= px_hi - px_lo);
    vec = kF % 4 == 0 && !m.f1 && __all_sync(0xffffffffu, whole && (3 * x0) % 4 == 0);
    vec_base = active ? 3 * x0 : -1;
    float wx[kF];
#pragma unroll
    for (int c = 0; c < PO; ++c) {
      int xa, xb;
      float w;
      roll_coord(p * PO + c, a.win_w, a.scale_x, xa, xb, w);
      if constexpr (RO::kGen) {  // the left tap; the right one is the next column
        xl[c] = xa;
        if (xb == xa) w = 0.0f;  // right clamp: p00 exactly, whatever the next column holds
      } else if (xb == xa) {
        // the periodic taps are (xf, xf + 1), xf = PI p + T(c); at the edges
        // they differ from the clamped ones but give p00 exactly:
        w = 0.0f;  // right clamp: xf == x0, any right tap
      } else if (xa == p * PI + RO::T(c) + 1) {
        w = 1.0f;  // left clamp: xf == -1, (p(-1), p(0)) at weight 1
      }
      wx[3 * c] = wx[3 * c + 1] = wx[3 * c + 2] = w;
    }
#pragma unroll
    for (int i = 0; i < kW; ++i) wx2[i] = pk2(wx[RO::e0(i)], wx[RO::e1(i)]);
  }

  // float4 slot swizzle of the row buffer on the float4 store path: lanes
  // write 6 float4 apart (2-way bank conflicts in a quarter warp); flipping
  // bit 0 of the slot in every odd group of 8 spreads them, and the readout's
  // 8 consecutive slots stay one aligned group (a permutation within it)
  static __device__ __forceinline__ int swz(int q) { return q ^ ((q >> 3) & 1); }

  // one output row from the blends of its two window rows
  template <bool kVec>
  __device__ __forceinline__ void emit(const RollArgs& a, const RollTap* tp, int r, float4* orow, int row_f4,
                                       const f32x2 (&A)[kP], const f32x2 (&B)[kP]) {
    const f32x2 wy2 = splat2(tp[r].wy);
    // pixel-pair major: the values of pixels 2j, 2j + 1 are done after step
    // j, so each float4 / word store issues as soon as its values exist and
    // few results are live at once
    float2 f[kP];
#pragma unroll
    for (int j = 0; j < RO::kNPP; ++j) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int i = c * RO::kNPP + j;
        // kOp = first op + 4 * second op (0 none, 1 proven normalize, 2
        // affine, 3 IEEE normalize; the second op is never the proven form:
        // its input is not a blend of bytes)
        constexpr int kOp0 = kOp & 3, kOp1 = kOp >> 2;
        f32x2 v = k.lerp(A[i], B[i], wy2);
        if (kOp0 == 1) v = k.normalize(v, splat2(sa[c]), splat2(sb[c]), splat2(sr_[c]));
        if (kOp0 == 2) v = k.add(k.mul(v, splat2(sa[c])), splat2(sb[c]));
        if (kOp1 == 2 && kOp0 != 3) v = k.add(k.mul(v, splat2(a.op2_a[c])), splat2(a.op2_b[c]));
        f[i] = up2(v);
        if (kOp0 == 3) {
          f[i].x = __fdiv_rn(__fsub_rn(f[i].x, a.op_a[c]), a.op_b[c]);
          f[i].y = __fdiv_rn(__fsub_rn(f[i].y, a.op_a[c]), a.op_b[c]);
          if (kOp1 == 2) {
            f[i].x = __fadd_rn(__fmul_rn(f[i].x, a.op2_a[c]), a.op2_b[c]);
            f[i].y = __fadd_rn(__fmul_rn(f[i].y, a.op2_a[c]), a.op2_b[c]);
          }
        }
        if (kOp1 == 3) {
          f[i].x = __fdiv_rn(__fsub_rn(f[i].x, a.op2_a[c]), a.op2_b[c]);
          f[i].y = __fdiv_rn(__fsub_rn(f[i].y, a.op2_a[c]), a.op2_b[c]);
        }
        if constexpr (!(kVec && kF % 4 == 0)) {
          const int e0 = RO::e0(i), e1 = RO::e1(i);
          buf[pos[e0 / 3] + e0 % 3] = f[i].x;
          if (e1 != e0) buf[pos[e1 / 3] + e1 % 3] = f[i].y;
        }
      }
      if constexpr (kVec && kF % 4 == 0) {
        auto val = [&](int e) { return RO::hi_of(e) ? f[RO::pair_of(e)].y : f[RO::pair_of(e)].x; };
        const int done = 6 * j + 6;  // values [0, done) exist
        const int q4 = (vec_base >> 2);  // the lane's first float4 (vec_base is 16-byte aligned)
#pragma unroll
        for (int q = 0; q < kF / 4; ++q)
          if (4 * q + 4 <= done && 4 * q + 4 > done - 6 && vec_base >= 0)
            reinterpret_cast<float4*>(buf)[swz(q4 + q)] =
                make_float4(val(4 * q), val(4 * q + 1), val(4 * q + 2), val(4 * q + 3));
      }
    }
    __syncwarp();
    float4* o = orow + static_cast<size_t>(r) * row_f4;
    const float4* b4 = reinterpret_cast<const float4*>(buf);
    // a stripe is <= 32 periods = 24 * PO floats: ceil(3 PO / 4) float4 per lane
#pragma unroll
    for (int it = 0; it < (3 * PO + 3) / 4; ++it) {
      const int c = lane + 32 * it;
      if (c < n4) st_cs_f4(o + c, b4[kVec && kF % 4 == 0 ? swz(c) : c]);
    }
    __syncwarp();
  }

  // walk the run: A / B hold the blends of window rows s and s + 1 (roles
  // swap every source row), each computed once
  template <bool kFlip, bool kVec>
  __device__ void walk(const RollArgs& a, const RollMeta& m, const uint8_t* stage, const RollTap* tp, int r_lo,
                       int r_hi) {
    float4* orow = reinterpret_cast<float4*>(a.out + (static_cast<size_t>(m.j) * a.out_h +
                                                       static_cast<size_t>(m.band) * a.band_rows) *
                                                          (3 * a.out_w) + 3 * px_lo);
    const int row_f4 = 3 * a.out_w / 4;
    const int b = kFlip ? m.adj + 3 * (a.win_w - 1 - PI * p - (RO::T(PO - 1) + 1)) : m.adj + 3 * (PI * p + RO::T(0));
    int offl[PO];  // general map: left-tap byte offsets in a staged row (crop A's flip mirrors them)
    if constexpr (RO::kGen) {
#pragma unroll
      for (int c = 0; c < PO; ++c) offl[c] = m.adj + 3 * (kFlip ? a.win_w - 1 - xl[c] : xl[c]);
    }
    auto hrow = [&](const uint8_t* row, f32x2(&H)[kP]) {
      if constexpr (RO::kGen) RO::template hrow_gen<kFlip>(row, offl, H, wx2, k);
      else RO::template hrow<kFlip>(row, b, H, wx2, k);
    };
    f32x2 A[kP], B[kP];
#pragma unroll
    for (int i = 0; i < kP; ++i) B[i] = splat2(0.0f);
    int r = r_lo;
    int sr = tp[r].y0;
    const int s_last = tp[r_hi - 1].y1;
    hrow(stage + (sr - m.wy_lo) * a.stage_stride, A);
    for (;;) {
      if (sr + 1 <= s_last) hrow(stage + (sr + 1 - m.wy_lo) * a.stage_stride, B);
      while (r < r_hi && tp[r].y0 == sr) emit<kVec>(a, tp, r++, orow, row_f4, A, B);
      if (r >= r_hi) break;
      ++sr;
      if (sr + 1 <= s_last) hrow(stage + (sr + 1 - m.wy_lo) * a.stage_stride, A);
      while (r < r_hi && tp[r].y0 == sr) emit<kVec>(a, tp, r++, orow, row_f4, B, A);
      if (r >= r_hi) break;
      ++sr;
    }
  }

  __device__ void item(const RollArgs& a, const RollMeta& m, const uint8_t* stage, const RollTap* taps) {
    const int r_lo = static_cast<int>((static_cast<int64_t>(run) * m.nrows) / a.runs);
    const int r_hi = static_cast<int>((static_cast<int64_t>(run + 1) * m.nrows) / a.runs);
    if (r_lo >= r_hi) return;
    if (m.ox1 != g_ox1 || m.f1 != g_f1) geometry(a, m);
    const RollTap* tp = taps + m.oy1 + m.band * a.band_rows;
    if (vec) {
      if (m.f0) walk<true, true>(a, m, stage, tp, r_lo, r_hi);
      else walk<false, true>(a, m, stage, tp, r_lo, r_hi);
    } else {
      if (m.f0) walk<true, false>(a, m, stage, tp, r_lo, r_hi);
      else walk<false, false>(a, m, stage, tp, r_lo, r_hi);
    }
  }
};

template <int PO, int PI, int kOp>
__global__ void __launch_bounds__(kRollMaxWarps * 32 + 32, 1) roll_kernel(RollArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kRollMaxStages], empty[kRollMaxStages];
  __shared__ RollMeta meta[kRollMaxStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  RollTap* taps = reinterpret_cast<RollTap*>(smem + a.taps_offset);
  for (int m = tid; m < a.mid_h; m += blockDim.x) {
    RollTap t;
    roll_coord(m, a.win_h, a.scale_y, t.y0, t.y1, t.wy);
    if (t.y1 == t.y0) t.wy = 0.0f;
    taps[m] = t;
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], a.cons_warps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t total = a.rows * a.bands;
  if (warp == a.cons_warps) {  // ---- producer warp ----
    const uint64_t pol = policy_evict_first();
    const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
    for (int64_t k0 = 0;; k0 += 32) {
      const int64_t item = blockIdx.x + (k0 + lane) * static_cast<int64_t>(gridDim.x);
      RollPlan p{};
      p.id = -1;
      if (item < total) {
        p.j = item / a.bands;
        p.band = static_cast<int>(item - p.j * a.bands);
        const int64_t row = a.order ? a.order[a.first + p.j] : a.first + p.j;
        const bool valid = row >= 0 && row < a.num_images;  // engine orders are in range by construction
        p.row = row;
        p.nrows = min(a.band_rows, a.out_h - p.band * a.band_rows);
        int oy0 = 0, ox0 = 0;
        if (valid) {
          p.id = a.ids.of(row);
          if (a.pre_mode == 1) {
            const CropParams cp = crop_params(a.pre_seed, p.id, a.in_h, a.in_w, a.win_h, a.win_w);
            oy0 = cp.oy;
            ox0 = cp.ox;
            p.f0 = a.pre_flip ? cp.flip : 0;
          } else if (a.pre_mode == 2) {
            oy0 = (a.in_h - a.win_h) / 2;
            ox0 = (a.in_w - a.win_w) / 2;
          }
          if (a.post_mode == 1) {
            const CropParams cp = crop_params(a.post_seed, p.id, a.mid_h, a.mid_w, a.out_h, a.out_w);
            p.oy1 = cp.oy;
            p.ox1 = cp.ox;
            p.f1 = a.post_flip ? cp.flip : 0;
          } else if (a.post_mode == 2) {
            p.oy1 = (a.mid_h - a.out_h) / 2;
            p.ox1 = (a.mid_w - a.out_w) / 2;
          }
          const int m_lo = p.oy1 + p.band * a.band_rows;
          p.wy_lo = taps[m_lo].y0;
          p.nsrc = taps[m_lo + p.nrows - 1].y1 - p.wy_lo + 1;
          p.src_row = oy0 + p.wy_lo;
          p.col0 = (3 * ox0) & ~15;
          p.bytes_row = ((3 * (ox0 + a.win_w) + 15) & ~15) - p.col0;
          p.adj = 3 * ox0 - p.col0;
        }
      }
      const int n = __popc(__ballot_sync(0xffffffffu, item < total));
      for (int t = 0; t < n; ++t) {
        const int64_t k = k0 + t;
        const int s = static_cast<int>(k % a.stages);
        if (k >= a.stages) mbar_wait(&empty[s], static_cast<uint32_t>((k / a.stages) - 1) & 1);
        const RollPlan q = shfl_plan(p, t);
        const bool valid = q.id >= 0;
        uint8_t* dst = smem + static_cast<size_t>(s) * a.stage_bytes + 16;
        if (lane == 0) {
          meta[s] = RollMeta{q.id, q.j, q.band, q.nrows, q.wy_lo, q.adj, q.f0, q.ox1, q.f1, q.oy1};
          mbar_arrive_expect_tx(&full[s], valid ? static_cast<uint32_t>(q.nsrc * q.bytes_row) : 0u);
        }
        __syncwarp();
        if (valid) {
          const uint8_t* src = a.images + (static_cast<size_t>(q.row) * a.in_h + q.src_row) * row_bytes + q.col0;
          if (static_cast<size_t>(q.bytes_row) == row_bytes) {  // whole rows: one contiguous copy
            if (lane == 0) bulk_g2s(dst, src, static_cast<uint32_t>(q.nsrc * q.bytes_row), &full[s], pol);
          } else {
            for (int r = lane; r < q.nsrc; r += 32)
              bulk_g2s(dst + r * a.stage_stride, src + r * row_bytes, static_cast<uint32_t>(q.bytes_row), &full[s],
                       pol);
          }
        }
        __syncwarp();
      }
      if (n < 32) break;
    }
    return;
  }
  if (warp > a.cons_warps) return;

  // ---- consumer warps: warp = run * stripes + stripe ----
  RollWarp<PO, PI, kOp> w;
  w.init(a, smem, warp, lane);
  int kq = 0;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x, ++kq) {
    const int s = kq % a.stages;
    mbar_wait(&full[s], (kq / a.stages) & 1);
    const RollMeta m = meta[s];
    if (m.id >= 0 && m.band == 0 && warp == 0 && lane == 0) a.out_ids[m.j] = m.id;
    if (m.id >= 0) w.item(a, m, smem + static_cast<size_t>(s) * a.stage_bytes + 16, taps);
    __syncwarp();
    if (lane == 0) roll_arrive(&empty[s]);
  }
}

// ---- host ----

float coord_scale(int in, int out) { return static_cast<float>(in) / static_cast<float>(out); }

// host twin of roll_coord
void host_coord(int d, int in, float scale, int& i0, int& i1) {
  float s = (static_cast<float>(d) + 0.5f) * scale - 0.5f;
  if (s < 0.0f) s = 0.0f;
  int a = static_cast<int>(s);
  if (a > in - 1) a = in - 1;
  i0 = a;
  i1 = a + 1 < in ? a + 1 : in - 1;
}

template <int PO, int PI>
bool periodic_map(int win_w, int mid_w) {
  if (win_w % PI || mid_w % PO || win_w / PI != mid_w / PO) return false;
  const float scale = coord_scale(win_w, mid_w);
  for (int x = 0; x < mid_w; ++x) {
    int x0, x1;
    host_coord(x, win_w, scale, x0, x1);
    const int xf = PI * (x / PO) + Roll<PO, PI, 0>::T(x % PO);
    const bool left_clamp = xf == -1 && x0 == 0;  // s < 0 clamped to 0: weight 0 -> (p(-1), p(0)) at weight 1
    if (x0 != xf && !left_clamp) return false;
    if (x1 != x0 + 1 && x1 != x0) return false;
  }
  return true;
}

int roll_env(const char* name, int fallback);

bool roll_in_device_memory(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // HBM, or pinned host memory: the TMA engine reads it over PCIe in bulk
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged ||
         (attr.type == cudaMemoryTypeHost && roll_env("DP_DEV_TMA_HOST", 1));
}

int roll_env(const char* name, int fallback) {  // development-only knob overrides (tools/dev)
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : fallback;
}

int roll_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int PO, int PI, int kOp>
int roll_launch(const RollArgs& a, size_t smem, cudaStream_t s) {
  auto kernel = roll_kernel<PO, PI, kOp>;
  static std::atomic<int> dev_set{-1};  // the smem attribute, set again when the device changes
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_set.load(std::memory_order_relaxed) != dev) {
    const int rc = cuda_status(
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kRollSmemMax)),
        "image_chain (roll) smem attribute");
    if (rc) return rc;
    dev_set.store(dev, std::memory_order_relaxed);
  }
  const int64_t items = a.rows * a.bands;
  const int grid = static_cast<int>(std::min<int64_t>(items, roll_sm_count()));
  kernel<<<grid, (a.cons_warps + 1) * 32, smem, s>>>(a);
  return launch_status("image_chain (roll)");
}

// The kernel's configuration for a chain (no buffers yet); false when the
// chain is not K10's.
struct RollPlanHost {
  RollArgs a;
  size_t smem;
  int PO, PI, op;
};

bool roll_plan(const dp_image_chain* c, int out_h, int out_w, RollPlanHost& h, bool allow_general) {
  if (!c->resize || c->num_pre_ops != 0 || c->num_post_ops > 2 || !roll_env("DP_DEV_ROLL", 1)) return false;
  const size_t row_bytes = static_cast<size_t>(c->in_w) * 3;
  if (row_bytes % 16 || out_w % 4) return false;
  RollArgs& a = h.a;
  a = RollArgs{};
  a.in_h = c->in_h;
  a.in_w = c->in_w;
  a.win_h = c->pre_mode ? c->pre_h : c->in_h;
  a.win_w = c->pre_mode ? c->pre_w : c->in_w;
  a.mid_h = c->rs_h;
  a.mid_w = c->rs_w;
  a.out_h = out_h;
  a.out_w = out_w;
  a.pre_mode = c->pre_mode;
  a.pre_flip = c->pre_flip;
  a.pre_seed = c->pre_seed;
  a.post_mode = c->post_mode;
  a.post_flip = c->post_flip;
  a.post_seed = c->post_seed;
  a.scale_y = coord_scale(a.win_h, a.mid_h);
  a.scale_x = coord_scale(a.win_w, a.mid_w);
  // the periodic column map
  int PO = 0, PI = 0;
  if (periodic_map<7, 10>(a.win_w, a.mid_w)) PO = 7, PI = 10;
  else if (periodic_map<7, 8>(a.win_w, a.mid_w)) PO = 7, PI = 8;
  else if (periodic_map<7, 5>(a.win_w, a.mid_w)) PO = 7, PI = 5;
  else if (periodic_map<8, 10>(a.win_w, a.mid_w)) PO = 8, PI = 10;  // 5:4 as two periods per lane (24 floats)
  else if (periodic_map<7, 9>(a.win_w, a.mid_w)) PO = 7, PI = 9;     // 288 -> 224
  else if (periodic_map<7, 12>(a.win_w, a.mid_w)) PO = 7, PI = 12;   // 384 -> 224
  else if (periodic_map<7, 6>(a.win_w, a.mid_w)) PO = 7, PI = 6;     // 192 -> 224
  else if (periodic_map<7, 4>(a.win_w, a.mid_w)) PO = 7, PI = 4;     // 128 -> 224
  else if (periodic_map<8, 12>(a.win_w, a.mid_w)) PO = 8, PI = 12;   // 3:2, e.g. 384 -> 256
  else if (periodic_map<8, 16>(a.win_w, a.mid_w)) PO = 8, PI = 16;   // 2:1
  // any other ratio of a chain: runtime taps (against K9: 240 -> 176 6.2 vs
  // 3.8 M img/s, 176 -> 224 5.7 vs 4.7); dp_k_resize_normalize_batch keeps
  // K4 for them (300 -> 224: K4 5.0, this form 4.1 M img/s)
  else if ((allow_general || roll_env("DP_DEV_K4_GENERAL", 0)) && roll_env("DP_DEV_ROLL_GENERAL", 1))
    PO = 8, PI = 0;
  else return false;
  // two pixel ops: the general form only (one instantiation set)
  if (c->num_post_ops == 2) {
    if (!allow_general || !roll_env("DP_DEV_ROLL_GENERAL", 1)) return false;
    PO = 8, PI = 0;
  }
  // the pixel op
  int op = 0;
  if (c->num_post_ops == 1) {
    for (int ch = 0; ch < 3; ++ch) {
      a.op_a[ch] = c->op_a[0][ch];
      a.op_b[ch] = c->op_b[0][ch];
      a.op_r[ch] = 1.0f / c->op_b[0][ch];  // RN(1 / std)
    }
    op = c->op_kind[0] == 1 ? 2 : (fast_div_proven(a.op_a, a.op_b) ? 1 : 3);
  }
  if (c->num_post_ops == 2) {
    for (int ch = 0; ch < 3; ++ch) {
      a.op_a[ch] = c->op_a[0][ch];
      a.op_b[ch] = c->op_b[0][ch];
      a.op_r[ch] = 1.0f / c->op_b[0][ch];
      a.op2_a[ch] = c->op_a[1][ch];
      a.op2_b[ch] = c->op_b[1][ch];
    }
    op = (c->op_kind[0] == 1 ? 2 : (fast_div_proven(a.op_a, a.op_b) ? 1 : 3)) + 4 * (c->op_kind[1] == 1 ? 2 : 3);
  }
  // stripes: output pixel ranges (multiples of 4) whose mid columns span <= 32 periods
  // for every crop-B offset the chain can draw
  const bool exact = c->post_mode != 1;  // crop B at a fixed offset (none / center): exact period count
  auto periods = [&](int lo, int hi) {
    if (!exact) return (hi - lo + PO - 1) / PO + 1;
    const int ox1 = c->post_mode == 2 ? (a.mid_w - out_w) / 2 : 0;
    return (ox1 + hi - 1) / PO - (ox1 + lo) / PO + 1;
  };
  a.stripes = 0;
  for (int n = 1; n <= kRollMaxStripes && !a.stripes; ++n) {
    bool fits = true;
    for (int t = 0; t < n && fits; ++t) {
      const int lo = ((t * out_w / n) / 4) * 4, hi = t + 1 == n ? out_w : (((t + 1) * out_w / n) / 4) * 4;
      fits = hi > lo && periods(lo, hi) <= 32;
    }
    if (!fits) continue;
    a.stripes = n;
    for (int t = 0; t < n; ++t) a.stripe_px[t] = ((t * out_w / n) / 4) * 4;
    a.stripe_px[n] = out_w;
  }
  if (!a.stripes) return false;
  const int warps = roll_env("DP_DEV_ROLL_WARPS", kRollMaxWarps);
  a.runs = std::max(1, warps / a.stripes);
  a.cons_warps = a.runs * a.stripes;
  if (a.cons_warps > kRollMaxWarps) return false;
  // bands: ~run_rows output rows per run, spread evenly over the image;
  // shorter runs when a ring of 2 stages does not fit
  const double scale = static_cast<double>(a.win_h) / a.mid_h;
  a.stage_stride = static_cast<int>(std::min<size_t>(row_bytes, ((3 * a.win_w + 15 + 15) / 16) * 16));
  if (a.win_w == c->in_w) a.stage_stride = static_cast<int>(row_bytes);
  a.buf_floats = ((3 * (a.stripe_px[1] - a.stripe_px[0]) + 3) / 4) * 4;
  for (int st = 1; st < a.stripes; ++st)
    a.buf_floats = std::max(a.buf_floats, ((3 * (a.stripe_px[st + 1] - a.stripe_px[st]) + 3) / 4) * 4);
  const size_t taps = ((static_cast<size_t>(a.mid_h) * sizeof(RollTap) + 127) / 128) * 128;
  const size_t bufs = static_cast<size_t>(a.cons_warps) * (a.buf_floats + 128) * sizeof(float);  // + trash slots
  const int want_stages = std::min(kRollMaxStages, std::max(2, roll_env("DP_DEV_ROLL_STAGES", kRollMaxStages)));
  size_t smem = 0;
  // tools/dev sweep: runs of 8 rows best for 160 -> 224 and 320 -> 256
  for (int run_rows = roll_env("DP_DEV_ROLL_RUN", 8); run_rows >= 1; --run_rows) {
    a.bands = std::max(1, (out_h + a.runs * run_rows - 1) / (a.runs * run_rows));
    a.band_rows = (out_h + a.bands - 1) / a.bands;
    a.bands = (out_h + a.band_rows - 1) / a.band_rows;
    const int max_src = std::min(a.win_h, static_cast<int>(a.band_rows * scale) + 3);
    a.stage_bytes = ((16 + max_src * a.stage_stride + 16 + 127) / 128) * 128;
    a.stages = want_stages;
    while (a.stages > 2 && static_cast<size_t>(a.stages) * a.stage_bytes + taps + bufs > kRollSmemMax) --a.stages;
    smem = static_cast<size_t>(a.stages) * a.stage_bytes + taps + bufs;
    if (smem <= kRollSmemMax && a.stages >= 2) break;
  }
  if (smem > kRollSmemMax || a.stages < 2) return false;
  a.taps_offset = a.stages * a.stage_bytes;
  a.buf_offset = static_cast<int>(a.taps_offset + taps);
  a.nc = NormConsts{};
  h.smem = smem;
  h.PO = PO;
  h.PI = PI;
  h.op = op;
  return true;
}

}  // namespace

// Returns DP_OK after launching, 1 when the chain is not this kernel's
// (the caller uses K9), or an error status.
int roll_chain_batch(const uint8_t* images, int64_t num_images, const int64_t* order, int64_t first, int64_t rows,
                     int64_t id_base, int64_t id_stride, int64_t id_block, const dp_image_chain* c, int out_h,
                     int out_w, int64_t* out_ids, float* out, cudaStream_t stream, bool allow_general) {
  if (reinterpret_cast<uintptr_t>(images) % 16 || reinterpret_cast<uintptr_t>(out) % 16 ||
      !roll_in_device_memory(images))
    return 1;
  RollPlanHost h;
  if (!roll_plan(c, out_h, out_w, h, allow_general)) return 1;
  RollArgs& a = h.a;
  a.images = images;
  a.order = order;
  a.first = first;
  a.rows = rows;
  a.num_images = num_images;
  a.out_ids = out_ids;
  a.out = out;
  a.ids = RollIds{id_base, id_stride, id_block};
  if (rows == 0) return DP_OK;
#define DP_ROLL(PO_, PI_)                                                        \
  if (h.PO == PO_ && h.PI == PI_) {                                              \
    switch (h.op) {                                                              \
      case 0: return roll_launch<PO_, PI_, 0>(a, h.smem, stream);                \
      case 1: return roll_launch<PO_, PI_, 1>(a, h.smem, stream);                \
      case 2: return roll_launch<PO_, PI_, 2>(a, h.smem, stream);                \
      case 3: return roll_launch<PO_, PI_, 3>(a, h.smem, stream);                \
      default: break;                                                            \
    }                                                                            \
  }
  DP_ROLL(7, 10)
  DP_ROLL(7, 8)
  DP_ROLL(7, 5)
  DP_ROLL(8, 10)
  DP_ROLL(7, 9)
  DP_ROLL(7, 12)
  DP_ROLL(7, 6)
  DP_ROLL(7, 4)
  DP_ROLL(8, 12)
  DP_ROLL(8, 16)
  DP_ROLL(8, 0)
#undef DP_ROLL
  if (h.PO == 8 && h.PI == 0) {  // two pixel ops (general form)
    switch (h.op) {
      case 1 + 8: return roll_launch<8, 0, 1 + 8>(a, h.smem, stream);
      case 2 + 8: return roll_launch<8, 0, 2 + 8>(a, h.smem, stream);
      case 3 + 8: return roll_launch<8, 0, 3 + 8>(a, h.smem, stream);
      case 1 + 12: return roll_launch<8, 0, 1 + 12>(a, h.smem, stream);
      case 2 + 12: return roll_launch<8, 0, 2 + 12>(a, h.smem, stream);
      case 3 + 12: return roll_launch<8, 0, 3 + 12>(a, h.smem, stream);
      default: break;
    }
  }
  return 1;
}

bool roll_chain_eligible(const dp_image_chain* c, int out_h, int out_w, bool allow_general) {
  RollPlanHost h;
  return roll_plan(c, out_h, out_w, h, allow_general);
}

}  // namespace dpk

extern "C" int dp_image_chain_kernel(const dp_image_chain* chain, int* kernel) {
  int oh, ow, f32;
  if (!kernel) return dpk::fail(DP_ERR_INVALID_ATTR, "image_chain_kernel: null argument");
  const int st = dp_image_chain_output(chain, &oh, &ow, &f32);
  if (st) return st;
  *kernel = f32 && dpk::roll_chain_eligible(chain, oh, ow, true) ? 10 : 9;
  return DP_OK;
}
