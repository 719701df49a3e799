// k_chain.cu -- K9: the general image map chain fused with Batch, and the
// plain u8 gather of a Batch with no map.
//
// The reference applies one opaque MapFn per map node per element
// (/root/reference/proj/src/runtime.cpp:480-535, udf.hpp:31) and batches the
// results (MapAndBatchIterator, runtime.cpp:1467-1721).  The device UDF
// library's chains that K3 (crop+flip+normalize) and K4 (resize+normalize)
// do not cover are lowered into ONE descriptor (dp_image_chain):
//     [crop A] [pixel ops] [resize] [crop B] [pixel ops]
// -- crops / flips are coordinate maps, pixel ops (normalize, affine, cast)
// are per-channel pointwise and commute with them, so only their position
// relative to the resize matters.  Every output value is computed from its
// source taps with the same rounded fp32 ops, in the same order, as the
// sequential restatement (oracle/chain.c); u8 stays u8 through crops.
//
// Both kernels are HBM-bound.  K9 chain: a CTA owns a band of output rows of
// one image, stages the source rows x window columns the band reads into
// shared memory with 16-byte non-allocating loads, then each thread writes
// 16-byte (fp32) / 4-byte (u8) streaming stores.  K9 gather: one CTA per
// (image, 48 KB chunk), 16-byte loads / streaming stores.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "common.cuh"
#include "fastdiv.hpp"
#include "roll.hpp"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;
constexpr size_t kChainSmem = 96 * 1024;  // staged bytes per CTA (2 CTAs per SM)

struct ChainIds {
  int64_t base, stride, block;
  __device__ __forceinline__ int64_t of(int64_t r) const {
    if (block == 1) return base + r * stride;
    const int64_t q = r / block;
    return (q * stride + base) * block + (r - q * block);
  }
};

struct ChainArgs {
  const uint8_t* images;
  const int64_t* order;
  int64_t first, num_images;
  int64_t* out_ids;
  void* out;
  dp_image_chain c;
  int out_h, out_w, win_h, win_w, mid_h, mid_w;
  int band_rows, bands, stage_cols;  // stage_cols: staged bytes per source row (multiple of 16 when aligned)
  float scale_y, scale_x;            // resize: win / mid, rounded once
  int h_offset;                      // resize: byte offset of the horizontal-pass rows in shared memory
  // ops normalizing values known to lie in [0, 255] with constants the
  // exhaustive proof covers (tools/prove_fast_div.c): the two-FMA exact
  // division with rcp = RN(1 / std) instead of the general IEEE sequence
  unsigned fast_mask;
  float op_rcp[4][3];
  ChainIds ids;
};

// Half-pixel-centre source coordinate (oracle/chain.c chain_coord), the
// scale in / out precomputed (IEEE division on the host = __fdiv_rn).
__device__ __forceinline__ void chain_coord(int d, int in, float scale, int& i0, int& i1, float& w) {
  float s = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(d), 0.5f), scale), 0.5f);
  if (s < 0.0f) s = 0.0f;
  int a = static_cast<int>(s);
  if (a > in - 1) a = in - 1;
  i0 = a;
  i1 = a + 1 < in ? a + 1 : in - 1;
  w = __fsub_rn(s, static_cast<float>(a));
}

// Pixel ops [from, from + n) on one value; constants a[k], b[k] (and
// r[k] = RN(1 / b[k]) for the proven-exact fast division, bit k of `fast`)
// of the value's channel, in registers; kinds a bit mask (bit k: affine).
// kN >= 0: unrolled at compile time; -1: the runtime count n.
template <int kN>
__device__ __forceinline__ float apply_ops(const float* a, const float* b, const float* r, unsigned kinds,
                                           unsigned fast, int from, int n, float v) {
#pragma unroll
  for (int i = 0; i < (kN >= 0 ? kN : 4); ++i) {
    if (kN < 0 && i >= n) break;
    const int k = from + i;
    if ((kinds >> k) & 1u) v = __fadd_rn(__fmul_rn(v, a[k]), b[k]);  // x * scale + shift
    else if ((fast >> k) & 1u) v = normalize_fast(v, a[k], b[k], r[k]);  // (x - mean) / std, proven exact
    else v = __fdiv_rn(__fsub_rn(v, a[k]), b[k]);                       // (x - mean) / std, IEEE
  }
  return v;
}

struct Geo {
  int oy0, ox0, f0, oy1, ox1, f1;
};

__device__ __forceinline__ Geo chain_geo(const ChainArgs& a, int64_t id) {
  Geo g{0, 0, 0, 0, 0, 0};
  const dp_image_chain& c = a.c;
  if (c.pre_mode == 1) {
    const CropParams p = crop_params(c.pre_seed, id, c.in_h, c.in_w, c.pre_h, c.pre_w);
    g.oy0 = p.oy;
    g.ox0 = p.ox;
    g.f0 = c.pre_flip ? p.flip : 0;
  } else if (c.pre_mode == 2) {
    g.oy0 = (c.in_h - c.pre_h) / 2;
    g.ox0 = (c.in_w - c.pre_w) / 2;
  }
  if (c.post_mode == 1) {
    const CropParams p = crop_params(c.post_seed, id, a.mid_h, a.mid_w, c.post_h, c.post_w);
    g.oy1 = p.oy;
    g.ox1 = p.ox;
    g.f1 = c.post_flip ? p.flip : 0;
  } else if (c.post_mode == 2) {
    g.oy1 = (a.mid_h - c.post_h) / 2;
    g.ox1 = (a.mid_w - c.post_w) / 2;
  }
  return g;
}

// source row (image coordinates) of window row wy
__device__ __forceinline__ int first_src_row(const ChainArgs& a, const Geo& g, int my) {
  if (!a.c.resize) return g.oy0 + my;
  int y0, y1;
  float w;
  chain_coord(my, a.win_h, a.scale_y, y0, y1, w);
  return g.oy0 + y0;
}
__device__ __forceinline__ int last_src_row(const ChainArgs& a, const Geo& g, int my) {
  if (!a.c.resize) return g.oy0 + my;
  int y0, y1;
  float w;
  chain_coord(my, a.win_h, a.scale_y, y0, y1, w);
  return g.oy0 + y1;
}

// Thread layout: thread t owns output column group q = t % qn (4
// consecutive values of a row: one float4 / one 4-byte u8 word; the
// unaligned variant owns 1 value) and rows rsub = t / qn, rsub + rpp, ...
// of the band, so the column taps of its values (window byte offsets,
// weights, channels) are computed once per CTA and live in registers; the
// row loop is smem byte loads, the rounded lerp / pixel-op sequence and one
// streaming store.
template <typename OutT, bool kAligned, bool kResize, int kPre, int kPost>
__global__ void __launch_bounds__(1024, 1) chain_kernel(ChainArgs a) {
  extern __shared__ __align__(16) uint8_t stage[];
  __shared__ float opc[4][9];
  __shared__ int rtap_row[2][64];
  __shared__ float rtap_w[64];
  constexpr int kVec = kAligned ? 4 : 1;
  if (threadIdx.x < 36) {
    const int k = threadIdx.x / 9, i = threadIdx.x % 9;
    opc[k][i] = i < 3 ? a.c.op_a[k][i] : i < 6 ? a.c.op_b[k][i - 3] : a.op_rcp[k][i - 6];
  }
  unsigned kinds = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) kinds |= (a.c.op_kind[k] == 1 ? 1u : 0u) << k;
  const int band = blockIdx.x % a.bands;
  const int64_t j = blockIdx.x / a.bands;
  const int64_t row = a.order ? a.order[a.first + j] : a.first + j;
  if (row < 0 || row >= a.num_images) return;  // engine orders are in range by construction
  const int64_t id = a.ids.of(row);
  if (band == 0 && threadIdx.x == 0) a.out_ids[j] = id;
  const dp_image_chain& c = a.c;
  const Geo g = chain_geo(a, id);

  const int y_begin = band * a.band_rows;
  const int nrows = min(a.band_rows, a.out_h - y_begin);
  const int sy_lo = first_src_row(a, g, g.oy1 + y_begin);
  const int sy_hi = last_src_row(a, g, g.oy1 + y_begin + nrows - 1);
  const size_t row_bytes = static_cast<size_t>(c.in_w) * 3;
  // first staged byte of a source row: 16-byte aligned, the staged span kept
  // inside the row (stage_cols <= row bytes, both multiples of 16)
  const int col0 = kAligned ? min((g.ox0 * 3) & ~15, static_cast<int>(row_bytes) - a.stage_cols) : g.ox0 * 3;
  const uint8_t* src = a.images + (static_cast<size_t>(row) * c.in_h + sy_lo) * row_bytes + col0;
  const int srows = sy_hi - sy_lo + 1;
  if (kAligned) {
    const int chunks = a.stage_cols >> 4;
    for (int t = threadIdx.x; t < srows * chunks; t += blockDim.x) {
      const int r = t / chunks, q = t - r * chunks;
      *reinterpret_cast<uint4*>(stage + r * a.stage_cols + q * 16) =
          ld_nc_na_u4(src + static_cast<size_t>(r) * row_bytes + q * 16);
    }
  } else {
    for (int t = threadIdx.x; t < srows * a.stage_cols; t += blockDim.x) {
      const int r = t / a.stage_cols, q = t - r * a.stage_cols;
      stage[r * a.stage_cols + q] = src[static_cast<size_t>(r) * row_bytes + q];
    }
  }

  // this thread's column taps (overlaps the staging loads in flight)
  const int seg = a.out_w * 3;
  const int qn = (seg + kVec - 1) / kVec;
  const int q = threadIdx.x % qn, rsub = threadIdx.x / qn, rpp = blockDim.x / qn;
  const int shift = g.ox0 * 3 - col0;
  int off0[kVec], off1[kVec], chs[kVec];
  float wxs[kVec];
  constexpr int kOps = kPre >= 0 && kPost >= 0 ? kPre + kPost : 4;  // op constants held per value
  float opa[kVec][kOps > 0 ? kOps : 1], opb[kVec][kOps > 0 ? kOps : 1], opr[kVec][kOps > 0 ? kOps : 1];
  const unsigned fast = a.fast_mask;
#pragma unroll
  for (int u = 0; u < kVec; ++u) {
    int e = kVec * q + u;
    if (e >= seg) e = seg - 1;  // (unaligned tail: computed, not stored)
    const int x = e / 3, ch = e - 3 * x;
    const int mx = g.ox1 + (g.f1 ? a.out_w - 1 - x : x);
    int x0 = mx, x1 = mx;
    float wx = 0.0f;
    if (kResize) chain_coord(mx, a.win_w, a.scale_x, x0, x1, wx);
    off0[u] = shift + (g.f0 ? a.win_w - 1 - x0 : x0) * 3 + ch;
    off1[u] = shift + (g.f0 ? a.win_w - 1 - x1 : x1) * 3 + ch;
    wxs[u] = wx;
    chs[u] = ch;
  }
  __syncthreads();  // the op table
#pragma unroll
  for (int u = 0; u < kVec; ++u)
#pragma unroll
    for (int k = 0; k < kOps; ++k) {
      opa[u][k] = opc[k][chs[u]];
      opb[u][k] = opc[k][3 + chs[u]];
      opr[u][k] = opc[k][6 + chs[u]];
    }
  __syncthreads();  // (blockDim = qn * rpp: every thread has a column group and a row phase)

  OutT* obase = static_cast<OutT*>(a.out) + (static_cast<size_t>(j) * a.out_h + y_begin) * seg;
  const int np = c.num_pre_ops, npost = c.num_post_ops;
  if constexpr (kResize) {
    // the band's row taps, once (rows <= 64 by construction)
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
      int y0, y1;
      float wy;
      chain_coord(g.oy1 + y_begin + r, a.win_h, a.scale_y, y0, y1, wy);
      rtap_row[0][r] = (g.oy0 + y0 - sy_lo) * seg;
      rtap_row[1][r] = (g.oy0 + y1 - sy_lo) * seg;
      rtap_w[r] = wy;
    }
    // Separable: the horizontal blend of a (window row, output column) pair
    // is the same rounded value for every output row that reads it, so it
    // is computed once per staged row into shared memory (H), then each
    // output value is one vertical blend of two H rows -- the same ops in
    // the same order as p00..p11 -> top, bot -> v.
    float* H = reinterpret_cast<float*>(stage + a.h_offset);
    for (int r = rsub; r < srows; r += rpp) {
      const uint8_t* sr = stage + r * a.stage_cols;
      float v[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u) {
        const int ch = chs[u];
        const float p0 = apply_ops<kPre>(opa[u], opb[u], opr[u], kinds, fast, 0, np, u8_to_f32(sr[off0[u]]));
        const float p1 = apply_ops<kPre>(opa[u], opb[u], opr[u], kinds, fast, 0, np, u8_to_f32(sr[off1[u]]));
        v[u] = __fadd_rn(p0, __fmul_rn(wxs[u], __fsub_rn(p1, p0)));
      }
      if (kAligned) reinterpret_cast<float4*>(H + r * seg)[q] = make_float4(v[0], v[1], v[2], v[3]);
      else if (q < seg) H[r * seg + q] = v[0];
    }
    __syncthreads();
    for (int r = rsub; r < nrows; r += rpp) {
      const float wy = rtap_w[r];
      const float* h0 = H + rtap_row[0][r];
      const float* h1 = H + rtap_row[1][r];
      OutT* orow = obase + static_cast<size_t>(r) * seg;
      if (kAligned) {
        const float4 t4 = reinterpret_cast<const float4*>(h0)[q], b4 = reinterpret_cast<const float4*>(h1)[q];
        const float t[4] = {t4.x, t4.y, t4.z, t4.w}, b[4] = {b4.x, b4.y, b4.z, b4.w};
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = apply_ops<kPost>(opa[u], opb[u], opr[u], kinds, fast, kPre >= 0 ? kPre : np, npost, __fadd_rn(t[u], __fmul_rn(wy, __fsub_rn(b[u], t[u]))));
        st_cs_f4(reinterpret_cast<float4*>(orow) + q, make_float4(v[0], v[1], v[2], v[3]));
      } else if (q < seg) {
        const float t = h0[q], b = h1[q];
        orow[q] = apply_ops<kPost>(opa[0], opb[0], opr[0], kinds, fast, kPre >= 0 ? kPre : np, npost, __fadd_rn(t, __fmul_rn(wy, __fsub_rn(b, t))));
      }
    }
    return;
  }
  for (int r = rsub; r < nrows; r += rpp) {
    const int my = g.oy1 + y_begin + r;
    const uint8_t* r0 = stage + (g.oy0 + my - sy_lo) * a.stage_cols;
    OutT* orow = obase + static_cast<size_t>(r) * seg;
    if constexpr (sizeof(OutT) == 1) {  // u8: crops only (no resize, no ops)
      if (kAligned) {
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < kVec; ++u) w |= static_cast<uint32_t>(r0[off0[u]]) << (8 * u);
        __stcs(reinterpret_cast<unsigned int*>(orow) + q, w);
      } else if (q < seg) {
        orow[q] = r0[off0[0]];
      }
    } else {
      float v[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u) v[u] = apply_ops<kPre>(opa[u], opb[u], opr[u], kinds, fast, 0, np, u8_to_f32(r0[off0[u]]));
      if (kAligned) st_cs_f4(reinterpret_cast<float4*>(orow) + q, make_float4(v[0], v[1], v[2], v[3]));
      else if (q < seg) orow[q] = v[0];
    }
  }
}

// K9 gather: out[j] = images[order[first + j]], bytes as they are.
constexpr int kCopyChunk = 48 * 1024;
template <bool kAligned>
__global__ void __launch_bounds__(kThreads)
gather_copy_kernel(const uint8_t* __restrict__ images, int64_t num_images, int64_t image_bytes,
                   const int64_t* __restrict__ order, int64_t first, int chunks, ChainIds ids,
                   int64_t* __restrict__ out_ids, uint8_t* __restrict__ out) {
  const int64_t j = blockIdx.x / chunks;
  const int chunk = blockIdx.x % chunks;
  const int64_t row = order ? order[first + j] : first + j;
  if (row < 0 || row >= num_images) return;
  if (chunk == 0 && threadIdx.x == 0) out_ids[j] = ids.of(row);
  const int64_t b0 = static_cast<int64_t>(chunk) * kCopyChunk;
  const int64_t b1 = b0 + kCopyChunk < image_bytes ? b0 + kCopyChunk : image_bytes;
  const uint8_t* s = images + row * image_bytes;
  uint8_t* d = out + j * image_bytes;
  if (kAligned) {
    for (int64_t b = b0 + 16 * threadIdx.x; b < b1; b += 16 * kThreads) {
      const uint4 v = ld_nc_na_u4(s + b);
      __stcs(reinterpret_cast<uint4*>(d + b), v);
    }
  } else {
    for (int64_t b = b0 + threadIdx.x; b < b1; b += kThreads) d[b] = s[b];
  }
}

}  // namespace
}  // namespace dpk

using namespace dpk;

extern "C" int dp_image_chain_output(const dp_image_chain* c, int* out_h, int* out_w, int* out_f32) {
  if (!c || !out_h || !out_w || !out_f32) return fail(DP_ERR_INVALID_ATTR, "image_chain: null argument");
  if (c->in_h < 1 || c->in_w < 1) return fail(DP_ERR_INVALID_ATTR, "image_chain: image dims must be >= 1");
  int h = c->in_h, w = c->in_w;
  if (c->pre_mode) {
    if (c->pre_mode < 0 || c->pre_mode > 2 || c->pre_h < 1 || c->pre_w < 1 || c->pre_h > h || c->pre_w > w)
      return fail(DP_ERR_INVALID_ATTR, "image_chain: first crop larger than the image");
    h = c->pre_h;
    w = c->pre_w;
  }
  if (c->resize) {
    if (c->rs_h < 1 || c->rs_w < 1) return fail(DP_ERR_INVALID_ATTR, "image_chain: resize dims must be >= 1");
    h = c->rs_h;
    w = c->rs_w;
  }
  if (c->post_mode) {
    if (c->post_mode < 0 || c->post_mode > 2 || c->post_h < 1 || c->post_w < 1 || c->post_h > h || c->post_w > w)
      return fail(DP_ERR_INVALID_ATTR, "image_chain: second crop larger than its input");
    h = c->post_h;
    w = c->post_w;
  }
  if (c->num_pre_ops < 0 || c->num_post_ops < 0 || c->num_pre_ops + c->num_post_ops > 4 ||
      (!c->resize && c->num_post_ops))
    return fail(DP_ERR_INVALID_ATTR, "image_chain: at most 4 pixel ops (post-resize ops need a resize)");
  for (int k = 0; k < c->num_pre_ops + c->num_post_ops; ++k)
    if (c->op_kind[k] != 0 && c->op_kind[k] != 1) return fail(DP_ERR_INVALID_ATTR, "image_chain: bad op kind");
  const int f32 = c->resize || c->num_pre_ops + c->num_post_ops > 0;
  if (c->out_f32 != f32) return fail(DP_ERR_INVALID_ATTR, "image_chain: out_f32 does not match the chain");
  *out_h = h;
  *out_w = w;
  *out_f32 = f32;
  return DP_OK;
}

extern "C" int dp_k_image_chain_batch(const uint8_t* images, int64_t num_images, const int64_t* order, int64_t first,
                                      int64_t rows, int64_t id_base, int64_t id_stride, int64_t id_block,
                                      const dp_image_chain* chain, int64_t* out_ids, void* out, void* stream) {
  int oh, ow, f32;
  int st = dp_image_chain_output(chain, &oh, &ow, &f32);
  if (st) return st;
  if (rows < 0) return fail(DP_ERR_INVALID_ATTR, "image_chain: rows must be >= 0");
  if (id_stride < 1 || id_block < 1 || id_base < 0 || id_base >= id_stride)
    return fail(DP_ERR_INVALID_ATTR, "image_chain: bad sharded residency (id_base/id_stride/id_block)");
  if (rows == 0) return DP_OK;
  if (!images || !out_ids || !out || num_images < 1) return fail(DP_ERR_INVALID_ATTR, "image_chain: null buffer");
  // resize chains over a periodic column map: K10 (k_roll.cu)
  if (f32) {
    const int rc = roll_chain_batch(images, num_images, order, first, rows, id_base, id_stride, id_block, chain, oh, ow,
                                    out_ids, static_cast<float*>(out), as_stream(stream), true);
    if (rc != 1) return rc;
  }
  ChainArgs a{};
  a.images = images;
  a.order = order;
  a.first = first;
  a.num_images = num_images;
  a.out_ids = out_ids;
  a.out = out;
  a.c = *chain;
  a.out_h = oh;
  a.out_w = ow;
  a.win_h = chain->pre_mode ? chain->pre_h : chain->in_h;
  a.win_w = chain->pre_mode ? chain->pre_w : chain->in_w;
  a.mid_h = chain->resize ? chain->rs_h : a.win_h;
  a.mid_w = chain->resize ? chain->rs_w : a.win_w;
  a.ids = ChainIds{id_base, id_stride, id_block};
  const size_t row_bytes = static_cast<size_t>(chain->in_w) * 3;
  // vector path: 16-byte staged rows and whole float4 / u8x4 groups per output row
  const bool aligned = row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(images) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(out) % 16 == 0 && (ow * 3) % 4 == 0;
  // staged window columns: the whole window, widened to 16-byte boundaries
  a.stage_cols = aligned ? static_cast<int>(((a.win_w * 3 + 15) / 16 + 1) * 16) : a.win_w * 3;
  if (aligned && static_cast<size_t>(a.stage_cols) > row_bytes) a.stage_cols = static_cast<int>(row_bytes);
  // band rows: the source rows one band reads (u8 stage, + their fp32
  // horizontal blends when resizing) must fit the CTA's shared memory
  const double scale = chain->resize ? static_cast<double>(a.win_h) / a.mid_h : 1.0;
  auto src_rows = [&](int b) { return std::min(chain->resize ? static_cast<int>(b * scale) + 3 : b, chain->in_h); };
  auto stage_bytes = [&](int b) { return ((static_cast<size_t>(src_rows(b)) * a.stage_cols + 15) / 16) * 16; };
  auto smem_for = [&](int b) {
    return stage_bytes(b) + (chain->resize ? static_cast<size_t>(src_rows(b)) * ow * 3 * sizeof(float) : 0);
  };
  int band = 32;  // <= 64: the row-tap table
  while (band > 1 && smem_for(band) > kChainSmem) band /= 2;
  const size_t smem = smem_for(band);
  a.h_offset = static_cast<int>(stage_bytes(band));
  if (smem > 200 * 1024)
    return fail(DP_ERR_INVALID_ATTR, "image_chain: one output row reads more source rows than shared memory holds");
  a.band_rows = std::min(band, oh);
  a.bands = (oh + a.band_rows - 1) / a.band_rows;
  const int64_t grid = rows * a.bands;
  if (grid > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "image_chain: batch too large");
  cudaStream_t s = as_stream(stream);
  const bool vec = aligned;
  const int qn = vec ? ow * 3 / 4 : ow * 3;
  // threads: whole rows of column groups, ~512 per CTA (<= 1024)
  const int rpp = std::max(1, std::min(a.band_rows, qn >= 1024 ? 1 : std::max(1, 512 / qn)));
  const int threads = qn >= 1024 ? 1024 : qn * rpp;
  if (qn > 1024 && !vec) return fail(DP_ERR_INVALID_ATTR, "image_chain: output rows wider than 1024 values");
  auto launch = [&](auto kernel) {
    if (smem > 48 * 1024) {
      const int rc = cuda_status(
          cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
          "image_chain smem attribute");
      if (rc) return rc;
    }
    kernel<<<static_cast<int>(grid), threads, smem, s>>>(a);
    return launch_status("image_chain");
  };
  if (qn > 1024) return fail(DP_ERR_INVALID_ATTR, "image_chain: output rows wider than 4096 values");
  // op 0 sees u8 taps (or their blend when it follows the resize): values
  // in [0, 255]; fast division where its equality with IEEE division is
  // proven for the constants (the ImageNet mean / std and cast's 0 / 1
  // offline by tools/prove_fast_div.c, anything else on the device at first
  // use: fastdiv.hpp)
  {
    const int nops = chain->num_pre_ops + chain->num_post_ops;
    for (int k = 0; k < nops; ++k)
      for (int c = 0; c < 3; ++c) a.op_rcp[k][c] = 1.0f / chain->op_b[k][c];
    if (nops > 0 && chain->op_kind[0] == 0 && fast_div_proven(chain->op_a[0], chain->op_b[0])) a.fast_mask = 1u;
  }
  a.scale_y = static_cast<float>(a.win_h) / static_cast<float>(a.mid_h);
  a.scale_x = static_cast<float>(a.win_w) / static_cast<float>(a.mid_w);
  if (!f32)
    return vec ? launch(chain_kernel<uint8_t, true, false, 0, 0>) : launch(chain_kernel<uint8_t, false, false, 0, 0>);
  const int np = chain->num_pre_ops, npost = chain->num_post_ops;
  // the common structures unrolled; anything else runs the runtime op loop
#define DP_CHAIN(R, PRE, POST)                                                                       \
  if (chain->resize == R && np == PRE && npost == POST)                                              \
    return vec ? launch(chain_kernel<float, true, R, PRE, POST>) : launch(chain_kernel<float, false, R, PRE, POST>);
  DP_CHAIN(1, 0, 0)
  DP_CHAIN(1, 0, 1)
  DP_CHAIN(1, 1, 0)
  DP_CHAIN(1, 0, 2)
  DP_CHAIN(1, 1, 1)
  DP_CHAIN(0, 1, 0)
  DP_CHAIN(0, 2, 0)
#undef DP_CHAIN
  if (chain->resize)
    return vec ? launch(chain_kernel<float, true, true, -1, -1>) : launch(chain_kernel<float, false, true, -1, -1>);
  return vec ? launch(chain_kernel<float, true, false, -1, -1>) : launch(chain_kernel<float, false, false, -1, -1>);
}

extern "C" int dp_k_gather_copy_batch(const uint8_t* images, int64_t num_images, int64_t image_bytes,
                                      const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                      int64_t id_stride, int64_t id_block, int64_t* out_ids, uint8_t* out,
                                      void* stream) {
  if (rows < 0 || image_bytes < 1) return fail(DP_ERR_INVALID_ATTR, "gather_copy: rows >= 0, image_bytes >= 1");
  if (id_stride < 1 || id_block < 1 || id_base < 0 || id_base >= id_stride)
    return fail(DP_ERR_INVALID_ATTR, "gather_copy: bad sharded residency (id_base/id_stride/id_block)");
  if (rows == 0) return DP_OK;
  if (!images || !out_ids || !out || num_images < 1) return fail(DP_ERR_INVALID_ATTR, "gather_copy: null buffer");
  const int chunks = static_cast<int>((image_bytes + kCopyChunk - 1) / kCopyChunk);
  const int64_t grid = rows * chunks;
  if (grid > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "gather_copy: batch too large");
  const bool aligned = image_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(images) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(out) % 16 == 0;
  const ChainIds ids{id_base, id_stride, id_block};
  cudaStream_t s = as_stream(stream);
  if (aligned)
    gather_copy_kernel<true><<<static_cast<int>(grid), kThreads, 0, s>>>(images, num_images, image_bytes, order,
                                                                          first, chunks, ids, out_ids, out);
  else
    gather_copy_kernel<false><<<static_cast<int>(grid), kThreads, 0, s>>>(images, num_images, image_bytes, order,
                                                                           first, chunks, ids, out_ids, out);
  return launch_status("gather_copy");
}
