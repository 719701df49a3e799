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
#include <cstdint>
#include <string>

#include "common.cuh"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;
constexpr size_t kChainSmem = 64 * 1024;  // staged bytes per CTA (3 CTAs per SM)

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
  ChainIds ids;
};

__device__ __forceinline__ void chain_coord(int d, int in, int out, int& i0, int& i1, float& w) {
  const float scale = __fdiv_rn(static_cast<float>(in), static_cast<float>(out));
  float s = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(d), 0.5f), scale), 0.5f);
  if (s < 0.0f) s = 0.0f;
  int a = static_cast<int>(s);
  if (a > in - 1) a = in - 1;
  i0 = a;
  i1 = a + 1 < in ? a + 1 : in - 1;
  w = __fsub_rn(s, static_cast<float>(a));
}

__device__ __forceinline__ float apply_ops(const dp_image_chain& c, int from, int to, int ch, float v) {
  for (int k = from; k < to; ++k) {
    if (c.op_kind[k] == 0) v = __fdiv_rn(__fsub_rn(v, c.op_a[k][ch]), c.op_b[k][ch]);  // (x - mean) / std
    else v = __fadd_rn(__fmul_rn(v, c.op_a[k][ch]), c.op_b[k][ch]);                    // x * scale + shift
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
  chain_coord(my, a.win_h, a.mid_h, y0, y1, w);
  return g.oy0 + y0;
}
__device__ __forceinline__ int last_src_row(const ChainArgs& a, const Geo& g, int my) {
  if (!a.c.resize) return g.oy0 + my;
  int y0, y1;
  float w;
  chain_coord(my, a.win_h, a.mid_h, y0, y1, w);
  return g.oy0 + y1;
}

template <typename OutT, bool kAligned>
__global__ void __launch_bounds__(kThreads) chain_kernel(ChainArgs a) {
  extern __shared__ __align__(16) uint8_t stage[];
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
    for (int t = threadIdx.x; t < srows * chunks; t += kThreads) {
      const int r = t / chunks, q = t - r * chunks;
      *reinterpret_cast<uint4*>(stage + r * a.stage_cols + q * 16) =
          ld_nc_na_u4(src + static_cast<size_t>(r) * row_bytes + q * 16);
    }
  } else {
    for (int t = threadIdx.x; t < srows * a.stage_cols; t += kThreads) {
      const int r = t / a.stage_cols, q = t - r * a.stage_cols;
      stage[r * a.stage_cols + q] = src[static_cast<size_t>(r) * row_bytes + q];
    }
  }
  __syncthreads();

  const int seg = a.out_w * 3;
  OutT* obase = static_cast<OutT*>(a.out) + (static_cast<size_t>(j) * a.out_h + y_begin) * seg;
  const int shift = g.ox0 * 3 - col0;
  // window pixel (wy, wx), channel ch, as staged
  auto win = [&](int wy, int wx, int ch) -> uint32_t {
    const int sx = g.f0 ? a.win_w - 1 - wx : wx;
    return stage[(g.oy0 + wy - sy_lo) * a.stage_cols + shift + sx * 3 + ch];
  };
  auto value = [&](int r, int e) -> float {
    const int x = e / 3, ch = e - 3 * (e / 3);
    const int my = g.oy1 + y_begin + r;
    const int mx = g.ox1 + (g.f1 ? a.out_w - 1 - x : x);
    if (!c.resize) return apply_ops(c, 0, c.num_pre_ops, ch, static_cast<float>(win(my, mx, ch)));
    int y0, y1, x0, x1;
    float wy, wx;
    chain_coord(my, a.win_h, a.mid_h, y0, y1, wy);
    chain_coord(mx, a.win_w, a.mid_w, x0, x1, wx);
    const int np = c.num_pre_ops;
    const float p00 = apply_ops(c, 0, np, ch, static_cast<float>(win(y0, x0, ch)));
    const float p01 = apply_ops(c, 0, np, ch, static_cast<float>(win(y0, x1, ch)));
    const float p10 = apply_ops(c, 0, np, ch, static_cast<float>(win(y1, x0, ch)));
    const float p11 = apply_ops(c, 0, np, ch, static_cast<float>(win(y1, x1, ch)));
    const float top = __fadd_rn(p00, __fmul_rn(wx, __fsub_rn(p01, p00)));
    const float bot = __fadd_rn(p10, __fmul_rn(wx, __fsub_rn(p11, p10)));
    const float v = __fadd_rn(top, __fmul_rn(wy, __fsub_rn(bot, top)));
    return apply_ops(c, np, np + c.num_post_ops, ch, v);
  };
  if constexpr (sizeof(OutT) == 1) {  // u8: crops only (no resize, no ops)
    if (kAligned && (seg & 3) == 0) {
      const int qn = seg >> 2;
      for (int t = threadIdx.x; t < nrows * qn; t += kThreads) {
        const int r = t / qn, q = t - r * qn;
        const int my = g.oy1 + y_begin + r;
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = 4 * q + u, x = e / 3, ch = e - 3 * (e / 3);
          const int mx = g.ox1 + (g.f1 ? a.out_w - 1 - x : x);
          w |= win(my, mx, ch) << (8 * u);
        }
        __stcs(reinterpret_cast<unsigned int*>(obase + static_cast<size_t>(r) * seg) + q, w);
      }
    } else {
      for (int t = threadIdx.x; t < nrows * seg; t += kThreads) {
        const int r = t / seg, e = t - r * seg, x = e / 3, ch = e - 3 * (e / 3);
        const int my = g.oy1 + y_begin + r;
        const int mx = g.ox1 + (g.f1 ? a.out_w - 1 - x : x);
        obase[static_cast<size_t>(r) * seg + e] = static_cast<OutT>(win(my, mx, ch));
      }
    }
  } else {
    if (kAligned && (seg & 3) == 0) {
      const int qn = seg >> 2;
      for (int t = threadIdx.x; t < nrows * qn; t += kThreads) {
        const int r = t / qn, q = t - r * qn;
        float4 v;
        v.x = value(r, 4 * q);
        v.y = value(r, 4 * q + 1);
        v.z = value(r, 4 * q + 2);
        v.w = value(r, 4 * q + 3);
        st_cs_f4(reinterpret_cast<float4*>(obase + static_cast<size_t>(r) * seg) + q, v);
      }
    } else {
      for (int t = threadIdx.x; t < nrows * seg; t += kThreads) {
        const int r = t / seg, e = t - r * seg;
        obase[static_cast<size_t>(r) * seg + e] = value(r, e);
      }
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
  const bool aligned = row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(images) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(out) % 16 == 0;
  // staged window columns: the whole window, widened to 16-byte boundaries
  a.stage_cols = aligned ? static_cast<int>(((a.win_w * 3 + 15) / 16 + 1) * 16) : a.win_w * 3;
  if (aligned && static_cast<size_t>(a.stage_cols) > row_bytes) a.stage_cols = static_cast<int>(row_bytes);
  // band rows: the source rows one band reads must fit the stage
  const double scale = chain->resize ? static_cast<double>(a.win_h) / a.mid_h : 1.0;
  int band = 32;
  auto src_rows = [&](int b) { return chain->resize ? static_cast<int>(b * scale) + 3 : b; };
  while (band > 1 && static_cast<size_t>(std::min(src_rows(band), chain->in_h)) * a.stage_cols > kChainSmem) band /= 2;
  const size_t smem = static_cast<size_t>(std::min(src_rows(band), chain->in_h)) * a.stage_cols;
  if (smem > 200 * 1024)
    return fail(DP_ERR_INVALID_ATTR, "image_chain: one output row reads more source rows than shared memory holds");
  a.band_rows = std::min(band, oh);
  a.bands = (oh + a.band_rows - 1) / a.band_rows;
  const int64_t grid = rows * a.bands;
  if (grid > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "image_chain: batch too large");
  cudaStream_t s = as_stream(stream);
  auto launch = [&](auto kernel) {
    if (smem > 48 * 1024) {
      const int rc = cuda_status(
          cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
          "image_chain smem attribute");
      if (rc) return rc;
    }
    kernel<<<static_cast<int>(grid), kThreads, smem, s>>>(a);
    return launch_status("image_chain");
  };
  if (f32) return aligned ? launch(chain_kernel<float, true>) : launch(chain_kernel<float, false>);
  return aligned ? launch(chain_kernel<uint8_t, true>) : launch(chain_kernel<uint8_t, false>);
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
