// k_image.cu -- K3 gather + random crop + flip + normalize + batch and
// K4 gather + bilinear resize + normalize + batch: one launch writes a whole
// batch slot (MapAndBatchIterator's job, /root/reference/proj/src/
// runtime.cpp:1467-1721, with the UDF applied per cell and no AssembleBatch
// copy, :617-628).
//
// Both kernels are HBM-bound: per image K3 reads the
// 150,528-byte crop window once and writes 602,112 bytes of fp32; K4 reads
// the 307,200-byte source once and writes 602,112 bytes.  A CTA owns a band
// of output rows of one image: it stages the source bytes the band needs in
// shared memory with 16-byte non-allocating loads, then every thread emits
// 16-byte streaming (.cs) stores of 4 normalized fp32 values, so the output
// (80% of the traffic) leaves the SM as fully coalesced 128-bit stores.
#include <cstdint>

#include "common.cuh"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;
constexpr int kCropBandRows = 16;
constexpr int kResizeBandRows = 16;

__device__ __forceinline__ float sel3(int c, float a, float b, float d) { return c == 0 ? a : (c == 1 ? b : d); }

struct ImageArgs {
  const uint8_t* images;
  const int64_t* order;
  int64_t first;
  int64_t* out_ids;
  float* out;
  int in_h, in_w, out_h, out_w;
  int bands;
  NormConsts nc;
};

// ---------------------------------------------------------------- K3 ----
template <bool kAligned>
__global__ void __launch_bounds__(kThreads)
crop_flip_norm_kernel(ImageArgs a, uint64_t seed, int do_flip, int sstride) {
  extern __shared__ __align__(16) uint8_t stage[];
  const int band = blockIdx.x % a.bands;
  const int64_t j = blockIdx.x / a.bands;
  const int64_t id = a.order ? a.order[a.first + j] : a.first + j;
  CropParams cp = crop_params(seed, id, a.in_h, a.in_w, a.out_h, a.out_w);
  if (!do_flip) cp.flip = 0;
  if (band == 0 && threadIdx.x == 0) a.out_ids[j] = id;

  const int y_begin = band * kCropBandRows;
  const int nrows = min(kCropBandRows, a.out_h - y_begin);
  const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
  const int seg = a.out_w * 3;  // bytes (= floats) per output row
  const uint8_t* img = a.images + static_cast<size_t>(id) * a.in_h * row_bytes;
  const uint8_t* src0 = img + static_cast<size_t>(cp.oy + y_begin) * row_bytes;
  const int start = cp.ox * 3;

  int shift;
  if (kAligned) {
    const int a0 = start & ~15;
    shift = start - a0;
    const int nchunks = (shift + seg + 15) >> 4;
    for (int t = threadIdx.x; t < nrows * nchunks; t += kThreads) {
      const int r = t / nchunks, c = t - r * nchunks;
      *reinterpret_cast<uint4*>(stage + r * sstride + c * 16) =
          ld_nc_na_u4(src0 + static_cast<size_t>(r) * row_bytes + a0 + c * 16);
    }
  } else {
    shift = 0;
    for (int t = threadIdx.x; t < nrows * seg; t += kThreads) {
      const int r = t / seg, c = t - r * seg;
      stage[r * sstride + c] = src0[static_cast<size_t>(r) * row_bytes + start + c];
    }
  }
  __syncthreads();

  float* obase = a.out + (static_cast<size_t>(j) * a.out_h + y_begin) * seg;
  const NormConsts& nc = a.nc;
  if (kAligned) {
    const int q_per_row = seg >> 2;
    for (int t = threadIdx.x; t < nrows * q_per_row; t += kThreads) {
      const int r = t / q_per_row, q = t - r * q_per_row;
      const uint8_t* srow = stage + r * sstride + shift;
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = 4 * q + u;
        const int x = e / 3;
        const int ch = e - 3 * x;
        const int sx = cp.flip ? (a.out_w - 1 - x) : x;
        v[u] = normalize_u8(static_cast<float>(srow[sx * 3 + ch]), sel3(ch, nc.mean[0], nc.mean[1], nc.mean[2]),
                            sel3(ch, nc.stdv[0], nc.stdv[1], nc.stdv[2]), sel3(ch, nc.rcp[0], nc.rcp[1], nc.rcp[2]));
      }
      st_cs_f4(reinterpret_cast<float4*>(obase + static_cast<size_t>(r) * seg + 4 * q),
               make_float4(v[0], v[1], v[2], v[3]));
    }
  } else {
    for (int t = threadIdx.x; t < nrows * seg; t += kThreads) {
      const int r = t / seg, e = t - r * seg;
      const int x = e / 3, ch = e - 3 * x;
      const int sx = cp.flip ? (a.out_w - 1 - x) : x;
      obase[static_cast<size_t>(r) * seg + e] =
          normalize_u8(static_cast<float>(stage[r * sstride + sx * 3 + ch]), sel3(ch, nc.mean[0], nc.mean[1], nc.mean[2]),
                       sel3(ch, nc.stdv[0], nc.stdv[1], nc.stdv[2]), sel3(ch, nc.rcp[0], nc.rcp[1], nc.rcp[2]));
    }
  }
}

// ---------------------------------------------------------------- K4 ----
// Half-pixel-centre source coordinate (the oracle's resize_coord, every op
// individually rounded).
__device__ __forceinline__ void resize_coord(int d, int in, int out, int& i0, int& i1, float& w) {
  const float scale = __fdiv_rn(static_cast<float>(in), static_cast<float>(out));
  float s = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(d), 0.5f), scale), 0.5f);
  if (s < 0.0f) s = 0.0f;
  int a = static_cast<int>(s);
  if (a > in - 1) a = in - 1;
  i0 = a;
  i1 = a + 1 < in ? a + 1 : in - 1;
  w = __fsub_rn(s, static_cast<float>(a));
}

__device__ __forceinline__ float lerp_rn(float p, float q, float w) {
  return __fadd_rn(p, __fmul_rn(w, __fsub_rn(q, p)));
}

template <bool kAligned>
__global__ void __launch_bounds__(kThreads)
resize_norm_kernel(ImageArgs a) {
  extern __shared__ __align__(16) uint8_t stage[];
  const int band = blockIdx.x % a.bands;
  const int64_t j = blockIdx.x / a.bands;
  const int64_t id = a.order ? a.order[a.first + j] : a.first + j;
  if (band == 0 && threadIdx.x == 0) a.out_ids[j] = id;

  const int y_begin = band * kResizeBandRows;
  const int nrows = min(kResizeBandRows, a.out_h - y_begin);
  int ys0, ys1, tmp;
  float wtmp;
  resize_coord(y_begin, a.in_h, a.out_h, ys0, tmp, wtmp);
  resize_coord(y_begin + nrows - 1, a.in_h, a.out_h, tmp, ys1, wtmp);
  const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
  const size_t span = static_cast<size_t>(ys1 - ys0 + 1) * row_bytes;  // contiguous source rows
  const uint8_t* src = a.images + (static_cast<size_t>(id) * a.in_h + ys0) * row_bytes;
  if (kAligned) {
    for (size_t t = threadIdx.x; t < span / 16; t += kThreads)
      *reinterpret_cast<uint4*>(stage + t * 16) = ld_nc_na_u4(src + t * 16);
  } else {
    for (size_t t = threadIdx.x; t < span; t += kThreads) stage[t] = src[t];
  }
  __syncthreads();

  const int seg = a.out_w * 3;
  float* obase = a.out + (static_cast<size_t>(j) * a.out_h + y_begin) * seg;
  const NormConsts& nc = a.nc;
  const int vec = kAligned ? 4 : 1;
  const int q_per_row = seg / vec;
  for (int t = threadIdx.x; t < nrows * q_per_row; t += kThreads) {
    const int r = t / q_per_row, q = t - r * q_per_row;
    int y0, y1;
    float wy;
    resize_coord(y_begin + r, a.in_h, a.out_h, y0, y1, wy);
    const uint8_t* row0 = stage + static_cast<size_t>(y0 - ys0) * row_bytes;
    const uint8_t* row1 = stage + static_cast<size_t>(y1 - ys0) * row_bytes;
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= vec) break;
      const int e = vec * q + u;
      const int x = e / 3;
      const int ch = e - 3 * x;
      int x0, x1;
      float wx;
      resize_coord(x, a.in_w, a.out_w, x0, x1, wx);
      const float p00 = row0[x0 * 3 + ch], p01 = row0[x1 * 3 + ch];
      const float p10 = row1[x0 * 3 + ch], p11 = row1[x1 * 3 + ch];
      const float top = lerp_rn(p00, p01, wx);
      const float bot = lerp_rn(p10, p11, wx);
      const float val = lerp_rn(top, bot, wy);
      v[u] = normalize_f32(val, sel3(ch, nc.mean[0], nc.mean[1], nc.mean[2]), sel3(ch, nc.stdv[0], nc.stdv[1], nc.stdv[2]));
    }
    if (kAligned) {
      st_cs_f4(reinterpret_cast<float4*>(obase + static_cast<size_t>(r) * seg + 4 * q),
               make_float4(v[0], v[1], v[2], v[3]));
    } else {
      obase[static_cast<size_t>(r) * seg + q] = v[0];
    }
  }
}

NormConsts make_norm(const float mean[3], const float stdv[3]) {
  NormConsts nc;
  for (int c = 0; c < 3; ++c) {
    nc.mean[c] = mean[c];
    nc.stdv[c] = stdv[c];
    nc.rcp[c] = 1.0f / stdv[c];  // host IEEE division: RN(1/std)
  }
  return nc;
}

template <typename K>
int ensure_smem(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return DP_OK;
  return cuda_status(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                     "image kernel smem attribute");
}

int check_common(const uint8_t* images, int64_t num_images, int in_h, int in_w, int64_t rows, int out_h, int out_w,
                 const int64_t* out_ids, const float* out, const char* what) {
  if (rows < 0) return fail(DP_ERR_INVALID_ATTR, std::string(what) + ": rows must be >= 0");
  if (in_h < 1 || in_w < 1 || out_h < 1 || out_w < 1)
    return fail(DP_ERR_INVALID_ATTR, std::string(what) + ": image dims must be >= 1");
  if (rows > 0 && (!images || !out_ids || !out || num_images < 1))
    return fail(DP_ERR_INVALID_ATTR, std::string(what) + ": null buffer");
  return DP_OK;
}

}  // namespace
}  // namespace dpk

using namespace dpk;

extern "C" int dp_k_crop_flip_normalize_batch(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                              const int64_t* order, int64_t first, int64_t rows, uint64_t udf_seed,
                                              int crop_h, int crop_w, int do_flip, const float mean[3],
                                              const float stdv[3], int64_t* out_ids, float* out, void* stream) {
  int st = check_common(images, num_images, in_h, in_w, rows, crop_h, crop_w, out_ids, out, "crop_flip_normalize");
  if (st) return st;
  if (crop_h > in_h || crop_w > in_w)
    return fail(DP_ERR_INVALID_ATTR, "crop_flip_normalize: crop larger than the image");
  if (rows == 0) return DP_OK;
  ImageArgs a{images, order, first, out_ids, out, in_h, in_w, crop_h, crop_w,
              (crop_h + kCropBandRows - 1) / kCropBandRows, make_norm(mean, stdv)};
  const size_t row_bytes = static_cast<size_t>(in_w) * 3;
  const bool aligned = (row_bytes % 16 == 0) && (reinterpret_cast<uintptr_t>(images) % 16 == 0) &&
                       (crop_w % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const int seg = crop_w * 3;
  const int sstride = aligned ? ((seg + 15 + 15) / 16) * 16 : seg;
  const size_t smem = static_cast<size_t>(kCropBandRows) * sstride;
  const int64_t grid = rows * a.bands;
  if (grid > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "crop_flip_normalize: batch too large");
  cudaStream_t s = as_stream(stream);
  if (aligned) {
    if ((st = ensure_smem(crop_flip_norm_kernel<true>, smem))) return st;
    crop_flip_norm_kernel<true><<<static_cast<int>(grid), kThreads, smem, s>>>(a, udf_seed, do_flip, sstride);
  } else {
    if ((st = ensure_smem(crop_flip_norm_kernel<false>, smem))) return st;
    crop_flip_norm_kernel<false><<<static_cast<int>(grid), kThreads, smem, s>>>(a, udf_seed, do_flip, sstride);
  }
  return launch_status("crop_flip_normalize");
}

extern "C" int dp_k_resize_normalize_batch(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                           const int64_t* order, int64_t first, int64_t rows, int out_h, int out_w,
                                           const float mean[3], const float stdv[3], int64_t* out_ids, float* out,
                                           void* stream) {
  int st = check_common(images, num_images, in_h, in_w, rows, out_h, out_w, out_ids, out, "resize_normalize");
  if (st) return st;
  if (rows == 0) return DP_OK;
  ImageArgs a{images, order, first, out_ids, out, in_h, in_w, out_h, out_w,
              (out_h + kResizeBandRows - 1) / kResizeBandRows, make_norm(mean, stdv)};
  const size_t row_bytes = static_cast<size_t>(in_w) * 3;
  const bool aligned = (row_bytes % 16 == 0) && (reinterpret_cast<uintptr_t>(images) % 16 == 0) &&
                       (out_w % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  // Worst-case source rows per band: ceil(band * scale) + 2.
  const double scale = static_cast<double>(in_h) / out_h;
  const int max_src_rows = static_cast<int>(kResizeBandRows * scale) + 3;
  const size_t smem = static_cast<size_t>(max_src_rows < in_h ? max_src_rows : in_h) * row_bytes;
  if (smem > 227 * 1024)
    return fail(DP_ERR_INVALID_ATTR, "resize_normalize: source band exceeds shared memory (downscale > ~9x)");
  const int64_t grid = rows * a.bands;
  if (grid > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "resize_normalize: batch too large");
  cudaStream_t s = as_stream(stream);
  if (aligned) {
    if ((st = ensure_smem(resize_norm_kernel<true>, smem))) return st;
    resize_norm_kernel<true><<<static_cast<int>(grid), kThreads, smem, s>>>(a);
  } else {
    if ((st = ensure_smem(resize_norm_kernel<false>, smem))) return st;
    resize_norm_kernel<false><<<static_cast<int>(grid), kThreads, smem, s>>>(a);
  }
  return launch_status("resize_normalize");
}
