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
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "fastdiv.hpp"
#include "roll.hpp"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;
constexpr int kCropBandRows = 16;
constexpr int kResizeBandRows = 16;
constexpr int kFastCropBandRows = 16;   // tools/dev/ksweep.py: 16 rows x 8 stages best on B200
constexpr int kFastResizeBandRows = 16;
constexpr int kCropStages = 8;
constexpr int kResizeStages = 4;
constexpr size_t kSmemBudget = 200 * 1024;
constexpr size_t kSmemBudgetMax = 224 * 1024;  // 227 KB opt-in minus static + reserved
constexpr int kResizePWarps = 25;              // ResizePOp consumer warps (21 / 25 / 29 instantiated)

__device__ __forceinline__ float sel3(int c, float a, float b, float d) { return c == 0 ? a : (c == 1 ? b : d); }

// Element id of resident row r (the Philox counter and the emitted id).
// Fully resident: id = r.  Sharded residency (one process per GPU holds
// blocks b % stride == base of `block` consecutive positions; block 1 =
// element shards, block R = the record files of an interleave's shard):
//   id = ((r / block) * stride + base) * block + r % block.
struct RowIds {
  int64_t base, stride, block;
  __device__ __forceinline__ int64_t of(int64_t r) const {
    if (block == 1) return base + r * stride;
    const int64_t q = r / block;
    return (q * stride + base) * block + (r - q * block);
  }
};

struct ImageArgs {
  const uint8_t* images;
  const int64_t* order;
  int64_t first;
  int64_t* out_ids;
  float* out;
  int64_t num_images;
  int in_h, in_w, out_h, out_w;
  int bands;
  NormConsts nc;
  RowIds ids;  // element id of resident row r = ids.of(r)
};

// ---------------------------------------------------------------- K3 ----
template <bool kAligned>
__global__ void __launch_bounds__(kThreads)
crop_generic_kernel(ImageArgs a, uint64_t seed, int do_flip, int sstride) {
  extern __shared__ __align__(16) uint8_t stage[];
  const int band = blockIdx.x % a.bands;
  const int64_t j = blockIdx.x / a.bands;
  const int64_t row = a.order ? a.order[a.first + j] : a.first + j;
  if (row < 0 || row >= a.num_images) return;  // engine orders are in range by construction
  const int64_t id = a.ids.of(row);  // element id (sharded residency)
  CropParams cp = do_flip < 0 ? CropParams{(a.in_h - a.out_h) / 2, (a.in_w - a.out_w) / 2, 0}  // center
                              : crop_params(seed, id, a.in_h, a.in_w, a.out_h, a.out_w);
  if (do_flip <= 0) cp.flip = 0;
  if (band == 0 && threadIdx.x == 0) a.out_ids[j] = id;

  const int y_begin = band * kCropBandRows;
  const int nrows = min(kCropBandRows, a.out_h - y_begin);
  const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
  const int seg = a.out_w * 3;  // bytes (= floats) per output row
  const uint8_t* img = a.images + static_cast<size_t>(row) * a.in_h * row_bytes;
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
        v[u] = normalize_fast(static_cast<float>(srow[sx * 3 + ch]), sel3(ch, nc.mean[0], nc.mean[1], nc.mean[2]),
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
          normalize_fast(static_cast<float>(stage[r * sstride + sx * 3 + ch]), sel3(ch, nc.mean[0], nc.mean[1], nc.mean[2]),
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
resize_generic_kernel(ImageArgs a) {
  extern __shared__ __align__(16) uint8_t stage[];
  const int band = blockIdx.x % a.bands;
  const int64_t j = blockIdx.x / a.bands;
  const int64_t row = a.order ? a.order[a.first + j] : a.first + j;
  if (row < 0 || row >= a.num_images) return;  // engine orders are in range by construction
  if (band == 0 && threadIdx.x == 0) a.out_ids[j] = a.ids.of(row);

  const int y_begin = band * kResizeBandRows;
  const int nrows = min(kResizeBandRows, a.out_h - y_begin);
  int ys0, ys1, tmp;
  float wtmp;
  resize_coord(y_begin, a.in_h, a.out_h, ys0, tmp, wtmp);
  resize_coord(y_begin + nrows - 1, a.in_h, a.out_h, tmp, ys1, wtmp);
  const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
  const size_t span = static_cast<size_t>(ys1 - ys0 + 1) * row_bytes;  // contiguous source rows
  const uint8_t* src = a.images + (static_cast<size_t>(row) * a.in_h + ys0) * row_bytes;
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
      v[u] = normalize_fast(val, sel3(ch, nc.mean[0], nc.mean[1], nc.mean[2]), sel3(ch, nc.stdv[0], nc.stdv[1], nc.stdv[2]),
                            sel3(ch, nc.rcp[0], nc.rcp[1], nc.rcp[2]));
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


// ===================================================================
// Fast path: persistent, warp-specialized CTAs over a kStages-deep TMA
// pipeline (one CTA per SM).
//
// Work item = (batch row j, band of `band_rows` output rows).  One producer
// warp resolves each item's gather index (and crop offsets), arms the
// stage's "full" mbarrier with the exact byte count and issues the
// cp.async.bulk copies (TMA engine, L2 evict-first) of the source bytes the
// band needs.  The consumer warps own one fixed float4 output column q per
// thread, so channel constants and smem offsets of their 4 outputs are
// computed once per kernel; the inner loop is 4 (K3) or 16 (K4) LDS.U8,
// exact normalizes and one 16-byte streaming store.  Each consumer warp
// releases a stage through the "empty" mbarrier on its own -- there is no
// CTA-wide barrier in the loop, so warps drift freely and the TMA reads of
// later items overlap the store stream of earlier ones.
// ===================================================================
constexpr int kMaxStages = 16;
constexpr int kFastConsumers = 672;  // 21 warps; + 1 producer warp


struct StageMeta {
  int64_t id;
  int64_t j;
  int band, nrows, shift, flip, ys0, pad;
};

// Everything the producer needs to issue one item; computed by one lane per
// item, 32 items at a time, so the gather-index loads and Philox draws of a
// whole group are in flight together instead of serialising per item.
struct Plan {
  int64_t id, j, row;  // element id, batch row, source image row
  int band, nrows, src_row, col, shift, flip;
  uint32_t bytes_row;
};

__device__ __forceinline__ Plan shfl_plan(const Plan& p, int src) {
  Plan o;
  o.id = __shfl_sync(0xffffffffu, p.id, src);
  o.j = __shfl_sync(0xffffffffu, p.j, src);
  o.row = __shfl_sync(0xffffffffu, p.row, src);
  o.band = __shfl_sync(0xffffffffu, p.band, src);
  o.nrows = __shfl_sync(0xffffffffu, p.nrows, src);
  o.src_row = __shfl_sync(0xffffffffu, p.src_row, src);
  o.col = __shfl_sync(0xffffffffu, p.col, src);
  o.shift = __shfl_sync(0xffffffffu, p.shift, src);
  o.flip = __shfl_sync(0xffffffffu, p.flip, src);
  o.bytes_row = __shfl_sync(0xffffffffu, p.bytes_row, src);
  return o;
}

struct FastArgs {
  const uint8_t* images;
  const int64_t* order;
  int64_t first, rows, num_images;
  int64_t* out_ids;
  float* out;
  int in_h, in_w, out_h, out_w;
  int band_rows, bands, q_per_row, rpp;
  int q_stride;  // threads per row group (>= q_per_row; a multiple of 32 keeps groups warp-uniform)
  int stage_stride, stage_bytes, stages;
  uint64_t seed;
  int do_flip;
  int center;  // K3: center_crop offsets instead of Philox draws
  NormConsts nc;
  RowIds ids;  // element id of resident row r = ids.of(r)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct RowTap {
  int y0, y1;
  float wy;
};

// ---- K3 stage operations ----
struct CropOp {
  static constexpr bool kWarpWide = false;
  static constexpr int kConsumers = kFastConsumers;
  float mu[4], sd[4], rc[4];
  int off_n[4], off_f[4];
  f32x2 mu2[2], nsd2[2], rc2[2];
  PkK k;

  __device__ void init(const FastArgs& a, int q, uint8_t*) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = 4 * q + u, x = e / 3, ch = e - 3 * x;
      mu[u] = sel3(ch, a.nc.mean[0], a.nc.mean[1], a.nc.mean[2]);
      sd[u] = sel3(ch, a.nc.stdv[0], a.nc.stdv[1], a.nc.stdv[2]);
      rc[u] = sel3(ch, a.nc.rcp[0], a.nc.rcp[1], a.nc.rcp[2]);
      off_n[u] = e;
      off_f[u] = (a.out_w - 1 - x) * 3 + ch;
    }
    k = PkK(a.nc);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      mu2[p] = pk2(mu[2 * p], mu[2 * p + 1]);
      nsd2[p] = pk2(-sd[2 * p], -sd[2 * p + 1]);
      rc2[p] = pk2(rc[2 * p], rc[2 * p + 1]);
    }
  }

  static __device__ Plan plan(const FastArgs& a, int64_t item, const uint8_t*) {
    Plan p;
    p.j = item / a.bands;
    p.band = static_cast<int>(item - p.j * a.bands);
    const int64_t row = a.order ? a.order[a.first + p.j] : a.first + p.j;
    const bool valid = row >= 0 && row < a.num_images;
    p.row = valid ? row : -1;
    p.id = valid ? a.ids.of(row) : -1;
    p.nrows = min(a.band_rows, a.out_h - p.band * a.band_rows);
    CropParams cp{0, 0, 0};
    if (valid) {
      if (a.center) cp = CropParams{(a.in_h - a.out_h) / 2, (a.in_w - a.out_w) / 2, 0};  // center_crop
      else cp = crop_params(a.seed, p.id, a.in_h, a.in_w, a.out_h, a.out_w);
    }
    const int start = cp.ox * 3;
    p.shift = start & 15;
    p.src_row = cp.oy + p.band * a.band_rows;  // first source row
    p.col = start - p.shift;                     // 16-byte aligned first source byte
    p.flip = a.do_flip ? cp.flip : 0;
    p.bytes_row = static_cast<uint32_t>((p.shift + a.out_w * 3 + 15) >> 4) << 4;
    return p;
  }

  // producer warp: fill meta + issue the row copies of one planned item
  static __device__ void issue(const FastArgs& a, const Plan& p, uint8_t* dst, StageMeta* meta, uint64_t* full,
                               int lane, uint64_t pol) {
    const bool valid = p.id >= 0;
    if (lane == 0) {
      *meta = StageMeta{p.id, p.j, p.band, p.nrows, p.shift, p.flip, 0, 0};
      mbar_arrive_expect_tx(full, valid ? p.bytes_row * p.nrows : 0u);
    }
    __syncwarp();
    if (valid) {
      const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
      const uint8_t* src0 = a.images + (static_cast<size_t>(p.row) * a.in_h + p.src_row) * row_bytes + p.col;
      for (int r = lane; r < p.nrows; r += 32)
        bulk_g2s(dst + r * a.stage_stride, src0 + r * row_bytes, p.bytes_row, full, pol);
    }
  }

  __device__ void consume(const FastArgs& a, const StageMeta& m, const uint8_t* stage, int q, int rsub,
                          const uint8_t*) const {
    const uint8_t* st = stage + m.shift;
    const int seg = a.out_w * 3;
    float4* ob = reinterpret_cast<float4*>(a.out + (static_cast<size_t>(m.j) * a.out_h +
                                                    static_cast<size_t>(m.band) * a.band_rows) * seg);
    for (int r = rsub; r < m.nrows; r += a.rpp) {
      const uint8_t* row = st + r * a.stage_stride;
      const int* off = m.flip ? off_f : off_n;
      float2 v[2];
#pragma unroll
      for (int p = 0; p < 2; ++p)  // packed pairs: the scalar normalize_fast ops, bit for bit
        v[p] = up2(k.normalize(k.u8x2(row[off[2 * p]], row[off[2 * p + 1]]), mu2[p], nsd2[p], rc2[p]));
      st_cs_f4(ob + static_cast<size_t>(r) * a.q_per_row + q, make_float4(v[0].x, v[0].y, v[1].x, v[1].y));
    }
  }
};

// ---- K4 stage operations ----
struct ResizeOp {
  static constexpr bool kWarpWide = false;
  static constexpr int kConsumers = kFastConsumers;
  float mu[4], sd[4], rc[4], wx[4];
  int o0[4], o1[4];
  f32x2 mu2[2], nsd2[2], rc2[2], wx2[2];
  PkK k;

  __device__ void init(const FastArgs& a, int q, uint8_t*) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = 4 * q + u, x = e / 3, ch = e - 3 * x;
      mu[u] = sel3(ch, a.nc.mean[0], a.nc.mean[1], a.nc.mean[2]);
      sd[u] = sel3(ch, a.nc.stdv[0], a.nc.stdv[1], a.nc.stdv[2]);
      rc[u] = sel3(ch, a.nc.rcp[0], a.nc.rcp[1], a.nc.rcp[2]);
      int x0, x1;
      resize_coord(x, a.in_w, a.out_w, x0, x1, wx[u]);
      // Right-edge clamp (x1 == x0 == in_w - 1): blending (x0 - 1, x0) with
      // weight 1 gives p(x0) exactly (integer-valued fp32), as the oracle's
      // p00 + wx * (p00 - p00) does; so the right tap is always o0 + 3 and its
      // load takes an immediate offset (in_w >= 16 on this path).
      if (x1 == x0) {
        x0 -= 1;
        wx[u] = 1.0f;
      }
      o0[u] = x0 * 3 + ch;
      o1[u] = o0[u] + 3;
    }
    k = PkK(a.nc);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      mu2[p] = pk2(mu[2 * p], mu[2 * p + 1]);
      nsd2[p] = pk2(-sd[2 * p], -sd[2 * p + 1]);
      rc2[p] = pk2(rc[2 * p], rc[2 * p + 1]);
      wx2[p] = pk2(wx[2 * p], wx[2 * p + 1]);
    }
  }

  static __device__ Plan plan(const FastArgs& a, int64_t item, const uint8_t* taps_raw) {
    const RowTap* taps = reinterpret_cast<const RowTap*>(taps_raw);
    Plan p;
    p.j = item / a.bands;
    p.band = static_cast<int>(item - p.j * a.bands);
    const int64_t row = a.order ? a.order[a.first + p.j] : a.first + p.j;
    const bool valid = row >= 0 && row < a.num_images;
    p.row = valid ? row : -1;
    p.id = valid ? a.ids.of(row) : -1;
    const int y_begin = p.band * a.band_rows;
    p.nrows = min(a.band_rows, a.out_h - y_begin);
    p.src_row = taps[y_begin].y0;
    const int ys1 = taps[y_begin + p.nrows - 1].y1;
    p.bytes_row = static_cast<uint32_t>((ys1 - p.src_row + 1) * a.in_w * 3);  // whole contiguous span
    p.col = 0;
    p.shift = 0;
    p.flip = 0;
    return p;
  }

  static __device__ void issue(const FastArgs& a, const Plan& p, uint8_t* dst, StageMeta* meta, uint64_t* full,
                               int lane, uint64_t pol) {
    const bool valid = p.id >= 0;
    if (lane == 0) {
      *meta = StageMeta{p.id, p.j, p.band, p.nrows, 0, 0, p.src_row, 0};
      mbar_arrive_expect_tx(full, valid ? p.bytes_row : 0u);
      if (valid)
        bulk_g2s(dst, a.images + (static_cast<size_t>(p.row) * a.in_h + p.src_row) * static_cast<size_t>(a.in_w) * 3,
                 p.bytes_row, full, pol);
    }
    __syncwarp();
  }

  __device__ void consume(const FastArgs& a, const StageMeta& m, const uint8_t* st, int q, int rsub,
                          const uint8_t* taps_raw) const {
    const RowTap* taps = reinterpret_cast<const RowTap*>(taps_raw);
    const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
    const int seg = a.out_w * 3;
    const int y_begin = m.band * a.band_rows;
    float4* ob = reinterpret_cast<float4*>(a.out + (static_cast<size_t>(m.j) * a.out_h + y_begin) * seg);
    for (int r = rsub; r < m.nrows; r += a.rpp) {
      const RowTap t = taps[y_begin + r];
      const uint8_t* row0 = st + static_cast<size_t>(t.y0 - m.ys0) * row_bytes;
      const uint8_t* row1 = st + static_cast<size_t>(t.y1 - m.ys0) * row_bytes;
      // lanes (u = 2p, 2p + 1) in packed pairs: the same rounded ops as the
      // scalar lerp_rn / normalize_fast (orc_resize_normalize), half the issues.
      // (Walking consecutive rows per thread to reuse a shared source row
      // measured slower: 0.51-0.54 vs 0.67 of HBM -- the reuse branches cut
      // the loads in flight per thread.)
      const f32x2 wy2 = splat2(t.wy);
      float2 v[2];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int u = 2 * p;
        const f32x2 top = k.lerp_u8(PkK::raw_u8x2(row0[o0[u]], row0[o0[u + 1]]),
                                    PkK::raw_u8x2(row0[o1[u]], row0[o1[u + 1]]), wx2[p]);
        const f32x2 bot = k.lerp_u8(PkK::raw_u8x2(row1[o0[u]], row1[o0[u + 1]]),
                                    PkK::raw_u8x2(row1[o1[u]], row1[o1[u + 1]]), wx2[p]);
        v[p] = up2(k.normalize(k.lerp(top, bot, wy2), mu2[p], nsd2[p], rc2[p]));
      }
      st_cs_f4(ob + static_cast<size_t>(r) * a.q_per_row + q, make_float4(v[0].x, v[0].y, v[1].x, v[1].y));
    }
  }
};

// K4 over a PERIODIC horizontal map: in_w = PI * G, out_w = PO * G, and
// every output column x takes source columns x0 = PI * (x / PO) + T(x % PO)
// and x0 + 1 (checked on the host against resize_coord for every x:
// periodic_ok).  One lane owns one period ("group": PO output pixels = 3 * PO
// floats from a window of source bytes it loads as 32-bit words), one warp
// one output row (G <= 32 groups).  The bytes are picked out of registers
// with PRMT at compile-time positions instead of one shared-memory byte load
// per tap (ResizeOp: 16 per float4, ~1.8-way bank conflicts), and the row is
// transposed through a per-warp shared buffer (stride 3 * PO words, odd:
// conflict-free) into coalesced float4 stores.  Same lerp / normalize ops,
// same order, as ResizeOp and the oracle (orc_resize_normalize).
template <int PO, int PI, int W>
struct ResizePOp {
  __host__ __device__ static constexpr int T(int x) { return ((2 * x + 1) * PI - PO) / (2 * PO); }
  static constexpr int kF = 3 * PO;                       // floats per group
  static constexpr int kPairs = (kF + 1) / 2;
  static constexpr int kSpan = 3 * (T(PO - 1) + 2);       // window bytes
  static constexpr int kOmax = (3 * PI) % 4 == 0 ? 0 : ((3 * PI) % 2 == 0 ? 2 : 3);
  static constexpr int kNW = (kOmax + kSpan + 3) / 4;     // 32-bit words per window
  static constexpr bool kWarpWide = true;
  static constexpr int kConsumers = W * 32;  // W consumer warps, one output row each
  f32x2 wx2[kPairs];
  f32x2 mu2[3], nsd2[3], rc2[3];  // by pair pattern (channel of the pair's first float: 0, 2, 1)
  PkK k;
  float* stg;  // this warp's row buffer: G * kF floats
  int byte0;   // the group's first source byte in a row

  __device__ void init(const FastArgs& a, int q, uint8_t* taps) {
    float wx[kF];
#pragma unroll
    for (int e = 0; e < kF; e += 3) {
      int x0, x1;
      resize_coord(q * PO + e / 3, a.in_w, a.out_w, x0, x1, wx[e]);
      wx[e + 1] = wx[e];
      wx[e + 2] = wx[e];
    }
#pragma unroll
    for (int i = 0; i < kPairs; ++i) wx2[i] = pk2(wx[2 * i], wx[2 * i + 1 < kF ? 2 * i + 1 : 2 * i]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int c1 = (c + 1) % 3;
      mu2[c] = pk2(a.nc.mean[c], a.nc.mean[c1]);
      nsd2[c] = pk2(-a.nc.stdv[c], -a.nc.stdv[c1]);
      rc2[c] = pk2(a.nc.rcp[c], a.nc.rcp[c1]);
    }
    k = PkK(a.nc);
    const size_t taps_bytes = ((static_cast<size_t>(a.out_h) * sizeof(RowTap) + 15) / 16) * 16;
    stg = reinterpret_cast<float*>(taps + taps_bytes) + static_cast<size_t>(threadIdx.x >> 5) * a.q_per_row * kF;
    byte0 = q * PI * 3;
  }

  static __device__ Plan plan(const FastArgs& a, int64_t item, const uint8_t* taps_raw) {
    return ResizeOp::plan(a, item, taps_raw);
  }
  static __device__ void issue(const FastArgs& a, const Plan& p, uint8_t* dst, StageMeta* meta, uint64_t* full,
                               int lane, uint64_t pol) {
    ResizeOp::issue(a, p, dst, meta, full, lane, pol);
  }

  // byte b of the (shifted) window as an exact fp32 (the 2^23 magic-number
  // conversion; PRMT builds 0x4B0000bb directly)
  static __device__ __forceinline__ uint32_t pick(const uint32_t* w, int b) {
    return __byte_perm(w[b >> 2], 0x4B000000u, 0x7440u | static_cast<uint32_t>(b & 3));
  }
  // two tap bytes as 2^23 + byte (exact "magic" floats, not yet converted)
  static __device__ __forceinline__ f32x2 raw2(const uint32_t* w, int b0, int b1) {
    return pk2(__uint_as_float(pick(w, b0)), __uint_as_float(pick(w, b1)));
  }


  __device__ void consume(const FastArgs& a, const StageMeta& m, const uint8_t* st, int q, int rsub,
                          const uint8_t* taps_raw) const {
    const RowTap* taps = reinterpret_cast<const RowTap*>(taps_raw);
    const size_t row_bytes = static_cast<size_t>(a.in_w) * 3;
    const int lane = threadIdx.x & 31;
    const int y_begin = m.band * a.band_rows;
    const int row_f4 = a.out_w * 3 / 4;
    float4* ob = reinterpret_cast<float4*>(a.out) + (static_cast<size_t>(m.j) * a.out_h + y_begin) * row_f4;
    const int sh = (byte0 & 3) * 8;
    const bool mine = q < a.q_per_row;  // a group of this row (else: store helper only)
    for (int r = rsub; r < m.nrows; r += a.rpp) {
      const RowTap t = taps[y_begin + r];
      if (mine) {
        const uint32_t* s0 =
            reinterpret_cast<const uint32_t*>(st + static_cast<size_t>(t.y0 - m.ys0) * row_bytes + (byte0 & ~3));
        const uint32_t* s1 =
            reinterpret_cast<const uint32_t*>(st + static_cast<size_t>(t.y1 - m.ys0) * row_bytes + (byte0 & ~3));
        uint32_t w0[kNW + 1], w1[kNW + 1];
#pragma unroll
        for (int i = 0; i < kNW; ++i) {
          w0[i] = s0[i];
          w1[i] = s1[i];
        }
        w0[kNW] = w1[kNW] = 0;
        if (kOmax) {
#pragma unroll
          for (int i = 0; i < kNW; ++i) {
            w0[i] = __funnelshift_r(w0[i], w0[i + 1], sh);
            w1[i] = __funnelshift_r(w1[i], w1[i + 1], sh);
          }
        }
        const f32x2 wy2 = splat2(t.wy);
        float* my = stg + lane * kF;
#pragma unroll
        for (int i = 0; i < kPairs; ++i) {
          const int e0 = 2 * i, e1 = 2 * i + 1 < kF ? 2 * i + 1 : 2 * i;
          const int l0 = 3 * T(e0 / 3) + e0 % 3, l1 = 3 * T(e1 / 3) + e1 % 3;  // left taps; right = +3
          // only the left tap is converted (PkK::lerp_u8)
          const f32x2 top = k.lerp_u8(raw2(w0, l0, l1), raw2(w0, l0 + 3, l1 + 3), wx2[i]);
          const f32x2 bot = k.lerp_u8(raw2(w1, l0, l1), raw2(w1, l0 + 3, l1 + 3), wx2[i]);
          const float2 v = up2(k.normalize(k.lerp(top, bot, wy2), mu2[e0 % 3], nsd2[e0 % 3], rc2[e0 % 3]));
          my[e0] = v.x;
          if (e1 != e0) my[e1] = v.y;
        }
      }
      __syncwarp();
      const float4* src = reinterpret_cast<const float4*>(stg);
      float4* orow = ob + static_cast<size_t>(r) * row_f4;
#pragma unroll
      for (int i = 0; i < (32 * kF + 127) / 128; ++i) {  // <= 32 groups per row
        const int c = lane + 32 * i;
        if (c < row_f4) st_cs_f4(orow + c, src[c]);
      }
      __syncwarp();
    }
  }
};

// Host twin of resize_coord's column taps: the periodic form holds when
// every x0 = PI * (x / PO) + T(x % PO) and x1 = x0 + 1 (no edge clamps).
template <int PO, int PI>
bool periodic_ok(int in_w, int out_w) {
  if (in_w % PI || out_w % PO || in_w / PI != out_w / PO || out_w / PO > 32) return false;
  const float scale = static_cast<float>(in_w) / static_cast<float>(out_w);
  for (int x = 0; x < out_w; ++x) {
    float sx = (static_cast<float>(x) + 0.5f) * scale - 0.5f;
    if (sx < 0.0f) sx = 0.0f;
    int a = static_cast<int>(sx);
    if (a > in_w - 1) a = in_w - 1;
    if (a + 1 >= in_w || a != PI * (x / PO) + ResizePOp<PO, PI, 1>::T(x % PO)) return false;
  }
  return true;
}

template <class Op>
__global__ void __launch_bounds__(Op::kConsumers + 32, 1) pipeline_kernel(FastArgs a) {
  // The next launch on the stream (the next launch group, another slot) may
  // start as SMs free up: it reads only the read-only dataset and plan and
  // writes a different slot (programmatic dependent launch).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ StageMeta meta[kMaxStages];
  const int kStages = a.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int consumers = a.q_stride * a.rpp;
  const int n_cwarps = (consumers + 31) >> 5;
  uint8_t* taps = smem + kStages * a.stage_bytes;  // resize row taps (unused by K3)

  for (int y = tid; y < a.out_h; y += blockDim.x) {
    RowTap t;
    resize_coord(y, a.in_h, a.out_h, t.y0, t.y1, t.wy);
    reinterpret_cast<RowTap*>(taps)[y] = t;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], n_cwarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t total = a.rows * a.bands;
  if (warp == n_cwarps) {  // ---- producer warp ----
    const uint64_t pol = policy_evict_first();
    for (int64_t k0 = 0;; k0 += 32) {
      const int64_t my_item = blockIdx.x + (k0 + lane) * static_cast<int64_t>(gridDim.x);
      Plan mine{};
      if (my_item < total) mine = Op::plan(a, my_item, taps);
      const int n = __popc(__ballot_sync(0xffffffffu, my_item < total));
      for (int t = 0; t < n; ++t) {
        const int64_t k = k0 + t;
        const int s = static_cast<int>(k % kStages);
        if (k >= kStages) mbar_wait(&empty[s], static_cast<uint32_t>((k / kStages) - 1) & 1);
        Op::issue(a, shfl_plan(mine, t), smem + s * a.stage_bytes, &meta[s], &full[s], lane, pol);
      }
      if (n < 32) break;
    }
    return;
  }
  // ---- consumer warps ----
  const int q = tid % a.q_stride, rsub = tid / a.q_stride;
  // warp-wide ops (ResizePOp) run every lane of a consumer warp: lanes past
  // the row's groups take part in the warp's transposed store
  const bool active = tid < consumers && (Op::kWarpWide || q < a.q_per_row);
  Op op;
  op.init(a, active ? q : 0, taps);
  int k = 0;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x, ++k) {
    const int s = k % kStages;
    mbar_wait(&full[s], (k / kStages) & 1);
    const StageMeta m = meta[s];
    if (m.id >= 0 && active) {
      if (m.band == 0 && tid == 0) a.out_ids[m.j] = m.id;
      op.consume(a, m, smem + s * a.stage_bytes, q, rsub, taps);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int env_int(const char* name, int fallback);

template <typename K>
int launch_persistent(K kernel, const FastArgs& a, size_t smem, cudaStream_t s, const char* what) {
  // cudaFuncSetAttribute / the occupancy query are host-synchronous-ish and
  // cost tens of microseconds: do them once per (device, kernel, smem, threads).
  struct Key {
    int dev;
    const void* fn;
    size_t smem;
    int threads;
    bool operator<(const Key& o) const {
      return std::tie(dev, fn, smem, threads) < std::tie(o.dev, o.fn, o.smem, o.threads);
    }
  };
  static std::mutex mu;
  static std::map<Key, int> occupancy;
  static std::map<std::pair<int, const void*>, size_t> smem_attr;  // max dynamic smem set per kernel
  int st;
  const int threads = ((a.q_stride * a.rpp + 31) / 32) * 32 + 32;
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    const Key key{dev, reinterpret_cast<const void*>(kernel), smem, threads};
    size_t& cur = smem_attr[{dev, reinterpret_cast<const void*>(kernel)}];
    if (smem > cur) {  // the attribute only ever grows, so cached keys stay launchable
      if ((st = cuda_status(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem)),
                            what)))
        return st;
      cur = smem;
    }
    auto it = occupancy.find(key);
    if (it != occupancy.end()) {
      per_sm = it->second;
    } else {
      if ((st = cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem), what)))
        return st;
      occupancy[key] = per_sm;
    }
  }
  if (per_sm < 1) return fail(DP_ERR_INVALID_ATTR, std::string(what) + ": kernel does not fit on an SM");
  const int64_t items = a.rows * a.bands;
  const int64_t grid = std::min<int64_t>(items, static_cast<int64_t>(per_sm) * sm_count());
  static const int pdl = env_int("DP_DEV_PDL", 0);
  if (pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_status(cudaLaunchKernelEx(&cfg, kernel, a), what);
  }
  kernel<<<static_cast<int>(grid), threads, smem, s>>>(a);
  return launch_status(what);
}

// Fast-path eligibility: 16B-aligned rows and buffers, whole float4 per
// thread column, a row of float4s fits one CTA; images in HBM or pinned
// host memory (cp.async.bulk reads both).
bool in_device_memory(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // pinned host memory too: the TMA engine reads it over PCIe in bulk
  // (end-to-end runs: 0.8-0.9 of the PCIe copy rate against ~0.7 for the
  // generic kernels' 16-byte loads)
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged ||
         (attr.type == cudaMemoryTypeHost && env_int("DP_DEV_TMA_HOST", 1));
}

bool fast_ok(const uint8_t* images, int in_w, int out_w, const float* out) {
  const int q = out_w * 3 / 4;
  return (static_cast<size_t>(in_w) * 3) % 16 == 0 && reinterpret_cast<uintptr_t>(images) % 16 == 0 &&
         out_w % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 && q <= kFastConsumers &&
         in_device_memory(images);
}

// Development-only overrides for tuning sweeps (tools/dev/kbench.py).
int env_int(const char* name, int fallback) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : fallback;
}

FastArgs make_fast(const uint8_t* images, int64_t num_images, int in_h, int in_w, const int64_t* order, int64_t first,
                   int64_t rows, int out_h, int out_w, const float mean[3], const float stdv[3], int64_t* out_ids,
                   float* out, int band_rows, int stages) {
  FastArgs a{};
  a.images = images;
  a.order = order;
  a.first = first;
  a.rows = rows;
  a.num_images = num_images;
  a.out_ids = out_ids;
  a.out = out;
  a.in_h = in_h;
  a.in_w = in_w;
  a.out_h = out_h;
  a.out_w = out_w;
  a.band_rows = band_rows < out_h ? band_rows : out_h;
  a.bands = (out_h + a.band_rows - 1) / a.band_rows;
  a.q_per_row = out_w * 3 / 4;
  a.q_stride = a.q_per_row;
  a.rpp = kFastConsumers / a.q_per_row;
  if (a.rpp > a.band_rows) a.rpp = a.band_rows;
  a.nc = make_norm(mean, stdv);
  a.stages = env_int("DP_DEV_STAGES", stages);
  if (a.stages < 2) a.stages = 2;
  if (a.stages > kMaxStages) a.stages = kMaxStages;
  return a;
}

}  // namespace
}  // namespace dpk

using namespace dpk;

static int crop_impl(const uint8_t* images, int64_t num_images, int in_h, int in_w, const int64_t* order, int64_t first,
                     int64_t rows, uint64_t udf_seed, int crop_h, int crop_w, int do_flip, const float mean[3],
                     const float stdv[3], int64_t* out_ids, float* out, void* stream, RowIds ids) {
  int st = check_common(images, num_images, in_h, in_w, rows, crop_h, crop_w, out_ids, out, "crop_flip_normalize");
  if (st) return st;
  if (crop_h > in_h || crop_w > in_w)
    return fail(DP_ERR_INVALID_ATTR, "crop_flip_normalize: crop larger than the image");
  if (rows == 0) return DP_OK;
  cudaStream_t s = as_stream(stream);
  if (!fast_div_proven(mean, stdv)) {
    // the two-FMA division is not exact for these constants: the same chain
    // through K9 with IEEE division
    dp_image_chain c{};
    c.in_h = in_h;
    c.in_w = in_w;
    c.pre_mode = do_flip < 0 ? 2 : 1;
    c.pre_h = crop_h;
    c.pre_w = crop_w;
    c.pre_flip = do_flip > 0 ? 1 : 0;
    c.pre_seed = udf_seed;
    c.num_pre_ops = 1;
    for (int ch = 0; ch < 3; ++ch) {
      c.op_a[0][ch] = mean[ch];
      c.op_b[0][ch] = stdv[ch];
    }
    c.out_f32 = 1;
    return dp_k_image_chain_batch(images, num_images, order, first, rows, ids.base, ids.stride, ids.block, &c, out_ids,
                                  out, stream);
  }
  if (fast_ok(images, in_w, crop_w, out)) {
    FastArgs f = make_fast(images, num_images, in_h, in_w, order, first, rows, crop_h, crop_w, mean, stdv, out_ids,
                           out, env_int("DP_DEV_CROP_BAND", kFastCropBandRows), kCropStages);
    f.ids = ids;
    f.seed = udf_seed;
    f.do_flip = do_flip > 0 ? 1 : 0;
    f.center = do_flip < 0 ? 1 : 0;
    f.stage_stride = ((crop_w * 3 + 15 + 15) / 16) * 16;
    f.stage_bytes = ((f.band_rows * f.stage_stride + 127) / 128) * 128;
    const size_t taps = static_cast<size_t>(crop_h) * sizeof(RowTap);
    while (f.stages > 2 && static_cast<size_t>(f.stages) * f.stage_bytes + taps > kSmemBudget) --f.stages;
    const size_t smem = static_cast<size_t>(f.stages) * f.stage_bytes + taps;
    if (smem <= kSmemBudget) return launch_persistent(pipeline_kernel<CropOp>, f, smem, s, "crop_flip_normalize");
  }
  ImageArgs a{images, order, first, out_ids, out, num_images, in_h, in_w, crop_h, crop_w,
              (crop_h + kCropBandRows - 1) / kCropBandRows, make_norm(mean, stdv), ids};
  const size_t row_bytes = static_cast<size_t>(in_w) * 3;
  const bool aligned = (row_bytes % 16 == 0) && (reinterpret_cast<uintptr_t>(images) % 16 == 0) &&
                       (crop_w % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const int seg = crop_w * 3;
  const int sstride = aligned ? ((seg + 15 + 15) / 16) * 16 : seg;
  const size_t smem = static_cast<size_t>(kCropBandRows) * sstride;
  const int64_t grid = rows * a.bands;
  if (grid > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "crop_flip_normalize: batch too large");
  if (aligned) {
    if ((st = ensure_smem(crop_generic_kernel<true>, smem))) return st;
    crop_generic_kernel<true><<<static_cast<int>(grid), kThreads, smem, s>>>(a, udf_seed, do_flip, sstride);
  } else {
    if ((st = ensure_smem(crop_generic_kernel<false>, smem))) return st;
    crop_generic_kernel<false><<<static_cast<int>(grid), kThreads, smem, s>>>(a, udf_seed, do_flip, sstride);
  }
  return launch_status("crop_flip_normalize");
}

static int resize_impl(const uint8_t* images, int64_t num_images, int in_h, int in_w, const int64_t* order,
                       int64_t first, int64_t rows, int out_h, int out_w, const float mean[3], const float stdv[3],
                       int64_t* out_ids, float* out, void* stream, RowIds ids) {
  int st = check_common(images, num_images, in_h, in_w, rows, out_h, out_w, out_ids, out, "resize_normalize");
  if (st) return st;
  if (rows == 0) return DP_OK;
  cudaStream_t s = as_stream(stream);
  const bool proven = fast_div_proven(mean, stdv);
  {
    // the same chain as a descriptor: K10 when the column map is periodic
    // (320 -> 224: 0.92 of HBM against this file's 0.81), K9 (IEEE
    // division) when the two-FMA division is not proven exact for the
    // constants, else the K4 kernels below
    dp_image_chain c{};
    c.in_h = in_h;
    c.in_w = in_w;
    c.resize = 1;
    c.rs_h = out_h;
    c.rs_w = out_w;
    c.num_post_ops = 1;
    for (int ch = 0; ch < 3; ++ch) {
      c.op_a[0][ch] = mean[ch];
      c.op_b[0][ch] = stdv[ch];
    }
    c.out_f32 = 1;
    if (!proven)
      return dp_k_image_chain_batch(images, num_images, order, first, rows, ids.base, ids.stride, ids.block, &c,
                                    out_ids, out, stream);
    const int rc = roll_chain_batch(images, num_images, order, first, rows, ids.base, ids.stride, ids.block, &c, out_h,
                                    out_w, out_ids, out, s, /*allow_general=*/false);
    if (rc != 1) return rc;
  }
  if (fast_ok(images, in_w, out_w, out)) {
    FastArgs f = make_fast(images, num_images, in_h, in_w, order, first, rows, out_h, out_w, mean, stdv, out_ids, out,
                           env_int("DP_DEV_RESIZE_BAND", kFastResizeBandRows), kResizeStages);
    f.ids = ids;
    const double sc = static_cast<double>(in_h) / out_h;
    int src_rows = static_cast<int>(f.band_rows * sc) + 3;
    if (src_rows > in_h) src_rows = in_h;
    f.stage_stride = in_w * 3;
    f.stage_bytes = static_cast<int>(((static_cast<size_t>(src_rows) * in_w * 3 + 127) / 128) * 128);
    const size_t taps = static_cast<size_t>(out_h) * sizeof(RowTap);
    while (f.stages > 2 && static_cast<size_t>(f.stages) * f.stage_bytes + taps > kSmemBudget) --f.stages;
    const size_t smem = static_cast<size_t>(f.stages) * f.stage_bytes + taps;
    // periodic column taps (320 -> 224, 256 -> 224): one period per lane
    const bool p710 = periodic_ok<7, 10>(in_w, out_w), p78 = !p710 && periodic_ok<7, 8>(in_w, out_w);
    if ((p710 || p78) && env_int("DP_DEV_RESIZE_PERIODIC", 1)) {
      const int warps = env_int("DP_DEV_RESIZEP_WARPS", kResizePWarps);
      FastArgs p = f;
      p.q_per_row = out_w / 7;  // groups per row (one lane each)
      p.q_stride = 32;
      p.rpp = warps;
      // two output rows per consumer warp per band (tools/dev/k4sweep*.sh:
      // 43.0 vs 44.8 us per 256-image batch at 320 -> 224), one when the
      // larger stage does not fit
      const size_t taps16 = ((taps + 15) / 16) * 16;
      const size_t stg = static_cast<size_t>(p.rpp) * out_w * 3 * sizeof(float);
      size_t psmem = 0;
      for (int rows_per_warp : {2, 1}) {
        p.band_rows = env_int("DP_DEV_RESIZE_PBAND", rows_per_warp * p.rpp);
        if (p.band_rows > out_h) p.band_rows = out_h;
        p.bands = (out_h + p.band_rows - 1) / p.band_rows;
        p.stages = env_int("DP_DEV_STAGES", kResizeStages);
        int prow = static_cast<int>(p.band_rows * sc) + 3;
        if (prow > in_h) prow = in_h;
        p.stage_bytes = static_cast<int>(((static_cast<size_t>(prow) * in_w * 3 + 127) / 128) * 128);
        while (p.stages > 2 && static_cast<size_t>(p.stages) * p.stage_bytes + taps16 + stg > kSmemBudgetMax)
          --p.stages;
        psmem = static_cast<size_t>(p.stages) * p.stage_bytes + taps16 + stg;
        if (psmem <= kSmemBudgetMax) break;
      }
      if (psmem <= kSmemBudgetMax) {
#define DP_LAUNCH_P(W)                                                                                   \
  if (warps == W)                                                                                        \
    return p710 ? launch_persistent(pipeline_kernel<ResizePOp<7, 10, W>>, p, psmem, s, "resize_normalize") \
                : launch_persistent(pipeline_kernel<ResizePOp<7, 8, W>>, p, psmem, s, "resize_normalize");
        DP_LAUNCH_P(21)
        DP_LAUNCH_P(25)
        DP_LAUNCH_P(29)
#undef DP_LAUNCH_P
      }
    }
    if (smem <= kSmemBudget)
      return launch_persistent(pipeline_kernel<ResizeOp>, f, smem, s, "resize_normalize");
  }
  ImageArgs a{images, order, first, out_ids, out, num_images, in_h, in_w, out_h, out_w,
              (out_h + kResizeBandRows - 1) / kResizeBandRows, make_norm(mean, stdv), ids};
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
  if (aligned) {
    if ((st = ensure_smem(resize_generic_kernel<true>, smem))) return st;
    resize_generic_kernel<true><<<static_cast<int>(grid), kThreads, smem, s>>>(a);
  } else {
    if ((st = ensure_smem(resize_generic_kernel<false>, smem))) return st;
    resize_generic_kernel<false><<<static_cast<int>(grid), kThreads, smem, s>>>(a);
  }
  return launch_status("resize_normalize");
}

extern "C" int dp_k_crop_flip_normalize_batch(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                              const int64_t* order, int64_t first, int64_t rows, uint64_t udf_seed,
                                              int crop_h, int crop_w, int do_flip, const float mean[3],
                                              const float stdv[3], int64_t* out_ids, float* out, void* stream) {
  return crop_impl(images, num_images, in_h, in_w, order, first, rows, udf_seed, crop_h, crop_w, do_flip, mean, stdv,
                   out_ids, out, stream, RowIds{0, 1, 1});
}

extern "C" int dp_k_crop_flip_normalize_batch_ex(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                                 const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                                 int64_t id_stride, int64_t id_block, uint64_t udf_seed, int crop_h,
                                                 int crop_w, int do_flip, const float mean[3], const float stdv[3],
                                                 int64_t* out_ids, float* out, void* stream) {
  if (id_stride < 1 || id_block < 1 || id_base < 0 || id_base >= id_stride)
    return fail(DP_ERR_INVALID_ATTR, "crop_flip_normalize: bad sharded residency (id_base/id_stride/id_block)");
  return crop_impl(images, num_images, in_h, in_w, order, first, rows, udf_seed, crop_h, crop_w, do_flip, mean, stdv,
                   out_ids, out, stream, RowIds{id_base, id_stride, id_block});
}

extern "C" int dp_k_center_crop_normalize_batch_ex(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                                   const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                                   int64_t id_stride, int64_t id_block, int crop_h, int crop_w,
                                                   const float mean[3], const float stdv[3], int64_t* out_ids,
                                                   float* out, void* stream) {
  if (id_stride < 1 || id_block < 1 || id_base < 0 || id_base >= id_stride)
    return fail(DP_ERR_INVALID_ATTR, "center_crop_normalize: bad sharded residency (id_base/id_stride/id_block)");
  // do_flip = -1 selects the center offsets inside crop_impl (no draws, no flip)
  return crop_impl(images, num_images, in_h, in_w, order, first, rows, 0, crop_h, crop_w, -1, mean, stdv, out_ids,
                   out, stream, RowIds{id_base, id_stride, id_block});
}

extern "C" int dp_k_resize_normalize_batch(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                           const int64_t* order, int64_t first, int64_t rows, int out_h, int out_w,
                                           const float mean[3], const float stdv[3], int64_t* out_ids, float* out,
                                           void* stream) {
  return resize_impl(images, num_images, in_h, in_w, order, first, rows, out_h, out_w, mean, stdv, out_ids, out,
                     stream, RowIds{0, 1, 1});
}

extern "C" int dp_k_resize_normalize_batch_ex(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                              const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                              int64_t id_stride, int64_t id_block, int out_h, int out_w,
                                              const float mean[3], const float stdv[3], int64_t* out_ids, float* out,
                                              void* stream) {
  if (id_stride < 1 || id_block < 1 || id_base < 0 || id_base >= id_stride)
    return fail(DP_ERR_INVALID_ATTR, "resize_normalize: bad sharded residency (id_base/id_stride/id_block)");
  return resize_impl(images, num_images, in_h, in_w, order, first, rows, out_h, out_w, mean, stdv, out_ids, out,
                     stream, RowIds{id_base, id_stride, id_block});
}
