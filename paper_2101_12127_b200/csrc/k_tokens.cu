// k_tokens.cu -- K5: Filter(len <= max_keep) as warp-ballot stream
// compaction + PaddedBatch.
//
// Filter: FilterIterator (/root/reference/proj/src/runtime.cpp:537-577)
// keeps element i iff pred(i) and preserves order.  Here the predicate is the
// length test, evaluated on the int32 length array only; the kept positions
// are produced by a three-kernel stable compaction (per-tile counts with
// __ballot_sync/__popc, one-CTA exclusive scan over tiles, per-tile scatter
// at the scanned offsets), so the result is order-preserving and bit exact.
// PaddedBatch (new kind): each batch of `batch` kept rows
// is padded to its own max length; the valid prefix of every row equals the
// reference's ragged Batch output.
#include <cstdint>

#include "common.cuh"
#include "dpcuda.h"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;  // consecutive elements per thread
constexpr int kTile = kThreads * kItems;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kThreads / 32 ? warp_sums[lane] : 0;
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(kFull, z, o);
      if (lane >= o) z += y;
    }
    if (lane < kThreads / 32) warp_sums[lane] = z - w;
    if (lane == kThreads / 32 - 1) *total = z;
  }
  __syncthreads();
  return x - v + warp_sums[warp];
}

// The predicate of one Filter: a conjunction of up to 8 terms on a quantity
// of the element at position p -- its token-sequence length, its int64
// value, or the position itself (range) -- after the affine maps beneath the
// filter (wrap-around int64, as K1).  % is C++'s truncated remainder.
struct FilterSpec {
  const int32_t* lengths;
  const int64_t* values;
  int64_t mul, add;
  int nterms;
  int op[8];
  int64_t a[8], b[8];

  __device__ __forceinline__ bool keep(int64_t p) const {
    int64_t v = lengths ? static_cast<int64_t>(lengths[p]) : values ? values[p] : p;
    v = static_cast<int64_t>(static_cast<uint64_t>(v) * static_cast<uint64_t>(mul) + static_cast<uint64_t>(add));
    bool k = true;
    for (int t = 0; t < nterms; ++t) {
      switch (op[t]) {
        case DP_PRED_LE: k = k && v <= a[t]; break;
        case DP_PRED_GE: k = k && v >= a[t]; break;
        case DP_PRED_LT: k = k && v < a[t]; break;
        case DP_PRED_MOD_EQ: k = k && v % a[t] == b[t]; break;
        default: k = k && v % a[t] != b[t]; break;
      }
    }
    return k;
  }
};

// Element i of the filtered sequence is source position in_map[i] (or i).
__device__ __forceinline__ int thread_keep_mask(const FilterSpec& f, const int64_t* __restrict__ in_map, int64_t n,
                                                int64_t base) {
  int mask = 0;
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const int64_t i = base + u;
    if (i < n && f.keep(in_map ? in_map[i] : i)) mask |= 1 << u;
  }
  return mask;
}

__global__ void __launch_bounds__(kThreads)
filter_count_kernel(FilterSpec f, const int64_t* __restrict__ in_map, int64_t n, int64_t* __restrict__ tile_counts) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + static_cast<int64_t>(threadIdx.x) * kItems;
  int c = __popc(thread_keep_mask(f, in_map, n, base));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  __shared__ int warp_counts[kThreads / 32];
  if ((threadIdx.x & 31) == 0) warp_counts[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += warp_counts[w];
    tile_counts[blockIdx.x] = t;
  }
}

// One CTA: exclusive scan of the tile counts in place; total -> *num_kept.
__global__ void __launch_bounds__(1024)
filter_scan_kernel(int64_t* __restrict__ tile_counts, int64_t tiles, int64_t* __restrict__ num_kept) {
  __shared__ int64_t warp_sums[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < tiles; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < tiles ? tile_counts[i] : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = warp_sums[lane];
      int64_t z = w;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(kFull, z, o);
        if (lane >= o) z += y;
      }
      warp_sums[lane] = z - w;
    }
    __syncthreads();
    const int64_t excl = x - v + warp_sums[warp] + carry;
    if (i < tiles) tile_counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *num_kept = carry;
}

__global__ void __launch_bounds__(kThreads)
filter_scatter_kernel(FilterSpec f, int64_t n, const int64_t* __restrict__ tile_offsets,
                      const int64_t* __restrict__ in_map, int64_t* __restrict__ kept) {
  __shared__ int warp_sums[kThreads / 32];
  __shared__ int total;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + static_cast<int64_t>(threadIdx.x) * kItems;
  const int mask = thread_keep_mask(f, in_map, n, base);
  int off = block_exclusive_scan(__popc(mask), warp_sums, &total);
  int64_t dst = tile_offsets[blockIdx.x] + off;
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    if (mask & (1 << u)) {
      const int64_t p = base + u;
      kept[dst++] = in_map ? in_map[p] : p;
    }
  }
}

// One warp per batch.
__global__ void __launch_bounds__(kThreads)
batch_max_len_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ kept, int64_t num_kept,
                     int64_t batch, int64_t num_batches, int32_t* __restrict__ lmax) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= num_batches) return;
  const int64_t r0 = w * batch;
  const int64_t r1 = r0 + batch < num_kept ? r0 + batch : num_kept;
  int32_t m = 0;
  for (int64_t r = r0 + lane; r < r1; r += 32) m = max(m, lengths[kept[r]]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if (lane == 0) lmax[w] = m;
}

// One warp per output row; coalesced 4-byte loads/stores.
__global__ void __launch_bounds__(kThreads)
padded_batch_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                    const int32_t* __restrict__ lengths, const int64_t* __restrict__ kept, int64_t first, int64_t rows,
                    int32_t lmax, int32_t pad, int32_t* __restrict__ out, int32_t* __restrict__ out_lengths) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t p = kept[first + r];
  const int32_t len = lengths[p];
  const int32_t* src = tokens + offsets[p];
  int32_t* dst = out + r * static_cast<int64_t>(lmax);
  for (int c = lane; c < lmax; c += 32) __stcs(dst + c, c < len ? __ldcs(src + c) : pad);
  if (lane == 0) out_lengths[r] = len;
}

// Rows [first_row, first_row + rows) of consecutive padded batches in one
// launch: row R belongs to batch j = R / batch, is padded to lmax[j] and
// lands at element offset boff[j] - boff[j0] + (R - j * batch) * lmax[j].
//
// Latency, not bandwidth, bounded the one-row-per-warp form (ncu: long
// scoreboard stalls on the order -> length/offset -> tokens chain).  Here a
// CTA takes a tile of kRowTile rows: its threads resolve the tile's
// (position, length, offset, lmax, destination) once, in parallel, into
// shared memory; then each warp streams its rows with kLoadsInFlight token
// loads per lane issued before their stores.
#ifndef DP_TOK_TILE
#define DP_TOK_TILE 128
#endif
constexpr int kRowTile = DP_TOK_TILE;
// padded batches: 64-row tiles (twice the CTAs, each preamble half as long;
// tile sweep 64 / 128 / 256: 0.92 / 0.89 / 0.86 of HBM on cfg4, while the
// ragged kernel stays best at 128)
#ifndef DP_TOK_PAD_TILE
#define DP_TOK_PAD_TILE 64
#endif
constexpr int kPadTile = DP_TOK_PAD_TILE;
#ifndef DP_TOK_RAGGED_THREADS
#define DP_TOK_RAGGED_THREADS 256
#endif
#ifndef DP_TOK_RAGGED_TILE
#define DP_TOK_RAGGED_TILE 128
#endif
constexpr int kRaggedThreads = DP_TOK_RAGGED_THREADS, kRaggedTile = DP_TOK_RAGGED_TILE;
#ifndef DP_TOK_LOADS
#define DP_TOK_LOADS 16
#endif
#ifndef DP_TOK_MINB
#define DP_TOK_MINB 1
#endif
constexpr int kLoadsInFlight = DP_TOK_LOADS;

__global__ void __launch_bounds__(kThreads, DP_TOK_MINB)
padded_batches_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                      const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t first_row,
                      int64_t rows, int64_t batch, const int32_t* __restrict__ lmax, const int64_t* __restrict__ boff,
                      int32_t pad, int32_t* __restrict__ out, int32_t* __restrict__ out_lengths) {
  __shared__ int64_t s_src[kPadTile], s_dst[kPadTile];
  __shared__ int32_t s_len[kPadTile], s_lm[kPadTile];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kPadTile;
  const int n = static_cast<int>(rows - r0 < kPadTile ? rows - r0 : kPadTile);
  const int64_t j0 = first_row / batch;
  for (int t = threadIdx.x; t < n; t += kThreads) {
    const int64_t R = first_row + r0 + t, j = R / batch;
    const int64_t p = order ? __ldcs(order + R) : R;
    const int32_t len = lengths[p];
    s_src[t] = offsets[p];
    s_len[t] = len;
    const int32_t lm = lmax[j];
    s_lm[t] = lm;
    s_dst[t] = (boff[j] - boff[j0]) + (R - j * batch) * static_cast<int64_t>(lm);
    out_lengths[r0 + t] = len;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  constexpr int kW = kThreads / 32;
  for (int t = threadIdx.x >> 5; t < n; t += 2 * kW) {  // rows t and t + kW
    const int b = t + kW, has_b = b < n;
    stream_row_pair<kLoadsInFlight>(tokens + s_src[t], s_len[t], s_lm[t], out + s_dst[t],
                                    has_b ? tokens + s_src[b] : tokens, has_b ? s_len[b] : 0,
                                    has_b ? s_lm[b] : 0, has_b ? out + s_dst[b] : out, pad, lane);
  }
}

// ---- ragged Batch of token sequences (the reference's Filter -> Batch,
// runtime.cpp:579-637: a batch of variable-length lists) ----
// prefix[i] = sum of lengths[order[j]] for j < i (int64), by tile sums, the
// one-CTA tile scan above and a per-tile apply.
__device__ __forceinline__ int64_t block_exclusive_scan64(int64_t v, int64_t* warp_sums) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int64_t w = lane < kThreads / 32 ? warp_sums[lane] : 0;
    int64_t z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, z, o);
      if (lane >= o) z += y;
    }
    if (lane < kThreads / 32) warp_sums[lane] = z - w;
  }
  __syncthreads();
  return x - v + warp_sums[warp];
}

__global__ void __launch_bounds__(kThreads)
len_tile_sum_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t n,
                    int64_t* __restrict__ tiles) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + static_cast<int64_t>(threadIdx.x) * kItems;
  int64_t v = 0;
#pragma unroll
  for (int u = 0; u < kItems; ++u)
    if (base + u < n) v += lengths[order ? order[base + u] : base + u];
  __shared__ int64_t ws[kThreads / 32];
  const int64_t excl = block_exclusive_scan64(v, ws);
  if (threadIdx.x == kThreads - 1) tiles[blockIdx.x] = excl + v;
}

__global__ void __launch_bounds__(kThreads)
len_prefix_apply_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t n,
                        const int64_t* __restrict__ tile_base, int64_t* __restrict__ prefix) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + static_cast<int64_t>(threadIdx.x) * kItems;
  int64_t len[kItems], v = 0;
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    len[u] = base + u < n ? lengths[order ? order[base + u] : base + u] : 0;
    v += len[u];
  }
  __shared__ int64_t ws[kThreads / 32];
  int64_t at = tile_base[blockIdx.x] + block_exclusive_scan64(v, ws);
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    if (base + u < n) prefix[base + u] = at;
    at += len[u];
  }
}

// Rows [first_row, first_row + rows) of an epoch's consecutive ragged
// batches of `batch` rows (the last one may be short: n_rows in the epoch):
// row R's tokens go to values[prefix[R] - prefix[first_row]]; batch j's
// row splits (rows_j + 1 int64, relative to the batch) follow the splits of
// the batches before it in the launch group.  Row tiles as padded_batches.
__global__ void __launch_bounds__(kRaggedThreads, DP_TOK_MINB)
ragged_batches_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                      const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t first_row,
                      int64_t rows, int64_t batch, int64_t n_rows, const int64_t* __restrict__ prefix,
                      int32_t* __restrict__ values, int64_t* __restrict__ splits) {
  __shared__ int64_t s_src[kRaggedTile], s_dst[kRaggedTile];
  __shared__ int32_t s_len[kRaggedTile];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRaggedTile;
  const int n = static_cast<int>(rows - r0 < kRaggedTile ? rows - r0 : kRaggedTile);
  const int64_t j0 = first_row / batch, base = prefix[first_row];
  for (int t = threadIdx.x; t < n; t += kRaggedThreads) {
    const int64_t R = first_row + r0 + t, j = R / batch, r = R - j * batch;
    const int64_t p = order ? __ldcs(order + R) : R;
    const int32_t len = lengths[p];
    s_src[t] = offsets[p];
    s_len[t] = len;
    s_dst[t] = prefix[R] - base;
    const int64_t slot = (R - first_row) + (j - j0), batch_start = prefix[j * batch];
    splits[slot] = prefix[R] - batch_start;
    const int64_t rows_j = n_rows - j * batch < batch ? n_rows - j * batch : batch;
    if (r == rows_j - 1) splits[slot + 1] = prefix[R] + len - batch_start;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  constexpr int kW = kRaggedThreads / 32;
  for (int t = threadIdx.x >> 5; t < n; t += 2 * kW) {  // rows t and t + kW
    const int b = t + kW, has_b = b < n;
    const int la = s_len[t], lb = has_b ? s_len[b] : 0;
    stream_row_pair<kLoadsInFlight>(tokens + s_src[t], la, la, values + s_dst[t], has_b ? tokens + s_src[b] : tokens,
                                    lb, lb, has_b ? values + s_dst[b] : values, 0, lane);
  }
}

}  // namespace
}  // namespace dpk

using namespace dpk;

namespace dpk {
namespace {
// Stages the rows of an epoch plan out of (mapped, pinned) host memory into
// a packed device buffer: row i of the plan = source row order[i] (or i),
// its tokens land at staged + prefix[i].  One warp per row, kStageLoads
// 4-byte loads per lane issued before their stores: every warp keeps
// kStageLoads x 128 B of PCIe reads in flight, so thousands of resident
// warps cover the PCIe round trip (the batch kernels then read HBM).
constexpr int kStageLoads = 8;
__global__ void __launch_bounds__(kThreads)
stage_rows_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                  const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t n,
                  const int64_t* __restrict__ prefix, int32_t* __restrict__ staged,
                  int32_t* __restrict__ staged_lengths) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const int64_t p = order ? order[i] : i;
    const int32_t len = lengths[p];
    const int32_t* src = tokens + offsets[p];
    int32_t* dst = staged + prefix[i];
    if (lane == 0) staged_lengths[i] = len;
    for (int c = lane; c < len; c += 32 * kStageLoads) {
      int32_t v[kStageLoads];
#pragma unroll
      for (int u = 0; u < kStageLoads; ++u) v[u] = c + 32 * u < len ? __ldcs(src + c + 32 * u) : 0;
#pragma unroll
      for (int u = 0; u < kStageLoads; ++u)
        if (c + 32 * u < len) dst[c + 32 * u] = v[u];
    }
  }
}
}  // namespace
}  // namespace dpk

extern "C" int dp_k_stage_rows(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                               const int64_t* order, int64_t n, const int64_t* prefix, int32_t* staged,
                               int32_t* staged_lengths, void* stream) {
  if (n < 0) return dpk::fail(DP_ERR_INVALID_ATTR, "stage_rows: n must be >= 0");
  if (n == 0) return DP_OK;
  if (!tokens || !offsets || !lengths || !prefix || !staged || !staged_lengths)
    return dpk::fail(DP_ERR_INVALID_ATTR, "stage_rows: null buffer");
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148LL * 8 * 4);
  dpk::stage_rows_kernel<<<static_cast<int>(blocks), dpk::kThreads, 0, dpk::as_stream(stream)>>>(
      tokens, offsets, lengths, order, n, prefix, staged, staged_lengths);
  return dpk::launch_status("stage_rows");
}

extern "C" int dp_k_padded_batches(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                                   const int64_t* order, int64_t first_row, int64_t rows, int64_t batch,
                                   const int32_t* lmax_dev, const int64_t* boff_dev, int32_t pad_value, int32_t* out,
                                   int32_t* out_lengths, void* stream) {
  if (rows < 0 || batch < 1) return fail(DP_ERR_INVALID_ATTR, "padded_batches: bad rows/batch");
  if (rows == 0) return DP_OK;
  const int64_t blocks = (rows + kPadTile - 1) / kPadTile;
  if (blocks > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "padded_batches: too many rows");
  padded_batches_kernel<<<static_cast<int>(blocks), kThreads, 0, as_stream(stream)>>>(
      tokens, offsets, lengths, order, first_row, rows, batch, lmax_dev, boff_dev, pad_value, out, out_lengths);
  return launch_status("padded_batches");
}

extern "C" size_t dp_k_filter_scratch_bytes(int64_t n) {
  int64_t tiles = (n + kTile - 1) / kTile;
  return static_cast<size_t>(tiles < 1 ? 1 : tiles) * sizeof(int64_t);
}

static int filter_impl(const FilterSpec& f, int64_t n, const int64_t* in_map, int64_t* kept, int64_t* num_kept_dev,
                       void* scratch, void* stream) {
  if (n < 0) return fail(DP_ERR_INVALID_ATTR, "filter: n must be >= 0");
  if (!num_kept_dev || !scratch) return fail(DP_ERR_INVALID_ATTR, "filter: null num_kept/scratch");
  cudaStream_t s = as_stream(stream);
  if (n == 0) return cuda_status(cudaMemsetAsync(num_kept_dev, 0, sizeof(int64_t), s), "filter: memset");
  const int64_t tiles = (n + kTile - 1) / kTile;
  if (tiles > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "filter: n too large");
  int64_t* tile = static_cast<int64_t*>(scratch);
  filter_count_kernel<<<static_cast<int>(tiles), kThreads, 0, s>>>(f, in_map, n, tile);
  filter_scan_kernel<<<1, 1024, 0, s>>>(tile, tiles, num_kept_dev);
  filter_scatter_kernel<<<static_cast<int>(tiles), kThreads, 0, s>>>(f, n, tile, in_map, kept);
  return launch_status("filter");
}

extern "C" int dp_k_filter_len_le(const int32_t* lengths, int64_t n, int32_t max_keep, const int64_t* in_map,
                                  int64_t* kept, int64_t* num_kept_dev, void* scratch, void* stream) {
  if (!lengths && n > 0) return fail(DP_ERR_INVALID_ATTR, "filter: null lengths");
  FilterSpec f{};
  f.lengths = lengths;
  f.mul = 1;
  f.nterms = 1;
  f.op[0] = DP_PRED_LE;
  f.a[0] = max_keep;
  return filter_impl(f, n, in_map, kept, num_kept_dev, scratch, stream);
}

extern "C" int dp_k_filter(const int32_t* lengths, const int64_t* values, int64_t n, int64_t mul, int64_t add,
                           const dp_predicate_term* terms, int num_terms, const int64_t* in_map, int64_t* kept,
                           int64_t* num_kept_dev, void* scratch, void* stream) {
  if (num_terms < 1 || num_terms > 8 || !terms) return fail(DP_ERR_INVALID_ATTR, "filter: 1..8 predicate terms");
  FilterSpec f{};
  f.lengths = lengths;
  f.values = lengths ? nullptr : values;
  f.mul = mul;
  f.add = add;
  f.nterms = num_terms;
  for (int t = 0; t < num_terms; ++t) {
    if (terms[t].op < DP_PRED_LE || terms[t].op > DP_PRED_MOD_NE)
      return fail(DP_ERR_INVALID_ATTR, "filter: unknown predicate op");
    if ((terms[t].op == DP_PRED_MOD_EQ || terms[t].op == DP_PRED_MOD_NE) && terms[t].a == 0)
      return fail(DP_ERR_INVALID_ATTR, "filter: modulus must be non-zero");
    f.op[t] = terms[t].op;
    f.a[t] = terms[t].a;
    f.b[t] = terms[t].b;
  }
  return filter_impl(f, n, in_map, kept, num_kept_dev, scratch, stream);
}

extern "C" int dp_k_batch_max_len(const int32_t* lengths, const int64_t* kept, int64_t num_kept, int64_t batch,
                                  int32_t* lmax, void* stream) {
  if (batch < 1) return fail(DP_ERR_INVALID_ATTR, "padded_batch: batch_size must be >= 1");
  if (num_kept <= 0) return DP_OK;
  const int64_t nb = (num_kept + batch - 1) / batch;
  const int64_t blocks = (nb + kThreads / 32 - 1) / (kThreads / 32);
  batch_max_len_kernel<<<static_cast<int>(blocks), kThreads, 0, as_stream(stream)>>>(lengths, kept, num_kept, batch,
                                                                                     nb, lmax);
  return launch_status("batch_max_len");
}

extern "C" int dp_k_padded_batch(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                                 const int64_t* kept, int64_t first, int64_t rows, int32_t lmax, int32_t pad_value,
                                 int32_t* out, int32_t* out_lengths, void* stream) {
  if (rows < 0 || lmax < 0) return fail(DP_ERR_INVALID_ATTR, "padded_batch: bad rows/lmax");
  if (rows == 0) return DP_OK;
  const int64_t blocks = (rows + kThreads / 32 - 1) / (kThreads / 32);
  padded_batch_kernel<<<static_cast<int>(blocks), kThreads, 0, as_stream(stream)>>>(
      tokens, offsets, lengths, kept, first, rows, lmax, pad_value, out, out_lengths);
  return launch_status("padded_batch");
}

extern "C" size_t dp_k_len_prefix_scratch_bytes(int64_t n) { return dp_k_filter_scratch_bytes(n); }

extern "C" int dp_k_len_prefix(const int32_t* lengths, const int64_t* order, int64_t n, int64_t* prefix,
                               void* scratch, void* stream) {
  if (n < 0 || !lengths || !prefix || !scratch) return fail(DP_ERR_INVALID_ATTR, "len_prefix: bad arguments");
  cudaStream_t s = as_stream(stream);
  if (n == 0) return cuda_status(cudaMemsetAsync(prefix, 0, sizeof(int64_t), s), "len_prefix: memset");
  const int64_t tiles = (n + kTile - 1) / kTile;
  if (tiles > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "len_prefix: n too large");
  int64_t* tile = static_cast<int64_t*>(scratch);
  len_tile_sum_kernel<<<static_cast<int>(tiles), kThreads, 0, s>>>(lengths, order, n, tile);
  filter_scan_kernel<<<1, 1024, 0, s>>>(tile, tiles, prefix + n);  // exclusive tile bases; prefix[n] = total
  len_prefix_apply_kernel<<<static_cast<int>(tiles), kThreads, 0, s>>>(lengths, order, n, tile, prefix);
  return launch_status("len_prefix");
}

extern "C" int dp_k_ragged_batches(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                                   const int64_t* order, int64_t first_row, int64_t rows, int64_t batch,
                                   int64_t n_rows, const int64_t* prefix, int32_t* values, int64_t* splits,
                                   void* stream) {
  if (rows < 0 || batch < 1 || first_row < 0 || first_row + rows > n_rows)
    return fail(DP_ERR_INVALID_ATTR, "ragged_batches: bad rows/batch");
  if (rows == 0) return DP_OK;
  const int64_t blocks = (rows + kRaggedTile - 1) / kRaggedTile;
  if (blocks > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "ragged_batches: too many rows");
  ragged_batches_kernel<<<static_cast<int>(blocks), kRaggedThreads, 0, as_stream(stream)>>>(
      tokens, offsets, lengths, order, first_row, rows, batch, n_rows, prefix, values, splits);
  return launch_status("ragged_batches");
}
