// k_bucket.cu -- K8: BucketByLength, tf.data's bucket_by_sequence_length:
// group_by_window with key = the bucket of the sequence length (bucket b
// holds boundaries[b-1] <= len < boundaries[b]), window = that bucket's batch
// size, reduce = a batch padded to its own max length.  Elements are taken in
// order; a bucket whose window fills emits its batch at once; at the end of
// the input the partial windows are emitted in ascending bucket order (the
// std::map order of GroupByWindowDataset's groups), unless drop_remainder.
// Like PaddedBatch it is a new kind: the reference has neither
// (SURVEY.md 8(a) a15); the contract is restated by the oracle
// (oracle/restate.c orc_bucket_by_length).
//
// The sequential window loop becomes a data-parallel plan:
//   1. per-tile bucket counts, a per-bucket scan over tiles, and a stable
//      scatter (__match_any_sync ranks) give each element its rank r within
//      its bucket and the bucket-grouped position list perm;
//   2. the element with rank r closes a batch iff (r + 1) % size[b] == 0, and
//      the batches come out in the order of their closing elements -- a
//      stable compaction of the closing flags (the K5 filter kernels);
//   3. the partial windows follow, ascending bucket;
//   4. one warp per batch takes its max length.
// The batch kernel then pads every batch of a launch group (one CTA per
// batch) exactly like K5.
#include <cstdint>

#include "common.cuh"
#include "dpcuda.h"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;  // element i = tile * kTile + round * kThreads + tid
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kFull = 0xffffffffu;

struct BucketSpec {
  int32_t bounds[DP_MAX_BUCKETS - 1];
  int64_t size[DP_MAX_BUCKETS];
  int num_bounds;
  int drop;
};

__device__ __forceinline__ int bucket_of(int32_t len, const BucketSpec& s) {
  int b = 0;
  for (int k = 0; k < s.num_bounds; ++k) b += len >= s.bounds[k];
  return b;
}

__device__ __forceinline__ int64_t position(const int64_t* order, int64_t i) { return order ? order[i] : i; }

// tile_counts[tile * K + b] = elements of bucket b in the tile
__global__ void __launch_bounds__(kThreads)
bucket_count_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t n, BucketSpec s,
                    int64_t* __restrict__ tile_counts) {
  __shared__ int cnt[DP_MAX_BUCKETS];
  const int K = s.num_bounds + 1;
  if (threadIdx.x < DP_MAX_BUCKETS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  for (int j = 0; j < kRounds; ++j) {
    const int64_t i = base + j * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[bucket_of(lengths[position(order, i)], s)], 1);
  }
  __syncthreads();
  if (threadIdx.x < K) tile_counts[static_cast<int64_t>(blockIdx.x) * K + threadIdx.x] = cnt[threadIdx.x];
}

// One CTA: warp b scans bucket b's tile counts (exclusive, in place);
// meta[b] = count of bucket b, meta[K + b] = its offset in perm.
__global__ void __launch_bounds__(1024)
bucket_scan_kernel(int64_t* __restrict__ tile_counts, int64_t tiles, int K, int64_t* __restrict__ meta) {
  __shared__ int64_t totals[DP_MAX_BUCKETS];
  const int lane = threadIdx.x & 31, b = threadIdx.x >> 5;
  if (b < K) {
    int64_t carry = 0;
    for (int64_t t0 = 0; t0 < tiles; t0 += 32) {
      const int64_t t = t0 + lane;
      const int64_t v = t < tiles ? tile_counts[t * K + b] : 0;
      int64_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (t < tiles) tile_counts[t * K + b] = carry + x - v;
      carry += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) totals[b] = carry;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int k = 0; k < K; ++k) {
      meta[k] = totals[k];
      meta[K + k] = off;
      off += totals[k];
    }
  }
}

// Stable ranks within buckets; perm[off[b] + r] = position; close[i] = 0 iff
// element i closes a batch (a "length" for the K5 compaction with max 0).
__global__ void __launch_bounds__(kThreads)
bucket_scatter_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ order, int64_t n, BucketSpec s,
                      const int64_t* __restrict__ tile_base, const int64_t* __restrict__ meta,
                      int64_t* __restrict__ perm, int32_t* __restrict__ close, int32_t* __restrict__ bucket,
                      int64_t* __restrict__ rank) {
  __shared__ int wcnt[kWarps][DP_MAX_BUCKETS];
  __shared__ int wpre[kWarps][DP_MAX_BUCKETS];
  __shared__ int64_t run[DP_MAX_BUCKETS];
  const int K = s.num_bounds + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  if (threadIdx.x < K) run[threadIdx.x] = tile_base[static_cast<int64_t>(blockIdx.x) * K + threadIdx.x];
  for (int j = 0; j < kRounds; ++j) {
    for (int t = threadIdx.x; t < kWarps * DP_MAX_BUCKETS; t += kThreads) (&wcnt[0][0])[t] = 0;
    __syncthreads();
    const int64_t i = base + j * kThreads + threadIdx.x;
    const bool valid = i < n;
    const int64_t p = valid ? position(order, i) : 0;
    const int b = valid ? bucket_of(lengths[p], s) : DP_MAX_BUCKETS;  // invalid lanes group apart
    const uint32_t peers = __match_any_sync(kFull, b);
    const int in_warp = __popc(peers & ((1u << lane) - 1u));
    if (valid && in_warp == 0) wcnt[warp][b] = __popc(peers);
    __syncthreads();
    if (threadIdx.x < K) {
      int acc = 0;
      for (int w = 0; w < kWarps; ++w) {
        wpre[w][threadIdx.x] = acc;
        acc += wcnt[w][threadIdx.x];
      }
      wcnt[0][threadIdx.x] = acc;  // this round's total (read after the barrier below)
    }
    __syncthreads();
    if (valid) {
      const int64_t r = run[b] + wpre[warp][b] + in_warp;
      perm[meta[K + b] + r] = p;
      close[i] = (r + 1) % s.size[b] == 0 ? 0 : 1;
      bucket[i] = b;
      rank[i] = r;
    }
    __syncthreads();
    if (threadIdx.x < K) run[threadIdx.x] += wcnt[0][threadIdx.x];
    __syncthreads();  // before the next round clears wcnt
  }
}

// Batch descriptors in emission order: the closing elements, then the
// partial windows (ascending bucket, unless drop).  The last CTA writes the
// tails and the total.
__global__ void __launch_bounds__(kThreads)
bucket_desc_kernel(const int64_t* __restrict__ closing, const int64_t* __restrict__ num_closing,
                   const int32_t* __restrict__ bucket, const int64_t* __restrict__ rank, BucketSpec s,
                   const int64_t* __restrict__ meta, int64_t* __restrict__ start, int32_t* __restrict__ rows,
                   int64_t* __restrict__ num_batches) {
  const int K = s.num_bounds + 1;
  const int64_t E = *num_closing;
  if (blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x == 0) {
      int64_t e = E;
      for (int b = 0; b < K; ++b) {
        const int64_t c = meta[b], full = c / s.size[b] * s.size[b];
        if (c > full && !s.drop) {
          start[e] = meta[K + b] + full;
          rows[e] = static_cast<int32_t>(c - full);
          ++e;
        }
      }
      *num_batches = e;
    }
    return;
  }
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (e >= E) return;
  const int64_t i = closing[e];
  const int b = bucket[i];
  start[e] = meta[K + b] + rank[i] / s.size[b] * s.size[b];
  rows[e] = static_cast<int32_t>(s.size[b]);
}

// One warp per batch: max length over its rows.
__global__ void __launch_bounds__(kThreads)
bucket_lmax_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ perm,
                   const int64_t* __restrict__ start, const int32_t* __restrict__ rows,
                   const int64_t* __restrict__ num_batches, int32_t* __restrict__ lmax) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= *num_batches) return;
  const int64_t s0 = start[e];
  int32_t m = 0;
  for (int r = lane; r < rows[e]; r += 32) m = max(m, lengths[perm[s0 + r]]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if (lane == 0) lmax[e] = m;
}

// The rows of batches [first, first + nb) in emission order, in tiles of
// kRowTile rows per CTA (as K5 padded_batches): each row finds its batch by a
// binary search over the row prefix roff, resolves (position, length,
// offset, destination) into shared memory, then warps stream the tile with
// kLoads token loads in flight per lane.
constexpr int kRowTile = 128;
#ifndef DP_TOK_LOADS
#define DP_TOK_LOADS 16
#endif
#ifndef DP_TOK_MINB
#define DP_TOK_MINB 1
#endif
constexpr int kLoads = DP_TOK_LOADS;

__global__ void __launch_bounds__(kThreads, DP_TOK_MINB)
bucket_batches_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                      const int32_t* __restrict__ lengths, const int64_t* __restrict__ perm,
                      const int64_t* __restrict__ start, const int32_t* __restrict__ lmax_of,
                      const int64_t* __restrict__ boff, const int64_t* __restrict__ roff, int64_t first, int64_t nb,
                      int32_t pad, int32_t* __restrict__ out, int32_t* __restrict__ out_lengths) {
  __shared__ int64_t s_src[kRowTile], s_dst[kRowTile];
  __shared__ int32_t s_len[kRowTile], s_lm[kRowTile];
  __shared__ int64_t s_e0;
  const int64_t r_first = roff[first], rows = roff[first + nb] - r_first;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRowTile;
  const int n = static_cast<int>(rows - t0 < kRowTile ? rows - t0 : kRowTile);
  if (threadIdx.x == 0) {  // the batch e with roff[e] <= R < roff[e + 1] for the tile's first row
    const int64_t R = r_first + t0;
    int64_t lo = first, hi = first + nb - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (roff[mid] <= R) lo = mid;
      else hi = mid - 1;
    }
    s_e0 = lo;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += kThreads) {
    const int64_t R = r_first + t0 + t;  // row in the epoch's emission order
    int64_t e = s_e0;                    // a tile spans few batches: walk forward
    while (roff[e + 1] <= R) ++e;
    const int64_t r = R - roff[e];
    const int64_t p = perm[start[e] + r];
    const int32_t len = lengths[p], lm = lmax_of[e];
    s_src[t] = offsets[p];
    s_len[t] = len;
    s_lm[t] = lm;
    s_dst[t] = (boff[e] - boff[first]) + r * lm;
    out_lengths[R - r_first] = len;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int t = threadIdx.x >> 5; t < n; t += 2 * kWarps) {  // rows t and t + kWarps
    const int b = t + kWarps, has_b = b < n;
    stream_row_pair<kLoads>(tokens + s_src[t], s_len[t], s_lm[t], out + s_dst[t], has_b ? tokens + s_src[b] : tokens,
                            has_b ? s_len[b] : 0, has_b ? s_lm[b] : 0, has_b ? out + s_dst[b] : out, pad, lane);
  }
}

// Per-row tables of an epoch's bucket plan (built once per epoch on the plan
// stream): emitted row R of batch e, row r, reads source position
// perm[start_e + r] and lands at boff_e + r * lmax_e, width lmax_e.  The
// batch kernel's preamble then needs one coalesced read per table plus the
// (length, offset) gather, as K5 padded_batches, instead of a batch search,
// a forward walk over roff and the dependent perm read per row.
__global__ void __launch_bounds__(kThreads)
bucket_rows_kernel(const int64_t* __restrict__ perm, const int64_t* __restrict__ start,
                   const int32_t* __restrict__ lmax_of, const int64_t* __restrict__ boff,
                   const int64_t* __restrict__ roff, int64_t* __restrict__ row_src, int64_t* __restrict__ row_dst,
                   int32_t* __restrict__ row_lm) {
  const int64_t e = blockIdx.x, r0 = roff[e], rows = roff[e + 1] - r0, s0 = start[e], b0 = boff[e];
  const int32_t lm = lmax_of[e];
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    row_src[r0 + r] = perm[s0 + r];
    row_dst[r0 + r] = b0 + r * lm;
    row_lm[r0 + r] = lm;
  }
}

__global__ void __launch_bounds__(kThreads, DP_TOK_MINB)
bucket_rows_batches_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                           const int32_t* __restrict__ lengths, const int64_t* __restrict__ row_src,
                           const int64_t* __restrict__ row_dst, const int32_t* __restrict__ row_lm, int64_t r_first,
                           int64_t b_first, int64_t rows, int32_t pad, int32_t* __restrict__ out,
                           int32_t* __restrict__ out_lengths) {
  __shared__ int64_t s_src[kRowTile], s_dst[kRowTile];
  __shared__ int32_t s_len[kRowTile], s_lm[kRowTile];
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRowTile;
  const int n = static_cast<int>(rows - t0 < kRowTile ? rows - t0 : kRowTile);
  for (int t = threadIdx.x; t < n; t += kThreads) {
    const int64_t R = r_first + t0 + t;
    const int64_t p = __ldcs(row_src + R);
    const int32_t len = lengths[p];
    s_src[t] = offsets[p];
    s_len[t] = len;
    s_lm[t] = __ldcs(row_lm + R);
    s_dst[t] = __ldcs(row_dst + R) - b_first;
    out_lengths[t0 + t] = len;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int t = threadIdx.x >> 5; t < n; t += 2 * kWarps) {  // rows t and t + kWarps
    const int b = t + kWarps, has_b = b < n;
    stream_row_pair<kLoads>(tokens + s_src[t], s_len[t], s_lm[t], out + s_dst[t], has_b ? tokens + s_src[b] : tokens,
                            has_b ? s_len[b] : 0, has_b ? s_lm[b] : 0, has_b ? out + s_dst[b] : out, pad, lane);
  }
}

struct PlanScratch {
  int64_t* tile_counts;
  int64_t* meta;
  int32_t* close;
  int32_t* bucket;
  int64_t* rank;
  int64_t* closing;
  int64_t* num_closing;
  void* filter_scratch;
};

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

PlanScratch carve(void* scratch, int64_t n, int K) {
  const int64_t tiles = (n + kTile - 1) / kTile;
  auto* p = static_cast<uint8_t*>(scratch);
  PlanScratch s;
  s.tile_counts = reinterpret_cast<int64_t*>(p);
  p += align256(sizeof(int64_t) * (tiles < 1 ? 1 : tiles) * K);
  s.meta = reinterpret_cast<int64_t*>(p);
  p += align256(sizeof(int64_t) * 2 * DP_MAX_BUCKETS);
  s.close = reinterpret_cast<int32_t*>(p);
  p += align256(sizeof(int32_t) * (n < 1 ? 1 : n));
  s.bucket = reinterpret_cast<int32_t*>(p);
  p += align256(sizeof(int32_t) * (n < 1 ? 1 : n));
  s.rank = reinterpret_cast<int64_t*>(p);
  p += align256(sizeof(int64_t) * (n < 1 ? 1 : n));
  s.closing = reinterpret_cast<int64_t*>(p);
  p += align256(sizeof(int64_t) * (n < 1 ? 1 : n));
  s.num_closing = reinterpret_cast<int64_t*>(p);
  p += align256(sizeof(int64_t));
  s.filter_scratch = p;
  return s;
}

int make_spec(const int32_t* boundaries, int num_boundaries, const int64_t* batch_sizes, int drop, BucketSpec& s) {
  if (num_boundaries < 0 || num_boundaries > DP_MAX_BUCKETS - 1 || (num_boundaries && !boundaries) || !batch_sizes)
    return fail(DP_ERR_INVALID_ATTR, "bucket_by_length: 0..31 boundaries and one batch size per bucket");
  s = BucketSpec{};
  s.num_bounds = num_boundaries;
  s.drop = drop ? 1 : 0;
  for (int k = 0; k < num_boundaries; ++k) {
    if (k && boundaries[k] <= boundaries[k - 1])
      return fail(DP_ERR_INVALID_ATTR, "bucket_by_length: boundaries must increase");
    s.bounds[k] = boundaries[k];
  }
  for (int k = 0; k <= num_boundaries; ++k) {
    if (batch_sizes[k] < 1) return fail(DP_ERR_INVALID_ATTR, "bucket_by_length: batch sizes must be >= 1");
    s.size[k] = batch_sizes[k];
  }
  return DP_OK;
}

}  // namespace
}  // namespace dpk

using namespace dpk;

extern "C" size_t dp_k_bucket_scratch_bytes(int64_t n, int num_buckets) {
  const int K = num_buckets < 1 ? 1 : num_buckets;
  const int64_t tiles = (n + kTile - 1) / kTile;
  const int64_t m = n < 1 ? 1 : n;
  return align256(sizeof(int64_t) * (tiles < 1 ? 1 : tiles) * K) + align256(sizeof(int64_t) * 2 * DP_MAX_BUCKETS) +
         2 * align256(sizeof(int32_t) * m) + 2 * align256(sizeof(int64_t) * m) + align256(sizeof(int64_t)) +
         dp_k_filter_scratch_bytes(n);
}

extern "C" int dp_k_bucket_plan(const int32_t* lengths, const int64_t* order, int64_t n, const int32_t* boundaries,
                                int num_boundaries, const int64_t* batch_sizes, int drop_remainder, int64_t* perm,
                                int64_t* batch_start, int32_t* batch_rows, int32_t* batch_lmax,
                                int64_t* num_batches_dev, void* scratch, void* stream) {
  BucketSpec spec;
  if (int st = make_spec(boundaries, num_boundaries, batch_sizes, drop_remainder, spec)) return st;
  if (n < 0 || !lengths || !perm || !batch_start || !batch_rows || !batch_lmax || !num_batches_dev || !scratch)
    return fail(DP_ERR_INVALID_ATTR, "bucket_by_length: null argument");
  cudaStream_t s = as_stream(stream);
  if (n == 0) return cuda_status(cudaMemsetAsync(num_batches_dev, 0, sizeof(int64_t), s), "bucket: memset");
  const int K = num_boundaries + 1;
  const int64_t tiles = (n + kTile - 1) / kTile;
  if (tiles > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "bucket_by_length: n too large");
  PlanScratch sc = carve(scratch, n, K);
  bucket_count_kernel<<<static_cast<int>(tiles), kThreads, 0, s>>>(lengths, order, n, spec, sc.tile_counts);
  bucket_scan_kernel<<<1, 1024, 0, s>>>(sc.tile_counts, tiles, K, sc.meta);
  bucket_scatter_kernel<<<static_cast<int>(tiles), kThreads, 0, s>>>(lengths, order, n, spec, sc.tile_counts, sc.meta,
                                                                     perm, sc.close, sc.bucket, sc.rank);
  if (int st = dp_k_filter_len_le(sc.close, n, 0, nullptr, sc.closing, sc.num_closing, sc.filter_scratch, s)) return st;
  const int64_t desc_blocks = (n + kThreads - 1) / kThreads + 1;
  bucket_desc_kernel<<<static_cast<int>(desc_blocks), kThreads, 0, s>>>(sc.closing, sc.num_closing, sc.bucket, sc.rank,
                                                                        spec, sc.meta, batch_start, batch_rows,
                                                                        num_batches_dev);
  const int64_t max_batches = n + K;
  bucket_lmax_kernel<<<static_cast<int>((max_batches + kWarps - 1) / kWarps), kThreads, 0, s>>>(
      lengths, perm, batch_start, batch_rows, num_batches_dev, batch_lmax);
  return launch_status("bucket_plan");
}

extern "C" int dp_k_bucket_rows(const int64_t* perm, const int64_t* batch_start, const int32_t* batch_lmax,
                                const int64_t* boff, const int64_t* roff, int64_t num_batches, int64_t* row_src,
                                int64_t* row_dst, int32_t* row_lm, void* stream) {
  if (num_batches < 0 || num_batches > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "bucket_rows: bad batch count");
  if (num_batches == 0) return DP_OK;
  bucket_rows_kernel<<<static_cast<int>(num_batches), kThreads, 0, as_stream(stream)>>>(
      perm, batch_start, batch_lmax, boff, roff, row_src, row_dst, row_lm);
  return launch_status("bucket_rows");
}

extern "C" int dp_k_bucket_rows_batches(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                                        const int64_t* row_src, const int64_t* row_dst, const int32_t* row_lm,
                                        int64_t first_row, int64_t first_elem, int64_t num_rows, int32_t pad_value,
                                        int32_t* out, int32_t* out_lengths, void* stream) {
  if (first_row < 0 || first_elem < 0 || num_rows < 0) return fail(DP_ERR_INVALID_ATTR, "bucket_batches: bad range");
  if (num_rows == 0) return DP_OK;
  const int64_t blocks = (num_rows + kRowTile - 1) / kRowTile;
  if (blocks > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "bucket_batches: too many rows");
  bucket_rows_batches_kernel<<<static_cast<int>(blocks), kThreads, 0, as_stream(stream)>>>(
      tokens, offsets, lengths, row_src, row_dst, row_lm, first_row, first_elem, num_rows, pad_value, out,
      out_lengths);
  return launch_status("bucket_batches");
}

extern "C" int dp_k_bucket_batches(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                                   const int64_t* perm, const int64_t* batch_start, const int32_t* batch_rows,
                                   const int32_t* batch_lmax, const int64_t* boff, const int64_t* roff, int64_t first,
                                   int64_t num, int64_t num_rows, int32_t pad_value, int32_t* out,
                                   int32_t* out_lengths, void* stream) {
  (void)batch_rows;  // implied by roff
  if (first < 0 || num < 0 || num_rows < 0) return fail(DP_ERR_INVALID_ATTR, "bucket_batches: bad range");
  if (num == 0 || num_rows == 0) return DP_OK;
  const int64_t blocks = (num_rows + kRowTile - 1) / kRowTile;
  if (blocks > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "bucket_batches: too many rows");
  bucket_batches_kernel<<<static_cast<int>(blocks), kThreads, 0, as_stream(stream)>>>(
      tokens, offsets, lengths, perm, batch_start, batch_lmax, boff, roff, first, num, pad_value, out, out_lengths);
  return launch_status("bucket_batches");
}
