// k_index.cu -- K1 range_affine_batch, K6 shard / interleave index mapping,
// K7 order digest, synthetic input generators.  All HBM-bound integer work.
#include <algorithm>
#include <cstdint>
#include <queue>
#include <vector>

#include "common.cuh"
#include "status.hpp"

namespace dpk {
namespace {

constexpr int kThreads = 256;

int grid_for(int64_t work_items, int per_thread) {
  int64_t blocks = (work_items + static_cast<int64_t>(kThreads) * per_thread - 1) /
                   (static_cast<int64_t>(kThreads) * per_thread);
  if (blocks < 1) blocks = 1;
  // Grid-stride loops cover the rest; 148 SMs x 8 resident 256-thread CTAs.
  const int64_t cap = 148LL * 8 * 16;
  return static_cast<int>(blocks < cap ? blocks : cap);
}

// K1: out[i] = (first + i) * a + b, two int64 per thread with one 16-byte
// streaming store when the slot is 16-byte aligned (engine slots always are).
__global__ void __launch_bounds__(kThreads)
range_affine_kernel(int64_t first, int64_t rows, int64_t a, int64_t b, int64_t* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (vec) {
    const int64_t pairs = rows >> 1;
    for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < pairs; p += stride) {
      int64_t x0 = (first + 2 * p) * a + b;
      int64_t x1 = (first + 2 * p + 1) * a + b;
      asm volatile("st.global.cs.v2.s64 [%0], {%1, %2};" ::"l"(out + 2 * p), "l"(x0), "l"(x1) : "memory");
    }
    if ((rows & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[rows - 1] = (first + rows - 1) * a + b;
  } else {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += stride)
      out[i] = (first + i) * a + b;
  }
}

// K1 general form: out[i] = v * a + b, v = values ? values[p] : p,
// p = order ? order[first + i] : first + i  (gathered int64 source).
__global__ void __launch_bounds__(kThreads)
gather_affine_kernel(const int64_t* __restrict__ values, const int64_t* __restrict__ order, int64_t first, int64_t rows,
                     int64_t a, int64_t b, int64_t* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += stride) {
    const int64_t p = order ? order[first + i] : first + i;
    const int64_t v = values ? values[p] : p;
    out[i] = v * a + b;
  }
}

// K6: closed form of the deterministic interleave over equal-length readers
// (validated against the reference runtime in tests/test_oracle.py): inputs
// are opened in groups of `cycle`; group G holds inputs G*c .. G*c+m-1 with
// m = min(c, M - G*c) live slots and emits `records` rounds of one element
// per live slot.  Input i is source ordinal shard_index + i * num_shards.
__global__ void __launch_bounds__(kThreads)
shard_interleave_kernel(int64_t m_inputs, int64_t num_shards, int64_t shard_index, int64_t cycle,
                        int64_t records, int64_t count, int64_t* __restrict__ out) {
  // inputs: source ordinal shard_index + i * num_shards, i < m_inputs
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t group_elems = cycle * records;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += stride) {
    int64_t g = t / group_elems;
    int64_t g0 = g * cycle;
    int64_t m = m_inputs - g0 < cycle ? m_inputs - g0 : cycle;
    int64_t p = t - g * group_elems;
    int64_t r = p / m;
    int64_t s = p - r * m;
    int64_t src = shard_index + (g0 + s) * num_shards;
    out[t] = src * records + r;
  }
}

__global__ void __launch_bounds__(kThreads)
shard_kernel(int64_t count, int64_t num_shards, int64_t shard_index, const int64_t* __restrict__ in_map,
             int64_t* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    int64_t p = shard_index + i * num_shards;
    out[i] = in_map ? in_map[p] : p;
  }
}

__device__ __forceinline__ uint64_t position_hash(uint64_t v, uint64_t i) {
  uint64_t s = v ^ (i * 0x9e3779b97f4a7c15ULL);
  return splitmix64_next(s);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
digest_kernel(const T* __restrict__ values, int64_t n, int64_t first, unsigned long long* digest) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint64_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    acc += position_hash(static_cast<uint64_t>(values[i]), static_cast<uint64_t>(first + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(digest, static_cast<unsigned long long>(acc));
}

// 16 pixels per thread: pixel g (global byte index from image first_id) is
// the top byte of SplitMix64Next(seed ^ (first_id * image_bytes + g)).
__global__ void __launch_bounds__(kThreads)
synth_images_kernel(uint8_t* __restrict__ images, uint64_t base, uint64_t total, uint64_t seed) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 16;
  for (uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16; g < total; g += stride) {
    if (g + 16 <= total) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint64_t s = seed ^ (base + g + q * 4 + u);
          acc |= static_cast<uint32_t>(splitmix64_next(s) >> 56) << (8 * u);
        }
        w[q] = acc;
      }
      *reinterpret_cast<uint4*>(images + g) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (uint64_t b = g; b < total; ++b) {
        uint64_t s = seed ^ (base + b);
        images[b] = static_cast<uint8_t>(splitmix64_next(s) >> 56);
      }
    }
  }
}

// One warp per sequence.
__global__ void __launch_bounds__(kThreads)
synth_tokens_kernel(int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n, uint64_t seed) {
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; i < n; i += warps) {
    int64_t off = offsets[i], len = offsets[i + 1] - off;
    for (int64_t j = lane; j < len; j += 32) {
      uint64_t s = seed ^ ((static_cast<uint64_t>(i) << 20) | static_cast<uint64_t>(j));
      tokens[off + j] = static_cast<int32_t>(splitmix64_next(s) & 0x7fffffffULL);
    }
  }
}

}  // namespace
}  // namespace dpk

using namespace dpk;

extern "C" int dp_k_range_affine_batch(int64_t first, int64_t rows, int64_t a, int64_t b, int64_t* out,
                                       void* stream) {
  if (rows < 0 || (rows > 0 && !out)) return fail(DP_ERR_INVALID_ATTR, "range_affine_batch: bad rows/out");
  if (rows == 0) return DP_OK;
  range_affine_kernel<<<grid_for((rows + 1) / 2, 1), kThreads, 0, as_stream(stream)>>>(first, rows, a, b, out);
  return launch_status("range_affine_batch");
}

extern "C" int dp_k_gather_affine_batch(const int64_t* values, const int64_t* order, int64_t first, int64_t rows,
                                        int64_t a, int64_t b, int64_t* out, void* stream) {
  if (rows < 0 || (rows > 0 && !out)) return fail(DP_ERR_INVALID_ATTR, "gather_affine_batch: bad rows/out");
  if (rows == 0) return DP_OK;
  gather_affine_kernel<<<grid_for(rows, 1), kThreads, 0, as_stream(stream)>>>(values, order, first, rows, a, b, out);
  return launch_status("gather_affine_batch");
}

extern "C" int dp_k_interleave_index(int64_t first, int64_t stride, int64_t m_inputs, int64_t cycle, int64_t records,
                                     int64_t* out, void* stream) {
  if (cycle < 1) return fail(DP_ERR_INVALID_ATTR, "interleave_index: cycle_length must be >= 1");
  if (records < 0 || m_inputs < 0) return fail(DP_ERR_INVALID_ATTR, "interleave_index: bad sizes");
  const int64_t count = m_inputs * records;
  if (count == 0) return DP_OK;
  shard_interleave_kernel<<<grid_for(count, 1), kThreads, 0, as_stream(stream)>>>(m_inputs, stride, first, cycle,
                                                                                    records, count, out);
  return launch_status("interleave_index");
}

namespace dpk {
namespace {
// K6 over readers of unequal lengths.  The host schedules the inputs
// (dp_interleave_schedule): input i runs in cycle slot slot[i] during visits
// ("rounds") [start[i], start[i] + len[i]), each slot's inputs back to back;
// end[s] = the round slot s goes dead.  Element j of input i is emitted at
// round r = start[i] + j and its position is
//   sum_s' min(end[s'], r) + #{s' < slot[i] : end[s'] > r}
// (every slot emits once per round until it is dead).  One CTA per input.
__global__ void __launch_bounds__(kThreads)
interleave_var_kernel(const int64_t* __restrict__ slot, const int64_t* __restrict__ start,
                      const int64_t* __restrict__ len, const int64_t* __restrict__ first_record,
                      const int64_t* __restrict__ end, int cycle, int64_t* __restrict__ out) {
  extern __shared__ int64_t s_end[];
  for (int s = threadIdx.x; s < cycle; s += blockDim.x) s_end[s] = end[s];
  __syncthreads();
  const int64_t i = blockIdx.x, sl = slot[i], st = start[i], rec = first_record[i];
  for (int64_t j = threadIdx.x; j < len[i]; j += blockDim.x) {
    const int64_t r = st + j;
    int64_t pos = 0;
    for (int s = 0; s < cycle; ++s) {
      const int64_t e = s_end[s];
      pos += e < r ? e : r;
      pos += (s < sl && e > r) ? 1 : 0;
    }
    out[pos] = rec + j;
  }
}
}  // namespace
}  // namespace dpk

extern "C" int dp_interleave_schedule(int64_t m_inputs, const int64_t* lengths, int64_t cycle, int64_t* slot,
                                      int64_t* start, int64_t* end) {
  if (m_inputs < 0 || cycle < 1 || (m_inputs && (!lengths || !slot || !start)) || !end)
    return fail(DP_ERR_INVALID_ATTR, "interleave_schedule: bad arguments");
  // (round, slot) of the visits that need a new input, smallest first: the
  // InterleaveIterator loop (runtime.cpp:1061-1120) opens inputs in visit
  // order, and an exhausted slot opens the next one in the same visit
  using Visit = std::pair<int64_t, int64_t>;
  std::priority_queue<Visit, std::vector<Visit>, std::greater<Visit>> need;
  for (int64_t s = 0; s < cycle; ++s) {
    need.push({0, s});
    end[s] = 0;
  }
  for (int64_t i = 0; i < m_inputs; ++i) {
    if (lengths[i] < 0) return fail(DP_ERR_INVALID_ATTR, "interleave_schedule: negative length");
    const Visit v = need.top();
    need.pop();
    slot[i] = v.second;
    start[i] = v.first;
    end[v.second] = v.first + lengths[i];
    need.push({end[v.second], v.second});
  }
  return DP_OK;
}

extern "C" int dp_k_interleave_var(int64_t m_inputs, const int64_t* slot, const int64_t* start, const int64_t* len,
                                   const int64_t* first_record, const int64_t* end, int64_t cycle, int64_t* out,
                                   void* stream) {
  if (m_inputs < 0 || cycle < 1 || cycle > 4096) return fail(DP_ERR_INVALID_ATTR, "interleave_var: bad sizes");
  if (m_inputs == 0) return DP_OK;
  if (m_inputs > 0x7fffffff) return fail(DP_ERR_INVALID_ATTR, "interleave_var: too many inputs");
  interleave_var_kernel<<<static_cast<int>(m_inputs), kThreads, sizeof(int64_t) * cycle, as_stream(stream)>>>(
      slot, start, len, first_record, end, static_cast<int>(cycle), out);
  return launch_status("interleave_var");
}

extern "C" int64_t dp_k_shard_interleave_count(int64_t n_sources, int64_t num_shards, int64_t shard_index,
                                               int64_t records) {
  if (num_shards < 1 || shard_index < 0 || shard_index >= num_shards || n_sources <= shard_index) return 0;
  int64_t m = (n_sources - shard_index + num_shards - 1) / num_shards;
  return m * records;
}

extern "C" int dp_k_shard_interleave_index(int64_t n_sources, int64_t num_shards, int64_t shard_index,
                                           int64_t cycle, int64_t records, int64_t* out, void* stream) {
  if (num_shards < 1 || shard_index < 0 || shard_index >= num_shards)
    return fail(DP_ERR_INVALID_ATTR, "shard_interleave_index: index must be in [0, num_shards)");
  if (cycle < 1) return fail(DP_ERR_INVALID_ATTR, "shard_interleave_index: cycle_length must be >= 1");
  if (records < 0) return fail(DP_ERR_INVALID_ATTR, "shard_interleave_index: records must be >= 0");
  int64_t count = dp_k_shard_interleave_count(n_sources, num_shards, shard_index, records);
  if (count == 0) return DP_OK;
  int64_t m = count / records;
  shard_interleave_kernel<<<grid_for(count, 1), kThreads, 0, as_stream(stream)>>>(m, num_shards, shard_index,
                                                                                    cycle, records, count, out);
  return launch_status("shard_interleave_index");
}

extern "C" int dp_k_shard_index(int64_t n, int64_t num_shards, int64_t shard_index, const int64_t* in_map,
                                int64_t* out, void* stream) {
  if (num_shards < 1 || shard_index < 0 || shard_index >= num_shards)
    return fail(DP_ERR_INVALID_ATTR, "shard_index: index must be in [0, num_shards)");
  if (n <= shard_index) return DP_OK;
  int64_t count = (n - shard_index + num_shards - 1) / num_shards;
  shard_kernel<<<grid_for(count, 1), kThreads, 0, as_stream(stream)>>>(count, num_shards, shard_index, in_map, out);
  return launch_status("shard_index");
}

extern "C" int dp_k_order_digest(const int64_t* values, int64_t n, int64_t first, uint64_t* digest_dev,
                                 void* stream) {
  if (n <= 0) return DP_OK;
  digest_kernel<int64_t><<<grid_for(n, 8), kThreads, 0, as_stream(stream)>>>(
      values, n, first, reinterpret_cast<unsigned long long*>(digest_dev));
  return launch_status("order_digest");
}

extern "C" int dp_k_word_digest(const uint32_t* words, int64_t n, int64_t first, uint64_t* digest_dev,
                                void* stream) {
  if (n <= 0) return DP_OK;
  digest_kernel<uint32_t><<<grid_for(n, 8), kThreads, 0, as_stream(stream)>>>(
      words, n, first, reinterpret_cast<unsigned long long*>(digest_dev));
  return launch_status("word_digest");
}

extern "C" int dp_k_synth_images_strided(uint8_t* images, uint64_t first_id, uint64_t id_stride, uint64_t count,
                                         uint64_t image_bytes, uint64_t seed, void* stream) {
  if (id_stride <= 1) return dp_k_synth_images(images, first_id, count, image_bytes, seed, stream);
  if (reinterpret_cast<uintptr_t>(images) & 15)
    return fail(DP_ERR_INVALID_ATTR, "synth_images: buffer must be 16-byte aligned");
  // one launch per row (setup path, not timed): rows are contiguous id runs of length 1
  for (uint64_t i = 0; i < count; ++i) {
    synth_images_kernel<<<grid_for(static_cast<int64_t>((image_bytes + 15) / 16), 4), kThreads, 0,
                          as_stream(stream)>>>(images + i * image_bytes, (first_id + i * id_stride) * image_bytes,
                                               image_bytes, seed);
  }
  return launch_status("synth_images_strided");
}

extern "C" int dp_k_synth_images(uint8_t* images, uint64_t first_id, uint64_t count, uint64_t image_bytes,
                                 uint64_t seed, void* stream) {
  uint64_t total = count * image_bytes;
  if (total == 0) return DP_OK;
  if (reinterpret_cast<uintptr_t>(images) & 15)
    return fail(DP_ERR_INVALID_ATTR, "synth_images: buffer must be 16-byte aligned");
  synth_images_kernel<<<grid_for(static_cast<int64_t>((total + 15) / 16), 4), kThreads, 0, as_stream(stream)>>>(
      images, first_id * image_bytes, total, seed);
  return launch_status("synth_images");
}

extern "C" int dp_k_synth_tokens(int32_t* tokens, const int64_t* offsets, int64_t n, uint64_t seed,
                                 void* stream) {
  if (n <= 0) return DP_OK;
  synth_tokens_kernel<<<grid_for(n * 32, 1), kThreads, 0, as_stream(stream)>>>(tokens, offsets, n, seed);
  return launch_status("synth_tokens");
}

namespace dpk {
namespace {
// rows x width bytes from a pitched source into a packed destination; the
// destination is typically mapped pinned host memory (an SM-side write over
// PCIe that does not queue behind the copy engines)
__global__ void copy_strided_kernel(const uint8_t* __restrict__ src, size_t pitch, size_t width, size_t rows,
                                    uint8_t* __restrict__ dst) {
  const size_t total = width * rows;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / width, c = i - r * width;
    dst[i] = src[r * pitch + c];
  }
}
}  // namespace
}  // namespace dpk

extern "C" int dp_k_copy_strided(const void* src, size_t src_pitch, size_t width, size_t rows, void* dst,
                                 void* stream) {
  if (width == 0 || rows == 0) return DP_OK;
  if (!src || !dst || src_pitch < width) return dpk::fail(DP_ERR_INVALID_ATTR, "copy_strided: bad arguments");
  const size_t total = width * rows;
  const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 4));
  dpk::copy_strided_kernel<<<blocks, 256, 0, dpk::as_stream(stream)>>>(static_cast<const uint8_t*>(src), src_pitch,
                                                                        width, rows, static_cast<uint8_t*>(dst));
  return dpk::launch_status("copy_strided");
}
