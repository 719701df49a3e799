// k_shuffle.cu -- K2 shuffle_plan: the exact emission order of the
// reference's windowed-reservoir shuffle, computed on the device.
//
// Reference: ShuffleIterator::Next, /root/reference/proj/src/runtime.cpp:
// 721-747 (prime `cap` = min(n, buffer) inputs; each step draws
// idx = Pcg32::Bounded(size) (random.hpp:57-63), emits buffer[idx], refills
// it with the next input, or, once the input is exhausted, moves back() into
// idx and pops).
//
// Two implementations of the same contract:
//  * the device-wide plan (default, below the warp kernel): grid passes over
//    all draws -- see its comment block;
//  * the single-warp kernel (degenerate buffers with F / cap > 256, where
//    slot buckets would be long), decomposed as follows.
// Decomposition:
//  * fill phase, steps k < F = n - cap: the bound is fixed at cap, so which
//    raw PCG outputs are rejected (r < 2^32 mod cap) does not depend on the
//    buffer.  One warp walks the PCG stream 32 raws per iteration, each lane
//    positioned with an O(log k) LCG jump; a ballot assigns draw numbers to
//    the accepted lanes.  The buffer dependency is "slot idx_k last written
//    by step k' < k holds ordinal cap + k'": lanes resolve earlier writers in
//    the same iteration with __match_any_sync and read older ones from the
//    slot table (shared memory when it fits).
//  * drain phase (cap steps, bound cap, cap-1, ..., 1): rejections are still
//    buffer independent; the warp finds them 32 draws at a time (assuming none,
//    then cutting at the first rejecting lane), and lane 0 applies the
//    swap-with-last updates in order.
// The result is bit-identical to the sequential reference for every n,
// buffer and seed (tests/test_gpu_parity.py).
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "status.hpp"

namespace dpk {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr size_t kMaxSmemBuffer = 200 * 1024;

__global__ void __launch_bounds__(32)
shuffle_plan_kernel(uint64_t n, uint32_t cap, uint64_t engine_seed, const int64_t* __restrict__ in_map,
                    int64_t* __restrict__ out, uint32_t* __restrict__ gbuf) {
  extern __shared__ uint32_t sbuf[];
  __shared__ LcgJump jumps[33];  // jumps[k] advances a lane by k raws
  uint32_t* buf = gbuf ? gbuf : sbuf;
  const int lane = threadIdx.x;
  const uint32_t lt = (1u << lane) - 1u;

  jumps[lane + 1] = lcg_jump(static_cast<uint64_t>(lane) + 1);
  if (lane == 0) jumps[0] = lcg_jump(0);
  for (uint32_t i = lane; i < cap; i += 32) buf[i] = i;
  __syncwarp();

  const uint64_t s0 = pcg_seeded_state(engine_seed);
  const uint64_t fill = n - cap;
  uint64_t s = lcg_apply(jumps[lane], s0);
  const LcgJump j32 = jumps[32];
  uint64_t raw_consumed = 0;

  // ---- fill phase ----
  {
    const uint32_t thr = (0u - cap) % cap;
    uint64_t k = 0;
    while (k < fill) {
      const uint32_t r = pcg_output(s);
      s = lcg_apply(j32, s);
      const bool acc = r >= thr;
      const uint32_t bal = __ballot_sync(kFull, acc);
      const uint64_t kk = k + __popc(bal & lt);
      const bool valid = acc && kk < fill;
      const uint32_t idx = r % cap;
      const uint32_t key = valid ? idx : (0x80000000u | static_cast<uint32_t>(lane));
      const uint32_t peers = __match_any_sync(kFull, key);
      const uint32_t below = peers & lt;
      const int pred = below ? 31 - __clz(below) : lane;
      const uint64_t kk_pred = __shfl_sync(kFull, kk, pred);
      const uint32_t cur = valid ? buf[idx] : 0u;
      __syncwarp();
      if (valid) {
        const uint64_t ord = below ? static_cast<uint64_t>(cap) + kk_pred : static_cast<uint64_t>(cur);
        out[kk] = in_map ? in_map[ord] : static_cast<int64_t>(ord);
        const bool last_writer = (peers & ~lt & ~(1u << lane)) == 0;
        if (last_writer) buf[idx] = static_cast<uint32_t>(cap + kk);
      }
      __syncwarp();
      const uint32_t nacc = __popc(bal);
      if (k + nacc >= fill) {
        const uint32_t m = __ballot_sync(kFull, valid && kk == fill - 1);
        raw_consumed += static_cast<uint64_t>(__ffs(m));  // lane of draw F-1, plus one
        k = fill;
      } else {
        k += nacc;
        raw_consumed += 32;
      }
    }
  }

  // ---- drain phase ----
  s = lcg_apply(lcg_jump(raw_consumed + static_cast<uint64_t>(lane)), s0);
  uint64_t pos = fill;
  uint32_t size = cap;
  while (size > 0) {
    const uint32_t r = pcg_output(s);
    const bool active = static_cast<uint32_t>(lane) < size;
    const uint32_t b = active ? size - static_cast<uint32_t>(lane) : 1u;
    const uint32_t thr = (0u - b) % b;
    const uint32_t rm = __ballot_sync(kFull, active && r < thr);
    const int f = rm ? __ffs(rm) - 1 : 32;
    const int avail = size < 32u ? static_cast<int>(size) : 32;
    const int ndraw = f < avail ? f : avail;
    const int nconsumed = f < avail ? f + 1 : ndraw;
    const uint32_t idx = r % b;
    for (int d = 0; d < ndraw; ++d) {
      const uint32_t id_d = __shfl_sync(kFull, idx, d);
      if (lane == 0) {
        const uint32_t v = buf[id_d];
        out[pos + d] = in_map ? in_map[v] : static_cast<int64_t>(v);
        buf[id_d] = buf[size - 1 - d];
      }
    }
    __syncwarp();
    pos += ndraw;
    size -= ndraw;
    s = lcg_apply(jumps[nconsumed], s);
  }
}


// ===================================================================
// Device-wide plan (the default): every step is a grid-wide pass, no
// per-draw sequential chain.
//
//  P1  raws      r_j = PCG output j (LCG jump-ahead per thread), j < R
//  P2  fill      accept = r_j >= 2^32 mod cap; stable compaction numbers
//                the accepted raws as draws k < F (tile counts, one-CTA
//                scan, scatter) -> slot_k = r % cap; also records how many
//                raws the fill consumed
//  P3  buckets   per-slot counts, scan, scatter k into its slot's bucket
//  P4  resolve   draw k's predecessor in its slot = max k' < k in the
//                bucket (buckets hold F/cap draws on average): out_k =
//                cap + pred, or the slot's initial ordinal; the slot's last
//                writer sets B[slot] = cap + k
//  P5  drain     one CTA: draw ids (bound cap - d) with an exact parallel
//                rejection fix-up, position buckets, P(d) / R(e) by bucket
//                scans, terminal ancestors T(e) along R, and
//                out[F + d] = B[cap-1-T(P(d))] or B[id_d]
// Degenerate buffers (F / cap > 256, e.g. buffer 1) keep the warp kernel.
// ===================================================================
constexpr int kPT = 256;        // threads per CTA for the grid passes
constexpr int kRawPer = 16;     // raws per thread in P1
constexpr int kTileK = 4096;    // draws per compaction tile (256 x 16)
constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ uint32_t raw_at_state(uint64_t s0, uint64_t j) {
  return pcg_output(lcg_apply(lcg_jump(j), s0));
}

__global__ void __launch_bounds__(kPT) p1_raws(uint64_t s0, uint64_t R, uint32_t* __restrict__ raws) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * kPT + threadIdx.x;
  const uint64_t j0 = t * kRawPer;
  if (j0 >= R) return;
  uint64_t s = lcg_apply(lcg_jump(j0), s0);
#pragma unroll
  for (int u = 0; u < kRawPer; ++u) {
    if (j0 + u < R) raws[j0 + u] = pcg_output(s);
    s = pcg_step(s);
  }
}

__global__ void __launch_bounds__(kPT) p2_count(const uint32_t* __restrict__ raws, uint64_t R, uint32_t thr,
                                                uint64_t* __restrict__ tiles) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTileK + threadIdx.x * 16ull;
  int c = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) c += (base + u < R && raws[base + u] >= thr);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  __shared__ int ws[kPT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kPT / 32; ++w) t += ws[w];
    tiles[blockIdx.x] = t;
  }
}

// one-CTA exclusive scan of n 64-bit counts (in place); total -> *total
__global__ void __launch_bounds__(1024) scan_u64(uint64_t* __restrict__ v, uint64_t n, uint64_t* __restrict__ total) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < n; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t x0 = i < n ? v[i] : 0;
    uint64_t x = x0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint64_t w = ws[lane];
      uint64_t z = w;
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFull, z, o);
        if (lane >= o) z += y;
      }
      ws[lane] = z - w;
    }
    __syncthreads();
    const uint64_t ex = x - x0 + ws[warp] + carry;
    if (i < n) v[i] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) carry = ex + x0;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kPT) p2_scatter(const uint32_t* __restrict__ raws, uint64_t R, uint32_t thr,
                                                  uint32_t cap, uint64_t F, const uint64_t* __restrict__ tiles,
                                                  uint32_t* __restrict__ slot_of, uint32_t* __restrict__ counts,
                                                  uint64_t* __restrict__ meta) {
  __shared__ int ws[kPT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTileK + threadIdx.x * 16ull;
  uint32_t mask = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) mask |= (base + u < R && raws[base + u] >= thr) ? (1u << u) : 0u;
  const int c = __popc(mask);
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < kPT / 32 ? ws[lane] : 0;
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, z, o);
      if (lane >= o) z += y;
    }
    if (lane < kPT / 32) ws[lane] = z - w;
  }
  __syncthreads();
  uint64_t k = tiles[blockIdx.x] + (x - c) + ws[warp];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    if (mask & (1u << u)) {
      if (k < F) {
        const uint32_t s = raws[base + u] % cap;
        slot_of[k] = s;
        atomicAdd(&counts[s], 1u);
        if (k == F - 1) meta[0] = base + u + 1;  // raws consumed by the fill
      }
      ++k;
    }
  }
}

constexpr int kScanT = 1024;

__global__ void __launch_bounds__(kScanT) scan_small_u32(const uint32_t* __restrict__ counts, uint32_t cap,
                                                      uint32_t* __restrict__ start) {
  // single 1024-thread CTA: start[s] = sum_{s' < s} counts[s'] (cap <= 2^31, totals < 2^32)
  __shared__ uint32_t ws[kScanT / 32];
  __shared__ uint32_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < cap; base += kScanT) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t x0 = i < cap ? counts[i] : 0;
    uint32_t x = x0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = lane < kScanT / 32 ? ws[lane] : 0;
      uint32_t z = w;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, z, o);
        if (lane >= o) z += y;
      }
      if (lane < kScanT / 32) ws[lane] = z - w;
    }
    __syncthreads();
    const uint32_t ex = x - x0 + ws[warp] + carry;
    if (i < cap) start[i] = ex;
    __syncthreads();
    if (threadIdx.x == kScanT - 1) carry = ex + x0;
    __syncthreads();
  }
  if (threadIdx.x == 0) start[cap] = carry;
}

__global__ void __launch_bounds__(kPT) p3_bucket(const uint32_t* __restrict__ slot_of, uint64_t F,
                                                 const uint32_t* __restrict__ start, uint32_t* __restrict__ cursor,
                                                 uint32_t* __restrict__ bucket) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kPT;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kPT + threadIdx.x; k < F; k += stride) {
    const uint32_t s = slot_of[k];
    bucket[start[s] + atomicAdd(&cursor[s], 1u)] = static_cast<uint32_t>(k);
  }
}

__global__ void __launch_bounds__(kPT) p4_resolve(const uint32_t* __restrict__ slot_of, uint64_t F, uint32_t cap,
                                                  const uint32_t* __restrict__ start,
                                                  const uint32_t* __restrict__ bucket, uint32_t* __restrict__ B,
                                                  const int64_t* __restrict__ in_map, int64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kPT;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kPT + threadIdx.x; k < F; k += stride) {
    const uint32_t s = slot_of[k];
    const uint32_t b0 = start[s], b1 = start[s + 1];
    uint32_t pred = kNone;
    bool last = true;
    for (uint32_t i = b0; i < b1; ++i) {
      const uint32_t kk = bucket[i];
      if (kk < k && (pred == kNone || kk > pred)) pred = kk;
      if (kk > k) last = false;
    }
    const uint64_t ord = pred == kNone ? static_cast<uint64_t>(s) : static_cast<uint64_t>(cap) + pred;
    out[k] = in_map ? in_map[ord] : static_cast<int64_t>(ord);
    if (last) B[s] = static_cast<uint32_t>(cap + k);
  }
}

__global__ void __launch_bounds__(kPT) init_slots(uint32_t* __restrict__ B, uint32_t* __restrict__ counts,
                                                  uint32_t* __restrict__ cursor, uint32_t cap) {
  for (uint32_t i = blockIdx.x * kPT + threadIdx.x; i < cap; i += gridDim.x * kPT) {
    B[i] = i;
    counts[i] = 0;
    cursor[i] = 0;
  }
}

// in-place exclusive scan of n u32 by the whole CTA (blockDim 1024)
__device__ void block_scan_u32(uint32_t* v, uint32_t n, uint32_t* ws, uint32_t* carry) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) *carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t x0 = i < n ? v[i] : 0;
    uint32_t x = x0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = ws[lane];
      uint32_t z = w;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, z, o);
        if (lane >= o) z += y;
      }
      ws[lane] = z - w;
    }
    __syncthreads();
    const uint32_t ex = x - x0 + ws[warp] + *carry;
    if (i < n) v[i] = ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) *carry = ex + x0;
    __syncthreads();
  }
}

// Drain, one CTA of 1024 threads.  dstate = ids[cap] | start[cap+1] |
// cursor[cap] (then terminal ancestors) | bucket[cap] | par[cap].
__global__ void __launch_bounds__(1024) p5_drain(uint64_t s0, const uint32_t* __restrict__ raws, uint64_t R,
                                                 const uint64_t* __restrict__ meta, uint64_t F, uint32_t cap,
                                                 const uint32_t* __restrict__ B, uint32_t* __restrict__ gstate,
                                                 const int64_t* __restrict__ in_map, int64_t* __restrict__ out) {
  // work arrays in shared memory when they fit (every phase is a chain of
  // dependent lookups: smem latency instead of L2 latency), else global
  extern __shared__ uint32_t sstate[];
  uint32_t* dstate = gstate ? gstate : sstate;
  uint32_t* ids = dstate;
  uint32_t* start = ids + cap;
  uint32_t* cursor = start + cap + 1;
  uint32_t* bucket = cursor + cap;
  uint32_t* par = bucket + cap;
  __shared__ uint32_t ws[32], carry, first_rej;
  const uint64_t consumed = F ? meta[0] : 0;
  auto raw = [&](uint64_t q) { return q < R ? raws[q] : raw_at_state(s0, q); };

  // (a) ids: draw d uses raw consumed + d + shift(d); a rejected draw
  //     retries with the next raw, shifting every later draw by one
  uint64_t shift = 0;
  uint32_t d_start = 0;
  for (;;) {
    if (threadIdx.x == 0) first_rej = kNone;
    __syncthreads();
    for (uint32_t d = d_start + threadIdx.x; d < cap; d += blockDim.x) {
      const uint32_t b = cap - d;
      const uint32_t r = raw(consumed + d + shift);
      if (r < (0u - b) % b) atomicMin(&first_rej, d);
      else ids[d] = r % b;
    }
    __syncthreads();
    const uint32_t fr = first_rej;
    __syncthreads();
    if (fr == kNone) break;
    shift += 1;
    d_start = fr;
  }
  // (b) group steps by the position they read
  for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) {
    start[i] = 0;
    cursor[i] = 0;
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < cap; d += blockDim.x) atomicAdd(&start[ids[d]], 1u);
  __syncthreads();
  block_scan_u32(start, cap + 1, ws, &carry);
  for (uint32_t d = threadIdx.x; d < cap; d += blockDim.x) {
    const uint32_t p = ids[d];
    bucket[start[p] + atomicAdd(&cursor[p], 1u)] = d;
  }
  __syncthreads();
  // (c) R(e): last step before e that selected the tail position cap-1-e
  for (uint32_t e = threadIdx.x; e < cap; e += blockDim.x) {
    const uint32_t p = cap - 1 - e;
    uint32_t best = kNone;
    for (uint32_t i = start[p]; i < start[p + 1]; ++i) {
      const uint32_t d = bucket[i];
      if (d < e && (best == kNone || d > best)) best = d;
    }
    par[e] = best;
  }
  __syncthreads();
  // (d) terminal ancestors along R (chains are short for random draws)
  for (uint32_t e = threadIdx.x; e < cap; e += blockDim.x) {
    uint32_t x = e;
    while (par[x] != kNone) x = par[x];
    cursor[e] = x;
  }
  __syncthreads();
  // (e) step d emits src(P(d)) = B[cap-1-T(P(d))], or B[id_d] when the
  //     position was never written before d
  for (uint32_t d = threadIdx.x; d < cap; d += blockDim.x) {
    const uint32_t p = ids[d];
    uint32_t pd = kNone;
    for (uint32_t i = start[p]; i < start[p + 1]; ++i) {
      const uint32_t x = bucket[i];
      if (x < d && (pd == kNone || x > pd)) pd = x;
    }
    const uint32_t v = pd == kNone ? B[p] : B[cap - 1 - cursor[pd]];
    out[F + d] = in_map ? in_map[v] : static_cast<int64_t>(v);
  }
}

struct Layout {
  uint64_t R, F, tiles;
  size_t off_raws, off_slot, off_bucket, off_start, off_counts, off_cursor, off_B, off_tiles, off_dstate, off_meta,
      total;
};

Layout plan_layout(uint64_t n, uint32_t cap) {
  Layout l{};
  l.F = n - cap;
  // raws: the fill's draws plus a margin far beyond the rejections
  // (Binomial(R, p), p = (2^32 mod cap) / 2^32 < 1/2) and the drain's draws
  const double p = static_cast<double>((0u - cap) % cap) / 4294967296.0;
  const double fp = static_cast<double>(l.F);
  const uint64_t margin = static_cast<uint64_t>(fp * p / (1.0 - p) * 1.5 + 64.0 * std::sqrt(fp * p + 1.0) + 4096.0);
  l.R = l.F + margin + cap + 64;
  l.tiles = (l.R + kTileK - 1) / kTileK;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  l.off_raws = take(l.R * 4);
  l.off_slot = take(l.F * 4 + 4);
  l.off_bucket = take(l.F * 4 + 4);
  l.off_start = take((static_cast<size_t>(cap) + 1) * 4);
  l.off_counts = take(static_cast<size_t>(cap) * 4);
  l.off_cursor = take(static_cast<size_t>(cap) * 4);
  l.off_B = take(static_cast<size_t>(cap) * 4);
  l.off_tiles = take((l.tiles + 1) * 8);
  l.off_dstate = take((5 * static_cast<size_t>(cap) + 1) * 4);
  l.off_meta = take(64);
  l.total = off;
  return l;
}

bool use_device_plan(uint64_t n, uint32_t cap) { return n - cap <= 256ull * cap; }

}  // namespace
}  // namespace dpk

using namespace dpk;

extern "C" size_t dp_k_shuffle_plan_scratch_bytes(uint64_t n, uint64_t buffer_size) {
  if (n == 0 || buffer_size == 0 || n >= (1ULL << 32)) return 0;
  const uint64_t cap64 = buffer_size < n ? buffer_size : n;
  if (cap64 >= (1ULL << 31)) return 0;
  const uint32_t cap = static_cast<uint32_t>(cap64);
  if (use_device_plan(n, cap)) return plan_layout(n, cap).total;
  const size_t bytes = static_cast<size_t>(cap) * sizeof(uint32_t);
  return bytes > kMaxSmemBuffer ? bytes : 0;
}

extern "C" int dp_k_shuffle_plan(uint64_t n, uint64_t buffer_size, uint64_t engine_seed, const int64_t* in_map,
                                 int64_t* out, void* scratch, void* stream) {
  if (buffer_size < 1) return fail(DP_ERR_INVALID_ATTR, "shuffle: buffer_size must be >= 1");
  if (n >= (1ULL << 32)) return fail(DP_ERR_INVALID_ATTR, "shuffle_plan: n must be < 2^32");
  if (n == 0) return DP_OK;
  const uint64_t cap64 = buffer_size < n ? buffer_size : n;
  if (cap64 >= (1ULL << 31)) return fail(DP_ERR_INVALID_ATTR, "shuffle_plan: buffer must be < 2^31");
  const uint32_t cap = static_cast<uint32_t>(cap64);
  cudaStream_t st = as_stream(stream);
  const char* force_warp = std::getenv("DP_DEV_SHUFFLE_WARP");  // development A/B only
  if (use_device_plan(n, cap) && !(force_warp && *force_warp == '1')) {
    if (!scratch) return fail(DP_ERR_INVALID_ATTR, "shuffle_plan: scratch required (dp_k_shuffle_plan_scratch_bytes)");
    const Layout l = plan_layout(n, cap);
    uint8_t* base = static_cast<uint8_t*>(scratch);
    uint32_t* raws = reinterpret_cast<uint32_t*>(base + l.off_raws);
    uint32_t* slot_of = reinterpret_cast<uint32_t*>(base + l.off_slot);
    uint32_t* bucket = reinterpret_cast<uint32_t*>(base + l.off_bucket);
    uint32_t* start = reinterpret_cast<uint32_t*>(base + l.off_start);
    uint32_t* counts = reinterpret_cast<uint32_t*>(base + l.off_counts);
    uint32_t* cursor = reinterpret_cast<uint32_t*>(base + l.off_cursor);
    uint32_t* B = reinterpret_cast<uint32_t*>(base + l.off_B);
    uint64_t* tiles = reinterpret_cast<uint64_t*>(base + l.off_tiles);
    uint32_t* dstate = reinterpret_cast<uint32_t*>(base + l.off_dstate);
    uint64_t* meta = reinterpret_cast<uint64_t*>(base + l.off_meta);
    const uint64_t s0 = pcg_seeded_state(engine_seed);
    const uint32_t thr = (0u - cap) % cap;
    const int slot_grid = static_cast<int>(std::min<uint64_t>((cap + kPT - 1) / kPT, 148 * 8));
    init_slots<<<slot_grid, kPT, 0, st>>>(B, counts, cursor, cap);
    if (l.F > 0) {
      const uint64_t raw_threads = (l.R + kRawPer - 1) / kRawPer;
      p1_raws<<<static_cast<unsigned>((raw_threads + kPT - 1) / kPT), kPT, 0, st>>>(s0, l.R, raws);
      p2_count<<<static_cast<unsigned>(l.tiles), kPT, 0, st>>>(raws, l.R, thr, tiles);
      scan_u64<<<1, 1024, 0, st>>>(tiles, l.tiles, meta + 1);
      p2_scatter<<<static_cast<unsigned>(l.tiles), kPT, 0, st>>>(raws, l.R, thr, cap, l.F, tiles, slot_of, counts,
                                                                   meta);
      scan_small_u32<<<1, kScanT, 0, st>>>(counts, cap, start);
      const int kgrid = static_cast<int>(std::min<uint64_t>((l.F + kPT - 1) / kPT, 148 * 16));
      p3_bucket<<<kgrid, kPT, 0, st>>>(slot_of, l.F, start, cursor, bucket);
      p4_resolve<<<kgrid, kPT, 0, st>>>(slot_of, l.F, cap, start, bucket, B, in_map, out);
    } else {
      // no fill: the drain starts at raw 0 (raws computed on demand)
    }
    const size_t dbytes = (5 * static_cast<size_t>(cap) + 1) * sizeof(uint32_t);
    constexpr size_t kDrainSmem = 200 * 1024;
    if (dbytes <= kDrainSmem) {
      static int attr_dev = -1;
      int dev = 0;
      cudaGetDevice(&dev);
      if (attr_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(p5_drain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kDrainSmem));
        if (e != cudaSuccess) return cuda_status(e, "shuffle_plan: smem attribute");
        attr_dev = dev;
      }
      p5_drain<<<1, 1024, dbytes, st>>>(s0, raws, l.F > 0 ? l.R : 0, meta, l.F, cap, B, nullptr, in_map, out);
    } else {
      p5_drain<<<1, 1024, 0, st>>>(s0, raws, l.F > 0 ? l.R : 0, meta, l.F, cap, B, dstate, in_map, out);
    }
    return launch_status("shuffle_plan");
  }
  const size_t bytes = static_cast<size_t>(cap) * sizeof(uint32_t);
  uint32_t* gbuf = nullptr;
  size_t smem = 0;
  if (bytes > kMaxSmemBuffer) {
    if (!scratch) return fail(DP_ERR_INVALID_ATTR, "shuffle_plan: scratch required for this buffer size");
    gbuf = static_cast<uint32_t*>(scratch);
  } else {
    smem = bytes;
    static bool attr_set = false;
    if (!attr_set) {
      cudaError_t e = cudaFuncSetAttribute(shuffle_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kMaxSmemBuffer));
      if (e != cudaSuccess) return cuda_status(e, "shuffle_plan: smem attribute");
      attr_set = true;
    }
  }
  shuffle_plan_kernel<<<1, 32, smem, st>>>(n, cap, engine_seed, in_map, out, gbuf);
  return launch_status("shuffle_plan");
}
