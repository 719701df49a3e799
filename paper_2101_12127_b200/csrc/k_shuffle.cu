// k_shuffle.cu -- K2 shuffle_plan: the exact emission order of the
// reference's windowed-reservoir shuffle, computed on the device.
//
// Reference: ShuffleIterator::Next, /root/reference/proj/src/runtime.cpp:
// 721-747 (prime `cap` = min(n, buffer) inputs; each step draws
// idx = Pcg32::Bounded(size) (random.hpp:57-63), emits buffer[idx], refills
// it with the next input, or, once the input is exhausted, moves back() into
// idx and pops).
//
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
#include <cstdint>

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

}  // namespace
}  // namespace dpk

using namespace dpk;

extern "C" size_t dp_k_shuffle_plan_scratch_bytes(uint64_t n, uint64_t buffer_size) {
  uint64_t cap = buffer_size < n ? buffer_size : n;
  size_t bytes = static_cast<size_t>(cap) * sizeof(uint32_t);
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
  shuffle_plan_kernel<<<1, 32, smem, as_stream(stream)>>>(n, cap, engine_seed, in_map, out, gbuf);
  return launch_status("shuffle_plan");
}
