// runtime.cpp -- MakeIterator / GetNext: lowers a graph onto the sm_100a
// kernels and runs it as a stream-ordered device pipeline.
//
// Reference path being replaced: the NodeIterator tree of
// /root/reference/proj/src/runtime.cpp -- FromMemory (386-414), Shuffle
// (688-768), Shard (770-800), Repeat (1130-1187), Prefetch (1193-1294),
// MapAndBatch (1467-1721), Interleave (1044-1128), Filter (537-577), Batch
// (579-637), GetNext (147-165, 2196-2199).
//
// Lowering.  A graph is split into
//   [prefetch]* [repeat] BATCH-STAGE INDEX-CHAIN SOURCE
// BATCH-STAGE  map_and_batch(f) | batch(map(f)) | batch | padded_batch |
//              bucket_by_length | (none: unbatched) -- one fused
//              gather+UDF+store kernel per group of batches (K1/K3/K4/K5/K8)
// INDEX-CHAIN  shard / interleave / filter / shuffle / repeat (+ maps, which
//              commute with them and run in the batch stage; a filter sees
//              the affine maps beneath it) -- computed once per epoch as a
//              device array of source positions (the "epoch plan": K6
//              shard/interleave index, K5 compaction, K2 exact shuffle
//              order), each stage mapping the previous one.
// Batch i of the stream is rows [i*b, i*b + rows_i) of the epoch plan; the
// fused kernel gathers its elements through the plan.  Nothing is copied or
// assembled on the host.
//
// Prefetch.  A ring of device slots, each holding a launch group of G
// consecutive batches (a power of two near 3.2 GB of output -- 16 cfg2
// batches; padded kinds: the whole epoch).  GetNext keeps `depth` groups in
// flight on the iterator's stream and returns batch i as an Element of device
// Tensor views whose owner is the group's lease on the slot; the slot is rewritten only
// after every batch of its group was handed out and dropped, and after
// consumer-stream work queued before the drop (one release event per group).
// `depth` = the prefetch buffer_size, or for AUTOTUNE a value chosen from the
// measured device time per group against the host issue time.  The per-batch
// path makes no CUDA call.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <future>
#include <map>
#include <mutex>
#include <random>
#include <set>
#include <sstream>

#include "../roll.hpp"
#include "dpb200/datapipe.hpp"
#include "dpcuda.h"
#include "engine/device_util.hpp"
#include "engine/lowering.hpp"

namespace datapipe::b200 {

using namespace detail;

// ----------------------------------------------------- epoch plans, slots --
namespace {

// An epoch of the index chain: `count` positions into the element source,
// materialised in `order` (null = identity), with `tail` extra slots after
// `count` for the head of the next epoch (batches that span epochs).
struct EpochPlan {
  int64_t epoch = -1;
  int64_t count = 0;
  std::shared_ptr<void> order;  // int64 [count + tail]
  int64_t tail = 0;
  // padded batches
  std::vector<int32_t> lmax;         // per batch of this epoch
  std::vector<int64_t> boff;         // per batch, exclusive prefix (elements)
  std::shared_ptr<void> lmax_dev, boff_dev;
  // bucket_by_length: order = the bucket-grouped positions; per batch its
  // start in order, rows and the exclusive row prefix
  std::vector<int64_t> rows, roff;
  std::shared_ptr<void> bstart_dev, rows_dev, roff_dev;
  std::shared_ptr<void> row_src_dev, row_dst_dev, row_lm_dev;  // per emitted row (dp_k_bucket_rows)
  // token sources in pinned host memory: the plan's rows staged into device
  // memory in consumption order (dp_k_stage_rows), read by the batch kernels
  // with the identity order
  bool staged = false;
  std::shared_ptr<void> st_tokens, st_offsets, st_lengths;
  cudaEvent_t ready = nullptr;
  int64_t ready_gen = 0;  // bumped whenever `ready` is recorded again (a head appended)
};

struct Slot {
  int device = 0;
  std::shared_ptr<void> a, b, c, ha, hb, hc;  // device outputs (+ pinned host mirrors); c: labels
  size_t a_bytes = 0, b_bytes = 0, c_bytes = 0;
  cudaEvent_t ready = nullptr, release = nullptr, start = nullptr;
  bool release_recorded = false;
  // group bookkeeping
  int64_t first_batch = 0, num_batches = 0;
  std::atomic<int64_t> handed_out{0};  // written by the GetNext thread only
  int64_t units = 0;  // what GetNext hands out from this slot: batches, or elements when unbatched
  // The group's lease: every handed-out unit holds a copy, the iterator holds
  // one until the last unit goes out (see Lease); set at issue.
  std::shared_ptr<void> lease;
  bool busy = false;
  std::vector<int64_t> batch_off_a, batch_off_b, batch_rows, batch_cols;
  ~Slot() {
    if (ready) cudaEventDestroy(ready);
    if (release) cudaEventDestroy(release);
    if (start) cudaEventDestroy(start);
  }
};

}  // namespace

// -------------------------------------------------------------- the pipeline --
class DevicePipeline {
 public:
  DevicePipeline(const Lowered& L, uint64_t base_seed, const IteratorOptions& opt)
      : L_(L), base_seed_(base_seed), opt_(opt) {
    DeviceGuard g(opt_.device);
    CudaCheck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    CudaCheck(cudaStreamCreateWithFlags(&plan_stream_, cudaStreamNonBlocking), "stream");
    if (opt_.host_output) CudaCheck(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "stream");
    consumer_ = opt_.consumer_stream ? static_cast<cudaStream_t>(opt_.consumer_stream) : stream_;
    depth_ = L_.prefetch > 0 ? L_.prefetch : 2;
    autotune_ = L_.prefetch == kAutotune;
    PlanEpochSizes();          // also finds the max sequence length (padded slots)
    batch_bytes_ = BatchBytes();
    labels_ = L_.source && L_.source->labels && L_.kind != BatchKind::kPadded;
    if (labels_) batch_bytes_.first += sizeof(int64_t) * L_.batch;  // counted with the ids for group sizing
    // group size: >= 256 MB of output per launch (amortises launch latency and
    // the persistent kernel's ramp-up / drain), at most one epoch of batches
    // Per-launch fixed costs (kernel ramp-up, tail imbalance, launch gap)
    // are ~10% of a 150 MB batch; 16 cfg2 batches per launch put the batch
    // stage at the HBM roofline (tools/dev/groupsweep.py).  Pinned host slots
    // (host_output) are kept smaller.
    size_t target = opt_.max_launch_bytes ? opt_.max_launch_bytes
                                          : (opt_.host_output ? size_t(512) << 20 : size_t(3200) << 20);
    if (const char* v = std::getenv("DP_DEV_GROUP_MB")) target = size_t(std::atoll(v)) << 20;  // tuning sweeps
    target = std::min(target, opt_.slot_memory_budget / 2);
    group_ = std::max<int64_t>(1, static_cast<int64_t>(target / std::max<size_t>(batch_bytes_.first + batch_bytes_.second, 1)));
    // a power of two, so groups tile power-of-two epochs without a ragged group
    int64_t pow2 = 1;
    while (pow2 * 2 <= group_) pow2 *= 2;
    // (padded kinds launch a whole epoch when it fits: their epochs have an
    // arbitrary batch count, so a power of two would leave a ragged tail group)
    if (L_.kind != BatchKind::kPadded || group_ < batches_per_epoch_) group_ = pow2;
    if (opt_.launch_batches > 0) group_ = opt_.launch_batches;
    group_ = std::min(group_, std::max<int64_t>(1, batches_per_epoch_));
    // the prefetch depth must fit the slot budget (at least double buffering)
    const size_t group_bytes = (batch_bytes_.first + batch_bytes_.second) * group_;
    depth_ = std::max<int64_t>(2, std::min<int64_t>(depth_, static_cast<int64_t>(opt_.slot_memory_budget /
                                                                                 std::max<size_t>(group_bytes, 1))));
    max_depth_ = autotune_ ? std::clamp<int64_t>(static_cast<int64_t>(opt_.slot_memory_budget /
                                                                      std::max<size_t>(group_bytes, 1)),
                                                 2, 4)
                           : depth_;
    if (span_epochs_) group_ = std::min<int64_t>(group_, std::max<int64_t>(1, epoch_count_ / std::max<int64_t>(L_.batch, 1)));
    // a first launch group of another size (then groups of group_ again)
    head_ = opt_.first_launch_batches;
    if (head_ <= 0 || head_ == group_ || (span_epochs_ ? head_ > group_ : head_ >= batches_per_epoch_)) head_ = 0;
    if (group_ > 1) {  // epoch 0 was planned with a one-group tail: re-plan lazily
      for (auto& [e, p] : plans_)
        if (p.ready) cudaEventDestroy(p.ready);
      cudaStreamSynchronize(plan_stream_);
      plans_.clear();
      DrainOpTimings(true);  // the sizing plan is not part of the stream's work
      op_ns_total_.clear();
      op_produced_.clear();
    }
  }

  ~DevicePipeline() {
    DeviceGuard g(opt_.device);
    {
      std::lock_guard lk(shared_->mu);
      shared_->alive = false;
    }
    for (auto& sl : slots_) sl->lease.reset();  // groups not fully handed out
    try {
      JoinPendingPlan();
    } catch (...) {  // an error of a plan nobody asked for: dropped with the pipeline
    }
    PrintDebugTiming();
    cudaStreamSynchronize(stream_);
    for (auto& t : timed_) event_pool_.push_back(t);
    for (auto& t : event_pool_) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.end);
    }
    cudaStreamSynchronize(plan_stream_);
    if (copy_stream_) cudaStreamSynchronize(copy_stream_);
    for (auto& [e, p] : plans_)
      if (p.ready) cudaEventDestroy(p.ready);
    plans_.clear();  // stream-ordered frees: before the streams go away
    cudaStreamSynchronize(plan_stream_);
    if (retire_ev_) cudaEventDestroy(retire_ev_);
    for (auto& t : op_timed_) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.end);
    }
    cudaStreamDestroy(stream_);
    cudaStreamDestroy(plan_stream_);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (rb_host_) cudaFreeHost(rb_host_);
  }

  // The per-batch fast path makes no CUDA call and takes no lock (the
  // group's lease is copied, see Lease): issuing, slot reuse, autotuning and the consumer-stream wait
  // happen at group boundaries, or when a released slot may let the next
  // group go out (Shared::slots_freed).
  std::optional<Element> Next() {
    if (done_) return std::nullopt;
    const int64_t u = next_batch_;  // the unit GetNext hands out: a batch, or an element when unbatched
    const int64_t total = L_.unbatched ? total_units_ : total_batches_;
    if (total >= 0 && u >= total) {
      done_ = true;
      return std::nullopt;
    }
    int64_t row = 0;
    const int64_t i = L_.unbatched ? BatchOfElement(u, row) : u;  // internal batch
    const int64_t grp = GroupOf(i);
    using Clock = std::chrono::steady_clock;
    const auto t0 = debug_timing_ ? Clock::now() : Clock::time_point{};
    const bool boundary = grp != cur_group_;
    const uint64_t freed = shared_->slots_freed.load(std::memory_order_acquire);
    if (boundary || freed != seen_freed_) {
      seen_freed_ = freed;
      DeviceGuard g(opt_.device);
      while (issued_groups_ <= grp) IssueGroup(issued_groups_);
      // keep `depth` groups in flight
      while (issued_groups_ < grp + depth_ && (total_groups_ < 0 || issued_groups_ < total_groups_)) {
        if (!TryIssueGroup(issued_groups_, /*may_grow=*/false)) break;
      }
      if (boundary) {
        cur_slot_ = group_slot_.at(grp);
        cur_group_ = grp;
        {
          // after a Seek into the middle of a group, the skipped units count as handed out
          std::lock_guard lk(shared_->mu);
          const int64_t before = UnitsBefore(*cur_slot_, i, row);
          if (cur_slot_->handed_out.load() < before) cur_slot_->handed_out.store(before);
        }
        // one wait per group: the slot's ready event covers all its batches
        if (consumer_ != stream_ && !opt_.host_output)
          CudaCheck(cudaStreamWaitEvent(consumer_, cur_slot_->ready, 0), "wait");
        // unbatched: element values are read on the host (the reference
        // returns int64 values, not device tensors)
        if (L_.unbatched) CudaCheck(cudaEventSynchronize(cur_slot_->ready), "unbatched values");
        MaybeAutotune();
      }
    }
    const auto t1 = debug_timing_ ? Clock::now() : Clock::time_point{};
    next_batch_++;
    produced_++;
    if (!debug_timing_) return L_.unbatched ? MakeUnitElement(cur_slot_, i, row) : MakeElement(cur_slot_, i);
    const auto t2 = Clock::now();
    auto e = L_.unbatched ? MakeUnitElement(cur_slot_, i, row) : MakeElement(cur_slot_, i);
    const auto t3 = Clock::now();
    dbg_[0] += std::chrono::duration<double>(t1 - t0).count();
    dbg_[1] += std::chrono::duration<double>(t2 - t1).count();
    dbg_[2] += std::chrono::duration<double>(t3 - t2).count();
    return e;
  }

  double dbg_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t plans_built_ = 0;
  void PrintDebugTiming() const {
    if (!std::getenv("DP_DEBUG_TIMING") || produced_ == 0) return;
    std::fprintf(stderr,
                 "[dp timing] per GetNext (us): issue %.1f autotune %.1f element %.1f | per group: find %.1f plan %.1f "
                 "launch %.1f events %.1f (%lld groups) | prefetched plan build %.1f (%lld plans)\n",
                 1e6 * dbg_[0] / produced_, 1e6 * dbg_[1] / produced_, 1e6 * dbg_[2] / produced_,
                 1e6 * dbg_[3] / std::max<int64_t>(issued_count_, 1), 1e6 * dbg_[4] / std::max<int64_t>(issued_count_, 1),
                 1e6 * dbg_[5] / std::max<int64_t>(issued_count_, 1), 1e6 * dbg_[6] / std::max<int64_t>(issued_count_, 1),
                 static_cast<long long>(issued_count_), 1e6 * dbg_[7] / std::max<int64_t>(plans_built_, 1),
                 static_cast<long long>(plans_built_));
  }

  int64_t delivered() const { return produced_; }
  int64_t depth() const { return depth_; }
  int64_t launches() const { return launches_; }
  int64_t batches_launched() const { return batches_launched_; }
  void* stream() const { return stream_; }
  int64_t batch_time_ns() const { return batch_ns_total_; }
  int64_t group_size() const { return group_; }
  std::string Describe() const {
    std::ostringstream os;
    const char* kinds[] = {"K1 gather_affine_batch", "K3 crop_flip_normalize_batch", "K4 resize_normalize_batch",
                           "K5 padded_batches",     "K1 gather_affine_batch",       "K9 image_chain_batch",
                           "K9 gather_copy_batch"};
    std::string kernel = kinds[static_cast<int>(L_.kind)];
    int k10 = 0;  // resize chains K10 takes (dp_image_chain_kernel)
    if (L_.kind == BatchKind::kChain && dp_image_chain_kernel(&L_.img_chain, &k10) == DP_OK && k10 == 10)
      kernel = "K10 image_chain_roll (via K9 image_chain_batch)";
    if (L_.kind == BatchKind::kResize) {
      dp_image_chain c{};  // resize + normalize as a chain: K10 when its column map is periodic
      c.in_h = static_cast<int>(L_.source->h);
      c.in_w = static_cast<int>(L_.source->w);
      c.resize = 1;
      c.rs_h = static_cast<int>(L_.resize.out_h);
      c.rs_w = static_cast<int>(L_.resize.out_w);
      c.num_post_ops = 1;
      for (int ch = 0; ch < 3; ++ch) {
        c.op_a[0][ch] = L_.norm.mean[ch];
        c.op_b[0][ch] = L_.norm.stdv[ch];
      }
      c.out_f32 = 1;
      if (dpk::roll_chain_eligible(&c, c.rs_h, c.rs_w, /*allow_general=*/false))  // as resize_normalize_batch
        kernel = "K10 image_chain_roll (via K4 resize_normalize_batch)";
    }
    os << "batch stage: " << kernel << " (batch " << L_.batch << (L_.drop ? ", drop" : "")
       << ", " << group_ << " batch(es) per launch, depth " << depth_ << (autotune_ ? " autotuned" : "") << ")\n";
    os << "index chain (bottom-up):";
    for (const auto& op : L_.chain) {
      const char* names[] = {"shard", "shuffle", "filter", "interleave", "repeat"};
      os << " " << names[static_cast<int>(op.kind)];
    }
    os << "\nsource positions: " << L_.source_count << ", epoch: " << epoch_count_ << " elements, "
       << batches_per_epoch_ << " batches" << (span_epochs_ ? " (batches span epochs)" : "") << "\n";
    return os.str();
  }

 private:
  // ---- sizes ----
  std::pair<size_t, size_t> BatchBytes() const {
    const int64_t b = L_.batch;
    switch (L_.kind) {
      case BatchKind::kAffine:
      case BatchKind::kIdentityInt: return {sizeof(int64_t) * b, 0};
      case BatchKind::kCrop: return {sizeof(int64_t) * b, sizeof(float) * b * L_.crop.out_h * L_.crop.out_w * 3};
      case BatchKind::kResize: return {sizeof(int64_t) * b, sizeof(float) * b * L_.resize.out_h * L_.resize.out_w * 3};
      case BatchKind::kChain:
      case BatchKind::kCopy:
        return {sizeof(int64_t) * b, (L_.img_f32 ? sizeof(float) : 1) * b * L_.img_h * L_.img_w * 3};
      case BatchKind::kPadded:
        if (L_.ragged) return {sizeof(int32_t) * b * std::max<int64_t>(max_len_, 1), sizeof(int64_t) * (b + 1)};
        return {sizeof(int32_t) * b * std::max<int64_t>(max_len_, 1), sizeof(int32_t) * b};
    }
    return {0, 0};
  }

  // Epoch length is the same every epoch (shuffle keeps the count; filter
  // predicates are deterministic); compute it once (may run the filter).
  void PlanEpochSizes() {
    span_epochs_ = false;
    int64_t inner_repeat = 1;
    for (const auto& op : L_.chain)
      if (op.kind == IndexOp::Kind::kRepeat) {
        span_epochs_ = true;
        inner_repeat = op.a;
      }
    if (L_.kind == BatchKind::kPadded) {
      // max sequence length over the source, for slot sizing
      std::vector<int32_t> lens(L_.source->count);
      CudaCheck(cudaMemcpy(lens.data(), L_.source->lengths.get(), sizeof(int32_t) * lens.size(), cudaMemcpyDefault),
                "lengths");
      max_len_ = lens.empty() ? 0 : *std::max_element(lens.begin(), lens.end());
      for (const auto& op : L_.chain)
        if (op.kind == IndexOp::Kind::kFilter && op.pred.on == DevicePredicate::On::kLength)
          max_len_ = std::min<int64_t>(max_len_, std::max<int64_t>(op.pred.MaxLen(), 0));
    }
    EpochPlan& p0 = Plan(0);
    epoch_count_ = p0.count;
    // (bucket_by_length: the same multiset of lengths every epoch, so the
    // same number of batches; only their order changes with the shuffle)
    const int64_t per = L_.bucketed ? static_cast<int64_t>(p0.rows.size())
                        : L_.drop   ? epoch_count_ / L_.batch
                                    : (epoch_count_ + L_.batch - 1) / L_.batch;
    if (span_epochs_) {
      if (inner_repeat == kInfiniteRepeat) {
        total_batches_ = epoch_count_ == 0 ? 0 : -1;
      } else {
        const int64_t total = epoch_count_ * inner_repeat;
        total_batches_ = L_.drop ? total / L_.batch : (total + L_.batch - 1) / L_.batch;
      }
      batches_per_epoch_ = std::max<int64_t>(1, epoch_count_ / L_.batch);
    } else {
      batches_per_epoch_ = per;
      if (L_.outer_repeat == kInfiniteRepeat) total_batches_ = per == 0 ? 0 : -1;
      else total_batches_ = per * L_.outer_repeat;
    }
    if (!span_epochs_) {
      const int64_t gpe = 0;  // groups per epoch fixed after group_ known (see GroupInfo)
      (void)gpe;
    }
    total_groups_ = -1;  // computed lazily via GroupRange
    if (L_.unbatched) {
      if (span_epochs_) {
        const int64_t rows = TotalRows();
        total_units_ = rows == INT64_MAX ? (epoch_count_ == 0 ? 0 : -1) : rows;
      } else {
        total_units_ = L_.outer_repeat == kInfiniteRepeat ? (epoch_count_ == 0 ? 0 : -1)
                                                          : epoch_count_ * L_.outer_repeat;
      }
    }
  }

  // Batches of group g: [first, first + n).  Groups never straddle the
  // boundary of a non-spanning epoch, so every group is one contiguous range
  // of one epoch plan (plus the next epoch's head when spanning).
  // Launch group holding batch i (inverse of GroupRange).
  // unbatched: element u -> internal batch and row (batches never straddle a
  // non-spanning epoch)
  int64_t BatchOfElement(int64_t u, int64_t& row) const {
    if (span_epochs_ || epoch_count_ == 0) {
      row = u % L_.batch;
      return u / L_.batch;
    }
    const int64_t e = u / epoch_count_, off = u - e * epoch_count_;
    row = off % L_.batch;
    return e * batches_per_epoch_ + off / L_.batch;
  }
  // units of `s` handed out before (batch i, row)
  int64_t UnitsBefore(const Slot& s, int64_t i, int64_t row) const {
    if (!L_.unbatched) return i - s.first_batch;
    int64_t n = row;
    for (int64_t b = s.first_batch; b < i; ++b) n += s.batch_rows[b - s.first_batch];
    return n;
  }

  // Groups tile the batch stream (spanning epochs) or each epoch from its
  // start; with a head (IteratorOptions::first_launch_batches) the first
  // group of the stream holds head_ batches and the tiling restarts after it.
  int64_t SegGroups(int64_t batches, int64_t head) const {
    if (batches <= 0) return 0;
    return head ? 1 + (batches - head + group_ - 1) / group_ : (batches + group_ - 1) / group_;
  }
  int64_t GroupInSeg(int64_t k, int64_t head) const {
    return head ? (k < head ? 0 : 1 + (k - head) / group_) : k / group_;
  }
  std::pair<int64_t, int64_t> SegRange(int64_t grp, int64_t head) const {  // (first, n) within the segment
    if (!head) return {grp * group_, group_};
    if (grp == 0) return {0, head};
    return {head + (grp - 1) * group_, group_};
  }

  int64_t GroupOf(int64_t i) const {
    if (span_epochs_) return GroupInSeg(i, head_);
    const int64_t bpe = std::max<int64_t>(batches_per_epoch_, 1);
    const int64_t e = i / bpe, k = i % bpe;
    if (e == 0) return GroupInSeg(k, head_);
    return SegGroups(bpe, head_) + (e - 1) * SegGroups(bpe, 0) + k / group_;
  }

 public:
  // O(1) repositioning of a fresh iterator at batch n (checkpoint restore):
  // the skipped batches are never computed.
  void Seek(int64_t n) {
    if (produced_ != 0 || issued_groups_ != 0)
      throw PipelineError(ErrorCode::kInternal, "Seek needs a fresh iterator");
    const int64_t total = L_.unbatched ? total_units_ : total_batches_;
    if (n < 0 || (total >= 0 && n > total))
      throw PipelineError(ErrorCode::kCorruptBlob, "checkpoint claims " + std::to_string(n) +
                                                       " delivered elements but the pipeline has " +
                                                       std::to_string(total));
    next_batch_ = n;
    produced_ = n;
    int64_t row = 0;
    issued_groups_ = GroupOf(L_.unbatched ? BatchOfElement(n, row) : n);
  }

 private:
  std::pair<int64_t, int64_t> GroupRange(int64_t g) const {
    if (span_epochs_) {
      auto [first, n] = SegRange(g, head_);
      if (total_batches_ >= 0) n = std::min(n, total_batches_ - first);
      return {first, std::max<int64_t>(n, 0)};
    }
    const int64_t bpe = batches_per_epoch_;
    const int64_t gpe0 = SegGroups(bpe, head_), gpe = SegGroups(bpe, 0);
    if (gpe == 0) return {0, 0};
    int64_t e = 0, k = g;
    if (g >= gpe0) {
      e = 1 + (g - gpe0) / gpe;
      k = (g - gpe0) % gpe;
    }
    auto [off, n] = SegRange(k, e == 0 ? head_ : 0);
    const int64_t first = e * bpe + off;
    n = std::min(n, bpe - off);
    if (total_batches_ >= 0 && first >= total_batches_) n = 0;
    return {first, n};
  }

  // salt for the shuffles of epoch e: base seed, re-salted per repeat epoch
  // (RepeatIterator::MakeChild runtime.cpp:1175-1177; fused shuffle :751)
  uint64_t EpochSalt(int64_t e) const {
    bool under_repeat = L_.outer_repeat != 1 || span_epochs_;
    return under_repeat ? MixSeeds(base_seed_, static_cast<uint64_t>(e)) : base_seed_;
  }

  void JoinPendingPlan() {
    if (pending_plan_.valid()) pending_plan_.get();  // rethrows the helper's error
  }

  // Plan read-backs (counts, batch shapes): a kernel on stream s writes the
  // bytes into mapped pinned host memory and s is synchronised -- no copy
  // engine involved, so they never queue behind a launch group's host_output
  // D2H copy (which held every token epoch's next plan for the length of a
  // 200 MB copy).  rows x width bytes at src_pitch (contiguous by default).
  void ReadBack(void* dst, const void* src, size_t width, cudaStream_t s, size_t rows = 1, size_t src_pitch = 0) {
    const size_t bytes = width * rows;
    if (!bytes) return;
    static const bool copy_engine = std::getenv("DP_DEV_RB_COPY") != nullptr;  // development A/B switch
    if (copy_engine) {
      CudaCheck(cudaMemcpy2DAsync(dst, width, src, src_pitch ? src_pitch : width, width, rows, cudaMemcpyDeviceToHost,
                                  s),
                "read-back");
      CudaCheck(cudaStreamSynchronize(s), "read-back");
      return;
    }
    std::lock_guard lk(rb_mu_);
    if (bytes > rb_cap_) {
      if (rb_host_) {
        CudaCheck(cudaStreamSynchronize(s), "read-back");
        cudaFreeHost(rb_host_);
        rb_host_ = nullptr;
      }
      rb_cap_ = std::max<size_t>(bytes, size_t(1) << 20);
      CudaCheck(cudaHostAlloc(&rb_host_, rb_cap_, cudaHostAllocMapped | cudaHostAllocPortable), "read-back buffer");
    }
    KCheck(dp_k_copy_strided(src, src_pitch ? src_pitch : width, width, rows, rb_host_, s), "read-back");
    CudaCheck(cudaStreamSynchronize(s), "read-back");
    std::memcpy(dst, rb_host_, bytes);
  }

  // Builds epoch e's plan on a helper thread (plan stream); Plan() joins it.
  void PrefetchPlan(int64_t e) {
    JoinPendingPlan();
    RetirePlansBefore(e);
    if (plans_.count(e)) return;
    pending_plan_ = std::async(std::launch::async, [this, e] {
      DeviceGuard g(opt_.device);
      EpochPlan p;
      p.epoch = e;
      const auto t0 = std::chrono::steady_clock::now();
      BuildPlan(p, e);
      const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::lock_guard lk(plans_mu_);
      dbg_[7] += dt;  // helper-thread plan build time (DP_DEBUG_TIMING)
      plans_built_++;
      plans_.emplace(e, std::move(p));
    });
  }

  // Retire the plans of epochs before `e - 1` (called whenever plan e is
  // asked for or prefetched; groups are issued in epoch order, so nothing
  // issued later reads them).  Their buffers are freed on the plan stream,
  // ordered after every batch kernel queued so far on the batch stream (the
  // last readers) -- no host synchronisation.
  void RetirePlansBefore(int64_t e) {
    for (auto jt = plans_.begin(); jt != plans_.end() && jt->first < e - 1;) {
      if (!retire_ev_) CudaCheck(cudaEventCreateWithFlags(&retire_ev_, cudaEventDisableTiming), "event");
      CudaCheck(cudaEventRecord(retire_ev_, stream_), "event");
      CudaCheck(cudaStreamWaitEvent(plan_stream_, retire_ev_, 0), "wait");
      if (jt->second.ready) cudaEventDestroy(jt->second.ready);
      for (auto at = appended_.begin(); at != appended_.end();)
        at = *at / 1000003 == jt->first ? appended_.erase(at) : std::next(at);
      jt = plans_.erase(jt);
    }
  }

 public:
  PipelineIterator::Stats stats() const {
    PipelineIterator::Stats st;
    st.live_plans = static_cast<int64_t>(plans_.size());
    st.slots = static_cast<int64_t>(slots_.size());
    st.slot_bytes = static_cast<int64_t>(slot_bytes_total_);
    st.prefetch_depth = depth_;
    st.group_batches = group_;
    const TunerState t = Tuner();
    st.max_depth = t.max_depth;
    st.producer_groups_per_s = t.producer_groups_per_s;
    st.consumer_groups_per_s = t.consumer_groups_per_s;
    st.p_empty = t.p_empty;
    return st;
  }

 private:
  // Folds the completed index-op timings into op_ns_total_ (wait: all).
  void DrainOpTimings(bool wait) {
    std::lock_guard lk(metrics_mu_);
    size_t k = 0;
    for (; k < op_timed_.size(); ++k) {
      auto& t = op_timed_[k];
      if (wait) cudaEventSynchronize(t.end);
      else if (cudaEventQuery(t.end) != cudaSuccess) {
        cudaGetLastError();
        break;
      }
      float ms = 0;
      if (cudaEventElapsedTime(&ms, t.start, t.end) == cudaSuccess) {
        op_ns_total_.resize(L_.chain.size(), 0);
        op_ns_total_[t.op] += static_cast<int64_t>(static_cast<double>(ms) * 1e6);
      }
      cudaGetLastError();
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.end);
    }
    op_timed_.erase(op_timed_.begin(), op_timed_.begin() + static_cast<std::ptrdiff_t>(k));
  }

  EpochPlan& Plan(int64_t e) {
    JoinPendingPlan();
    DrainOpTimings(false);
    RetirePlansBefore(e);
    auto it = plans_.find(e);
    if (it != plans_.end()) return it->second;
    EpochPlan& p = plans_[e];
    p.epoch = e;
    BuildPlan(p, e);
    return p;
  }

  void BuildPlan(EpochPlan& p, int64_t e) {
    cudaStream_t s = plan_stream_;
    const uint64_t salt = EpochSalt(e);
    // state: identity over [0, count) or an array
    int64_t count = L_.source_count;
    std::shared_ptr<void> cur;  // int64 order (null = identity)
    const int64_t tail = std::max<int64_t>(L_.batch * group_, 1);
    // every plan buffer is stream-ordered on the plan stream (see Plan() for
    // how retirement orders the free after the batch kernels' last use)
    auto dalloc = [&](size_t bytes) { return DeviceAllocAsync(bytes, opt_.device, plan_stream_, plan_stream_); };
    auto alloc = [&](int64_t n) { return dalloc(sizeof(int64_t) * (n + tail)); };
    for (size_t oi = 0; oi < L_.chain.size(); ++oi) {
      const auto& op = L_.chain[oi];
      // self time of this index op (its plan kernels; Metrics())
      cudaEvent_t t0 = nullptr, t1 = nullptr;
      CudaCheck(cudaEventCreate(&t0), "event");
      CudaCheck(cudaEventCreate(&t1), "event");
      CudaCheck(cudaEventRecord(t0, s), "event");
      switch (op.kind) {
        case IndexOp::Kind::kShard: {
          const int64_t m = count > op.b ? (count - op.b + op.a - 1) / op.a : 0;
          auto out = alloc(m);
          KCheck(dp_k_shard_index(count, op.a, op.b, P<int64_t>(cur), P<int64_t>(out), s), "shard");
          launches_++;
          cur = out;
          count = m;
          break;
        }
        case IndexOp::Kind::kInterleave: {
          // inputs are the current positions = source ordinals; they are an
          // arithmetic sequence here (identity or shards of it)
          int64_t first = 0, stride = 1;
          ArithmeticOf(count, first, stride);
          if (L_.records_local) first = 0, stride = 1;  // block residency: input j of the shard = held file j
          if (op.b == 0 && L_.records && L_.records->kind == SourceData::Kind::kRecords) {
            BuildVarInterleave(first, stride, op.a, cur, count);
            break;
          }
          const int64_t m = count * op.b;
          auto out = alloc(m);
          KCheck(dp_k_interleave_index(first, stride, count, op.a, op.b, P<int64_t>(out), s), "interleave");
          launches_++;
          cur = out;
          count = m;
          break;
        }
        case IndexOp::Kind::kFilter: {
          auto out = alloc(count);
          auto nk = dalloc(sizeof(int64_t));
          auto scratch = dalloc(dp_k_filter_scratch_bytes(count));
          std::vector<dp_predicate_term> terms;
          for (const auto& t : op.pred.terms) terms.push_back({static_cast<int>(t.op), t.a, t.b});
          const bool on_len = op.pred.on == DevicePredicate::On::kLength;
          // value predicates: from_memory values, else the position (range /
          // interleaved record indices)
          const int64_t* vals =
              !on_len && L_.source && L_.source->kind == SourceData::Kind::kInt64 ? P<int64_t>(L_.source->values)
                                                                                  : nullptr;
          KCheck(dp_k_filter(on_len ? P<int32_t>(L_.source->lengths) : nullptr, vals, count, op.mul, op.add,
                             terms.data(), static_cast<int>(terms.size()), P<int64_t>(cur), P<int64_t>(out),
                             P<int64_t>(nk), scratch.get(), s),
                 "filter");
          launches_ += 3;
          int64_t m = 0;
          ReadBack(&m, nk.get(), sizeof(int64_t), s);
          cur = out;
          count = m;
          break;
        }
        case IndexOp::Kind::kShuffle: {
          auto out = alloc(count);
          const uint64_t seed = ShuffleEngineSeed(salt, op.seed);
          size_t sb = dp_k_shuffle_plan_scratch_bytes(static_cast<uint64_t>(count), static_cast<uint64_t>(op.a));
          std::shared_ptr<void> scratch = sb ? dalloc(sb) : nullptr;
          KCheck(dp_k_shuffle_plan(count, op.a, seed, P<int64_t>(cur), P<int64_t>(out), scratch.get(), s), "shuffle");
          launches_++;
          cur = out;
          count = count;
          break;
        }
        case IndexOp::Kind::kRepeat:
          break;
      }
      CudaCheck(cudaEventRecord(t1, s), "event");
      std::lock_guard lk(metrics_mu_);
      op_timed_.push_back({static_cast<int>(oi), t0, t1});
      if (op_produced_.size() < L_.chain.size()) op_produced_.resize(L_.chain.size(), 0);
      op_produced_[oi] += count;
    }
    if (!cur && (span_epochs_ || L_.kind == BatchKind::kPadded)) {
      // materialise the identity so spanning batches can append the next head
      cur = alloc(count);
      KCheck(dp_k_shard_index(count, 1, 0, nullptr, P<int64_t>(cur), s), "identity");
      launches_++;
    }
    p.count = count;
    p.order = cur;
    p.tail = cur ? tail : 0;
    if (L_.bucketed) {
      BuildBucketPlan(p, cur, count);
    } else if (L_.ragged) {
      BuildRaggedPlan(p, cur, count);
    } else if (L_.kind == BatchKind::kPadded) {
      const int64_t nb = (count + L_.batch - 1) / L_.batch;
      p.lmax.assign(nb, 0);
      p.boff.assign(nb + 1, 0);
      if (nb) {
        auto lm = dalloc(sizeof(int32_t) * nb);
        KCheck(dp_k_batch_max_len(P<int32_t>(L_.source->lengths), P<int64_t>(cur), count, L_.batch, P<int32_t>(lm), s),
               "batch_max_len");
        launches_++;
        ReadBack(p.lmax.data(), lm.get(), sizeof(int32_t) * nb, s);
        for (int64_t j = 0; j < nb; ++j) {
          const int64_t rows = std::min<int64_t>(L_.batch, count - j * L_.batch);
          p.boff[j + 1] = p.boff[j] + rows * p.lmax[j];
        }
        p.lmax_dev = lm;
        p.boff_dev = dalloc(sizeof(int64_t) * (nb + 1));
        CudaCheck(cudaMemcpyAsync(p.boff_dev.get(), p.boff.data(), sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, s),
                  "boff");
      }
    }
    if (L_.kind == BatchKind::kPadded && L_.source->residency == Residency::kHost) StageRows(p);
    CudaCheck(cudaEventCreateWithFlags(&p.ready, cudaEventDisableTiming), "event");
    CudaCheck(cudaEventRecord(p.ready, s), "event");
    p.ready_gen = 1;
  }

  // Pinned-host token source (end-to-end runs): one PCIe pass per epoch
  // moves exactly the rows the plan consumes, in consumption order, into a
  // packed device buffer (warp-per-row kernel with 8 loads in flight per
  // lane); the batch kernels then stream HBM.  Rows: the plan order
  // (padded / ragged) or the bucket plan's emitted rows (then re-indexed
  // 0..n-1).
  void StageRows(EpochPlan& p) {
    cudaStream_t s = plan_stream_;
    auto dalloc = [&](size_t bytes) { return DeviceAllocAsync(bytes, opt_.device, plan_stream_, plan_stream_); };
    const int64_t* ord = L_.bucketed ? P<int64_t>(p.row_src_dev) : P<int64_t>(p.order);
    const int64_t n = L_.bucketed ? (p.roff.empty() ? 0 : p.roff.back()) : p.count;
    std::shared_ptr<void> prefix;
    if (L_.ragged) {
      prefix = p.roff_dev;  // the ragged plan's length prefix over the same order
    } else {
      prefix = dalloc(sizeof(int64_t) * (n + 1));
      auto scratch = dalloc(dp_k_len_prefix_scratch_bytes(n));
      KCheck(dp_k_len_prefix(P<int32_t>(L_.source->lengths), ord, n, P<int64_t>(prefix), scratch.get(), s),
             "stage prefix");
      launches_ += 3;
    }
    int64_t total = 0;
    ReadBack(&total, P<int64_t>(prefix) + n, sizeof(int64_t), s);
    p.st_tokens = dalloc(sizeof(int32_t) * std::max<int64_t>(total, 1));
    p.st_lengths = dalloc(sizeof(int32_t) * std::max<int64_t>(n, 1));
    p.st_offsets = prefix;
    KCheck(dp_k_stage_rows(P<int32_t>(L_.source->tokens), P<int64_t>(L_.source->offsets),
                           P<int32_t>(L_.source->lengths), ord, n, P<int64_t>(prefix), P<int32_t>(p.st_tokens),
                           P<int32_t>(p.st_lengths), s),
           "stage rows");
    launches_++;
    if (L_.bucketed && n > 0) {  // emitted row k is staged row k
      KCheck(dp_k_range_affine_batch(0, n, 1, 0, P<int64_t>(p.row_src_dev), s), "stage iota");
      launches_++;
    }
    p.staged = true;
  }

  // Interleave over record files of unequal sizes: the host schedules the
  // inputs over the cycle slots (O(inputs log cycle), dp_interleave_schedule),
  // the device writes every record's position (K6 interleave_var).
  void BuildVarInterleave(int64_t first, int64_t stride, int64_t cycle, std::shared_ptr<void>& cur, int64_t& count) {
    cudaStream_t s = plan_stream_;
    const auto& fr = L_.records->file_records;
    std::vector<int64_t> file_start(fr.size() + 1, 0);
    for (size_t f = 0; f < fr.size(); ++f) file_start[f + 1] = file_start[f] + fr[f];
    const int64_t m = count;
    std::vector<int64_t> host(5 * std::max<int64_t>(m, 1) + cycle, 0);  // slot | start | len | first_record | end
    int64_t* slot = host.data();
    int64_t* start = slot + m;
    int64_t* len = start + m;
    int64_t* rec = len + m;
    int64_t* end = rec + m;
    int64_t total = 0;
    for (int64_t i = 0; i < m; ++i) {
      const int64_t x = first + i * stride;
      if (x < 0 || x >= static_cast<int64_t>(fr.size()))
        throw PipelineError(ErrorCode::kMalformedInput, "interleave: input " + std::to_string(x) + " has no record file (" +
                                                            std::to_string(fr.size()) + " files)");
      len[i] = fr[x];
      rec[i] = file_start[x];
      total += len[i];
    }
    KCheck(dp_interleave_schedule(m, len, cycle, slot, start, end), "interleave schedule");
    auto dalloc = [&](size_t bytes) { return DeviceAllocAsync(bytes, opt_.device, plan_stream_, plan_stream_); };
    auto meta = dalloc(sizeof(int64_t) * host.size());
    CudaCheck(cudaMemcpyAsync(meta.get(), host.data(), sizeof(int64_t) * host.size(), cudaMemcpyHostToDevice, s),
              "interleave schedule");
    const int64_t tail = std::max<int64_t>(L_.batch * group_, 1);
    auto out = dalloc(sizeof(int64_t) * (total + tail));
    const int64_t* d = P<int64_t>(meta);
    KCheck(dp_k_interleave_var(m, d, d + m, d + 2 * m, d + 3 * m, d + 4 * m, cycle, P<int64_t>(out), s),
           "interleave_var");
    launches_++;
    CudaCheck(cudaStreamSynchronize(s), "interleave schedule");  // `host` is read by the copy
    cur = out;
    count = total;
  }

  // Ragged batches: the epoch's length prefix over its kept rows; the batch
  // boundaries' prefixes are read back for the elements' shapes.
  void BuildRaggedPlan(EpochPlan& p, const std::shared_ptr<void>& cur, int64_t count) {
    cudaStream_t s = plan_stream_;
    auto dalloc = [&](size_t bytes) { return DeviceAllocAsync(bytes, opt_.device, plan_stream_, plan_stream_); };
    auto prefix = dalloc(sizeof(int64_t) * (count + 1));
    auto scratch = dalloc(dp_k_len_prefix_scratch_bytes(count));
    KCheck(dp_k_len_prefix(P<int32_t>(L_.source->lengths), P<int64_t>(cur), count, P<int64_t>(prefix), scratch.get(),
                           s),
           "len_prefix");
    launches_ += 3;
    const int64_t B = L_.batch, nb = L_.drop ? count / B : (count + B - 1) / B;
    p.boff.assign(nb + 1, 0);
    if (nb) {  // prefix[j * B] for j < nb, then the end of the last batch
      ReadBack(p.boff.data(), prefix.get(), sizeof(int64_t), s, nb, sizeof(int64_t) * B);  // prefix[j * B]
      ReadBack(&p.boff[nb], P<int64_t>(prefix) + std::min(nb * B, count), sizeof(int64_t), s);
    }
    p.lmax.assign(nb, 0);
    for (int64_t j = 0; j < nb; ++j) p.lmax[j] = static_cast<int32_t>(p.boff[j + 1] - p.boff[j]);  // tokens
    p.roff_dev = prefix;
  }

  // K8: the bucket plan of one epoch (k_bucket.cu) -- batches, their rows
  // and lengths read back for the elements' shapes, prefixes uploaded.
  void BuildBucketPlan(EpochPlan& p, const std::shared_ptr<void>& cur, int64_t count) {
    cudaStream_t s = plan_stream_;
    auto dalloc = [&](size_t bytes) { return DeviceAllocAsync(bytes, opt_.device, plan_stream_, plan_stream_); };
    const int K = static_cast<int>(L_.bucket_sizes.size());
    const int64_t maxb = count + K;
    auto perm = dalloc(sizeof(int64_t) * std::max<int64_t>(count, 1));
    auto bstart = dalloc(sizeof(int64_t) * maxb), brows = dalloc(sizeof(int32_t) * maxb);
    auto blmax = dalloc(sizeof(int32_t) * maxb), nbd = dalloc(sizeof(int64_t));
    auto scratch = dalloc(dp_k_bucket_scratch_bytes(count, K));
    KCheck(dp_k_bucket_plan(P<int32_t>(L_.source->lengths), P<int64_t>(cur), count, L_.bucket_bounds.data(),
                            static_cast<int>(L_.bucket_bounds.size()), L_.bucket_sizes.data(), L_.drop ? 1 : 0,
                            P<int64_t>(perm), P<int64_t>(bstart), P<int32_t>(brows), P<int32_t>(blmax),
                            P<int64_t>(nbd), scratch.get(), s),
           "bucket_plan");
    launches_ += 8;
    int64_t nb = 0;
    ReadBack(&nb, nbd.get(), sizeof(int64_t), s);
    std::vector<int32_t> rows32(nb);
    p.lmax.assign(nb, 0);
    if (nb) {
      ReadBack(rows32.data(), brows.get(), sizeof(int32_t) * nb, s);
      ReadBack(p.lmax.data(), blmax.get(), sizeof(int32_t) * nb, s);
    }
    p.rows.assign(rows32.begin(), rows32.end());
    p.boff.assign(nb + 1, 0);
    std::vector<int64_t> roff(nb + 1, 0);
    for (int64_t j = 0; j < nb; ++j) {
      p.boff[j + 1] = p.boff[j] + p.rows[j] * p.lmax[j];
      roff[j + 1] = roff[j] + p.rows[j];
    }
    p.boff_dev = dalloc(sizeof(int64_t) * (nb + 1));
    p.roff_dev = dalloc(sizeof(int64_t) * (nb + 1));
    CudaCheck(cudaMemcpyAsync(p.boff_dev.get(), p.boff.data(), sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, s),
              "boff");
    CudaCheck(cudaMemcpyAsync(p.roff_dev.get(), roff.data(), sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, s),
              "roff");
    // per-row tables for the batch kernel (one pass per epoch, plan stream)
    const int64_t nrows = roff[nb];
    p.row_src_dev = dalloc(sizeof(int64_t) * std::max<int64_t>(nrows, 1));
    p.row_dst_dev = dalloc(sizeof(int64_t) * std::max<int64_t>(nrows, 1));
    p.row_lm_dev = dalloc(sizeof(int32_t) * std::max<int64_t>(nrows, 1));
    KCheck(dp_k_bucket_rows(P<int64_t>(perm), P<int64_t>(bstart), P<int32_t>(blmax), P<int64_t>(p.boff_dev),
                            P<int64_t>(p.roff_dev), nb, P<int64_t>(p.row_src_dev), P<int64_t>(p.row_dst_dev),
                            P<int32_t>(p.row_lm_dev), s),
           "bucket_rows");
    launches_++;
    // the host vectors are read by the copies: keep them alive until done
    CudaCheck(cudaStreamSynchronize(s), "bucket upload");
    p.roff = std::move(roff);
    p.order = perm;
    p.bstart_dev = bstart;
    p.rows_dev = brows;
    p.lmax_dev = blmax;
  }

  // The current positions before an interleave are source ordinals produced
  // by shards only: recover (first, stride) symbolically.
  void ArithmeticOf(int64_t /*count*/, int64_t& first, int64_t& stride) const {
    first = 0;
    stride = 1;
    for (const auto& op : L_.chain) {
      if (op.kind == IndexOp::Kind::kInterleave) break;
      first += op.b * stride;
      stride *= op.a;
    }
  }

  // Ensure epoch plan e exists and, for spanning batches, that the head of
  // epoch e+1 follows it in memory.
  void EnsurePlanFor(int64_t first_batch, int64_t nb) {
    if (!span_epochs_) {
      Plan(first_batch / std::max<int64_t>(batches_per_epoch_, 1));
      return;
    }
    const int64_t r0 = first_batch * L_.batch;
    const int64_t r1 = std::min(r0 + nb * L_.batch, total_batches_ >= 0 ? TotalRows() : INT64_MAX);
    const int64_t e0 = epoch_count_ ? r0 / epoch_count_ : 0;
    const int64_t e1 = epoch_count_ ? (r1 - 1) / epoch_count_ : 0;
    EpochPlan& p = Plan(e0);
    for (int64_t e = e0 + 1; e <= e1; ++e) {
      EpochPlan& q = Plan(e);
      // append epoch e's head after epoch e0's end (only e0 + 1 can be needed: tail = one group)
      const int64_t off = (e - e0) * epoch_count_;
      const int64_t need = std::min<int64_t>(q.count, p.count + p.tail - off);
      if (need > 0 && !appended_.count(e0 * 1000003 + e)) {
        CudaCheck(cudaStreamWaitEvent(plan_stream_, q.ready, 0), "wait");
        CudaCheck(cudaMemcpyAsync(P<int64_t>(p.order) + off, q.order.get(), sizeof(int64_t) * need,
                                  cudaMemcpyDeviceToDevice, plan_stream_),
                  "append head");
        CudaCheck(cudaEventRecord(p.ready, plan_stream_), "event");
        p.ready_gen++;
        appended_.insert(e0 * 1000003 + e);
      }
    }
  }

  bool MoreEpochsAfter(int64_t e) const {
    if (span_epochs_) {
      const int64_t rows = TotalRows();
      return rows == INT64_MAX || (e + 1) * epoch_count_ < rows;
    }
    if (L_.outer_repeat == kInfiniteRepeat) return true;
    return e + 1 < L_.outer_repeat;
  }

  int64_t TotalRows() const {
    int64_t inner = 1;
    for (const auto& op : L_.chain)
      if (op.kind == IndexOp::Kind::kRepeat) inner = op.a;
    return inner < 0 ? INT64_MAX : epoch_count_ * inner;
  }

  std::shared_ptr<Slot> NewSlot() {
    auto slot = std::make_shared<Slot>();
    slot->device = opt_.device;
    const int64_t cap = std::max(group_, head_);  // batches a slot holds (the head group may be larger)
    const size_t label_bytes = labels_ ? sizeof(int64_t) * L_.batch : 0;
    slot->a_bytes = (batch_bytes_.first - label_bytes) * cap;
    slot->b_bytes = batch_bytes_.second * cap;
    slot->c_bytes = label_bytes * cap;
    slot->a = DeviceAlloc(slot->a_bytes, opt_.device);
    if (slot->b_bytes) slot->b = DeviceAlloc(slot->b_bytes, opt_.device);
    if (slot->c_bytes) slot->c = DeviceAlloc(slot->c_bytes, opt_.device);
    if (opt_.host_output) {
      slot->ha = PinnedAlloc(slot->a_bytes);
      if (slot->b_bytes) slot->hb = PinnedAlloc(slot->b_bytes);
      if (slot->c_bytes) slot->hc = PinnedAlloc(slot->c_bytes);
    } else if (L_.unbatched && L_.ragged) {
      slot->hb = PinnedAlloc(slot->b_bytes);  // host copy of the row splits
    } else if (L_.unbatched) {
      slot->ha = PinnedAlloc(slot->a_bytes);  // host copy of the values / ids
      if (slot->c_bytes) slot->hc = PinnedAlloc(slot->c_bytes);  // and of the labels
    }
    CudaCheck(cudaEventCreateWithFlags(&slot->ready, cudaEventDisableTiming), "event");
    CudaCheck(cudaEventCreateWithFlags(&slot->release, cudaEventDisableTiming), "event");
    CudaCheck(cudaEventCreate(&slot->start), "event");
    slot_bytes_total_ += slot->a_bytes + slot->b_bytes + slot->c_bytes;
    slots_.push_back(slot);
    return slot;
  }

  std::shared_ptr<Slot> FindFreeSlot(bool may_grow) {
    if (autotune_ && !slots_preallocated_) {
      // every slot the tuner may use, once, so a depth change never allocates
      slots_preallocated_ = true;
      while (static_cast<int64_t>(slots_.size()) < max_depth_) NewSlot();
    }
    for (auto& s : slots_) {
      // free = never used, or its release event was recorded (which happens
      // only after every unit was handed out and dropped, see Lease)
      std::lock_guard lk(shared_->mu);
      if (!s->busy || s->release_recorded) return s;
    }
    const size_t need = (batch_bytes_.first + batch_bytes_.second) * std::max(group_, head_);
    if (static_cast<int64_t>(slots_.size()) < std::max(depth_, max_depth_) || may_grow) {
      if (slot_bytes_total_ + need > opt_.slot_memory_budget && !slots_.empty())
        throw PipelineError(ErrorCode::kInternal,
                            "prefetch slots exhausted: every device batch slot is still held by the consumer "
                            "(drop returned Elements before requesting more, or raise slot_memory_budget)");
      return NewSlot();
    }
    return nullptr;
  }

  void IssueGroup(int64_t g) {
    if (!TryIssueGroup(g, /*may_grow=*/true)) throw PipelineError(ErrorCode::kInternal, "could not issue batch group");
  }

  bool TryIssueGroup(int64_t g, bool may_grow) {
    auto [first, nb] = GroupRange(g);
    if (nb <= 0) {
      total_groups_ = g;
      return false;
    }
    auto slot = FindFreeSlot(may_grow);
    if (!slot) return false;
    const auto t0 = std::chrono::steady_clock::now();
    {
      std::lock_guard lk(shared_->mu);
      if (slot->busy) {
        // host_output: the previous D2H copy out of this slot (copy stream)
        if (opt_.host_output) CudaCheck(cudaStreamWaitEvent(stream_, slot->ready, 0), "wait copy");
        // consumer-stream work queued before the last drop; a release
        // recorded on this very stream is already ordered before the launch
        if (slot->release_recorded && consumer_ != stream_)
          CudaCheck(cudaStreamWaitEvent(stream_, slot->release, 0), "wait release");
      }
      slot->busy = true;
      slot->release_recorded = false;
      slot->first_batch = first;
      slot->num_batches = nb;
      slot->units = nb;  // unbatched: set to the element count below
      slot->handed_out = 0;
      slot->lease = std::shared_ptr<void>(
          nullptr,
          [slot_ref = slot, consumer = consumer_, shared = shared_](void*) {
            // the last holder of the group is gone: every unit was handed out
            // and dropped.  Record the release (one API call per group).
            std::lock_guard lk(shared->mu);
            if (shared->alive && !slot_ref->release_recorded) {
              cudaEventRecord(slot_ref->release, consumer);
              slot_ref->release_recorded = true;
              shared->slots_freed.fetch_add(1, std::memory_order_release);
            }
          },
          PoolAllocator<char>());
    }
    const auto tA = std::chrono::steady_clock::now();
    dbg_[3] += std::chrono::duration<double>(tA - t0).count();
    EnsurePlanFor(first, nb);
    const int64_t epoch = span_epochs_ ? (epoch_count_ ? first * L_.batch / epoch_count_ : 0)
                                       : first / std::max<int64_t>(batches_per_epoch_, 1);
    EpochPlan& plan = Plan(epoch);
    if (waited_plan_ != std::make_pair(epoch, plan.ready_gen)) {  // once per plan (re)record
      CudaCheck(cudaStreamWaitEvent(stream_, plan.ready, 0), "wait plan");
      waited_plan_ = {epoch, plan.ready_gen};
    }
    // Plan the next epoch on the side stream now, so its index kernels
    // overlap this epoch's batch kernels instead of stalling the next one.
    if (MoreEpochsAfter(epoch)) {
      if (L_.kind == BatchKind::kPadded) PrefetchPlan(epoch + 1);
      else Plan(epoch + 1);
    }
    // rows of this group inside the epoch plan
    const int64_t row0 = span_epochs_ ? first * L_.batch - epoch * epoch_count_
                                      : (first - epoch * batches_per_epoch_) * L_.batch;
    int64_t rows_total = 0;
    slot->batch_rows.assign(nb, 0);
    slot->batch_cols.assign(nb, 0);
    slot->batch_off_a.assign(nb, 0);
    slot->batch_off_b.assign(nb, 0);
    const int64_t avail = span_epochs_ ? plan.count + plan.tail : plan.count;
    for (int64_t k = 0; k < nb && !L_.bucketed; ++k) {
      int64_t rows = std::min<int64_t>(L_.batch, (span_epochs_ ? TotalRows() - (first + k) * L_.batch
                                                               : plan.count - (row0 + k * L_.batch)));
      rows = std::min<int64_t>(rows, avail - (row0 + k * L_.batch));
      slot->batch_rows[k] = rows;
      rows_total += rows;
    }
    const auto tB = std::chrono::steady_clock::now();
    dbg_[4] += std::chrono::duration<double>(tB - tA).count();
    TimedLaunch tl = NewTimedLaunch();
    CudaCheck(cudaEventRecord(tl.start, stream_), "event");
    const int64_t* order = P<int64_t>(plan.order);
    const float mean[3] = {L_.norm.mean[0], L_.norm.mean[1], L_.norm.mean[2]};
    const float stdv[3] = {L_.norm.stdv[0], L_.norm.stdv[1], L_.norm.stdv[2]};
    switch (L_.kind) {
      case BatchKind::kAffine:
      case BatchKind::kIdentityInt: {
        const int64_t* values = L_.source ? P<int64_t>(L_.source->values) : nullptr;
        if (!values && !order) {
          KCheck(dp_k_range_affine_batch(row0, rows_total, L_.affine_a, L_.affine_b, P<int64_t>(slot->a), stream_), "K1");
        } else {
          KCheck(dp_k_gather_affine_batch(values, order, row0, rows_total, L_.affine_a, L_.affine_b, P<int64_t>(slot->a),
                                          stream_),
                 "K1");
        }
        launches_++;
        int64_t off = 0;
        for (int64_t k = 0; k < nb; ++k) {
          slot->batch_off_a[k] = off * sizeof(int64_t);
          off += slot->batch_rows[k];
        }
        break;
      }
      case BatchKind::kCrop:
      case BatchKind::kResize: {
        const auto& src = *L_.source;
        const int oh = static_cast<int>(L_.kind == BatchKind::kCrop ? L_.crop.out_h : L_.resize.out_h);
        const int ow = static_cast<int>(L_.kind == BatchKind::kCrop ? L_.crop.out_w : L_.resize.out_w);
        if (L_.kind == BatchKind::kCrop && L_.crop.op == MapStep::Op::kCenterCrop)
          KCheck(dp_k_center_crop_normalize_batch_ex(P<uint8_t>(src.values), src.count, static_cast<int>(src.h),
                                                     static_cast<int>(src.w), order, row0, rows_total, src.shard_index,
                                                     src.shard_count, src.shard_block, oh, ow, mean, stdv,
                                                     P<int64_t>(slot->a), P<float>(slot->b), stream_),
                 "K3 center");
        else if (L_.kind == BatchKind::kCrop)
          KCheck(dp_k_crop_flip_normalize_batch_ex(P<uint8_t>(src.values), src.count, static_cast<int>(src.h),
                                                   static_cast<int>(src.w), order, row0, rows_total, src.shard_index,
                                                   src.shard_count, src.shard_block, L_.crop.seed, oh, ow, L_.crop.flip ? 1 : 0, mean,
                                                   stdv, P<int64_t>(slot->a), P<float>(slot->b), stream_),
                 "K3");
        else
          KCheck(dp_k_resize_normalize_batch_ex(P<uint8_t>(src.values), src.count, static_cast<int>(src.h),
                                                static_cast<int>(src.w), order, row0, rows_total, src.shard_index,
                                                src.shard_count, src.shard_block, oh, ow, mean, stdv, P<int64_t>(slot->a),
                                                P<float>(slot->b), stream_),
                 "K4");
        launches_++;
        int64_t off = 0;
        for (int64_t k = 0; k < nb; ++k) {
          slot->batch_off_a[k] = off * sizeof(int64_t);
          slot->batch_off_b[k] = off * sizeof(float) * oh * ow * 3;
          off += slot->batch_rows[k];
        }
        break;
      }
      case BatchKind::kChain:
      case BatchKind::kCopy: {
        const auto& src = *L_.source;
        if (L_.kind == BatchKind::kChain)
          KCheck(dp_k_image_chain_batch(P<uint8_t>(src.values), src.count, order, row0, rows_total, src.shard_index,
                                        src.shard_count, src.shard_block, &L_.img_chain, P<int64_t>(slot->a),
                                        slot->b.get(), stream_),
                 "K9 image chain");
        else
          KCheck(dp_k_gather_copy_batch(P<uint8_t>(src.values), src.count, src.h * src.w * 3, order, row0, rows_total,
                                        src.shard_index, src.shard_count, src.shard_block, P<int64_t>(slot->a),
                                        P<uint8_t>(slot->b), stream_),
                 "K9 gather");
        launches_++;
        const size_t img_bytes = (L_.img_f32 ? sizeof(float) : 1) * L_.img_h * L_.img_w * 3;
        int64_t off = 0;
        for (int64_t k = 0; k < nb; ++k) {
          slot->batch_off_a[k] = off * sizeof(int64_t);
          slot->batch_off_b[k] = off * img_bytes;
          off += slot->batch_rows[k];
        }
        break;
      }
      case BatchKind::kPadded: {
        const int64_t j0 = row0 / L_.batch;
        // staged plans: rows in consumption order in device memory
        const int32_t* tok = plan.staged ? P<int32_t>(plan.st_tokens) : P<int32_t>(L_.source->tokens);
        const int64_t* offs = plan.staged ? P<int64_t>(plan.st_offsets) : P<int64_t>(L_.source->offsets);
        const int32_t* lens = plan.staged ? P<int32_t>(plan.st_lengths) : P<int32_t>(L_.source->lengths);
        const int64_t* ord = plan.staged ? nullptr : order;
        if (L_.bucketed) {
          int64_t group_rows = 0;
          for (int64_t k = 0; k < nb; ++k) group_rows += slot->batch_rows[k] = plan.rows[j0 + k];
          KCheck(dp_k_bucket_rows_batches(tok, offs, lens, P<int64_t>(plan.row_src_dev),
                                          P<int64_t>(plan.row_dst_dev), P<int32_t>(plan.row_lm_dev), plan.roff[j0],
                                          plan.boff[j0], group_rows, static_cast<int32_t>(L_.pad),
                                          P<int32_t>(slot->a), P<int32_t>(slot->b), stream_),
                 "K8");
        } else if (L_.ragged) {
          KCheck(dp_k_ragged_batches(tok, offs, lens, ord, row0, rows_total, L_.batch, plan.count,
                                     P<int64_t>(plan.roff_dev), P<int32_t>(slot->a), P<int64_t>(slot->b), stream_),
                 "K5 ragged");
        } else {
          KCheck(dp_k_padded_batches(tok, offs, lens, ord, row0, rows_total, L_.batch,
                                     P<int32_t>(plan.lmax_dev), P<int64_t>(plan.boff_dev),
                                     static_cast<int32_t>(L_.pad), P<int32_t>(slot->a), P<int32_t>(slot->b), stream_),
                 "K5");
        }
        launches_++;
        int64_t off = 0;
        for (int64_t k = 0; k < nb; ++k) {
          slot->batch_cols[k] = plan.lmax[j0 + k];
          slot->batch_off_a[k] = (plan.boff[j0 + k] - plan.boff[j0]) * sizeof(int32_t);
          slot->batch_off_b[k] = L_.ragged ? (off + k) * sizeof(int64_t) : off * sizeof(int32_t);
          off += slot->batch_rows[k];
        }
        break;
      }
    }
    if (labels_) {  // the label component: labels[p] of every gathered row (K1 gather)
      KCheck(dp_k_gather_affine_batch(P<int64_t>(L_.source->labels), order, row0, rows_total, 1, 0,
                                      P<int64_t>(slot->c), stream_),
             "labels");
      launches_++;
    }
    const auto tC = std::chrono::steady_clock::now();
    dbg_[5] += std::chrono::duration<double>(tC - tB).count();
    CudaCheck(cudaEventRecord(tl.end, stream_), "event");
    batches_launched_ += nb;
    timed_.push_back(tl);
    if (opt_.host_output) {
      CudaCheck(cudaEventRecord(slot->ready, stream_), "event");
      CudaCheck(cudaStreamWaitEvent(copy_stream_, slot->ready, 0), "wait");
      const size_t a_used = UsedBytesA(*slot), b_used = UsedBytesB(*slot);
      CudaCheck(cudaMemcpyAsync(slot->ha.get(), slot->a.get(), a_used, cudaMemcpyDeviceToHost, copy_stream_), "d2h");
      if (b_used) CudaCheck(cudaMemcpyAsync(slot->hb.get(), slot->b.get(), b_used, cudaMemcpyDeviceToHost, copy_stream_), "d2h");
      const size_t c_used = labels_ ? a_used : 0;  // one int64 label per row, like the ids
      if (c_used) CudaCheck(cudaMemcpyAsync(slot->hc.get(), slot->c.get(), c_used, cudaMemcpyDeviceToHost, copy_stream_), "d2h");
      CudaCheck(cudaEventRecord(slot->ready, copy_stream_), "event");
      d2h_bytes_ += a_used + b_used + c_used;
    } else if (L_.unbatched && L_.ragged) {
      // single token sequences: the row splits locate them in the values
      CudaCheck(cudaMemcpyAsync(slot->hb.get(), slot->b.get(), UsedBytesB(*slot), cudaMemcpyDeviceToHost, stream_),
                "d2h splits");
      CudaCheck(cudaEventRecord(slot->ready, stream_), "event");
    } else if (L_.unbatched) {
      // element values / ids are served as host int64 values
      CudaCheck(cudaMemcpyAsync(slot->ha.get(), slot->a.get(), UsedBytesA(*slot), cudaMemcpyDeviceToHost, stream_),
                "d2h values");
      if (labels_)
        CudaCheck(cudaMemcpyAsync(slot->hc.get(), slot->c.get(), UsedBytesA(*slot), cudaMemcpyDeviceToHost, stream_),
                  "d2h labels");
      CudaCheck(cudaEventRecord(slot->ready, stream_), "event");
    } else {
      CudaCheck(cudaEventRecord(slot->ready, stream_), "event");
    }
    if (L_.unbatched) {
      std::lock_guard lk(shared_->mu);
      int64_t units = 0;
      for (auto r : slot->batch_rows) units += r;
      slot->units = units;
    }
    group_slot_[g] = slot;
    for (auto it = group_slot_.begin(); it != group_slot_.end() && it->first < g - 2 * depth_ - 4;)
      it = group_slot_.erase(it);
    issued_groups_ = std::max(issued_groups_, g + 1);
    dbg_[6] += std::chrono::duration<double>(std::chrono::steady_clock::now() - tC).count();
    host_issue_ns_ += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    issued_count_++;
    return true;
  }

  size_t UsedBytesA(const Slot& s) const {
    if (L_.ragged) {
      size_t t = 0;
      for (auto c : s.batch_cols) t += c * sizeof(int32_t);
      return t;
    }
    if (L_.kind == BatchKind::kPadded) {
      size_t t = 0;
      for (size_t k = 0; k < s.batch_rows.size(); ++k) t += s.batch_rows[k] * s.batch_cols[k] * sizeof(int32_t);
      return t;
    }
    int64_t rows = 0;
    for (auto r : s.batch_rows) rows += r;
    return rows * sizeof(int64_t);
  }
  size_t UsedBytesB(const Slot& s) const {
    int64_t rows = 0;
    for (auto r : s.batch_rows) rows += r;
    if (L_.ragged) return (rows + static_cast<int64_t>(s.batch_rows.size())) * sizeof(int64_t);
    if (L_.kind == BatchKind::kPadded) return rows * sizeof(int32_t);
    if (L_.kind == BatchKind::kCrop) return rows * sizeof(float) * L_.crop.out_h * L_.crop.out_w * 3;
    if (L_.kind == BatchKind::kResize) return rows * sizeof(float) * L_.resize.out_h * L_.resize.out_w * 3;
    if (L_.kind == BatchKind::kChain || L_.kind == BatchKind::kCopy)
      return rows * (L_.img_f32 ? sizeof(float) : 1) * L_.img_h * L_.img_w * 3;
    return 0;
  }

  // A lease on `slot` for one handed-out unit: a copy of the group's lease,
  // and for the group's last unit the iterator's own reference, moved.  The
  // group's deleter therefore runs on the drop of whichever unit goes last,
  // never before the last unit was handed out, and records the release event
  // under the lock; the slot is reused only after that (FindFreeSlot /
  // TryIssueGroup), and the event orders every unit's consumer-stream work
  // before the rewrite.  Per unit: one refcount increment, no allocation.
  std::shared_ptr<void> Lease(const std::shared_ptr<Slot>& slot) {
    const int64_t h = slot->handed_out.load(std::memory_order_relaxed) + 1;
    slot->handed_out.store(h, std::memory_order_relaxed);
    if (h >= slot->units) return std::move(slot->lease);
    return slot->lease;
  }

  Element MakeElement(const std::shared_ptr<Slot>& slot, int64_t i) {
    const int64_t k = i - slot->first_batch;
    const int64_t rows = slot->batch_rows[k];
    std::shared_ptr<void> lease = Lease(slot);
    const bool host = opt_.host_output;
    auto base_a = static_cast<uint8_t*>(host ? slot->ha.get() : slot->a.get()) + slot->batch_off_a[k];
    auto base_b = slot->b ? static_cast<uint8_t*>(host ? slot->hb.get() : slot->b.get()) + slot->batch_off_b[k] : nullptr;
    auto base_c = slot->c ? static_cast<uint8_t*>(host ? slot->hc.get() : slot->c.get()) + slot->batch_off_a[k] : nullptr;
    // the last component takes the lease itself (one refcount round trip fewer)
    auto mk = [&](DType dt, std::vector<int64_t> shape, void* data, bool last = false) {
      Tensor t;
      t.dtype = dt;
      t.shape = std::move(shape);
      t.data = data;
      t.residency = host ? Residency::kHost : Residency::kDevice;
      t.device = opt_.device;
      t.owner = last ? std::move(lease) : lease;
      t.ready = slot->ready;
      return Value::FromTensor(std::allocate_shared<Tensor>(PoolAllocator<Tensor>(), std::move(t)));
    };
    std::vector<Value> comps;
    comps.reserve(2);
    switch (L_.kind) {
      case BatchKind::kAffine:
      case BatchKind::kIdentityInt:
        comps.push_back(mk(DType::kInt64, {rows}, base_a, true));
        break;
      case BatchKind::kCrop:
        comps.push_back(mk(DType::kInt64, {rows}, base_a));
        comps.push_back(mk(DType::kFloat32, {rows, L_.crop.out_h, L_.crop.out_w, 3}, base_b, !labels_));
        break;
      case BatchKind::kResize:
        comps.push_back(mk(DType::kInt64, {rows}, base_a));
        comps.push_back(mk(DType::kFloat32, {rows, L_.resize.out_h, L_.resize.out_w, 3}, base_b, !labels_));
        break;
      case BatchKind::kChain:
      case BatchKind::kCopy:
        comps.push_back(mk(DType::kInt64, {rows}, base_a));
        comps.push_back(mk(L_.img_f32 ? DType::kFloat32 : DType::kUInt8, {rows, L_.img_h, L_.img_w, 3}, base_b,
                           !labels_));
        break;
      case BatchKind::kPadded:
        if (L_.ragged) {  // (values, row splits)
          comps.push_back(mk(DType::kInt32, {slot->batch_cols[k]}, base_a));
          comps.push_back(mk(DType::kInt64, {rows + 1}, base_b, true));
          break;
        }
        comps.push_back(mk(DType::kInt32, {rows, slot->batch_cols[k]}, base_a));
        comps.push_back(mk(DType::kInt32, {rows}, base_b, true));
        break;
    }
    if (labels_) comps.push_back(mk(DType::kInt64, {rows}, base_c, true));
    return Element(std::move(comps));
  }

  // unbatched: element `row` of internal batch i -- (int64 value) or (int64
  // id, tensor [h, w, 3] view into the slot), as MapIterator delivers them
  Element MakeUnitElement(const std::shared_ptr<Slot>& slot, int64_t i, int64_t row) {
    const int64_t k = i - slot->first_batch;
    std::shared_ptr<void> lease = Lease(slot);
    if (L_.ragged) {  // one token sequence: a device view into the batch's values
      const int64_t* splits = reinterpret_cast<const int64_t*>(static_cast<const uint8_t*>(slot->hb.get()) +
                                                               slot->batch_off_b[k]);
      Tensor t;
      t.dtype = DType::kInt32;
      t.shape = {splits[row + 1] - splits[row]};
      t.data = static_cast<uint8_t*>(slot->a.get()) + slot->batch_off_a[k] + splits[row] * sizeof(int32_t);
      t.residency = Residency::kDevice;
      t.device = opt_.device;
      t.owner = std::move(lease);
      t.ready = slot->ready;
      std::vector<Value> one;
      one.push_back(Value::FromTensor(std::move(t)));
      return Element(std::move(one));
    }
    const int64_t idx = slot->batch_off_a[k] / static_cast<int64_t>(sizeof(int64_t)) + row;
    const int64_t value = static_cast<const int64_t*>(slot->ha.get())[idx];
    std::vector<Value> comps;
    comps.reserve(3);
    comps.push_back(Value::Int64(value));
    if (IsImageKind()) {
      const int64_t oh = ImgH(), ow = ImgW();
      const size_t el = L_.kind == BatchKind::kCopy || (L_.kind == BatchKind::kChain && !L_.img_f32) ? 1 : sizeof(float);
      Tensor t;
      t.dtype = el == 1 ? DType::kUInt8 : DType::kFloat32;
      t.shape = {oh, ow, 3};
      t.data = static_cast<uint8_t*>(slot->b.get()) + slot->batch_off_b[k] + row * oh * ow * 3 * el;
      t.residency = Residency::kDevice;
      t.device = opt_.device;
      t.owner = std::move(lease);
      t.ready = slot->ready;
      comps.push_back(Value::FromTensor(std::move(t)));
      if (labels_) comps.push_back(Value::Int64(static_cast<const int64_t*>(slot->hc.get())[idx]));
    }
    // (int64 values were copied out: the slot can go as soon as this returns)
    Element e(std::move(comps));
    if (!IsImageKind()) lease.reset();
    return e;
  }

  bool IsImageKind() const {
    return L_.kind == BatchKind::kCrop || L_.kind == BatchKind::kResize || L_.kind == BatchKind::kChain ||
           L_.kind == BatchKind::kCopy;
  }
  int64_t ImgH() const {
    return L_.kind == BatchKind::kCrop ? L_.crop.out_h : L_.kind == BatchKind::kResize ? L_.resize.out_h : L_.img_h;
  }
  int64_t ImgW() const {
    return L_.kind == BatchKind::kCrop ? L_.crop.out_w : L_.kind == BatchKind::kResize ? L_.resize.out_w : L_.img_w;
  }

  // AUTOTUNE prefetch: depth = ceil(host issue time / device time per group)
  // + 2, re-evaluated from CUDA-event timings every 16 groups.
  struct TimedLaunch {
    cudaEvent_t start = nullptr, end = nullptr;
  };
  TimedLaunch NewTimedLaunch() {
    if (!event_pool_.empty()) {
      TimedLaunch t = event_pool_.back();
      event_pool_.pop_back();
      return t;
    }
    TimedLaunch t;
    CudaCheck(cudaEventCreate(&t.start), "event");
    CudaCheck(cudaEventCreate(&t.end), "event");
    return t;
  }

  // Accumulates the device duration of every completed batch-stage launch
  // (events recorded around the launch on the launching stream).
  void DrainTimings(bool wait) {
    while (!timed_.empty()) {
      TimedLaunch t = timed_.front();
      if (wait) {
        cudaEventSynchronize(t.end);
      } else if (cudaEventQuery(t.end) != cudaSuccess) {
        cudaGetLastError();
        break;
      }
      float ms = 0;
      if (cudaEventElapsedTime(&ms, t.start, t.end) == cudaSuccess) {
        batch_ns_total_ += static_cast<int64_t>(static_cast<double>(ms) * 1e6);
        timed_groups_++;
      }
      cudaGetLastError();
      timed_.pop_front();
      event_pool_.push_back(t);
    }
  }

 public:
  // Device time of the batch-stage launches completed so far (waits for all
  // issued ones) -> (total ns, launches).
  std::pair<int64_t, int64_t> BatchStageTiming() {
    DeviceGuard g(opt_.device);
    DrainTimings(true);
    return {batch_ns_total_, timed_groups_};
  }

 private:
  // AUTOTUNE prefetch depth from the reference's model (SURVEY.md 8(f)
  // next #3): the ring is an M/M/1/k queue (model.cpp:262-266, the kAsyncQueue
  // case) with producer rate x = launch groups/s the device writes (CUDA-
  // event self time of the batch stage, EWMA) and consumer rate y = groups/s
  // the consumer asks for (host time between group boundaries, EWMA), both
  // with RecordSelfTime's one-second half-life (model.cpp:47-64).  The
  // buffered groups n are the smallest whose PEmpty (model.cpp:29-42) is
  // <= 2%, or past which one more group lowers it by < 0.5% (a producer-
  // bound ring); depth = n + 1 (the group being consumed), capped by the
  // slots pre-allocated within slot_memory_budget at the first issue, so
  // a depth change never allocates.
  static double PEmpty(double n, double x, double y) {
    const double r = x / y;
    if (std::abs(r - 1.0) < 1e-9) return 1.0 / (n + 1.0);
    return std::clamp((1.0 - r) / (1.0 - std::pow(r, n + 1.0)), 0.0, 1.0);
  }
  static void Ewma(double& acc, bool& has, std::chrono::steady_clock::time_point& last, double sample) {
    const auto now = std::chrono::steady_clock::now();
    if (!has) {
      acc = sample;
      has = true;
    } else {
      const double dt = std::chrono::duration<double, std::nano>(now - last).count();
      const double w = std::min(std::exp2(-std::max(dt, 0.0) / 1e9), 0.95);
      acc = w * acc + (1.0 - w) * sample;
    }
    last = now;
  }
  void MaybeAutotune() {
    const int64_t done_before = timed_groups_;
    const int64_t ns_before = batch_ns_total_;
    DrainTimings(false);
    if (timed_groups_ > done_before)
      Ewma(prod_ns_, has_prod_, prod_last_, static_cast<double>(batch_ns_total_ - ns_before) /
                                                static_cast<double>(timed_groups_ - done_before));
    const auto now = std::chrono::steady_clock::now();
    if (has_boundary_)
      Ewma(cons_ns_, has_cons_, cons_last_, std::chrono::duration<double, std::nano>(now - last_boundary_).count());
    last_boundary_ = now;
    has_boundary_ = true;
    if (!autotune_ || !has_prod_ || !has_cons_) return;
    const double x = 1e9 / std::max(prod_ns_, 1.0), y = 1e9 / std::max(cons_ns_, 1.0);
    int64_t n = 1;
    while (n + 1 < max_depth_) {
      const double p = PEmpty(static_cast<double>(n), x, y);
      if (p <= 0.02 || p - PEmpty(static_cast<double>(n + 1), x, y) < 0.005) break;
      ++n;
    }
    depth_ = std::clamp<int64_t>(n + 1, 2, max_depth_);
    last_pempty_ = PEmpty(static_cast<double>(depth_ - 1), x, y);
  }

 public:
  struct TunerState {
    double producer_groups_per_s = 0, consumer_groups_per_s = 0, p_empty = 0;
    int64_t depth = 0, max_depth = 0;
  };
  TunerState Tuner() const {
    TunerState t;
    t.producer_groups_per_s = has_prod_ ? 1e9 / std::max(prod_ns_, 1.0) : 0;
    t.consumer_groups_per_s = has_cons_ ? 1e9 / std::max(cons_ns_, 1.0) : 0;
    t.p_empty = last_pempty_;
    t.depth = depth_;
    t.max_depth = max_depth_;
    return t;
  }

 private:

 public:
  int64_t d2h_bytes() const { return d2h_bytes_; }

  // Per-node rows in the reference's shape (runtime.hpp:46-51, Metrics()):
  // path, label, self time, elements produced.  Self time is device time
  // from CUDA events for the stages that run kernels (the fused batch stage;
  // each index op's per-epoch plan kernels), host issue time for prefetch;
  // maps fused into the batch stage report 0 (their work is the batch
  // stage's).
  std::vector<NodeMetricsRow> Metrics() {
    DeviceGuard g(opt_.device);
    DrainTimings(true);
    DrainOpTimings(true);
    std::vector<int64_t> op_ns(L_.chain.size(), 0);
    {
      std::lock_guard lk(metrics_mu_);
      for (size_t i = 0; i < op_ns_total_.size() && i < op_ns.size(); ++i) op_ns[i] = op_ns_total_[i];
    }
    std::vector<NodeMetricsRow> rows;
    for (const auto& path : L_.node_paths) {
      const std::string label = path.substr(path.rfind('/') + 1, path.rfind('@') - path.rfind('/') - 1);
      NodeMetricsRow r{path, label, 0, 0};
      if (path == L_.batch_node_path) {
        r.label += " (device: fused batch stage)";
        r.self_time_ns = batch_ns_total_;
        r.elements_produced = produced_;
      } else if (label == "prefetch") {
        r.label += " (device ring, depth " + std::to_string(depth_) + ")";
        r.self_time_ns = host_issue_ns_;
        r.elements_produced = produced_;
      } else if (label == "repeat" && path == L_.node_paths.front()) {
        r.elements_produced = produced_;
      } else {
        for (size_t i = 0; i < L_.chain.size(); ++i)
          if (L_.chain[i].path == path) {
            r.label += " (device: epoch plan)";
            r.self_time_ns = op_ns[i];
            std::lock_guard lk(metrics_mu_);
            r.elements_produced = i < op_produced_.size() ? op_produced_[i] : 0;
          }
      }
      rows.push_back(std::move(r));
    }
    return rows;
  }
  // State shared with outstanding slot leases (they may outlive the pipeline).
  struct Shared {
    std::mutex mu;
    bool alive = true;
    std::atomic<uint64_t> slots_freed{0};  // bumped when a slot's last batch is dropped
  };
  std::shared_ptr<Shared> shared_ = std::make_shared<Shared>();
  void Shutdown() {
    std::lock_guard lk(shared_->mu);
    shared_->alive = false;
  }

 private:
  Lowered L_;
  uint64_t base_seed_;
  IteratorOptions opt_;
  cudaStream_t stream_ = nullptr, plan_stream_ = nullptr, copy_stream_ = nullptr, consumer_ = nullptr;
  std::mutex rb_mu_;  // the plan read-back buffer (mapped pinned host memory)
  void* rb_host_ = nullptr;
  size_t rb_cap_ = 0;
  int64_t depth_ = 2;
  int64_t max_depth_ = 2;  // AUTOTUNE ceiling: the slots pre-allocated within the budget
  bool autotune_ = false;
  bool slots_preallocated_ = false;
  // AUTOTUNE model state (EWMAs of device ns per group, host ns per group)
  double prod_ns_ = 0, cons_ns_ = 0, last_pempty_ = 0;
  bool has_prod_ = false, has_cons_ = false, has_boundary_ = false;
  std::chrono::steady_clock::time_point prod_last_{}, cons_last_{}, last_boundary_{};
  const bool debug_timing_ = std::getenv("DP_DEBUG_TIMING") != nullptr;
  int64_t cur_group_ = -1;            // group of the last batch handed out
  uint64_t seen_freed_ = 0;           // Shared::slots_freed at the last issue attempt
  std::shared_ptr<Slot> cur_slot_;
  std::pair<size_t, size_t> batch_bytes_;
  int64_t max_len_ = 0;
  int64_t group_ = 1;
  bool labels_ = false;  // images with labels: a third component (int64 per row)
  int64_t head_ = 0;  // batches of the stream's first launch group (0: group_)
  bool span_epochs_ = false;
  int64_t epoch_count_ = 0, batches_per_epoch_ = 0, total_batches_ = 0, total_groups_ = -1;
  int64_t total_units_ = 0;  // unbatched: elements (-1 = infinite)
  std::map<int64_t, EpochPlan> plans_;
  std::pair<int64_t, int64_t> waited_plan_{-1, -1};  // (epoch, ready_gen) the batch stream last waited on
  cudaEvent_t retire_ev_ = nullptr;
  int64_t batches_launched_ = 0;
  std::set<int64_t> appended_;
  std::vector<std::shared_ptr<Slot>> slots_;
  std::map<int64_t, std::shared_ptr<Slot>> group_slot_;
  size_t slot_bytes_total_ = 0;
  int64_t issued_groups_ = 0, next_batch_ = 0, produced_ = 0;
  std::atomic<int64_t> launches_{0};  // also counted by the plan-prefetch thread
  // padded kinds: the next epoch's plan (which reads counts back to the host)
  // is built by a helper thread while this one serves GetNext
  std::future<void> pending_plan_;
  std::mutex plans_mu_;
  int64_t host_issue_ns_ = 0, issued_count_ = 0, batch_ns_total_ = 0, timed_groups_ = 0;
  std::deque<TimedLaunch> timed_;
  std::vector<TimedLaunch> event_pool_;
  int64_t d2h_bytes_ = 0;
  bool done_ = false;
  // index-op self time (plan kernels, built on the helper thread too)
  struct OpTimed {
    int op;
    cudaEvent_t start, end;
  };
  std::mutex metrics_mu_;
  std::vector<OpTimed> op_timed_;
  std::vector<int64_t> op_ns_total_, op_produced_;
};

// ---------------------------------------------------------- PipelineIterator --
PipelineIterator::PipelineIterator(DatasetGraph graph, const UdfRegistry& registry, IteratorOptions options)
    : graph_(std::move(graph)), options_(options) {
  if (!graph_.root()) throw PipelineError(ErrorCode::kValidationFailed, "empty graph");
  // UDF validation (runtime.cpp:2117-2156): every referenced UDF must exist
  std::function<void(const DatasetNode&)> validate = [&](const DatasetNode& n) {
    if (n.HasAttr("udf")) registry.Get(n.GetString("udf"));
    if (n.HasAttr("fused_filter_udf")) registry.Get(n.GetString("fused_filter_udf"));
    for (const auto& in : n.inputs()) validate(*in);
  };
  validate(*graph_.root());
  if (options_.seed_override) {
    base_seed_ = *options_.seed_override;
  } else {
    std::random_device rd;
    base_seed_ = MixSeeds(rd(), rd());
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw DeviceError("no CUDA device: the B200 engine has no CPU fallback");
  }
  Lowered L = Lower(graph_, registry);
  impl_ = std::make_unique<DevicePipeline>(L, base_seed_, options_);
}

PipelineIterator::~PipelineIterator() {
  if (impl_) impl_->Shutdown();
}

std::optional<Element> PipelineIterator::GetNext() {
  std::lock_guard lock(mu_);
  auto e = impl_->Next();
  if (e && !Conforms(*e, graph_.element_spec()))
    throw PipelineError(ErrorCode::kTypeMismatch,
                        "produced " + e->ToString() + " not conforming to " + graph_.element_spec().ToString());
  return e;
}

int64_t PipelineIterator::root_delivered() const {
  std::lock_guard lock(mu_);
  return impl_->delivered();
}

std::vector<NodeMetricsRow> PipelineIterator::Metrics() const {
  std::lock_guard lock(mu_);
  return impl_->Metrics();
}

void* PipelineIterator::stream() const { return impl_->stream(); }
int64_t PipelineIterator::prefetch_depth() const { return impl_->depth(); }
PipelineIterator::Stats PipelineIterator::stats() const {
  std::lock_guard lock(mu_);
  return impl_->stats();
}
int64_t PipelineIterator::kernel_launches() const { return impl_->launches(); }
int64_t PipelineIterator::batches_launched() const { return impl_->batches_launched(); }
void PipelineIterator::Seek(int64_t batches) {
  std::lock_guard lock(mu_);
  impl_->Seek(batches);
}
std::pair<int64_t, int64_t> PipelineIterator::BatchStageTiming() const {
  std::lock_guard lock(mu_);
  return impl_->BatchStageTiming();
}
std::string PipelineIterator::LoweringPlan() const { return impl_->Describe(); }

std::unique_ptr<PipelineIterator> MakeIterator(const DatasetGraph& graph, const UdfRegistry& registry,
                                               IteratorOptions options) {
  return std::make_unique<PipelineIterator>(graph, registry, options);
}

}  // namespace datapipe::b200
