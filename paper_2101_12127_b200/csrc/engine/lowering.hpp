// lowering.hpp -- the lowered form of a graph (engine-internal): the batch
// stage, the index chain and the source a DevicePipeline runs (lowering.cpp
// builds it; runtime.cpp runs it).
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "dpb200/datapipe.hpp"
#include "dpcuda.h"

namespace datapipe::b200::detail {

struct IndexOp {
  enum class Kind { kShard, kShuffle, kFilter, kInterleave, kRepeat } kind;
  int64_t a = 0, b = 0;  // shard(k, i) | shuffle(buffer) | filter(max_len) | interleave(cycle, records) | repeat(count)
  std::optional<uint64_t> seed;
  std::string path;
  int64_t parallel = 1;  // interleave num_parallel_calls
  // filter: the predicate, and the affine maps beneath it (v -> v * mul + add)
  DevicePredicate pred;
  int64_t mul = 1, add = 0;
  bool opaque = false;  // a non-affine map lies beneath the filter
};

// kChain: K9's general image map chain; kCopy: images batched with no map
enum class BatchKind { kAffine, kCrop, kResize, kPadded, kIdentityInt, kChain, kCopy };

struct Lowered {
  int64_t prefetch = 0;  // 0: none, -1: AUTOTUNE, else depth
  int64_t outer_repeat = 1;
  BatchKind kind = BatchKind::kIdentityInt;
  int64_t batch = 1;     // bucket_by_length: the largest bucket batch size
  bool drop = false;
  // no batch stage: GetNext delivers single elements (MapIterator and the
  // index ops as roots, runtime.cpp:480-535); the device still works in
  // internal batches of `batch` elements, served one by one
  bool unbatched = false;
  // bucket_by_length (a padded kind with per-bucket windows, K8)
  bool bucketed = false;
  // Batch of token sequences: ragged (values + row splits), a padded kind
  // without padding
  bool ragged = false;
  std::vector<int32_t> bucket_bounds;
  std::vector<int64_t> bucket_sizes;
  int64_t pad = 0;
  std::vector<MapStep> steps;
  int64_t affine_a = 1, affine_b = 0;
  MapStep crop{}, resize{}, norm{};
  dp_image_chain img_chain{};      // kChain
  int64_t img_h = 0, img_w = 0;    // kChain / kCopy: output image dims
  bool img_f32 = false;            // kChain: fp32 output (else u8)
  std::vector<IndexOp> chain;  // bottom-up
  SourcePtr source;            // element data (images / tokens / int64 values); null for range
  int64_t source_count = 0;    // positions entering the index chain
  SourcePtr records;           // interleave record source
  bool records_local = false;  // records hold only this shard's files (block residency): index held files
  std::vector<std::string> node_paths;  // root first
  std::string batch_node_path;
};

// Splits `g` into [prefetch]* [repeat] BATCH-STAGE INDEX-CHAIN SOURCE (see
// runtime.cpp); kInvalidAttr "device lowering: ..." for graphs the device
// path does not run (there is no CPU fallback).
Lowered Lower(const DatasetGraph& g, const UdfRegistry& reg);

}  // namespace datapipe::b200::detail
