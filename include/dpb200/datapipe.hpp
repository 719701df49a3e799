// dpb200/datapipe.hpp -- the Dataset / Iterator operator API of the B200
// engine: graph builders (ops::*), the UDF registry with device UDF
// descriptors, the static optimizer, and MakeIterator / GetNext.
//
// Drop-in surface for the reference's path:
//   ops::* builders     -- /root/reference/proj/include/datapipe/graph.hpp:134-165
//   Build / DatasetGraph -- graph.hpp:68-131
//   UdfRegistry          -- udf.hpp:41-87 (plus device descriptors)
//   Optimize / RuleSet   -- optimizer.hpp:22-75
//   MakeIterator / PipelineIterator::GetNext / IteratorOptions
//                        -- runtime.hpp:35-100
// The kinds on the path are supported; Range, TensorSlices, TokenSequences
// and PaddedBatch are the new kinds the north star names.  Graphs that do
// not lower onto the device path are rejected at MakeIterator with
// PipelineError(kInvalidAttr) -- there is no CPU fallback.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <variant>
#include <vector>

#include "dpb200/core.hpp"

namespace datapipe::b200 {

constexpr int64_t kAutotune = -1;        // graph.hpp:34
constexpr int64_t kInfiniteRepeat = -1;  // graph.hpp:36

enum class NodeKind : uint8_t {
  // reference kinds on the path (numbering of graph.hpp:38-56)
  kFromMemory = 0,
  kFromFile = 1,
  kInterleave = 5,
  kBatch = 6,
  kPrefetch = 8,
  kRepeat = 9,
  kShuffle = 10,
  kShard = 11,
  kMap = 2,
  kFilter = 3,
  kMapAndBatch = 16,
  // new kinds
  kRange = 32,
  kTensorSlices = 33,
  kTokenSequences = 34,
  kPaddedBatch = 35,
  kBucketByLength = 36,
};

const char* NodeKindName(NodeKind kind);

// ---- source data (device resident, or pinned host for end-to-end runs) ----
struct SourceData {
  // kRecords: length-prefixed record files (from_file); payloads packed
  // back to back in `values` (record_len bytes each when uniform, else 0)
  enum class Kind { kInt64, kImages, kTokens, kRecords } kind;
  int64_t record_len = 0;
  std::vector<int64_t> file_records;  // kRecords: records per file, in path order
  std::vector<int64_t> host_int64;    // kInt64 from_memory: the values (graph serialization)
  int64_t count = 0;
  // kInt64: values[count] (device);  kImages: u8 [count, h, w, c]
  // kTokens: lengths i32[count], offsets i64[count+1], tokens i32[total]
  std::shared_ptr<void> values, lengths, offsets, tokens;
  int64_t h = 0, w = 0, c = 0, total_tokens = 0;
  Residency residency = Residency::kDevice;
  int device = 0;
  // Sharded residency (one process per GPU): this process
  // holds only the elements with position p % shard_count == shard_index of a
  // `global_count`-element dataset, row r = position shard_index + r *
  // shard_count.  The graph must apply shard(shard_count, shard_index) to it
  // first (checked at MakeIterator).  shard_count 1 = fully resident.
  // shard_block R > 1: the record blocks of an interleave's shard -- this
  // process holds the R records of every interleave input (file) x with
  // x % shard_count == shard_index, row r = record (x * R + r % R) of file
  // x = (r / R) * shard_count + shard_index; the graph applies
  // shard(shard_count, shard_index) to the interleave's inputs.
  int64_t global_count = 0, shard_count = 1, shard_index = 0, shard_block = 1;
  // kImages: an int64 label per held row (the element is then (int64 id,
  // image, int64 label), FromMemory's tuple elements, element.hpp:30-184);
  // same residency as the images
  std::shared_ptr<void> labels;
};
using SourcePtr = std::shared_ptr<const SourceData>;

// Synthetic inputs, generated on the device.
SourcePtr SynthImages(int64_t count, int64_t h, int64_t w, uint64_t seed, int device = 0);
// Only shard `index` of `num_shards` of a `global_count`-image dataset is
// generated and held (pixels keyed by the global element id).
SourcePtr SynthImagesSharded(int64_t global_count, int64_t h, int64_t w, uint64_t seed, int64_t num_shards,
                             int64_t index, int device = 0);
// Synthetic records for interleave: `num_files` inputs of `records_per_file`
// images (record r of file x = image id x * R + r); this process holds only
// the files x % num_shards == index (all of them when num_shards is 1).
SourcePtr SynthRecordsSharded(int64_t num_files, int64_t records_per_file, int64_t h, int64_t w, uint64_t seed,
                              int64_t num_shards, int64_t index, int device = 0);
// A view of `s` declaring its residency: it holds shard `index` of
// `num_shards` of a `global_count`-element dataset in blocks of `block`
// consecutive positions (block 1 = element shards; block R = the files of an
// interleave's shard).  kInvalidAttr unless s->count is that shard's size.
SourcePtr AsShard(const SourcePtr& s, int64_t global_count, int64_t num_shards, int64_t index, int64_t block = 1);
// A view of image source `s` carrying an int64 label per held row (copied to
// the device, or to pinned host memory when `s` is host resident).
SourcePtr WithLabels(const SourcePtr& s, const int64_t* labels, int64_t count);
SourcePtr SynthTokens(int64_t count, uint32_t max_len, uint64_t len_seed, uint64_t tok_seed, int device = 0);
// Uploads host data (copied); images: u8 [count, h, w, 3].
SourcePtr ImagesFromHost(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device = 0);
// Wraps pinned host memory (not copied, must outlive the graph); the device
// kernels read it over PCIe (end-to-end runs).
SourcePtr ImagesFromPinnedHost(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device = 0);
SourcePtr Int64FromHost(const int64_t* values, int64_t count, int device = 0);
SourcePtr TokensFromHost(const int32_t* lengths, int64_t count, const int32_t* tokens, int device = 0);
// Token sequences copied into pinned, device-mapped host memory: the kernels
// read them over PCIe (end-to-end runs of the token configs).
SourcePtr TokensFromPinnedHost(const int32_t* lengths, int64_t count, const int32_t* tokens, int device = 0);
// Length-prefixed record files (formats.md:67-74) read in order; payloads
// packed into device memory.
// num_shards > 1: read only the files f % num_shards == index (an
// interleave's shard of the file list; every held file must hold the same
// record count R -- the reader's).
SourcePtr RecordsFromFiles(const std::vector<std::string>& paths, int device = 0, int64_t num_shards = 1,
                           int64_t index = 0);
// WriteRecordFile (runtime.hpp:102-107): [u32 LE length][payload] per record.
void WriteRecordFile(const std::string& path, const std::vector<std::string>& payloads);

// ---- graph IR ----
using AttrValue =
    std::variant<int64_t, uint64_t, double, bool, std::string, std::vector<std::string>, SourcePtr, std::vector<int64_t>>;
using Attrs = std::map<std::string, AttrValue>;

class DatasetNode {
 public:
  DatasetNode(NodeKind kind, std::vector<std::shared_ptr<const DatasetNode>> inputs, Attrs attrs, ElementSpec spec)
      : kind_(kind), inputs_(std::move(inputs)), attrs_(std::move(attrs)), spec_(std::move(spec)) {}
  NodeKind kind() const { return kind_; }
  const std::vector<std::shared_ptr<const DatasetNode>>& inputs() const { return inputs_; }
  const Attrs& attrs() const { return attrs_; }
  const ElementSpec& output_spec() const { return spec_; }
  bool HasAttr(const std::string& k) const { return attrs_.count(k) > 0; }
  int64_t GetInt(const std::string& k) const;
  int64_t GetIntOr(const std::string& k, int64_t fallback) const;
  uint64_t GetUint(const std::string& k) const;
  bool GetBoolOr(const std::string& k, bool fallback) const;
  const std::string& GetString(const std::string& k) const;
  const SourcePtr& GetSource(const std::string& k) const;

 private:
  NodeKind kind_;
  std::vector<std::shared_ptr<const DatasetNode>> inputs_;
  Attrs attrs_;
  ElementSpec spec_;
};
using NodePtr = std::shared_ptr<const DatasetNode>;

class DatasetGraph {
 public:
  DatasetGraph() = default;
  explicit DatasetGraph(NodePtr root) : root_(std::move(root)) {}
  const NodePtr& root() const { return root_; }
  const ElementSpec& element_spec() const { return root_->output_spec(); }
  std::string ToString() const;

 private:
  NodePtr root_;
};

// ---- device UDFs ----
// One step of a map UDF chain; consecutive steps are fused into one batch
// kernel at lowering time (K1 affine, K3 crop+flip+normalize, K4 resize +
// normalize).
struct MapStep {
  // kDecodeRaw: a from_file record (bytes) holding a raw uint8 HWC image of
  // out_h x out_w x 3 -> (int64 record ordinal, tensor u8[out_h, out_w, 3])
  // kCenterCrop: out_h x out_w window at ((H - out_h) / 2, (W - out_w) / 2)
  // kImageAffine: fp32 x * scale_c + shift_c per channel (two rounded ops)
  enum class Op { kAffine, kRandomCropFlip, kResizeBilinear, kNormalize, kDecodeRaw, kCenterCrop, kImageAffine } op;
  int64_t a = 1, b = 0;                 // affine
  int64_t out_h = 0, out_w = 0;         // crop / resize
  uint64_t seed = 0;                    // crop: Philox key
  bool flip = true;                     // crop: random horizontal flip
  std::array<float, 3> mean{}, stdv{};  // normalize
  std::array<float, 3> scale{}, shift{};  // image affine
};

// Device predicate for Filter: a conjunction of terms on one quantity of
// the element -- a token sequence's LENGTH (the cfg4 filter), or an int64
// element's VALUE (after the affine maps beneath the filter; the reference's
// keep_even / keep_odd, pipeline_spec.cpp:234-243).  % is C++'s truncated
// remainder, as in those UDFs.
struct PredicateTerm {
  enum class Op { kLE, kGE, kLT, kModEq, kModNe } op;
  int64_t a = 0, b = 0;  // v <= a | v >= a | v < a | v % a == b | v % a != b
};
struct DevicePredicate {
  enum class On { kLength, kValue } on = On::kLength;
  std::vector<PredicateTerm> terms;  // conjunction, at most 8
  int64_t MaxLen() const;            // kLength: the tightest v <= a bound (INT64_MAX if none)
};

// Interleave reader: input element x opens a dataset of `records` records
// valued x * records + r (index into the record source).
struct RecordReader {
  int64_t records = 0;
};

class UdfRegistry {
 public:
  struct Entry {
    std::vector<MapStep> map;              // map / map_and_batch
    std::optional<DevicePredicate> predicate;
    std::optional<RecordReader> reader;    // interleave
    std::optional<int64_t> cost_hint_ns;
  };
  UdfRegistry() = default;
  UdfRegistry(const UdfRegistry&) = delete;
  UdfRegistry& operator=(const UdfRegistry&) = delete;

  void Register(const std::string& name, Entry entry);  // kDuplicateName
  void RegisterAffine(const std::string& name, int64_t a, int64_t b);
  void RegisterRandomCropFlip(const std::string& name, int64_t crop_h, int64_t crop_w, uint64_t seed, bool flip);
  void RegisterResizeBilinear(const std::string& name, int64_t out_h, int64_t out_w);
  void RegisterNormalize(const std::string& name, std::array<float, 3> mean, std::array<float, 3> stdv);
  // cast: u8 image -> fp32 (exact), lowered as normalize(mean 0, std 1) --
  // (x - 0) / 1 is x exactly under the kernels' IEEE-exact normalize
  void RegisterCast(const std::string& name);
  void RegisterDecodeRaw(const std::string& name, int64_t h, int64_t w);
  // center crop (no randomness, no flip), dtype preserved
  void RegisterCenterCrop(const std::string& name, int64_t crop_h, int64_t crop_w);
  // per-channel x * scale_c + shift_c on an image (u8 or fp32) -> fp32
  void RegisterImageAffine(const std::string& name, std::array<float, 3> scale, std::array<float, 3> shift);
  void RegisterLengthFilter(const std::string& name, int64_t max_len);  // keep len <= max_len
  void RegisterValueFilter(const std::string& name, std::vector<PredicateTerm> terms);
  // keep_even / keep_odd / keep_all on int64 elements (the reference's
  // EnsurePredicates, pipeline_spec.cpp:234-243)
  void RegisterStandardPredicates();
  void RegisterRecordReader(const std::string& name, int64_t records);
  bool Contains(const std::string& name) const;
  const Entry& Get(const std::string& name) const;  // kUnknownUdf
  ElementSpec MapOutputSpec(const std::string& name, const ElementSpec& in) const;

 private:
  mutable std::mutex mu_;
  std::map<std::string, std::unique_ptr<Entry>> entries_;
};

ElementSpec ApplyMapSteps(const std::vector<MapStep>& steps, const ElementSpec& in);

NodePtr Build(NodeKind kind, std::vector<NodePtr> inputs, Attrs attrs, const UdfRegistry& reg);

namespace ops {
DatasetGraph Range(int64_t n, const UdfRegistry& reg);
DatasetGraph FromMemory(const std::vector<int64_t>& values, const UdfRegistry& reg, int device = 0);
DatasetGraph TensorSlices(SourcePtr images, const UdfRegistry& reg);
DatasetGraph TokenSequences(SourcePtr tokens, const UdfRegistry& reg);
// ops::FromFile (graph.hpp:137; record format formats.md:67-74): the files'
// length-prefixed records, in file order, become (bytes) elements.  Read and
// validated here (kMissingFile, kMalformedInput); payloads are packed into
// device memory once.
DatasetGraph FromFile(const std::vector<std::string>& paths, const UdfRegistry& reg, int device = 0);
DatasetGraph Map(const DatasetGraph& in, const std::string& udf, int64_t num_parallel_calls, const UdfRegistry& reg);
DatasetGraph Filter(const DatasetGraph& in, const std::string& udf, const UdfRegistry& reg);
DatasetGraph Interleave(const DatasetGraph& in, const std::string& udf, int64_t cycle_length,
                        int64_t num_parallel_calls, SourcePtr records, const UdfRegistry& reg);
DatasetGraph Batch(const DatasetGraph& in, int64_t batch_size, bool drop_remainder, const UdfRegistry& reg);
DatasetGraph PaddedBatch(const DatasetGraph& in, int64_t batch_size, int64_t padding_value, bool drop_remainder,
                         const UdfRegistry& reg);
// tf.data bucket_by_sequence_length over token sequences (cfg4 "/
// bucket-by-length"; a new kind like PaddedBatch): bucket b holds
// boundaries[b-1] <= len < boundaries[b] and is batched by batch_sizes[b]
// (boundaries.size() + 1 entries, <= 32 buckets); each batch is padded to its
// own max length with padding_value.  Batches come out as their windows fill,
// then the partial windows in ascending bucket order unless drop_remainder.
DatasetGraph BucketByLength(const DatasetGraph& in, const std::vector<int64_t>& boundaries,
                            const std::vector<int64_t>& batch_sizes, int64_t padding_value, bool drop_remainder,
                            const UdfRegistry& reg);
DatasetGraph Prefetch(const DatasetGraph& in, int64_t buffer_size, const UdfRegistry& reg);
DatasetGraph Repeat(const DatasetGraph& in, int64_t count, const UdfRegistry& reg);
DatasetGraph Shuffle(const DatasetGraph& in, int64_t buffer_size, std::optional<uint64_t> seed,
                     const UdfRegistry& reg);
DatasetGraph Shard(const DatasetGraph& in, int64_t num_shards, int64_t index, const UdfRegistry& reg);
}  // namespace ops

// ---- static optimizer (optimizer.hpp:22-75; formats.md:152-186) ----
inline constexpr const char* kMapMapFusion = "map_map_fusion";
inline constexpr const char* kFilterFilterFusion = "filter_filter_fusion";
inline constexpr const char* kMapFilterFusion = "map_filter_fusion";
inline constexpr const char* kMapVectorization = "map_vectorization";
inline constexpr const char* kMapBatchFusion = "map_batch_fusion";
inline constexpr const char* kShuffleRepeatFusion = "shuffle_repeat_fusion";

class RuleSet {
 public:
  static RuleSet Default();
  static RuleSet None() { return RuleSet(); }
  void Disable(const std::string& name);
  bool IsEnabled(const std::string& name) const;
  const std::vector<std::string>& order() const { return order_; }
  static const std::vector<std::string>& AllRuleNames();

 private:
  std::vector<std::string> order_;
};

struct RewriteRecord {
  std::string rule, node_path;
};
struct RewriteReport {
  std::vector<RewriteRecord> applied;
  int iterations = 0;
  std::string ToString() const;
};

std::pair<DatasetGraph, RewriteReport> Optimize(const DatasetGraph& graph, const RuleSet& rules,
                                                UdfRegistry& registry);

// ---- runtime ----
struct IteratorOptions {
  bool deterministic = true;
  std::optional<uint64_t> seed_override;  // base seed (runtime.hpp:35-44)
  // B200 extensions --------------------------------------------------------
  int device = 0;
  // Stream (cudaStream_t) the consumer reads batches on; batch i is made
  // ready on it with cudaStreamWaitEvent, and a released slot is reused only
  // after the consumer's work queued on it so far.  nullptr = the iterator's
  // own stream (consumer work queued there is ordered by construction).
  void* consumer_stream = nullptr;
  // Copy each batch into pinned host memory before returning it.
  bool host_output = false;
  // Upper bound on device memory for prefetch slots (bytes).
  size_t slot_memory_budget = size_t(8) << 30;
  // Output bytes one fused launch may produce (consecutive batches are
  // grouped into one launch up to this size); 0 = 3.2 GB (512 MB with
  // host_output).
  size_t max_launch_bytes = 0;
  // Batches per fused launch, exactly (0 = from max_launch_bytes, rounded
  // down to a power of two).  Launch groups never straddle an epoch of a
  // per-epoch batch stage, so the last group of an epoch may be shorter.
  int64_t launch_batches = 0;
  // Batches of the stream's first launch group only (0 = launch_batches);
  // the groups after it tile the stream (or epoch 0) from there.
  int64_t first_launch_batches = 0;
};

struct NodeMetricsRow {
  std::string path, label;
  int64_t self_time_ns = 0;
  int64_t elements_produced = 0;
};

class DevicePipeline;  // lowering + device state (runtime.cpp)

class PipelineIterator {
 public:
  PipelineIterator(DatasetGraph graph, const UdfRegistry& registry, IteratorOptions options);
  ~PipelineIterator();
  PipelineIterator(const PipelineIterator&) = delete;
  PipelineIterator& operator=(const PipelineIterator&) = delete;

  // Next batch, or nullopt after the end (sticky).  Thread-safe.  Returned
  // tensors are ready on options().consumer_stream; Tensor::ready is the
  // producing event for other streams.
  std::optional<Element> GetNext();

  const DatasetGraph& graph() const { return graph_; }
  const IteratorOptions& options() const { return options_; }
  uint64_t base_seed() const { return base_seed_; }
  int64_t root_delivered() const;
  std::vector<NodeMetricsRow> Metrics() const;
  void* stream() const;                 // the iterator's producer stream
  int64_t prefetch_depth() const;       // device slots in use (autotuned)
  int64_t kernel_launches() const;      // sm_100a kernels issued so far
  int64_t batches_launched() const;     // batches covered by issued batch-stage launches
  struct Stats {
    int64_t live_plans = 0, slots = 0, slot_bytes = 0, prefetch_depth = 0, group_batches = 0, max_depth = 0;
    double producer_groups_per_s = 0, consumer_groups_per_s = 0, p_empty = 0;
  };
  Stats stats() const;
  // Checkpoint in the reference's DPC1 layout (checkpoint.hpp:36-49,
  // formats.md:76-94).  Restore() seeks instead of replaying.
  std::string Save() const;
  // Repositions a fresh iterator at batch `batches` without computing the
  // skipped ones (kCorruptBlob past the end).
  void Seek(int64_t batches);
  // Device time (CUDA events around each launch, on the launching stream)
  // of the fused batch-stage launches issued so far: {total ns, launches}.
  std::pair<int64_t, int64_t> BatchStageTiming() const;
  std::string LoweringPlan() const;     // human-readable lowering

 private:
  DatasetGraph graph_;
  IteratorOptions options_;
  uint64_t base_seed_;
  std::unique_ptr<DevicePipeline> impl_;
  mutable std::mutex mu_;
};

std::unique_ptr<PipelineIterator> MakeIterator(const DatasetGraph& graph, const UdfRegistry& registry,
                                               IteratorOptions options = {});

// Restore(graph, registry, blob) (checkpoint.cpp:50-105): validates magic
// (kCorruptBlob), version (kVersionMismatch) and the seed-invariant graph
// fingerprint (kFingerprintMismatch), then MakeIterator with the recorded
// base seed and Seek to the saved position.
std::unique_ptr<PipelineIterator> Restore(const DatasetGraph& graph, const UdfRegistry& registry,
                                          const std::string& blob, IteratorOptions options = {});

// ---- pipeline description text (formats.md "Pipeline description text
// format"; pipeline_spec.hpp ParsePipelineSpec) for device pipelines: the
// reference's stanza grammar with the device UDF library (see
// engine/pipeline_spec.cpp for the stanzas).  Errors: kParseError with
// "line L, col C: ...".
struct ParsedPipeline {
  DatasetGraph graph;
  IteratorOptions options;
  int epochs = 5;
  std::vector<std::string> disabled_rules;
  struct TunableRef {
    std::string name;  // "map@0.parallel", "prefetch@1.buffer"
    std::string attr;  // "num_parallel_calls" | "buffer_size"
  };
  std::vector<TunableRef> tunables;
};
ParsedPipeline ParsePipelineSpec(const std::string& text, UdfRegistry& registry, int device = 0);
ParsedPipeline ParsePipelineSpecFile(const std::string& path, UdfRegistry& registry, int device = 0);

// ---- graph serialization (formats.md "Graph serialization"; serialize.hpp) ----
// DPG1 bytes, canonical (preorder nodes, attrs in ascending key order).
// Kinds and attrs shared with the reference encode exactly as the
// reference's Serialize does (from_memory -> "elements" element list of int64
// scalars, from_file -> "paths"), so those graphs' bytes and fingerprints are
// the reference's.  Device data with no reference encoding (tensor_slices /
// token_sequences sources, interleave records) is written as a descriptor
// (attr tag 32: kind and shape, not the data) and re-bound at Deserialize from
// `sources`, consumed in preorder; a descriptor mismatch is kValidationFailed.
std::string Serialize(const DatasetGraph& graph);
DatasetGraph Deserialize(const std::string& bytes, const UdfRegistry& registry,
                         const std::vector<SourcePtr>& sources = {}, int device = 0);
// SHA-256 of the serialization with every "seed" attr zeroed
// (GraphFingerprint, serialize.cpp:213-216): the checkpoint fingerprint.
std::array<uint8_t, 32> GraphFingerprint(const DatasetGraph& graph);
std::string FingerprintHex(const std::array<uint8_t, 32>& fp);
std::array<uint8_t, 32> Sha256Digest(const void* data, size_t n);  // FIPS 180-4

// PRNG contract helpers (random.hpp:24-34; runtime.cpp:713-718).
uint64_t MixSeeds(uint64_t a, uint64_t b);
uint64_t ShuffleEngineSeed(uint64_t epoch_salt, std::optional<uint64_t> attr_seed);

}  // namespace datapipe::b200
