// capi_pipeline.cpp -- extern "C" binding of the operator API
// (include/dpcuda_pipeline.h -> include/dpb200/datapipe.hpp).  Exceptions
// never cross the boundary: PipelineError -> its ErrorCode + 1, DeviceError
// -> DP_ERR_CUDA, anything else -> DP_ERR_INTERNAL; the message goes to
// dp_last_error().
#include <cuda_runtime.h>

#include <cstring>
#include <sstream>

#include "dpb200/datapipe.hpp"
#include "dpcuda_pipeline.h"
#include "status.hpp"

using namespace datapipe::b200;

struct dp_registry {
  UdfRegistry reg;
};
struct dp_graph {
  DatasetGraph g;
};
struct dp_source {
  SourcePtr s;
};
struct dp_iterator {
  std::unique_ptr<PipelineIterator> it;
};

namespace {

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return DP_OK;
  } catch (const DeviceError& e) {
    return dpk::fail(DP_ERR_CUDA, e.what());
  } catch (const PipelineError& e) {
    return dpk::fail(static_cast<int>(e.code()) + 1, e.what());
  } catch (const std::exception& e) {
    return dpk::fail(DP_ERR_INTERNAL, e.what());
  }
}

int NullArg(const char* what) { return dpk::fail(DP_ERR_INVALID_ATTR, std::string("null argument: ") + what); }

void CopyOut(const std::string& s, char* buf, size_t len) {
  if (!buf || !len) return;
  std::strncpy(buf, s.c_str(), len - 1);
  buf[len - 1] = '\0';
}

int Emit(dp_graph** out, DatasetGraph g) {
  *out = new dp_graph{std::move(g)};
  return DP_OK;
}

}  // namespace

#define DP_REQUIRE(x) \
  if (!(x)) return NullArg(#x)

extern "C" {

int dp_registry_create(dp_registry** out) {
  DP_REQUIRE(out);
  return Guard([&] { *out = new dp_registry(); });
}
void dp_registry_destroy(dp_registry* reg) { delete reg; }

int dp_registry_register_affine(dp_registry* reg, const char* name, int64_t a, int64_t b) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterAffine(name, a, b); });
}
int dp_registry_register_random_crop_flip(dp_registry* reg, const char* name, int64_t crop_h, int64_t crop_w,
                                          uint64_t seed, int flip) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterRandomCropFlip(name, crop_h, crop_w, seed, flip != 0); });
}
int dp_registry_register_resize_bilinear(dp_registry* reg, const char* name, int64_t out_h, int64_t out_w) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterResizeBilinear(name, out_h, out_w); });
}
int dp_registry_register_normalize(dp_registry* reg, const char* name, const float mean[3], const float stdv[3]) {
  DP_REQUIRE(reg && name && mean && stdv);
  return Guard([&] { reg->reg.RegisterNormalize(name, {mean[0], mean[1], mean[2]}, {stdv[0], stdv[1], stdv[2]}); });
}
int dp_registry_register_cast(dp_registry* reg, const char* name) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterCast(name); });
}
int dp_registry_register_center_crop(dp_registry* reg, const char* name, int64_t crop_h, int64_t crop_w) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterCenterCrop(name, crop_h, crop_w); });
}
int dp_registry_register_image_affine(dp_registry* reg, const char* name, const float scale[3],
                                      const float shift[3]) {
  DP_REQUIRE(reg && name && scale && shift);
  return Guard(
      [&] { reg->reg.RegisterImageAffine(name, {scale[0], scale[1], scale[2]}, {shift[0], shift[1], shift[2]}); });
}
int dp_registry_register_length_filter(dp_registry* reg, const char* name, int64_t max_len) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterLengthFilter(name, max_len); });
}
int dp_registry_register_value_filter(dp_registry* reg, const char* name, const dp_predicate_term* terms,
                                      int num_terms) {
  DP_REQUIRE(reg && name && (terms || num_terms == 0));
  return Guard([&] {
    std::vector<PredicateTerm> t;
    for (int i = 0; i < num_terms; ++i) {
      if (terms[i].op < DP_PRED_LE || terms[i].op > DP_PRED_MOD_NE)
        throw PipelineError(ErrorCode::kInvalidAttr, "value filter: unknown predicate op");
      t.push_back({static_cast<PredicateTerm::Op>(terms[i].op), terms[i].a, terms[i].b});
    }
    reg->reg.RegisterValueFilter(name, std::move(t));
  });
}
int dp_registry_register_standard_predicates(dp_registry* reg) {
  DP_REQUIRE(reg);
  return Guard([&] { reg->reg.RegisterStandardPredicates(); });
}
int dp_registry_register_record_reader(dp_registry* reg, const char* name, int64_t records) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterRecordReader(name, records); });
}
int dp_registry_register_decode_raw(dp_registry* reg, const char* name, int64_t h, int64_t w) {
  DP_REQUIRE(reg && name);
  return Guard([&] { reg->reg.RegisterDecodeRaw(name, h, w); });
}
int dp_registry_contains(const dp_registry* reg, const char* name) {
  return reg && name && reg->reg.Contains(name) ? 1 : 0;
}

// ---- sources ----
int dp_source_synthetic_images(int64_t count, int64_t h, int64_t w, uint64_t seed, int device, dp_source** out) {
  DP_REQUIRE(out);
  return Guard([&] { *out = new dp_source{SynthImages(count, h, w, seed, device)}; });
}
int dp_source_synthetic_images_sharded(int64_t global_count, int64_t h, int64_t w, uint64_t seed,
                                       int64_t num_shards, int64_t index, int device, dp_source** out) {
  DP_REQUIRE(out);
  return Guard([&] { *out = new dp_source{SynthImagesSharded(global_count, h, w, seed, num_shards, index, device)}; });
}
int dp_source_synthetic_records_sharded(int64_t num_files, int64_t records_per_file, int64_t h, int64_t w,
                                        uint64_t seed, int64_t num_shards, int64_t index, int device,
                                        dp_source** out) {
  DP_REQUIRE(out);
  return Guard([&] {
    *out = new dp_source{SynthRecordsSharded(num_files, records_per_file, h, w, seed, num_shards, index, device)};
  });
}
int dp_source_as_shard(const dp_source* src, int64_t global_count, int64_t num_shards, int64_t index,
                       int64_t block, dp_source** out) {
  DP_REQUIRE(src && out);
  return Guard([&] { *out = new dp_source{AsShard(src->s, global_count, num_shards, index, block)}; });
}
int dp_source_with_labels(const dp_source* images, const int64_t* labels, int64_t count, dp_source** out) {
  DP_REQUIRE(images && out && (labels || count == 0));
  return Guard([&] { *out = new dp_source{WithLabels(images->s, labels, count)}; });
}
int dp_source_images_from_host(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device,
                               dp_source** out) {
  DP_REQUIRE(data && out);
  return Guard([&] { *out = new dp_source{ImagesFromHost(data, count, h, w, device)}; });
}
int dp_source_images_pinned_host(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device,
                                 dp_source** out) {
  DP_REQUIRE(data && out);
  return Guard([&] { *out = new dp_source{ImagesFromPinnedHost(data, count, h, w, device)}; });
}
int dp_source_synthetic_tokens(int64_t count, uint32_t max_len, uint64_t len_seed, uint64_t tok_seed, int device,
                               dp_source** out) {
  DP_REQUIRE(out);
  return Guard([&] { *out = new dp_source{SynthTokens(count, max_len, len_seed, tok_seed, device)}; });
}
int dp_source_tokens_from_host(const int32_t* lengths, int64_t count, const int32_t* tokens, int device,
                               dp_source** out) {
  DP_REQUIRE(lengths && out);
  return Guard([&] { *out = new dp_source{TokensFromHost(lengths, count, tokens, device)}; });
}
int dp_source_tokens_pinned_host(const int32_t* lengths, int64_t count, const int32_t* tokens, int device,
                                 dp_source** out) {
  DP_REQUIRE(out && count >= 0 && (lengths || count == 0));
  return Guard([&] { *out = new dp_source{TokensFromPinnedHost(lengths, count, tokens, device)}; });
}
int dp_source_records_from_files(const char* const* paths, int64_t num_paths, int device, dp_source** out) {
  return dp_source_records_from_files_sharded(paths, num_paths, 1, 0, device, out);
}
int dp_source_records_from_files_sharded(const char* const* paths, int64_t num_paths, int64_t num_shards,
                                         int64_t index, int device, dp_source** out) {
  DP_REQUIRE(out && (paths || num_paths == 0) && num_paths >= 0);
  return Guard([&] {
    std::vector<std::string> p;
    for (int64_t i = 0; i < num_paths; ++i) {
      if (!paths[i]) throw PipelineError(ErrorCode::kInvalidAttr, "records_from_files: null path");
      p.emplace_back(paths[i]);
    }
    *out = new dp_source{RecordsFromFiles(p, device, num_shards, index)};
  });
}
void dp_source_release(dp_source* src) { delete src; }

// ---- graphs ----
int dp_graph_range(const dp_registry* reg, int64_t n, dp_graph** out) {
  DP_REQUIRE(reg && out);
  return Guard([&] { Emit(out, ops::Range(n, reg->reg)); });
}
int dp_graph_from_memory_i64(const dp_registry* reg, const int64_t* values, int64_t n, int device, dp_graph** out) {
  DP_REQUIRE(reg && out && (values || n == 0));
  return Guard([&] { Emit(out, ops::FromMemory(std::vector<int64_t>(values, values + n), reg->reg, device)); });
}
int dp_graph_tensor_slices(const dp_registry* reg, const dp_source* images, dp_graph** out) {
  DP_REQUIRE(reg && images && out);
  return Guard([&] { Emit(out, ops::TensorSlices(images->s, reg->reg)); });
}
int dp_graph_from_file(const dp_registry* reg, const char* const* paths, int64_t num_paths, int device,
                       dp_graph** out) {
  DP_REQUIRE(reg && out && (paths || num_paths == 0) && num_paths >= 0);
  return Guard([&] {
    std::vector<std::string> p;
    for (int64_t i = 0; i < num_paths; ++i) {
      if (!paths[i]) throw PipelineError(ErrorCode::kInvalidAttr, "from_file: null path");
      p.emplace_back(paths[i]);
    }
    Emit(out, ops::FromFile(p, reg->reg, device));
  });
}
int dp_write_record_file(const char* path, const uint8_t* data, const int64_t* offsets, int64_t count) {
  DP_REQUIRE(path && offsets && count >= 0 && (data || count == 0));
  return Guard([&] {
    std::vector<std::string> payloads;
    payloads.reserve(count);
    for (int64_t i = 0; i < count; ++i) {
      if (offsets[i + 1] < offsets[i]) throw PipelineError(ErrorCode::kInvalidAttr, "write_record_file: offsets");
      payloads.emplace_back(reinterpret_cast<const char*>(data) + offsets[i], offsets[i + 1] - offsets[i]);
    }
    WriteRecordFile(path, payloads);
  });
}
int dp_graph_token_sequences(const dp_registry* reg, const dp_source* tokens, dp_graph** out) {
  DP_REQUIRE(reg && tokens && out);
  return Guard([&] { Emit(out, ops::TokenSequences(tokens->s, reg->reg)); });
}
int dp_graph_map(const dp_graph* in, const char* udf, int64_t p, const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && udf && reg && out);
  return Guard([&] { Emit(out, ops::Map(in->g, udf, p, reg->reg)); });
}
int dp_graph_filter(const dp_graph* in, const char* udf, const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && udf && reg && out);
  return Guard([&] { Emit(out, ops::Filter(in->g, udf, reg->reg)); });
}
int dp_graph_interleave(const dp_graph* in, const char* udf, int64_t cycle, int64_t p, const dp_source* records,
                        const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && udf && reg && out);
  return Guard([&] { Emit(out, ops::Interleave(in->g, udf, cycle, p, records ? records->s : nullptr, reg->reg)); });
}
int dp_graph_batch(const dp_graph* in, int64_t b, int drop, const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] { Emit(out, ops::Batch(in->g, b, drop != 0, reg->reg)); });
}
int dp_graph_padded_batch(const dp_graph* in, int64_t b, int64_t pad, int drop, const dp_registry* reg,
                          dp_graph** out) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] { Emit(out, ops::PaddedBatch(in->g, b, pad, drop != 0, reg->reg)); });
}
int dp_graph_bucket_by_length(const dp_graph* in, const int64_t* boundaries, int64_t num_boundaries,
                              const int64_t* batch_sizes, int64_t pad, int drop, const dp_registry* reg,
                              dp_graph** out) {
  DP_REQUIRE(in && reg && out && batch_sizes && num_boundaries >= 0 && (boundaries || num_boundaries == 0));
  return Guard([&] {
    std::vector<int64_t> b(boundaries, boundaries + num_boundaries), s(batch_sizes, batch_sizes + num_boundaries + 1);
    Emit(out, ops::BucketByLength(in->g, b, s, pad, drop != 0, reg->reg));
  });
}
int dp_graph_prefetch(const dp_graph* in, int64_t buffer_size, const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] { Emit(out, ops::Prefetch(in->g, buffer_size, reg->reg)); });
}
int dp_graph_repeat(const dp_graph* in, int64_t count, const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] { Emit(out, ops::Repeat(in->g, count, reg->reg)); });
}
int dp_graph_shuffle(const dp_graph* in, int64_t buffer_size, int has_seed, uint64_t seed, const dp_registry* reg,
                     dp_graph** out) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] {
    Emit(out, ops::Shuffle(in->g, buffer_size, has_seed ? std::optional<uint64_t>(seed) : std::nullopt, reg->reg));
  });
}
int dp_graph_shard(const dp_graph* in, int64_t k, int64_t index, const dp_registry* reg, dp_graph** out) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] { Emit(out, ops::Shard(in->g, k, index, reg->reg)); });
}
int dp_graph_optimize(const dp_graph* in, dp_registry* reg, const char* disabled, dp_graph** out, char* report,
                      size_t report_len) {
  DP_REQUIRE(in && reg && out);
  return Guard([&] {
    RuleSet rules = RuleSet::Default();
    if (disabled && *disabled) {
      std::stringstream ss(disabled);
      std::string r;
      while (std::getline(ss, r, ','))
        if (!r.empty()) rules.Disable(r);
    }
    auto [g, rep] = Optimize(in->g, rules, reg->reg);
    CopyOut(rep.ToString(), report, report_len);
    Emit(out, std::move(g));
  });
}
int dp_graph_root_kind(const dp_graph* g, char* buf, size_t len) {
  DP_REQUIRE(g && buf);
  CopyOut(NodeKindName(g->g.root()->kind()), buf, len);
  return DP_OK;
}
int dp_graph_to_string(const dp_graph* g, char* buf, size_t len) {
  DP_REQUIRE(g && buf);
  CopyOut(g->g.ToString(), buf, len);
  return DP_OK;
}
int dp_graph_serialize(const dp_graph* g, uint8_t* buf, size_t cap, size_t* len) {
  DP_REQUIRE(g && len && (buf || cap == 0));
  return Guard([&] {
    const std::string b = Serialize(g->g);
    *len = b.size();
    if (cap) std::memcpy(buf, b.data(), std::min(cap, b.size()));
  });
}
int dp_graph_deserialize(const dp_registry* reg, const uint8_t* bytes, size_t len, const dp_source* const* sources,
                         int64_t num_sources, int device, dp_graph** out) {
  DP_REQUIRE(reg && out && (bytes || len == 0) && num_sources >= 0 && (sources || num_sources == 0));
  return Guard([&] {
    std::vector<SourcePtr> src;
    for (int64_t i = 0; i < num_sources; ++i) src.push_back(sources[i] ? sources[i]->s : nullptr);
    Emit(out, Deserialize(std::string(reinterpret_cast<const char*>(bytes), len), reg->reg, src, device));
  });
}
int dp_graph_from_spec(dp_registry* reg, const char* text, int device, dp_graph** out, int* epochs, int* has_seed,
                       uint64_t* seed, int* deterministic, char* disabled, size_t len) {
  DP_REQUIRE(reg && text && out);
  return Guard([&] {
    ParsedPipeline p = ParsePipelineSpec(text, reg->reg, device);
    if (epochs) *epochs = p.epochs;
    if (has_seed) *has_seed = p.options.seed_override.has_value() ? 1 : 0;
    if (seed) *seed = p.options.seed_override.value_or(0);
    if (deterministic) *deterministic = p.options.deterministic ? 1 : 0;
    std::string d;
    for (const auto& r : p.disabled_rules) d += (d.empty() ? "" : ",") + r;
    if (disabled) CopyOut(d, disabled, len);
    Emit(out, std::move(p.graph));
  });
}
int dp_graph_fingerprint(const dp_graph* g, char* hex) {
  DP_REQUIRE(g && hex);
  return Guard([&] {
    const std::string h = FingerprintHex(GraphFingerprint(g->g));
    std::memcpy(hex, h.c_str(), h.size() + 1);
  });
}
void dp_graph_release(dp_graph* g) { delete g; }

// ---- iterators ----
void dp_iterator_options_default(dp_iterator_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->deterministic = 1;
}

int dp_iterator_create(const dp_graph* g, const dp_registry* reg, const dp_iterator_options* opt, dp_iterator** out) {
  DP_REQUIRE(g && reg && out);
  return Guard([&] {
    IteratorOptions o;
    if (opt) {
      o.deterministic = opt->deterministic != 0;
      if (opt->has_seed_override) o.seed_override = opt->seed_override;
      o.device = opt->device;
      o.consumer_stream = opt->consumer_stream;
      o.host_output = opt->host_output != 0;
      if (opt->slot_memory_budget) o.slot_memory_budget = opt->slot_memory_budget;
      o.max_launch_bytes = opt->max_launch_bytes;
      o.launch_batches = opt->launch_batches;
      o.first_launch_batches = opt->first_launch_batches;
    }
    *out = new dp_iterator{MakeIterator(g->g, reg->reg, o)};
  });
}

int dp_iterator_get_next(dp_iterator* it, dp_batch* batch) {
  DP_REQUIRE(it && batch);
  std::memset(batch, 0, sizeof(*batch));
  bool eof = false;
  int st = Guard([&] {
    auto e = it->it->GetNext();
    if (!e) {
      eof = true;
      return;
    }
    auto* held = new Element(std::move(*e));
    batch->handle = held;
    batch->num_components = static_cast<int>(std::min<size_t>(held->arity(), 4));
    batch->index = it->it->root_delivered() - 1;
    for (int c = 0; c < batch->num_components; ++c) {
      dp_tensor& d = batch->components[c];
      const Value& v = held->component(c);
      if (v.kind() == Value::Kind::kInt64) {  // unbatched int64 value: a 0-d host tensor
        d.dtype = static_cast<int>(DType::kInt64);
        d.ndim = 0;
        d.data = const_cast<int64_t*>(v.int64_ptr());
        d.on_host = 1;
        continue;
      }
      const Tensor& t = v.tensor();
      d.dtype = static_cast<int>(t.dtype);
      d.ndim = static_cast<int>(std::min<size_t>(t.shape.size(), 6));
      for (int k = 0; k < d.ndim; ++k) d.shape[k] = t.shape[k];
      d.data = t.data;
      d.on_host = t.residency == Residency::kHost;
      batch->ready_event = t.ready;
    }
  });
  if (st != DP_OK) return st;
  if (eof) return dpk::fail(DP_ERR_END_OF_SEQUENCE, "end of sequence");
  return DP_OK;
}

int dp_batch_release(dp_batch* batch) {
  DP_REQUIRE(batch);
  delete static_cast<Element*>(batch->handle);
  batch->handle = nullptr;
  return DP_OK;
}

int dp_iterator_save(const dp_iterator* it, void* buf, size_t cap, size_t* len) {
  DP_REQUIRE(it && len);
  std::string blob;
  int st = Guard([&] { blob = it->it->Save(); });
  if (st != DP_OK) return st;
  *len = blob.size();
  if (!buf || cap < blob.size()) return dpk::fail(DP_ERR_INVALID_ATTR, "checkpoint buffer too small");
  std::memcpy(buf, blob.data(), blob.size());
  return DP_OK;
}

int dp_iterator_restore(const dp_graph* g, const dp_registry* reg, const void* blob, size_t len,
                        const dp_iterator_options* opt, dp_iterator** out) {
  DP_REQUIRE(g && reg && out && (blob || len == 0));
  return Guard([&] {
    IteratorOptions o;
    if (opt) {
      o.device = opt->device;
      o.consumer_stream = opt->consumer_stream;
      o.host_output = opt->host_output != 0;
      if (opt->slot_memory_budget) o.slot_memory_budget = opt->slot_memory_budget;
      o.max_launch_bytes = opt->max_launch_bytes;
      o.launch_batches = opt->launch_batches;
      o.first_launch_batches = opt->first_launch_batches;
    }
    std::string b(static_cast<const char*>(blob), len);
    *out = new dp_iterator{Restore(g->g, reg->reg, b, o)};
  });
}

int dp_iterator_skip(dp_iterator* it, int64_t n, int64_t* produced) {
  DP_REQUIRE(it && produced);
  *produced = 0;
  return Guard([&] {
    for (int64_t i = 0; i < n; ++i) {
      if (!it->it->GetNext()) break;
      ++*produced;
    }
  });
}

int dp_batch_wait(const dp_batch* batch) {
  DP_REQUIRE(batch && batch->handle);
  return Guard([&] {
    if (batch->ready_event) {
      cudaError_t err = cudaEventSynchronize(static_cast<cudaEvent_t>(batch->ready_event));
      if (err != cudaSuccess) throw DeviceError(cudaGetErrorString(err));
    }
  });
}

int dp_tensor_copy_to_host(const dp_batch* batch, int component, void* dst, size_t bytes) {
  DP_REQUIRE(batch && batch->handle && dst);
  return Guard([&] {
    const auto* e = static_cast<const Element*>(batch->handle);
    if (component < 0 || component >= static_cast<int>(e->arity()))
      throw PipelineError(ErrorCode::kInvalidAttr, "component out of range");
    if (e->component(component).kind() == Value::Kind::kInt64) {
      if (bytes < sizeof(int64_t)) throw PipelineError(ErrorCode::kInvalidAttr, "destination too small");
      std::memcpy(dst, e->component(component).int64_ptr(), sizeof(int64_t));
      return;
    }
    const Tensor& t = e->component(component).tensor();
    if (bytes < t.nbytes()) throw PipelineError(ErrorCode::kInvalidAttr, "destination too small");
    if (t.ready) {
      cudaError_t err = cudaEventSynchronize(static_cast<cudaEvent_t>(t.ready));
      if (err != cudaSuccess) throw DeviceError(cudaGetErrorString(err));
    }
    if (t.residency == Residency::kHost) {
      std::memcpy(dst, t.data, t.nbytes());
    } else {
      cudaError_t err = cudaMemcpy(dst, t.data, t.nbytes(), cudaMemcpyDeviceToHost);
      if (err != cudaSuccess) throw DeviceError(cudaGetErrorString(err));
    }
  });
}

void* dp_iterator_stream(const dp_iterator* it) { return it ? it->it->stream() : nullptr; }
int64_t dp_iterator_kernel_launches(const dp_iterator* it) { return it ? it->it->kernel_launches() : 0; }
int64_t dp_iterator_batches_launched(const dp_iterator* it) { return it ? it->it->batches_launched() : 0; }
int dp_iterator_batch_stage_timing(const dp_iterator* it, int64_t* total_ns, int64_t* launches) {
  DP_REQUIRE(it && total_ns && launches);
  return Guard([&] {
    auto [ns, n] = it->it->BatchStageTiming();
    *total_ns = ns;
    *launches = n;
  });
}
int64_t dp_iterator_prefetch_depth(const dp_iterator* it) { return it ? it->it->prefetch_depth() : 0; }
int dp_iterator_get_stats(const dp_iterator* it, dp_iterator_stats* out) {
  DP_REQUIRE(it && out);
  return Guard([&] {
    const auto st = it->it->stats();
    *out = dp_iterator_stats{st.live_plans,    st.slots,
                             st.slot_bytes,    st.prefetch_depth,
                             st.group_batches, st.max_depth,
                             st.producer_groups_per_s, st.consumer_groups_per_s,
                             st.p_empty};
  });
}
int dp_iterator_metrics(const dp_iterator* it, dp_node_metrics* rows, int cap, int* count) {
  DP_REQUIRE(it && count && (rows || cap == 0));
  return Guard([&] {
    const auto m = it->it->Metrics();
    *count = static_cast<int>(m.size());
    for (int i = 0; i < cap && i < static_cast<int>(m.size()); ++i) {
      std::memset(&rows[i], 0, sizeof(rows[i]));
      std::strncpy(rows[i].path, m[i].path.c_str(), sizeof(rows[i].path) - 1);
      std::strncpy(rows[i].label, m[i].label.c_str(), sizeof(rows[i].label) - 1);
      rows[i].self_time_ns = m[i].self_time_ns;
      rows[i].elements_produced = m[i].elements_produced;
    }
  });
}
int64_t dp_iterator_root_delivered(const dp_iterator* it) { return it ? it->it->root_delivered() : 0; }
uint64_t dp_iterator_base_seed(const dp_iterator* it) { return it ? it->it->base_seed() : 0; }
int dp_iterator_describe(const dp_iterator* it, char* buf, size_t len) {
  DP_REQUIRE(it && buf);
  return Guard([&] { CopyOut(it->it->LoweringPlan(), buf, len); });
}
void dp_iterator_destroy(dp_iterator* it) { delete it; }

}  // extern "C"
