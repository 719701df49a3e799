// graph.cpp -- graph IR, attribute validation, output-spec derivation, the
// ops:: builders and the UDF registry (include/dpb200/datapipe.hpp).
//
// Validation and spec rules follow the reference (graph.cpp:159-378 there):
// batch wraps every component and its leading length is static only with
// drop_remainder (BatchWrapSpec, graph.cpp:159-170); AUTOTUNE (-1) is legal
// for num_parallel_calls / buffer_size; shard index in [0, num_shards).
#include <algorithm>
#include <functional>
#include <sstream>

#include "dpb200/datapipe.hpp"

namespace datapipe::b200 {

const char* NodeKindName(NodeKind kind) {
  switch (kind) {
    case NodeKind::kFromMemory: return "from_memory";
    case NodeKind::kFromFile: return "from_file";
    case NodeKind::kMap: return "map";
    case NodeKind::kFilter: return "filter";
    case NodeKind::kInterleave: return "interleave";
    case NodeKind::kBatch: return "batch";
    case NodeKind::kPrefetch: return "prefetch";
    case NodeKind::kRepeat: return "repeat";
    case NodeKind::kShuffle: return "shuffle";
    case NodeKind::kShard: return "shard";
    case NodeKind::kMapAndBatch: return "map_and_batch";
    case NodeKind::kRange: return "range";
    case NodeKind::kTensorSlices: return "tensor_slices";
    case NodeKind::kTokenSequences: return "token_sequences";
    case NodeKind::kPaddedBatch: return "padded_batch";
    case NodeKind::kBucketByLength: return "bucket_by_length";
  }
  return "?";
}

// random.hpp:24-34
uint64_t MixSeeds(uint64_t a, uint64_t b) {
  uint64_t s = a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2));
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// runtime.cpp:713-718
uint64_t ShuffleEngineSeed(uint64_t epoch_salt, std::optional<uint64_t> attr_seed) {
  return MixSeeds(epoch_salt, attr_seed.value_or(0x9d2c5680u));
}

// ------------------------------------------------------------ node attrs --
namespace {
[[noreturn]] void BadAttr(NodeKind k, const std::string& msg) {
  throw PipelineError(ErrorCode::kInvalidAttr, std::string(NodeKindName(k)) + ": " + msg);
}
PipelineError TypeMismatchError(const std::string& what, const ElementSpec& got) {
  return PipelineError(ErrorCode::kTypeMismatch, what + ", got " + got.ToString());
}
}  // namespace

int64_t DatasetNode::GetInt(const std::string& k) const {
  auto it = attrs_.find(k);
  if (it == attrs_.end() || !std::holds_alternative<int64_t>(it->second)) BadAttr(kind_, "missing int attr " + k);
  return std::get<int64_t>(it->second);
}
int64_t DatasetNode::GetIntOr(const std::string& k, int64_t fallback) const { return HasAttr(k) ? GetInt(k) : fallback; }
uint64_t DatasetNode::GetUint(const std::string& k) const {
  auto it = attrs_.find(k);
  if (it == attrs_.end() || !std::holds_alternative<uint64_t>(it->second)) BadAttr(kind_, "missing uint attr " + k);
  return std::get<uint64_t>(it->second);
}
bool DatasetNode::GetBoolOr(const std::string& k, bool fallback) const {
  auto it = attrs_.find(k);
  if (it == attrs_.end()) return fallback;
  if (!std::holds_alternative<bool>(it->second)) BadAttr(kind_, k + " must be a bool");
  return std::get<bool>(it->second);
}
const std::string& DatasetNode::GetString(const std::string& k) const {
  auto it = attrs_.find(k);
  if (it == attrs_.end() || !std::holds_alternative<std::string>(it->second)) BadAttr(kind_, "missing string attr " + k);
  return std::get<std::string>(it->second);
}
const SourcePtr& DatasetNode::GetSource(const std::string& k) const {
  auto it = attrs_.find(k);
  if (it == attrs_.end() || !std::holds_alternative<SourcePtr>(it->second)) BadAttr(kind_, "missing source attr " + k);
  return std::get<SourcePtr>(it->second);
}

std::string DatasetGraph::ToString() const {
  std::ostringstream os;
  std::function<void(const DatasetNode&, int)> walk = [&](const DatasetNode& n, int depth) {
    os << std::string(2 * depth, ' ') << NodeKindName(n.kind());
    for (const auto& [k, v] : n.attrs()) {
      os << " " << k << "=";
      std::visit(
          [&](const auto& x) {
            using T = std::decay_t<decltype(x)>;
            if constexpr (std::is_same_v<T, SourcePtr>) os << "<source " << (x ? x->count : 0) << ">";
            else if constexpr (std::is_same_v<T, std::vector<std::string>>) os << "[" << x.size() << "]";
            else if constexpr (std::is_same_v<T, std::vector<int64_t>>) {
              os << "[";
              for (size_t i = 0; i < x.size(); ++i) os << (i ? "," : "") << x[i];
              os << "]";
            } else os << x;
          },
          v);
    }
    os << " : " << n.output_spec().ToString() << "\n";
    for (const auto& in : n.inputs()) walk(*in, depth + 1);
  };
  if (root_) walk(*root_, 0);
  return os.str();
}

// ------------------------------------------------------------ UDF registry --
void UdfRegistry::Register(const std::string& name, Entry entry) {
  std::lock_guard lock(mu_);
  if (entries_.count(name)) throw PipelineError(ErrorCode::kDuplicateName, "UDF already registered: " + name);
  entries_[name] = std::make_unique<Entry>(std::move(entry));
}

void UdfRegistry::RegisterAffine(const std::string& name, int64_t a, int64_t b) {
  Entry e;
  MapStep s{MapStep::Op::kAffine};
  s.a = a;
  s.b = b;
  e.map.push_back(s);
  Register(name, std::move(e));
}

void UdfRegistry::RegisterRandomCropFlip(const std::string& name, int64_t crop_h, int64_t crop_w, uint64_t seed,
                                         bool flip) {
  if (crop_h < 1 || crop_w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "crop size must be >= 1");
  Entry e;
  MapStep s{MapStep::Op::kRandomCropFlip};
  s.out_h = crop_h;
  s.out_w = crop_w;
  s.seed = seed;
  s.flip = flip;
  e.map.push_back(s);
  Register(name, std::move(e));
}

void UdfRegistry::RegisterResizeBilinear(const std::string& name, int64_t out_h, int64_t out_w) {
  if (out_h < 1 || out_w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "resize size must be >= 1");
  Entry e;
  MapStep s{MapStep::Op::kResizeBilinear};
  s.out_h = out_h;
  s.out_w = out_w;
  e.map.push_back(s);
  Register(name, std::move(e));
}

void UdfRegistry::RegisterNormalize(const std::string& name, std::array<float, 3> mean, std::array<float, 3> stdv) {
  Entry e;
  MapStep s{MapStep::Op::kNormalize};
  s.mean = mean;
  s.stdv = stdv;
  e.map.push_back(s);
  Register(name, std::move(e));
}

void UdfRegistry::RegisterCast(const std::string& name) { RegisterNormalize(name, {0.f, 0.f, 0.f}, {1.f, 1.f, 1.f}); }

void UdfRegistry::RegisterCenterCrop(const std::string& name, int64_t crop_h, int64_t crop_w) {
  if (crop_h < 1 || crop_w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "crop size must be >= 1");
  Entry e;
  MapStep s{MapStep::Op::kCenterCrop};
  s.out_h = crop_h;
  s.out_w = crop_w;
  s.flip = false;
  e.map.push_back(s);
  Register(name, std::move(e));
}

void UdfRegistry::RegisterImageAffine(const std::string& name, std::array<float, 3> scale,
                                      std::array<float, 3> shift) {
  Entry e;
  MapStep s{MapStep::Op::kImageAffine};
  s.scale = scale;
  s.shift = shift;
  e.map.push_back(s);
  Register(name, std::move(e));
}

void UdfRegistry::RegisterDecodeRaw(const std::string& name, int64_t h, int64_t w) {
  if (h < 1 || w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "decode_raw: shape must be >= 1");
  Entry e;
  MapStep s{MapStep::Op::kDecodeRaw};
  s.out_h = h;
  s.out_w = w;
  e.map.push_back(s);
  Register(name, std::move(e));
}

int64_t DevicePredicate::MaxLen() const {
  int64_t m = INT64_MAX;
  for (const auto& t : terms)
    if (t.op == PredicateTerm::Op::kLE) m = std::min(m, t.a);
  return m;
}

void UdfRegistry::RegisterLengthFilter(const std::string& name, int64_t max_len) {
  Entry e;
  e.predicate = DevicePredicate{DevicePredicate::On::kLength, {{PredicateTerm::Op::kLE, max_len, 0}}};
  Register(name, std::move(e));
}

void UdfRegistry::RegisterValueFilter(const std::string& name, std::vector<PredicateTerm> terms) {
  if (terms.empty() || terms.size() > 8)
    throw PipelineError(ErrorCode::kInvalidAttr, "value filter: 1..8 terms");
  for (const auto& t : terms)
    if ((t.op == PredicateTerm::Op::kModEq || t.op == PredicateTerm::Op::kModNe) && t.a == 0)
      throw PipelineError(ErrorCode::kInvalidAttr, "value filter: modulus must be non-zero");
  Entry e;
  e.predicate = DevicePredicate{DevicePredicate::On::kValue, std::move(terms)};
  Register(name, std::move(e));
}

void UdfRegistry::RegisterStandardPredicates() {
  if (Contains("keep_even")) return;
  RegisterValueFilter("keep_even", {{PredicateTerm::Op::kModEq, 2, 0}});
  RegisterValueFilter("keep_odd", {{PredicateTerm::Op::kModNe, 2, 0}});
  RegisterValueFilter("keep_all", {{PredicateTerm::Op::kGE, INT64_MIN, 0}});
}

void UdfRegistry::RegisterRecordReader(const std::string& name, int64_t records) {
  if (records < 0) throw PipelineError(ErrorCode::kInvalidAttr, "records must be >= 0");
  Entry e;
  e.reader = RecordReader{records};
  Register(name, std::move(e));
}

bool UdfRegistry::Contains(const std::string& name) const {
  std::lock_guard lock(mu_);
  return entries_.count(name) > 0;
}

const UdfRegistry::Entry& UdfRegistry::Get(const std::string& name) const {
  std::lock_guard lock(mu_);
  auto it = entries_.find(name);
  if (it == entries_.end()) throw PipelineError(ErrorCode::kUnknownUdf, "UDF not registered: " + name);
  return *it->second;
}

ElementSpec ApplyMapSteps(const std::vector<MapStep>& steps, const ElementSpec& in) {
  ElementSpec cur = in;
  // (int64 id, tensor[h, w, 3]) or (int64 id, tensor[h, w, 3], int64 label):
  // image maps transform the tensor and pass the other components through
  auto image_spec = [&](const char* what) -> const TypeSpec& {
    if ((cur.arity() != 2 && cur.arity() != 3) || cur.components()[0].kind() != Value::Kind::kInt64 ||
        cur.components()[1].kind() != Value::Kind::kTensor || cur.components()[1].shape().size() != 3 ||
        cur.components()[1].shape()[2] != 3 ||
        (cur.arity() == 3 && cur.components()[2].kind() != Value::Kind::kInt64))
      throw TypeMismatchError(what, cur);
    return cur.components()[1];
  };
  auto with_image = [&](TypeSpec t) {
    std::vector<TypeSpec> c{TypeSpec::Int64(), std::move(t)};
    if (cur.arity() == 3) c.push_back(TypeSpec::Int64());
    return ElementSpec(std::move(c));
  };
  for (const auto& s : steps) {
    switch (s.op) {
      case MapStep::Op::kAffine:
        if (cur.arity() != 1 || cur.components()[0].kind() != Value::Kind::kInt64)
          throw TypeMismatchError("affine expects (int64)", cur);
        break;
      case MapStep::Op::kRandomCropFlip: {
        const TypeSpec& t = image_spec("random_crop expects (int64 id, tensor[h,w,3])");
        if (t.shape()[0] < s.out_h || t.shape()[1] < s.out_w)
          throw PipelineError(ErrorCode::kTypeMismatch, "random_crop: crop larger than the image");
        cur = with_image(TypeSpec::OfTensor(t.dtype(), {s.out_h, s.out_w, 3}));
        break;
      }
      case MapStep::Op::kCenterCrop: {
        const TypeSpec& t = image_spec("center_crop expects (int64 id, tensor[h,w,3])");
        if (t.shape()[0] < s.out_h || t.shape()[1] < s.out_w)
          throw PipelineError(ErrorCode::kTypeMismatch, "center_crop: crop larger than the image");
        cur = with_image(TypeSpec::OfTensor(t.dtype(), {s.out_h, s.out_w, 3}));
        break;
      }
      case MapStep::Op::kResizeBilinear: {
        image_spec("resize expects (int64 id, tensor[h,w,3])");
        cur = with_image(TypeSpec::OfTensor(DType::kFloat32, {s.out_h, s.out_w, 3}));
        break;
      }
      case MapStep::Op::kImageAffine: {
        const TypeSpec& t = image_spec("image affine expects (int64 id, tensor[h,w,3])");
        cur = with_image(TypeSpec::OfTensor(DType::kFloat32, t.shape()));
        break;
      }
      case MapStep::Op::kDecodeRaw:
        if (cur.arity() != 1 || cur.components()[0].kind() != Value::Kind::kBytes)
          throw TypeMismatchError("decode_raw expects (bytes) records", cur);
        cur = ElementSpec({TypeSpec::Int64(), TypeSpec::OfTensor(DType::kUInt8, {s.out_h, s.out_w, 3})});
        break;
      case MapStep::Op::kNormalize: {
        const TypeSpec& t = image_spec("normalize expects (int64 id, tensor[h,w,3])");
        cur = with_image(TypeSpec::OfTensor(DType::kFloat32, t.shape()));
        break;
      }
    }
  }
  return cur;
}

ElementSpec UdfRegistry::MapOutputSpec(const std::string& name, const ElementSpec& in) const {
  if (!Contains(name)) return in;  // identity when unregistered (udf.cpp:89-95)
  return ApplyMapSteps(Get(name).map, in);
}

// -------------------------------------------------------------------- Build --
namespace {

int64_t RequireInt(NodeKind k, const Attrs& a, const std::string& key) {
  auto it = a.find(key);
  if (it == a.end() || !std::holds_alternative<int64_t>(it->second)) BadAttr(k, "'" + key + "' must be an int");
  return std::get<int64_t>(it->second);
}

void RequireString(NodeKind k, const Attrs& a, const std::string& key) {
  auto it = a.find(key);
  if (it == a.end() || !std::holds_alternative<std::string>(it->second)) BadAttr(k, "'" + key + "' must be a string");
}

void CheckKeys(NodeKind k, const Attrs& a, std::initializer_list<const char*> required,
               std::initializer_list<const char*> optional) {
  for (const char* r : required)
    if (!a.count(r)) BadAttr(k, std::string("missing attr '") + r + "'");
  for (const auto& [key, v] : a) {
    bool ok = std::any_of(required.begin(), required.end(), [&](const char* r) { return key == r; }) ||
              std::any_of(optional.begin(), optional.end(), [&](const char* r) { return key == r; });
    if (!ok) BadAttr(k, "unknown attr '" + key + "'");
  }
}

void CheckTunable(NodeKind k, const Attrs& a, const std::string& key) {
  int64_t v = RequireInt(k, a, key);
  if (v != kAutotune && v < 1) BadAttr(k, key + " must be >= 1 or AUTOTUNE");
}

TypeSpec BatchWrap(const TypeSpec& c, std::optional<int64_t> len) {
  int64_t n = len ? *len : -1;
  if (c.kind() == Value::Kind::kInt64) return TypeSpec::OfTensor(DType::kInt64, {n});
  if (c.kind() == Value::Kind::kTensor) {
    std::vector<int64_t> shape{n};
    shape.insert(shape.end(), c.shape().begin(), c.shape().end());
    return TypeSpec::OfTensor(c.dtype(), shape);
  }
  return TypeSpec::List(c, len ? std::optional<uint64_t>(*len) : std::nullopt);
}

// A batch of variable-length 1-D tensors (token sequences) is ragged: the
// reference's list of lists (runtime.cpp:579-637) becomes two components,
// the rows' values back to back and int64 row splits (rows + 1).
ElementSpec BatchWrapSpec(const ElementSpec& in, int64_t b, bool drop) {
  std::vector<TypeSpec> out;
  for (const auto& c : in.components()) {
    if (c.kind() == Value::Kind::kTensor && c.shape().size() == 1 && c.shape()[0] < 0) {
      out.push_back(TypeSpec::OfTensor(c.dtype(), {-1}));
      out.push_back(TypeSpec::OfTensor(DType::kInt64, {drop ? b + 1 : -1}));
      continue;
    }
    out.push_back(BatchWrap(c, drop ? std::optional<int64_t>(b) : std::nullopt));
  }
  return ElementSpec(std::move(out));
}

ElementSpec SourceSpec(const SourceData& s) {
  switch (s.kind) {
    case SourceData::Kind::kInt64: return ElementSpec({TypeSpec::Int64()});
    case SourceData::Kind::kImages:
      if (s.labels)
        return ElementSpec(
            {TypeSpec::Int64(), TypeSpec::OfTensor(DType::kUInt8, {s.h, s.w, s.c}), TypeSpec::Int64()});
      return ElementSpec({TypeSpec::Int64(), TypeSpec::OfTensor(DType::kUInt8, {s.h, s.w, s.c})});
    case SourceData::Kind::kTokens: return ElementSpec({TypeSpec::OfTensor(DType::kInt32, {-1})});
    case SourceData::Kind::kRecords: return ElementSpec({TypeSpec::Bytes()});
  }
  return ElementSpec();
}

void ValidateAttrs(NodeKind kind, const Attrs& a) {
  switch (kind) {
    case NodeKind::kRange:
      CheckKeys(kind, a, {"count"}, {});
      if (RequireInt(kind, a, "count") < 0) BadAttr(kind, "count must be >= 0");
      break;
    case NodeKind::kFromMemory:
    case NodeKind::kFromFile:
    case NodeKind::kTensorSlices:
    case NodeKind::kTokenSequences: {
      if (kind == NodeKind::kFromFile) {
        CheckKeys(kind, a, {"source", "paths"}, {});
        auto p = a.find("paths");
        if (!std::holds_alternative<std::vector<std::string>>(p->second) ||
            std::get<std::vector<std::string>>(p->second).empty())
          BadAttr(kind, "'paths' must be a non-empty list of strings");
      } else {
        CheckKeys(kind, a, {"source"}, {});
      }
      auto it = a.find("source");
      if (!std::holds_alternative<SourcePtr>(it->second) || !std::get<SourcePtr>(it->second))
        BadAttr(kind, "'source' must be a source");
      if (std::get<SourcePtr>(it->second)->count < 1 && kind == NodeKind::kFromMemory)
        BadAttr(kind, "'elements' must be non-empty");
      break;
    }
    case NodeKind::kMap:
      CheckKeys(kind, a, {"udf", "num_parallel_calls"}, {"fused_filter_udf"});
      RequireString(kind, a, "udf");
      CheckTunable(kind, a, "num_parallel_calls");
      if (a.count("fused_filter_udf")) RequireString(kind, a, "fused_filter_udf");
      break;
    case NodeKind::kFilter:
      CheckKeys(kind, a, {"udf"}, {});
      RequireString(kind, a, "udf");
      break;
    case NodeKind::kInterleave: {
      CheckKeys(kind, a, {"udf", "cycle_length", "num_parallel_calls"}, {"records"});
      RequireString(kind, a, "udf");
      int64_t cycle = RequireInt(kind, a, "cycle_length");
      if (cycle < 1) BadAttr(kind, "cycle_length must be >= 1");
      int64_t p = RequireInt(kind, a, "num_parallel_calls");
      if (p != kAutotune && (p < 1 || p > cycle)) BadAttr(kind, "num_parallel_calls must be in [1, cycle_length]");
      break;
    }
    case NodeKind::kBatch:
      CheckKeys(kind, a, {"batch_size"}, {"drop_remainder"});
      if (RequireInt(kind, a, "batch_size") < 1) BadAttr(kind, "batch_size must be >= 1");
      break;
    case NodeKind::kPaddedBatch:
      CheckKeys(kind, a, {"batch_size", "padding_value"}, {"drop_remainder"});
      if (RequireInt(kind, a, "batch_size") < 1) BadAttr(kind, "batch_size must be >= 1");
      RequireInt(kind, a, "padding_value");
      break;
    case NodeKind::kBucketByLength: {
      CheckKeys(kind, a, {"bucket_boundaries", "bucket_batch_sizes", "padding_value"}, {"drop_remainder"});
      RequireInt(kind, a, "padding_value");
      auto ints = [&](const char* k) -> const std::vector<int64_t>& {
        const auto& v = a.at(k);
        if (!std::holds_alternative<std::vector<int64_t>>(v)) BadAttr(kind, std::string("'") + k + "' must be an int list");
        return std::get<std::vector<int64_t>>(v);
      };
      const auto& bounds = ints("bucket_boundaries");
      const auto& sizes = ints("bucket_batch_sizes");
      if (bounds.size() > 31) BadAttr(kind, "at most 31 boundaries (32 buckets)");
      if (sizes.size() != bounds.size() + 1) BadAttr(kind, "bucket_batch_sizes needs one entry per bucket");
      for (size_t k = 0; k < bounds.size(); ++k)
        if (bounds[k] < 0 || bounds[k] > INT32_MAX || (k && bounds[k] <= bounds[k - 1]))
          BadAttr(kind, "bucket_boundaries must be increasing non-negative int32");
      for (int64_t b : sizes)
        if (b < 1 || b > INT32_MAX) BadAttr(kind, "bucket batch sizes must be in [1, 2^31)");
      break;
    }
    case NodeKind::kMapAndBatch:
      CheckKeys(kind, a, {"udf", "batch_size", "num_parallel_calls"}, {"drop_remainder"});
      RequireString(kind, a, "udf");
      if (RequireInt(kind, a, "batch_size") < 1) BadAttr(kind, "batch_size must be >= 1");
      CheckTunable(kind, a, "num_parallel_calls");
      break;
    case NodeKind::kPrefetch:
      CheckKeys(kind, a, {"buffer_size"}, {});
      CheckTunable(kind, a, "buffer_size");
      break;
    case NodeKind::kRepeat: {
      CheckKeys(kind, a, {"count"}, {});
      int64_t c = RequireInt(kind, a, "count");
      if (c != kInfiniteRepeat && c < 1) BadAttr(kind, "count must be >= 1 or INFINITE");
      break;
    }
    case NodeKind::kShuffle:
      CheckKeys(kind, a, {"buffer_size"}, {"seed", "fused_with_repeat"});
      if (RequireInt(kind, a, "buffer_size") < 1) BadAttr(kind, "buffer_size must be >= 1");
      if (a.count("seed") && !std::holds_alternative<uint64_t>(a.at("seed"))) BadAttr(kind, "seed must be unsigned");
      if (a.count("fused_with_repeat") && !std::holds_alternative<bool>(a.at("fused_with_repeat")))
        BadAttr(kind, "fused_with_repeat must be a bool");
      break;
    case NodeKind::kShard: {
      CheckKeys(kind, a, {"num_shards", "index"}, {});
      int64_t k = RequireInt(kind, a, "num_shards"), i = RequireInt(kind, a, "index");
      if (k < 1) BadAttr(kind, "num_shards must be >= 1");
      if (i < 0 || i >= k) BadAttr(kind, "index must be in [0, num_shards)");
      break;
    }
  }
}

int Arity(NodeKind kind) {
  switch (kind) {
    case NodeKind::kRange:
    case NodeKind::kFromMemory:
    case NodeKind::kFromFile:
    case NodeKind::kTensorSlices:
    case NodeKind::kTokenSequences:
      return 0;
    default:
      return 1;
  }
}

bool GetBool(const Attrs& a, const char* key) {
  auto it = a.find(key);
  return it != a.end() && std::get<bool>(it->second);
}

ElementSpec DeriveSpec(NodeKind kind, const std::vector<NodePtr>& in, const Attrs& a, const UdfRegistry& reg) {
  switch (kind) {
    case NodeKind::kRange: return ElementSpec({TypeSpec::Int64()});
    case NodeKind::kFromMemory:
    case NodeKind::kFromFile:
    case NodeKind::kTensorSlices:
    case NodeKind::kTokenSequences: return SourceSpec(*std::get<SourcePtr>(a.at("source")));
    case NodeKind::kMap: return reg.MapOutputSpec(std::get<std::string>(a.at("udf")), in[0]->output_spec());
    case NodeKind::kFilter:
    case NodeKind::kPrefetch:
    case NodeKind::kRepeat:
    case NodeKind::kShuffle:
    case NodeKind::kShard: return in[0]->output_spec();
    case NodeKind::kInterleave: {
      const auto& udf = std::get<std::string>(a.at("udf"));
      const auto& e = reg.Get(udf);
      if (!e.reader) BadAttr(kind, "UDF '" + udf + "' is not a record reader");
      if (in[0]->output_spec() != ElementSpec({TypeSpec::Int64()}))
        throw PipelineError(ErrorCode::kTypeMismatch, "interleave: input must be (int64) source ordinals");
      auto it = a.find("records");
      if (it != a.end()) return SourceSpec(*std::get<SourcePtr>(it->second));
      return ElementSpec({TypeSpec::Int64()});
    }
    case NodeKind::kBatch:
      return BatchWrapSpec(in[0]->output_spec(), std::get<int64_t>(a.at("batch_size")), GetBool(a, "drop_remainder"));
    case NodeKind::kPaddedBatch: {
      const auto& s = in[0]->output_spec();
      if (s.arity() != 1 || s.components()[0].kind() != Value::Kind::kTensor || s.components()[0].shape().size() != 1)
        throw PipelineError(ErrorCode::kTypeMismatch, "padded_batch expects (tensor[?]) sequences");
      int64_t n = GetBool(a, "drop_remainder") ? std::get<int64_t>(a.at("batch_size")) : -1;
      return ElementSpec({TypeSpec::OfTensor(s.components()[0].dtype(), {n, -1}), TypeSpec::OfTensor(DType::kInt32, {n})});
    }
    case NodeKind::kBucketByLength: {
      const auto& s = in[0]->output_spec();
      if (s.arity() != 1 || s.components()[0].kind() != Value::Kind::kTensor || s.components()[0].shape().size() != 1)
        throw PipelineError(ErrorCode::kTypeMismatch, "bucket_by_length expects (tensor[?]) sequences");
      return ElementSpec({TypeSpec::OfTensor(s.components()[0].dtype(), {-1, -1}), TypeSpec::OfTensor(DType::kInt32, {-1})});
    }
    case NodeKind::kMapAndBatch: {
      ElementSpec mapped = reg.MapOutputSpec(std::get<std::string>(a.at("udf")), in[0]->output_spec());
      return BatchWrapSpec(mapped, std::get<int64_t>(a.at("batch_size")), GetBool(a, "drop_remainder"));
    }
  }
  throw PipelineError(ErrorCode::kInternal, "unhandled node kind");
}

}  // namespace

NodePtr Build(NodeKind kind, std::vector<NodePtr> inputs, Attrs attrs, const UdfRegistry& reg) {
  if (static_cast<int>(inputs.size()) != Arity(kind))
    throw PipelineError(ErrorCode::kInvalidArity, std::string(NodeKindName(kind)) + ": expected " +
                                                      std::to_string(Arity(kind)) + " inputs, got " +
                                                      std::to_string(inputs.size()));
  for (const auto& in : inputs)
    if (!in) throw PipelineError(ErrorCode::kInvalidArity, "null input node");
  ValidateAttrs(kind, attrs);
  ElementSpec spec = DeriveSpec(kind, inputs, attrs, reg);
  return std::make_shared<const DatasetNode>(kind, std::move(inputs), std::move(attrs), std::move(spec));
}

namespace ops {

DatasetGraph Range(int64_t n, const UdfRegistry& reg) {
  return DatasetGraph(Build(NodeKind::kRange, {}, {{"count", n}}, reg));
}
DatasetGraph FromMemory(const std::vector<int64_t>& values, const UdfRegistry& reg, int device) {
  return DatasetGraph(Build(NodeKind::kFromMemory, {},
                            {{"source", Int64FromHost(values.data(), static_cast<int64_t>(values.size()), device)}}, reg));
}
DatasetGraph FromFile(const std::vector<std::string>& paths, const UdfRegistry& reg, int device) {
  return DatasetGraph(Build(NodeKind::kFromFile, {}, {{"source", RecordsFromFiles(paths, device)}, {"paths", paths}}, reg));
}
DatasetGraph TensorSlices(SourcePtr images, const UdfRegistry& reg) {
  if (!images || images->kind != SourceData::Kind::kImages)
    throw PipelineError(ErrorCode::kInvalidAttr, "tensor_slices: source must be an image tensor");
  return DatasetGraph(Build(NodeKind::kTensorSlices, {}, {{"source", std::move(images)}}, reg));
}
DatasetGraph TokenSequences(SourcePtr tokens, const UdfRegistry& reg) {
  if (!tokens || tokens->kind != SourceData::Kind::kTokens)
    throw PipelineError(ErrorCode::kInvalidAttr, "token_sequences: source must be token sequences");
  return DatasetGraph(Build(NodeKind::kTokenSequences, {}, {{"source", std::move(tokens)}}, reg));
}
DatasetGraph Map(const DatasetGraph& in, const std::string& udf, int64_t p, const UdfRegistry& reg) {
  return DatasetGraph(Build(NodeKind::kMap, {in.root()}, {{"udf", udf}, {"num_parallel_calls", p}}, reg));
}
DatasetGraph Filter(const DatasetGraph& in, const std::string& udf, const UdfRegistry& reg) {
  return DatasetGraph(Build(NodeKind::kFilter, {in.root()}, {{"udf", udf}}, reg));
}
DatasetGraph Interleave(const DatasetGraph& in, const std::string& udf, int64_t cycle, int64_t p, SourcePtr records,
                        const UdfRegistry& reg) {
  Attrs a{{"udf", udf}, {"cycle_length", cycle}, {"num_parallel_calls", p}};
  if (records) a["records"] = std::move(records);
  return DatasetGraph(Build(NodeKind::kInterleave, {in.root()}, std::move(a), reg));
}
DatasetGraph Batch(const DatasetGraph& in, int64_t b, bool drop, const UdfRegistry& reg) {
  Attrs a{{"batch_size", b}};
  if (drop) a["drop_remainder"] = true;
  return DatasetGraph(Build(NodeKind::kBatch, {in.root()}, std::move(a), reg));
}
DatasetGraph PaddedBatch(const DatasetGraph& in, int64_t b, int64_t pad, bool drop, const UdfRegistry& reg) {
  Attrs a{{"batch_size", b}, {"padding_value", pad}};
  if (drop) a["drop_remainder"] = true;
  return DatasetGraph(Build(NodeKind::kPaddedBatch, {in.root()}, std::move(a), reg));
}
DatasetGraph BucketByLength(const DatasetGraph& in, const std::vector<int64_t>& boundaries,
                            const std::vector<int64_t>& batch_sizes, int64_t pad, bool drop, const UdfRegistry& reg) {
  Attrs a{{"bucket_boundaries", boundaries}, {"bucket_batch_sizes", batch_sizes}, {"padding_value", pad}};
  if (drop) a["drop_remainder"] = true;
  return DatasetGraph(Build(NodeKind::kBucketByLength, {in.root()}, std::move(a), reg));
}
DatasetGraph Prefetch(const DatasetGraph& in, int64_t buffer_size, const UdfRegistry& reg) {
  return DatasetGraph(Build(NodeKind::kPrefetch, {in.root()}, {{"buffer_size", buffer_size}}, reg));
}
DatasetGraph Repeat(const DatasetGraph& in, int64_t count, const UdfRegistry& reg) {
  return DatasetGraph(Build(NodeKind::kRepeat, {in.root()}, {{"count", count}}, reg));
}
DatasetGraph Shuffle(const DatasetGraph& in, int64_t buffer_size, std::optional<uint64_t> seed,
                     const UdfRegistry& reg) {
  Attrs a{{"buffer_size", buffer_size}};
  if (seed) a["seed"] = *seed;
  return DatasetGraph(Build(NodeKind::kShuffle, {in.root()}, std::move(a), reg));
}
DatasetGraph Shard(const DatasetGraph& in, int64_t k, int64_t i, const UdfRegistry& reg) {
  return DatasetGraph(Build(NodeKind::kShard, {in.root()}, {{"num_shards", k}, {"index", i}}, reg));
}

}  // namespace ops
}  // namespace datapipe::b200
