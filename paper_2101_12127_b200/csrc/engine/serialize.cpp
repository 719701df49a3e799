// serialize.cpp -- DPG1 graph serialization and the graph fingerprint
// (/root/reference/proj/docs/formats.md "Graph serialization" / "Fingerprint";
// reference src/serialize.cpp Serialize / Deserialize / GraphFingerprint).
//
//   graph := "DPG1" version:u16(=1) node_count:u32 node
//   node  := kind:u8 num_inputs:u8 num_attrs:u8 attr* node*     (preorder)
//   attr  := key:str tag:u8 payload      (ascending key order)
//
// Tags 0-6 are the reference's (int64, uint64, float64, bool, string,
// string list, element list).  Node attrs that hold device data map onto the
// reference encoding where one exists -- from_memory's int64 source is the
// "elements" element list, from_file's source is implied by its "paths" --
// so a graph both engines can build serializes to the same bytes and has the
// same fingerprint.  The remaining device sources (tensor_slices /
// token_sequences data, interleave records) have no reference encoding: tag
// 32 writes a descriptor (kind, count, shape) and Deserialize re-binds the
// caller's sources in preorder.
#include <algorithm>
#include <cstring>

#include "dpb200/datapipe.hpp"

namespace datapipe::b200 {
namespace {

constexpr char kMagic[4] = {'D', 'P', 'G', '1'};
constexpr uint16_t kVersion = 1;
enum Tag : uint8_t {
  kTagInt64 = 0,
  kTagUint64 = 1,
  kTagFloat64 = 2,
  kTagBool = 3,
  kTagString = 4,
  kTagStringList = 5,
  kTagElementList = 6,
  kTagDeviceSource = 32,  // this engine's extensions: a device-source descriptor,
  kTagInt64List = 33,     // an int64 list (bucket_by_length boundaries / sizes)
};

struct Out {
  std::string b;
  template <typename T>
  void Le(T v) {
    uint64_t u;
    if constexpr (std::is_same_v<T, double>) {
      std::memcpy(&u, &v, 8);
    } else {
      u = static_cast<uint64_t>(v);
    }
    for (size_t i = 0; i < sizeof(T); ++i) b.push_back(static_cast<char>((u >> (8 * i)) & 0xff));
  }
  void Str(const std::string& s) {
    Le<uint32_t>(static_cast<uint32_t>(s.size()));
    b += s;
  }
};

struct In {
  const std::string& b;
  size_t pos = 0;
  [[noreturn]] void Bad(const std::string& what) const {
    throw PipelineError(ErrorCode::kMalformedInput, "at byte " + std::to_string(pos) + ": " + what);
  }
  void Need(size_t n) {
    if (pos + n > b.size()) Bad("truncated graph");
  }
  template <typename T>
  T Le() {
    Need(sizeof(T));
    uint64_t u = 0;
    for (size_t i = 0; i < sizeof(T); ++i) u |= static_cast<uint64_t>(static_cast<uint8_t>(b[pos + i])) << (8 * i);
    pos += sizeof(T);
    if constexpr (std::is_same_v<T, double>) {
      double d;
      std::memcpy(&d, &u, 8);
      return d;
    } else {
      return static_cast<T>(u);
    }
  }
  std::string Str() {
    const uint32_t n = Le<uint32_t>();
    Need(n);
    std::string s = b.substr(pos, n);
    pos += n;
    return s;
  }
};

uint32_t CountNodes(const DatasetNode& n) {
  uint32_t c = 1;
  for (const auto& in : n.inputs()) c += CountNodes(*in);
  return c;
}

// The serialized (key, value) list of a node, in ascending key order.
using Item = std::pair<std::string, const AttrValue*>;
std::vector<Item> SerializedAttrs(const DatasetNode& n) {
  std::vector<Item> items;
  for (const auto& [k, v] : n.attrs()) {
    if (k == "source" && n.kind() == NodeKind::kFromFile) continue;  // implied by "paths"
    if (k == "source" && n.kind() == NodeKind::kFromMemory) {
      items.emplace_back("elements", &v);
      continue;
    }
    items.emplace_back(k, &v);
  }
  std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.first < b.first; });
  return items;
}

void EncodeSource(const std::string& key, const SourceData& s, Out& w) {
  if (key == "elements") {  // from_memory: element := arity:u8 value; value := tag 0 (int64) i64
    if (s.host_int64.size() != static_cast<size_t>(s.count))
      throw PipelineError(ErrorCode::kInternal, "from_memory source lost its host values");
    w.Le<uint8_t>(kTagElementList);
    w.Le<uint32_t>(static_cast<uint32_t>(s.count));
    for (int64_t v : s.host_int64) {
      w.Le<uint8_t>(1);
      w.Le<uint8_t>(0);
      w.Le<int64_t>(v);
    }
    return;
  }
  w.Le<uint8_t>(kTagDeviceSource);
  // kind, bit 7 = the images carry labels (a third element component)
  w.Le<uint8_t>(static_cast<uint8_t>(static_cast<uint8_t>(s.kind) | (s.labels ? 0x80 : 0)));
  for (int64_t v : {s.count, s.h, s.w, s.c, s.total_tokens, s.record_len, s.global_count, s.shard_count, s.shard_index,
                    s.shard_block})
    w.Le<int64_t>(v);
}

void EncodeNode(const DatasetNode& n, Out& w, bool zero_seeds) {
  const auto items = SerializedAttrs(n);
  w.Le<uint8_t>(static_cast<uint8_t>(n.kind()));
  w.Le<uint8_t>(static_cast<uint8_t>(n.inputs().size()));
  w.Le<uint8_t>(static_cast<uint8_t>(items.size()));
  for (const auto& [key, value] : items) {
    w.Str(key);
    if (zero_seeds && key == "seed") {
      w.Le<uint8_t>(kTagUint64);
      w.Le<uint64_t>(0);
      continue;
    }
    std::visit(
        [&](const auto& v) {
          using T = std::decay_t<decltype(v)>;
          if constexpr (std::is_same_v<T, int64_t>) {
            w.Le<uint8_t>(kTagInt64);
            w.Le<int64_t>(v);
          } else if constexpr (std::is_same_v<T, uint64_t>) {
            w.Le<uint8_t>(kTagUint64);
            w.Le<uint64_t>(v);
          } else if constexpr (std::is_same_v<T, double>) {
            w.Le<uint8_t>(kTagFloat64);
            w.Le<double>(v);
          } else if constexpr (std::is_same_v<T, bool>) {
            w.Le<uint8_t>(kTagBool);
            w.Le<uint8_t>(v ? 1 : 0);
          } else if constexpr (std::is_same_v<T, std::string>) {
            w.Le<uint8_t>(kTagString);
            w.Str(v);
          } else if constexpr (std::is_same_v<T, std::vector<std::string>>) {
            w.Le<uint8_t>(kTagStringList);
            w.Le<uint32_t>(static_cast<uint32_t>(v.size()));
            for (const auto& s : v) w.Str(s);
          } else if constexpr (std::is_same_v<T, std::vector<int64_t>>) {
            w.Le<uint8_t>(kTagInt64List);
            w.Le<uint32_t>(static_cast<uint32_t>(v.size()));
            for (int64_t x : v) w.Le<int64_t>(x);
          } else {  // SourcePtr
            EncodeSource(key, *v, w);
          }
        },
        *value);
  }
  for (const auto& in : n.inputs()) EncodeNode(*in, w, zero_seeds);
}

std::string SerializeImpl(const DatasetGraph& g, bool zero_seeds) {
  if (!g.root()) throw PipelineError(ErrorCode::kValidationFailed, "empty graph");
  Out w;
  w.b.append(kMagic, 4);
  w.Le<uint16_t>(kVersion);
  w.Le<uint32_t>(CountNodes(*g.root()));
  EncodeNode(*g.root(), w, zero_seeds);
  return std::move(w.b);
}

bool KnownKind(uint8_t k) {
  switch (static_cast<NodeKind>(k)) {
    case NodeKind::kFromMemory:
    case NodeKind::kFromFile:
    case NodeKind::kMap:
    case NodeKind::kFilter:
    case NodeKind::kInterleave:
    case NodeKind::kBatch:
    case NodeKind::kPrefetch:
    case NodeKind::kRepeat:
    case NodeKind::kShuffle:
    case NodeKind::kShard:
    case NodeKind::kMapAndBatch:
    case NodeKind::kRange:
    case NodeKind::kTensorSlices:
    case NodeKind::kTokenSequences:
    case NodeKind::kPaddedBatch:
    case NodeKind::kBucketByLength:
      return true;
  }
  return false;
}

struct Decoder {
  In r;
  const UdfRegistry& reg;
  const std::vector<SourcePtr>& sources;
  int device;
  size_t next_source = 0;
  uint32_t nodes = 0;

  SourcePtr BindSource(In& in) {
    const uint8_t kind_byte = in.Le<uint8_t>();
    const auto kind = static_cast<SourceData::Kind>(kind_byte & 0x7f);
    const bool labels = (kind_byte & 0x80) != 0;
    int64_t d[10];
    for (auto& v : d) v = in.Le<int64_t>();
    if (next_source >= sources.size())
      throw PipelineError(ErrorCode::kValidationFailed,
                          "graph references device source #" + std::to_string(next_source) +
                              ": pass the sources (device data is not serialized)");
    SourcePtr s = sources[next_source++];
    if (!s) throw PipelineError(ErrorCode::kValidationFailed, "null device source");
    const int64_t have[10] = {s->count, s->h, s->w, s->c, s->total_tokens, s->record_len,
                              s->global_count, s->shard_count, s->shard_index, s->shard_block};
    if (s->kind != kind || (s->labels != nullptr) != labels || std::memcmp(d, have, sizeof(d)) != 0)
      throw PipelineError(ErrorCode::kValidationFailed,
                          "device source #" + std::to_string(next_source - 1) + " does not match the serialized one");
    return s;
  }

  AttrValue DecodeAttr(NodeKind kind, const std::string& key, std::string& out_key) {
    out_key = key;
    const size_t at = r.pos;
    const uint8_t tag = r.Le<uint8_t>();
    switch (tag) {
      case kTagInt64:
        return r.Le<int64_t>();
      case kTagUint64:
        return r.Le<uint64_t>();
      case kTagFloat64:
        return r.Le<double>();
      case kTagBool:
        return r.Le<uint8_t>() != 0;
      case kTagString:
        return r.Str();
      case kTagStringList: {
        const uint32_t n = r.Le<uint32_t>();
        std::vector<std::string> v;
        for (uint32_t i = 0; i < n; ++i) v.push_back(r.Str());
        return v;
      }
      case kTagElementList: {
        if (kind != NodeKind::kFromMemory || key != "elements")
          throw PipelineError(ErrorCode::kValidationFailed, "element list attr '" + key + "' is not on the device path");
        const uint32_t n = r.Le<uint32_t>();
        std::vector<int64_t> v;
        v.reserve(n);
        for (uint32_t i = 0; i < n; ++i) {
          const uint8_t arity = r.Le<uint8_t>();
          const uint8_t vt = arity == 1 ? r.Le<uint8_t>() : 0xff;
          if (arity != 1 || vt != 0)
            throw PipelineError(ErrorCode::kValidationFailed,
                                "from_memory elements must be int64 scalars on the device path");
          v.push_back(r.Le<int64_t>());
        }
        out_key = "source";
        return Int64FromHost(v.data(), static_cast<int64_t>(v.size()), device);
      }
      case kTagDeviceSource:
        return BindSource(r);
      case kTagInt64List: {
        const uint32_t n = r.Le<uint32_t>();
        std::vector<int64_t> v;
        for (uint32_t i = 0; i < n; ++i) v.push_back(r.Le<int64_t>());
        return v;
      }
      default:
        r.pos = at;
        r.Bad("unknown attr tag " + std::to_string(tag));
    }
  }

  NodePtr Node() {
    const size_t at = r.pos;
    const uint8_t k = r.Le<uint8_t>();
    if (!KnownKind(k)) {
      if (k <= 16)  // a reference kind off the device path (flat_map, unbatch, zip, ...)
        throw PipelineError(ErrorCode::kValidationFailed,
                            "decoded graph failed validation: node kind " + std::to_string(k) +
                                " is not on the device path");
      r.pos = at;
      r.Bad("unknown node kind " + std::to_string(k));
    }
    const auto kind = static_cast<NodeKind>(k);
    const uint8_t ni = r.Le<uint8_t>(), na = r.Le<uint8_t>();
    Attrs attrs;
    for (uint8_t i = 0; i < na; ++i) {
      std::string key = r.Str(), out_key;
      AttrValue v = DecodeAttr(kind, key, out_key);
      attrs.emplace(std::move(out_key), std::move(v));
    }
    if (kind == NodeKind::kFromFile) {  // the records are re-read from "paths"
      auto p = attrs.find("paths");
      if (p == attrs.end() || !std::holds_alternative<std::vector<std::string>>(p->second))
        throw PipelineError(ErrorCode::kValidationFailed, "decoded graph failed validation: from_file needs 'paths'");
      attrs["source"] = RecordsFromFiles(std::get<std::vector<std::string>>(p->second), device);
    }
    std::vector<NodePtr> inputs;
    for (uint8_t i = 0; i < ni; ++i) inputs.push_back(Node());
    ++nodes;
    try {
      return Build(kind, std::move(inputs), std::move(attrs), reg);
    } catch (const PipelineError& e) {
      if (e.code() == ErrorCode::kUnknownUdf) throw;
      throw PipelineError(ErrorCode::kValidationFailed, std::string("decoded graph failed validation: ") + e.what());
    }
  }
};

}  // namespace

std::string Serialize(const DatasetGraph& graph) { return SerializeImpl(graph, false); }

DatasetGraph Deserialize(const std::string& bytes, const UdfRegistry& registry, const std::vector<SourcePtr>& sources,
                         int device) {
  if (bytes.size() < 4 || bytes.compare(0, 4, kMagic, 4) != 0)
    throw PipelineError(ErrorCode::kMalformedInput, "at byte 0: bad magic");
  Decoder d{In{bytes, 4}, registry, sources, device};
  const uint16_t version = d.r.Le<uint16_t>();
  if (version != kVersion)
    throw PipelineError(ErrorCode::kVersionMismatch, "unsupported graph format version " + std::to_string(version));
  const uint32_t declared = d.r.Le<uint32_t>();
  NodePtr root = d.Node();
  if (d.nodes != declared)
    d.r.Bad("node count mismatch: header says " + std::to_string(declared) + ", decoded " + std::to_string(d.nodes));
  if (d.r.pos != bytes.size()) d.r.Bad("trailing bytes");
  return DatasetGraph(std::move(root));
}

std::array<uint8_t, 32> GraphFingerprint(const DatasetGraph& graph) {
  const std::string s = SerializeImpl(graph, true);
  return Sha256Digest(s.data(), s.size());
}

}  // namespace datapipe::b200
