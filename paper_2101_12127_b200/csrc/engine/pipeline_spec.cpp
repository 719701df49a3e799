// pipeline_spec.cpp -- the reference's line-oriented pipeline description
// (docs/formats.md "Pipeline description text format"; reference
// src/pipeline_spec.cpp ParsePipelineSpec) for DEVICE pipelines.
//
// The reference's stanzas model host work (`map work_ms=...`, sleep/busy
// sources), which has no device meaning; here the same stanza grammar --
// `#` comments, one `source` first, ops applied in order, trailers, AUTO for
// tunables, `ParseError` with line and column -- describes the device UDF
// library instead:
//
//   source range count=<n>
//   source memory values=<v1,v2,...>
//   source images count=<n> h=<h> w=<w> [seed=<s>]
//   source tokens count=<n> max_len=<m> [seed=<s>]
//   source file path=<p> [path=<p> ...]
//   map affine a=<a> b=<b> [parallel=<n>|AUTO]
//   map crop h=<h> w=<w> [seed=<s>] [flip=true|false]
//   map resize h=<h> w=<w>
//   map normalize [mean=<m0,m1,m2>] [std=<s0,s1,s2>]
//   map cast                              (u8 -> fp32)
//   map center_crop h=<h> w=<w>
//   map scale scale=<a0,a1,a2> [shift=<b0,b1,b2>]   (x * a_c + b_c -> fp32)
//   map decode h=<h> w=<w>
//   filter keep=even|odd|all | filter len_le=<n>
//   shuffle buffer=<n> [seed=<s>]        shard shards=<k> index=<i>
//   batch size=<b> [drop_remainder=true]  padded_batch size=<b> [pad=<v>]
//   bucket boundaries=<b1,b2,...> sizes=<s1,...> [pad=<v>]
//   prefetch buffer=<n>|AUTO             repeat count=<n>
//   options [deterministic=true|false] [seed=<s>]
//   epochs <n>
//   disable rule=<rewrite-rule-name>
//
// UDFs get names derived from the stanza ("affine(3,1)", "crop(224,224,7,1)",
// ...) so re-parsing a document reuses the registry's entries, as the
// reference does.
#include <cstdint>
#include <fstream>
#include <sstream>

#include "dpb200/datapipe.hpp"

namespace datapipe::b200 {
namespace {

struct Arg {
  std::string key, value;
  int column;
};
struct Line {
  int number = 0, column = 0;
  std::string stanza, subkind;
  std::vector<Arg> args;
  std::vector<std::string> words;  // bare words after the stanza (e.g. `epochs 5`)
};

[[noreturn]] void Fail(int line, int col, const std::string& msg) {
  throw PipelineError(ErrorCode::kParseError, "line " + std::to_string(line) + ", col " + std::to_string(col) + ": " +
                                                  msg);
}

std::vector<Line> Tokenize(const std::string& text) {
  std::vector<Line> out;
  std::istringstream in(text);
  std::string raw;
  int number = 0;
  while (std::getline(in, raw)) {
    ++number;
    const size_t hash = raw.find('#');
    if (hash != std::string::npos) raw.resize(hash);
    Line line;
    line.number = number;
    size_t i = 0;
    int token = 0;
    while (i < raw.size()) {
      while (i < raw.size() && std::isspace(static_cast<unsigned char>(raw[i]))) ++i;
      if (i >= raw.size()) break;
      const size_t start = i;
      while (i < raw.size() && !std::isspace(static_cast<unsigned char>(raw[i]))) ++i;
      const std::string word = raw.substr(start, i - start);
      const int col = static_cast<int>(start) + 1;
      const size_t eq = word.find('=');
      if (token == 0) {
        line.stanza = word;
        line.column = col;
      } else if (eq == std::string::npos) {
        if (line.subkind.empty() && line.args.empty() && line.words.empty() &&
            (line.stanza == "source" || line.stanza == "map" || line.stanza == "filter")) {
          line.subkind = word;
        } else {
          line.words.push_back(word);
        }
      } else {
        if (eq == 0) Fail(number, col, "argument without a key");
        line.args.push_back({word.substr(0, eq), word.substr(eq + 1), col});
      }
      ++token;
    }
    if (!line.stanza.empty()) out.push_back(std::move(line));
  }
  return out;
}

class StanzaArgs {
 public:
  explicit StanzaArgs(const Line& l) : l_(l), used_(l.args.size(), false) {}
  std::optional<std::string> Value(const std::string& k) {
    for (size_t i = 0; i < l_.args.size(); ++i)
      if (l_.args[i].key == k) {
        used_[i] = true;
        return l_.args[i].value;
      }
    return std::nullopt;
  }
  std::vector<std::string> AllValues(const std::string& k) {
    std::vector<std::string> v;
    for (size_t i = 0; i < l_.args.size(); ++i)
      if (l_.args[i].key == k) {
        used_[i] = true;
        v.push_back(l_.args[i].value);
      }
    return v;
  }
  int64_t Integer(const std::string& k, std::optional<int64_t> fallback = {}) {
    auto v = Value(k);
    if (!v) {
      if (fallback) return *fallback;
      Fail(l_.number, l_.column, l_.stanza + ": missing '" + k + "'");
    }
    return ToInt(*v, k);
  }
  uint64_t Unsigned(const std::string& k, uint64_t fallback) {
    auto v = Value(k);
    if (!v) return fallback;
    try {
      size_t idx = 0;
      const uint64_t x = std::stoull(*v, &idx, 0);
      if (idx != v->size()) throw std::invalid_argument("trailing");
      return x;
    } catch (const std::exception&) {
      Fail(l_.number, ColumnOfKey(k), "'" + k + "' must be an unsigned integer, got '" + *v + "'");
    }
  }
  int64_t IntOrAuto(const std::string& k, int64_t fallback) {
    auto v = Value(k);
    if (!v) return fallback;
    if (*v == "AUTO") return kAutotune;
    return ToInt(*v, k);
  }
  bool Flag(const std::string& k, bool fallback) {
    auto v = Value(k);
    if (!v) return fallback;
    if (*v == "true" || *v == "1") return true;
    if (*v == "false" || *v == "0") return false;
    Fail(l_.number, ColumnOfKey(k), "'" + k + "' must be true or false");
  }
  std::vector<int64_t> Integers(const std::string& k) {
    auto v = Value(k);
    if (!v) Fail(l_.number, l_.column, l_.stanza + ": missing '" + k + "'");
    std::vector<int64_t> out;
    std::stringstream ss(*v);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(ToInt(item, k));
    return out;
  }
  std::vector<float> Floats(const std::string& k, std::vector<float> fallback) {
    auto v = Value(k);
    if (!v) return fallback;
    std::vector<float> out;
    std::stringstream ss(*v);
    std::string item;
    while (std::getline(ss, item, ',')) {
      try {
        out.push_back(std::stof(item));
      } catch (const std::exception&) {
        Fail(l_.number, ColumnOfKey(k), "'" + k + "' must be a list of numbers");
      }
    }
    return out;
  }
  void CheckAllUsed() {
    for (size_t i = 0; i < l_.args.size(); ++i)
      if (!used_[i]) Fail(l_.number, l_.args[i].column, l_.stanza + ": unknown argument '" + l_.args[i].key + "'");
    if (!l_.words.empty() && l_.stanza != "epochs")
      Fail(l_.number, l_.column, l_.stanza + ": unexpected '" + l_.words[0] + "'");
  }

 private:
  int64_t ToInt(const std::string& v, const std::string& k) {
    try {
      size_t idx = 0;
      const int64_t x = std::stoll(v, &idx, 0);
      if (idx != v.size()) throw std::invalid_argument("trailing");
      return x;
    } catch (const std::exception&) {
      Fail(l_.number, ColumnOfKey(k), "'" + k + "' must be an integer, got '" + v + "'");
    }
  }
  int ColumnOfKey(const std::string& k) const {
    for (const auto& a : l_.args)
      if (a.key == k) return a.column;
    return l_.column;
  }
  const Line& l_;
  std::vector<bool> used_;
};

}  // namespace

ParsedPipeline ParsePipelineSpec(const std::string& text, UdfRegistry& reg, int device) {
  ParsedPipeline out;
  DatasetGraph g;
  bool have_source = false;
  for (const Line& line : Tokenize(text)) {
    StanzaArgs args(line);
    const int L = line.number, C = line.column;
    const std::string& s = line.stanza;
    auto need_source = [&] {
      if (!have_source) Fail(L, C, "'" + s + "' before a source stanza");
    };
    try {
      if (s == "source") {
        if (have_source) Fail(L, C, "multiple source stanzas");
        const std::string& k = line.subkind;
        if (k == "range") {
          g = ops::Range(args.Integer("count"), reg);
        } else if (k == "memory") {
          auto v = args.Value("values");
          if (!v) Fail(L, C, "memory source requires values=1,2,3");
          std::vector<int64_t> vals;
          std::stringstream ss(*v);
          std::string item;
          while (std::getline(ss, item, ',')) {
            try {
              vals.push_back(std::stoll(item));
            } catch (const std::exception&) {
              Fail(L, C, "values must be integers");
            }
          }
          g = ops::FromMemory(vals, reg, device);
        } else if (k == "images") {
          const int64_t n = args.Integer("count"), h = args.Integer("h"), w = args.Integer("w");
          g = ops::TensorSlices(SynthImages(n, h, w, args.Unsigned("seed", 0x5EED), device), reg);
        } else if (k == "tokens") {
          const int64_t n = args.Integer("count"), m = args.Integer("max_len");
          const uint64_t seed = args.Unsigned("seed", 4);
          g = ops::TokenSequences(SynthTokens(n, static_cast<uint32_t>(m), seed, seed, device), reg);
        } else if (k == "file") {
          auto paths = args.AllValues("path");
          if (paths.empty()) Fail(L, C, "file source requires path=...");
          g = ops::FromFile(paths, reg, device);
        } else {
          Fail(L, C, "usage: source range|memory|images|tokens|file ...");
        }
        have_source = true;
      } else if (s == "map") {
        need_source();
        const std::string& k = line.subkind;
        std::string name;
        if (k == "affine") {
          const int64_t a = args.Integer("a"), b = args.Integer("b", 0);
          name = "affine(" + std::to_string(a) + "," + std::to_string(b) + ")";
          if (!reg.Contains(name)) reg.RegisterAffine(name, a, b);
        } else if (k == "crop") {
          const int64_t h = args.Integer("h"), w = args.Integer("w");
          const uint64_t seed = args.Unsigned("seed", 7);
          const bool flip = args.Flag("flip", true);
          name = "crop(" + std::to_string(h) + "," + std::to_string(w) + "," + std::to_string(seed) + "," +
                 (flip ? "1" : "0") + ")";
          if (!reg.Contains(name)) reg.RegisterRandomCropFlip(name, h, w, seed, flip);
        } else if (k == "resize") {
          const int64_t h = args.Integer("h"), w = args.Integer("w");
          name = "resize(" + std::to_string(h) + "," + std::to_string(w) + ")";
          if (!reg.Contains(name)) reg.RegisterResizeBilinear(name, h, w);
        } else if (k == "normalize") {
          auto m = args.Floats("mean", {123.675f, 116.28f, 103.53f});
          auto d = args.Floats("std", {58.395f, 57.12f, 57.375f});
          if (m.size() != 3 || d.size() != 3) Fail(L, C, "normalize: mean and std take 3 values");
          std::ostringstream nm;
          nm << "normalize(" << m[0] << "," << m[1] << "," << m[2] << ";" << d[0] << "," << d[1] << "," << d[2] << ")";
          name = nm.str();
          if (!reg.Contains(name)) reg.RegisterNormalize(name, {m[0], m[1], m[2]}, {d[0], d[1], d[2]});
        } else if (k == "cast") {
          name = "cast";
          if (!reg.Contains(name)) reg.RegisterCast(name);
        } else if (k == "center_crop") {
          const int64_t h = args.Integer("h"), w = args.Integer("w");
          name = "center_crop(" + std::to_string(h) + "," + std::to_string(w) + ")";
          if (!reg.Contains(name)) reg.RegisterCenterCrop(name, h, w);
        } else if (k == "scale") {
          auto a = args.Floats("scale", {1.f, 1.f, 1.f});
          auto b = args.Floats("shift", {0.f, 0.f, 0.f});
          if (a.size() != 3 || b.size() != 3) Fail(L, C, "scale: scale and shift take 3 values");
          std::ostringstream nm;
          nm << "scale(" << a[0] << "," << a[1] << "," << a[2] << ";" << b[0] << "," << b[1] << "," << b[2] << ")";
          name = nm.str();
          if (!reg.Contains(name)) reg.RegisterImageAffine(name, {a[0], a[1], a[2]}, {b[0], b[1], b[2]});
        } else if (k == "decode") {
          const int64_t h = args.Integer("h"), w = args.Integer("w");
          name = "decode_raw(" + std::to_string(h) + "," + std::to_string(w) + ")";
          if (!reg.Contains(name)) reg.RegisterDecodeRaw(name, h, w);
        } else {
          Fail(L, C, "usage: map affine|crop|center_crop|resize|normalize|scale|cast|decode ...");
        }
        const int64_t p = args.IntOrAuto("parallel", 1);
        out.tunables.push_back({"map@" + std::to_string(out.tunables.size()) + ".parallel", "num_parallel_calls"});
        g = ops::Map(g, name, p, reg);
      } else if (s == "filter") {
        need_source();
        std::string name;
        if (auto keep = args.Value("keep")) {
          reg.RegisterStandardPredicates();
          if (*keep != "even" && *keep != "odd" && *keep != "all") Fail(L, C, "filter requires keep=even|odd|all");
          name = "keep_" + *keep;
        } else if (auto le = args.Value("len_le")) {
          name = "len_le(" + *le + ")";
          if (!reg.Contains(name)) reg.RegisterLengthFilter(name, std::stoll(*le));
        } else {
          Fail(L, C, "filter requires keep=even|odd|all or len_le=<n>");
        }
        g = ops::Filter(g, name, reg);
      } else if (s == "shuffle") {
        need_source();
        const int64_t b = args.Integer("buffer");
        auto seed = args.Value("seed");
        g = ops::Shuffle(g, b, seed ? std::optional<uint64_t>(std::stoull(*seed, nullptr, 0)) : std::nullopt, reg);
      } else if (s == "shard") {
        need_source();
        g = ops::Shard(g, args.Integer("shards"), args.Integer("index"), reg);
      } else if (s == "batch") {
        need_source();
        g = ops::Batch(g, args.Integer("size"), args.Flag("drop_remainder", false), reg);
      } else if (s == "padded_batch") {
        need_source();
        g = ops::PaddedBatch(g, args.Integer("size"), args.Integer("pad", 0), args.Flag("drop_remainder", false), reg);
      } else if (s == "bucket") {
        need_source();
        const auto b = args.Integers("boundaries"), z = args.Integers("sizes");
        g = ops::BucketByLength(g, b, z, args.Integer("pad", 0), args.Flag("drop_remainder", false), reg);
      } else if (s == "prefetch") {
        need_source();
        out.tunables.push_back({"prefetch@" + std::to_string(out.tunables.size()) + ".buffer", "buffer_size"});
        g = ops::Prefetch(g, args.IntOrAuto("buffer", kAutotune), reg);
      } else if (s == "repeat") {
        need_source();
        g = ops::Repeat(g, args.Integer("count"), reg);
      } else if (s == "options") {
        out.options.deterministic = args.Flag("deterministic", true);
        if (auto seed = args.Value("seed")) out.options.seed_override = std::stoull(*seed, nullptr, 0);
      } else if (s == "epochs") {
        if (line.words.size() != 1) Fail(L, C, "usage: epochs <n>");
        out.epochs = static_cast<int>(std::stoll(line.words[0]));
        if (out.epochs < 1) Fail(L, C, "epochs must be >= 1");
      } else if (s == "disable") {
        auto rule = args.Value("rule");
        if (!rule) Fail(L, C, "usage: disable rule=<name>");
        out.disabled_rules.push_back(*rule);
      } else {
        Fail(L, C, "unknown stanza '" + s + "'");
      }
      args.CheckAllUsed();
    } catch (const PipelineError& e) {
      if (e.code() == ErrorCode::kParseError) throw;
      Fail(L, C, e.what());  // a builder's validation error, located
    } catch (const std::invalid_argument&) {
      Fail(L, C, "malformed number");
    } catch (const std::out_of_range&) {
      Fail(L, C, "number out of range");
    }
  }
  if (!have_source) Fail(1, 1, "no source stanza");
  out.graph = g;
  return out;
}

ParsedPipeline ParsePipelineSpecFile(const std::string& path, UdfRegistry& reg, int device) {
  std::ifstream f(path);
  if (!f) throw PipelineError(ErrorCode::kMissingFile, "no such file: " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ParsePipelineSpec(ss.str(), reg, device);
}

}  // namespace datapipe::b200
