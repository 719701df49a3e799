// checkpoint.cpp -- Save / Restore of device iterators in the reference's
// DPC1 layout (/root/reference/proj/docs/formats.md:76-94,
// src/checkpoint.cpp:30-105):
//
//   "DPC1" version:u16=1 fingerprint:32B base_seed:u64 deterministic:u8
//   root_delivered:u64 entry_count:u32 { path:str(u32 len + bytes) delivered:u64 }*
//
// (little endian).  The reference restores by REPLAYING root_delivered
// GetNext calls.  The device path is a pure function of (base seed,
// position) -- epoch plans are recomputed from the seeds and every batch is
// a gather through its plan -- so Restore SEEKS: the new iterator starts at
// batch root_delivered without computing the skipped batches, and produces
// exactly the batches the replay would have (tests/test_gpu_pipeline.py).
//
// Fingerprint: GraphFingerprint (serialize.cpp in this engine), SHA-256 of
// the DPG1 serialization with the seed attrs zeroed -- byte-identical to the
// reference's for the graphs both engines express (tests/test_serialize.py
// pins it against the compiled reference), so such checkpoints carry the
// same fingerprint in both.
#include <array>
#include <cstring>
#include <sstream>

#include "dpb200/datapipe.hpp"

namespace datapipe::b200 {

namespace {

constexpr char kMagic[4] = {'D', 'P', 'C', '1'};
constexpr uint16_t kVersion = 1;

// ---- SHA-256 (FIPS 180-4) ----
struct Sha256 {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  uint64_t len = 0;
  uint8_t buf[64];
  size_t fill = 0;

  static uint32_t Rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

  void Block(const uint8_t* p) {
    static const uint32_t k[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
        0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
        0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
        0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
        0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
        0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
        0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
        0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t(p[4 * i]) << 24) | (uint32_t(p[4 * i + 1]) << 16) | (uint32_t(p[4 * i + 2]) << 8) | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      uint32_t s0 = Rotr(w[i - 15], 7) ^ Rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      uint32_t s1 = Rotr(w[i - 2], 17) ^ Rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      uint32_t t1 = hh + (Rotr(e, 6) ^ Rotr(e, 11) ^ Rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
      uint32_t t2 = (Rotr(a, 2) ^ Rotr(a, 13) ^ Rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a;
    h[1] += b;
    h[2] += c;
    h[3] += d;
    h[4] += e;
    h[5] += f;
    h[6] += g;
    h[7] += hh;
  }

  void Update(const void* data, size_t n) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    len += n;
    while (n) {
      size_t take = std::min(n, size_t(64) - fill);
      std::memcpy(buf + fill, p, take);
      fill += take;
      p += take;
      n -= take;
      if (fill == 64) {
        Block(buf);
        fill = 0;
      }
    }
  }

  std::array<uint8_t, 32> Final() {
    uint64_t bits = len * 8;
    uint8_t pad = 0x80;
    Update(&pad, 1);
    uint8_t zero = 0;
    while (fill != 56) Update(&zero, 1);
    uint8_t lenb[8];
    for (int i = 0; i < 8; ++i) lenb[i] = static_cast<uint8_t>(bits >> (56 - 8 * i));
    Update(lenb, 8);
    std::array<uint8_t, 32> out;
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) out[4 * i + j] = static_cast<uint8_t>(h[i] >> (24 - 8 * j));
    return out;
  }
};

struct Writer {
  std::string out;
  void Raw(const void* p, size_t n) { out.append(static_cast<const char*>(p), n); }
  template <typename T>
  void Le(T v) {
    for (size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<char>((static_cast<uint64_t>(v) >> (8 * i)) & 0xff));
  }
  void Str(const std::string& s) {
    Le<uint32_t>(static_cast<uint32_t>(s.size()));
    out += s;
  }
};

struct Reader {
  const std::string& in;
  size_t pos = 0;
  void Need(size_t n) {
    if (pos + n > in.size()) throw PipelineError(ErrorCode::kCorruptBlob, "truncated checkpoint at byte " + std::to_string(pos));
  }
  template <typename T>
  T Le() {
    Need(sizeof(T));
    uint64_t v = 0;
    for (size_t i = 0; i < sizeof(T); ++i) v |= static_cast<uint64_t>(static_cast<uint8_t>(in[pos + i])) << (8 * i);
    pos += sizeof(T);
    return static_cast<T>(v);
  }
  std::string Str() {
    uint32_t n = Le<uint32_t>();
    Need(n);
    std::string s = in.substr(pos, n);
    pos += n;
    return s;
  }
};

}  // namespace

std::array<uint8_t, 32> Sha256Digest(const void* data, size_t n) {
  Sha256 sha;
  sha.Update(data, n);
  return sha.Final();
}

std::string FingerprintHex(const std::array<uint8_t, 32>& fp) {
  static const char* kHex = "0123456789abcdef";
  std::string s;
  for (uint8_t b : fp) {
    s.push_back(kHex[b >> 4]);
    s.push_back(kHex[b & 0xf]);
  }
  return s;
}

std::string PipelineIterator::Save() const {
  Writer w;
  w.Raw(kMagic, 4);
  w.Le<uint16_t>(kVersion);
  const auto fp = GraphFingerprint(graph_);
  w.Raw(fp.data(), fp.size());
  w.Le<uint64_t>(base_seed_);
  w.Le<uint8_t>(options_.deterministic ? 1 : 0);
  const int64_t delivered = root_delivered();
  w.Le<uint64_t>(static_cast<uint64_t>(delivered));
  w.Le<uint32_t>(1);  // per-node progress: the root (the fused stage has no finer counters)
  w.Str("/" + std::string(NodeKindName(graph_.root()->kind())) + "@0");
  w.Le<uint64_t>(static_cast<uint64_t>(delivered));
  return w.out;
}

std::unique_ptr<PipelineIterator> Restore(const DatasetGraph& graph, const UdfRegistry& registry,
                                          const std::string& blob, IteratorOptions options) {
  if (blob.size() < 6 || blob.compare(0, 4, kMagic, 4) != 0)
    throw PipelineError(ErrorCode::kCorruptBlob, "bad checkpoint magic");
  Reader r{blob};
  r.pos = 4;
  const uint16_t version = r.Le<uint16_t>();
  if (version != kVersion)
    throw PipelineError(ErrorCode::kVersionMismatch, "unsupported checkpoint version " + std::to_string(version));
  std::array<uint8_t, 32> saved;
  for (auto& b : saved) b = r.Le<uint8_t>();
  const uint64_t base_seed = r.Le<uint64_t>();
  const bool deterministic = r.Le<uint8_t>() != 0;
  const uint64_t delivered = r.Le<uint64_t>();
  const uint32_t entries = r.Le<uint32_t>();
  for (uint32_t i = 0; i < entries; ++i) {
    r.Str();
    r.Le<uint64_t>();
  }
  if (r.pos != blob.size()) throw PipelineError(ErrorCode::kCorruptBlob, "trailing bytes in checkpoint");
  if (GraphFingerprint(graph) != saved)
    throw PipelineError(ErrorCode::kFingerprintMismatch, "checkpoint was taken from a different pipeline");
  options.deterministic = deterministic;
  options.seed_override = base_seed;
  auto it = MakeIterator(graph, registry, options);
  it->Seek(static_cast<int64_t>(delivered));
  return it;
}

}  // namespace datapipe::b200
