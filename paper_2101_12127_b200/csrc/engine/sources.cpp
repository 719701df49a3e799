// sources.cpp -- the device-resident (or pinned-host) element sources:
// synthetic images / tokens (SURVEY.md 8(d) generators, keyed like the
// oracle's), uploads from host arrays, pinned-host images for end-to-end
// runs, and length-prefixed record files (FromFileIterator,
// /root/reference/proj/src/runtime.cpp:416-474; WriteRecordFile 2251-2266).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "dpb200/datapipe.hpp"
#include "dpcuda.h"
#include "engine/device_util.hpp"

namespace datapipe::b200 {
using namespace detail;

SourcePtr SynthImages(int64_t count, int64_t h, int64_t w, uint64_t seed, int device) {
  if (count < 1 || h < 1 || w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "synth images: bad shape");
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kImages;
  s->count = count;
  s->h = h;
  s->w = w;
  s->c = 3;
  s->device = device;
  const size_t bytes = static_cast<size_t>(count) * h * w * 3;
  s->values = DeviceAlloc(bytes, device);
  DeviceGuard g(device);
  KCheck(dp_k_synth_images(P<uint8_t>(s->values), 0, count, h * w * 3, seed, nullptr), "synth images");
  CudaCheck(cudaDeviceSynchronize(), "synth images");
  return s;
}

SourcePtr SynthImagesSharded(int64_t global_count, int64_t h, int64_t w, uint64_t seed, int64_t num_shards,
                             int64_t index, int device) {
  if (num_shards < 1 || index < 0 || index >= num_shards || global_count <= index)
    throw PipelineError(ErrorCode::kInvalidAttr, "synth images: shard index must be in [0, num_shards) and < count");
  if (h < 1 || w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "synth images: bad shape");
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kImages;
  s->count = (global_count - index + num_shards - 1) / num_shards;
  s->global_count = global_count;
  s->shard_count = num_shards;
  s->shard_index = index;
  s->h = h;
  s->w = w;
  s->c = 3;
  s->device = device;
  s->values = DeviceAlloc(static_cast<size_t>(s->count) * h * w * 3, device);
  DeviceGuard g(device);
  KCheck(dp_k_synth_images_strided(P<uint8_t>(s->values), index, num_shards, s->count, h * w * 3, seed, nullptr),
         "synth images");
  CudaCheck(cudaDeviceSynchronize(), "synth images");
  return s;
}

SourcePtr SynthRecordsSharded(int64_t num_files, int64_t records_per_file, int64_t h, int64_t w, uint64_t seed,
                              int64_t num_shards, int64_t index, int device) {
  if (num_shards < 1 || index < 0 || index >= num_shards || num_files <= index)
    throw PipelineError(ErrorCode::kInvalidAttr, "synth records: shard index must be in [0, num_shards) and < files");
  if (records_per_file < 1 || h < 1 || w < 1) throw PipelineError(ErrorCode::kInvalidAttr, "synth records: bad shape");
  const int64_t files = (num_files - index + num_shards - 1) / num_shards, R = records_per_file;
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kImages;
  s->count = files * R;
  s->h = h;
  s->w = w;
  s->c = 3;
  s->device = device;
  if (num_shards > 1) {
    s->global_count = num_files * R;
    s->shard_count = num_shards;
    s->shard_index = index;
    s->shard_block = R;
  }
  const size_t image = static_cast<size_t>(h) * w * 3;
  s->values = DeviceAlloc(static_cast<size_t>(s->count) * image, device);
  DeviceGuard g(device);
  for (int64_t j = 0; j < files; ++j)  // held file j = file x: ids x * R .. x * R + R - 1 (setup, not timed)
    KCheck(dp_k_synth_images(P<uint8_t>(s->values) + j * R * image, (index + j * num_shards) * R, R, image, seed,
                             nullptr),
           "synth records");
  CudaCheck(cudaDeviceSynchronize(), "synth records");
  return s;
}

SourcePtr AsShard(const SourcePtr& s, int64_t global_count, int64_t num_shards, int64_t index, int64_t block) {
  if (!s) throw PipelineError(ErrorCode::kInvalidAttr, "as_shard: null source");
  if (s->shard_count != 1) throw PipelineError(ErrorCode::kInvalidAttr, "as_shard: source is already a shard");
  if (num_shards < 1 || index < 0 || index >= num_shards || block < 1 || global_count < 1)
    throw PipelineError(ErrorCode::kInvalidAttr, "as_shard: need 0 <= index < num_shards, block >= 1");
  const int64_t blocks = (global_count + block - 1) / block;
  const int64_t mine = blocks > index ? (blocks - index + num_shards - 1) / num_shards : 0;
  int64_t held = mine * block;
  if (mine > 0 && (index + (mine - 1) * num_shards) == blocks - 1) held -= blocks * block - global_count;
  if (held != s->count)
    throw PipelineError(ErrorCode::kInvalidAttr, "as_shard: shard " + std::to_string(index) + " of " +
                                                     std::to_string(num_shards) + " holds " + std::to_string(held) +
                                                     " elements, the source " + std::to_string(s->count));
  auto v = std::make_shared<SourceData>(*s);
  v->global_count = global_count;
  v->shard_count = num_shards;
  v->shard_index = index;
  v->shard_block = block;
  return v;
}

SourcePtr WithLabels(const SourcePtr& s, const int64_t* labels, int64_t count) {
  if (!s || s->kind != SourceData::Kind::kImages)
    throw PipelineError(ErrorCode::kInvalidAttr, "labels: the source must hold images");
  if (count != s->count)
    throw PipelineError(ErrorCode::kInvalidAttr, "labels: " + std::to_string(count) + " labels for " +
                                                     std::to_string(s->count) + " images");
  if (count > 0 && !labels) throw PipelineError(ErrorCode::kInvalidAttr, "labels: null");
  auto v = std::make_shared<SourceData>(*s);
  const size_t bytes = sizeof(int64_t) * std::max<int64_t>(count, 1);
  DeviceGuard g(s->device);
  if (s->residency == Residency::kHost) {
    v->labels = PinnedAlloc(bytes);  // mapped: the kernels read it over PCIe like the images
    if (count) std::memcpy(v->labels.get(), labels, sizeof(int64_t) * count);
  } else {
    v->labels = DeviceAlloc(bytes, s->device);
    if (count)
      CudaCheck(cudaMemcpy(v->labels.get(), labels, sizeof(int64_t) * count, cudaMemcpyHostToDevice), "labels");
  }
  return v;
}

SourcePtr SynthTokens(int64_t count, uint32_t max_len, uint64_t len_seed, uint64_t tok_seed, int device) {
  if (count < 1 || max_len < 1) throw PipelineError(ErrorCode::kInvalidAttr, "synth tokens: bad shape");
  // lengths: Pcg32(len_seed).Bounded(max_len) + 1 drawn in order (random.hpp:41-63)
  std::vector<int32_t> lens(count);
  uint64_t st = 0;
  auto next = [&]() {
    uint64_t old = st;
    st = old * 6364136223846793005ULL + 1442695040888963407ULL;
    uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((-rot) & 31u));
  };
  next();
  st += len_seed;
  next();
  const uint32_t thr = (0u - max_len) % max_len;
  for (auto& l : lens) {
    uint32_t r;
    do r = next();
    while (r < thr);
    l = static_cast<int32_t>(r % max_len) + 1;
  }
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kTokens;
  s->count = count;
  s->device = device;
  std::vector<int64_t> offs(count + 1, 0);
  for (int64_t i = 0; i < count; ++i) offs[i + 1] = offs[i] + lens[i];
  s->total_tokens = offs[count];
  s->lengths = DeviceAlloc(sizeof(int32_t) * count, device);
  s->offsets = DeviceAlloc(sizeof(int64_t) * (count + 1), device);
  s->tokens = DeviceAlloc(sizeof(int32_t) * std::max<int64_t>(s->total_tokens, 1), device);
  DeviceGuard g(device);
  CudaCheck(cudaMemcpy(s->lengths.get(), lens.data(), sizeof(int32_t) * count, cudaMemcpyHostToDevice), "upload");
  CudaCheck(cudaMemcpy(s->offsets.get(), offs.data(), sizeof(int64_t) * (count + 1), cudaMemcpyHostToDevice), "upload");
  KCheck(dp_k_synth_tokens(P<int32_t>(s->tokens), P<int64_t>(s->offsets), count, tok_seed, nullptr), "synth tokens");
  CudaCheck(cudaDeviceSynchronize(), "synth tokens");
  return s;
}

SourcePtr ImagesFromHost(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device) {
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kImages;
  s->count = count;
  s->h = h;
  s->w = w;
  s->c = 3;
  s->device = device;
  const size_t bytes = static_cast<size_t>(count) * h * w * 3;
  s->values = DeviceAlloc(bytes, device);
  DeviceGuard g(device);
  CudaCheck(cudaMemcpy(s->values.get(), data, bytes, cudaMemcpyHostToDevice), "upload images");
  return s;
}

SourcePtr ImagesFromPinnedHost(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device) {
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kImages;
  s->count = count;
  s->h = h;
  s->w = w;
  s->c = 3;
  s->device = device;
  s->residency = Residency::kHost;
  DeviceGuard g(device);
  void* dptr = nullptr;
  const size_t bytes = static_cast<size_t>(count) * h * w * 3;
  bool registered = false;
  if (cudaHostGetDevicePointer(&dptr, const_cast<uint8_t*>(data), 0) != cudaSuccess) {
    cudaGetLastError();
    CudaCheck(cudaHostRegister(const_cast<uint8_t*>(data), bytes, cudaHostRegisterMapped | cudaHostRegisterPortable),
              "cudaHostRegister");
    registered = true;
    CudaCheck(cudaHostGetDevicePointer(&dptr, const_cast<uint8_t*>(data), 0), "cudaHostGetDevicePointer");
  }
  void* host = const_cast<uint8_t*>(data);
  s->values = std::shared_ptr<void>(dptr, [host, registered](void*) {
    if (registered) cudaHostUnregister(host);
  });
  return s;
}

// FromFileIterator::Next (/root/reference/proj/src/runtime.cpp:416-474):
// records are [u32 little-endian length][payload], files read in order; a
// truncated length or payload is MalformedInput, a missing file MissingFile.
SourcePtr RecordsFromFiles(const std::vector<std::string>& paths, int device, int64_t num_shards, int64_t index) {
  if (paths.empty()) throw PipelineError(ErrorCode::kInvalidAttr, "from_file: 'paths' must be non-empty");
  if (num_shards < 1 || index < 0 || index >= num_shards || static_cast<int64_t>(paths.size()) <= index)
    throw PipelineError(ErrorCode::kInvalidAttr, "records: shard index must be in [0, num_shards) and < files");
  auto held = [&](size_t fi) { return static_cast<int64_t>(fi) % num_shards == index; };
  // Pass 1: walk the length headers (seeking over payloads) -- validates the
  // framing and sizes everything.  Pass 2 reads the payloads straight into
  // one pinned staging buffer (one host copy of the data), then one H2D copy.
  struct Rec {
    size_t file;
    long pos;
    uint32_t len;
  };
  std::vector<Rec> recs;
  std::vector<int64_t> offsets{0};
  std::vector<int64_t> per_file;
  int64_t uniform = -1;
  for (size_t fi = 0; fi < paths.size(); ++fi) {
    if (!held(fi)) continue;
    const std::string& path = paths[fi];
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw PipelineError(ErrorCode::kMissingFile, "no such file: " + path);
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    const size_t before = recs.size();
    long pos = 0;
    while (pos < size) {
      unsigned char lb[4];
      if (pos + 4 > size || std::fread(lb, 1, 4, f) != 4) {
        std::fclose(f);
        throw PipelineError(ErrorCode::kMalformedInput,
                            "at byte " + std::to_string(pos) + ": truncated record length in " + path);
      }
      const uint32_t len = lb[0] | (lb[1] << 8) | (lb[2] << 16) | (static_cast<uint32_t>(lb[3]) << 24);
      pos += 4;
      if (pos + static_cast<long>(len) > size) {
        std::fclose(f);
        throw PipelineError(ErrorCode::kMalformedInput,
                            "at byte " + std::to_string(pos) + ": truncated record payload in " + path);
      }
      recs.push_back({fi, pos, len});
      offsets.push_back(offsets.back() + len);
      uniform = (uniform < 0 || uniform == static_cast<int64_t>(len)) ? len : -2;
      pos += len;
      std::fseek(f, pos, SEEK_SET);
    }
    std::fclose(f);
    per_file.push_back(static_cast<int64_t>(recs.size() - before));
  }
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kRecords;
  s->count = static_cast<int64_t>(recs.size());
  s->record_len = uniform >= 0 ? uniform : 0;
  if (num_shards > 1) {  // block residency: every held file holds R records
    for (int64_t c : per_file)
      if (c != per_file[0])
        throw PipelineError(ErrorCode::kMalformedInput,
                            "sharded records: held files hold " + std::to_string(per_file[0]) + " and " +
                                std::to_string(c) + " records (block residency needs equal files)");
    s->shard_count = num_shards;
    s->shard_index = index;
    s->shard_block = std::max<int64_t>(per_file[0], 1);
    s->global_count = per_file[0] * static_cast<int64_t>(paths.size());
  }
  s->file_records = std::move(per_file);
  s->device = device;
  const size_t total = static_cast<size_t>(offsets.back());
  auto staging = PinnedAlloc(std::max<size_t>(total, 16));
  char* dst = static_cast<char*>(staging.get());
  for (size_t fi = 0, r = 0; fi < paths.size(); ++fi) {
    if (!held(fi)) continue;
    FILE* f = std::fopen(paths[fi].c_str(), "rb");
    if (!f) throw PipelineError(ErrorCode::kMissingFile, "no such file: " + paths[fi]);
    for (; r < recs.size() && recs[r].file == fi; ++r) {
      std::fseek(f, recs[r].pos, SEEK_SET);
      if (std::fread(dst + offsets[r], 1, recs[r].len, f) != recs[r].len) {
        std::fclose(f);
        throw PipelineError(ErrorCode::kMalformedInput, "file changed while reading: " + paths[fi]);
      }
    }
    std::fclose(f);
  }
  s->values = DeviceAlloc(std::max<size_t>(total, 16), device);
  s->offsets = DeviceAlloc(sizeof(int64_t) * offsets.size(), device);
  DeviceGuard g(device);
  CudaCheck(cudaMemcpy(s->values.get(), staging.get(), total, cudaMemcpyHostToDevice), "upload records");
  CudaCheck(cudaMemcpy(s->offsets.get(), offsets.data(), sizeof(int64_t) * offsets.size(), cudaMemcpyHostToDevice),
            "upload offsets");
  return s;
}

// runtime.cpp:2251-2266
void WriteRecordFile(const std::string& path, const std::vector<std::string>& payloads) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw PipelineError(ErrorCode::kMissingFile, "cannot write: " + path);
  for (const auto& p : payloads) {
    const uint32_t len = static_cast<uint32_t>(p.size());
    unsigned char lb[4] = {static_cast<unsigned char>(len), static_cast<unsigned char>(len >> 8),
                           static_cast<unsigned char>(len >> 16), static_cast<unsigned char>(len >> 24)};
    std::fwrite(lb, 1, 4, f);
    std::fwrite(p.data(), 1, p.size(), f);
  }
  std::fclose(f);
}

SourcePtr Int64FromHost(const int64_t* values, int64_t count, int device) {
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kInt64;
  s->count = count;
  s->device = device;
  if (count) s->host_int64.assign(values, values + count);
  // Without a CUDA device the graph still builds (and serializes); the device
  // copy is made here when a device exists, and MakeIterator fails loudly
  // without one -- nothing is computed on the host.
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return s;
  }
  s->values = DeviceAlloc(sizeof(int64_t) * std::max<int64_t>(count, 1), device);
  DeviceGuard g(device);
  if (count) CudaCheck(cudaMemcpy(s->values.get(), values, sizeof(int64_t) * count, cudaMemcpyHostToDevice), "upload");
  return s;
}

SourcePtr TokensFromPinnedHost(const int32_t* lengths, int64_t count, const int32_t* tokens, int device) {
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kTokens;
  s->count = count;
  s->device = device;
  s->residency = Residency::kHost;
  DeviceGuard g(device);
  s->lengths = PinnedAlloc(sizeof(int32_t) * std::max<int64_t>(count, 1));
  s->offsets = PinnedAlloc(sizeof(int64_t) * (count + 1));
  int64_t* offs = P<int64_t>(s->offsets);
  offs[0] = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (lengths[i] < 0) throw PipelineError(ErrorCode::kInvalidAttr, "token lengths must be >= 0");
    offs[i + 1] = offs[i] + lengths[i];
  }
  s->total_tokens = offs[count];
  if (s->total_tokens > 0 && tokens == nullptr)
    throw PipelineError(ErrorCode::kInvalidAttr, "token sequences: tokens is null but the lengths sum to " +
                                                     std::to_string(s->total_tokens));
  s->tokens = PinnedAlloc(sizeof(int32_t) * std::max<int64_t>(s->total_tokens, 1));
  if (count) std::memcpy(s->lengths.get(), lengths, sizeof(int32_t) * count);
  if (s->total_tokens) std::memcpy(s->tokens.get(), tokens, sizeof(int32_t) * s->total_tokens);
  return s;  // mapped + portable pinned memory: under UVA the host pointers are the device pointers
}

SourcePtr TokensFromHost(const int32_t* lengths, int64_t count, const int32_t* tokens, int device) {
  auto s = std::make_shared<SourceData>();
  s->kind = SourceData::Kind::kTokens;
  s->count = count;
  s->device = device;
  std::vector<int64_t> offs(count + 1, 0);
  for (int64_t i = 0; i < count; ++i) {
    if (lengths[i] < 0) throw PipelineError(ErrorCode::kInvalidAttr, "token lengths must be >= 0");
    offs[i + 1] = offs[i] + lengths[i];
  }
  s->total_tokens = offs[count];
  if (s->total_tokens > 0 && tokens == nullptr)
    throw PipelineError(ErrorCode::kInvalidAttr, "token sequences: tokens is null but the lengths sum to " +
                                                     std::to_string(s->total_tokens));
  s->lengths = DeviceAlloc(sizeof(int32_t) * std::max<int64_t>(count, 1), device);
  s->offsets = DeviceAlloc(sizeof(int64_t) * (count + 1), device);
  s->tokens = DeviceAlloc(sizeof(int32_t) * std::max<int64_t>(s->total_tokens, 1), device);
  DeviceGuard g(device);
  CudaCheck(cudaMemcpy(s->lengths.get(), lengths, sizeof(int32_t) * count, cudaMemcpyHostToDevice), "upload");
  CudaCheck(cudaMemcpy(s->offsets.get(), offs.data(), sizeof(int64_t) * (count + 1), cudaMemcpyHostToDevice), "upload");
  if (s->total_tokens)
    CudaCheck(cudaMemcpy(s->tokens.get(), tokens, sizeof(int32_t) * s->total_tokens, cudaMemcpyHostToDevice), "upload");
  return s;
}

}  // namespace datapipe::b200
