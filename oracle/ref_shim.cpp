// oracle/ref_shim.cpp -- extern "C" driver over the COMPILED REFERENCE.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile together with the
// reference's own sources (compiled in place from /root/reference/proj/src,
// never copied) into oracle/_ref/libdpref.so.  Used by tests/ to pin the
// oracle restatement (oracle/restate.c) and to generate tests/golden/, and by
// bench.py --impl reference / cpu_baseline as the reference CPU pipeline.
//
// Every pipeline here is built through the reference's public operator API
// (datapipe::ops::*, include/datapipe/graph.hpp:134-165), optimized with
// datapipe::Optimize (include/datapipe/optimizer.hpp:73-75) and drained
// through MakeIterator / PipelineIterator::GetNext
// (include/datapipe/runtime.hpp:68,98-100) with seed_override set (SURVEY.md
// 0.3 #5).  The map UDFs are the oracle restatement registered through
// UdfRegistry::RegisterMap (include/datapipe/udf.hpp:61-63).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "datapipe/checkpoint.hpp"
#include "datapipe/element.hpp"
#include "datapipe/errors.hpp"
#include "datapipe/graph.hpp"
#include "datapipe/optimizer.hpp"
#include "datapipe/runtime.hpp"
#include "datapipe/serialize.hpp"
#include "datapipe/udf.hpp"
#include "restate.h"

using namespace datapipe;

namespace {

thread_local std::string g_err;

int Fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

std::vector<Element> IntRange(int64_t n) {
  std::vector<Element> out;
  out.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out.push_back(Element::Scalar(Value::Int64(i)));
  return out;
}

IteratorOptions Seeded(uint64_t base_seed) {
  IteratorOptions o;
  o.deterministic = true;
  o.seed_override = base_seed;
  return o;
}

void RegisterAffine(UdfRegistry& reg, const std::string& name, int64_t a,
                    int64_t b) {
  if (reg.Contains(name)) return;
  reg.RegisterMap(name, [a, b](const Element& e) {
    return Element::Scalar(Value::Int64(e.component(0).int64() * a + b));
  });
}

struct ImageUdfParams {
  int mode;  // 0 crop+flip+normalize, 1 resize+normalize, 2 crop+normalize
  int in_h, in_w, out_h, out_w;
  uint64_t udf_seed;
};

std::string ImageUdfName(const ImageUdfParams& p) {
  return "img_udf(mode=" + std::to_string(p.mode) + ",in=" +
         std::to_string(p.in_h) + "x" + std::to_string(p.in_w) + ",out=" +
         std::to_string(p.out_h) + "x" + std::to_string(p.out_w) + ",seed=" +
         std::to_string(p.udf_seed) + ")";
}

// (int64 id, bytes uint8 HWC) -> (int64 id, bytes fp32 HWC little endian).
void RegisterImageUdf(UdfRegistry& reg, const ImageUdfParams& p) {
  std::string name = ImageUdfName(p);
  if (reg.Contains(name)) return;
  reg.RegisterMap(name, [p](const Element& e) {
    int64_t id = e.component(0).int64();
    const std::string& img = e.component(1).bytes();
    std::string out(static_cast<size_t>(p.out_h) * p.out_w * 3 * sizeof(float),
                    '\0');
    float* o = reinterpret_cast<float*>(out.data());
    const uint8_t* in = reinterpret_cast<const uint8_t*>(img.data());
    if (p.mode == 1) {
      orc_resize_normalize(in, p.in_h, p.in_w, p.out_h, p.out_w, o);
    } else {
      orc_crop_flip_normalize(in, p.in_h, p.in_w, id, p.udf_seed, p.out_h,
                              p.out_w, p.mode == 0 ? 1 : 0, o);
    }
    std::vector<Value> c;
    c.push_back(Value::Int64(id));
    c.push_back(Value::Bytes(std::move(out)));
    return Element(std::move(c));
  });
}

std::vector<Element> SynthImages(int64_t n, int h, int w, uint64_t pix_seed) {
  std::vector<Element> out;
  out.reserve(static_cast<size_t>(n));
  size_t bytes = static_cast<size_t>(h) * w * 3;
  std::string buf(bytes, '\0');
  for (int64_t i = 0; i < n; ++i) {
    orc_synth_images(pix_seed, static_cast<uint64_t>(i), 1, bytes,
                     reinterpret_cast<uint8_t*>(buf.data()));
    std::vector<Value> c;
    c.push_back(Value::Int64(i));
    c.push_back(Value::Bytes(buf));
    out.push_back(Element(std::move(c)));
  }
  return out;
}

struct ImagePipelineArgs {
  ImageUdfParams udf;
  int64_t n;
  int64_t shard_k, shard_g;    // shard_k 0 => no shard
  int64_t shuffle_buffer;      // 0 => no shuffle
  int has_shuffle_seed;
  uint64_t shuffle_seed;
  int64_t batch;
  int drop_remainder;
  int64_t parallel;            // num_parallel_calls of the map
  int64_t prefetch;            // 0 => none; -1 AUTOTUNE
  uint64_t pix_seed;
};

DatasetGraph BuildImageGraph(UdfRegistry& reg, const ImagePipelineArgs& a,
                             std::vector<Element> elements) {
  RegisterImageUdf(reg, a.udf);
  DatasetGraph g = ops::FromMemory(std::move(elements), reg);
  if (a.shard_k > 0) g = ops::Shard(g, a.shard_k, a.shard_g, reg);
  if (a.shuffle_buffer > 0) {
    std::optional<uint64_t> seed;
    if (a.has_shuffle_seed) seed = a.shuffle_seed;
    g = ops::Shuffle(g, a.shuffle_buffer, seed, reg);
  }
  g = ops::Map(g, ImageUdfName(a.udf), a.parallel, reg);
  g = ops::Batch(g, a.batch, a.drop_remainder != 0, reg);
  if (a.prefetch != 0) g = ops::Prefetch(g, a.prefetch, reg);
  auto [opt, report] = Optimize(g, RuleSet::Default(), reg);
  return opt;
}

// One image-chain step as its own reference map UDF: (int64 id, bytes img
// [, int64 label]) -> the same with the step applied (oracle/chain.c); the
// input dims / dtype of the step are fixed by the chain prefix.
std::string RegisterChainStep(UdfRegistry& reg, const orc_map_step& s, int index, int in_h, int in_w, int in_f32) {
  std::string name = "chain_step(" + std::to_string(index) + ",op=" + std::to_string(s.op) + ")";
  reg.RegisterMap(name, [s, in_h, in_w, in_f32](const Element& e) {
    int oh = 0, ow = 0, of = 0;
    if (orc_chain_output(&s, 1, in_h, in_w, &oh, &ow, &of)) throw std::runtime_error("chain step: bad shape");
    of = of || in_f32;
    const int64_t id = e.component(0).int64();
    std::string out(static_cast<size_t>(oh) * ow * 3 * (of ? sizeof(float) : 1), '\0');
    if (orc_apply_step(e.component(1).bytes().data(), in_h, in_w, in_f32, id, &s, out.data()))
      throw std::runtime_error("chain step failed");
    std::vector<Value> c;
    c.push_back(Value::Int64(id));
    c.push_back(Value::Bytes(std::move(out)));
    if (e.arity() == 3) c.push_back(e.component(2));
    return Element(std::move(c));
  });
  return name;
}

}  // namespace

extern "C" {

// from_memory(n synthetic images [, labels]) -> [shuffle] -> map(step_0) ->
// ... -> map(step_k) -> batch(b), optimized (map_map_fusion composes the
// steps, map_batch_fusion fuses the batch), drained by GetNext.  Outputs the
// ids, the output image bytes back to back, the labels and the batch sizes.
int ref_image_chain_pipeline(const orc_map_step* steps, int nsteps, int in_h, int in_w, uint64_t pix_seed, int64_t n,
                             const int64_t* labels, int64_t shuffle_buffer, uint64_t shuffle_seed, int64_t batch,
                             int drop_remainder, uint64_t base_seed, int64_t* out_ids, uint8_t* out_images,
                             int64_t* out_labels, int64_t* out_batch_sizes, int64_t* num_batches) {
  try {
    UdfRegistry reg;
    std::vector<Element> elems = SynthImages(n, in_h, in_w, pix_seed);
    if (labels)
      for (int64_t i = 0; i < n; ++i) {
        std::vector<Value> c{elems[i].component(0), elems[i].component(1), Value::Int64(labels[i])};
        elems[i] = Element(std::move(c));
      }
    DatasetGraph g = ops::FromMemory(std::move(elems), reg);
    if (shuffle_buffer > 0) g = ops::Shuffle(g, shuffle_buffer, shuffle_seed, reg);
    int h = in_h, w = in_w, f = 0;
    for (int i = 0; i < nsteps; ++i) {
      g = ops::Map(g, RegisterChainStep(reg, steps[i], i, h, w, f), 1, reg);
      int oh, ow, of;
      if (orc_chain_output(&steps[i], 1, h, w, &oh, &ow, &of)) throw std::runtime_error("bad chain");
      h = oh;
      w = ow;
      f = f || of;
    }
    g = ops::Batch(g, batch, drop_remainder != 0, reg);
    g = Optimize(g, RuleSet::Default(), reg).first;
    auto it = MakeIterator(g, reg, Seeded(base_seed));
    const size_t per = static_cast<size_t>(h) * w * 3 * (f ? sizeof(float) : 1);
    int64_t k = 0, nb = 0;
    while (auto e = it->GetNext()) {
      const auto& ids = e->component(0).items();
      const auto& imgs = e->component(1).items();
      for (size_t i = 0; i < ids.size(); ++i, ++k) {
        out_ids[k] = ids[i].int64();
        if (imgs[i].bytes().size() != per) throw std::runtime_error("chain output size");
        std::memcpy(out_images + static_cast<size_t>(k) * per, imgs[i].bytes().data(), per);
        if (labels) out_labels[k] = e->component(2).items()[i].int64();
      }
      out_batch_sizes[nb++] = static_cast<int64_t>(ids.size());
    }
    *num_batches = nb;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}


const char* ref_last_error(void) { return g_err.c_str(); }

// cfg1: from_memory(IntRange(n)) -> map(x*a+b, p) -> batch(b) [-> Optimize].
// out_values[n] (flattened batches), out_batch_sizes[], *num_batches; writes
// the root node kind after Optimize into root_kind (>= 32 bytes).
int ref_range_map_batch(int64_t n, int64_t a, int64_t b, int64_t batch,
                        int drop_remainder, int64_t parallel, int optimize,
                        uint64_t base_seed, int64_t* out_values,
                        int64_t* out_batch_sizes, int64_t* num_batches,
                        char* root_kind) {
  try {
    UdfRegistry reg;
    std::string udf = "affine(" + std::to_string(a) + "," + std::to_string(b) + ")";
    RegisterAffine(reg, udf, a, b);
    DatasetGraph g = ops::FromMemory(IntRange(n), reg);
    g = ops::Map(g, udf, parallel, reg);
    g = ops::Batch(g, batch, drop_remainder != 0, reg);
    if (optimize) g = Optimize(g, RuleSet::Default(), reg).first;
    std::snprintf(root_kind, 32, "%s", NodeKindName(g.root()->kind()));
    auto it = MakeIterator(g, reg, Seeded(base_seed));
    int64_t k = 0, nb = 0;
    while (auto e = it->GetNext()) {
      const auto& items = e->component(0).items();
      for (const auto& v : items) out_values[k++] = v.int64();
      out_batch_sizes[nb++] = static_cast<int64_t>(items.size());
    }
    *num_batches = nb;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// from_memory(IntRange(n)) [-> shard(k, g)] -> shuffle(buffer, seed) [->
// repeat(epochs)]; writes the emitted values (input ordinals) to out.
int ref_shuffle_ids(int64_t n, int64_t shard_k, int64_t shard_g,
                    int64_t buffer, int has_seed, uint64_t seed,
                    uint64_t base_seed, int64_t epochs, int optimize,
                    int64_t* out, int64_t* count) {
  try {
    UdfRegistry reg;
    DatasetGraph g = ops::FromMemory(IntRange(n), reg);
    if (shard_k > 0) g = ops::Shard(g, shard_k, shard_g, reg);
    std::optional<uint64_t> s;
    if (has_seed) s = seed;
    g = ops::Shuffle(g, buffer, s, reg);
    if (epochs > 1) g = ops::Repeat(g, epochs, reg);
    if (optimize) g = Optimize(g, RuleSet::Default(), reg).first;
    auto it = MakeIterator(g, reg, Seeded(base_seed));
    int64_t k = 0;
    while (auto e = it->GetNext()) out[k++] = e->component(0).int64();
    *count = k;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// Image pipelines (cfg2 / cfg3 shapes) at parity sizes.  Outputs the batch
// ids (int64), the fp32 pixels (out_h*out_w*3 per image) and batch sizes.
int ref_image_pipeline(int mode, int in_h, int in_w, int out_h, int out_w,
                       uint64_t udf_seed, uint64_t pix_seed, int64_t n,
                       int64_t shard_k, int64_t shard_g, int64_t shuffle_buffer,
                       int has_shuffle_seed, uint64_t shuffle_seed,
                       int64_t batch, int drop_remainder, int64_t parallel,
                       int64_t prefetch, uint64_t base_seed, int64_t* out_ids,
                       float* out_pixels, int64_t* out_batch_sizes,
                       int64_t* num_batches) {
  try {
    UdfRegistry reg;
    ImagePipelineArgs a{{mode, in_h, in_w, out_h, out_w, udf_seed},
                        n, shard_k, shard_g, shuffle_buffer, has_shuffle_seed,
                        shuffle_seed, batch, drop_remainder, parallel,
                        prefetch, pix_seed};
    DatasetGraph g = BuildImageGraph(reg, a, SynthImages(n, in_h, in_w, pix_seed));
    auto it = MakeIterator(g, reg, Seeded(base_seed));
    size_t per = static_cast<size_t>(out_h) * out_w * 3;
    int64_t k = 0, nb = 0;
    while (auto e = it->GetNext()) {
      const auto& ids = e->component(0).items();
      const auto& imgs = e->component(1).items();
      for (size_t i = 0; i < ids.size(); ++i, ++k) {
        out_ids[k] = ids[i].int64();
        std::memcpy(out_pixels + static_cast<size_t>(k) * per,
                    imgs[i].bytes().data(), per * sizeof(float));
      }
      out_batch_sizes[nb++] = static_cast<int64_t>(ids.size());
    }
    *num_batches = nb;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// cfg4 at parity sizes: from_memory(list[int64] token sequences) ->
// filter(len <= max_keep) -> batch(b) (ragged, the reference has no
// padded_batch).  Outputs per emitted row its length
// and tokens (concatenated), and the batch sizes.
int ref_filter_batch_tokens(int64_t n, uint64_t len_seed, uint32_t max_len,
                            uint64_t tok_seed, int32_t max_keep, int64_t batch,
                            int drop_remainder, int64_t* out_row_lengths,
                            int64_t* out_tokens, int64_t* out_batch_sizes,
                            int64_t* num_batches, int64_t* num_rows,
                            int64_t* num_tokens) {
  try {
    UdfRegistry reg;
    std::string pred = "len_le(" + std::to_string(max_keep) + ")";
    reg.RegisterPredicate(pred, [max_keep](const Element& e) {
      return static_cast<int64_t>(e.component(0).items().size()) <= max_keep;
    });
    std::vector<int32_t> lens(static_cast<size_t>(n));
    orc_synth_lengths(len_seed, max_len, static_cast<uint64_t>(n), lens.data());
    std::vector<Element> elems;
    elems.reserve(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      std::vector<Value> toks;
      toks.reserve(static_cast<size_t>(lens[i]));
      for (int32_t j = 0; j < lens[i]; ++j)
        toks.push_back(Value::Int64(orc_synth_token(tok_seed, i, j)));
      elems.push_back(Element::Scalar(Value::List(std::move(toks))));
    }
    DatasetGraph g = ops::FromMemory(std::move(elems), reg);
    g = ops::Filter(g, pred, reg);
    g = ops::Batch(g, batch, drop_remainder != 0, reg);
    g = Optimize(g, RuleSet::Default(), reg).first;
    auto it = MakeIterator(g, reg, Seeded(1));
    int64_t nb = 0, nr = 0, nt = 0;
    while (auto e = it->GetNext()) {
      const auto& rows = e->component(0).items();
      for (const auto& row : rows) {
        out_row_lengths[nr++] = static_cast<int64_t>(row.items().size());
        for (const auto& t : row.items()) out_tokens[nt++] = t.int64();
      }
      out_batch_sizes[nb++] = static_cast<int64_t>(rows.size());
    }
    *num_batches = nb;
    *num_rows = nr;
    *num_tokens = nt;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// cfg5 index stage: from_memory(shard ids 0..S-1) -> shard(k, g) ->
// interleave(reader of R records valued id*R + r, cycle, parallel) [->
// shuffle(buffer, seed)].  Emits the record values.
int ref_interleave_ids(int64_t num_sources, int64_t shard_k, int64_t shard_g,
                       int64_t cycle, int64_t parallel, int64_t records,
                       int64_t shuffle_buffer, uint64_t shuffle_seed,
                       uint64_t base_seed, int64_t* out, int64_t* count) {
  try {
    UdfRegistry reg;
    std::string udf = "reader(" + std::to_string(records) + ")";
    reg.RegisterDataset(
        udf,
        [&reg, records](const Element& e) {
          int64_t s = e.component(0).int64();
          std::vector<Element> recs;
          for (int64_t r = 0; r < records; ++r)
            recs.push_back(Element::Scalar(Value::Int64(s * records + r)));
          return ops::FromMemory(std::move(recs), reg);
        },
        ElementSpec({TypeSpec::Int64()}));
    DatasetGraph g = ops::FromMemory(IntRange(num_sources), reg);
    if (shard_k > 0) g = ops::Shard(g, shard_k, shard_g, reg);
    g = ops::Interleave(g, udf, cycle, parallel, reg);
    if (shuffle_buffer > 0) g = ops::Shuffle(g, shuffle_buffer, shuffle_seed, reg);
    auto it = MakeIterator(g, reg, Seeded(base_seed));
    int64_t k = 0;
    while (auto e = it->GetNext()) out[k++] = e->component(0).int64();
    *count = k;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// Value filters (the reference's keep_even / keep_odd, pipeline_spec.cpp:
// 234-243): from_memory(IntRange(n)) -> map(x * a + b) -> filter(keep_*)
// [-> shuffle(buffer, 42)] -> batch(64) [-> Optimize: map_filter_fusion,
// map_batch_fusion].  Emits the values.
int ref_filter_values(int64_t n, int64_t a, int64_t b, int odd, int64_t shuffle_buffer, int optimize,
                      int64_t* out, int64_t* count, char* root_kind, size_t root_len) {
  try {
    UdfRegistry reg;
    const std::string f = "affine(" + std::to_string(a) + "," + std::to_string(b) + ")";
    RegisterAffine(reg, f, a, b);
    reg.RegisterPredicate("keep_even", [](const Element& e) { return e.component(0).int64() % 2 == 0; });
    reg.RegisterPredicate("keep_odd", [](const Element& e) { return e.component(0).int64() % 2 != 0; });
    DatasetGraph g = ops::Map(ops::FromMemory(IntRange(n), reg), f, 1, reg);
    g = ops::Filter(g, odd ? "keep_odd" : "keep_even", reg);
    if (shuffle_buffer > 0) g = ops::Shuffle(g, shuffle_buffer, uint64_t{42}, reg);
    g = ops::Batch(g, 64, false, reg);
    if (optimize) g = Optimize(g, RuleSet::Default(), reg).first;
    std::string chain;  // root first: kind<-kind<-...
    for (const DatasetNode* nd = g.root().get(); nd; nd = nd->inputs().empty() ? nullptr : nd->inputs()[0].get())
      chain += std::string(chain.empty() ? "" : "<-") + NodeKindName(nd->kind());
    std::snprintf(root_kind, root_len, "%s", chain.c_str());
    auto it = MakeIterator(g, reg, Seeded(1));
    int64_t k = 0;
    while (auto e = it->GetNext())
      for (const auto& v : e->component(0).items()) out[k++] = v.int64();
    *count = k;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// Interleave over readers of unequal lengths: from_memory(0..S-1) [->
// shard(k, g)] -> interleave(reader: input s opens lengths[s] records valued
// start_s + r, start_s = sum of earlier lengths; cycle, parallel).
int ref_interleave_var_ids(int64_t num_sources, const int64_t* lengths, int64_t shard_k, int64_t shard_g,
                           int64_t cycle, int64_t parallel, uint64_t base_seed, int64_t* out, int64_t* count) {
  try {
    UdfRegistry reg;
    std::vector<int64_t> len(lengths, lengths + num_sources), start(num_sources + 1, 0);
    for (int64_t s = 0; s < num_sources; ++s) start[s + 1] = start[s] + len[s];
    reg.RegisterDataset(
        "reader_var",
        [&reg, len, start](const Element& e) {
          const int64_t s = e.component(0).int64();
          std::vector<Element> recs;
          for (int64_t r = 0; r < len[s]; ++r) recs.push_back(Element::Scalar(Value::Int64(start[s] + r)));
          if (recs.empty())  // an empty reader: one element filtered out (from_memory must be non-empty)
            return ops::Filter(ops::FromMemory({Element::Scalar(Value::Int64(0))}, reg), "none", reg);
          return ops::FromMemory(std::move(recs), reg);
        },
        ElementSpec({TypeSpec::Int64()}));
    reg.RegisterPredicate("none", [](const Element&) { return false; });
    DatasetGraph g = ops::FromMemory(IntRange(num_sources), reg);
    if (shard_k > 0) g = ops::Shard(g, shard_k, shard_g, reg);
    g = ops::Interleave(g, "reader_var", cycle, parallel, reg);
    auto it = MakeIterator(g, reg, Seeded(base_seed));
    int64_t k = 0;
    while (auto e = it->GetNext()) out[k++] = e->component(0).int64();
    *count = k;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// CPU baseline timing (bench::Run methodology, src/bench.cpp:192-249): the
// image pipeline over `n` resident synthetic images with map parallelism
// `parallel`, optimized to map_and_batch, prefetch(prefetch).  One warm-up
// epoch is discarded; each measured epoch is a fresh iterator drained to EOF.
// Writes the per-epoch wall seconds into epoch_s[epochs].
int ref_time_image_pipeline(int mode, int in_h, int in_w, int out_h, int out_w,
                            uint64_t udf_seed, uint64_t pix_seed, int64_t n,
                            int64_t shuffle_buffer, uint64_t shuffle_seed,
                            int64_t batch, int64_t parallel, int64_t prefetch,
                            uint64_t base_seed, int epochs, double* epoch_s,
                            int64_t* elements_per_epoch) {
  try {
    UdfRegistry reg;
    ImagePipelineArgs a{{mode, in_h, in_w, out_h, out_w, udf_seed},
                        n, 0, 0, shuffle_buffer, 1, shuffle_seed, batch, 0,
                        parallel, prefetch, pix_seed};
    DatasetGraph g = BuildImageGraph(reg, a, SynthImages(n, in_h, in_w, pix_seed));
    for (int ep = 0; ep <= epochs; ++ep) {
      auto it = MakeIterator(g, reg, Seeded(base_seed));
      auto t0 = std::chrono::steady_clock::now();
      int64_t count = 0;
      while (auto e = it->GetNext()) count += static_cast<int64_t>(e->component(0).items().size());
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (ep > 0) epoch_s[ep - 1] = s;
      *elements_per_epoch = count;
    }
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// bench.py --impl reference: the reference pipeline for the image configs
// over a resident sample of `n` synthetic images, repeated indefinitely
// (repeat(INFINITE) above the shuffle), optimized to map_and_batch with
// num_parallel_calls = `parallel`, prefetch(2).  Pulls `warmup` batches,
// then times `steps` GetNext calls (one batch each).  Returns seconds.
int ref_time_image_steps(int mode, int in_h, int in_w, int out_h, int out_w, uint64_t udf_seed,
                         uint64_t pix_seed, int64_t n, int64_t shuffle_buffer, uint64_t shuffle_seed,
                         int64_t batch, int64_t parallel, int64_t warmup, int64_t steps,
                         double* seconds, int64_t* elements) {
  try {
    UdfRegistry reg;
    ImageUdfParams p{mode, in_h, in_w, out_h, out_w, udf_seed};
    RegisterImageUdf(reg, p);
    DatasetGraph g = ops::FromMemory(SynthImages(n, in_h, in_w, pix_seed), reg);
    if (shuffle_buffer > 0) g = ops::Shuffle(g, shuffle_buffer, shuffle_seed, reg);
    g = ops::Repeat(g, kInfiniteRepeat, reg);
    g = ops::Map(g, ImageUdfName(p), parallel, reg);
    g = ops::Batch(g, batch, false, reg);
    g = ops::Prefetch(g, kAutotune, reg);  // prefetch(AUTOTUNE)
    g = Optimize(g, RuleSet::Default(), reg).first;
    auto it = MakeIterator(g, reg, Seeded(1));
    for (int64_t i = 0; i < warmup; ++i) it->GetNext();
    int64_t count = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < steps; ++i) {
      auto e = it->GetNext();
      count += static_cast<int64_t>(e->component(0).items().size());
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *elements = count;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// CPU baseline for the chain configs: from_memory(n synthetic images) ->
// shuffle -> repeat -> one map node per chain step (num_parallel_calls =
// parallel; map_map_fusion composes them) -> batch -> prefetch(AUTOTUNE),
// optimized; `steps` timed GetNext calls after `warmup`.
int ref_time_chain_steps(const orc_map_step* chain, int nsteps, int in_h, int in_w, uint64_t pix_seed, int64_t n,
                         int64_t shuffle_buffer, uint64_t shuffle_seed, int64_t batch, int64_t parallel,
                         int64_t warmup, int64_t steps, double* seconds, int64_t* elements) {
  try {
    UdfRegistry reg;
    DatasetGraph g = ops::FromMemory(SynthImages(n, in_h, in_w, pix_seed), reg);
    if (shuffle_buffer > 0) g = ops::Shuffle(g, shuffle_buffer, shuffle_seed, reg);
    g = ops::Repeat(g, kInfiniteRepeat, reg);
    int h = in_h, w = in_w, f = 0;
    for (int i = 0; i < nsteps; ++i) {
      g = ops::Map(g, RegisterChainStep(reg, chain[i], i, h, w, f), parallel, reg);
      int oh, ow, of;
      if (orc_chain_output(&chain[i], 1, h, w, &oh, &ow, &of)) throw std::runtime_error("bad chain");
      h = oh;
      w = ow;
      f = f || of;
    }
    g = ops::Batch(g, batch, false, reg);
    g = ops::Prefetch(g, kAutotune, reg);
    g = Optimize(g, RuleSet::Default(), reg).first;
    auto it = MakeIterator(g, reg, Seeded(1));
    for (int64_t i = 0; i < warmup; ++i) it->GetNext();
    int64_t count = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < steps; ++i) {
      auto e = it->GetNext();
      count += static_cast<int64_t>(e->component(0).items().size());
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *elements = count;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// CPU baseline for cfg5: from_memory(file ids 0..files-1) -> interleave(
// reader: file s opens `records` images valued (s * records + r, image bytes),
// cycle, parallel) -> shuffle -> repeat -> map(img udf, parallel) -> batch ->
// prefetch(AUTOTUNE), optimized.  The readers copy their records out of a
// resident sample of `sample` synthetic images (record i = sample[i % sample]).
int ref_time_interleave_image_steps(int mode, int in_h, int in_w, int out_h, int out_w, uint64_t udf_seed,
                                    uint64_t pix_seed, int64_t sample, int64_t files, int64_t records,
                                    int64_t cycle, int64_t interleave_parallel, int64_t shuffle_buffer,
                                    uint64_t shuffle_seed, int64_t batch, int64_t parallel, int64_t warmup,
                                    int64_t steps, double* seconds, int64_t* elements) {
  try {
    UdfRegistry reg;
    ImageUdfParams p{mode, in_h, in_w, out_h, out_w, udf_seed};
    RegisterImageUdf(reg, p);
    auto imgs = std::make_shared<std::vector<Element>>(SynthImages(sample, in_h, in_w, pix_seed));
    reg.RegisterDataset(
        "image_reader",
        [&reg, imgs, records](const Element& e) {
          const int64_t s = e.component(0).int64();
          std::vector<Element> recs;
          for (int64_t r = 0; r < records; ++r) {
            const int64_t id = s * records + r;
            std::vector<Value> c;
            c.push_back(Value::Int64(id));
            c.push_back(Value::Bytes((*imgs)[static_cast<size_t>(id) % imgs->size()].component(1).bytes()));
            recs.push_back(Element(std::move(c)));
          }
          return ops::FromMemory(std::move(recs), reg);
        },
        ElementSpec({TypeSpec::Int64(), TypeSpec::Bytes()}));
    DatasetGraph g = ops::FromMemory(IntRange(files), reg);
    g = ops::Interleave(g, "image_reader", cycle, interleave_parallel, reg);
    if (shuffle_buffer > 0) g = ops::Shuffle(g, shuffle_buffer, shuffle_seed, reg);
    g = ops::Repeat(g, kInfiniteRepeat, reg);
    g = ops::Map(g, ImageUdfName(p), parallel, reg);
    g = ops::Batch(g, batch, false, reg);
    g = ops::Prefetch(g, kAutotune, reg);
    g = Optimize(g, RuleSet::Default(), reg).first;
    auto it = MakeIterator(g, reg, Seeded(1));
    for (int64_t i = 0; i < warmup; ++i) it->GetNext();
    int64_t count = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < steps; ++i) {
      auto e = it->GetNext();
      count += static_cast<int64_t>(e->component(0).items().size());
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *elements = count;
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// CPU baseline for cfg1 (range -> map -> batch, optimized).
int ref_time_range_map_batch(int64_t n, int64_t batch, int64_t parallel,
                             int epochs, double* epoch_s) {
  try {
    UdfRegistry reg;
    RegisterAffine(reg, "affine(3,1)", 3, 1);
    DatasetGraph g = ops::FromMemory(IntRange(n), reg);
    g = ops::Map(g, "affine(3,1)", parallel, reg);
    g = ops::Batch(g, batch, false, reg);
    g = Optimize(g, RuleSet::Default(), reg).first;
    for (int ep = 0; ep <= epochs; ++ep) {
      auto it = MakeIterator(g, reg, Seeded(1));
      auto t0 = std::chrono::steady_clock::now();
      while (auto e = it->GetNext()) {
      }
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (ep > 0) epoch_s[ep - 1] = s;
    }
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// CPU baseline for cfg4: token sequences -> filter(len <= max_keep) ->
// batch (the reference has no padded_batch; its ragged Batch is the same
// selection and order), optimized.  Elements are built once, outside timing.
int ref_time_filter_batch_tokens(int64_t n, uint64_t len_seed, uint32_t max_len, uint64_t tok_seed,
                                 int32_t max_keep, int64_t batch, int epochs, double* epoch_s) {
  try {
    UdfRegistry reg;
    std::string pred = "len_le(" + std::to_string(max_keep) + ")";
    reg.RegisterPredicate(pred, [max_keep](const Element& e) {
      return static_cast<int64_t>(e.component(0).items().size()) <= max_keep;
    });
    std::vector<int32_t> lens(static_cast<size_t>(n));
    orc_synth_lengths(len_seed, max_len, static_cast<uint64_t>(n), lens.data());
    std::vector<Element> elems;
    elems.reserve(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      std::vector<Value> toks;
      toks.reserve(static_cast<size_t>(lens[i]));
      for (int32_t j = 0; j < lens[i]; ++j) toks.push_back(Value::Int64(orc_synth_token(tok_seed, i, j)));
      elems.push_back(Element::Scalar(Value::List(std::move(toks))));
    }
    DatasetGraph g = ops::FromMemory(std::move(elems), reg);
    g = ops::Filter(g, pred, reg);
    g = ops::Batch(g, batch, false, reg);
    g = Optimize(g, RuleSet::Default(), reg).first;
    for (int ep = 0; ep <= epochs; ++ep) {
      auto it = MakeIterator(g, reg, Seeded(1));
      auto t0 = std::chrono::steady_clock::now();
      while (auto e = it->GetNext()) {
      }
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (ep > 0) epoch_s[ep - 1] = s;
    }
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// Graph serialization known answers (formats.md "Graph serialization",
// src/serialize.cpp Serialize / GraphFingerprint) for the pipeline shapes
// both engines express.  which:
//   0 from_memory(0..9) -> map(affine(3,1), 4) -> batch(4)
//   1 the same, Optimize(Default)                    (-> map_and_batch)
//   2 from_memory(0..99) -> shuffle(10, seed 42) -> repeat(3) -> batch(8)
//     -> prefetch(AUTOTUNE), Optimize(Default)       (shuffle_repeat fusion)
//   3 from_memory(0..63) -> shard(4, 1) -> shuffle(50) -> map(affine(3,1), -1)
//     -> map(affine(2,0), 2) -> batch(16, drop) -> prefetch(2), Optimize
//   4 from_memory(0..7) -> interleave(reader(3), 2, 1) -> batch(5)
//   5 from_file(part-0.rec, part-1.rec) -> batch(2)
// Writes the serialized bytes (up to cap) and the fingerprint as 64 hex chars.
namespace {
DatasetGraph KnownPipeline(int which, UdfRegistry& reg) {
    RegisterAffine(reg, "affine(3,1)", 3, 1);
    RegisterAffine(reg, "affine(2,0)", 2, 0);
    reg.RegisterDataset(
        "reader(3)",
        [&reg](const Element& e) {
          std::vector<Element> recs;
          for (int64_t r = 0; r < 3; ++r) recs.push_back(Element::Scalar(Value::Int64(e.component(0).int64() * 3 + r)));
          return ops::FromMemory(std::move(recs), reg);
        },
        ElementSpec({TypeSpec::Int64()}));
    DatasetGraph g;
    switch (which) {
      case 0:
      case 1:
        g = ops::Batch(ops::Map(ops::FromMemory(IntRange(10), reg), "affine(3,1)", 4, reg), 4, false, reg);
        if (which == 1) g = Optimize(g, RuleSet::Default(), reg).first;
        break;
      case 2:
        g = ops::Shuffle(ops::FromMemory(IntRange(100), reg), 10, uint64_t{42}, reg);
        g = ops::Prefetch(ops::Batch(ops::Repeat(g, 3, reg), 8, false, reg), kAutotune, reg);
        g = Optimize(g, RuleSet::Default(), reg).first;
        break;
      case 3:
        g = ops::Shuffle(ops::Shard(ops::FromMemory(IntRange(64), reg), 4, 1, reg), 50, std::nullopt, reg);
        g = ops::Map(ops::Map(g, "affine(3,1)", kAutotune, reg), "affine(2,0)", 2, reg);
        g = ops::Prefetch(ops::Batch(g, 16, true, reg), 2, reg);
        g = Optimize(g, RuleSet::Default(), reg).first;
        break;
      case 4:
        g = ops::Batch(ops::Interleave(ops::FromMemory(IntRange(8), reg), "reader(3)", 2, 1, reg), 5, false, reg);
        break;
      case 5:
        g = ops::Batch(ops::FromFile({"part-0.rec", "part-1.rec"}, reg), 2, false, reg);
        break;
      default:
        throw PipelineError(ErrorCode::kInvalidAttr, "unknown pipeline");
    }
    return g;
}
}  // namespace

int ref_serialize_pipeline(int which, uint8_t* buf, size_t cap, size_t* len, char* fp_hex) {
  try {
    UdfRegistry reg;
    DatasetGraph g = KnownPipeline(which, reg);
    const std::string bytes = Serialize(g);
    *len = bytes.size();
    std::memcpy(buf, bytes.data(), std::min(cap, bytes.size()));
    const std::string hex = GraphFingerprint(g).ToHex();
    std::memcpy(fp_hex, hex.c_str(), hex.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

// DPC1 checkpoint (src/checkpoint.cpp Save) of known pipeline `which` after
// `k` GetNext calls, base seed 1, deterministic.
int ref_checkpoint_after(int which, int64_t k, uint8_t* buf, size_t cap, size_t* len) {
  try {
    UdfRegistry reg;
    DatasetGraph g = KnownPipeline(which, reg);
    auto it = MakeIterator(g, reg, Seeded(1));
    for (int64_t i = 0; i < k; ++i)
      if (!it->GetNext()) throw PipelineError(ErrorCode::kInvalidAttr, "pipeline ended before k");
    const CheckpointBlob blob = Save(*it);
    *len = blob.bytes.size();
    std::memcpy(buf, blob.bytes.data(), std::min(cap, blob.bytes.size()));
    return 0;
  } catch (const std::exception& e) {
    return Fail(e);
  }
}

int ref_hardware_concurrency(void) {
  return static_cast<int>(std::thread::hardware_concurrency());
}

}  // extern "C"
