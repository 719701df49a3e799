// A reference user's program, ported by changing the include and namespace:
// builds the cfg1 graph with ops::*, optimizes it to map_and_batch, drains
// it with GetNext and prints the SURVEY.md Appendix A known answers; then a
// cfg2-shaped image pipeline, with a checkpoint Save/Restore in the middle;
// the reference's graph serialization / fingerprint; bucket_by_length.
#include <cuda_runtime.h>

#include <cstdio>
#include <numeric>
#include <vector>

#include "dpb200/datapipe.hpp"

using namespace datapipe::b200;

int main() {
  UdfRegistry reg;
  reg.RegisterAffine("affine(3,1)", 3, 1);
  DatasetGraph g = ops::Batch(ops::Map(ops::Range(1000000, reg), "affine(3,1)", 1, reg), 1024, false, reg);
  auto [opt, report] = Optimize(g, RuleSet::Default(), reg);
  IteratorOptions o;
  o.seed_override = 1;
  auto it = MakeIterator(opt, reg, o);
  uint64_t h = 0xcbf29ce484222325ULL;
  int64_t sum = 0, batches = 0, last = 0;
  std::vector<int64_t> host;
  while (auto e = it->GetNext()) {
    const Tensor& t = e->component(0).tensor();
    host.resize(t.shape[0]);
    cudaEventSynchronize(static_cast<cudaEvent_t>(t.ready));
    cudaMemcpy(host.data(), t.data, t.nbytes(), cudaMemcpyDeviceToHost);
    for (int64_t v : host) {
      h = (h ^ static_cast<uint64_t>(v)) * 0x100000001b3ULL;
      sum += v;
    }
    last = t.shape[0];
    ++batches;
  }
  std::printf("cfg1 root=%s batches=%lld last=%lld sum=%lld fnv=%016llx\n", NodeKindName(opt.root()->kind()),
              static_cast<long long>(batches), static_cast<long long>(last), static_cast<long long>(sum),
              static_cast<unsigned long long>(h));

  reg.RegisterRandomCropFlip("crop", 224, 224, 7, true);
  reg.RegisterNormalize("norm", {123.675f, 116.28f, 103.53f}, {58.395f, 57.12f, 57.375f});
  auto images = SynthImages(4096, 256, 256, 0x5EED);
  DatasetGraph p = ops::TensorSlices(images, reg);
  p = ops::Shuffle(p, 1000, 42, reg);
  p = ops::Map(p, "crop", kAutotune, reg);
  p = ops::Map(p, "norm", kAutotune, reg);
  p = ops::Prefetch(ops::Batch(p, 256, false, reg), kAutotune, reg);
  auto popt = Optimize(p, RuleSet::Default(), reg).first;
  auto pit = MakeIterator(popt, reg, o);
  for (int i = 0; i < 5; ++i) pit->GetNext();
  std::string blob = pit->Save();
  auto a = pit->GetNext();
  auto restored = Restore(popt, reg, blob);
  auto b = restored->GetNext();
  std::vector<int64_t> ia(256), ib(256);
  cudaDeviceSynchronize();
  cudaMemcpy(ia.data(), a->component(0).tensor().data, 2048, cudaMemcpyDeviceToHost);
  cudaMemcpy(ib.data(), b->component(0).tensor().data, 2048, cudaMemcpyDeviceToHost);
  std::printf("cfg2 restore_matches=%d first_id=%lld plan:\n%s", ia == ib ? 1 : 0, static_cast<long long>(ia[0]),
              pit->LoweringPlan().c_str());

  // DPG1 bytes + fingerprint: from_memory(0..9) -> map(affine(3,1), 4) -> batch(4)
  std::vector<int64_t> ten(10);
  std::iota(ten.begin(), ten.end(), 0);
  DatasetGraph s = ops::Batch(ops::Map(ops::FromMemory(ten, reg), "affine(3,1)", 4, reg), 4, false, reg);
  const std::string bytes = Serialize(s);
  std::printf("fingerprint=%s roundtrip=%d\n", FingerprintHex(GraphFingerprint(s)).c_str(),
              Serialize(Deserialize(bytes, reg)) == bytes ? 1 : 0);

  // bucket_by_length over 5,000 token sequences
  auto tokens = SynthTokens(5000, 300, 6, 6);
  DatasetGraph bk = ops::BucketByLength(ops::TokenSequences(tokens, reg), {100, 200}, {16, 8, 4}, 0, false, reg);
  auto bit = MakeIterator(bk, reg, o);
  int64_t rows = 0, nb = 0;
  while (auto e = bit->GetNext()) {
    rows += e->component(1).tensor().shape[0];
    ++nb;
  }
  std::printf("bucket rows=%lld batches=%lld\n", static_cast<long long>(rows), static_cast<long long>(nb));

  // (image, label) elements through RandomResizedCrop (crop >> resize >>
  // normalize, K9), with per-node metrics and the tuner's state
  std::vector<int64_t> labels(512);
  for (size_t i = 0; i < labels.size(); ++i) labels[i] = static_cast<int64_t>(i % 10);
  reg.RegisterRandomCropFlip("crop160", 160, 160, 3, true);
  reg.RegisterResizeBilinear("resize224", 224, 224);
  DatasetGraph rrc = ops::TensorSlices(WithLabels(SynthImages(512, 256, 256, 0x5EED), labels.data(), 512), reg);
  rrc = ops::Map(ops::Map(ops::Map(ops::Shuffle(rrc, 128, 9, reg), "crop160", 1, reg), "resize224", 1, reg), "norm",
                 1, reg);
  rrc = ops::Prefetch(ops::Batch(rrc, 64, false, reg), kAutotune, reg);
  auto rit = MakeIterator(Optimize(rrc, RuleSet::Default(), reg).first, reg, o);
  int64_t label_sum = 0, imgs = 0;
  std::vector<int64_t> lab(64);
  while (auto e = rit->GetNext()) {
    const Tensor& l = e->component(2).tensor();
    cudaEventSynchronize(static_cast<cudaEvent_t>(l.ready));
    cudaMemcpy(lab.data(), l.data, l.nbytes(), cudaMemcpyDeviceToHost);
    for (int64_t k = 0; k < l.shape[0]; ++k) label_sum += lab[k];
    imgs += e->component(1).tensor().shape[0];
  }
  std::printf("rrc images=%lld label_sum=%lld shape=%s\n", static_cast<long long>(imgs),
              static_cast<long long>(label_sum), rrc.element_spec().ToString().c_str());
  for (const auto& row : rit->Metrics())
    std::printf("metrics %s %s self_ns=%lld produced=%lld\n", row.path.c_str(), row.label.c_str(),
                static_cast<long long>(row.self_time_ns), static_cast<long long>(row.elements_produced));
  return ia == ib ? 0 : 1;
}
