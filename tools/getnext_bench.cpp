// Host cost of GetNext + drop on a device-light pipeline (cfg1 shape): the
// per-batch overhead that bounds small-batch configs.  Development aid.
//   g++ -std=c++20 -O2 -Iinclude -I/usr/local/cuda/include tools/getnext_bench.cpp \
//       -Lpaper_2101_12127_b200/lib -ldpcuda -Wl,-rpath,$PWD/paper_2101_12127_b200/lib -o /tmp/gnb
#include <chrono>
#include <cstdio>

#include "dpb200/datapipe.hpp"

using namespace datapipe::b200;

int main() {
  UdfRegistry reg;
  reg.RegisterAffine("a", 3, 1);
  DatasetGraph g = ops::Repeat(ops::Batch(ops::Map(ops::Range(1 << 24, reg), "a", 1, reg), 1024, false, reg), -1, reg);
  IteratorOptions o;
  o.seed_override = 1;
  auto it = MakeIterator(Optimize(g, RuleSet::Default(), reg).first, reg, o);
  for (int i = 0; i < 20000; ++i) it->GetNext();
  const int n = 200000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) it->GetNext();
  const double ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count() / n;
  std::printf("GetNext + drop: %.1f ns per batch (%.3g elements/s host bound)\n", ns, 1024 / ns * 1e9);
  return 0;
}
