// Multi-threaded stress of the device pipeline's host runtime, built with
// ThreadSanitizer against a TSAN-instrumented libdpcuda.so
// (tests/test_gpu_tsan.py): several threads call GetNext on one iterator
// (GetNext is thread-safe, as the reference's PipelineIterator), hand the
// batches to other threads that drop them after queueing consumer-stream
// work, while another thread takes checkpoints (Save) and reads Metrics().
// Batches are small and launch groups short, so slots are reused (the
// lease / release-event path of runtime.cpp) thousands of times.
// Prints "stress ok batches=N unique=N" when every batch id was delivered
// exactly once.
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <deque>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "dpb200/datapipe.hpp"

using namespace datapipe::b200;

int main() {
  UdfRegistry reg;
  reg.RegisterAffine("a", 1, 0);
  const int64_t n = 1 << 18;
  DatasetGraph g = ops::Batch(ops::Map(ops::Range(n, reg), "a", 1, reg), 64, false, reg);
  g = ops::Prefetch(g, kAutotune, reg);
  auto opt = Optimize(g, RuleSet::Default(), reg).first;
  cudaStream_t consumer;
  cudaStreamCreateWithFlags(&consumer, cudaStreamNonBlocking);
  IteratorOptions o;
  o.seed_override = 3;
  o.consumer_stream = consumer;
  o.launch_batches = 2;
  auto it = MakeIterator(opt, reg, o);

  std::mutex mu;
  std::condition_variable cv;
  std::deque<Element> queue;
  bool done = false;
  std::atomic<int64_t> batches{0};
  std::mutex seen_mu;
  std::set<int64_t> firsts;
  int64_t* dev_sink = nullptr;
  cudaMalloc(&dev_sink, sizeof(int64_t) * 64);

  auto producer = [&] {
    for (;;) {
      auto e = it->GetNext();
      if (!e) break;
      batches.fetch_add(1);
      std::lock_guard<std::mutex> lk(mu);
      queue.push_back(std::move(*e));
      cv.notify_one();
    }
  };
  auto dropper = [&] {
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return !queue.empty() || done; });
      if (queue.empty()) return;
      Element e = std::move(queue.front());
      queue.pop_front();
      lk.unlock();
      const Tensor& t = e.component(0).tensor();
      // consumer-stream work on the batch, queued before the drop
      cudaStreamWaitEvent(consumer, static_cast<cudaEvent_t>(t.ready), 0);
      cudaMemcpyAsync(dev_sink, t.data, sizeof(int64_t), cudaMemcpyDeviceToDevice, consumer);
      int64_t first = -1;
      cudaMemcpyAsync(&first, t.data, sizeof(int64_t), cudaMemcpyDeviceToHost, consumer);
      cudaStreamSynchronize(consumer);
      {
        std::lock_guard<std::mutex> sl(seen_mu);
        firsts.insert(first);
      }
    }  // the element (and its lease) is dropped here, on this thread
  };
  std::atomic<bool> stop_observer{false};
  auto observer = [&] {
    while (!stop_observer.load()) {
      (void)it->Save();
      (void)it->Metrics();
      std::this_thread::yield();
    }
  };

  std::vector<std::thread> ths;
  for (int i = 0; i < 3; ++i) ths.emplace_back(dropper);
  std::thread obs(observer);
  std::vector<std::thread> prods;
  for (int i = 0; i < 3; ++i) prods.emplace_back(producer);
  for (auto& t : prods) t.join();
  {
    std::lock_guard<std::mutex> lk(mu);
    done = true;
  }
  cv.notify_all();
  for (auto& t : ths) t.join();
  stop_observer = true;
  obs.join();
  cudaDeviceSynchronize();
  const int64_t expect = n / 64;
  std::printf("stress %s batches=%lld unique=%zu\n",
              batches.load() == expect && static_cast<int64_t>(firsts.size()) == expect ? "ok" : "FAILED",
              static_cast<long long>(batches.load()), firsts.size());
  cudaFree(dev_sink);
  cudaStreamDestroy(consumer);
  return 0;
}
