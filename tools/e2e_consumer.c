/* e2e_consumer.c -- the end-to-end consumer loop of bench.py's token
 * configs, in C over the C ABI (include/dpcuda_pipeline.h): what a C / FFI
 * user of the pipeline writes.  Each batch is fetched with
 * dp_iterator_get_next, waited on until its bytes are in pinned host memory
 * (host_output iterator: dp_batch_wait), read on the host (its first and
 * last token words folded into a checksum: the bytes arrived) and released.
 * Python's per-call overhead (~10 us per batch through ctypes) would
 * otherwise bound the tiny (128-sequence) token batches.  Benchmark
 * harness, not product: built by __graft_entry__.build() into
 * tools/bin/libdpe2e.so.
 */
#include <stdint.h>

#include "dpcuda_pipeline.h"

/* n batches; *rows += rows batched (ragged: row_splits - 1); returns DP_OK,
 * DP_ERR_END_OF_SEQUENCE (with *done = batches consumed) or an error. */
int dpe2e_consume_host_batches(dp_iterator* it, int64_t n, int ragged, int64_t* rows, uint64_t* checksum,
                               int64_t* done) {
  *done = 0;
  for (int64_t i = 0; i < n; ++i) {
    dp_batch b;
    int st = dp_iterator_get_next(it, &b);
    if (st) return st;
    st = dp_batch_wait(&b);
    if (st) {
      dp_batch_release(&b);
      return st;
    }
    const dp_tensor* c0 = &b.components[0];
    const dp_tensor* c1 = &b.components[1];
    *rows += ragged ? c1->shape[0] - 1 : c1->shape[0];
    int64_t words = 1;
    for (int d = 0; d < c0->ndim; ++d) words *= c0->shape[d];
    if (words > 0 && c0->on_host) {
      const int32_t* w = (const int32_t*)c0->data;
      *checksum += (uint64_t)(uint32_t)w[0] * 0x9e3779b97f4a7c15ULL + (uint32_t)w[words - 1];
    }
    st = dp_batch_release(&b);
    if (st) return st;
    ++*done;
  }
  return 0;
}
