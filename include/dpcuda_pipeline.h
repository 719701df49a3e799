/*
 * dpcuda_pipeline.h -- C ABI of the Dataset / Iterator operator API
 * (libdpcuda.so).  Each entry point is the FFI binding of one reference
 * operator; the reference interface it replaces is cited beside it
 * (paths under /root/reference/proj/).  Status codes: include/dpcuda.h.
 *
 * Ownership: every dp_registry / dp_graph / dp_iterator handle is released
 * with its *_release / *_destroy call; a dp_batch returned by
 * dp_iterator_get_next holds a lease on a device prefetch slot until
 * dp_batch_release.
 */
#ifndef DPCUDA_PIPELINE_H_
#define DPCUDA_PIPELINE_H_

#include <stddef.h>
#include <stdint.h>

#include "dpcuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dp_registry dp_registry;
typedef struct dp_graph dp_graph;
typedef struct dp_iterator dp_iterator;
typedef struct dp_source dp_source;

#define DP_AUTOTUNE (-1)
#define DP_INFINITE (-1)

/* ---- UDF registry: include/datapipe/udf.hpp:41-87 (UdfRegistry) ---- */
int dp_registry_create(dp_registry** out);
void dp_registry_destroy(dp_registry* reg);
/* map x -> x*a + b on int64 elements (the cfg1 UDF) */
int dp_registry_register_affine(dp_registry* reg, const char* name, int64_t a, int64_t b);
/* random crop (Philox key = seed, counter = element id) + optional flip */
int dp_registry_register_random_crop_flip(dp_registry* reg, const char* name, int64_t crop_h, int64_t crop_w,
                                          uint64_t seed, int flip);
/* bilinear resize, half-pixel centres */
int dp_registry_register_resize_bilinear(dp_registry* reg, const char* name, int64_t out_h, int64_t out_w);
/* per-channel (x - mean[c]) / std[c] to fp32 */
int dp_registry_register_normalize(dp_registry* reg, const char* name, const float mean[3], const float stdv[3]);
/* cast u8 -> fp32 (the north star's Map library "cast"): exact, = normalize(mean 0, std 1) */
int dp_registry_register_cast(dp_registry* reg, const char* name);
/* center crop (offsets ((H - h) / 2, (W - w) / 2), no flip; dtype kept) */
int dp_registry_register_center_crop(dp_registry* reg, const char* name, int64_t crop_h, int64_t crop_w);
/* per-channel x * scale[c] + shift[c] on an image -> fp32 (two rounded ops) */
int dp_registry_register_image_affine(dp_registry* reg, const char* name, const float scale[3], const float shift[3]);
/* predicate: keep sequences with length <= max_len */
int dp_registry_register_length_filter(dp_registry* reg, const char* name, int64_t max_len);
/* predicate on int64 element values (after the maps beneath the filter):
 * a conjunction of 1..8 terms (dp_predicate_term, include/dpcuda.h) */
int dp_registry_register_value_filter(dp_registry* reg, const char* name, const dp_predicate_term* terms,
                                      int num_terms);
/* keep_even / keep_odd / keep_all (pipeline_spec.cpp:234-243 EnsurePredicates) */
int dp_registry_register_standard_predicates(dp_registry* reg);
/* interleave dataset UDF: element x opens records x*records .. x*records+records-1 */
int dp_registry_register_record_reader(dp_registry* reg, const char* name, int64_t records);
/* decode a from_file record holding a raw u8 HWC image of h x w x 3 ->
 * (int64 ordinal, u8[h,w,3]); must be the first map after from_file */
int dp_registry_register_decode_raw(dp_registry* reg, const char* name, int64_t h, int64_t w);
int dp_registry_contains(const dp_registry* reg, const char* name);

/* ---- sources (new kinds) ---- */
int dp_source_synthetic_images(int64_t count, int64_t h, int64_t w, uint64_t seed, int device, dp_source** out);
/* Sharded residency: only elements p % num_shards == index of a global_count
 * dataset are generated/held; graphs must start with shard(num_shards, index). */
int dp_source_synthetic_images_sharded(int64_t global_count, int64_t h, int64_t w, uint64_t seed,
                                       int64_t num_shards, int64_t index, int device, dp_source** out);
/* synthetic records of an interleave over `num_files` inputs of
 * `records_per_file` images each (record r of file x = image id x * R + r);
 * this process holds only the files x % num_shards == index (block residency:
 * the graph applies shard(num_shards, index) to the interleave's inputs) */
int dp_source_synthetic_records_sharded(int64_t num_files, int64_t records_per_file, int64_t h, int64_t w,
                                        uint64_t seed, int64_t num_shards, int64_t index, int device,
                                        dp_source** out);
/* a view of `src` declaring that it holds shard `index` of `num_shards` of a
 * `global_count`-element dataset, in blocks of `block` consecutive positions
 * (1: element shards; R: the record files of an interleave's shard) */
int dp_source_as_shard(const dp_source* src, int64_t global_count, int64_t num_shards, int64_t index,
                       int64_t block, dp_source** out);
int dp_source_images_from_host(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device,
                               dp_source** out);
/* `images` with an int64 label per held row (copied): tensor_slices over it
 * yields (int64 id, u8 image, int64 label) elements -- FromMemory's tuple
 * elements (include/datapipe/graph.hpp:136, element.hpp:30-184); maps
 * transform the image and pass the label through, Batch stacks it. */
int dp_source_with_labels(const dp_source* images, const int64_t* labels, int64_t count, dp_source** out);
/* pinned/registered host memory read by the kernels over PCIe (end-to-end runs; not copied) */
int dp_source_images_pinned_host(const uint8_t* data, int64_t count, int64_t h, int64_t w, int device,
                                 dp_source** out);
int dp_source_synthetic_tokens(int64_t count, uint32_t max_len, uint64_t len_seed, uint64_t tok_seed, int device,
                               dp_source** out);
int dp_source_tokens_from_host(const int32_t* lengths, int64_t count, const int32_t* tokens, int device,
                               dp_source** out);
/* token sequences in pinned, device-mapped host memory (copied in), read by the kernels over PCIe */
int dp_source_tokens_pinned_host(const int32_t* lengths, int64_t count, const int32_t* tokens, int device,
                                 dp_source** out);
/* length-prefixed record files (formats.md:67-74) read in order into device
 * memory: the records of an interleave over files (file x = input element x,
 * every file holding the reader's record count; ops::Interleave over
 * ops::FromFile readers, runtime.cpp:1044-1128) */
int dp_source_records_from_files(const char* const* paths, int64_t num_paths, int device, dp_source** out);
/* only the files f % num_shards == index are read (each process of a
 * sharded interleave reads its own files; held files must hold equal counts) */
int dp_source_records_from_files_sharded(const char* const* paths, int64_t num_paths, int64_t num_shards,
                                         int64_t index, int device, dp_source** out);
void dp_source_release(dp_source* src);

/* ---- graph builders: include/datapipe/graph.hpp:134-165 (ops::*) ---- */
int dp_graph_range(const dp_registry* reg, int64_t n, dp_graph** out);                  /* source synthetic count=n */
int dp_graph_from_memory_i64(const dp_registry* reg, const int64_t* values, int64_t n, int device,
                             dp_graph** out);                                           /* ops::FromMemory */
int dp_graph_tensor_slices(const dp_registry* reg, const dp_source* images, dp_graph** out);
/* ops::FromFile (graph.hpp:137): length-prefixed record files (formats.md:67-74)
 * read in order into device memory.  kMissingFile / kMalformedInput as the
 * reference's FromFileIterator (runtime.cpp:416-474), raised here, before any
 * iteration. */
int dp_graph_from_file(const dp_registry* reg, const char* const* paths, int64_t num_paths, int device,
                       dp_graph** out);
/* WriteRecordFile (runtime.hpp:102-107): [u32 LE length][payload] per record;
 * payload i = data[offsets[i] .. offsets[i+1]) */
int dp_write_record_file(const char* path, const uint8_t* data, const int64_t* offsets, int64_t count);
int dp_graph_token_sequences(const dp_registry* reg, const dp_source* tokens, dp_graph** out);
int dp_graph_map(const dp_graph* in, const char* udf, int64_t num_parallel_calls, const dp_registry* reg,
                 dp_graph** out);                                                       /* ops::Map */
int dp_graph_filter(const dp_graph* in, const char* udf, const dp_registry* reg, dp_graph** out); /* ops::Filter */
int dp_graph_interleave(const dp_graph* in, const char* udf, int64_t cycle_length, int64_t num_parallel_calls,
                        const dp_source* records, const dp_registry* reg, dp_graph** out); /* ops::Interleave */
int dp_graph_batch(const dp_graph* in, int64_t batch_size, int drop_remainder, const dp_registry* reg,
                   dp_graph** out);                                                     /* ops::Batch */
int dp_graph_padded_batch(const dp_graph* in, int64_t batch_size, int64_t padding_value, int drop_remainder,
                          const dp_registry* reg, dp_graph** out);                      /* new kind */
/* tf.data bucket_by_sequence_length (new kind; K8): num_boundaries <= 31
 * increasing boundaries, num_boundaries + 1 batch sizes */
int dp_graph_bucket_by_length(const dp_graph* in, const int64_t* boundaries, int64_t num_boundaries,
                              const int64_t* batch_sizes, int64_t padding_value, int drop_remainder,
                              const dp_registry* reg, dp_graph** out);
int dp_graph_prefetch(const dp_graph* in, int64_t buffer_size, const dp_registry* reg, dp_graph** out);
int dp_graph_repeat(const dp_graph* in, int64_t count, const dp_registry* reg, dp_graph** out);
int dp_graph_shuffle(const dp_graph* in, int64_t buffer_size, int has_seed, uint64_t seed, const dp_registry* reg,
                     dp_graph** out);                                                   /* ops::Shuffle */
int dp_graph_shard(const dp_graph* in, int64_t num_shards, int64_t index, const dp_registry* reg,
                   dp_graph** out);                                                     /* ops::Shard */
/* Optimize(graph, RuleSet::Default() minus the comma-separated
 * disabled_rules, registry): include/datapipe/optimizer.hpp:73-75.
 * report (optional) receives RewriteReport::ToString(). */
int dp_graph_optimize(const dp_graph* in, dp_registry* reg, const char* disabled_rules, dp_graph** out,
                      char* report, size_t report_len);
/* kind name of the root node ("map_and_batch", ...) and the graph dump */
int dp_graph_root_kind(const dp_graph* g, char* buf, size_t len);
int dp_graph_to_string(const dp_graph* g, char* buf, size_t len);
/* Serialize (serialize.hpp; formats.md "Graph serialization"): DPG1 bytes.
 * Writes min(len, cap) bytes and sets *len to the full size (call with
 * cap = 0 to size the buffer). */
int dp_graph_serialize(const dp_graph* g, uint8_t* buf, size_t cap, size_t* len);
/* Deserialize: device sources with no reference encoding are re-bound from
 * `sources` in preorder (descriptor-checked, kValidationFailed otherwise). */
int dp_graph_deserialize(const dp_registry* reg, const uint8_t* bytes, size_t len, const dp_source* const* sources,
                         int64_t num_sources, int device, dp_graph** out);
/* GraphFingerprint (serialize.cpp:213-216): SHA-256 of the seed-zeroed
 * serialization as 64 hex chars + NUL (hex must hold 65 bytes). */
int dp_graph_fingerprint(const dp_graph* g, char* hex);
/* ParsePipelineSpec (pipeline_spec.hpp; formats.md "Pipeline description
 * text format") over the device UDF library.  Out: the graph, the `epochs`
 * trailer, the `options` trailer (has_seed / seed / deterministic) and the
 * `disable rule=` names comma-separated into `disabled` (len bytes). */
int dp_graph_from_spec(dp_registry* reg, const char* text, int device, dp_graph** out, int* epochs, int* has_seed,
                       uint64_t* seed, int* deterministic, char* disabled, size_t len);
void dp_graph_release(dp_graph* g);

/* ---- iterator: include/datapipe/runtime.hpp:35-100 ---- */
typedef struct {
  int deterministic;          /* IteratorOptions::deterministic */
  int has_seed_override;      /* IteratorOptions::seed_override */
  uint64_t seed_override;
  int device;                 /* CUDA device ordinal */
  void* consumer_stream;      /* cudaStream_t the batches are consumed on (NULL: iterator stream) */
  int host_output;            /* copy batches to pinned host memory */
  uint64_t slot_memory_budget;/* bytes of device prefetch slots (0: default 8 GiB) */
  uint64_t max_launch_bytes;  /* output bytes per fused launch (0: default) */
  int64_t launch_batches;     /* batches per fused launch, exactly (0: from max_launch_bytes) */
  int64_t first_launch_batches; /* batches of the first launch only (0: launch_batches) */
} dp_iterator_options;

typedef enum { DP_U8 = 0, DP_I32 = 1, DP_I64 = 2, DP_F32 = 3 } dp_dtype;

typedef struct {
  int dtype;          /* dp_dtype */
  int ndim;
  int64_t shape[6];
  void* data;         /* device pointer (or pinned host with host_output) */
  int on_host;
} dp_tensor;

typedef struct {
  void* handle;       /* lease; pass to dp_batch_release */
  int num_components;
  dp_tensor components[4];
  void* ready_event;  /* cudaEvent_t completing when the batch is written */
  int64_t index;      /* batch ordinal in the stream */
} dp_batch;

void dp_iterator_options_default(dp_iterator_options* o);
/* MakeIterator (runtime.hpp:98-100): validates UDFs (UnknownUdf) and lowers
 * the graph onto the device (InvalidAttr if it has no device lowering). */
int dp_iterator_create(const dp_graph* g, const dp_registry* reg, const dp_iterator_options* opt, dp_iterator** out);
/* PipelineIterator::GetNext (runtime.hpp:68): DP_OK with *batch filled, or
 * DP_ERR_END_OF_SEQUENCE (sticky). */
int dp_iterator_get_next(dp_iterator* it, dp_batch* batch);
/* Ends the lease.  The slot is rewritten only after the work queued on the
 * iterator's consumer_stream before this call. */
int dp_batch_release(dp_batch* batch);
/* Checkpoint (include/datapipe/checkpoint.hpp:36-49, DPC1 layout of
 * docs/formats.md:76-94).  dp_iterator_save writes the blob into buf (cap
 * bytes) and its size into *len; with buf == NULL or cap too small it only
 * reports *len and returns DP_ERR_INVALID_ATTR.  dp_iterator_restore validates
 * magic / version / fingerprint (CorruptBlob, VersionMismatch,
 * FingerprintMismatch) and seeks a fresh iterator to the saved position. */
int dp_iterator_save(const dp_iterator* it, void* buf, size_t cap, size_t* len);
int dp_iterator_restore(const dp_graph* g, const dp_registry* reg, const void* blob, size_t len,
                        const dp_iterator_options* opt, dp_iterator** out);
/* GetNext `n` times, dropping every batch (a consumer that only advances the
 * stream, like tf.data's skip); *produced = batches actually delivered. */
int dp_iterator_skip(dp_iterator* it, int64_t n, int64_t* produced);
/* Blocks the calling host thread until the batch is written (and, with
 * host_output, copied to its pinned host slot). */
int dp_batch_wait(const dp_batch* batch);
/* Copies a batch component to host memory (waits for the batch). */
int dp_tensor_copy_to_host(const dp_batch* batch, int component, void* dst, size_t bytes);
void* dp_iterator_stream(const dp_iterator* it);
int64_t dp_iterator_kernel_launches(const dp_iterator* it);
/* Batches covered by the fused batch-stage launches issued so far. */
int64_t dp_iterator_batches_launched(const dp_iterator* it);
/* Device time of the fused batch-stage launches so far (CUDA events around
 * each launch on the launching stream; waits for issued launches). */
int dp_iterator_batch_stage_timing(const dp_iterator* it, int64_t* total_ns, int64_t* launches);
int64_t dp_iterator_prefetch_depth(const dp_iterator* it);
/* Resource counters of the device pipeline (no reference counterpart: the
 * reference's buffers are per-element heap objects). */
typedef struct {
  int64_t live_plans;     /* epoch plans held (current, next, one back) */
  int64_t slots;          /* device batch slots allocated (prefetch ring) */
  int64_t slot_bytes;     /* their device bytes */
  int64_t prefetch_depth; /* groups kept in flight */
  int64_t group_batches;  /* batches per fused launch */
  /* AUTOTUNE (the reference's M/M/1/k model, model.cpp:29-42, 262-266) */
  int64_t max_depth;              /* slots pre-allocated for the tuner */
  double producer_groups_per_s;   /* device rate (CUDA-event self time, EWMA) */
  double consumer_groups_per_s;   /* host request rate (EWMA) */
  double p_empty;                 /* PEmpty(depth - 1, producer, consumer) */
} dp_iterator_stats;
/* Metrics() (runtime.hpp:46-51, 76): one row per graph node, root first. */
typedef struct {
  char path[192];
  char label[96];
  int64_t self_time_ns;
  int64_t elements_produced;
} dp_node_metrics;
/* Fills up to cap rows; *count = the node count (rows beyond cap dropped). */
int dp_iterator_metrics(const dp_iterator* it, dp_node_metrics* rows, int cap, int* count);
int dp_iterator_get_stats(const dp_iterator* it, dp_iterator_stats* out);
int64_t dp_iterator_root_delivered(const dp_iterator* it);
uint64_t dp_iterator_base_seed(const dp_iterator* it);
int dp_iterator_describe(const dp_iterator* it, char* buf, size_t len);
void dp_iterator_destroy(dp_iterator* it);

#ifdef __cplusplus
}
#endif

#endif /* DPCUDA_PIPELINE_H_ */
