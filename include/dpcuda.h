/*
 * dpcuda.h -- the C ABI of the B200 datapipe engine (libdpcuda.so).
 *
 * This is the drop-in boundary for the reference's fused
 * shuffle -> map -> batch -> prefetch path.  The reference
 * ("datapipe", /root/reference/proj) exposes that path only as a C++ operator
 * API; it has no C ABI or FFI of its own.  The entry points below are what an
 * FFI binding of that API would bind, in two layers:
 *
 *   1. dp_graph_* / dp_iterator_*  -- the Dataset/Iterator operator API
 *      (ops::*, Optimize, MakeIterator, GetNext), backed by the C++ host
 *      engine in paper_2101_12127_b200/csrc/engine/ which lowers the graph
 *      onto the sm_100a kernels.  Declared in dpcuda_pipeline.h.
 *   2. dp_k_* (this file)          -- one entry per sm_100a kernel family,
 *      taking device pointers, sizes and an explicit cudaStream_t (passed as
 *      void*); asynchronous on that stream.  Used by the engine and by the
 *      parity tests.
 *
 * Conventions:
 *   - every function returns 0 (DP_OK) or a dp_status; no exception crosses
 *     the boundary.  dp_last_error() returns a thread-local message.
 *   - dp_status values 1..19 mirror datapipe::ErrorCode
 *     (/root/reference/proj/include/datapipe/errors.hpp:25-45) + 1.
 *   - no hidden allocation on launch paths; callers own device buffers.
 */
#ifndef DPCUDA_H_
#define DPCUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DP_OK = 0,
  /* datapipe::ErrorCode + 1 (errors.hpp:25-45) */
  DP_ERR_INVALID_ARITY = 1,
  DP_ERR_INVALID_ATTR = 2,
  DP_ERR_TYPE_MISMATCH = 3,
  DP_ERR_MALFORMED_INPUT = 4,
  DP_ERR_VALIDATION_FAILED = 5,
  DP_ERR_DUPLICATE_NAME = 6,
  DP_ERR_UNKNOWN_UDF = 7,
  DP_ERR_MISSING_FILE = 8,
  DP_ERR_UDF_ERROR = 9,
  DP_ERR_FINGERPRINT_MISMATCH = 10,
  DP_ERR_VERSION_MISMATCH = 11,
  DP_ERR_CORRUPT_BLOB = 12,
  DP_ERR_CONCURRENT_CACHE_FILL = 13,
  DP_ERR_REWRITE_DIVERGED = 14,
  DP_ERR_RULE_PRODUCED_INVALID_GRAPH = 15,
  DP_ERR_DOMAIN_ERROR = 16,
  DP_ERR_GRID_TOO_LARGE = 17,
  DP_ERR_PARSE_ERROR = 18,
  DP_ERR_INTERNAL = 19,
  /* device-side failures (no reference counterpart) */
  DP_ERR_CUDA = 100,
  DP_ERR_OUT_OF_MEMORY = 101,
  DP_ERR_END_OF_SEQUENCE = 102
} dp_status;

/* Thread-local message of the last failing call on this thread. */
const char* dp_last_error(void);
/* Library version / build string ("libdpcuda sm_100a ..."). */
const char* dp_build_info(void);
/* Number of visible CUDA devices (0 when there is no GPU). */
int dp_device_count(int* count);

/* ---------------------------------------------------------------------- */
/* K1  range_affine_batch -- FromMemory(IntRange) + Map(x*a+b) + Batch     */
/*     replaces FromMemoryIterator::Next + MapIterator + BatchIterator /   */
/*     MapAndBatchIterator (src/runtime.cpp:386-414, 480-535, 579-637,     */
/*     1467-1721) for an int64 range source.                               */
/*     out[i] = (first + i) * a + b,  i < rows  (int64, wrap-around).      */
int dp_k_range_affine_batch(int64_t first, int64_t rows, int64_t a, int64_t b,
                            int64_t* out, void* stream);

/* K1 general form (gathered int64 source): out[i] = v * a + b with       */
/* v = values ? values[p] : p and p = order ? order[first + i] : first + i. */
int dp_k_gather_affine_batch(const int64_t* values, const int64_t* order, int64_t first, int64_t rows,
                             int64_t a, int64_t b, int64_t* out, void* stream);

/* ---------------------------------------------------------------------- */
/* K2  shuffle_plan -- ShuffleIterator (src/runtime.cpp:688-768) with the  */
/*     PCG32 contract (include/datapipe/random.hpp:39-74).                 */
/*     Emission order of a windowed reservoir of `buffer_size` over the    */
/*     input ordinals 0..n-1 seeded with `engine_seed` (= MixSeeds(salt,   */
/*     seed|0x9d2c5680), runtime.cpp:713-718).  out[k] = in_map[ord_k] if  */
/*     in_map != NULL else ord_k.  `scratch` must hold min(n,buffer_size)  */
/*     uint32 when that exceeds the kernel's shared-memory buffer (pass    */
/*     NULL otherwise; see dp_k_shuffle_plan_scratch_bytes).               */
size_t dp_k_shuffle_plan_scratch_bytes(uint64_t n, uint64_t buffer_size);
int dp_k_shuffle_plan(uint64_t n, uint64_t buffer_size, uint64_t engine_seed,
                      const int64_t* in_map, int64_t* out, void* scratch,
                      void* stream);

/* ---------------------------------------------------------------------- */
/* K3  gather + random crop + flip + normalize + batch (one launch per     */
/*     batch) -- MapAndBatchIterator::WorkerLoop + the crop UDF +          */
/*     AssembleBatch (src/runtime.cpp:1574-1670, 617-628).                 */
/*     images: uint8 [num_images, in_h, in_w, 3] (HWC), device resident.   */
/*     order:  int64 gather positions (NULL = identity); element j of the  */
/*     batch is images[order[first + j]], its id = that position.          */
/*     out_ids: int64 [rows]; out: fp32 [rows, crop_h, crop_w, 3].         */
/*     Crop offsets / flip: Philox4x32-10(key = udf_seed, ctr = id).       */
/*     normalize: (x - mean[c]) / std[c] rounded as IEEE fp32 division.    */
int dp_k_crop_flip_normalize_batch(const uint8_t* images, int64_t num_images,
                                   int in_h, int in_w, const int64_t* order,
                                   int64_t first, int64_t rows,
                                   uint64_t udf_seed, int crop_h, int crop_w,
                                   int do_flip, const float mean[3],
                                   const float stdv[3], int64_t* out_ids,
                                   float* out, void* stream);

/* K4  gather + bilinear resize (half-pixel centres, edge clamp) +         */
/*     normalize + batch.  Same layout conventions as K3.                  */
int dp_k_resize_normalize_batch(const uint8_t* images, int64_t num_images,
                                int in_h, int in_w, const int64_t* order,
                                int64_t first, int64_t rows, int out_h,
                                int out_w, const float mean[3],
                                const float stdv[3], int64_t* out_ids,
                                float* out, void* stream);

/* Sharded residency (one process per GPU holds shard `id_base` of
 * `id_stride`, in blocks of `id_block` consecutive ids): `images` row r is
 * element ((r / id_block) * id_stride + id_base) * id_block + r % id_block
 * (id_block 1: id_base + r * id_stride); the gather order indexes rows, ids
 * (Philox counter, out_ids) are global. */
int dp_k_crop_flip_normalize_batch_ex(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                      const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                      int64_t id_stride, int64_t id_block, uint64_t udf_seed, int crop_h,
                                      int crop_w, int do_flip, const float mean[3], const float stdv[3],
                                      int64_t* out_ids, float* out, void* stream);
/* K3 with center_crop offsets ((in_h - crop_h) / 2, (in_w - crop_w) / 2), no
 * flip: center_crop >> normalize (an eval-time chain). */
int dp_k_center_crop_normalize_batch_ex(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                        const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                        int64_t id_stride, int64_t id_block, int crop_h, int crop_w,
                                        const float mean[3], const float stdv[3], int64_t* out_ids, float* out,
                                        void* stream);
int dp_k_resize_normalize_batch_ex(const uint8_t* images, int64_t num_images, int in_h, int in_w,
                                   const int64_t* order, int64_t first, int64_t rows, int64_t id_base,
                                   int64_t id_stride, int64_t id_block, int out_h, int out_w,
                                   const float mean[3], const float stdv[3], int64_t* out_ids, float* out,
                                   void* stream);

/* ---------------------------------------------------------------------- */
/* K5  filter(len <= max_keep) stream compaction + padded_batch.           */
/*     FilterIterator (src/runtime.cpp:537-577) + BatchIterator on ragged  */
/*     (element i of the filtered sequence has length lengths[in_map[i]])  */
/*     lists (579-637); padded_batch is a new kind.   */
/*     kept: int64 [n] out (stable order), *num_kept written to device     */
/*     memory `num_kept_dev` (int64).  scratch: dp_k_filter_scratch_bytes. */
size_t dp_k_filter_scratch_bytes(int64_t n);
/* General device predicate (FilterIterator runtime.cpp:556-571 with the     */
/* predicate UDF as a descriptor): keep element i iff every term holds on   */
/* v = mul * q + add (wrap-around int64), q = lengths[p] if lengths, else    */
/* values[p] if values, else the position p itself (range); p = in_map[i].  */
/* % is C's truncated remainder (the reference's keep_even/keep_odd,        */
/* pipeline_spec.cpp:234-243).  terms: host array, 1..8.                   */
#define DP_PRED_LE 0     /* v <= a      */
#define DP_PRED_GE 1     /* v >= a      */
#define DP_PRED_LT 2     /* v < a       */
#define DP_PRED_MOD_EQ 3 /* v % a == b  */
#define DP_PRED_MOD_NE 4 /* v % a != b  */
typedef struct dp_predicate_term {
  int op;
  int64_t a, b;
} dp_predicate_term;
int dp_k_filter(const int32_t* lengths, const int64_t* values, int64_t n,
                int64_t mul, int64_t add, const dp_predicate_term* terms,
                int num_terms, const int64_t* in_map, int64_t* kept,
                int64_t* num_kept_dev, void* scratch, void* stream);
int dp_k_filter_len_le(const int32_t* lengths, int64_t n, int32_t max_keep,
                       const int64_t* in_map, int64_t* kept,
                       int64_t* num_kept_dev, void* scratch, void* stream);
/* Per-batch max row length: lmax[j] = max over the rows of batch j of     */
/* lengths[kept[j*batch + r]]  (rows of the last batch may be fewer).      */
int dp_k_batch_max_len(const int32_t* lengths, const int64_t* kept,
                       int64_t num_kept, int64_t batch, int32_t* lmax,
                       void* stream);
/* One padded batch: out[r, 0:lmax] = tokens of row r then pad_value;      */
/* out_lengths[r] = its length.  rows <= batch.                            */
int dp_k_padded_batch(const int32_t* tokens, const int64_t* offsets,
                      const int32_t* lengths, const int64_t* kept,
                      int64_t first, int64_t rows, int32_t lmax,
                      int32_t pad_value, int32_t* out, int32_t* out_lengths,
                      void* stream);

/* Grouped form: rows [first_row, first_row + rows) of consecutive padded  */
/* batches of `batch` rows in one launch; lmax_dev[j] / boff_dev[j] are    */
/* the epoch's per-batch max length and element offset (exclusive prefix   */
/* of rows_j * lmax_j); `out` is the element offset boff_dev[first_row /   */
/* batch].  order = the epoch's kept positions.                            */
int dp_k_padded_batches(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                        const int64_t* order, int64_t first_row, int64_t rows, int64_t batch,
                        const int32_t* lmax_dev, const int64_t* boff_dev, int32_t pad_value,
                        int32_t* out, int32_t* out_lengths, void* stream);

/* Ragged Batch of token sequences (the reference's Filter -> Batch lists, */
/* runtime.cpp:579-637): prefix[i] = sum of lengths[order[j]], j < i, and  */
/* prefix[n] = the total (int64 [n + 1]; order null = identity).          */
/* Stages plan rows into device memory (token configs with a pinned host
 * source, end to end): staged[prefix[i] ..] = tokens[offsets[p_i] ..
 * + lengths[p_i]), staged_lengths[i] = lengths[p_i], p_i = order ? order[i]
 * : i; prefix from dp_k_len_prefix over the same order.  The batch kernels
 * then read the staged rows (order = identity, offsets = prefix) from HBM
 * instead of gathering 4-byte words over PCIe. */
int dp_k_stage_rows(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths, const int64_t* order,
                    int64_t n, const int64_t* prefix, int32_t* staged, int32_t* staged_lengths, void* stream);
size_t dp_k_len_prefix_scratch_bytes(int64_t n);
int dp_k_len_prefix(const int32_t* lengths, const int64_t* order, int64_t n,
                    int64_t* prefix, void* scratch, void* stream);
/* Rows [first_row, first_row + rows) of an epoch of n_rows kept rows in   */
/* batches of `batch`: tokens packed into values (offset prefix[R] -       */
/* prefix[first_row]); each batch's rows_j + 1 row splits (int64, relative */
/* to the batch) one after another in `splits`.                           */
int dp_k_ragged_batches(const int32_t* tokens, const int64_t* offsets, const int32_t* lengths,
                        const int64_t* order, int64_t first_row, int64_t rows, int64_t batch,
                        int64_t n_rows, const int64_t* prefix, int32_t* values, int64_t* splits,
                        void* stream);

/* ---------------------------------------------------------------------- */
/* K8  bucket_by_length -- tf.data bucket_by_sequence_length              */
/*     (group_by_window: key = bucket of the length, window = the bucket's */
/*     batch size, reduce = padded batch); a new kind like padded_batch,  */
/*     absent from the reference (graph.hpp:38-56).   */
/*     Bucket b holds boundaries[b-1] <= len < boundaries[b]; batches are */
/*     emitted when their window fills, then the partial windows in       */
/*     ascending bucket order (unless drop_remainder).                    */
#define DP_MAX_BUCKETS 32
size_t dp_k_bucket_scratch_bytes(int64_t n, int num_buckets);
/* Plan over the n elements of `order` (positions; null = identity):      */
/*   perm[n]: positions grouped by bucket, arrival order within a bucket; */
/*   per emitted batch e < *num_batches_dev (<= n + buckets):             */
/*   batch_start[e] (into perm), batch_rows[e], batch_lmax[e].            */
/*   boundaries / batch_sizes are HOST arrays (num_boundaries + 1 sizes). */
int dp_k_bucket_plan(const int32_t* lengths, const int64_t* order, int64_t n,
                     const int32_t* boundaries, int num_boundaries,
                     const int64_t* batch_sizes, int drop_remainder,
                     int64_t* perm, int64_t* batch_start, int32_t* batch_rows,
                     int32_t* batch_lmax, int64_t* num_batches_dev,
                     void* scratch, void* stream);
/* Pads batches [first, first + num) of a plan into `out` (element offset */
/* boff[e] - boff[first], row-major [rows_e, lmax_e]) and their lengths   */
/* into out_lengths (offset roff[e] - roff[first]); boff / roff are the   */
/* exclusive prefixes of rows_e * lmax_e and rows_e (device arrays);      */
/* num_rows = roff[first + num] - roff[first] (host value, grid size).    */
int dp_k_bucket_batches(const int32_t* tokens, const int64_t* offsets,
                        const int32_t* lengths, const int64_t* perm,
                        const int64_t* batch_start, const int32_t* batch_rows,
                        const int32_t* batch_lmax, const int64_t* boff,
                        const int64_t* roff, int64_t first, int64_t num,
                        int64_t num_rows, int32_t pad_value, int32_t* out,
                        int32_t* out_lengths, void* stream);

/* The same batches from per-row tables of a plan (dp_k_bucket_rows, once  */
/* per epoch): row R reads position row_src[R], writes row_lm[R] tokens at */
/* row_dst[R] - first_elem; rows [first_row, first_row + num_rows).  The    */
/* engine's path (a shallower per-row dependency chain than the search).   */
int dp_k_bucket_rows(const int64_t* perm, const int64_t* batch_start,
                     const int32_t* batch_lmax, const int64_t* boff,
                     const int64_t* roff, int64_t num_batches,
                     int64_t* row_src, int64_t* row_dst, int32_t* row_lm,
                     void* stream);
int dp_k_bucket_rows_batches(const int32_t* tokens, const int64_t* offsets,
                             const int32_t* lengths, const int64_t* row_src,
                             const int64_t* row_dst, const int32_t* row_lm,
                             int64_t first_row, int64_t first_elem,
                             int64_t num_rows, int32_t pad_value,
                             int32_t* out, int32_t* out_lengths, void* stream);

/* ---------------------------------------------------------------------- */
/* K6  shard + interleave index mapping -- ShardIterator (runtime.cpp:     */
/*     770-800) + (Parallel)InterleaveIterator (1044-1128, 1727-2021) over */
/*     equal-length readers.  Inputs are the source ordinals p < n_sources */
/*     with p % num_shards == shard_index; each opens a reader of          */
/*     `records` elements valued p * records + r; cycle = cycle_length.    */
/*     out: int64 [count] where count = dp_k_shard_interleave_count(...).  */
int64_t dp_k_shard_interleave_count(int64_t n_sources, int64_t num_shards,
                                    int64_t shard_index, int64_t records);
int dp_k_shard_interleave_index(int64_t n_sources, int64_t num_shards,
                                int64_t shard_index, int64_t cycle,
                                int64_t records, int64_t* out, void* stream);
/* General form over inputs first + i * stride, i < m_inputs. */
int dp_k_interleave_index(int64_t first, int64_t stride, int64_t m_inputs, int64_t cycle,
                          int64_t records, int64_t* out, void* stream);
/* Readers of unequal lengths (record files of different sizes): host      */
/* schedule of the InterleaveIterator loop (runtime.cpp:1061-1120) --      */
/* input i (in input order, lengths[i] records) runs in cycle slot slot[i] */
/* from visit round start[i]; end[s] = the round slot s goes dead (cycle   */
/* entries).  O(m log cycle) on the host: control, not data.              */
int dp_interleave_schedule(int64_t m_inputs, const int64_t* lengths, int64_t cycle,
                           int64_t* slot, int64_t* start, int64_t* end);
/* Device order from that schedule (all arrays device memory):            */
/* out[pos(i, j)] = first_record[i] + j for j < len[i].                   */
int dp_k_interleave_var(int64_t m_inputs, const int64_t* slot, const int64_t* start,
                        const int64_t* len, const int64_t* first_record,
                        const int64_t* end, int64_t cycle, int64_t* out, void* stream);
/* Shard alone: out[i] = shard_index + i * num_shards (or in_map of it). */
int dp_k_shard_index(int64_t n, int64_t num_shards, int64_t shard_index,
                     const int64_t* in_map, int64_t* out, void* stream);

/* ---------------------------------------------------------------------- */
/* ---------------------------------------------------------------------- */
/* K9  general image map chain + Batch (MapAndBatchIterator, src/runtime.  */
/*     cpp:1467-1721, over the device UDF library's chains that K3 / K4 do  */
/*     not cover): [crop A][pixel ops][resize][crop B][pixel ops], each    */
/*     value from its source taps with the sequential chain's rounded fp32 */
/*     ops (oracle/chain.c).  Crop modes: 0 none, 1 random (Philox key =   */
/*     seed, counter = element id; flip bit used when *_flip), 2 center.   */
/*     Pixel ops (op_kind): 0 normalize (x - a_c) / b_c, 1 affine          */
/*     x * a_c + b_c; the first num_pre_ops act on source taps (before the */
/*     resize), the next num_post_ops on the blend.  out_f32 = resize or   */
/*     any op (else u8 output: crops only).                                */
typedef struct {
  int in_h, in_w;
  int pre_mode, pre_h, pre_w, pre_flip;
  uint64_t pre_seed;
  int resize, rs_h, rs_w;
  int post_mode, post_h, post_w, post_flip;
  uint64_t post_seed;
  int num_pre_ops, num_post_ops;
  int op_kind[4];
  float op_a[4][3], op_b[4][3];
  int out_f32;
} dp_image_chain;
/* Output shape / dtype of a chain (validates it). */
int dp_image_chain_output(const dp_image_chain* chain, int* out_h, int* out_w, int* out_f32);
/* out[j] = chain(images[p_j]), p_j = order ? order[first + j] : first + j;
 * out_ids[j] = the element id of p_j (sharded residency as K3's _ex). */
int dp_k_image_chain_batch(const uint8_t* images, int64_t num_images, const int64_t* order, int64_t first,
                           int64_t rows, int64_t id_base, int64_t id_stride, int64_t id_block,
                           const dp_image_chain* chain, int64_t* out_ids, void* out, void* stream);
/* Which kernel runs a chain on HBM-resident, 16-byte aligned buffers: 10  */
/* (K10, below) or 9 (K9).                                                 */
int dp_image_chain_kernel(const dp_image_chain* chain, int* kernel);
/* K10 (k_roll.cu): the resize chains [crop A] -> resize -> [crop B] ->     */
/*     [one or two pixel ops] whose column map is periodic (10:7,           */
/*     8:7, 5:7, 5:4, 9:7, 12:7, 6:7, 4:7, 3:2, 2:1; any other ratio of a   */
/*     chain with runtime taps), run by                                     */
/*     dp_k_image_chain_batch / dp_k_resize_normalize_batch: horizontal blends */
/*     computed once per (source row, column) and rolled in registers.      */
/* Whether normalize(mean, std)'s two-FMA division equals IEEE division    */
/* for every fp32 in [+0, 255] (checked exhaustively on the device at first */
/* use, cached); the kernels use IEEE division where it does not.          */
int dp_fast_div_proven(const float mean[3], const float stdv[3], int* proven);
/* Batch with no map (BatchIterator over (id, u8 image), runtime.cpp:579-
 * 637): out[j] = images[p_j] byte for byte (image_bytes each). */
int dp_k_gather_copy_batch(const uint8_t* images, int64_t num_images, int64_t image_bytes, const int64_t* order,
                           int64_t first, int64_t rows, int64_t id_base, int64_t id_stride, int64_t id_block,
                           int64_t* out_ids, uint8_t* out, void* stream);

/* K7  order digest (the multi-GPU "final ordering check") */
/*     position-keyed, parallel: D = sum_i SplitMix64Next(v_i ^ (i *      */
/*     0x9e3779b97f4a7c15)) mod 2^64 (state passed by value).  Accumulates */
/*     into *digest_dev (uint64) for positions first..first+n-1.           */
int dp_k_order_digest(const int64_t* values, int64_t n, int64_t first,
                      uint64_t* digest_dev, void* stream);
/* Same over raw 32-bit words (fp32 batch payloads, bit-exact check). */
int dp_k_word_digest(const uint32_t* words, int64_t n, int64_t first,
                     uint64_t* digest_dev, void* stream);

/* rows x width bytes of a pitched (device) source, packed into dst --    */
/* typically mapped pinned host memory: an SM-side read-back that does not */
/* queue behind the copy engines (the plan's small read-backs while a      */
/* launch group's host_output copy is in flight).                          */
int dp_k_copy_strided(const void* src, size_t src_pitch, size_t width, size_t rows, void* dst, void* stream);

/* ---------------------------------------------------------------------- */
/* Synthetic inputs (same generators as oracle/restate.c). */
/* images[i, off] = top byte of SplitMix64Next(seed ^ ((first_id + i) *    */
/* image_bytes + off)).                                                    */
int dp_k_synth_images(uint8_t* images, uint64_t first_id, uint64_t count,
                      uint64_t image_bytes, uint64_t seed, void* stream);
/* Row i holds image id first_id + i * id_stride (a Shard's residency). */
int dp_k_synth_images_strided(uint8_t* images, uint64_t first_id, uint64_t id_stride, uint64_t count,
                              uint64_t image_bytes, uint64_t seed, void* stream);
/* tokens[offsets[i] + j] = SplitMix64Next(seed ^ (i << 20 | j)) & 0x7fffffff */
int dp_k_synth_tokens(int32_t* tokens, const int64_t* offsets, int64_t n,
                      uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DPCUDA_H_ */
