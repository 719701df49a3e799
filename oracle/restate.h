/*
 * oracle/restate.h -- CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2101_12127_b200/,
 * include/) links, loads or calls this code.  Only tests/, the smoke() check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg use
 * it, and only as the checker or the reported CPU baseline.
 *
 * Two parity levels:
 *  1. ordering / batching / filtering / sharding (integer, bit exact): a plain
 *     C restatement of the reference runtime, pinned against the compiled
 *     reference (oracle/_ref, oracle/ref_shim.cpp) and against the known
 *     answers in SURVEY.md Appendix A (tests/golden/).
 *  2. map-UDF arithmetic (crop / flip / resize / normalize): PARITY UNPINNED
 *     by the reference, which has no image UDFs, so this
 *     file DEFINES them (as does orc_bucket_by_length for that new kind).  The same C
 *     functions are registered into the reference's UdfRegistry by
 *     oracle/ref_shim.cpp, so the compiled reference pipeline and this
 *     restatement agree by construction on the arithmetic; the order in which
 *     elements reach the UDF is what the reference pins.
 *
 * Compiled with -O2 -ffp-contract=off and no -march (matches the reference's
 * Release flags, /root/reference/proj/CMakeLists.txt:7-9): every fp32 op is
 * individually rounded, no FMA contraction.
 */
#ifndef DP_ORACLE_RESTATE_H_
#define DP_ORACLE_RESTATE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- PRNG contract: /root/reference/proj/include/datapipe/random.hpp ---- */
uint64_t orc_splitmix64_next(uint64_t* state);           /* random.hpp:24-29 */
uint64_t orc_mix_seeds(uint64_t a, uint64_t b);          /* random.hpp:31-34 */
typedef struct { uint64_t state; } orc_pcg32;
void orc_pcg32_init(orc_pcg32* g, uint64_t seed);        /* random.hpp:41-46 */
uint32_t orc_pcg32_next(orc_pcg32* g);                   /* random.hpp:48-54 */
uint32_t orc_pcg32_bounded(orc_pcg32* g, uint32_t bound);/* random.hpp:57-63 */

/* ShuffleIterator::DeriveSeed, runtime.cpp:713-718: attr seed absent -> the
 * constant 0x9d2c5680. */
uint64_t orc_shuffle_seed(uint64_t epoch_salt, int has_attr_seed,
                          uint64_t attr_seed);

/* ShuffleIterator::Next, runtime.cpp:721-747 (and ReferenceEval
 * reference.cpp:47-73): windowed reservoir over the input ordinals 0..n-1.
 * out[k] = input ordinal emitted at step k.  n, buffer >= 1. */
void orc_shuffle_order(uint64_t n, uint64_t buffer_size, uint64_t engine_seed,
                       uint32_t* out);

/* ---- digest ---- */
uint64_t orc_digest_init(void);
uint64_t orc_digest_i64(uint64_t h, const int64_t* v, size_t n);
uint64_t orc_digest_u32(uint64_t h, const uint32_t* v, size_t n);

/* ---- synthetic inputs ---- */
/* pixel byte `off` of image `id` (image of `image_bytes` bytes): top byte of
 * SplitMix64Next(seed ^ (id * image_bytes + off)). */
uint8_t orc_synth_pixel(uint64_t seed, uint64_t id, uint64_t image_bytes,
                        uint64_t off);
void orc_synth_images(uint64_t seed, uint64_t first_id, uint64_t count,
                      uint64_t image_bytes, uint8_t* out);
/* token sequences: len_i = Pcg32(len_seed).Bounded(max_len) + 1 drawn in
 * order; token (i, j) = SplitMix64Next(tok_seed ^ (i << 20 | j)) & 0x7fffffff. */
void orc_synth_lengths(uint64_t len_seed, uint32_t max_len, uint64_t n,
                       int32_t* lengths);
int32_t orc_synth_token(uint64_t tok_seed, uint64_t i, uint64_t j);

/* ---- Philox4x32-10 (Salmon et al. 2011); the crop/flip randomness
 * contract of this build: key = udf seed, counter =
 * element id. ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                       uint32_t out[4]);
void orc_crop_params(uint64_t seed, int64_t id, int in_h, int in_w, int crop_h,
                     int crop_w, int* oy, int* ox, int* flip);

/* ---- map UDF arithmetic ---- */
extern const float ORC_MEAN[3];
extern const float ORC_STD[3];
/* random crop (crop_h x crop_w at Philox offsets) + optional horizontal flip
 * + per-channel normalize (x - M_c) / S_c, HWC fp32 out.  `do_flip` = 0
 * disables the flip draw (crop only). */
void orc_crop_flip_normalize(const uint8_t* img, int in_h, int in_w,
                             int64_t id, uint64_t seed, int crop_h, int crop_w,
                             int do_flip, float* out);
/* bilinear resize alone (fp32 out), the same rounded ops. */
void orc_resize(const uint8_t* img, int in_h, int in_w, int out_h, int out_w, float* out);
/* bilinear resize (half-pixel centres, edge clamp) + normalize. */
void orc_resize_normalize(const uint8_t* img, int in_h, int in_w, int out_h,
                          int out_w, float* out);
float orc_normalize(float v, int c);

/* ---- filter + padded batch (cfg4) ---- */
/* Stable compaction of the positions with lengths[i] <= max_keep.  Returns
 * the kept count; kept[] gets the source positions in order. */
uint64_t orc_filter_len_le(const int32_t* lengths, uint64_t n,
                           int32_t max_keep, uint32_t* kept);

/* bucket_by_length (cfg4 "/ bucket-by-length"): tf.data's
 * bucket_by_sequence_length = group_by_window(key = #boundaries <= len,
 * window = batch_sizes[key], reduce = padded batch).  The reference has no
 * such kind (graph.hpp:38-56), so this sequential loop DEFINES the contract
 * (parity unpinned by the reference; TF's GroupByWindowDataset flushes the
 * remaining groups from a std::map, i.e. ascending key).  Walks order[0..n)
 * (positions into `lengths`); writes the emitted batches' positions back to
 * back into out_positions and each batch's row count into out_batch_rows;
 * returns the number of batches. */
int64_t orc_bucket_by_length(const int32_t* lengths, const int64_t* order,
                             int64_t n, const int32_t* boundaries,
                             int num_boundaries, const int64_t* batch_sizes,
                             int drop_remainder, int64_t* out_positions,
                             int64_t* out_batch_rows);

/* ---- shard / interleave index mapping (cfg3/cfg5) ---- */
/* ShardIterator, runtime.cpp:785-792: positions p with p % k == g. */
uint64_t orc_shard_positions(uint64_t n, uint64_t k, uint64_t g,
                             uint64_t* out);
/* InterleaveIterator (cycle c) over M inputs, each opening a reader of L
 * records (input m, record r) -> m * L + r.  runtime.cpp:1061-1120. */
uint64_t orc_interleave_order(uint64_t m_inputs, const uint64_t* inputs,
                              uint64_t cycle, uint64_t records,
                              uint64_t* out);
/* The same loop for readers of different lengths: input ordinal m opens
 * lengths[m] records valued starts[m] + r (record files of unequal sizes). */
uint64_t orc_interleave_var(uint64_t m_inputs, const uint64_t* inputs,
                            uint64_t cycle, const uint64_t* lengths,
                            const uint64_t* starts, uint64_t* out);

/* ---- image map UDF chain (oracle/chain.c): each step a MapFn on the whole
 * element, applied in order; u8 stays u8 through crops, resize / normalize /
 * affine / cast make fp32. ---- */
enum {
  ORC_STEP_RANDOM_CROP = 1, /* h, w, seed, flip: Philox offsets (orc_crop_params) */
  ORC_STEP_CENTER_CROP = 2, /* h, w: offsets ((H - h) / 2, (W - w) / 2), no flip */
  ORC_STEP_RESIZE = 3,      /* h, w: bilinear, half-pixel centres (orc_resize) */
  ORC_STEP_NORMALIZE = 4,   /* a = mean[3], b = std[3]: (x - a_c) / b_c */
  ORC_STEP_AFFINE = 5,      /* a = scale[3], b = shift[3]: x * a_c + b_c */
  ORC_STEP_CAST = 6         /* u8 -> fp32, exact */
};
typedef struct {
  int op, h, w, flip;
  uint64_t seed;
  float a[3], b[3];
} orc_map_step;
/* one step on an element image (u8 or fp32 HWC); out sized for its output */
int orc_apply_step(const void* in, int in_h, int in_w, int in_f32, int64_t id, const orc_map_step* step,
                   void* out);
/* output dims / dtype of a chain over an in_h x in_w x 3 u8 image; -1 if invalid */
int orc_chain_output(const orc_map_step* steps, int nsteps, int in_h, int in_w, int* out_h, int* out_w,
                     int* out_f32);
/* element (id, img) through the chain; out holds the result (u8 or fp32) */
int orc_apply_chain(const uint8_t* img, int in_h, int in_w, int64_t id, const orc_map_step* steps, int nsteps,
                    void* out);
/* Whole-epoch output digest: images ids[0..n) (synthetic pixels, seed
 * pix_seed) through the chain, output k's little-endian u32 words w hashed
 * at position k * words + w with K7's position hash and summed mod 2^64
 * (the device's dp_k_word_digest over the epoch's batches). */
uint64_t orc_epoch_image_digest(const orc_map_step* steps, int nsteps, uint64_t pix_seed, const int64_t* ids,
                                int64_t n, int in_h, int in_w, int threads, int* err);

#ifdef __cplusplus
}
#endif

#endif /* DP_ORACLE_RESTATE_H_ */
