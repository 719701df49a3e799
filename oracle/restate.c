/*
 * oracle/restate.c -- CPU restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see restate.h).  Each function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/.
 */
#include "restate.h"

#include <stdlib.h>
#include <string.h>

/* include/datapipe/random.hpp:24-29 */
uint64_t orc_splitmix64_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* include/datapipe/random.hpp:31-34 */
uint64_t orc_mix_seeds(uint64_t a, uint64_t b) {
  uint64_t s = a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2));
  return orc_splitmix64_next(&s);
}

#define ORC_PCG_MULT 6364136223846793005ULL
#define ORC_PCG_INC 1442695040888963407ULL /* random.hpp:72 kStream */

/* include/datapipe/random.hpp:48-54 */
uint32_t orc_pcg32_next(orc_pcg32* g) {
  uint64_t old = g->state;
  g->state = old * ORC_PCG_MULT + ORC_PCG_INC;
  uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = (uint32_t)(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((-rot) & 31u));
}

/* include/datapipe/random.hpp:41-46 */
void orc_pcg32_init(orc_pcg32* g, uint64_t seed) {
  g->state = 0;
  orc_pcg32_next(g);
  g->state += seed;
  orc_pcg32_next(g);
}

/* include/datapipe/random.hpp:57-63 */
uint32_t orc_pcg32_bounded(orc_pcg32* g, uint32_t bound) {
  uint32_t threshold = (-bound) % bound;
  for (;;) {
    uint32_t r = orc_pcg32_next(g);
    if (r >= threshold) return r % bound;
  }
}

/* src/runtime.cpp:713-718 */
uint64_t orc_shuffle_seed(uint64_t epoch_salt, int has_attr_seed,
                          uint64_t attr_seed) {
  return orc_mix_seeds(epoch_salt, has_attr_seed ? attr_seed : 0x9d2c5680u);
}

/* src/runtime.cpp:721-747: prime the buffer with the first `buffer_size`
 * inputs, then each step draws idx = Bounded(size), emits buffer[idx] and
 * refills it from the input, or on drain moves back() into idx and pops. */
void orc_shuffle_order(uint64_t n, uint64_t buffer_size, uint64_t engine_seed,
                       uint32_t* out) {
  orc_pcg32 g;
  orc_pcg32_init(&g, engine_seed);
  uint64_t cap = buffer_size < n ? buffer_size : n;
  uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (cap ? cap : 1));
  uint64_t size = 0, next_in = 0;
  while (size < buffer_size && next_in < n) buf[size++] = (uint32_t)next_in++;
  uint64_t k = 0;
  while (size > 0) {
    uint32_t idx = orc_pcg32_bounded(&g, (uint32_t)size);
    out[k++] = buf[idx];
    if (next_in < n) {
      buf[idx] = (uint32_t)next_in++;
    } else {
      buf[idx] = buf[size - 1];
      size--;
    }
  }
  free(buf);
}

uint64_t orc_digest_init(void) { return 0xcbf29ce484222325ULL; }

uint64_t orc_digest_i64(uint64_t h, const int64_t* v, size_t n) {
  for (size_t i = 0; i < n; ++i) h = (h ^ (uint64_t)v[i]) * 0x100000001b3ULL;
  return h;
}

uint64_t orc_digest_u32(uint64_t h, const uint32_t* v, size_t n) {
  for (size_t i = 0; i < n; ++i) h = (h ^ (uint64_t)v[i]) * 0x100000001b3ULL;
  return h;
}

uint8_t orc_synth_pixel(uint64_t seed, uint64_t id, uint64_t image_bytes,
                        uint64_t off) {
  uint64_t s = seed ^ (id * image_bytes + off);
  return (uint8_t)(orc_splitmix64_next(&s) >> 56);
}

void orc_synth_images(uint64_t seed, uint64_t first_id, uint64_t count,
                      uint64_t image_bytes, uint8_t* out) {
  for (uint64_t i = 0; i < count; ++i)
    for (uint64_t off = 0; off < image_bytes; ++off)
      out[i * image_bytes + off] =
          orc_synth_pixel(seed, first_id + i, image_bytes, off);
}

void orc_synth_lengths(uint64_t len_seed, uint32_t max_len, uint64_t n,
                       int32_t* lengths) {
  orc_pcg32 g;
  orc_pcg32_init(&g, len_seed);
  for (uint64_t i = 0; i < n; ++i)
    lengths[i] = (int32_t)orc_pcg32_bounded(&g, max_len) + 1;
}

int32_t orc_synth_token(uint64_t tok_seed, uint64_t i, uint64_t j) {
  uint64_t s = tok_seed ^ ((i << 20) | j);
  return (int32_t)(orc_splitmix64_next(&s) & 0x7fffffffULL);
}

/* Philox4x32-10, Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers:
 * as easy as 1, 2, 3" (Random123 reference constants). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                       uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void orc_crop_params(uint64_t seed, int64_t id, int in_h, int in_w, int crop_h,
                     int crop_w, int* oy, int* ox, int* flip) {
  uint32_t ctr[4] = {(uint32_t)(uint64_t)id, (uint32_t)((uint64_t)id >> 32), 0,
                     0};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t r[4];
  orc_philox4x32_10(ctr, key, r);
  *oy = (int)(r[0] % (uint32_t)(in_h - crop_h + 1));
  *ox = (int)(r[1] % (uint32_t)(in_w - crop_w + 1));
  *flip = (int)(r[2] & 1u);
}

/* ImageNet mean / std scaled to [0, 255]. */
const float ORC_MEAN[3] = {123.675f, 116.28f, 103.53f};
const float ORC_STD[3] = {58.395f, 57.12f, 57.375f};

/* One subtract, one IEEE divide; with -ffp-contract=off both round once. */
float orc_normalize(float v, int c) {
  float d = v - ORC_MEAN[c];
  return d / ORC_STD[c];
}

void orc_crop_flip_normalize(const uint8_t* img, int in_h, int in_w,
                             int64_t id, uint64_t seed, int crop_h, int crop_w,
                             int do_flip, float* out) {
  int oy, ox, flip;
  orc_crop_params(seed, id, in_h, in_w, crop_h, crop_w, &oy, &ox, &flip);
  if (!do_flip) flip = 0;
  for (int y = 0; y < crop_h; ++y) {
    const uint8_t* row = img + (size_t)(oy + y) * in_w * 3;
    for (int x = 0; x < crop_w; ++x) {
      int sx = ox + (flip ? crop_w - 1 - x : x);
      for (int c = 0; c < 3; ++c)
        out[((size_t)y * crop_w + x) * 3 + c] =
            orc_normalize((float)row[sx * 3 + c], c);
    }
  }
}

/* Half-pixel-centre bilinear source coordinate, clamped at 0 and at the last
 * row/column: s = (d + 0.5) * (in / out) - 0.5, every op rounded in fp32. */
static void resize_coord(int d, int in, int out, int* i0, int* i1, float* w) {
  float scale = (float)in / (float)out;
  float t = (float)d + 0.5f;
  float u = t * scale;
  float s = u - 0.5f;
  if (s < 0.0f) s = 0.0f;
  int a = (int)s;
  if (a > in - 1) a = in - 1;
  *i0 = a;
  *i1 = a + 1 < in ? a + 1 : in - 1;
  *w = s - (float)a;
}

void orc_resize(const uint8_t* img, int in_h, int in_w, int out_h, int out_w, float* out) {
  for (int y = 0; y < out_h; ++y) {
    int y0, y1;
    float wy;
    resize_coord(y, in_h, out_h, &y0, &y1, &wy);
    for (int x = 0; x < out_w; ++x) {
      int x0, x1;
      float wx;
      resize_coord(x, in_w, out_w, &x0, &x1, &wx);
      for (int c = 0; c < 3; ++c) {
        float p00 = (float)img[((size_t)y0 * in_w + x0) * 3 + c];
        float p01 = (float)img[((size_t)y0 * in_w + x1) * 3 + c];
        float p10 = (float)img[((size_t)y1 * in_w + x0) * 3 + c];
        float p11 = (float)img[((size_t)y1 * in_w + x1) * 3 + c];
        float top = p00 + wx * (p01 - p00);
        float bot = p10 + wx * (p11 - p10);
        out[((size_t)y * out_w + x) * 3 + c] = top + wy * (bot - top);
      }
    }
  }
}

void orc_resize_normalize(const uint8_t* img, int in_h, int in_w, int out_h,
                          int out_w, float* out) {
  for (int y = 0; y < out_h; ++y) {
    int y0, y1;
    float wy;
    resize_coord(y, in_h, out_h, &y0, &y1, &wy);
    for (int x = 0; x < out_w; ++x) {
      int x0, x1;
      float wx;
      resize_coord(x, in_w, out_w, &x0, &x1, &wx);
      for (int c = 0; c < 3; ++c) {
        float p00 = (float)img[((size_t)y0 * in_w + x0) * 3 + c];
        float p01 = (float)img[((size_t)y0 * in_w + x1) * 3 + c];
        float p10 = (float)img[((size_t)y1 * in_w + x0) * 3 + c];
        float p11 = (float)img[((size_t)y1 * in_w + x1) * 3 + c];
        float d0 = p01 - p00;
        float m0 = wx * d0;
        float top = p00 + m0;
        float d1 = p11 - p10;
        float m1 = wx * d1;
        float bot = p10 + m1;
        float dv = bot - top;
        float mv = wy * dv;
        float v = top + mv;
        out[((size_t)y * out_w + x) * 3 + c] = orc_normalize(v, c);
      }
    }
  }
}

/* FilterIterator, src/runtime.cpp:556-571, with the len <= max predicate. */
uint64_t orc_filter_len_le(const int32_t* lengths, uint64_t n,
                           int32_t max_keep, uint32_t* kept) {
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (lengths[i] <= max_keep) kept[m++] = (uint32_t)i;
  return m;
}

/* ShardIterator::Next, src/runtime.cpp:785-792. */
uint64_t orc_shard_positions(uint64_t n, uint64_t k, uint64_t g,
                             uint64_t* out) {
  uint64_t m = 0;
  for (uint64_t p = 0; p < n; ++p)
    if (p % k == g) out[m++] = p;
  return m;
}

/* InterleaveIterator::Next / OpenNext, src/runtime.cpp:1061-1120, simulated
 * step by step for sub-datasets of `records` elements each. */
uint64_t orc_interleave_order(uint64_t m_inputs, const uint64_t* inputs,
                              uint64_t cycle, uint64_t records,
                              uint64_t* out) {
  typedef struct { int open, dead; uint64_t input, pos; } slot_t;
  slot_t* slots = (slot_t*)calloc(cycle, sizeof(slot_t));
  uint64_t cursor = 0, next_input = 0, k = 0;
  int inputs_done = 0;
  for (;;) {
    uint64_t dead_streak = 0;
    int produced = 0;
    while (dead_streak < cycle) {
      slot_t* s = &slots[cursor];
      if (!s->open && !s->dead) {
        if (inputs_done || next_input >= m_inputs) {
          inputs_done = 1;
          s->dead = 1;
        } else {
          s->open = 1;
          s->input = inputs[next_input++];
          s->pos = 0;
        }
      }
      if (s->dead) {
        cursor = (cursor + 1) % cycle;
        dead_streak++;
        continue;
      }
      if (s->pos < records) {
        out[k++] = s->input * records + s->pos++;
        cursor = (cursor + 1) % cycle;
        produced = 1;
        break;
      }
      s->open = 0; /* exhausted: same cycle position opens the next input */
    }
    if (!produced) break;
  }
  free(slots);
  return k;
}

/* InterleaveIterator::Next / OpenNext (src/runtime.cpp:1061-1120) with
 * per-input lengths: an exhausted slot opens the next input in the same
 * visit (no turn is lost; empty inputs are skipped in place); a slot finding
 * no input left is dead. */
uint64_t orc_interleave_var(uint64_t m_inputs, const uint64_t* inputs,
                            uint64_t cycle, const uint64_t* lengths,
                            const uint64_t* starts, uint64_t* out) {
  typedef struct { int open, dead; uint64_t input, pos; } slot_t;
  slot_t* slots = (slot_t*)calloc(cycle, sizeof(slot_t));
  uint64_t cursor = 0, next_input = 0, k = 0;
  for (;;) {
    uint64_t dead_streak = 0;
    int produced = 0;
    while (dead_streak < cycle) {
      slot_t* s = &slots[cursor];
      if (!s->open && !s->dead) {
        if (next_input >= m_inputs) {
          s->dead = 1;
        } else {
          s->open = 1;
          s->input = inputs[next_input++];
          s->pos = 0;
        }
      }
      if (s->dead) {
        cursor = (cursor + 1) % cycle;
        dead_streak++;
        continue;
      }
      if (s->pos < lengths[s->input]) {
        out[k++] = starts[s->input] + s->pos++;
        cursor = (cursor + 1) % cycle;
        produced = 1;
        break;
      }
      s->open = 0; /* exhausted: same cycle position opens the next input */
    }
    if (!produced) break;
  }
  free(slots);
  return k;
}

/* group_by_window, sequentially (see restate.h). */
int64_t orc_bucket_by_length(const int32_t* lengths, const int64_t* order,
                             int64_t n, const int32_t* boundaries,
                             int num_boundaries, const int64_t* batch_sizes,
                             int drop_remainder, int64_t* out_positions,
                             int64_t* out_batch_rows) {
  const int nb = num_boundaries + 1;
  int64_t* window[33];
  int64_t fill[33];
  int64_t batches = 0, w = 0;
  for (int b = 0; b < nb; ++b) {
    window[b] = (int64_t*)malloc(sizeof(int64_t) * (size_t)batch_sizes[b]);
    fill[b] = 0;
  }
  for (int64_t i = 0; i < n; ++i) {
    const int64_t p = order ? order[i] : i;
    int b = 0;
    for (int k = 0; k < num_boundaries; ++k) b += lengths[p] >= boundaries[k];
    window[b][fill[b]++] = p;
    if (fill[b] == batch_sizes[b]) { /* the window is full: emit it */
      for (int64_t r = 0; r < fill[b]; ++r) out_positions[w++] = window[b][r];
      out_batch_rows[batches++] = fill[b];
      fill[b] = 0;
    }
  }
  for (int b = 0; b < nb; ++b) { /* end of input: ascending key */
    if (fill[b] && !drop_remainder) {
      for (int64_t r = 0; r < fill[b]; ++r) out_positions[w++] = window[b][r];
      out_batch_rows[batches++] = fill[b];
    }
    free(window[b]);
  }
  return batches;
}
