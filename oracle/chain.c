/*
 * oracle/chain.c -- CPU restatement of the device image-map UDF library as a
 * sequential chain of per-element map functions.  TEST INFRASTRUCTURE ONLY
 * (see restate.h).
 *
 * The reference's Map applies one opaque MapFn per element per map node
 * (/root/reference/proj/src/runtime.cpp:480-535, udf.hpp:31); a chain
 * map(f).map(g) is g(f(e)) (optimizer.cpp:165-188 composes the names as
 * "(f)>>(g)").  The reference has no image UDFs, so each
 * step below DEFINES one: it runs on a whole intermediate image (u8 or
 * fp32, HWC, 3 channels) exactly as a MapFn would, every fp32 op rounded
 * once (-ffp-contract=off).  The device kernels fuse the chain; they must
 * produce these bytes.
 */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "restate.h"

/* resize_coord of restate.c (half-pixel centres, clamped) */
static void chain_coord(int d, int in, int out, int* i0, int* i1, float* w) {
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

typedef struct {
  int h, w, f32; /* f32: values are float, else uint8 */
  uint8_t* u8;
  float* f;
} orc_img;

static float px(const orc_img* m, size_t i) { return m->f32 ? m->f[i] : (float)m->u8[i]; }

static void img_alloc(orc_img* m, int h, int w, int f32) {
  m->h = h;
  m->w = w;
  m->f32 = f32;
  size_t n = (size_t)h * w * 3;
  m->u8 = f32 ? NULL : (uint8_t*)malloc(n ? n : 1);
  m->f = f32 ? (float*)malloc(sizeof(float) * (n ? n : 1)) : NULL;
}
static void img_free(orc_img* m) {
  free(m->u8);
  free(m->f);
  m->u8 = NULL;
  m->f = NULL;
}

/* one step applied to `cur` (replaced) */
static int chain_step(orc_img* cur, const orc_map_step* s, int64_t id) {
  orc_img nx;
  switch (s->op) {
    case ORC_STEP_RANDOM_CROP:
    case ORC_STEP_CENTER_CROP: {
      if (s->h > cur->h || s->w > cur->w || s->h < 1 || s->w < 1) return -1;
      int oy, ox, fl = 0;
      if (s->op == ORC_STEP_RANDOM_CROP) {
        orc_crop_params(s->seed, id, cur->h, cur->w, s->h, s->w, &oy, &ox, &fl);
        if (!s->flip) fl = 0;
      } else {
        oy = (cur->h - s->h) / 2;
        ox = (cur->w - s->w) / 2;
      }
      img_alloc(&nx, s->h, s->w, cur->f32);
      for (int y = 0; y < s->h; ++y)
        for (int x = 0; x < s->w; ++x) {
          int sx = ox + (fl ? s->w - 1 - x : x);
          size_t si = ((size_t)(oy + y) * cur->w + sx) * 3, di = ((size_t)y * s->w + x) * 3;
          for (int c = 0; c < 3; ++c) {
            if (cur->f32) nx.f[di + c] = cur->f[si + c];
            else nx.u8[di + c] = cur->u8[si + c];
          }
        }
      break;
    }
    case ORC_STEP_RESIZE: {
      if (s->h < 1 || s->w < 1) return -1;
      img_alloc(&nx, s->h, s->w, 1);
      for (int y = 0; y < s->h; ++y) {
        int y0, y1;
        float wy;
        chain_coord(y, cur->h, s->h, &y0, &y1, &wy);
        for (int x = 0; x < s->w; ++x) {
          int x0, x1;
          float wx;
          chain_coord(x, cur->w, s->w, &x0, &x1, &wx);
          for (int c = 0; c < 3; ++c) {
            float p00 = px(cur, ((size_t)y0 * cur->w + x0) * 3 + c);
            float p01 = px(cur, ((size_t)y0 * cur->w + x1) * 3 + c);
            float p10 = px(cur, ((size_t)y1 * cur->w + x0) * 3 + c);
            float p11 = px(cur, ((size_t)y1 * cur->w + x1) * 3 + c);
            float d0 = p01 - p00;
            float m0 = wx * d0;
            float top = p00 + m0;
            float d1 = p11 - p10;
            float m1 = wx * d1;
            float bot = p10 + m1;
            float dv = bot - top;
            float mv = wy * dv;
            nx.f[((size_t)y * s->w + x) * 3 + c] = top + mv;
          }
        }
      }
      break;
    }
    case ORC_STEP_NORMALIZE:
    case ORC_STEP_AFFINE:
    case ORC_STEP_CAST: {
      img_alloc(&nx, cur->h, cur->w, 1);
      size_t n = (size_t)cur->h * cur->w;
      for (size_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) {
          float v = px(cur, i * 3 + c);
          if (s->op == ORC_STEP_NORMALIZE) {
            float d = v - s->a[c]; /* (x - mean) / std: one subtract, one IEEE divide */
            v = d / s->b[c];
          } else if (s->op == ORC_STEP_AFFINE) {
            float m = v * s->a[c]; /* x * scale + shift: two rounded ops */
            v = m + s->b[c];
          }
          nx.f[i * 3 + c] = v;
        }
      break;
    }
    default:
      return -1;
  }
  img_free(cur);
  *cur = nx;
  return 0;
}

int orc_apply_step(const void* in, int in_h, int in_w, int in_f32, int64_t id, const orc_map_step* step,
                   void* out) {
  orc_img cur;
  img_alloc(&cur, in_h, in_w, in_f32);
  const size_t n = (size_t)in_h * in_w * 3;
  if (in_f32) memcpy(cur.f, in, sizeof(float) * n);
  else memcpy(cur.u8, in, n);
  if (chain_step(&cur, step, id)) {
    img_free(&cur);
    return -1;
  }
  const size_t m = (size_t)cur.h * cur.w * 3;
  if (cur.f32) memcpy(out, cur.f, sizeof(float) * m);
  else memcpy(out, cur.u8, m);
  img_free(&cur);
  return 0;
}

int orc_chain_output(const orc_map_step* steps, int nsteps, int in_h, int in_w, int* out_h, int* out_w,
                     int* out_f32) {
  int h = in_h, w = in_w, f = 0;
  for (int i = 0; i < nsteps; ++i) {
    const orc_map_step* s = &steps[i];
    if (s->op == ORC_STEP_RANDOM_CROP || s->op == ORC_STEP_CENTER_CROP) {
      if (s->h > h || s->w > w || s->h < 1 || s->w < 1) return -1;
      h = s->h;
      w = s->w;
    } else if (s->op == ORC_STEP_RESIZE) {
      h = s->h;
      w = s->w;
      f = 1;
    } else if (s->op == ORC_STEP_NORMALIZE || s->op == ORC_STEP_AFFINE || s->op == ORC_STEP_CAST) {
      f = 1;
    } else {
      return -1;
    }
  }
  *out_h = h;
  *out_w = w;
  *out_f32 = f;
  return 0;
}

int orc_apply_chain(const uint8_t* img, int in_h, int in_w, int64_t id, const orc_map_step* steps, int nsteps,
                    void* out) {
  orc_img cur;
  img_alloc(&cur, in_h, in_w, 0);
  memcpy(cur.u8, img, (size_t)in_h * in_w * 3);
  for (int i = 0; i < nsteps; ++i)
    if (chain_step(&cur, &steps[i], id)) {
      img_free(&cur);
      return -1;
    }
  size_t n = (size_t)cur.h * cur.w * 3;
  if (cur.f32) memcpy(out, cur.f, sizeof(float) * n);
  else memcpy(out, cur.u8, n);
  img_free(&cur);
  return 0;
}

/* K7's position hash (SplitMix64Next of v ^ (pos * golden)), summed. */
static uint64_t pos_hash(uint64_t v, uint64_t pos) {
  uint64_t s = v ^ (pos * 0x9E3779B97F4A7C15ULL);
  return orc_splitmix64_next(&s);
}

typedef struct {
  const orc_map_step* steps;
  int nsteps, in_h, in_w;
  uint64_t pix_seed;
  const int64_t* ids;
  int64_t begin, end;
  uint64_t words; /* u32 words per output image */
  uint64_t sum;
  int err;
} digest_job;

static void* digest_worker(void* p) {
  digest_job* j = (digest_job*)p;
  const uint64_t ibytes = (uint64_t)j->in_h * j->in_w * 3;
  uint8_t* img = (uint8_t*)malloc(ibytes);
  uint32_t* out = (uint32_t*)malloc(j->words * 4);
  uint64_t acc = 0;
  for (int64_t k = j->begin; k < j->end; ++k) {
    orc_synth_images(j->pix_seed, (uint64_t)j->ids[k], 1, ibytes, img);
    if (orc_apply_chain(img, j->in_h, j->in_w, j->ids[k], j->steps, j->nsteps, out)) {
      j->err = 1;
      break;
    }
    const uint64_t base = (uint64_t)k * j->words;
    for (uint64_t w = 0; w < j->words; ++w) acc += pos_hash(out[w], base + w);
  }
  j->sum = acc;
  free(img);
  free(out);
  return NULL;
}

uint64_t orc_epoch_image_digest(const orc_map_step* steps, int nsteps, uint64_t pix_seed, const int64_t* ids,
                                int64_t n, int in_h, int in_w, int threads, int* err) {
  int oh, ow, f32;
  *err = 0;
  if (orc_chain_output(steps, nsteps, in_h, in_w, &oh, &ow, &f32) || ((uint64_t)oh * ow * 3 * (f32 ? 4 : 1)) % 4) {
    *err = 1;
    return 0;
  }
  const uint64_t words = (uint64_t)oh * ow * 3 * (f32 ? 4 : 1) / 4;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  digest_job jobs[256];
  pthread_t th[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (digest_job){steps, nsteps, in_h, in_w, pix_seed, ids, n * t / threads, n * (t + 1) / threads, words,
                           0, 0};
    pthread_create(&th[t], NULL, digest_worker, &jobs[t]);
  }
  uint64_t sum = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    sum += jobs[t].sum;
    *err |= jobs[t].err;
  }
  return sum;
}
