/* Exhaustive proof that the device normalize's division sequence
 *   d = RN(v - M);  q = RN(d * r);  rem = RN(d - q*s) (fma);  q' = RN(q + rem*r) (fma)
 * with r = RN(1/s) equals IEEE RN(d / s) for EVERY fp32 v in [0, 255] and the
 * three ImageNet channels (every value K4's bilinear blend can produce).
 * Build: gcc -O2 -ffp-contract=off -fopenmp tools/prove_fast_div.c -lm
 * (fmaf from libm is correctly rounded).  Prints mismatches; 0 == proven. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
static float f_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
int main(void) {
  const float M[3] = {123.675f, 116.28f, 103.53f}, S[3] = {58.395f, 57.12f, 57.375f};
  const uint32_t hi = 0x437f0000u; /* 255.0f */
  long long bad = 0;
  for (int c = 0; c < 3; ++c) {
    const float s = S[c], r = 1.0f / s, m = M[c];
    long long badc = 0;
#pragma omp parallel for reduction(+ : badc) schedule(static, 1 << 20)
    for (long long u = 0; u <= (long long)hi; ++u) {
      float v = f_of((uint32_t)u);
      volatile float d = v - m;
      volatile float want = d / s;
      volatile float q = d * r;
      float rem = fmaf(-q, s, d);
      float got = fmaf(rem, r, q);
      if (memcmp(&got, (const void*)&want, 4) != 0) badc++;
    }
    printf("channel %d: %lld mismatches over %u inputs\n", c, badc, hi + 1);
    bad += badc;
  }
  printf("TOTAL mismatches: %lld\n", bad);
  return bad != 0;
}
