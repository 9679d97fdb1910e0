/* Exhaustive check of the fp32-only quantizer thresholds (mkv_common.cuh group_thresholds_fast)
 * against the double-precision definition (group_thresholds) for EVERY positive fp32 scale in
 * [2^-100, 2^100] -- the fp16 input domain needs [2^-26, 2^16].
 *   T_k = the smallest float >= m_k * sc, m_k = midpoint of c_k = k + 0.5 and its predecessor
 *       = c_k - d_k with d_k = 2^-26, 2^-24, 2^-23.
 * fp32 method: ds = sc * d_k (exact), y = fma(c_k, sc, -ds) (= fl(m_k * sc)), r = fma(-c_k, sc, y)
 * (= y - c_k * sc exactly), T_k = (r >= -ds) ? y : nextup(y).
 *   gcc -O2 -ffp-contract=off -o /tmp/thr tools/threshold_fp32_check.c -lm && /tmp/thr */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static float f_of(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t b_of(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

int main(void) {
    const float c[3] = {0.5f, 1.5f, 2.5f};
    const float d[3] = {0x1p-26f, 0x1p-24f, 0x1p-23f};
    for (int k = 0; k < 3; ++k) { /* d_k is exactly c_k minus the midpoint below it */
        const double m = 0.5 * ((double)nextafterf(c[k], 0.0f) + (double)c[k]);
        if ((double)c[k] - m != (double)d[k]) { printf("bad d[%d]\n", k); return 1; }
    }
    const uint32_t b0 = b_of(0x1p-100f), b1 = b_of(0x1p100f);
    uint64_t n = 0, bad = 0;
    for (uint32_t b = b0; b <= b1; ++b) {
        const float sc = f_of(b);
        for (int k = 0; k < 3; ++k) {
            const double m = (double)c[k] - (double)d[k];
            const double prod = m * (double)sc;
            float x = (float)prod;
            if ((double)x < prod) x = nextafterf(x, INFINITY);
            const float ds = sc * d[k];
            const float y = fmaf(c[k], sc, -ds);
            const float r = fmaf(-c[k], sc, y);
            const float t = (r >= -ds) ? y : f_of(b_of(y) + 1u);
            if (b_of(t) != b_of(x)) {
                if (bad < 10) printf("mismatch sc=%a k=%d double=%a fp32=%a\n", sc, k, x, t);
                ++bad;
            }
            ++n;
        }
    }
    printf("checked %llu (scale, k) pairs over [2^-100, 2^100]: %llu mismatches\n", (unsigned long long)n,
           (unsigned long long)bad);
    return bad != 0;
}
