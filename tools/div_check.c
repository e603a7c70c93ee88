/* Pins the camera_ray division in csrc/device_common.cuh: for a = px + sx
 * (px an integer pixel index < 2^16, sx in [0, 1) a 53-bit sample offset)
 * and b = width < 2^16, with y = RN(1/b) from the host,
 *   q0 = RN(a y), q = RN(q0 + RN?(a - q0 b) y)  [two fmas]
 * equals the IEEE quotient a / b. Every width 1..65535 is checked with
 * random and edge numerators (px = 0 / b - 1, sx = 0 / 0.5 / 1 - 2^-53).
 * Build: gcc -O2 -mfma -ffp-contract=off tools/div_check.c -o div_check -lm
 * Usage: div_check [random cases per width]  -> "<bad> mismatches of <n>" */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t st = 88172645463325252ULL;
static uint64_t xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }

static long long bad = 0, n = 0;
static void check(double a, double b, double y) {
    const double q0 = a * y;
    const double q = fma(fma(-q0, b, a), y, q0);
    const double ref = a / b;
    ++n;
    if (memcmp(&q, &ref, 8) != 0) {
        if (bad < 5) printf("mismatch a=%a b=%a got=%a want=%a\n", a, b, q, ref);
        ++bad;
    }
}
int main(int argc, char** argv) {
    const long long per = argc > 1 ? atoll(argv[1]) : 300;
    for (int w = 1; w < 65536; ++w) {
        const double b = (double)w, y = 1.0 / b;
        const double sxs[3] = {0.0, 0.5, 1.0 - 0x1p-53};
        for (int k = 0; k < 3; ++k) {
            check(0.0 + sxs[k], b, y);
            check((double)(w - 1) + sxs[k], b, y);
        }
        for (long long i = 0; i < per; ++i) {
            const double px = (double)(xr() % (uint64_t)w);
            const double sx = (double)(xr() >> 11) * 0x1.0p-53;
            check(px + sx, b, y);
        }
    }
    printf("%lld mismatches of %lld\n", bad, n);
    return bad != 0;
}
