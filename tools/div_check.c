/* Pins the reciprocal-corrected divisions (csrc/table.cu div_by: general
 * operands, see main) and the camera_ray division in csrc/device_common.cuh:
 * for a = px + sx
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
static double make(int emin, int emax, int ones) {
    uint64_t m = xr() & ((1ULL << 52) - 1);
    if (ones) m |= ((1ULL << 52) - 1) ^ (xr() & 0xff);  /* mantissas near all ones */
    const int e = emin + (int)(xr() % (uint64_t)(emax - emin + 1));
    const uint64_t bits = ((uint64_t)(e + 1023) << 52) | m;
    double d;
    memcpy(&d, &bits, 8);
    return d;
}
int main(int argc, char** argv) {
    const long long per = argc > 1 ? atoll(argv[1]) : 300;
    /* general operands (table.cu div_by): |a| in [2^-900, 2^900], b in [2^-60, 2^60] */
    for (long long i = 0; i < 400 * per; ++i) {
        const double b = make(-60, 60, (i & 7) == 0);
        const double a = make(-900, 899, (i & 7) == 1) * ((i & 1) ? -1.0 : 1.0);
        check(a, b, 1.0 / b);
    }
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
