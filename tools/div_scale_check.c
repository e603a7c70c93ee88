/* Pins the exactness claim of err_ratio() in csrc/trace_reference.cu:
 * for 2^-900 <= |e| < 2^-120 and 2^-45 <= s <= 2^40,
 * RN(RN(e * 2^900) / s) * 2^-900 == RN(e / s) (IEEE binary64).
 * Build: gcc -O2 -ffp-contract=off tools/div_scale_check.c -o div_scale_check -lm
 * Usage: div_scale_check [cases]  -> "<bad> mismatches of <n>", exit 1 on any */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t st = 88172645463325252ULL;
static uint64_t xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
static double make(int emin, int emax) {
    uint64_t m = xr() & ((1ULL << 52) - 1);
    if (!(xr() & 7)) m |= ((1ULL << 52) - 1) ^ (xr() & 0xff);  /* mantissas near all ones */
    int e = emin + (int)(xr() % (uint64_t)(emax - emin + 1));
    uint64_t b = ((uint64_t)(e + 1023) << 52) | m;
    if (xr() & 1) b |= 1ULL << 63;
    double d;
    memcpy(&d, &b, 8);
    return d;
}
int main(int argc, char** argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 100000000LL, bad = 0;
    for (long long i = 0; i < n; i++) {
        double e = make(-900, -121), s = fabs(make(-45, 39));
        volatile double a = e * 0x1p900;
        volatile double q = a / s;
        double r = q * 0x1p-900, ref = e / s;
        if (memcmp(&r, &ref, 8) != 0) {
            if (bad < 5) printf("mismatch e=%a s=%a got=%a want=%a\n", e, s, r, ref);
            bad++;
        }
    }
    printf("%lld mismatches of %lld\n", bad, n);
    return bad != 0;
}
