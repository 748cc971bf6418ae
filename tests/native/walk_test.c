/* Brute-force check of fl_walk (paper_1701_03572_b200/csrc/walk.h) against
 * k sequential IEEE additions.  Test infrastructure. */
#include <stdint.h>
#include <string.h>

#include "../../paper_1701_03572_b200/csrc/walk.h"

static uint64_t st;
static uint64_t nx(void) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static double u01(void) { return (double)(nx() >> 11) * 0x1.0p-53; }

/* returns the number of mismatching (s0, d, n) cases out of `cases` */
long long walk_check(uint64_t seed, long long cases, int maxn, double smax, double* worst) {
    st = seed;
    long long bad = 0;
    for (long long c = 0; c < cases; ++c) {
        double s0 = (u01() * 2 - 1) * smax;
        if ((nx() & 7) == 0) s0 = (double)(int64_t)(s0);       /* integer starts */
        double d = 0.4 + 1.2 * u01();
        if (nx() & 1) d = -d;
        if ((nx() & 15) == 0) d = 1.0;                          /* exact steps */
        if ((nx() & 15) == 0) d = ldexp(u01() + 1.0, -(int)(nx() % 6)); /* small steps */
        const int n = (int)(nx() % (uint64_t)maxn);
        double s = s0;
        int ok = 1;
        for (int k = 1; k <= n; ++k) {
            s = s + d;
            if ((k & 63) == 0 || k == n) {
                const double e = fl_walk(s0, d, k);
                if (memcmp(&e, &s, sizeof s) != 0) {
                    ok = 0;
                    if (worst) *worst = s0;
                    break;
                }
            }
        }
        bad += !ok;
    }
    return bad;
}

double walk_eval(double s0, double d, long long n) { return fl_walk(s0, d, n); }
