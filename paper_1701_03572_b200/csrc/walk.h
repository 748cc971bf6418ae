// walk.h — exact closed form of the reference's row-incremental coordinate
// walk (warp_similarity, image_ops.cpp:124-131):
//
//     s_0 = row start;  s_{k+1} = fl(s_k + d)   (k sequential IEEE additions)
//
// A direct s_0 + k*d differs from the walk by a few ulps, which is enough to
// move a bilinear sample across a .5 rounding tie.  Inside one binade
// [2^e, 2^(e+1)) every s_k is a multiple of ulp_e, and fl(s_k + d) adds the
// same multiple of ulp_e each step — except in a round-half-even tie, where
// the first step lands on an even multiple and every later step then adds a
// constant again.  So: take real steps until two consecutive increments
// agree, jump in one exact multiply-add to just before the binade edge, and
// take real steps across the edge.  Cost ~10 fp ops per binade crossed.
// Verified against brute force in tests/test_walk.py.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define WALK_HD __host__ __device__ __forceinline__
#else
#define WALK_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define WALK_ADD(a, b) __dadd_rn((a), (b))
#define WALK_MUL(a, b) __dmul_rn((a), (b))
#else
#define WALK_ADD(a, b) ((a) + (b))
#define WALK_MUL(a, b) ((a) * (b))
#endif

// fl-walk of n steps of +d from s (n >= 0).
WALK_HD double fl_walk(double s, double d, long long n) {
    if (d == 0.0) return s;
    const double ad = fabs(d);
    double prev_inc = 0.0;
    int agree = 0;  // consecutive steps with equal increments seen
    while (n > 0) {
        const double as = fabs(s);
        if (as >= 8.0 * ad && agree >= 2) {
            // binade of s and the safe interval for pre-step values
            int e;
            frexp(as, &e);  // as in [2^(e-1), 2^e)
            const double lo = ldexp(1.0, e - 1), hi = ldexp(1.0, e);
            // |s_j| must stay in [lo + 2|d|, hi - 2|d|] so s_j + d stays in the binade
            const double inc = prev_inc;  // constant increment (exact multiple of ulp)
            const double ainc = fabs(inc);
            if (ainc > 0.0) {
                // |s| moves by +-ainc per step (same sign as inc * s)
                const int grows = (inc > 0.0) == (s > 0.0);
                const double room = grows ? (hi - 2.0 * ad) - as : as - (lo + 2.0 * ad);
                long long k = room > 0.0 ? (long long)floor(room / ainc) : 0;
                if (k > n) k = n;
                if (k > 0) {
                    s = WALK_ADD(s, WALK_MUL((double)k, inc));  // exact: stays on the ulp grid
                    n -= k;
                    if (n == 0) break;
                }
            }
            agree = 0;  // re-establish the increment after the boundary
        }
        const double t = WALK_ADD(s, d);
        const double inc = t - s;  // exact (Sterbenz) whenever it matters
        int es, et;
        frexp(s, &es);
        frexp(t, &et);
        const int same_binade = es == et && ((s > 0.0) == (t > 0.0)) && s != 0.0 && t != 0.0;
        if (!same_binade) agree = 0;
        else agree = (agree > 0 && inc == prev_inc) ? agree + 1 : 1;
        prev_inc = inc;
        s = t;
        --n;
    }
    return s;
}
