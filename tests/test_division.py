"""K5 divides by the level's determinant with one reciprocal per level and a
Markstein correction per iteration (k_lk.cu div_rn_recip): q0 = RN(a*y),
r = fma(-q0, b, a), q = fma(r, y, q0) with y = RN(1/b).  The claim is that q
equals the IEEE quotient RN(a/b) bit for bit.  This checks it on the host
(same IEEE binary64 FMA semantics as DFMA) over random operands, including
divisors whose significands are all ones or near powers of two."""
import os
import shutil
import subprocess
import tempfile

import pytest

SRC = r"""
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double mk(int hard) {
    uint64_t m = rnd() & ((1ull << 52) - 1);
    if (hard == 1) m |= ((1ull << 52) - 1) & ~((1ull << (rnd() % 20)) - 1);
    if (hard == 2) m &= (1ull << (rnd() % 20)) - 1;
    int e = -80 + (int)(rnd() % 161);
    uint64_t bits = ((uint64_t)(e + 1023) << 52) | m | ((rnd() & 1) << 63);
    double d;
    memcpy(&d, &bits, 8);
    return d;
}
int main(int argc, char** argv) {
    long n = atol(argv[1]), bad = 0;
    for (long i = 0; i < n; ++i) {
        double a = mk((int)(rnd() % 3)), b = mk((int)(rnd() % 3));
        volatile double y = 1.0 / b;
        volatile double q0 = a * y;
        double q = fma(fma(-q0, b, a), y, q0);
        if (q != a / b) ++bad;
    }
    printf("%ld\n", bad);
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_markstein_division_is_correctly_rounded():
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c, "w").write(SRC.replace("#include <string.h>", "#include <string.h>\n#include <stdlib.h>"))
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", c, "-o", exe, "-lm"], check=True)
        out = subprocess.run([exe, "20000000"], capture_output=True, text=True, check=True).stdout
    assert int(out) == 0
