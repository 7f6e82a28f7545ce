"""The restated libm log (paper_2512_19925_b200/csrc/libm_log.h) against the
host's own log(), bit for bit, on the transport kernels' input domain (uniform
deviates ((u >> 11) + 0.5) * 2^-53), the near-1 branch and random doubles.
Compiled on the fly with gcc (no FMA contraction) — runs on CPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r"""
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
#include "libm_log.h"
static uint64_t s[4] = {11, 22, 33, 44};
static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static uint64_t nx(void) { uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45); return r; }
int main(int argc, char** argv) {
  long n = atol(argv[1]), bad = 0;
  for (long i = 0; i < n; ++i) {
    double u = ((double)(nx() >> 11) + 0.5) * 0x1.0p-53;
    if (hwwg_libm_log(u) != log(u)) ++bad;
    double v = 0.9375 + 0.13 * u;
    if (hwwg_libm_log(v) != log(v)) ++bad;
    uint64_t b = nx() & 0x7fffffffffffffffULL; double x; memcpy(&x, &b, 8);
    double a = hwwg_libm_log(x), c = log(x);
    if (!(a == c || (isnan(a) && isnan(c)))) ++bad;
  }
  printf("%ld\n", bad);
  return 0;
}
"""


def test_restated_log_is_bit_exact(tmp_path):
    inc = [os.path.join(ROOT, "paper_2512_19925_b200", "csrc"),
           os.path.join(ROOT, "paper_2512_19925_b200", "_build")]
    if not os.path.exists(os.path.join(inc[1], "libm_log_table.h")):
        pytest.skip("engine not built")
    c = tmp_path / "t.c"
    c.write_text(SRC.replace("#include <stdio.h>", "#include <stdio.h>\n#include <stdlib.h>"))
    exe = tmp_path / "t"
    subprocess.run(["/usr/bin/gcc", "-O2", "-ffp-contract=off", "-I", inc[0], "-I", inc[1],
                    str(c), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe), "3000000"], check=True, capture_output=True, text=True)
    assert int(out.stdout.strip()) == 0
