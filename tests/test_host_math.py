"""Host-side checks of integer helpers the remap kernels rely on (no GPU): the fast-division
multiplier of psm_device.cuh (make_fastdiv / fast_div, used to decode tile indices in
k_remap.cu) must give n / d exactly for every 32-bit n; checked here by compiling a small
program against the header with the device __umulhi replaced by its definition (high 32 bits
of the 64-bit product) and comparing with plain division over edge cases and random n."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2502_20049_b200", "csrc")

PROG = r"""
#include <cstdio>
#include <cstdint>
#include <random>
#include "psm_device.cuh"
static uint32_t umulhi(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
static uint32_t fdiv(uint32_t n, const psm::FastDiv& f) {
  return (uint32_t)(((uint64_t)umulhi(n, f.m) + n) >> f.l);  // fast_div with __umulhi spelled out
}
int main() {
  std::mt19937_64 rng(7);
  const uint32_t ds[] = {1u, 2u, 3u, 5u, 7u, 16u, 17u, 31u, 32u, 33u, 100u, 128u, 129u, 255u,
                         4096u, 65535u, 65536u, 524287u, 1u << 20, (1u << 20) + 3u, 2147483647u,
                         2147483648u, 4294967295u};
  long bad = 0, n_checked = 0;
  for (uint32_t d : ds) {
    const psm::FastDiv f = psm::make_fastdiv(d);
    const uint32_t edge[] = {0u, 1u, d - 1u, d, d + 1u, 2u * d - 1u, 2u * d, 4294967295u,
                             4294967294u, 2147483647u, 2147483648u};
    for (uint32_t n : edge) { ++n_checked; if (fdiv(n, f) != n / d) ++bad; }
    for (int k = 0; k < 200000; ++k) {
      const uint32_t n = (uint32_t)rng();
      ++n_checked;
      if (fdiv(n, f) != n / d) ++bad;
      const uint32_t q = (uint32_t)rng() % 4096u, r = (uint32_t)rng() % d;  // exact multiples
      const uint64_t nn = (uint64_t)q * d + r;
      if (nn <= 4294967295ull) { ++n_checked; if (fdiv((uint32_t)nn, f) != q) ++bad; }
    }
  }
  for (uint32_t d = 1; d < 3000; ++d) {  // every small divisor, the tile-grid range
    const psm::FastDiv f = psm::make_fastdiv(d);
    for (uint32_t n = 0; n < 200000; n += 7) { ++n_checked; if (fdiv(n, f) != n / d) ++bad; }
  }
  std::printf("%ld %ld\n", n_checked, bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_fastdiv_exact_for_all_tested_numerators():
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "fd.cpp")
        exe = os.path.join(td, "fd")
        with open(src, "w") as fh:
            fh.write(PROG)
        subprocess.run(["g++", "-std=c++17", "-O2", "-I", CSRC, "-I", "/usr/local/cuda/include",
                        src, "-o", exe], check=True, capture_output=True)
        out = subprocess.run([exe], capture_output=True, text=True)
        checked, bad = map(int, out.stdout.split())
        assert checked > 5_000_000
        assert bad == 0 and out.returncode == 0
