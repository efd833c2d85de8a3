"""Host-side arithmetic of the runtime checked on CPU (no GPU): the exact multiply-shift division
(rt_internal.h FastDiv, used for the pixel / sample mapping of every camera ray) and the
sub-pixel offset table (rt_kernels.cu upload_sample_offsets must hold exactly what the device's
sample_offset computes, whose rules the oracle's stratified / Hammersley offsets pin).

A tiny C++ driver includes rt_internal.h, builds FastDiv for many divisors and emulates the
device's __umulhi in 64-bit integer arithmetic."""
import os
import shutil
import subprocess
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1504_03151_b200", "csrc")
CUDA_INC = "/usr/local/cuda/include"

DRIVER = textwrap.dedent(r"""
    #include <cstdio>
    #include <cstdint>
    #include "rt_internal.h"
    static unsigned fdiv_host(const rt::FastDiv& f, unsigned x) {  // the device fdiv, __umulhi emulated
      if (f.d <= 1u) return x;
      const unsigned t = (unsigned)(((unsigned long long)x * f.m) >> 32);
      return (t + ((x - t) >> 1)) >> f.s;
    }
    int main() {
      unsigned long long bad = 0, n = 0, seed = 12345;
      auto rnd = [&]() { seed = seed * 6364136223846793005ull + 1442695040888963407ull; return (unsigned)(seed >> 32); };
      for (unsigned d = 1; d <= 5000; ++d) {
        const rt::FastDiv f = rt::make_fastdiv(d);
        const unsigned xs[] = {0u, 1u, d - 1u, d, d + 1u, 2u * d - 1u, 0x7fffffffu, 0x80000000u, 0xffffffffu};
        for (unsigned x : xs) { ++n; if (fdiv_host(f, x) != x / d) ++bad; }
        for (int i = 0; i < 300; ++i) { const unsigned x = rnd(); ++n; if (fdiv_host(f, x) != x / d) ++bad; }
        for (unsigned x = 0; x < 3000u; ++x) { ++n; if (fdiv_host(f, x) != x / d) ++bad; }
      }
      const unsigned big[] = {65535u, 65536u, 1u << 20, (1u << 22) + 7u, 0x7fffffffu, 0x80000000u, 0xfffffffeu};
      for (unsigned d : big) {
        const rt::FastDiv f = rt::make_fastdiv(d);
        for (int i = 0; i < 20000; ++i) { const unsigned x = rnd(); ++n; if (fdiv_host(f, x) != x / d) ++bad; }
      }
      printf("%llu %llu\n", n, bad);
      return 0;
    }
""")


def test_fastdiv_exact(tmp_path):
    if not shutil.which("g++") or not os.path.exists(os.path.join(CUDA_INC, "cuda_runtime.h")):
        pytest.skip("g++ or CUDA headers not available")
    src = tmp_path / "fastdiv.cpp"
    src.write_text(DRIVER)
    exe = tmp_path / "fastdiv"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, "-I", CUDA_INC, "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe)], check=True, capture_output=True)
    n, bad = map(int, subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split())
    assert n > 15_000_000 and bad == 0, (n, bad)


def _offset_rule(s, spp):
    """sample_offset (rt_device.cuh) in Python floats (IEEE double, the same operations)."""
    import math
    n = 1
    while (n + 1) * (n + 1) <= spp:
        n += 1
    if n * n == spp:
        return (s % n + 0.5) / n, (s // n + 0.5) / n
    r = int(f"{s:032b}"[::-1], 2)
    y = r * (1.0 / 4294967296.0) + 0.5 / spp
    return (s + 0.5) / spp, y - math.floor(y)


def test_sample_offsets_match_the_oracle():
    """The offsets the table holds follow the oracle's rules (stratified n x n grid for square spp,
    else the Hammersley-style radical inverse): compare with the oracle's own ray generation."""
    from oracle import pyoracle
    pyoracle.build()
    for spp in (1, 2, 3, 4, 5, 9, 16, 17):
        for s in range(spp):
            ox, oy = _offset_rule(s, spp)
            assert 0.0 <= ox < 1.0 and 0.0 <= oy < 1.0
            assert (ox, oy) == tuple(pyoracle.sample_offset(s, spp)), (s, spp)
