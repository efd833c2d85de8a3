#!/usr/bin/env python
"""Mutation check of the oracle's pins: apply one plausible mistake at a time to a copy of
oracle/oracle.c and run the CPU oracle tests against it; every mutation must fail a test.

    python tools/oracle_mutations.py [--out profiles/r02_oracle_mutations.txt]

Each mutation names the reading it breaks (DESIGN.md R#n / SPEC.md S:n). Runs on CPU only.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, reading, old, new, occurrence index or None for all)
MUTATIONS = [
    ("schlick (1-c)^5 -> (1-c)^4", "S:179", "m * m * m * m * m", "m * m * m * m", None),
    ("exit-side Schlick cosine cos_t -> cos_i", "S:300, R#10",
     "double c = entering ? ci : sqrt(1.0 - sin2t);", "double c = ci;", None),
    ("DIFFUSE-kr weight T*=kr -> T*=rho", "S:299, R#8", "T = scl(T, kr);", "T = mulv(T, rho);", None),
    ("drop REFRACTIVE T*=rho", "S:300, R#9", "      T = mulv(T, rho);\n      An_next = eta", "      An_next = eta", None),
    ("shadow origin p + EPS_T n -> p", "S:157, R#12", "v3 os = add(p, scl(n, EPS_T));", "v3 os = p;", 0),
    ("ambient at every hit", "R#4",
     "      L = add(L, mulv(T, mulv(rho, amb))); /* ambient, unshadowed (reading R#4) */\n", "", None),
    ("RNG key pixel+1 -> pixel", "S:307-314",
     "uint64_t x = seed ^ ((pixel_index + 1ULL) * GOLDEN);\n  x = orc_mix64(x);\n  x = orc_mix64(x ^ ((((uint64_t)sample",
     "uint64_t x = seed ^ ((pixel_index) * GOLDEN);\n  x = orc_mix64(x);\n  x = orc_mix64(x ^ ((((uint64_t)sample", None),
    ("closest-hit ties -> last index (<=)", "S:73, R#16",
     "if (prim_hit(P, k, o, d, &t) && t < tbest) { tbest = t; best = k; }\n    }\n    cnt->sphere_tests",
     "if (prim_hit(P, k, o, d, &t) && t <= tbest) { tbest = t; best = k; }\n    }\n    cnt->sphere_tests", None),
    # (a sphere root equal to EPS_T is unreachable from float inputs: the stable-root arithmetic
    # never lands on the double nearest 1e-4; the plane root dp / den does)
    ("EPS_T acceptance >= -> > (planes)", "S:63, S:104, R#12", "if (tt >= EPS_T) { *t = tt; return 1; }",
     "if (tt > EPS_T) { *t = tt; return 1; }", None),
    ("EPS_T 1e-4 -> 1e-5", "S:104, R#12", "#define EPS_T 1e-4", "#define EPS_T 1e-5", None),
    ("normal not flipped toward the ray", "S:47, R#17", "v3 n = entering ? ng : scl(ng, -1.0);", "v3 n = ng;", None),
    ("Phong (s+2)/(2pi) -> (s+1)/(2pi)", "R#3", "(shininess + 2.0) / (2.0 * PI)", "(shininess + 1.0) / (2.0 * PI)", None),
    ("point-light falloff cos/d^2 -> cos/d", "Eq. 3, R#2", "double g = cos_t / d2;", "double g = cos_t / sqrt(d2);", None),
    ("shadow interval [EPS,t_max) -> [EPS,t_max]", "S:157, R#13",
     "if (prim_hit(P, k, os, ds, &t) && t < tmax) { occluded = 1; break; }\n        }\n        if (want_margin) {\n          int self_in",
     "if (prim_hit(P, k, os, ds, &t) && t <= tmax + 1.0) { occluded = 1; break; }\n        }\n        if (want_margin) {\n          int self_in", None),
    ("refraction eta entering 1/ior -> ior", "S:88, R#10", "double eta = entering ? 1.0 / ior : ior;",
     "double eta = entering ? ior : 1.0 / ior;", None),
    ("camera right = up x f (left-handed)", "S:229, R#18", "cam.r = normalize(cross(cam.f, ld3(sc->up)));",
     "cam.r = normalize(cross(ld3(sc->up), cam.f));", None),
]


def apply(src: str, old: str, new: str, occ):
    if old not in src:
        raise ValueError(f"pattern not found: {old[:60]!r}")
    if occ is None:
        return src.replace(old, new)
    i = -1
    for _ in range(occ + 1):
        i = src.index(old, i + 1)
    return src[:i] + new + src[i + len(old):]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--tests", default="tests/test_oracle_continuation.py tests/test_oracle_render.py "
                                        "tests/test_oracle_geometry.py tests/test_oracle_next.py tests/test_oracle_alg1.py")
    a = ap.parse_args()
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    lines = []
    ok_all = True
    for name, reading, old, new, occ in MUTATIONS:
        tmp = tempfile.mkdtemp(prefix="orcmut")
        try:
            shutil.copytree(ROOT, os.path.join(tmp, "r"), ignore=shutil.ignore_patterns(
                ".git", "gpurun_out", "*.so", "__pycache__", "baseline"))
            r = os.path.join(tmp, "r")
            open(os.path.join(r, "oracle", "oracle.c"), "w").write(apply(src, old, new, occ))
            res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "not gpu",
                                  *a.tests.split()], cwd=r, capture_output=True, text=True, timeout=1800)
            failed = [ln.split(" - ")[0].replace("FAILED ", "") for ln in res.stdout.splitlines()
                      if ln.startswith("FAILED")]
            caught = res.returncode != 0 and bool(failed)
            ok_all &= caught
            first = failed[0] if failed else "(none)"
            lines.append(f"{'CAUGHT ' if caught else 'MISSED '} {name:48s} [{reading}]  {len(failed)} failing, e.g. {first}")
            print(lines[-1], flush=True)
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
    txt = "\n".join(lines) + f"\n{'all mutations caught' if ok_all else 'SOME MUTATIONS MISSED'}\n"
    if a.out:
        open(a.out, "w").write(txt)
    return 0 if ok_all else 1


if __name__ == "__main__":
    sys.exit(main())
