"""Pins for the oracle's continuation weights, Schlick arithmetic, shadow-ray origin, ambient rule,
RNG composition and test counting (CPU, no GPU).

Each test is a closed form or a hand count for a scene built so that one reading of the paper /
SPEC decides the result, chosen so that a plausible mistake in that part of oracle.c (a wrong
exponent, the wrong cosine, a dropped or swapped weight, a missing offset) changes the value:

  * Schlick's approximation F = R0 + (1 - R0)(1 - c)^5 and its cosine on the less
    dense side (R#10): exit-side Fresnel uses cos(theta_t), not cos(theta_i);
  * the DIFFUSE-kr mirror weight T *= kr and the REFRACTIVE weight T *= rho (PAPER.md
    P:212-222 reflection/refraction continuation; R#8, R#9);
  * the shadow ray leaves from p + EPS_T n (R#12);
  * ambient at DIFFUSE hits only (BASELINE.json north_star "shadowed points get ambient only"; R#4);
  * the counter RNG is splitmix64 keyed by (pixel + 1) then by the (sample, depth) word
    (§8(c).1 step 9), checked against an independent splitmix64 stream;
  * algorithmic test counts in index order with the Alg. 1 `break` (§8(c).1 step 11).
"""
import math

import numpy as np
import pytest

import scenegen
from scenegen import DIFFUSE, REFRACTIVE, SPECULAR, SplitMix64

_MASK = (1 << 64) - 1
_G = 0x9E3779B97F4A7C15


def _f32(x):
    return float(np.float32(x))


# ---- Schlick ---------------------------------------------------------------------------
def test_schlick_closed_forms(oracle_lib):
    # R0 = ((1 - 1.5) / (1 + 1.5))^2 = 0.04; at c = 1/2: 0.04 + 0.96 / 32 = 0.07
    assert oracle_lib.schlick(1.5, 0.5) == pytest.approx(0.07, rel=1e-14)
    assert oracle_lib.schlick(1.5, 1.0) == pytest.approx(0.04, rel=1e-14)
    assert oracle_lib.schlick(1.5, 0.0) == pytest.approx(1.0, rel=1e-15)
    # ior 2: R0 = 1/9; c = 3/4: 1/9 + (8/9) / 4^5 = 1/9 + 1/1152
    assert oracle_lib.schlick(2.0, 0.75) == pytest.approx(1 / 9 + 1 / 1152, rel=1e-14)
    # ior 1: R0 = 0, F = (1 - c)^5; c = 0.8 -> 0.2^5
    assert oracle_lib.schlick(1.0, 0.8) == pytest.approx(0.2 ** 5, rel=1e-12)


def _exit_scene(seed, albedo=(1, 1, 1), bg=(0.25, 0.5, 0.75), max_depth=1):
    """Camera inside a glass sphere (ior 1.5) centred (0.6, 0, 0), r = 1, looking +z: the camera
    ray leaves the sphere at z = sqrt(1 - 0.6^2) with cos(theta_i) = 0.8 on the dense side."""
    b = scenegen.builder()
    b.sphere((0.6, 0, 0), 1.0, b.material(REFRACTIVE, albedo, ior=1.5))
    return b.build("exit", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                   max_depth=max_depth, spp=1, background=bg, seed=seed)


def test_schlick_exit_side_uses_transmitted_cosine(oracle_lib):
    # Leaving the glass, Schlick's cosine is the one on the less dense side (R#10):
    # sin^2(theta_t) = ior^2 (1 - cos^2 theta_i) = 2.25 cx^2, c = sqrt(1 - sin^2 theta_t).
    cx = _f32(0.6)
    F_exit = 0.04 + 0.96 * (1 - math.sqrt(1 - 2.25 * cx * cx)) ** 5   # ~0.0950
    F_inc = 0.04 + 0.96 * (1 - math.sqrt(1 - cx * cx)) ** 5           # ~0.0403 (the wrong cosine)
    bg = (0.25, 0.5, 0.75)
    in_band = 0
    for seed in range(3000):
        u = oracle_lib.rng(seed, 0, 0, 0)
        if abs(u - F_exit) < 1e-9:
            continue
        r = oracle_lib.render(_exit_scene(seed))
        if u < F_exit:
            # internal reflection: the ray stays inside, hits the (non-emissive) glass again at
            # depth 1 = max_depth and ends with nothing added
            assert r.rgb[0].tolist() == [0.0, 0.0, 0.0], seed
            assert list(r.hit_ids[0, 0]) == [0, 0], seed
        else:
            # refraction out of the sphere, miss -> background with T = rho = 1
            assert r.rgb[0].tolist() == [_f32(x) for x in bg], seed
            assert list(r.hit_ids[0, 0]) == [0, -1], seed
        in_band += F_inc <= u < F_exit
    assert in_band >= 50  # the draws that separate the two cosine choices were exercised


# ---- continuation weights -------------------------------------------------------------
def _diffuse_mirrors(D, kr=0.25, rho=(0.9, 0.6, 0.3), ambient=(0, 0, 0)):
    b = scenegen.builder()
    m = b.material(DIFFUSE, rho, emission=(1, 1, 1), kr=kr)
    b.plane((0, 0, 1), 0.0, m)
    b.plane((0, 0, 1), 10.0, m)
    return b.build("kr-mirrors", eye=(0, 0, 5), look_at=(0, 0, 6), up=(0, 1, 0), vfov=30, width=1, height=1,
                   max_depth=D, spp=1, ambient=ambient)


@pytest.mark.parametrize("D", [0, 1, 2, 5, 8])
def test_diffuse_kr_mirror_weight(oracle_lib, D):
    # DIFFUSE with kr > 0 mirrors with weight kr, not rho (R#8): no lights, no ambient, emission 1
    # at every hit -> L = sum_{i<=D} kr^i in every channel (exact in binary for kr = 1/4)
    r = oracle_lib.render(_diffuse_mirrors(D))
    want = sum(0.25 ** i for i in range(D + 1))
    assert r.rgb[0].tolist() == [want] * 3
    assert r.bounces[0, 0] == D
    # kr = 0 stops the path at the first hit (Whitted: no diffuse bounce)
    r0 = oracle_lib.render(_diffuse_mirrors(D, kr=0.0))
    assert r0.rgb[0].tolist() == [1.0] * 3 and r0.bounces[0, 0] == 0


def test_coloured_glass_weights(oracle_lib):
    # W5 with coloured glass rho = (1/2, 1/4, 1): normal incidence keeps the direction; the branch
    # taken is a pure function of the integer RNG (T *= rho per glass bounce):
    #   refract in, refract out, miss   -> background * rho^2
    #   reflect at entry, miss           -> background * rho
    #   refract in, reflect inside, stop -> 0 (max_depth 2 reached inside, no emission)
    rho = (0.5, 0.25, 1.0)
    bg = (0.25, 0.5, 0.75)
    seen = set()
    b = scenegen.builder()
    b.sphere((0, 0, 5), 1.0, b.material(REFRACTIVE, rho, ior=1.5))
    for seed in range(80):
        sc = b.build("glass", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                     max_depth=2, spp=1, background=bg, seed=seed)
        u0, u1 = oracle_lib.rng(seed, 0, 0, 0), oracle_lib.rng(seed, 0, 0, 1)
        r = oracle_lib.render(sc)
        if u0 >= 0.04 and u1 >= 0.04:
            assert r.rgb[0].tolist() == [bg[c] * rho[c] ** 2 for c in range(3)], seed
            seen.add("tt")
        elif u0 < 0.04:
            assert r.rgb[0].tolist() == [bg[c] * rho[c] for c in range(3)], seed
            seen.add("r")
        else:
            assert r.rgb[0].tolist() == [0.0, 0.0, 0.0], seed
            seen.add("tr")
    assert "tt" in seen and len(seen) >= 2


# ---- shadow-ray origin --------------------------------------------------------------------
def _offset_scene(gap):
    """A DIFFUSE floor y = 0 and a second plane y = gap above it; the camera sits between them
    (y = 7.5e-5) looking down at 30 degrees, so its ray meets the floor at t = 1.5e-4 >= EPS_T.
    A light 10 units straight above the hit point."""
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.5, 0.5, 0.5)))
    b.plane((0, 1, 0), gap, b.material(DIFFUSE, (0.5, 0.5, 0.5)))
    b.light((0, 10, 0), (200 * math.pi,) * 3)
    y = 7.5e-5
    return b.build("offset", eye=(0, y, 0), look_at=(0, y - 0.5, math.sqrt(0.75)), up=(0, 1, 0), vfov=30,
                   width=1, height=1, max_depth=0, spp=1, ambient=(0.1, 0.1, 0.1))


def test_shadow_origin_offset_decides_occlusion(oracle_lib):
    # gap 1.5e-4: from o_s = p + EPS_T n the second plane lies at t = 0.5e-4 < EPS_T (not an
    # occluder) -> lit; traced from p itself it would be at 1.5e-4 >= EPS_T -> occluded
    r = oracle_lib.render(_offset_scene(1.5e-4))
    amb = 0.5 * _f32(0.1)
    lit = 0.5 / math.pi * _f32(200 * math.pi) / 100.0 + amb  # rho/pi I cos / d^2, cos ~ 1, d^2 ~ 100
    assert r.hit_ids[0, 0, 0] == 0 and r.counts["shadow"] == 1
    assert r.rgb[0, 0] == pytest.approx(lit, rel=1e-6)
    # gap 2.5e-4: the plane is 1.5e-4 >= EPS_T beyond the offset origin -> occluded, ambient only
    r2 = oracle_lib.render(_offset_scene(2.5e-4))
    assert r2.rgb[0].tolist() == [amb] * 3


# ---- ambient rule (R#4) -----------------------------------------------------------------------------
@pytest.mark.parametrize("D", [0, 3, 5])
def test_ambient_only_at_diffuse_hits(oracle_lib, D):
    # W4's SPECULAR mirrors with a non-zero ambient: delta materials get no ambient term, so the
    # closed form sum 0.5^i is unchanged
    b = scenegen.builder()
    m = b.material(SPECULAR, (0.5, 0.5, 0.5), emission=(1, 1, 1))
    b.plane((0, 0, 1), 0.0, m)
    b.plane((0, 0, 1), 10.0, m)
    sc = b.build("W4amb", eye=(0, 0, 5), look_at=(0, 0, 6), up=(0, 1, 0), vfov=30, width=1, height=1,
                 max_depth=D, spp=1, ambient=(0.5, 0.5, 0.5))
    assert oracle_lib.render(sc).rgb[0, 0] == 2 - 0.5 ** D
    # DIFFUSE kr-mirrors with ambient A: every hit adds T rho A as well -> sum kr^i (1 + rho A)
    r = oracle_lib.render(_diffuse_mirrors(D, rho=(0.5, 0.5, 0.5), ambient=(0.5, 0.5, 0.5)))
    assert r.rgb[0, 0] == pytest.approx(sum(0.25 ** i for i in range(D + 1)) * 1.25, rel=1e-15)


# ---- RNG composition ------------------------------------------------------------------
def _splitmix_first(state):
    """First output of Vigna's splitmix64 seeded with `state` (scenegen's independent copy)."""
    return SplitMix64(state).next_u64()


def test_rng_matches_independent_splitmix_stream(oracle_lib):
    # seed 0: the first mix is output number pixel + 1 of splitmix64 seeded with 0; the second mix
    # of (that ^ word * G) is the first output of splitmix64 seeded with (that ^ word * G) - G
    g = SplitMix64(0)
    outs = [g.next_u64() for _ in range(40)]
    for pix in range(40):
        for s, depth in ((0, 0), (0, 3), (5, 0), (7, 2)):
            word = ((s << 32) + depth) * _G & _MASK
            x = _splitmix_first(((outs[pix] ^ word) - _G) & _MASK)
            assert oracle_lib.rng(0, pix, s, depth) == (x >> 40) * 2.0 ** -24, (pix, s, depth)
    # a non-zero seed enters by XOR with (pixel + 1) G before the first mix
    seed = 0x1234_5678_9ABC_DEF0
    for pix in (0, 1, 99):
        h = _splitmix_first(((seed ^ ((pix + 1) * _G & _MASK)) - _G) & _MASK)
        x = _splitmix_first(((h ^ ((3 << 32) + 1) * _G & _MASK) - _G) & _MASK)
        assert oracle_lib.rng(seed, pix, 3, 1) == (x >> 40) * 2.0 ** -24


# ---- test counts in index order (§8(c).1 step 11; Alg. 1 `break`) ------------------------------------
@pytest.mark.parametrize("order,hit,sph,pl", [
    ("S0 S1 P", 0, 4, 1),   # closest: 2 spheres + 1 plane; shadow: S0, S1 (occluder) -> stop
    ("P S0 S1", 1, 4, 2),   # shadow: P, S0, S1 (occluder)
    ("S0 P S1", 0, 4, 2),   # shadow: S0, P, S1 (occluder)
    ("S1 S0 P", 1, 3, 1),   # shadow: S1 occludes first -> 1 sphere test
])
def test_counts_follow_index_order(oracle_lib, order, hit, sph, pl):
    # W2's occluded configuration with a far plane y = -5 (parallel to the camera ray, below every
    # shadow ray) inserted at different indices: primary 1, shadow 1, counted by hand
    b = scenegen.builder()
    mt = b.material(DIFFUSE, (0.5, 0.5, 0.5))
    for tok in order.split():
        if tok == "S0":
            b.sphere((0, 0, 5), 1.0, mt)
        elif tok == "S1":
            b.sphere((0, 1.5, 2.5), 0.5, mt)
        else:
            b.plane((0, 1, 0), -5.0, mt)
    b.light((0, 3, 1), (36 * math.pi,) * 3)
    sc = b.build("counts", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=1, height=1,
                 max_depth=0, spp=1, ambient=(0.1, 0.1, 0.1), keep_order=True)
    r = oracle_lib.render(sc)
    assert r.hit_ids[0, 0, 0] == hit
    assert r.rgb[0, 0] == 0.5 * _f32(0.1)
    assert (r.counts["primary"], r.counts["shadow"], r.counts["secondary"]) == (1, 1, 0)
    assert (r.counts["sphere_tests"], r.counts["plane_tests"]) == (sph, pl)


# ---- ties, the EPS_T threshold, the shadow interval's far end -----------------------------------------
@pytest.mark.parametrize("order,want", [("S0 S1", 0), ("S1 S0", 0), ("P S", 0), ("S P", 0)])
def test_ties_go_to_the_lowest_index(oracle_lib, order, want):
    # "two identical coincident spheres -> Hit carries the lower object_index"; the
    # same rule between a sphere and a plane tangent to it at the hit point (both exactly t = 4:
    # sphere c = (0,0,5), r = 1 on the axis; plane z = 4). Each primitive emits a different colour.
    b = scenegen.builder()
    red = b.material(DIFFUSE, (0, 0, 0), emission=(1, 0, 0))
    green = b.material(DIFFUSE, (0, 0, 0), emission=(0, 1, 0))
    for k, tok in enumerate(order.split()):
        m = red if k == 0 else green
        if tok.startswith("S"):
            b.sphere((0, 0, 5), 1.0, m)
        else:
            b.plane((0, 0, 1), 4.0, m)
    sc = b.build("tie", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                 max_depth=0, spp=1, keep_order=True)
    r = oracle_lib.render(sc)
    assert r.hit_ids[0, 0, 0] == want
    assert r.rgb[0].tolist() == [1.0, 0.0, 0.0]


def test_eps_t_threshold_is_inclusive(oracle_lib):
    # S:63 "smallest root t with t >= EPS_T" (EPS_T = 1e-4): a plane root of exactly 1e-4
    # (dp / den = 1e-4 / 1) is accepted, the next double below is rejected
    o, d, n = (0.0, 0.0, 0.0), (0.0, 0.0, 1.0), (0.0, 0.0, 1.0)
    assert oracle_lib.intersect_plane(o, d, n, 1e-4) == 1e-4
    assert oracle_lib.intersect_plane(o, d, n, float(np.nextafter(1e-4, 0.0))) is None
    # sphere: origin at the centre of a sphere of radius r: the exit root is r (S:69 example form)
    t = oracle_lib.intersect_sphere((0.0, 0.0, 0.0), d, (0.0, 0.0, 0.0), 2e-4)
    assert t == pytest.approx(2e-4, rel=1e-15)
    assert oracle_lib.intersect_sphere((0.0, 0.0, 0.0), d, (0.0, 0.0, 0.0), 0.5e-4) is None


def test_occluder_beyond_the_light_does_not_shadow(oracle_lib):
    # occluded iff a root lies in [EPS_T, |P_l - o_s|): a sphere on the shadow ray's line
    # just beyond the light (roots ~0.3-0.7 past t_max) leaves the pixel bit-identical
    def scene(extra):
        b = scenegen.builder()
        m = b.material(DIFFUSE, (0.5, 0.5, 0.5))
        b.sphere((0, 0, 5), 1.0, m)
        if extra:
            # p ~ (0, 0, 4), light (0, 2, 2): direction (0, 1, -1)/sqrt 2, t_max ~ 2.83; centre at t ~ 3.3
            s = 3.3 / math.sqrt(2)
            b.sphere((0, s, 4 - s), 0.2, m)
        b.light((0, 2, 2), (50.0,) * 3)
        return b.build("beyond", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                       max_depth=0, spp=1, ambient=(0.1, 0.1, 0.1))
    a, b_ = oracle_lib.render(scene(False)), oracle_lib.render(scene(True))
    assert a.rgb[0, 0] > 0.5 and (a.rgb == b_.rgb).all()
    # moved to t ~ 2.3 (before the light) it occludes: ambient only
    bb = scenegen.builder()
    m = bb.material(DIFFUSE, (0.5, 0.5, 0.5))
    bb.sphere((0, 0, 5), 1.0, m)
    s = 2.3 / math.sqrt(2)
    bb.sphere((0, s, 4 - s), 0.2, m)
    bb.light((0, 2, 2), (50.0,) * 3)
    sc = bb.build("before", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                  max_depth=0, spp=1, ambient=(0.1, 0.1, 0.1))
    assert oracle_lib.render(sc).rgb[0].tolist() == [0.5 * _f32(0.1)] * 3


@pytest.mark.parametrize("order,sph,pl", [("S0 S1 Pocc", 4, 1), ("S1 S0 Pocc", 3, 1), ("Pocc S0 S1", 2, 2),
                                          ("S0 Pocc S1", 3, 2)])
def test_counts_with_an_occluding_plane(oracle_lib, order, sph, pl):
    # as above with a plane y = 2 that also blocks the shadow ray (between the shading point and the
    # light, parallel to the camera ray): the first occluder in index order stops the count
    b = scenegen.builder()
    mt = b.material(DIFFUSE, (0.5, 0.5, 0.5))
    for tok in order.split():
        if tok == "S0":
            b.sphere((0, 0, 5), 1.0, mt)
        elif tok == "S1":
            b.sphere((0, 1.5, 2.5), 0.5, mt)
        else:
            b.plane((0, 1, 0), 2.0, mt)
    b.light((0, 3, 1), (36 * math.pi,) * 3)
    sc = b.build("counts2", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=1, height=1,
                 max_depth=0, spp=1, ambient=(0.1, 0.1, 0.1), keep_order=True)
    r = oracle_lib.render(sc)
    assert r.rgb[0, 0] == 0.5 * _f32(0.1)
    assert (r.counts["sphere_tests"], r.counts["plane_tests"]) == (sph, pl)
