"""Pins for the oracle's shading, bounce loop and whole-frame invariants (CPU, no GPU).

Worked examples W1-W6 are hand-derived closed forms (tests/golden/worked_examples.json,
SURVEY.md §8(c).3); the rest are invariants that any correct implementation satisfies.
"""
import json
import math
import os

import numpy as np
import pytest

import scenegen
from scenegen import DIFFUSE, REFRACTIVE, SPECULAR

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _w1_scene(light=(0, 0, 0), I=16 * math.pi, ks=0.0, shin=1.0, occluder=False, ambient=0.1):
    b = scenegen.builder()
    m = b.material(DIFFUSE, (0.5, 0.5, 0.5), ks=ks, shininess=shin)
    b.sphere((0, 0, 5), 1.0, m)
    if occluder:
        b.sphere((0, 1.5, 2.5), 0.5, b.material(DIFFUSE, (0.5, 0.5, 0.5)))
    b.light(light, (I, I, I))
    return b.build("W1", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=1, height=1,
                   max_depth=0, spp=1, ambient=(ambient,) * 3)


def _f32(x):
    return float(np.float32(x))


def test_w1_lambert(oracle_lib):
    r = oracle_lib.render(_w1_scene())
    # I is stored as float32(16 pi); the closed form uses the same stored value
    want = 0.5 / math.pi * _f32(16 * math.pi) / 16 + 0.5 * _f32(0.1)
    assert r.rgb[0] == pytest.approx([want] * 3, rel=1e-14)
    assert want == pytest.approx(GOLDEN["W1_lambert"]["L"], rel=1e-6)
    assert oracle_lib.tonemap8(r.rgb[0, 0]) == GOLDEN["W1_lambert"]["tonemap8"]
    assert r.hit_ids[0, 0, 0] == 0 and r.counts["primary"] == 1 and r.counts["shadow"] == 1


def test_w2_shadow_and_occluder(oracle_lib):
    I = _f32(36 * math.pi)
    r = oracle_lib.render(_w1_scene(light=(0, 3, 1), I=36 * math.pi))
    want = 0.5 / math.pi * I / 18 / math.sqrt(2) + 0.5 * _f32(0.1)
    assert r.rgb[0, 0] == pytest.approx(want, rel=1e-12)
    assert want == pytest.approx(GOLDEN["W2_shadow"]["L_lit"], rel=1e-6)
    r2 = oracle_lib.render(_w1_scene(light=(0, 3, 1), I=36 * math.pi, occluder=True))
    # ambient only: "shadowed points get ambient only" (BASELINE.json north_star)
    assert r2.rgb[0, 0] == 0.5 * _f32(0.1)
    assert oracle_lib.tonemap8(r2.rgb[0, 0]) == GOLDEN["W2_shadow"]["tonemap8_shadowed"]
    assert r2.counts["primary"] == 1 and r2.counts["shadow"] == 1
    assert r2.hit_ids[0, 0, 0] == 0  # the camera ray misses the occluder


def test_w6_phong(oracle_lib):
    r = oracle_lib.render(_w1_scene(ks=0.5, shin=10))
    want = 0.5 / math.pi * _f32(16 * math.pi) / 16 + 0.5 * 12 / (2 * math.pi) * _f32(16 * math.pi) / 16 + 0.5 * _f32(0.1)
    assert r.rgb[0, 0] == pytest.approx(want, rel=1e-12)
    assert want == pytest.approx(GOLDEN["W6_phong"]["L"], rel=1e-6)


def test_light_behind_surface_casts_no_shadow_ray(oracle_lib):
    # emitter behind the surface contributes 0 and (our reading) casts no shadow ray
    r = oracle_lib.render(_w1_scene(light=(0, 0, 10), I=100.0))
    assert r.rgb[0, 0] == 0.5 * _f32(0.1)
    assert r.counts["shadow"] == 0


def _mirror_scene(D):
    b = scenegen.builder()
    m = b.material(SPECULAR, (0.5, 0.5, 0.5), emission=(1, 1, 1))
    b.plane((0, 0, 1), 0.0, m)
    b.plane((0, 0, 1), 10.0, m)
    return b.build("W4", eye=(0, 0, 5), look_at=(0, 0, 6), up=(0, 1, 0), vfov=30, width=1, height=1,
                   max_depth=D, spp=1)


@pytest.mark.parametrize("D", [0, 1, 2, 3, 5, 8])
def test_w4_parallel_mirrors_closed_form(oracle_lib, D):
    # sum_{i<=D} k^i L_e, exact in binary
    r = oracle_lib.render(_mirror_scene(D))
    assert r.rgb[0, 0] == GOLDEN["W4_mirrors"]["L_by_depth"].get(str(D), 2 - 0.5 ** D)
    assert r.rgb[0, 0] == 2 - 0.5 ** D
    assert r.bounces[0, 0] == D and r.counts["secondary"] == D
    ids = r.hit_ids[0, 0]
    assert list(ids) == [1 if i % 2 == 0 else 0 for i in range(D + 1)]


def test_w5_refraction_head_on(oracle_lib):
    b = scenegen.builder()
    b.sphere((0, 0, 5), 1.0, b.material(REFRACTIVE, (1, 1, 1), ior=1.5))
    bg = (0.25, 0.5, 0.75)
    assert oracle_lib.schlick(1.5, 1.0) == pytest.approx(GOLDEN["W5_refraction"]["R0"], rel=1e-12)
    assert oracle_lib.schlick(1.5, 0.0) == pytest.approx(1.0, abs=1e-15)
    found = 0
    for seed in range(40):
        sc = b.build("W5", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                     max_depth=2, spp=1, background=bg, seed=seed)
        u0, u1 = oracle_lib.rng(seed, 0, 0, 0), oracle_lib.rng(seed, 0, 0, 1)
        r = oracle_lib.render(sc)
        if u0 >= 0.04 and u1 >= 0.04:
            # refract in (direction unchanged), refract out, miss -> background with T = 1
            assert r.rgb[0].tolist() == [_f32(x) for x in bg]
            assert list(r.hit_ids[0, 0]) == [0, 0, -1] and r.bounces[0, 0] == 2
            found += 1
        elif u0 < 0.04:
            # mirror reflection straight back: miss -> background, one bounce
            assert r.rgb[0].tolist() == [_f32(x) for x in bg]
            assert list(r.hit_ids[0, 0]) == [0, -1, -2]
        else:
            # refract in, internal reflection, then max_depth reached inside: no emission -> 0
            assert r.rgb[0].tolist() == [0.0, 0.0, 0.0]
    assert found > 30


def test_miss_returns_background_bit_exact(oracle_lib):
    b = scenegen.builder()
    b.sphere((0, 0, -5), 1.0, b.material(DIFFUSE, (1, 1, 1)))  # behind the camera
    b.light((0, 5, 0), (10, 10, 10))
    bg = (0.1, 0.2, 0.3)
    sc = b.build("miss", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=8, height=6,
                 max_depth=4, spp=4, background=bg)
    r = oracle_lib.render(sc)
    assert (r.rgb == np.array([_f32(x) for x in bg])[None, :]).all()
    assert r.counts["secondary"] == 0 and r.counts["shadow"] == 0
    assert r.counts["primary"] == 8 * 6 * 4
    assert (r.hit_ids[..., 0] == -1).all() and (r.hit_ids[..., 1:] == -2).all()


def _hemisphere_quadrature(fn, n=64):
    """Gauss-Legendre n x n over (cos theta in [0,1], phi in [0, 2 pi]) of fn(w) * cos(theta)."""
    x, w = np.polynomial.legendre.leggauss(n)
    mu = 0.5 * (x + 1)
    wmu = 0.5 * w
    phi = np.pi * (x + 1)
    wphi = np.pi * w
    tot = 0.0
    for i in range(n):
        st = math.sqrt(1 - mu[i] ** 2)
        for j in range(n):
            wi = (st * math.cos(phi[j]), st * math.sin(phi[j]), mu[i])
            tot += wmu[i] * wphi[j] * fn(wi) * mu[i]
    return tot


def test_brdf_values_and_normalisation(oracle_lib):
    n = (0, 0, 1)
    # S:141-144
    f = oracle_lib.brdf(0, (0.5, 0.5, 0.5), 0.0, 1.0, (0, 0, 1), (0, 0, 1), n)
    np.testing.assert_allclose(f, [0.5 / math.pi] * 3, rtol=1e-15)
    assert f[0] == pytest.approx(0.15915, abs=1e-5)
    assert (oracle_lib.brdf(0, (0, 0, 0), 0.0, 1.0, (0, 0, 1), (0, 0, 1), n) == 0).all()
    assert (oracle_lib.brdf(1, (1, 1, 1), 0.5, 8.0, (0, 0, 1), (0, 0, 1), n) == 0).all()
    # S:173 Lambert: integral of f cos = albedo within 1e-3
    val = _hemisphere_quadrature(lambda wi: oracle_lib.brdf(0, (0.7, 0.7, 0.7), 0.0, 1.0, wi, (0, 0, 1), n)[0], 32)
    assert val == pytest.approx(0.7, abs=1e-3)
    # normalised Phong: with w_o = n the lobe integrates to exactly ks (pins (s+2)/(2 pi), R#3)
    for s in (1.0, 10.0, 32.0):
        val = _hemisphere_quadrature(lambda wi: oracle_lib.brdf(0, (0, 0, 0), 1.0, s, wi, (0, 0, 1), n)[0], 48)
        assert val == pytest.approx(1.0, abs=1e-3), s
    # Helmholtz reciprocity for the Lambert + Phong lobe
    rng = np.random.default_rng(5)
    for _ in range(50):
        a, b_ = rng.normal(size=3), rng.normal(size=3)
        a[2], b_[2] = abs(a[2]), abs(b_[2])
        a /= np.linalg.norm(a)
        b_ /= np.linalg.norm(b_)
        f1 = oracle_lib.brdf(0, (0.3, 0.4, 0.5), 0.4, 12.0, a, b_, n)
        f2 = oracle_lib.brdf(0, (0.3, 0.4, 0.5), 0.4, 12.0, b_, a, n)
        np.testing.assert_allclose(f1, f2, rtol=1e-12)


def _scaled(sc, k):
    import dataclasses
    return dataclasses.replace(sc, light_intensity=sc.light_intensity * np.float32(k),
                               mat_emission=sc.mat_emission * np.float32(k))


def test_linearity_in_sources(oracle_lib):
    # S:175 monotone/linear in L_e and I; with ambient = background = 0 and k = 4 (a power of two)
    import dataclasses
    for seed in range(3):
        sc = scenegen.random_tiny(seed, width=10, height=8)
        sc = dataclasses.replace(sc, ambient=np.zeros(3, np.float32), background=np.zeros(3, np.float32))
        sc.mat_emission[:] = np.float32(0.25)
        r1 = oracle_lib.render(sc)
        r4 = oracle_lib.render(_scaled(sc, 4))
        assert (r4.rgb == 4 * r1.rgb).all()


def test_depth_monotonicity(oracle_lib):
    # adding a bounce only adds non-negative terms (same RNG draws per depth index)
    for seed in range(4):
        sc = scenegen.random_tiny(seed, width=10, height=8)
        prev = None
        for D in range(0, 5):
            r = oracle_lib.render(sc.with_frame(max_depth=D))
            assert np.isfinite(r.rgb).all() and (r.rgb >= 0).all()
            if prev is not None:
                assert (r.rgb >= prev).all()
            prev = r.rgb


def test_partition_invariance(oracle_lib):
    # the image is a pure function of the scene, not of the pixel order/partition
    sc = scenegen.random_tiny(11, width=13, height=7, spp=4)
    full = oracle_lib.render(sc)
    perm = np.random.default_rng(0).permutation(13 * 7)
    part = oracle_lib.render(sc, pixels=perm)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    assert (part.rgb[inv] == full.rgb).all()
    assert (part.hit_ids[inv] == full.hit_ids).all()
    assert full.counts["primary"] == 13 * 7 * 4


def test_ray_counts_2x2(oracle_lib):
    # a 2x2 image traces exactly 4 camera rays per pass
    sc = scenegen.random_tiny(2, width=2, height=2)
    assert oracle_lib.render(sc).counts["primary"] == 4


def _bruteforce_first_hit(sc, o, d):
    """Independent nearest-hit search: bisection on each primitive's implicit function along the
    ray (Eq. 9 for spheres, n.x - d for planes), then the smallest t (ties -> lowest index)."""
    best_t, best_k = math.inf, -1
    for k in range(sc.n_prims):
        p = sc.prim_p[k].astype(np.float64)
        if sc.prim_type[k] == scenegen.PLANE:
            n = p[:3] / np.linalg.norm(p[:3])
            dp = p[3] / np.linalg.norm(p[:3])
            f = lambda t: float(n @ (o + t * d) - dp)
        else:
            c, r = p[:3], p[3]
            f = lambda t: float((o + t * d - c) @ (o + t * d - c) - r * r)
        ts = np.linspace(1e-4, 200, 40001)
        vals = np.array([f(t) for t in ts[:1]])
        P = o[None, :] + ts[:, None] * d[None, :]
        if sc.prim_type[k] == scenegen.PLANE:
            vals = P @ n - dp
        else:
            Q = P - c[None, :]
            vals = (Q * Q).sum(1) - r * r
        sgn = np.sign(vals)
        ch = np.nonzero(sgn[1:] != sgn[0])[0]
        if len(ch) == 0:
            continue
        j = ch[0]
        lo, hi = ts[j], ts[j + 1]
        s0 = np.sign(f(lo))
        for _ in range(100):
            mid = 0.5 * (lo + hi)
            if np.sign(f(mid)) == s0:
                lo = mid
            else:
                hi = mid
        t = 0.5 * (lo + hi)
        if t < best_t:
            best_t, best_k = t, k
    return best_k, best_t


def test_primary_hits_match_bruteforce(oracle_lib):
    checked = 0
    for seed in range(3):
        sc = scenegen.random_tiny(seed, width=12, height=9)
        r = oracle_lib.render(sc)
        for pix in range(sc.width * sc.height):
            if r.margin[pix, 0] < 1e-3:
                continue  # near-tangent / near-tie samples are grid-ambiguous for the brute force
            px, py = pix % sc.width, pix // sc.width
            o, d = oracle_lib.camera_ray(sc, sc.width, sc.height, px, py)
            k, _ = _bruteforce_first_hit(sc, o, d)
            assert r.hit_ids[pix, 0, 0] == k, (seed, pix)
            checked += 1
    assert checked > 150


def test_margins_flag_tangent_and_clear_rays(oracle_lib):
    # a camera ray that grazes a sphere silhouette exactly has margin ~0; a clear ray is large
    b = scenegen.builder()
    b.sphere((0, 1, 5), 1.0, b.material(DIFFUSE, (0.5, 0.5, 0.5)))
    sc = b.build("tan", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                 max_depth=0, spp=1)
    assert oracle_lib.render(sc).margin[0, 0] < 1e-12
    b = scenegen.builder()
    b.sphere((0, 0, 5), 1.0, b.material(DIFFUSE, (0.5, 0.5, 0.5)))
    sc = b.build("clear", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                 max_depth=0, spp=1)
    assert oracle_lib.render(sc).margin[0, 0] > 1e-3


def test_perturbation_replicas_are_close(oracle_lib):
    # the classification replicas (Monte Carlo arithmetic) stay within ~1e-5 on a smooth scene
    sc = scenegen.get("C1")
    r0 = oracle_lib.render(sc)
    r1 = oracle_lib.render(sc, perturb=2.0 ** -22, perturb_seed=1)
    ok = (r0.margin.min(1) > 1e-3)
    rel = np.abs(r1.rgb - r0.rgb) / (np.abs(r0.rgb) + 1e-6)
    assert np.median(rel[ok]) < 1e-5
