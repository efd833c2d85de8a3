"""Pins of the NEXT-1 / NEXT-2 oracle extensions: spherical area lights sampled
one point per emitter (Eq. 8 as a one-sample estimator), the global integrator's
cosine-weighted diffuse bounce and progressive passes.

Every pin is fixed by mathematics outside the oracle: closed forms (sphere irradiance, the
analytic cosine-lobe moments, geometric series of a furnace), an independent numerical
quadrature, exact special cases, or invariants of the definitions (resume, stream 0 = the hot
path's RNG). A dropped cos term, a wrong pdf, a wrong sign of the bounce or an emitter that
shadows its own sample fails one of them."""
import math

import numpy as np
import pytest

import scenegen
from scenegen import DIFFUSE, SPECULAR

SQ = math.sqrt


# ---- sample_light_point ---------------------------------------------------------
def test_sample_sphere_spec_examples(oracle_lib):
    x, nl, pdf = oracle_lib.sample_sphere((0, 0, 0), 1.0, 0.0, 0.0)
    assert np.allclose(x, (0, 0, 1), atol=0) and np.allclose(nl, (0, 0, 1), atol=0)
    assert pdf == pytest.approx(1 / (4 * math.pi), rel=1e-15)
    _, _, pdf2 = oracle_lib.sample_sphere((0, 0, 0), 2.0, 0.3, 0.7)
    assert pdf2 == pytest.approx(1 / (16 * math.pi), rel=1e-15)
    # u1 = 1/2, u2 = 1/4: equator at phi = pi/2
    x, nl, _ = oracle_lib.sample_sphere((1, 2, 3), 0.5, 0.5, 0.25)
    assert np.allclose(x, (1, 2.5, 3), atol=1e-15)


def test_sample_sphere_uniform_on_the_surface(oracle_lib):
    po = oracle_lib
    c, r = np.array([0.3, -1.0, 2.0]), 1.7
    n = 100_000
    xs = np.empty((n, 3))
    for i in range(n):
        u1 = po.rng_stream(11, i, 0, 0, 5)
        u2 = po.rng_stream(11, i, 0, 0, 6)
        x, nl, _ = po.sample_sphere(c, r, u1, u2)
        xs[i] = x
    rad = np.linalg.norm(xs - c, axis=1)
    assert np.abs(rad - r).max() < 1e-12                                   # on the sphere
    assert np.abs(xs.mean(0) - c).max() < 0.02 * r                          # S:150 symmetry
    # Archimedes: z is uniform on [-r, r] for a uniform point on the sphere
    z = (xs[:, 2] - c[2]) / r
    for lo, hi in [(-1, -0.5), (-0.5, 0), (0, 0.5), (0.5, 1)]:
        assert abs(((z >= lo) & (z < hi)).mean() - 0.25) < 0.006


# ---- orthonormal basis + cosine-weighted direction -----------------------------
@pytest.mark.parametrize("n", [(0, 0, 1), (0, 0, -1), (1, 0, 0), (0, 1, 0), (0.6, 0, -0.8),
                               (0.48, 0.6, 0.64), (-0.36, 0.48, -0.8), (1e-9, 0, -1.0)])
def test_onb_is_orthonormal_and_right_handed(oracle_lib, n):
    n = np.array(n, float)
    n /= np.linalg.norm(n)
    t1, t2 = oracle_lib.onb(n)
    M = np.stack([t1, t2, n])
    assert np.allclose(M @ M.T, np.eye(3), atol=1e-14)
    assert np.allclose(np.cross(t1, t2), n, atol=1e-14)


def test_cosine_direction_closed_form_point(oracle_lib):
    # n = +z: t1 = x, t2 = y exactly; u1 = u2 = 1/2 -> (sqrt(1/2) cos pi, sqrt(1/2) sin pi, sqrt(1/2))
    d = oracle_lib.cosine_direction((0, 0, 1), 0.5, 0.5)
    assert np.allclose(d, (-SQ(0.5), 0.0, SQ(0.5)), atol=1e-15)


def test_cosine_direction_moments(oracle_lib):
    po = oracle_lib
    n = np.array([0.48, 0.6, 0.64])
    t1, t2 = po.onb(n)
    N = 100_000
    c = np.empty(N)
    a1 = np.empty(N)
    for i in range(N):
        d = po.cosine_direction(n, po.rng_stream(5, i, 0, 0, 3), po.rng_stream(5, i, 0, 0, 4))
        assert abs(np.linalg.norm(d) - 1) < 1e-13
        c[i] = d @ n
        a1[i] = d @ t1
    assert c.min() >= 0.0                                       # hemisphere
    assert abs(c.mean() - 2 / 3) < 0.01                          # E[cos] = 2/3
    assert abs((c * c).mean() - 0.5) < 0.01                      # E[cos^2] = 1/2 for pdf cos/pi
    assert abs(a1.mean()) < 0.01                                 # azimuthal symmetry


# ---- RNG streams (R#42) ---------------------------------------------------------------------
def test_rng_stream0_is_the_hot_path_rng(oracle_lib):
    po = oracle_lib
    for (seed, pix, s, d) in [(0, 0, 0, 0), (7, 123456, 3, 5), (2**63 + 5, 2**40, 15, 255)]:
        assert po.rng_stream(seed, pix, s, d, 0) == po.rng(seed, pix, s, d)


def test_rng_streams_uniform_and_decorrelated(oracle_lib):
    po = oracle_lib
    u = np.array([po.rng_stream(3, i, 7, 2, 9) for i in range(200_000)])
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.002
    a = [po.rng_stream(3, 10, s, 0, 1) for s in range(100)]
    b = [po.rng_stream(3, 11, s, 0, 1) for s in range(100)]
    c = [po.rng_stream(3, 10, s, 0, 2) for s in range(100)]
    assert sum(x != y for x, y in zip(a, b)) >= 95 and sum(x != y for x, y in zip(a, c)) >= 95


# ---- direct lighting from a spherical emitter (Eq. 8 one-sample estimator) ------------------
def _emitter_over_plane(center, R, Le, rho, eye, look):
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (rho, rho, rho)))
    b.sphere(center, R, b.material(DIFFUSE, (0, 0, 0), emission=(Le, Le, Le)))
    return b.build("emitter", eye=eye, look_at=look, up=(0, 1, 0), vfov=0.5, width=1, height=1,
                   max_depth=0, spp=1)


def _hit_point(po, sc):
    o, d = po.camera_ray(sc, 1, 1, 0, 0, 0, 1)
    t = po.intersect_plane(o, d, (0, 1, 0), 0.0)
    return o + t * d


def test_area_light_estimator_matches_sphere_irradiance_closed_form(oracle_lib):
    """A sphere of uniform radiance Le fully above the tangent plane gives the irradiance
    E = pi Le (R/D)^2 cos(theta) (sin^2 of the half-angle times the cosine): L_o = rho E / pi."""
    po = oracle_lib
    sc = _emitter_over_plane((0.7, 3.0, 0.4), 0.8, 20.0, 0.6, eye=(0, 1.5, -1.5), look=(0, 0, 0))
    N = 20_000
    r = po.render(sc, spp=N, area_lights=1, jitter=0)
    p = _hit_point(po, sc)
    c = np.array([0.7, 3.0, 0.4])
    D = np.linalg.norm(c - p)
    cos_t = (c - p)[1] / D
    expected = 0.6 / math.pi * math.pi * 20.0 * (0.8 / D) ** 2 * cos_t
    s = r.sample_rgb[0, :, 0]
    se = s.std() / math.sqrt(N)
    assert r.hit_ids[0, :, 0].tolist() == [0] * N
    assert abs(s.mean() - expected) < 4 * se + 1e-9, (s.mean(), expected, se)
    assert se < 0.02 * expected  # the estimator is informative at this N
    assert r.counts["shadow"] <= N and r.counts["sphere_tests"] == N  # emitter never tested by its shadow rays


def test_area_light_estimator_matches_quadrature_across_the_horizon(oracle_lib):
    """Emitter partly below the tangent plane (closed form breaks): compare with an independent
    Gauss-Legendre quadrature of Le max(0, cos_s) max(0, cos_l) / d^2 over the sphere."""
    po = oracle_lib
    c, R, Le, rho = np.array([2.0, 0.3, 1.0]), 1.0, 10.0, 0.8
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (rho, rho, rho)))
    b.sphere(tuple(c), R, b.material(DIFFUSE, (0, 0, 0), emission=(Le, Le, Le)))
    sc = b.build("horizon", eye=(-0.5, 1.0, -1.5), look_at=(-0.5, 0, 0), up=(0, 1, 0), vfov=0.5,
                 width=1, height=1, max_depth=0, spp=1)
    p = _hit_point(po, sc)
    # quadrature over (cos theta, phi) of the emitter surface, z-pole parametrisation
    xg, wg = np.polynomial.legendre.leggauss(400)
    ct = xg
    ph = math.pi * (xg + 1)
    CT, PH = np.meshgrid(ct, ph, indexing="ij")
    W = np.outer(wg, wg) * math.pi  # d(cos t) d(phi) = R^2 dA / R^2
    ST = np.sqrt(1 - CT ** 2)
    nl = np.stack([ST * np.cos(PH), ST * np.sin(PH), CT], -1)
    x = c + R * nl
    w = x - p
    d2 = (w * w).sum(-1)
    wi = w / np.sqrt(d2)[..., None]
    cs = np.maximum(0, wi[..., 1])
    cl = np.maximum(0, -(wi * nl).sum(-1))
    E = (Le * cs * cl / d2 * R * R * W).sum()
    # the plane hides nothing here (the emitter is the only other object), so visibility = 1
    expected = rho / math.pi * E
    N = 20_000
    r = po.render(sc, spp=N, area_lights=1)
    s = r.sample_rgb[0, :, 0]
    se = s.std() / math.sqrt(N)
    assert abs(s.mean() - expected) < 4 * se + 1e-9, (s.mean(), expected, se)


def test_emitter_behind_an_occluder_gives_zero(oracle_lib):
    po = oracle_lib
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.8, 0.8, 0.8)))
    b.sphere((0, 2.0, 0), 0.5, b.material(DIFFUSE, (0.5, 0.5, 0.5)))        # blocker
    b.sphere((0, 6.0, 0), 0.3, b.material(DIFFUSE, (0, 0, 0), emission=(50, 50, 50)))
    sc = b.build("blocked", eye=(0, 0.5, -1.0), look_at=(0, 0, 0), up=(0, 1, 0), vfov=0.5,
                 width=1, height=1, max_depth=0, spp=64)
    r = po.render(sc, area_lights=1)
    assert r.hit_ids[0, :, 0].tolist() == [0] * 64
    assert (r.sample_rgb == 0).all()
    # about half of the uniform surface points face away (cos_l <= 0: no shadow ray)
    assert 10 < r.counts["shadow"] < 54


def test_point_lights_unchanged_by_area_light_mode_without_emitters(oracle_lib):
    po = oracle_lib
    sc = scenegen.get("C2").with_frame(width=24, height=18)
    a = po.render(sc)
    b = po.render(sc, area_lights=1)
    assert np.array_equal(a.sample_rgb, b.sample_rgb) and a.counts == b.counts


# ---- global integrator (NEXT-2) ------------------------------------------------------------
def test_global_furnace_is_a_geometric_series(oracle_lib):
    """Camera inside a closed diffuse sphere of albedo rho and emission Le, no area-light
    sampling: every bounce stays inside and collects Le, so each sample is exactly
    Le (1 - rho^(D+1)) / (1 - rho) — independent of the random directions."""
    po = oracle_lib
    rho, Le, D = 0.5, 2.0, 5
    b = scenegen.builder()
    b.sphere((0, 0, 0), 10.0, b.material(DIFFUSE, (rho, rho, rho), emission=(Le, Le, Le)))
    sc = b.build("furnace", eye=(1, 2, 3), look_at=(0, 0, 9), up=(0, 1, 0), vfov=60,
                 width=6, height=5, max_depth=D, spp=3, background=(7, 7, 7))
    r = po.render(sc, integrator=1)
    expected = Le * (1 - rho ** (D + 1)) / (1 - rho)
    assert np.allclose(r.sample_rgb, expected, rtol=1e-12)
    assert (r.bounces == D).all() and (r.hit_ids == 0).all()
    assert r.counts["secondary"] == 6 * 5 * 3 * D


def test_global_diffuse_plane_under_a_constant_sky(oracle_lib):
    """One diffuse plane under background B: every cosine-weighted bounce escapes, so each
    sample is exactly rho * B (f_r cos / pdf = rho), and the bounce is in the upper hemisphere."""
    po = oracle_lib
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.25, 0.5, 0.75)))
    sc = b.build("sky", eye=(0, 2, -3), look_at=(0, 0, 2), up=(0, 1, 0), vfov=40, width=8, height=6,
                 max_depth=3, spp=2, background=(2.0, 4.0, 8.0))
    r = po.render(sc, integrator=1)
    assert np.allclose(r.sample_rgb, np.array([0.5, 2.0, 6.0]), rtol=1e-12)
    assert (r.bounces == 1).all() and (r.hit_ids[:, :, 1] == -1).all()


def test_global_max_depth0_emitter_is_le_exactly(oracle_lib):
    po = oracle_lib
    b = scenegen.builder()
    b.sphere((0, 0, 5), 1.0, b.material(DIFFUSE, (0.3, 0.3, 0.3), emission=(5, 5, 5)))
    sc = b.build("e0", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=5, width=3, height=3,
                 max_depth=0, spp=1)
    r = po.render(sc, integrator=1, area_lights=1)
    assert np.array_equal(r.sample_rgb, np.full((9, 1, 3), 5.0))


def test_global_black_albedo_is_first_hit_emission(oracle_lib):
    po = oracle_lib
    sc = scenegen.random_tiny(4, n_spheres=6, n_emitters=2, n_lights=0, max_depth=4, spp=2)
    sc.mat_albedo[:] = 0.0
    sc.mat_ks[:] = 0.0
    sc.ambient[:] = 0.0
    sc.background[:] = 0.0
    r = po.render(sc, integrator=1, area_lights=1)
    first = r.hit_ids[:, :, 0]
    le = np.where(first[..., None] >= 0, sc.mat_emission[sc.prim_mat[np.maximum(first, 0)]], 0.0)
    # refractive/specular hits with black albedo carry nothing onward either
    assert np.allclose(r.sample_rgb, le, rtol=1e-15, atol=0)


def test_global_equals_whitted_when_diffuse_albedo_is_zero(oracle_lib):
    """S:318 local/global consistency: with zero diffuse albedo and no mirror term the global
    bounce carries T = 0, so the two integrators agree per sample (bounce counts aside)."""
    po = oracle_lib
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0, 0, 0), ks=0.5, shininess=8))
    b.sphere((0, 1, 4), 1.0, b.material(SPECULAR, (0.9, 0.9, 0.9)))
    b.light((2, 5, 1), (40, 40, 40))
    sc = b.build("zero", eye=(0, 1.5, -3), look_at=(0, 1, 4), up=(0, 1, 0), vfov=50, width=10,
                 height=8, max_depth=3, spp=1, background=(0.2, 0.3, 0.4))
    a = po.render(sc)
    g = po.render(sc, integrator=1)
    assert np.allclose(a.sample_rgb, g.sample_rgb, rtol=1e-12, atol=1e-15)


def test_nee_double_count_rule(oracle_lib):
    """With area-light sampling a cosine bounce that lands on an emitter adds nothing (the
    emitter was sampled at the previous vertex); without sampling it adds T Le."""
    po = oracle_lib
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.5, 0.5, 0.5)))
    b.sphere((0, 1.2, 0), 1.0, b.material(DIFFUSE, (0, 0, 0), emission=(3, 3, 3)))
    sc = b.build("nee", eye=(0, 0.3, -4), look_at=(0, 0, 0), up=(0, 1, 0), vfov=2, width=1,
                 height=1, max_depth=1, spp=400, background=(0, 0, 0))
    off = po.render(sc, integrator=1, area_lights=0)
    on = po.render(sc, integrator=1, area_lights=1)
    hit_emitter = off.hit_ids[0, :, 1] == 1
    assert hit_emitter.any() and (~hit_emitter).any()
    # without NEE: the sample is 0.5 * 3 when the bounce hits the emitter, else 0
    assert np.allclose(off.sample_rgb[0, :, 0], np.where(hit_emitter, 1.5, 0.0), rtol=1e-15)
    # with NEE: the same paths, and only the direct term (bounce emission dropped)
    assert np.array_equal(on.hit_ids, off.hit_ids)
    d = po.render(sc.with_frame(max_depth=0), integrator=1, area_lights=1)
    assert np.allclose(on.sample_rgb, d.sample_rgb, rtol=1e-15)


# ---- progressive passes ---------------------------------------------------------
def test_progressive_resume_is_bit_identical(oracle_lib):
    po = oracle_lib
    sc = scenegen.random_tiny(2, n_spheres=5, n_emitters=1, n_lights=1, max_depth=3)
    kw = dict(integrator=1, area_lights=1, jitter=1)
    full = po.render(sc, spp=6, sample_base=0, **kw)
    a = po.render(sc, spp=2, sample_base=0, **kw)
    b = po.render(sc, spp=4, sample_base=2, **kw)
    assert np.array_equal(full.sample_rgb, np.concatenate([a.sample_rgb, b.sample_rgb], 1))
    assert np.array_equal(full.hit_ids, np.concatenate([a.hit_ids, b.hit_ids], 1))
    assert {k: a.counts[k] + b.counts[k] for k in a.counts} == full.counts


def test_random_jitter_stays_inside_the_pixel(oracle_lib):
    """jitter = 1 draws the sub-pixel offset from streams 1/2: the ray passes through the
    pixel's footprint, and different passes use different offsets."""
    po = oracle_lib
    b = scenegen.builder()
    b.plane((0, 0, -1), -10.0, b.material(DIFFUSE, (1, 1, 1), emission=(1, 1, 1)))
    sc = b.build("wall", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=90, width=4,
                 height=4, max_depth=0, spp=8)
    r = po.render(sc, jitter=1, pixels=np.array([5]))  # px = 1, py = 1
    assert (r.hit_ids == 0).all()
    # footprint of pixel (1, 1) on the wall z = 10 (h = tan 45 = 1, aspect 1): x in [-5, 0], y in [0, 5]
    for s in range(8):
        ox = po.rng_stream(0, 5, s, 0, 1)
        oy = po.rng_stream(0, 5, s, 0, 2)
        assert 0 <= ox < 1 and 0 <= oy < 1
        x = (2 * (1 + ox) / 4 - 1) * 10
        y = (1 - 2 * (1 + oy) / 4) * 10
        assert -5 <= x <= 0 and 0 <= y <= 5
    assert len({po.rng_stream(0, 5, s, 0, 1) for s in range(8)}) == 8
