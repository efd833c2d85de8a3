"""The oracle's closed-form pin scenes (tests/test_oracle_continuation.py) through the CUDA path.

Each scene isolates one reading (Schlick's exit-side cosine, the DIFFUSE-kr and coloured-glass
weights, the p + EPS_T n shadow origin, the [EPS_T, t_max) interval, ties to the lowest index,
test counts in primitive order). A reading shared wrongly by both sides would pass a plain
GPU-vs-oracle parity test; here the GPU must also reproduce the hand-derived values, and hit ids,
bounce counts and every statistic must equal the oracle's exactly (both decide in FP64).
"""
import math

import numpy as np
import pytest

import scenegen
from scenegen import DIFFUSE, REFRACTIVE
from tests import parity
from tests.gpu_helpers import gpu_render
from tests.test_oracle_continuation import _diffuse_mirrors, _exit_scene, _offset_scene

pytestmark = pytest.mark.gpu
VARIANTS = ["wavefront", "megakernel"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    yield


def _f32(x):
    return float(np.float32(x))


def _same(oracle_lib, sc, variant, rel=2e-6):
    g = gpu_render(sc, variant=variant)
    ref = oracle_lib.render(sc)
    assert (g["ids"] == ref.hit_ids).all(), (g["ids"], ref.hit_ids)
    assert (g["bounces"] == ref.bounces).all()
    ok, msg = parity.counts_equal(g["stats"], ref.counts)
    assert ok, msg
    np.testing.assert_allclose(g["rgb"], ref.rgb, rtol=rel, atol=1e-7)
    return g


@pytest.mark.parametrize("variant", VARIANTS)
def test_exit_side_schlick_cosine(oracle_lib, variant):
    cx = _f32(0.6)
    F_exit = 0.04 + 0.96 * (1 - math.sqrt(1 - 2.25 * cx * cx)) ** 5
    F_inc = 0.04 + 0.96 * (1 - math.sqrt(1 - cx * cx)) ** 5
    band = 0
    for seed in range(400):
        u = oracle_lib.rng(seed, 0, 0, 0)
        if abs(u - F_exit) < 1e-9:
            continue
        g = _same(oracle_lib, _exit_scene(seed), variant)
        want = [0.0, 0.0, 0.0] if u < F_exit else [_f32(x) for x in (0.25, 0.5, 0.75)]
        assert g["rgb"][0].tolist() == want, seed
        band += F_inc <= u < F_exit
    assert band >= 5


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("D", [0, 2, 5])
def test_diffuse_kr_weight(oracle_lib, variant, D):
    g = _same(oracle_lib, _diffuse_mirrors(D), variant)
    assert g["rgb"][0].tolist() == [sum(0.25 ** i for i in range(D + 1))] * 3  # exact in float32


@pytest.mark.parametrize("variant", VARIANTS)
def test_coloured_glass(oracle_lib, variant):
    rho, bg = (0.5, 0.25, 1.0), (0.25, 0.5, 0.75)
    b = scenegen.builder()
    b.sphere((0, 0, 5), 1.0, b.material(REFRACTIVE, rho, ior=1.5))
    seen = set()
    for seed in range(60):
        sc = b.build("glass", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=30, width=1, height=1,
                     max_depth=2, spp=1, background=bg, seed=seed)
        g = _same(oracle_lib, sc, variant)
        u0, u1 = oracle_lib.rng(seed, 0, 0, 0), oracle_lib.rng(seed, 0, 0, 1)
        if u0 >= 0.04 and u1 >= 0.04:
            assert g["rgb"][0].tolist() == [bg[c] * rho[c] ** 2 for c in range(3)]
            seen.add("tt")
        elif u0 < 0.04:
            assert g["rgb"][0].tolist() == [bg[c] * rho[c] for c in range(3)]
            seen.add("r")
    assert "tt" in seen


@pytest.mark.parametrize("variant", VARIANTS)
def test_shadow_origin_offset(oracle_lib, variant):
    amb = 0.5 * _f32(0.1)
    g = _same(oracle_lib, _offset_scene(1.5e-4), variant)
    assert g["rgb"][0, 0] > 0.9 and g["stats"]["shadow"] == 1
    g = _same(oracle_lib, _offset_scene(2.5e-4), variant)
    assert g["rgb"][0].tolist() == [np.float32(amb)] * 3


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("order", ["S0 S1", "S1 S0", "P S", "S P"])
def test_ties_lowest_index(oracle_lib, variant, order):
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
    g = _same(oracle_lib, sc, variant)
    assert g["ids"][0, 0, 0] == 0 and g["rgb"][0].tolist() == [1.0, 0.0, 0.0]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("order,sph,pl", [("S0 S1 P", 4, 1), ("P S0 S1", 4, 2), ("S0 P S1", 4, 2),
                                          ("S1 S0 P", 3, 1), ("S0 S1 Pocc", 4, 1), ("S1 S0 Pocc", 3, 1),
                                          ("Pocc S0 S1", 2, 2), ("S0 Pocc S1", 3, 2)])
def test_counts_in_primitive_order(oracle_lib, variant, order, sph, pl):
    # W2's occluded pixel; "Pocc" is a plane that also occludes the shadow ray (y = 2, above the
    # shading point, below the light, parallel to the camera ray): with spheres listed before it the
    # first occluder in index order is still a sphere, which the GPU finds after testing planes first
    b = scenegen.builder()
    mt = b.material(DIFFUSE, (0.5, 0.5, 0.5))
    for tok in order.split():
        if tok == "S0":
            b.sphere((0, 0, 5), 1.0, mt)
        elif tok == "S1":
            b.sphere((0, 1.5, 2.5), 0.5, mt)
        elif tok == "P":
            b.plane((0, 1, 0), -5.0, mt)
        else:
            b.plane((0, 1, 0), 2.0, mt)
    b.light((0, 3, 1), (36 * math.pi,) * 3)
    sc = b.build("counts", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=1, height=1,
                 max_depth=0, spp=1, ambient=(0.1, 0.1, 0.1), keep_order=True)
    g = _same(oracle_lib, sc, variant)
    assert (g["stats"]["sphere_tests"], g["stats"]["plane_tests"]) == (sph, pl)
