"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Rule: tests/parity.py. Full frames where the oracle finishes in
seconds; at BASELINE.json's full sizes (C3, C4) the GPU renders the whole frame in the bench's
launch configuration and the oracle computes a seeded sample of pixels one by one.
"""
import math

import numpy as np
import pytest

import scenegen
from tests import parity
from tests.gpu_helpers import gpu_render

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    yield


def _check(oracle_lib, sc, pixels=None, label="", variant="wavefront"):
    g = gpu_render(sc, variant=variant)
    ref = oracle_lib.render(sc, pixels=pixels)
    pix = ref.pixels
    cls = parity.classify(oracle_lib, sc, ref, pixels if pixels is not None else None)
    rep = parity.compare(g["rgb"][pix], g["ids"][pix], g["bounces"][pix], ref, cls)
    print(f"[{label or sc.name}] {rep}")
    assert rep.ok, f"{label or sc.name}: {rep}"
    # every discrete decision is taken in FP64 on both sides: hit ids and bounce counts match on
    # (almost) every pixel, edge-class ones included
    frac = parity.exact_id_fraction(g["ids"][pix], g["bounces"][pix], ref)
    print(f"[{label or sc.name}] bit-exact hit ids + bounces: {frac:.5%} of {len(pix)} pixels")
    assert frac >= parity.MIN_EXACT_ID_FRAC, frac
    if pixels is None:
        ok, msg = parity.ray_budget_ok(g["stats"], ref.counts, ref, cls, sc.n_lights)
        print(f"[{label or sc.name}] rays: {msg}")
        assert ok, msg
        ok, msg = parity.counts_equal(g["stats"], ref.counts)
        print(f"[{label or sc.name}] counts: {msg}")
        assert ok, msg
    return g, ref, rep


VARIANTS = ["wavefront", "megakernel"]


@pytest.mark.parametrize("variant", VARIANTS)
def test_c1_full_frame(oracle_lib, variant):
    _check(oracle_lib, scenegen.get("C1"), variant=variant, label=f"C1/{variant}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_c2_full_frame(oracle_lib, variant):
    _check(oracle_lib, scenegen.get("C2"), variant=variant, label=f"C2/{variant}")


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_variants_bit_identical(name):
    # the wavefront and megakernel organisations compute the same terms in the same order
    sc = scenegen.get(name)
    if name in ("C3", "C4"):
        sc = sc.with_frame(width=480, height=270)
    a = gpu_render(sc, variant="wavefront")
    b = gpu_render(sc, variant="megakernel")
    assert (a["rgba"].view(np.uint32) == b["rgba"].view(np.uint32)).all()
    assert (a["ids"] == b["ids"]).all() and (a["bounces"] == b["bounces"]).all()
    for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests"):
        assert a["stats"][k] == b["stats"][k], k


def test_c2_ragged_deeper_supersampled(oracle_lib):
    # ragged against 8x4 tiles, non-square spp (Hammersley), deeper bounces
    sc = scenegen.get("C2").with_frame(width=67, height=45, max_depth=6, spp=3)
    _check(oracle_lib, sc, label="C2-ragged")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("seed,W,H,D,spp", [(0, 13, 7, 3, 1), (1, 9, 9, 6, 4), (2, 17, 5, 0, 2),
                                            (3, 8, 4, 2, 5), (4, 31, 3, 5, 9), (5, 1, 1, 4, 16)])
def test_tiny_random_scenes(oracle_lib, seed, W, H, D, spp, variant):
    sc = scenegen.random_tiny(seed, n_spheres=7, n_planes=2, n_lights=3, width=W, height=H, max_depth=D, spp=spp)
    _check(oracle_lib, sc, label=f"tiny{seed}/{variant}", variant=variant)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("seed,W,H,D,spp", [(20, 13, 7, 4, 1), (21, 9, 9, 6, 4), (22, 17, 5, 3, 2), (23, 11, 10, 5, 1)])
def test_interleaved_order_and_tinted_glass(oracle_lib, seed, W, H, D, spp, variant):
    """Primitive orders other than planes-first (two planes inserted between the spheres: ties
    and test counts follow primitive indices, §8(c).1 step 11) and coloured glass (the
    REFRACTIVE weight T *= rho); exact counts against the oracle."""
    sc = scenegen.random_tiny(seed, n_spheres=8, n_planes=2, n_lights=3, width=W, height=H, max_depth=D, spp=spp,
                              glass_tint=True, interleave=True)
    assert list(sc.prim_type[:5]) == [0, 0, 0, 0, 1]  # spheres before the planes
    assert (sc.mat_albedo[sc.mat_kind == scenegen.REFRACTIVE] < 1).any()
    _check(oracle_lib, sc, label=f"interleaved{seed}/{variant}", variant=variant)


def _sweep_cases():
    """Seeded sweep over the scene shapes the kernels branch on: sphere counts around the pair /
    batch / AUTO boundaries (1, 2, 15, 16, 17, 63, 64, 65, 150, 300; dense, so the eye often sits
    inside spheres), 0-2 planes, planes-first or interleaved orders, 0-30 point lights (light-origin
    scans up to 30), depths 0-6, 1-5 spp, ragged frames."""
    g = np.random.default_rng(2024)
    cases = []
    for i, ns in enumerate([1, 2, 15, 16, 17, 63, 64, 65, 150, 300, 40, 9]):
        cases.append(dict(seed=300 + i, n_spheres=ns, n_planes=int(g.integers(0, 3)), n_lights=int(g.choice([0, 1, 5, 12, 30])),
                          width=int(g.integers(5, 19)), height=int(g.integers(3, 13)), max_depth=int(g.integers(0, 7)),
                          spp=int(g.integers(1, 6)), glass_tint=bool(g.integers(0, 2)), interleave=bool(g.integers(0, 2))))
    return cases


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"s{c['seed']}-n{c['n_spheres']}-l{c['n_lights']}")
def test_random_sweep(oracle_lib, variant, case):
    sc = scenegen.random_tiny(**case)
    _check(oracle_lib, sc, label=f"sweep {case['seed']}/{variant}", variant=variant)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n_lights", [29, 30, 31, 32])
def test_many_point_lights(oracle_lib, variant, n_lights):
    """Up to 30 point lights are scanned from the light (one lane each in wf_shade's slot
    reservation), 31-32 (RT_MAX_LIGHTS) through the general scan: both sides of the limit."""
    sc = scenegen.random_tiny(40 + n_lights, n_spheres=9, n_planes=1, n_lights=n_lights, width=23, height=11,
                              max_depth=3, spp=1)
    _check(oracle_lib, sc, label=f"{n_lights} lights/{variant}", variant=variant)


def _shared_origin_scene(case):
    """Edge cases of the shared-origin tangent test (camera rays and light-origin shadow scans,
    rt_kernels.cu neg_tangent): the eye or a light inside a sphere, the eye exactly on a surface, a
    light within 1e-6 S of one (always a candidate), 1e-4 and 1e-3 off one (tested); a ground
    plane tilted by 1e-8 gives shading points at t ~ 2e8 (the light-origin scan drops nothing
    past t_l > 1e6 S)."""
    g = scenegen.SplitMix64(900 + case)
    b = scenegen.builder()
    f32 = lambda x: float(np.float32(x))
    dif = b.material(scenegen.DIFFUSE, (0.7, 0.6, 0.5), ks=0.3, shininess=20.0, kr=0.2)
    mir = b.material(scenegen.SPECULAR, (0.9, 0.9, 0.9))
    gls = b.material(scenegen.REFRACTIVE, (1, 1, 1), ior=1.5)
    for i in range(40):
        c = (g.uniform(-6, 6), g.uniform(-2, 4) if case < 3 else g.uniform(1.5, 5), g.uniform(3, 16))
        b.sphere(tuple(f32(x) for x in c), f32(g.uniform(0.3, 1.2)), (dif, mir, gls)[i % 3])
    # case 3: a ground plane tilted by 1e-8: the image's centre row (dy = 0) meets it at t ~ 2e8
    b.plane((0, 1, -1e-8) if case == 3 else (0, 1, 0), -2.0, dif)
    eye = (0.0, 0.0, 0.0)
    if case == 0:    # eye inside a glass sphere; a light inside another sphere
        b.sphere((0.25, 0.0, 0.5), 1.0, gls)
        b.sphere((5.0, 6.0, 9.0), 0.5, dif)
        b.light((5.0, 6.0, 9.0), (60, 60, 60))
    elif case == 1:  # eye exactly on a sphere's surface; a light 1e-3 off another's (tested, h ~ 0.045)
        # (a light exactly ON a surface is no parity case: every shadow ray toward it meets that
        # sphere at t = t_max, decided by the last bit of FP64 rounding, and nvcc contracts the
        # FP64 dot products into FMAs where the oracle's gcc build does not)
        b.sphere((0.0, 0.0, -1.0), 1.0, dif)
        b.sphere((3.0, 5.0, 8.0), 1.0, dif)
        b.light((3.0, 3.999, 8.0), (60, 60, 60))
    elif case == 2:  # within 1e-6 S (always candidates) and at 1e-4 of the surface (tested)
        b.sphere((0.0, 0.0, f32(-1.0 - 2e-6)), 1.0, mir)
        b.sphere((3.0, 5.0, 8.0), 1.0, dif)
        b.light((3.0, f32(4.0 - 2e-6), 8.0), (60, 60, 60))
        b.light((-3.0, f32(4.0 - 1e-4), 8.0), (40, 40, 40))
        b.sphere((-3.0, 5.0, 8.0), 1.0, gls)
    else:            # far shading points: t_l ~ 2e8 > 1e6 S
        b.light((0.0, 3.0, 6.0), (80, 80, 80))
    b.light((-4.0, 8.0, 2.0), (50, 50, 50))
    return b.build(f"shared-origin-{case}", eye=eye, look_at=(0.0, 0.0, 1.0), up=(0, 1, 0), vfov=60,
                   width=48, height=33, max_depth=3, spp=1, background=(0.1, 0.2, 0.3))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_shared_origin_edge_cases(oracle_lib, variant, case):
    _check(oracle_lib, _shared_origin_scene(case), label=f"shared-origin {case}/{variant}", variant=variant)


@pytest.mark.parametrize("spp", [255, 256, 257, 300])
def test_sub_pixel_offsets_table_and_computed(oracle_lib, spp):
    """spp <= 256 reads the sub-pixel offsets from the constant table, beyond that they are
    computed per sample (the same IEEE values): both against the oracle."""
    sc = scenegen.random_tiny(91, n_spheres=6, n_planes=1, n_lights=2, width=3, height=2, max_depth=2, spp=spp)
    _check(oracle_lib, sc, label=f"spp {spp}", variant="wavefront")


@pytest.mark.parametrize("split", [-1, 2, 8])
def test_light_origin_tables_beyond_64k(oracle_lib, split):
    """16 point lights x 1100 spheres: the lights' -h columns (70 KB) no longer fit the short-list
    scan's staging, which then works light by light like the long-list scan; forced splits (2, 8
    parts) run that path on every list. Full-frame parity with exact counts."""
    from paper_1504_03151_b200 import rt
    sc = scenegen.random_tiny(77, n_spheres=1100, n_planes=1, n_lights=16, width=20, height=12, max_depth=3, spp=2)
    rt.set_scan_split(split)
    try:
        _check(oracle_lib, sc, label=f"16 lights x 1100 spheres, split {split}", variant="wavefront")
    finally:
        rt.set_scan_split(-1)


@pytest.mark.parametrize("variant", VARIANTS)
def test_tinted_glass_c2_shaped(oracle_lib, variant):
    """C2-sized frame of a scene with many coloured-glass spheres (every third material glass)."""
    sc = scenegen.random_tiny(31, n_spheres=12, n_planes=1, n_lights=2, width=96, height=64, max_depth=5, spp=1,
                              glass_tint=True)
    _check(oracle_lib, sc, label=f"tinted/{variant}", variant=variant)


def test_c3_full_size_sampled(oracle_lib):
    sc = scenegen.get("C3")
    pix = np.random.default_rng(33).choice(sc.width * sc.height, 6000, replace=False)
    _check(oracle_lib, sc, pixels=pix, label="C3@1080p")


@pytest.mark.parametrize("variant", VARIANTS)
def test_c4_full_size_sampled(oracle_lib, variant):
    sc = scenegen.get("C4")
    pix = np.random.default_rng(44).choice(sc.width * sc.height, 3000, replace=False)
    _check(oracle_lib, sc, pixels=pix, label=f"C4@1080p/{variant}", variant=variant)


def test_c5_full_size_sampled(oracle_lib):
    # 3840x2160, 16 spp, depth 8: 132.7 M paths -> 32 wavefront chunks; oracle on sampled pixels
    sc = scenegen.get("C5")
    pix = np.sort(np.random.default_rng(55).choice(sc.width * sc.height, 1200, replace=False))
    g = gpu_render(sc, pixels=pix)
    ref = oracle_lib.render(sc, pixels=pix)
    cls = parity.classify(oracle_lib, sc, ref, pix)
    rep = parity.compare(g["rgb"], g["ids"], g["bounces"], ref, cls)
    print(f"[C5@4K] {rep}")
    assert rep.ok, rep
    assert g["stats"]["primary"] == sc.width * sc.height * sc.spp


def test_c4_full_size_counts_consistent(oracle_lib):
    # rays-per-pixel statistics of the full-size GPU frame agree with the oracle sample
    sc = scenegen.get("C4")
    g = gpu_render(sc, debug=False)
    st = g["stats"]
    assert st["primary"] == sc.width * sc.height * sc.spp
    pix = np.random.default_rng(45).choice(sc.width * sc.height, 3000, replace=False)
    ref = oracle_lib.render(sc, pixels=pix)
    for k in ("shadow", "secondary", "sphere_tests"):
        gpu_rate = st[k] / st["primary"]
        orc_rate = ref.counts[k] / ref.counts["primary"]
        assert gpu_rate == pytest.approx(orc_rate, rel=0.1), k


def test_worked_examples_on_gpu():
    # W1, W2, W4 closed forms (tests/golden/worked_examples.json) through the CUDA path
    b = scenegen.builder()
    b.sphere((0, 0, 5), 1.0, b.material(scenegen.DIFFUSE, (0.5, 0.5, 0.5)))
    b.light((0, 0, 0), (16 * math.pi,) * 3)
    sc = b.build("W1", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=1, height=1,
                 max_depth=0, spp=1, ambient=(0.1,) * 3)
    g = gpu_render(sc)
    assert g["rgb"][0] == pytest.approx([0.55] * 3, rel=2e-6)
    assert g["stats"]["shadow"] == 1
    for D in (0, 1, 3, 5, 8):
        b = scenegen.builder()
        m = b.material(scenegen.SPECULAR, (0.5, 0.5, 0.5), emission=(1, 1, 1))
        b.plane((0, 0, 1), 0.0, m)
        b.plane((0, 0, 1), 10.0, m)
        sc = b.build("W4", eye=(0, 0, 5), look_at=(0, 0, 6), up=(0, 1, 0), vfov=30, width=1, height=1,
                     max_depth=D, spp=1)
        g = gpu_render(sc)
        assert g["rgb"][0, 0] == 2 - 0.5 ** D  # exact in float32 too
        assert g["bounces"][0, 0] == D


def test_empty_and_planes_only_scenes(oracle_lib):
    b = scenegen.builder()
    b.material(scenegen.DIFFUSE, (0.5, 0.5, 0.5))
    sc = b.build("empty", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=19, height=6,
                 max_depth=3, spp=2, background=(0.25, 0.5, 0.125))
    g = gpu_render(sc)
    assert (g["rgb"] == np.array([0.25, 0.5, 0.125], np.float32)).all()
    assert (g["rgba"][:, 3] == 1.0).all()
    assert g["stats"]["primary"] == 19 * 6 * 2 and g["stats"]["secondary"] == 0
    b = scenegen.builder()
    b.plane((0, 1, 0), 0.0, b.material(scenegen.DIFFUSE, (0.6, 0.6, 0.6), kr=0.5))
    b.plane((0, -1, 0), -6.0, b.material(scenegen.SPECULAR, (0.8, 0.8, 0.8)))
    b.light((0, 3, 4), (50, 50, 50))
    sc = b.build("planes", eye=(0, 1, -5), look_at=(0, 1, 0), up=(0, 1, 0), vfov=70, width=24, height=20,
                 max_depth=4, spp=1, background=(0.1, 0.1, 0.1), ambient=(0.05, 0.05, 0.05))
    _check(oracle_lib, sc, label="planes-only")


@pytest.mark.parametrize("name,variant", [("C2", "auto"), ("C2", "wavefront"), ("C4", "wavefront"),
                                          ("C5", "wavefront")])
def test_host_and_device_outputs_identical(name, variant):
    """Host framebuffers (the wavefront copies each chunk's finished rows on a second stream while
    later chunks render; C4 = 2 chunks, C5 = 32) equal device ones bit for bit."""
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get(name)
    if name == "C5":
        sc = sc.with_frame(spp=4, max_depth=2)
    rt.set_variant(variant)
    rt.load_scene(sc)
    dev = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    rt.render(sc.width, sc.height, sc.max_depth, sc.spp, dev)
    host = np.empty((sc.height, sc.width, 4), np.float32)
    rt.render(sc.width, sc.height, sc.max_depth, sc.spp, host)
    torch.cuda.synchronize()
    assert (dev.cpu().numpy().view(np.uint32) == host.view(np.uint32)).all()
    again = torch.empty_like(dev)
    rt.render(sc.width, sc.height, sc.max_depth, sc.spp, again)
    assert torch.equal(again, dev)  # deterministic
    rt.set_variant("auto")


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_assemble_bit_identical(world):
    # SURVEY §4 level (i): every rank's shard rendered on one GPU, gathered by concatenation
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C2").with_frame(width=203, height=117, spp=2)
    rt.load_scene(sc)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    full = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    rt.render(W, H, D, S, full)
    ref_stats = rt.stats()
    tpr, sb = rt.shard_layout(W, H, world)
    gathered = torch.zeros(world * sb, dtype=torch.uint8, device="cuda")
    for r in range(world):
        rt.render_shard(W, H, D, S, r, world, gathered[r * sb:(r + 1) * sb])
    out = torch.empty_like(full)
    rt.assemble_tiles(gathered, W, H, world, out)
    st = rt.stats()
    torch.cuda.synchronize()
    assert torch.equal(out, full)
    for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests"):
        assert st[k] == ref_stats[k], k


def test_tonemap_kernel_matches_spec():
    import torch
    from paper_1504_03151_b200 import rt
    v = np.random.default_rng(0).uniform(-0.2, 1.3, (1000, 4)).astype(np.float32)
    v[:5, 0] = [0.0, 0.5, 1.0, 2.0, -1.0]
    dev = torch.from_numpy(v).cuda()
    out = torch.empty((1000, 4), dtype=torch.uint8, device="cuda")
    rt.tonemap_rgba8(dev, out)
    got = out.cpu().numpy()
    want = parity.tonemap8(v[:, :3])
    assert (got[:, :3] == want).all() and (got[:, 3] == 255).all()
    assert list(got[:5, 0]) == [0, 186, 255, 255, 0]


def test_validation_errors():
    from paper_1504_03151_b200 import rt
    sc = scenegen.get("C1")
    prims, mats, lights, env = rt.pack_scene(sc)
    bad = prims.copy()
    bad["p"][2, 3] = -1.0
    with pytest.raises(rt.RtError) as e:
        rt.scene_upload(bad, mats, lights, env)
    assert e.value.code == -1 and "prim 2" in e.value.msg and "radius" in e.value.msg
    bad = prims.copy()
    bad["material"][1] = 99
    with pytest.raises(rt.RtError) as e:
        rt.scene_upload(bad, mats, lights, env)
    assert "prim 1" in e.value.msg
    badm = mats.copy()
    badm["albedo"][0, 1] = 1.5
    with pytest.raises(rt.RtError) as e:
        rt.scene_upload(prims, badm, lights, env)
    assert "material 0" in e.value.msg
    with pytest.raises(rt.RtError) as e:
        rt.camera_set((0, 0, 0), (0, 0, 0), (0, 1, 0), 60)
    assert e.value.code == -1
    with pytest.raises(rt.RtError) as e:
        rt.camera_set((0, 0, 0), (0, 1, 0), (0, 1, 0), 60)  # up parallel to view
    with pytest.raises(rt.RtError) as e:
        rt.camera_set((0, 0, 0), (0, 0, 1), (0, 1, 0), 180)
    rt.load_scene(sc)
    import torch
    out = torch.empty((4, 4, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(rt.RtError) as e:
        rt.render(4, 4, -1, 1, out)
    assert e.value.code == -1
    with pytest.raises(rt.RtError):
        rt.render(0, 4, 1, 1, out)
    with pytest.raises(rt.RtError):
        rt.render(4, 4, 1, 0, out)
    with pytest.raises(rt.RtError):
        rt.render_shard(4, 4, 1, 1, 2, 2, out)  # rank >= world
    # state is unchanged after errors: a valid render still works
    rt.render(4, 4, 1, 1, out)


def _big_scene():
    g = scenegen.SplitMix64(77)
    b = scenegen.builder()
    mats = [b.material(scenegen.DIFFUSE, (0.7, 0.5, 0.3), ks=0.2, shininess=16.0),
            b.material(scenegen.SPECULAR, (0.9, 0.9, 0.9)),
            b.material(scenegen.REFRACTIVE, (1, 1, 1), ior=1.5),
            b.material(scenegen.DIFFUSE, (0.4, 0.6, 0.8), kr=0.4)]
    for i in range(12000):
        c = (g.uniform(-40, 40), g.uniform(-20, 20), g.uniform(10, 90))
        b.sphere(tuple(float(np.float32(x)) for x in c), float(np.float32(g.uniform(0.2, 0.8))), mats[i % 4])
    b.light((0, 30, 50), (3000, 3000, 3000))
    b.light((-20, 0, 0), (800, 800, 800))
    return b.build("big", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60, width=160, height=90,
                   max_depth=3, spp=1, background=(0.1, 0.1, 0.2))


def test_tiled_scan_bit_identical_and_faster():
    """Scenes beyond shared memory: the TMA-tiled scans (two 16 KB tiles per CTA in flight) and the
    global-memory scans produce the same frame, counts included; the tiled ones are timed too."""
    import torch
    from paper_1504_03151_b200 import rt
    sc = _big_scene().with_frame(width=640, height=360)
    rt.set_variant("wavefront")
    rt.load_scene(sc)
    res = {}
    try:
        for tiled in (0, 1):
            rt.set_tiled_scan(tiled)
            out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
            ms = []
            for _ in range(4):
                rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
                st = rt.stats()
                ms.append(st["last_render_ms"])
            torch.cuda.synchronize()
            res[tiled] = (out.clone(), {k: st[k] for k in ("primary", "shadow", "secondary", "sphere_tests")}, min(ms))
    finally:
        rt.set_tiled_scan(1)
        rt.set_variant("auto")
    assert torch.equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]
    print(f"12k spheres 640x360: global {res[0][2]:.3f} ms, tiled {res[1][2]:.3f} ms")


@pytest.mark.parametrize("variant", VARIANTS)
def test_scene_beyond_shared_memory(oracle_lib, variant):
    """12 000 spheres > RT_SMEM_SPHERES (10 240): the scans stream the scene through TMA-loaded
    tiles (or read it from global memory: megakernel, split scans) instead of the TMA-staged
    shared-memory copy; sampled parity vs the oracle."""
    sc = _big_scene()
    pix = np.random.default_rng(5).choice(sc.width * sc.height, 300, replace=False)
    _check(oracle_lib, sc, pixels=pix, label=f"12k spheres/{variant}", variant=variant)
