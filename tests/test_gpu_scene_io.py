"""NEXT-4 on the GPU: scene text round trip (a parsed scene renders bit-identically to the
uploaded one), the P6 PPM writer's exact bytes and the CLI end to end
(exit 0, determinism, snapshots = the mean of the first K passes)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import scenegen
from tests import parity
from tests.gpu_helpers import gpu_render

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    yield


def _render_parsed(sc, text, integrator="whitted", area=False):
    import torch
    from paper_1504_03151_b200 import rt
    rt.set_variant("auto")
    rt.set_integrator(integrator, area)
    rt.scene_parse(text)
    rt.set_seed(sc.seed)
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    rt.render(sc.width, sc.height, sc.max_depth, sc.spp, out)
    st = rt.stats()
    rt.set_integrator("whitted", False)
    return out.reshape(-1, 4).cpu().numpy(), st


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_parsed_scene_renders_bit_identically(name):
    sc = scenegen.get(name)
    ref = gpu_render(sc, debug=False, variant="auto")
    img, st = _render_parsed(sc, scenegen.to_text(sc))
    assert np.array_equal(img, ref["rgba"])
    for k in ("primary", "shadow", "secondary", "sphere_tests", "plane_tests"):
        assert st[k] == ref["stats"][k]


def test_parsed_scene_with_emitters_global():
    sc = scenegen.random_tiny(3, n_spheres=6, n_emitters=2, width=40, height=30, max_depth=4, spp=2)
    ref = gpu_render(sc, debug=False, variant="auto", integrator="global", area_lights=True)
    img, _ = _render_parsed(sc, scenegen.to_text(sc), "global", True)
    assert np.array_equal(img, ref["rgba"])


def _ppm(path):
    b = open(path, "rb").read()
    parts = b.split(b"\n", 3)
    assert parts[0] == b"P6" and parts[2] == b"255"
    w, h = map(int, parts[1].split())
    px = np.frombuffer(parts[3], np.uint8)
    assert px.size == w * h * 3
    return w, h, px.reshape(h, w, 3), b


def test_ppm_exact_bytes(tmp_path):
    import torch
    from paper_1504_03151_b200 import rt
    one = torch.ones((1, 1, 4), dtype=torch.float32, device="cuda")
    rt.write_ppm(one, 1, 1, str(tmp_path / "a.ppm"))
    assert open(tmp_path / "a.ppm", "rb").read() == b"P6\n1 1\n255\n\xff\xff\xff"
    zero = torch.zeros((2, 2, 4), dtype=torch.float32, device="cuda")
    rt.write_ppm(zero, 2, 2, str(tmp_path / "b.ppm"))
    assert open(tmp_path / "b.ppm", "rb").read() == b"P6\n2 2\n255\n" + bytes(12)
    img = torch.rand((5, 7, 4), dtype=torch.float32, device="cuda") * 1.2
    rt.write_ppm(img, 7, 5, str(tmp_path / "c.ppm"))
    w, h, px, _ = _ppm(tmp_path / "c.ppm")
    assert (w, h) == (7, 5)
    assert np.abs(px.astype(int) - parity.tonemap8(img[..., :3].cpu().numpy())).max() <= 1
    with pytest.raises(rt.RtError) as e:
        rt.write_ppm(img, 7, 5, str(tmp_path / "no" / "such" / "dir.ppm"))
    assert e.value.code == -8


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1504_03151_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_end_to_end(tmp_path):
    scene = os.path.join(ROOT, "scenes", "cornell.scene")
    a, b = tmp_path / "a.ppm", tmp_path / "b.ppm"
    r = _cli("--scene", scene, "--passes", "4", "--width", "64", "--height", "48", "--seed", "7", "--out", str(a))
    assert r.returncode == 0, r.stderr
    w, h, px, ba = _ppm(a)
    assert (w, h) == (64, 48) and px.max() > 0
    r = _cli("--scene", scene, "--passes", "4", "--width", "64", "--height", "48", "--seed", "7", "--out", str(b))
    assert r.returncode == 0 and open(b, "rb").read() == ba                                # S:503 determinism
    # snapshots: the pass-2 snapshot of a 4-pass run equals a 2-pass run byte for byte
    c, d = tmp_path / "c.ppm", tmp_path / "d.ppm"
    assert _cli("--scene", scene, "--passes", "4", "--width", "64", "--height", "48", "--snapshot-every", "2",
                "--out", str(c)).returncode == 0
    assert _cli("--scene", scene, "--passes", "2", "--width", "64", "--height", "48", "--out", str(d)).returncode == 0
    assert open(tmp_path / "c_pass2.ppm", "rb").read() == open(d, "rb").read()
    assert open(c, "rb").read() == _cli_bytes(scene, tmp_path)


def _cli_bytes(scene, tmp_path):
    e = tmp_path / "e.ppm"
    assert _cli("--scene", scene, "--passes", "4", "--width", "64", "--height", "48", "--out", str(e)).returncode == 0
    return open(e, "rb").read()
