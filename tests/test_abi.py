"""CPU-side checks of the C ABI boundary: the library builds, loads, exports every function that
include/rt.h declares, and fails loudly (never falls back to the CPU) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1504_03151_b200 import build as rtbuild
from paper_1504_03151_b200 import rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    rtbuild.build()
    return rt.lib()


def test_header_declares_the_north_star_calls():
    names = rt.declared_functions()
    for f in ("rt_scene_upload", "rt_camera_set", "rt_render", "rt_stats"):
        assert f in names


def test_library_exports_every_declared_symbol(lib):
    missing = [f for f in rt.declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_struct_layouts_match_header(tmp_path):
    # rt_primitive 24 B, rt_material 48 B, rt_light 24 B, rt_env 24 B, rt_ray_stats 112 B
    assert rt.PRIM_DTYPE.itemsize == 24 and rt.MAT_DTYPE.itemsize == 48
    assert rt.LIGHT_DTYPE.itemsize == 24 and rt.ENV_DTYPE.itemsize == 24
    assert ctypes.sizeof(rt.RayStats) == 112
    # every rt_ray_stats field of the binding sits at the offset the C compiler gives the header's
    fields = [f for f, _ in rt.RayStats._fields_]
    src = "#include <stddef.h>\n#include <stdio.h>\n#include \"rt.h\"\nint main(void) {\n"
    src += f'  printf("%zu\\n", sizeof(rt_ray_stats));\n'
    for f in fields:
        src += f'  printf("%zu\\n", offsetof(rt_ray_stats, {f}));\n'
    src += "  return 0;\n}\n"
    (tmp_path / "t.c").write_text(src)
    import subprocess
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), "-o", str(tmp_path / "t"),
                           str(tmp_path / "t.c")])
    out = [int(x) for x in subprocess.check_output([str(tmp_path / "t")]).split()]
    assert out[0] == ctypes.sizeof(rt.RayStats)
    assert out[1:] == [getattr(rt.RayStats, f).offset for f in fields]
    hdr = open(os.path.join(ROOT, "include", "rt.h")).read()
    assert re.search(r"RT_TILE_W = 8", hdr) and re.search(r"RT_TILE_H = 4", hdr)


def test_shard_layout_is_host_only(lib):
    # no device needed: pure arithmetic
    tpr, sb = rt.shard_layout(1920, 1080, 8)
    tiles = (1920 // 8) * (1080 // 4)
    assert tpr == -(-tiles // 8) and sb == tpr * 32 * 16 + 64
    tpr, sb = rt.shard_layout(13, 7, 3)
    assert tpr == -(-(2 * 2) // 3)
    with pytest.raises(rt.RtError) as e:
        rt.shard_layout(0, 5, 1)
    assert e.value.code == -1


def test_no_cpu_fallback_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    from scenegen import get
    sc = get("C1")
    with pytest.raises(rt.RtError) as e:
        rt.load_scene(sc)
    assert e.value.code == -4  # RT_ERR_CUDA, not a silent host computation
    out = np.zeros((4, 4, 4), np.float32)
    with pytest.raises(rt.RtError):
        rt.render(4, 4, 1, 1, out)
    assert (out == 0).all()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(rt, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(rt, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rt.lib()


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1504_03151_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|pyoracle|orc_render|oracle/)", src), f
