"""Race and bounds evidence without compute-sanitizer (closed on this pool):

* the checked build (-DRT_CHECKS=1: every kernel checks its queue, list and slot indices and the
  capacities of every reservation; rt_check_status) renders every kernel organisation and mode,
  through tools/sanitize_run.py, in its own process: no check may fail;
* schedule fuzzing (rt_set_schedule_jitter): random spin kernels at every stream fork, join and
  pipeline-slot start change how the concurrent kernels interleave; every fuzzed frame must equal
  the in-order render (one stream, rt_set_concurrency(0)) bit for bit, statistics included. A
  missing stream dependency (a race between the shadow side stream, the next closest scan and the
  chunk slots) would show as a different frame.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import scenegen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("primary", "shadow", "secondary", "sphere_tests", "plane_tests", "closest_sphere_tests")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_03151_b200 import build
    build.build()
    yield


def test_checked_build_reports_no_violation():
    from paper_1504_03151_b200 import build
    lib = build.build_checked()
    code = ("import sys; sys.path.insert(0, %r); import runpy; runpy.run_path(%r, run_name='__main__'); "
            "from paper_1504_03151_b200 import rt; print('CHECK', *rt.check_status())"
            % (ROOT, os.path.join(ROOT, "tools", "sanitize_run.py")))
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, B200RT_LIB=lib), capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("CHECK")][-1]
    first, compiled = line.split()[1:]
    assert compiled == "True" and first == "0", line


def test_default_build_has_no_checks():
    from paper_1504_03151_b200 import rt
    assert rt.check_status() == (0, False)


@pytest.mark.parametrize("name,frame", [("C4", dict(width=480, height=270)), ("C3", dict(width=480, height=270)),
                                        ("C2", dict(width=256, height=256))])
def test_schedule_fuzzing_bit_identical(name, frame):
    import torch
    from paper_1504_03151_b200 import rt
    sc = scenegen.get(name).with_frame(**frame)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    rt.set_variant("wavefront")
    rt.load_scene(sc)
    out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    rt.set_graphs(False)
    try:
        rt.set_concurrency(False)
        rt.render(W, H, D, S, out)
        st = rt.stats()
        ref, ref_st = out.clone(), {k: st[k] for k in KEYS}
        rt.set_concurrency(True)
        for slots in (2, 3, 4):
            rt.set_pipeline(slots)
            for seed in (1, 2, 3):
                rt.set_schedule_jitter(seed * 7919 + slots)
                out.fill_(float("nan"))
                rt.render(W, H, D, S, out)
                st = rt.stats()
                torch.cuda.synchronize()
                assert torch.equal(out, ref), (slots, seed)
                assert {k: st[k] for k in KEYS} == ref_st, (slots, seed)
    finally:
        rt.set_schedule_jitter(0)
        rt.set_pipeline(0)
        rt.set_concurrency(True)
        rt.set_graphs(True)
        rt.set_variant("auto")
