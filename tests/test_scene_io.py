"""NEXT-4 on the CPU: the scene-text parser of the C ABI (rt_scene_parse; SPEC
parse_scene S:217-225) — examples, error lines, a fuzz property — the CLI's exit codes
(S:495-504), and the text serializer's float32 round trip. Parsing happens before any device
call, so on a machine without a GPU a valid text ends in RT_ERR_CUDA (at upload), an invalid
one in RT_ERR_PARSE."""
import os
import subprocess
import sys

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import scenegen
from paper_1504_03151_b200 import build as rtbuild
from paper_1504_03151_b200 import rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PARSE, CUDA = -7, -4
MIN = "camera 0 0 -10  0 0 0  0 1 0  45\nsphere 1  0 0 5  0 0 0  0.5 0.5 0.5  diffuse\n"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    rtbuild.build()
    yield


def _rc(text):
    b = text.encode() if isinstance(text, str) else text
    rc = rt.lib().rt_scene_parse(b, len(b))
    return rc, rt.lib().rt_last_error().decode(errors="replace")


def _valid(rc):
    # valid text: parse succeeded, then upload needs a device (no GPU here) or succeeds (GPU box)
    return rc in (0, CUDA)


def test_spec_minimal_file_is_valid():
    rc, msg = _rc(MIN)
    assert _valid(rc), msg


@pytest.mark.parametrize("text,line,why", [
    ("sphere 1 0 0 5 0 0 0 0.5 0.5 0.5 diffuse\n", 1, "missing camera"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere -1 0 0 5 0 0 0 0.5 0.5 0.5 diffuse\n", 2, "radius <= 0"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\ncamera 0 0 -10 0 0 0 0 1 0 45\n", 2, "duplicate camera"),
    ("camera 0 0 -10 0 0 0 0 1 0\n", 1, "bad arity"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\n\n# c\nsphere 1 0 0 5 0 0 0 1.5 0.5 0.5 diffuse\n", 4, "albedo outside [0,1]"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere 1 0 0 x 0 0 0 0.5 0.5 0.5 diffuse\n", 2, "non-numeric field 'x'"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere 1 0 0 5 0 0 0 0.5 0.5 0.5 metal\n", 2, "unknown kind 'metal'"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere 1 0 0 5 0 0 0 0.5 0.5 0.5 refractive 0.9\n", 2, "ior must be >= 1"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere 1 0 0 5 0 0 0 0.5 0.5 0.5 diffuse glow=1\n", 2, "unknown option 'glow'"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere 1 0 0 5 -1 0 0 0.5 0.5 0.5 diffuse\n", 2, "emission must be >= 0"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nplane 0 0 0 1 0 0 0 0.5 0.5 0.5 diffuse\n", 2, "plane normal is zero"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nteapot 1 2 3\n", 2, "unknown directive 'teapot'"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nlight 0 5 0 1 1\n", 2, "bad arity"),
    ("camera 0 0 -10 0 0 0 0 1 0 45\nsphere 1 0 0 inf 0 0 0 0.5 0.5 0.5 diffuse\n", 2, "non-numeric field 'inf'"),
    ("camera 0 0 0 0 0 0 0 1 0 45\n", 1, "camera: eye == look_at"),
    ("camera 0 0 -10 0 0 0 0 0 1 45\n", 1, "camera: up is zero or parallel"),
    ("camera 0 0 -10 0 0 0 0 1 0 180\n", 1, "camera: vfov"),
])
def test_parse_errors_name_the_line(text, line, why):
    rc, msg = _rc(text)
    assert rc == PARSE, (rc, msg)
    assert msg.startswith(f"line {line}: ") and why in msg, msg


def test_full_grammar_and_comments_parse():
    text = ("# comment\n\n  camera 0 1 -5   0 1 0   0 1 0   50  # trailing comment\r\n"
            "background 0.1 0.2 0.3\nambient 0.01 0.01 0.01\nlight 0 5 0  10 10 10\n"
            "plane 0 1 0 0  0 0 0  0.8 0.8 0.8  diffuse kr=0.2\n"
            "sphere 1  0 1 3  0 0 0  0.9 0.9 0.9  specular\n"
            "sphere 0.5  1 0.5 2  0 0 0  1 1 1  refractive\n"
            "sphere 0.5  -1 0.5 2  0 0 0  1 1 1  refractive 1.33 ks=0.1\n"
            "sphere 0.3  0 3 2  5 5 5  0 0 0  diffuse shininess=8 ks=0.5\n")
    rc, msg = _rc(text)
    assert _valid(rc), msg


def test_empty_and_lights_only():
    assert _rc("")[0] == PARSE and "missing camera" in _rc("")[1]
    rc, msg = _rc("camera 0 0 -1 0 0 0 0 1 0 45\nlight 1 1 1 1 1 1\n")
    assert _valid(rc), msg


@settings(max_examples=300, deadline=None)
@given(st.binary(max_size=300))
def test_parser_never_crashes_on_arbitrary_bytes(data):   # S:235 fuzz property
    rc, msg = _rc(data)
    assert rc in (0, PARSE, CUDA), (rc, msg)
    if rc == PARSE:
        assert msg.startswith("line ") and msg.isprintable()


@settings(max_examples=300, deadline=None)
@given(st.integers(0, len(MIN) - 1), st.binary(min_size=1, max_size=4))
def test_parser_never_crashes_on_mutated_scenes(pos, ins):
    data = MIN.encode()[:pos] + ins + MIN.encode()[pos + 1:]
    rc, _ = _rc(data)
    assert rc in (0, PARSE, CUDA)


def test_serializer_round_trips_float32():
    for name in ("C0", "C2", "C3"):
        sc = scenegen.get(name)
        text = scenegen.to_text(sc)
        rc, msg = _rc(text)
        assert _valid(rc), (name, msg)
        nums = [t for line in text.splitlines() if not line.startswith("#")
                for t in line.split()[1:] if t[0] in "-0123456789"]
        for t in nums:  # %.9g of a float32 parses back to the same float32
            assert np.float32(float(t)) == np.float32(t)
    assert open(os.path.join(ROOT, "scenes", "cornell.scene")).read() == scenegen.to_text(scenegen.get("C0"))


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1504_03151_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_cli_exit_codes(tmp_path):
    assert _cli().returncode == 1                                              # usage: --scene required
    assert _cli("--scene", "x", "--passes", "0").returncode == 1
    r = _cli("--scene", str(tmp_path / "missing.scene"))
    assert r.returncode == 3 and "missing.scene" in r.stderr
    bad = tmp_path / "bad.scene"
    bad.write_text("camera 0 0 -10 0 0 0 0 1 0 45\nsphere -1 0 0 5 0 0 0 0.5 0.5 0.5 diffuse\n")
    r = _cli("--scene", str(bad))
    assert r.returncode == 2 and "line 2" in r.stderr
