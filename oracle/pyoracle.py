"""ctypes wrapper around liboracle.so (the plain C oracle).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "oracle.c")]
_HDR = os.path.join(_HERE, "oracle.h")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C11, IEEE double, no FP contraction)."""
    newest = max(os.path.getmtime(p) for p in _SRC + [_HDR])
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-Wall", "-o", tmp] + _SRC + ["-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Scene(C.Structure):
    _fields_ = [
        ("n_prims", C.c_int32), ("prim_type", C.c_void_p), ("prim_mat", C.c_void_p),
        ("prim_p", C.c_void_p), ("n_mats", C.c_int32), ("mat_kind", C.c_void_p),
        ("mat_albedo", C.c_void_p), ("mat_emission", C.c_void_p), ("mat_ior", C.c_void_p),
        ("mat_ks", C.c_void_p), ("mat_shininess", C.c_void_p), ("mat_kr", C.c_void_p),
        ("n_lights", C.c_int32), ("light_pos", C.c_void_p), ("light_intensity", C.c_void_p),
        ("background", C.c_void_p), ("ambient", C.c_void_p), ("eye", C.c_void_p),
        ("look_at", C.c_void_p), ("up", C.c_void_p), ("vfov_deg", C.c_float),
    ]


class _Frame(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("max_depth", C.c_int32),
                ("spp", C.c_int32), ("seed", C.c_uint64), ("perturb", C.c_double),
                ("perturb_seed", C.c_uint64), ("integrator", C.c_int32), ("area_lights", C.c_int32),
                ("jitter", C.c_int32), ("pad_", C.c_int32), ("sample_base", C.c_int64)]


class _Counts(C.Structure):
    _fields_ = [("primary", C.c_uint64), ("shadow", C.c_uint64), ("secondary", C.c_uint64),
                ("sphere_tests", C.c_uint64), ("plane_tests", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        _lib.orc_render.restype = C.c_int
        _lib.orc_render.argtypes = [C.POINTER(_Scene), C.POINTER(_Frame), C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(_Counts)]
        _lib.orc_solve_quadratic.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        _lib.orc_intersect_sphere.argtypes = [dp, dp, dp, C.c_double, dp]
        _lib.orc_intersect_plane.argtypes = [dp, dp, dp, C.c_double, dp]
        _lib.orc_reflect.argtypes = [dp, dp, dp]
        _lib.orc_refract.argtypes = [dp, dp, C.c_double, dp]
        _lib.orc_sample_offset.argtypes = [C.c_int32, C.c_int32, dp, dp]
        _lib.orc_camera_ray.argtypes = [C.POINTER(_Scene), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, dp, dp]
        _lib.orc_mix64.restype = C.c_uint64
        _lib.orc_mix64.argtypes = [C.c_uint64]
        _lib.orc_rng.restype = C.c_double
        _lib.orc_rng.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
        _lib.orc_rng_stream.restype = C.c_double
        _lib.orc_rng_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        _lib.orc_sample_sphere.restype = C.c_double
        _lib.orc_sample_sphere.argtypes = [dp, C.c_double, C.c_double, C.c_double, dp, dp]
        _lib.orc_onb.argtypes = [dp, dp, dp]
        _lib.orc_cosine_direction.argtypes = [dp, C.c_double, C.c_double, dp]
        _lib.orc_render_local_grid.restype = C.c_int
        _lib.orc_render_local_grid.argtypes = [C.POINTER(_Scene), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                               C.c_void_p]
        _lib.orc_brdf.argtypes = [C.c_int32, dp, C.c_double, C.c_double, dp, dp, dp, dp]
        _lib.orc_schlick.restype = C.c_double
        _lib.orc_schlick.argtypes = [C.c_double, C.c_double]
        _lib.orc_tonemap8.restype = C.c_int32
        _lib.orc_tonemap8.argtypes = [C.c_double, C.c_double, C.c_double]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class _SceneHolder:
    """Keeps contiguous float32/int32 copies alive while the C struct points at them."""

    def __init__(self, sc):
        f, i = np.float32, np.int32
        self.arrs = dict(
            prim_type=np.ascontiguousarray(sc.prim_type, i), prim_mat=np.ascontiguousarray(sc.prim_mat, i),
            prim_p=np.ascontiguousarray(sc.prim_p, f), mat_kind=np.ascontiguousarray(sc.mat_kind, i),
            mat_albedo=np.ascontiguousarray(sc.mat_albedo, f), mat_emission=np.ascontiguousarray(sc.mat_emission, f),
            mat_ior=np.ascontiguousarray(sc.mat_ior, f), mat_ks=np.ascontiguousarray(sc.mat_ks, f),
            mat_shininess=np.ascontiguousarray(sc.mat_shininess, f), mat_kr=np.ascontiguousarray(sc.mat_kr, f),
            light_pos=np.ascontiguousarray(sc.light_pos, f).reshape(-1, 3),
            light_intensity=np.ascontiguousarray(sc.light_intensity, f).reshape(-1, 3),
            background=np.ascontiguousarray(sc.background, f), ambient=np.ascontiguousarray(sc.ambient, f),
            eye=np.ascontiguousarray(sc.eye, f), look_at=np.ascontiguousarray(sc.look_at, f),
            up=np.ascontiguousarray(sc.up, f))
        a = self.arrs
        self.s = _Scene(
            n_prims=len(a["prim_type"]), prim_type=_ptr(a["prim_type"]), prim_mat=_ptr(a["prim_mat"]),
            prim_p=_ptr(a["prim_p"]), n_mats=len(a["mat_kind"]), mat_kind=_ptr(a["mat_kind"]),
            mat_albedo=_ptr(a["mat_albedo"]), mat_emission=_ptr(a["mat_emission"]), mat_ior=_ptr(a["mat_ior"]),
            mat_ks=_ptr(a["mat_ks"]), mat_shininess=_ptr(a["mat_shininess"]), mat_kr=_ptr(a["mat_kr"]),
            n_lights=len(a["light_pos"]), light_pos=_ptr(a["light_pos"]),
            light_intensity=_ptr(a["light_intensity"]), background=_ptr(a["background"]),
            ambient=_ptr(a["ambient"]), eye=_ptr(a["eye"]), look_at=_ptr(a["look_at"]), up=_ptr(a["up"]),
            vfov_deg=float(sc.vfov))


@dataclass
class OracleResult:
    rgb: np.ndarray        # [n,3] float64 mean radiance
    hit_ids: np.ndarray    # [n,spp,max_depth+1] int32
    bounces: np.ndarray    # [n,spp] int32
    margin: np.ndarray     # [n,spp] float64
    sample_rgb: np.ndarray  # [n,spp,3]
    counts: dict
    pixels: np.ndarray     # [n] int64 pixel indices


def render(sc, pixels=None, perturb: float = 0.0, perturb_seed: int = 0,
           width=None, height=None, max_depth=None, spp=None, seed=None,
           integrator: int = 0, area_lights: int = 0, jitter: int = 0, sample_base: int = 0) -> OracleResult:
    L = lib()
    W = sc.width if width is None else width
    H = sc.height if height is None else height
    D = sc.max_depth if max_depth is None else max_depth
    S = sc.spp if spp is None else spp
    sd = sc.seed if seed is None else seed
    holder = _SceneHolder(sc)
    fr = _Frame(width=W, height=H, max_depth=D, spp=S, seed=sd, perturb=perturb, perturb_seed=perturb_seed,
                integrator=integrator, area_lights=area_lights, jitter=jitter, sample_base=sample_base)
    if pixels is None:
        pix = np.arange(W * H, dtype=np.int64)
        ppix = None
    else:
        pix = np.ascontiguousarray(pixels, dtype=np.int64)
        ppix = _ptr(pix)
    n = len(pix)
    rgb = np.zeros((n, 3), np.float64)
    ids = np.zeros((n, S, D + 1), np.int32)
    bn = np.zeros((n, S), np.int32)
    mg = np.zeros((n, S), np.float64)
    srgb = np.zeros((n, S, 3), np.float64)
    cnt = _Counts()
    rc = L.orc_render(C.byref(holder.s), C.byref(fr), ppix, n, _ptr(rgb), _ptr(ids), _ptr(bn), _ptr(mg),
                      _ptr(srgb), C.byref(cnt))
    if rc != 0:
        raise ValueError(f"orc_render failed rc={rc}")
    counts = {k: int(getattr(cnt, k)) for k, _ in _Counts._fields_}
    return OracleResult(rgb, ids, bn, mg, srgb, counts, pix)


def render_local_grid(sc, light_grid: int, rays_per_pixel: int, width=None, height=None) -> np.ndarray:
    """NEXT-3: the literal Alg. 1 light-grid quadrature (local illumination); [H*W, 3] float64."""
    W = sc.width if width is None else width
    H = sc.height if height is None else height
    holder = _SceneHolder(sc)
    rgb = np.zeros((W * H, 3), np.float64)
    rc = lib().orc_render_local_grid(C.byref(holder.s), W, H, light_grid, rays_per_pixel, _ptr(rgb))
    if rc != 0:
        raise ValueError(f"orc_render_local_grid failed rc={rc}")
    return rgb


def render_rgb_only(sc, pixels=None, integrator: int = 0, area_lights: int = 0, jitter: int = 0,
                    sample_base: int = 0) -> tuple:
    """Cheaper call for timing (cpu baseline): only the image and the counts."""
    L = lib()
    W, H = sc.width, sc.height
    holder = _SceneHolder(sc)
    fr = _Frame(width=W, height=H, max_depth=sc.max_depth, spp=sc.spp, seed=sc.seed, perturb=0.0, perturb_seed=0,
                integrator=integrator, area_lights=area_lights, jitter=jitter, sample_base=sample_base)
    if pixels is None:
        n, ppix = W * H, None
    else:
        pix = np.ascontiguousarray(pixels, dtype=np.int64)
        n, ppix = len(pix), _ptr(pix)
    rgb = np.zeros((n, 3), np.float64)
    cnt = _Counts()
    rc = L.orc_render(C.byref(holder.s), C.byref(fr), ppix, n, _ptr(rgb), None, None, None, None, C.byref(cnt))
    if rc != 0:
        raise ValueError(f"orc_render failed rc={rc}")
    return rgb, {k: int(getattr(cnt, k)) for k, _ in _Counts._fields_}


# ---- thin wrappers for the unit pins --------------------------------------------------------
def _d3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def solve_quadratic(a, b, c):
    r = (C.c_double * 2)()
    n = lib().orc_solve_quadratic(a, b, c, r)
    return [r[i] for i in range(n)]


def intersect_sphere(o, d, c, r):
    t = C.c_double()
    return t.value if lib().orc_intersect_sphere(_d3(o), _d3(d), _d3(c), r, C.byref(t)) else None


def intersect_plane(o, d, n, dp):
    t = C.c_double()
    return t.value if lib().orc_intersect_plane(_d3(o), _d3(d), _d3(n), dp, C.byref(t)) else None


def reflect(d, n):
    out = (C.c_double * 3)()
    lib().orc_reflect(_d3(d), _d3(n), out)
    return np.array(list(out))


def refract(d, n, eta):
    out = (C.c_double * 3)()
    ok = lib().orc_refract(_d3(d), _d3(n), eta, out)
    return np.array(list(out)) if ok else None


def sample_offset(s, spp):
    ox, oy = C.c_double(), C.c_double()
    lib().orc_sample_offset(s, spp, C.byref(ox), C.byref(oy))
    return ox.value, oy.value


def camera_ray(sc, width, height, px, py, s=0, spp=1):
    h = _SceneHolder(sc)
    o, d = (C.c_double * 3)(), (C.c_double * 3)()
    lib().orc_camera_ray(C.byref(h.s), width, height, px, py, s, spp, o, d)
    return np.array(list(o)), np.array(list(d))


def mix64(x):
    return int(lib().orc_mix64(x))


def rng(seed, pixel, sample, depth):
    return float(lib().orc_rng(seed, pixel, sample, depth))


def rng_stream(seed, pixel, sample, depth, stream):
    return float(lib().orc_rng_stream(seed, pixel, sample, depth, stream))


def sample_sphere(c, r, u1, u2):
    x, nl = (C.c_double * 3)(), (C.c_double * 3)()
    pdf = lib().orc_sample_sphere(_d3(c), r, u1, u2, x, nl)
    return np.array(list(x)), np.array(list(nl)), float(pdf)


def onb(n):
    t1, t2 = (C.c_double * 3)(), (C.c_double * 3)()
    lib().orc_onb(_d3(n), t1, t2)
    return np.array(list(t1)), np.array(list(t2))


def cosine_direction(n, u1, u2):
    out = (C.c_double * 3)()
    lib().orc_cosine_direction(_d3(n), u1, u2, out)
    return np.array(list(out))


def brdf(kind, albedo, ks, shininess, wi, wo, n):
    f = (C.c_double * 3)()
    lib().orc_brdf(kind, _d3(albedo), ks, shininess, _d3(wi), _d3(wo), _d3(n), f)
    return np.array(list(f))


def schlick(ior, c):
    return float(lib().orc_schlick(ior, c))


def tonemap8(v, exposure=1.0, gamma=2.2):
    return int(lib().orc_tonemap8(v, exposure, gamma))
