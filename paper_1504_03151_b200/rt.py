"""Thin ctypes binding to libb200rt.so (include/rt.h). Argument marshalling only: every step of
the ray-tracing path runs in the library's CUDA kernels. There is no CPU fallback — if the
library is missing or a call fails, this module raises.

Buffers may be torch tensors (device memory; PyTorch is used for allocation and streams) or
numpy arrays (host memory; the library stages through the device and copies back).
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B200RT_LIB", os.path.join(HERE, "libb200rt.so"))  # override: A/B builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "rt.h")

RT_OK = 0
STATUS = {0: "RT_OK", -1: "RT_ERR_INVALID_ARG", -2: "RT_ERR_NO_SCENE", -3: "RT_ERR_NO_CAMERA",
          -4: "RT_ERR_CUDA", -5: "RT_ERR_OOM", -6: "RT_ERR_STATE", -7: "RT_ERR_PARSE", -8: "RT_ERR_IO"}
TILE_W, TILE_H = 8, 4

PRIM_DTYPE = np.dtype([("type", "<u4"), ("material", "<u4"), ("p", "<f4", (4,))])
MAT_DTYPE = np.dtype([("kind", "<u4"), ("albedo", "<f4", (3,)), ("emission", "<f4", (3,)), ("ior", "<f4"),
                      ("ks", "<f4"), ("shininess", "<f4"), ("kr", "<f4"), ("_pad", "<f4")])
LIGHT_DTYPE = np.dtype([("position", "<f4", (3,)), ("intensity", "<f4", (3,))])
ENV_DTYPE = np.dtype([("background", "<f4", (3,)), ("ambient", "<f4", (3,))])
assert PRIM_DTYPE.itemsize == 24 and MAT_DTYPE.itemsize == 48 and LIGHT_DTYPE.itemsize == 24


class RtError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class RayStats(C.Structure):
    _fields_ = [("primary", C.c_uint64), ("shadow", C.c_uint64), ("secondary", C.c_uint64),
                ("sphere_tests", C.c_uint64), ("plane_tests", C.c_uint64), ("last_render_ms", C.c_double),
                ("closest_sphere_tests", C.c_uint64), ("isect_closest_ms", C.c_double),
                ("isect_shadow_ms", C.c_double), ("launches", C.c_uint32), ("variant", C.c_int32),
                ("shade_ms", C.c_double), ("isect_eye_ms", C.c_double), ("graph", C.c_int32), ("_pad", C.c_int32),
                ("accumulate_ms", C.c_double)]


_lib = None


def declared_functions() -> list[str]:
    """Names of every function declared in include/rt.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rt_[a-z0-9_]+)\s*\(", src)))


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python paper_1504_03151_b200/build.py` "
                           "(no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "rt_scene_upload": [vp, i32, vp, i32, vp, i32, vp],
        "rt_camera_set": [vp, vp, vp, C.c_float],
        "rt_render": [i32, i32, i32, i32, vp],
        "rt_stats": [C.POINTER(RayStats)],
        "rt_set_stream": [vp],
        "rt_set_seed": [C.c_uint64],
        "rt_set_variant": [i32],
        "rt_shard_layout": [i32, i32, i32, C.POINTER(i32), C.POINTER(i64)],
        "rt_render_shard": [i32, i32, i32, i32, i32, i32, vp],
        "rt_assemble_tiles": [vp, i32, i32, i32, vp],
        "rt_render_debug": [i32, i32, i32, i32, vp, vp, vp],
        "rt_tonemap_rgba8": [vp, vp, i64, C.c_float, C.c_float],
        "rt_set_integrator": [i32, i32],
        "rt_set_concurrency": [i32],
        "rt_set_pipeline": [i32],
        "rt_set_tiled_scan": [i32],
        "rt_set_schedule_jitter": [C.c_uint64],
        "rt_check_status": [C.POINTER(C.c_uint32), C.POINTER(i32)],
        "rt_set_graphs": [i32],
        "rt_set_scan_split": [i32],
        "rt_render_shard_direct": [i32, i32, i32, i32, i32, i32, vp, vp],
        "rt_sum_shard_stats": [vp, i32],
        "rt_ipc_alloc": [i64, C.POINTER(vp), C.c_char_p],
        "rt_ipc_open": [C.c_char_p, C.POINTER(vp)],
        "rt_ipc_close": [vp],
        "rt_ipc_free": [vp],
        "rt_scene_parse": [C.c_char_p, i64],
        "rt_scene_load": [C.c_char_p],
        "rt_write_ppm": [vp, i32, i32, C.c_float, C.c_float, C.c_char_p],
        "rt_render_passes": [i32, i32, i32, i64, i32, vp, vp],
        "rt_render_passes_debug": [i32, i32, i32, i64, i32, vp, vp, vp, vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.rt_last_error.argtypes = []
    L.rt_last_error.restype = C.c_char_p
    _lib = L
    return L


def _check(fn: str, rc: int):
    if rc != RT_OK:
        raise RtError(fn, rc, lib().rt_last_error().decode(errors="replace"))


def _ptr(buf) -> int:
    """Raw address of a torch tensor or numpy array (marshalling only)."""
    if hasattr(buf, "data_ptr"):
        if not buf.is_contiguous():
            raise ValueError("buffer must be contiguous")
        return buf.data_ptr()
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("buffer must be C-contiguous")
        return buf.ctypes.data
    raise TypeError(f"unsupported buffer type {type(buf)}")


# ---- scene marshalling (scenegen.Scene -> C structs) ------------------------------------------
def pack_scene(sc):
    prims = np.zeros(sc.n_prims, PRIM_DTYPE)
    prims["type"] = sc.prim_type
    prims["material"] = sc.prim_mat
    prims["p"] = sc.prim_p
    mats = np.zeros(len(sc.mat_kind), MAT_DTYPE)
    mats["kind"] = sc.mat_kind
    mats["albedo"] = sc.mat_albedo
    mats["emission"] = sc.mat_emission
    mats["ior"] = sc.mat_ior
    mats["ks"] = sc.mat_ks
    mats["shininess"] = sc.mat_shininess
    mats["kr"] = sc.mat_kr
    lights = np.zeros(sc.n_lights, LIGHT_DTYPE)
    lights["position"] = sc.light_pos
    lights["intensity"] = sc.light_intensity
    env = np.zeros(1, ENV_DTYPE)
    env["background"] = sc.background
    env["ambient"] = sc.ambient
    return prims, mats, lights, env


def scene_upload(prims, mats, lights, env=None):
    _check("rt_scene_upload", lib().rt_scene_upload(
        prims.ctypes.data if len(prims) else None, len(prims), mats.ctypes.data, len(mats),
        lights.ctypes.data if len(lights) else None, len(lights), env.ctypes.data if env is not None else None))


def camera_set(eye, look_at, up, vfov_deg: float):
    e, l, u = (np.ascontiguousarray(v, np.float32) for v in (eye, look_at, up))
    _check("rt_camera_set", lib().rt_camera_set(e.ctypes.data, l.ctypes.data, u.ctypes.data, float(vfov_deg)))


def set_seed(seed: int):
    _check("rt_set_seed", lib().rt_set_seed(int(seed)))


VARIANTS = {"auto": -1, "megakernel": 0, "wavefront": 1}


def set_variant(name: str):
    """Kernel organisation: "auto" (default), "wavefront" or "megakernel" (bit-identical results)."""
    _check("rt_set_variant", lib().rt_set_variant(VARIANTS[name]))


def set_concurrency(on: bool):
    """Wavefront: shadow scans concurrent with the next closest scan (default) or all in order."""
    _check("rt_set_concurrency", lib().rt_set_concurrency(1 if on else 0))


def set_tiled_scan(on: bool):
    """Scenes beyond shared memory: scans over TMA-loaded tiles (default) or global loads."""
    _check("rt_set_tiled_scan", lib().rt_set_tiled_scan(1 if on else 0))


def set_schedule_jitter(seed: int = 0):
    """Test support: random spin kernels at every stream fork/join of plain launches (0 = off)."""
    _check("rt_set_schedule_jitter", lib().rt_set_schedule_jitter(int(seed)))


def check_status() -> tuple[int, bool]:
    """Test support: (id of the first failed device check since the last call or 0, checks compiled)."""
    v, c = C.c_uint32(), C.c_int32()
    _check("rt_check_status", lib().rt_check_status(C.byref(v), C.byref(c)))
    return int(v.value), bool(c.value)


def set_pipeline(slots: int = 0):
    """Wavefront: chunk pipelining over 1..4 buffer-set slots; 0 = AUTO (the default: 2, or 3 for
    frames of >= 8 chunks)."""
    _check("rt_set_pipeline", lib().rt_set_pipeline(int(slots)))


def set_graphs(on: bool):
    """Wavefront: replay a CUDA graph of the launch sequence for repeated identical renders (default)."""
    _check("rt_set_graphs", lib().rt_set_graphs(1 if on else 0))


def set_scan_split(parts: int = -1):
    """Wavefront scans: -1 split short queues only (default); 1/2/4/8 force that many parts."""
    _check("rt_set_scan_split", lib().rt_set_scan_split(int(parts)))


def set_stream(stream):
    """stream: torch.cuda.Stream, a raw cudaStream_t int, or None (default stream)."""
    h = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    _check("rt_set_stream", lib().rt_set_stream(h))


def load_scene(sc):
    """Upload a scenegen.Scene and set its camera and seed (the usual three calls)."""
    scene_upload(*pack_scene(sc))
    camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)
    set_seed(sc.seed)


def render(width: int, height: int, max_depth: int, spp: int, out):
    """out: float32 buffer of width*height*4 (torch CUDA tensor or numpy host array)."""
    _check("rt_render", lib().rt_render(width, height, max_depth, spp, _ptr(out)))
    return out


def render_debug(width, height, max_depth, spp, out, hit_ids, bounces):
    _check("rt_render_debug", lib().rt_render_debug(width, height, max_depth, spp, _ptr(out), _ptr(hit_ids),
                                                    _ptr(bounces)))
    return out, hit_ids, bounces


def scene_parse(text):
    """NEXT-4: parse scene text (grammar in include/rt.h), upload it and set its camera."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    _check("rt_scene_parse", lib().rt_scene_parse(b, len(b)))


def scene_load(path: str):
    _check("rt_scene_load", lib().rt_scene_load(os.fsencode(path)))


def write_ppm(rgba, width: int, height: int, path: str, exposure: float = 1.0, gamma: float = 2.2):
    """rgba: float32 CUDA tensor of width*height*4 (tone-mapped on the device)."""
    _check("rt_write_ppm", lib().rt_write_ppm(_ptr(rgba), width, height, exposure, gamma, os.fsencode(path)))


INTEGRATORS = {"whitted": 0, "global": 1}


def set_integrator(name: str = "whitted", area_lights: bool = False):
    """NEXT-1 / NEXT-2 (include/rt.h rt_set_integrator): "whitted" (the hot path) or "global"
    (cosine-weighted diffuse bounce); area_lights samples every emissive sphere as a light."""
    _check("rt_set_integrator", lib().rt_set_integrator(INTEGRATORS[name], 1 if area_lights else 0))


def render_passes(width, height, max_depth, pass_begin, n_passes, accum, out=None):
    """Progressive passes: accum (float64 CUDA tensor [H, W, 3], zeroed before pass 0) += the
    radiance of passes pass_begin .. pass_begin + n_passes - 1; out (optional) = the mean."""
    _check("rt_render_passes", lib().rt_render_passes(width, height, max_depth, int(pass_begin), n_passes,
                                                      _ptr(accum), _ptr(out) if out is not None else None))
    return accum


def render_passes_debug(width, height, max_depth, pass_begin, n_passes, accum, out, hit_ids, bounces):
    _check("rt_render_passes_debug", lib().rt_render_passes_debug(
        width, height, max_depth, int(pass_begin), n_passes, _ptr(accum), _ptr(out), _ptr(hit_ids), _ptr(bounces)))
    return accum, out, hit_ids, bounces


def stats() -> dict:
    s = RayStats()
    _check("rt_stats", lib().rt_stats(C.byref(s)))
    return {k: getattr(s, k) for k, _ in RayStats._fields_}


def shard_layout(width, height, world):
    tpr, sb = C.c_int32(), C.c_int64()
    _check("rt_shard_layout", lib().rt_shard_layout(width, height, world, C.byref(tpr), C.byref(sb)))
    return tpr.value, sb.value


def render_shard(width, height, max_depth, spp, rank, world, slab):
    _check("rt_render_shard", lib().rt_render_shard(width, height, max_depth, spp, rank, world, _ptr(slab)))
    return slab


def render_shard_direct(width, height, max_depth, spp, rank, world, frame_ptr: int, records_ptr: int):
    """Fused render + gather: this rank's pixels go straight into the (peer) frame (rt.h)."""
    _check("rt_render_shard_direct", lib().rt_render_shard_direct(width, height, max_depth, spp, rank, world,
                                                                  frame_ptr, records_ptr))


def sum_shard_stats(records_ptr: int, world: int):
    _check("rt_sum_shard_stats", lib().rt_sum_shard_stats(records_ptr, world))


def ipc_alloc(nbytes: int) -> tuple[int, bytes]:
    ptr, h = C.c_void_p(), C.create_string_buffer(64)
    _check("rt_ipc_alloc", lib().rt_ipc_alloc(nbytes, C.byref(ptr), h))
    return ptr.value, h.raw


def ipc_open(handle: bytes) -> int:
    ptr = C.c_void_p()
    _check("rt_ipc_open", lib().rt_ipc_open(C.create_string_buffer(bytes(handle), 64), C.byref(ptr)))
    return ptr.value


def ipc_close(ptr: int):
    _check("rt_ipc_close", lib().rt_ipc_close(ptr))


def ipc_free(ptr: int):
    _check("rt_ipc_free", lib().rt_ipc_free(ptr))


class DeviceArray:
    """A raw device allocation seen by torch without a copy (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def assemble_tiles(gathered, width, height, world, out):
    _check("rt_assemble_tiles", lib().rt_assemble_tiles(_ptr(gathered), width, height, world, _ptr(out)))
    return out


def tonemap_rgba8(rgba, out, exposure=1.0, gamma=2.2):
    n = (rgba.numel() if hasattr(rgba, "numel") else rgba.size) // 4
    _check("rt_tonemap_rgba8", lib().rt_tonemap_rgba8(_ptr(rgba), _ptr(out), n, float(exposure), float(gamma)))
    return out
