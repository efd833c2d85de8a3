"""Seeded synthetic scene generator shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO ray-tracing arithmetic (no intersection, shading, camera or bounce math):
it only draws scene parameters from a counter-based generator and packs them into float32
arrays. Both sides of every parity check (``oracle/`` and the CUDA library) consume the exact
float32 values produced here.

Workloads follow BASELINE.json ``configs`` (BJ:7-11) with the recipes of SURVEY.md §8(d).1:
  C1  64x64, 3 spheres + ground plane, 1 point light, max_depth 1, 1 spp (hand-authored)
  C2  512x512, 10 spheres + plane, 2 lights, reflective materials, max_depth 3, 1 spp
  C3  1920x1080, 100 spheres + 2 planes, 4 lights, reflection + refraction, max_depth 5, 1 spp
  C4  1920x1080, 1000 random spheres, 8 lights, max_depth 5, 4 spp
  C5  3840x2160, 1000 spheres + 2 planes, 8 lights, max_depth 8, 16 spp
The paper's own scene ("provided by David Bucciarelli") is not recoverable;
these are sphere/plane scenes shaped like the paper's workload (spheres only).

Primitive convention (shared input contract, not method arithmetic):
  type 0 = sphere, p = (cx, cy, cz, radius)
  type 1 = plane,  p = (nx, ny, nz, d) with unit n and n.x = d
Planes are emitted before spheres so that index order == "planes first" order (except
``build(keep_order=True)`` / ``random_tiny(interleave=True)``: interleaved-order parity cases).
Material kinds: 0 DIFFUSE, 1 SPECULAR, 2 REFRACTIVE.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
import numpy as np

SPHERE, PLANE = 0, 1
DIFFUSE, SPECULAR, REFRACTIVE = 0, 1, 2

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


class SplitMix64:
    """Counter-based splitmix64 stream used only to draw scene parameters."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + _GOLDEN) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = (self.next_u64() >> 40) * (1.0 / (1 << 24))
        return lo + (hi - lo) * u


@dataclass
class Scene:
    name: str
    prim_type: np.ndarray        # int32 [N]
    prim_mat: np.ndarray         # int32 [N]
    prim_p: np.ndarray           # float32 [N,4]
    mat_kind: np.ndarray         # int32 [M]
    mat_albedo: np.ndarray       # float32 [M,3]
    mat_emission: np.ndarray     # float32 [M,3]
    mat_ior: np.ndarray          # float32 [M]
    mat_ks: np.ndarray           # float32 [M]
    mat_shininess: np.ndarray    # float32 [M]
    mat_kr: np.ndarray           # float32 [M]
    light_pos: np.ndarray        # float32 [L,3]
    light_intensity: np.ndarray  # float32 [L,3]
    background: np.ndarray       # float32 [3]
    ambient: np.ndarray          # float32 [3]
    eye: np.ndarray              # float32 [3]
    look_at: np.ndarray          # float32 [3]
    up: np.ndarray               # float32 [3]
    vfov: float                  # degrees (stored as an exact float32 value)
    width: int
    height: int
    max_depth: int
    spp: int
    seed: int = 0
    notes: str = field(default="")

    @property
    def n_prims(self) -> int:
        return int(self.prim_type.shape[0])

    @property
    def n_spheres(self) -> int:
        return int((self.prim_type == SPHERE).sum())

    @property
    def n_planes(self) -> int:
        return int((self.prim_type == PLANE).sum())

    @property
    def n_lights(self) -> int:
        return int(self.light_pos.shape[0])

    def with_frame(self, width=None, height=None, max_depth=None, spp=None, seed=None) -> "Scene":
        return replace(self,
                       width=self.width if width is None else int(width),
                       height=self.height if height is None else int(height),
                       max_depth=self.max_depth if max_depth is None else int(max_depth),
                       spp=self.spp if spp is None else int(spp),
                       seed=self.seed if seed is None else int(seed))

    def describe(self) -> dict:
        return {"workload": self.name, "width": self.width, "height": self.height,
                "max_depth": self.max_depth, "spp": self.spp, "spheres": self.n_spheres,
                "planes": self.n_planes, "lights": self.n_lights}


class _Builder:
    def __init__(self):
        self.prims = []   # (type, mat, p4)
        self.mats = []    # dict
        self.lights = []  # (pos3, I3)

    def material(self, kind, albedo, emission=(0, 0, 0), ior=1.0, ks=0.0, shininess=1.0, kr=0.0) -> int:
        self.mats.append(dict(kind=kind, albedo=albedo, emission=emission, ior=ior, ks=ks,
                              shininess=shininess, kr=kr))
        return len(self.mats) - 1

    def plane(self, n, d, mat):
        self.prims.append((PLANE, mat, (n[0], n[1], n[2], d)))

    def sphere(self, c, r, mat):
        self.prims.append((SPHERE, mat, (c[0], c[1], c[2], r)))

    def light(self, pos, intensity):
        self.lights.append((pos, intensity))

    def build(self, name, eye, look_at, up, vfov, width, height, max_depth, spp,
              background=(0, 0, 0), ambient=(0, 0, 0), seed=0, notes="", keep_order=False) -> Scene:
        # planes first (stable) by default, so index order equals the "planes, then spheres" order
        # of the generated configs; keep_order=True keeps the insertion order (interleaved
        # sphere/plane indices: tie-break and test-count parity cases)
        if keep_order:
            prims = list(self.prims)
        else:
            prims = [p for p in self.prims if p[0] == PLANE] + [p for p in self.prims if p[0] == SPHERE]
        f32 = np.float32
        m = self.mats
        L = self.lights
        return Scene(
            name=name,
            prim_type=np.array([p[0] for p in prims], dtype=np.int32),
            prim_mat=np.array([p[1] for p in prims], dtype=np.int32),
            prim_p=np.array([p[2] for p in prims], dtype=f32).reshape(-1, 4),
            mat_kind=np.array([x["kind"] for x in m], dtype=np.int32),
            mat_albedo=np.array([x["albedo"] for x in m], dtype=f32).reshape(-1, 3),
            mat_emission=np.array([x["emission"] for x in m], dtype=f32).reshape(-1, 3),
            mat_ior=np.array([x["ior"] for x in m], dtype=f32),
            mat_ks=np.array([x["ks"] for x in m], dtype=f32),
            mat_shininess=np.array([x["shininess"] for x in m], dtype=f32),
            mat_kr=np.array([x["kr"] for x in m], dtype=f32),
            light_pos=np.array([l[0] for l in L], dtype=f32).reshape(-1, 3),
            light_intensity=np.array([l[1] for l in L], dtype=f32).reshape(-1, 3),
            background=np.array(background, dtype=f32),
            ambient=np.array(ambient, dtype=f32),
            eye=np.array(eye, dtype=f32), look_at=np.array(look_at, dtype=f32),
            up=np.array(up, dtype=f32), vfov=float(np.float32(vfov)),
            width=int(width), height=int(height), max_depth=int(max_depth), spp=int(spp),
            seed=int(seed), notes=notes)


def _f32(x: float) -> float:
    return float(np.float32(x))


def _no_overlap(c, r, placed, pad=0.05):
    for (c2, r2) in placed:
        dx, dy, dz = c[0] - c2[0], c[1] - c2[1], c[2] - c2[2]
        if dx * dx + dy * dy + dz * dz < (r + r2 + pad) ** 2:
            return False
    return True


def config_c1() -> Scene:
    """BJ:7 — hand-authored 64x64 scene, SURVEY.md §8(d).1 row C1."""
    b = _Builder()
    ground = b.material(DIFFUSE, (0.8, 0.8, 0.8))
    b.plane((0, 1, 0), 0.0, ground)
    b.sphere((-1.25, 1, 0), 1.0, b.material(DIFFUSE, (0.9, 0.2, 0.2), ks=0.5, shininess=32))
    b.sphere((1.25, 1, 0), 1.0, b.material(SPECULAR, (0.9, 0.9, 0.9)))
    b.sphere((0, 0.5, -1.5), 0.5, b.material(REFRACTIVE, (1, 1, 1), ior=1.5))
    b.light((3, 5, -3), (60, 60, 60))
    return b.build("C1", eye=(0, 1, -4), look_at=(0, 1, 0), up=(0, 1, 0), vfov=60,
                   width=64, height=64, max_depth=1, spp=1,
                   background=(0.2, 0.3, 0.5), ambient=(0.05, 0.05, 0.05))


def config_c2(seed: int = 2) -> Scene:
    """BJ:8 — 512x512, 10 spheres + plane, 2 lights, reflective materials, depth 3."""
    g = SplitMix64(seed)
    b = _Builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.75, 0.75, 0.7), ks=0.1, shininess=8))
    placed = []
    while len(placed) < 10:
        r = _f32(g.uniform(0.4, 1.2))
        c = (_f32(g.uniform(-6, 6)), r, _f32(g.uniform(-2, 10)))
        if not _no_overlap(c, r, placed):
            continue
        k = len(placed) % 3
        col = (_f32(g.uniform(0.3, 1)), _f32(g.uniform(0.3, 1)), _f32(g.uniform(0.3, 1)))
        if k == 0:
            a = _f32(g.uniform(0.7, 1.0))
            m = b.material(SPECULAR, (a, a, a))
        elif k == 1:
            m = b.material(DIFFUSE, col, ks=0.3, shininess=64, kr=0.5)
        else:
            m = b.material(DIFFUSE, col, ks=0.2, shininess=16)
        b.sphere(c, r, m)
        placed.append((c, r))
    for sx in (-6, 6):
        I = _f32(g.uniform(80, 150))
        b.light((sx, 8, -4), (I, I, I))
    return b.build("C2", eye=(0, 3, -8), look_at=(0, 1, 4), up=(0, 1, 0), vfov=50,
                   width=512, height=512, max_depth=3, spp=1,
                   background=(0.1, 0.12, 0.2), ambient=(0.03, 0.03, 0.03), seed=0)


def _mixed_material(b: _Builder, g: SplitMix64, kr_diffuse: float, refr_lo=1.3, refr_hi=1.8) -> int:
    """50% DIFFUSE (half with kr), 25% SPECULAR, 25% REFRACTIVE."""
    u = g.uniform()
    col = (_f32(g.uniform(0.2, 1)), _f32(g.uniform(0.2, 1)), _f32(g.uniform(0.2, 1)))
    if u < 0.25:
        return b.material(DIFFUSE, col, ks=_f32(g.uniform(0, 0.5)), shininess=_f32(g.uniform(4, 64)))
    if u < 0.5:
        return b.material(DIFFUSE, col, ks=_f32(g.uniform(0, 0.5)), shininess=_f32(g.uniform(4, 64)),
                          kr=kr_diffuse)
    if u < 0.75:
        a = _f32(g.uniform(0.7, 0.98))
        return b.material(SPECULAR, (a, a, a))
    return b.material(REFRACTIVE, (1, 1, 1), ior=_f32(g.uniform(refr_lo, refr_hi)))


def config_c3(seed: int = 3) -> Scene:
    """BJ:9 — 1920x1080, 100 spheres + planes, 4 lights, reflection + refraction, depth 5."""
    g = SplitMix64(seed)
    b = _Builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.7, 0.7, 0.7)))
    b.plane((0, 0, -1), -40.0, b.material(DIFFUSE, (0.6, 0.65, 0.8), ks=0.2, shininess=16))
    placed = []
    while len(placed) < 100:
        r = _f32(g.uniform(0.3, 1.5))
        c = (_f32(g.uniform(-15, 15)), r, _f32(g.uniform(0, 35)))
        if not _no_overlap(c, r, placed):
            continue
        b.sphere(c, r, _mixed_material(b, g, 0.3))
        placed.append((c, r))
    for _ in range(4):
        I = _f32(g.uniform(200, 400))
        b.light((_f32(g.uniform(-15, 15)), _f32(g.uniform(8, 15)), _f32(g.uniform(-5, 30))), (I, I, I))
    return b.build("C3", eye=(0, 4, -12), look_at=(0, 1, 15), up=(0, 1, 0), vfov=55,
                   width=1920, height=1080, max_depth=5, spp=1,
                   background=(0.05, 0.07, 0.12), ambient=(0.02, 0.02, 0.02))


def config_c4(seed: int = 4) -> Scene:
    """BJ:10 — 1920x1080, 1000 random spheres (overlaps allowed), 8 lights, depth 5, 4 spp."""
    g = SplitMix64(seed)
    b = _Builder()
    spheres = []
    for _ in range(1000):
        c = (_f32(g.uniform(-30, 30)), _f32(g.uniform(-15, 15)), _f32(g.uniform(10, 70)))
        r = _f32(g.uniform(0.3, 1.2))
        u = g.uniform()
        col = (_f32(g.uniform(0.2, 1)), _f32(g.uniform(0.2, 1)), _f32(g.uniform(0.2, 1)))
        if u < 0.4:
            m = b.material(DIFFUSE, col, ks=_f32(g.uniform(0, 0.4)), shininess=_f32(g.uniform(4, 48)))
        elif u < 0.6:
            m = b.material(DIFFUSE, col, ks=_f32(g.uniform(0, 0.4)), shininess=_f32(g.uniform(4, 48)), kr=0.4)
        elif u < 0.8:
            a = _f32(g.uniform(0.7, 0.98))
            m = b.material(SPECULAR, (a, a, a))
        else:
            m = b.material(REFRACTIVE, (1, 1, 1), ior=_f32(g.uniform(1.3, 1.8)))
        b.sphere(c, r, m)
        spheres.append((c, r))
    n_l = 0
    while n_l < 8:
        p = (_f32(g.uniform(-30, 30)), _f32(g.uniform(-15, 15)), _f32(g.uniform(10, 70)))
        if not _no_overlap(p, 0.0, spheres, pad=0.2):
            continue
        I = _f32(g.uniform(100, 300))
        b.light(p, (I, I, I))
        n_l += 1
    return b.build("C4", eye=(0, 0, 0), look_at=(0, 0, 1), up=(0, 1, 0), vfov=60,
                   width=1920, height=1080, max_depth=5, spp=4,
                   background=(0.15, 0.18, 0.25), ambient=(0.02, 0.02, 0.02))


def config_c5(seed: int = 5) -> Scene:
    """BJ:11 — 3840x2160, 1000 spheres + 2 planes, 8 lights, depth 8, 16 spp."""
    g = SplitMix64(seed)
    b = _Builder()
    b.plane((0, 1, 0), 0.0, b.material(DIFFUSE, (0.7, 0.7, 0.7)))
    b.plane((0, 0, -1), -100.0, b.material(DIFFUSE, (0.6, 0.65, 0.8), ks=0.2, shininess=16))
    placed = []
    while len(placed) < 1000:
        r = _f32(g.uniform(0.3, 1.5))
        c = (_f32(g.uniform(-40, 40)), r, _f32(g.uniform(0, 90)))
        if not _no_overlap(c, r, placed):
            continue
        b.sphere(c, r, _mixed_material(b, g, 0.3))
        placed.append((c, r))
    for _ in range(8):
        I = _f32(g.uniform(200, 400))
        b.light((_f32(g.uniform(-40, 40)), _f32(g.uniform(8, 20)), _f32(g.uniform(-5, 80))), (I, I, I))
    return b.build("C5", eye=(0, 6, -20), look_at=(0, 1, 40), up=(0, 1, 0), vfov=55,
                   width=3840, height=2160, max_depth=8, spp=16,
                   background=(0.05, 0.07, 0.12), ambient=(0.02, 0.02, 0.02))


def config_c0() -> Scene:
    """Paper-shaped workload for NEXT-1 / NEXT-2 (SURVEY §8(d).1 "C0", §8(f) NEXT-2): a Cornell
    box of 5 planes + 3 spheres + 1 spherical area light at 640x480, depth 6 (P:241, P:275,
    P:290), rendered with the global integrator and area lights in progressive passes. No point
    lights, no ambient, black background: all light comes from the emitter."""
    b = _Builder()
    white = b.material(DIFFUSE, (0.75, 0.75, 0.75))
    red = b.material(DIFFUSE, (0.75, 0.25, 0.25))
    green = b.material(DIFFUSE, (0.25, 0.75, 0.25))
    b.plane((0, 1, 0), 0.0, white)      # floor y = 0
    b.plane((0, -1, 0), -5.0, white)    # ceiling y = 5
    b.plane((1, 0, 0), -2.5, red)       # left wall x = -2.5
    b.plane((-1, 0, 0), -2.5, green)    # right wall x = 2.5
    b.plane((0, 0, -1), -5.0, white)    # back wall z = 5
    b.sphere((-1.1, 0.9, 3.2), 0.9, b.material(SPECULAR, (0.95, 0.95, 0.95)))
    b.sphere((1.1, 0.9, 2.0), 0.9, b.material(REFRACTIVE, (1.0, 1.0, 1.0), ior=1.5))
    b.sphere((0.6, 0.5, 4.2), 0.5, b.material(DIFFUSE, (0.6, 0.6, 0.9), ks=0.3, shininess=32.0))
    b.sphere((0.0, 4.3, 2.8), 0.4, b.material(DIFFUSE, (0.0, 0.0, 0.0), emission=(25.0, 25.0, 25.0)))
    return b.build("C0", eye=(0, 2.5, -6.5), look_at=(0, 2.5, 0), up=(0, 1, 0), vfov=45,
                   width=640, height=480, max_depth=6, spp=1, background=(0, 0, 0), ambient=(0, 0, 0),
                   notes="Cornell box; render with integrator=global, area_lights=1, progressive passes")


CONFIGS = {"C0": config_c0, "C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}


def get(name: str) -> Scene:
    return CONFIGS[name.upper()]()


def random_tiny(seed: int, n_spheres: int = 6, n_planes: int = 1, n_lights: int = 2,
                width: int = 12, height: int = 9, max_depth: int = 3, spp: int = 1,
                n_emitters: int = 0, glass_tint: bool = False, interleave: bool = False) -> Scene:
    """Tiny random scenes for brute-force and randomized parity tests (all material kinds).
    glass_tint: REFRACTIVE materials get a random albedo in [0.3, 1]^3 instead of (1, 1, 1) (the
    glass weight T *= rho, is then visible). interleave: the planes are inserted between
    the spheres and the primitive order is kept (plane indices interleaved with sphere indices)."""
    g = SplitMix64(0xC0FFEE ^ seed)
    b = _Builder()

    def material():
        m = _mixed_material(b, g, 0.5)
        if glass_tint and b.mats[m]["kind"] == REFRACTIVE:
            b.mats[m]["albedo"] = (_f32(g.uniform(0.3, 1)), _f32(g.uniform(0.3, 1)), _f32(g.uniform(0.3, 1)))
        return m

    def add_planes():
        for i in range(n_planes):
            if i == 0:
                b.plane((0, 1, 0), 0.0, material())
            else:
                b.plane((0, 0, -1), -12.0, material())

    if not interleave:
        add_planes()
    for k in range(n_spheres):
        if interleave and k == n_spheres // 2:
            add_planes()
        r = _f32(g.uniform(0.3, 1.5))
        c = (_f32(g.uniform(-4, 4)), _f32(g.uniform(0.2, 3)), _f32(g.uniform(2, 9)))
        b.sphere(c, r, material())
    if interleave and n_spheres == 0:
        add_planes()
    for _ in range(n_emitters):  # spherical area lights (NEXT-1): emissive DIFFUSE spheres
        r = _f32(g.uniform(0.2, 0.6))
        c = (_f32(g.uniform(-4, 4)), _f32(g.uniform(3, 6)), _f32(g.uniform(1, 8)))
        le = _f32(g.uniform(5, 20))
        b.sphere(c, r, b.material(DIFFUSE, (_f32(g.uniform(0, 0.5)),) * 3, emission=(le, le * 0.9, le * 0.7)))
    for _ in range(n_lights):
        I = _f32(g.uniform(20, 80))
        b.light((_f32(g.uniform(-5, 5)), _f32(g.uniform(4, 8)), _f32(g.uniform(-2, 6))), (I, I * 0.9, I * 0.8))
    return b.build(f"tiny{seed}", eye=(0, 2, -6), look_at=(0, 1, 5), up=(0, 1, 0), vfov=55,
                   width=width, height=height, max_depth=max_depth, spp=spp,
                   background=(0.1, 0.2, 0.3), ambient=(0.03, 0.03, 0.03), seed=seed, keep_order=interleave)


_KIND_NAMES = {DIFFUSE: "diffuse", SPECULAR: "specular", REFRACTIVE: "refractive"}


def _g(x) -> str:
    """float32 value as the shortest decimal that round-trips through strtof (%.9g)."""
    return "%.9g" % float(np.float32(x))


def to_text(sc: Scene) -> str:
    """Scene -> the text format of include/rt.h (rt_scene_parse; SPEC S:246-249 grammar extended
    with planes, point lights and environment). Every value is printed so that strtof returns the
    same float32, so parsing the text reproduces the scene exactly (one material per primitive)."""
    out = [f"# {sc.name}: {sc.notes}".rstrip(": ") if sc.notes else f"# {sc.name}",
           "camera " + "  ".join(" ".join(_g(v) for v in vec) for vec in (sc.eye, sc.look_at, sc.up)) + "  " + _g(sc.vfov),
           "background " + " ".join(_g(v) for v in sc.background),
           "ambient " + " ".join(_g(v) for v in sc.ambient)]
    for p, I in zip(sc.light_pos, sc.light_intensity):
        out.append("light " + " ".join(_g(v) for v in p) + "  " + " ".join(_g(v) for v in I))
    for t, m, q in zip(sc.prim_type, sc.prim_mat, sc.prim_p):
        geo = (f"sphere {_g(q[3])}  {_g(q[0])} {_g(q[1])} {_g(q[2])}" if t == SPHERE
               else f"plane {_g(q[0])} {_g(q[1])} {_g(q[2])} {_g(q[3])}")
        kind = int(sc.mat_kind[m])
        mat = (" ".join(_g(v) for v in sc.mat_emission[m]) + "  " + " ".join(_g(v) for v in sc.mat_albedo[m])
               + "  " + _KIND_NAMES[kind])
        if kind == REFRACTIVE:
            mat += " " + _g(sc.mat_ior[m])
        mat += f" ks={_g(sc.mat_ks[m])} shininess={_g(sc.mat_shininess[m])} kr={_g(sc.mat_kr[m])}"
        out.append(geo + "  " + mat)
    return "\n".join(out) + "\n"


def builder() -> _Builder:
    """Hand-authoring entry point for worked examples in tests."""
    return _Builder()
