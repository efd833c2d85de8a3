"""Parity rule between the CUDA path and the oracle (BASELINE.json
north_star).

Classification (oracle side only):
  * a sample is exact-class when its oracle decision margin (slack of every discrete decision
    divided by that decision's first-order sensitivity, oracle.c *_margin) is >= MARGIN_THR, and
  * the pixel is well-conditioned: Monte Carlo arithmetic replicas of the oracle (every ray origin
    and direction perturbed by a relative PERTURB = 2^-18, i.e. 64 float32 ulps) keep the same hit
    ids and move the radiance by <= COND_REL_THR = the radiance tolerance. A pixel that stays
    within tolerance under 64-ulp perturbations of every ray is insensitive to the float32 path's
    rounding (measured effective error: a few to ~50 ulps after curved mirrors).
  A pixel is exact-class when all its samples are; otherwise it is edge-class.
Pass condition:
  R1  exact-class pixels: hit ids and bounce counts bit-exact; every channel
      |g - o| <= 1e-4 |o| + 1e-6; 8-bit tone-mapped difference <= 1.
  R2  pixels whose 8-bit value differs by more than 1 are at most 0.1 % of the compared pixels
      and all edge-class.
  R3  primary ray counts equal; shadow/secondary totals differ by no more than the ray budget of
      edge-class samples.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MARGIN_THR = 1e-4
PERTURB = 2.0 ** -18
COND_REL_THR = 1e-4
REL_TOL = 1e-4
ABS_TOL = 1e-6
MAX_DIFF_FRAC = 1e-3
MIN_EXACT_ID_FRAC = 0.999  # hit ids + bounce counts bit-exact on >= 99.9 % of all pixels
COUNT_KEYS = ("primary", "shadow", "secondary", "sphere_tests", "plane_tests")


def tonemap8(v):
    """SPEC tone_map, vectorised in float64."""
    x = np.clip(np.asarray(v, np.float64), 0.0, 1.0)
    return np.floor(255.0 * x ** (1.0 / 2.2) + 0.5).astype(np.int32)


@dataclass
class Classified:
    exact: np.ndarray   # [n] bool, exact-class pixels
    margin_ok: np.ndarray
    cond_ok: np.ndarray


def classify(oracle_mod, sc, ref, pixels, n_replicas=2, **okw) -> Classified:
    """okw: the oracle's mode arguments of `ref` (integrator, area_lights, jitter, sample_base,
    spp ...), repeated for the perturbed replicas."""
    margin_ok = (ref.margin >= MARGIN_THR).all(axis=1)
    cond_ok = np.ones(len(ref.rgb), bool)
    for k in range(n_replicas):
        rp = oracle_mod.render(sc, pixels=pixels, perturb=PERTURB, perturb_seed=1 + k, **okw)
        same_ids = (rp.hit_ids == ref.hit_ids).all(axis=(1, 2))
        rel = (np.abs(rp.rgb - ref.rgb) / (np.abs(ref.rgb) + 1e-6)).max(axis=1)
        cond_ok &= same_ids & (rel <= COND_REL_THR)
    return Classified(margin_ok & cond_ok, margin_ok, cond_ok)


@dataclass
class Report:
    n: int
    n_exact: int
    exact_fail: int
    exact_id_fail: int
    exact_rad_fail: int
    exact_8bit_fail: int
    diff8: int
    diff8_exact: int
    max_rel_exact: float
    nan: int

    @property
    def ok(self) -> bool:
        return (self.exact_fail == 0 and self.diff8 <= MAX_DIFF_FRAC * self.n and self.diff8_exact == 0
                and self.nan == 0)

    def __str__(self):
        return (f"n={self.n} exact={self.n_exact} ({self.n_exact / max(self.n, 1):.1%}) exact_fail={self.exact_fail} "
                f"(ids {self.exact_id_fail}, rad {self.exact_rad_fail}, 8bit {self.exact_8bit_fail}) "
                f"diff8={self.diff8} ({self.diff8 / max(self.n, 1):.4%}, exact {self.diff8_exact}) "
                f"max_rel_exact={self.max_rel_exact:.3g} nan={self.nan}")


def compare(g_rgb, g_ids, g_bounces, ref, cls: Classified) -> Report:
    """g_rgb [n,3] float32 (GPU), g_ids [n,spp,D+1], g_bounces [n,spp]; ref = oracle result."""
    o = ref.rgb
    g = np.asarray(g_rgb, np.float64)
    nan = int((~np.isfinite(g)).any(axis=1).sum())
    ids_ok = (np.asarray(g_ids) == ref.hit_ids).all(axis=(1, 2)) & (np.asarray(g_bounces) == ref.bounces).all(axis=1)
    err = np.abs(g - o)
    rad_ok = (err <= REL_TOL * np.abs(o) + ABS_TOL).all(axis=1)
    d8 = np.abs(tonemap8(g) - tonemap8(o)).max(axis=1)
    ok8 = d8 <= 1
    ex = cls.exact
    rel = (err / (np.abs(o) + 1e-30)).max(axis=1)
    return Report(
        n=len(o), n_exact=int(ex.sum()),
        exact_fail=int((ex & ~(ids_ok & rad_ok & ok8)).sum()),
        exact_id_fail=int((ex & ~ids_ok).sum()), exact_rad_fail=int((ex & ~rad_ok).sum()),
        exact_8bit_fail=int((ex & ~ok8).sum()),
        diff8=int((~ok8).sum()), diff8_exact=int((ex & ~ok8).sum()),
        max_rel_exact=float(rel[ex].max()) if ex.any() else 0.0, nan=nan)


def ray_budget_ok(g_stats: dict, ref_counts: dict, ref, cls: Classified, n_lights: int) -> tuple[bool, str]:
    """R3: primary equal; shadow/secondary differences bounded by edge-class samples' budgets."""
    edge_samples = int((~cls.exact).sum()) * ref.hit_ids.shape[1]
    D = ref.hit_ids.shape[2] - 1
    budget_sec = edge_samples * D
    budget_sh = edge_samples * (D + 1) * n_lights
    dp = g_stats["primary"] - ref_counts["primary"]
    ds = g_stats["shadow"] - ref_counts["shadow"]
    dsec = g_stats["secondary"] - ref_counts["secondary"]
    ok = dp == 0 and abs(ds) <= budget_sh and abs(dsec) <= budget_sec
    return ok, f"d_primary={dp} d_shadow={ds} (budget {budget_sh}) d_secondary={dsec} (budget {budget_sec})"


def exact_id_fraction(g_ids, g_bounces, ref) -> float:
    """Fraction of ALL compared pixels (exact- and edge-class) whose hit ids and bounce counts
    equal the oracle's bit for bit (both sides decide in FP64)."""
    ok = (np.asarray(g_ids) == ref.hit_ids).all(axis=(1, 2)) & (np.asarray(g_bounces) == ref.bounces).all(axis=1)
    return float(ok.mean()) if len(ok) else 1.0


def counts_equal(g_stats: dict, ref_counts: dict) -> tuple[bool, str]:
    """Full frames: the algorithmic counts (rays and sphere/plane tests, §8(c).1 step 11; the
    roofline's numerator) equal the oracle's exactly."""
    diff = {k: int(g_stats[k]) - int(ref_counts[k]) for k in COUNT_KEYS}
    return all(v == 0 for v in diff.values()), " ".join(f"d_{k}={v}" for k, v in diff.items())
