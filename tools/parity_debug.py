"""Debug aid: render a config on the GPU and print the worst parity offenders (test tooling)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import scenegen  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from tests import parity  # noqa: E402
from tests.gpu_helpers import gpu_render  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="C2")
    ap.add_argument("--n", type=int, default=0, help="sample n pixels (0 = full frame)")
    ap.add_argument("--top", type=int, default=8)
    a = ap.parse_args()
    sc = scenegen.get(a.config)
    g = gpu_render(sc)
    pix = None
    if a.n:
        pix = np.random.default_rng(1).choice(sc.width * sc.height, a.n, replace=False)
    ref = po.render(sc, pixels=pix)
    p = ref.pixels
    cls = parity.classify(po, sc, ref, pix)
    rep = parity.compare(g["rgb"][p], g["ids"][p], g["bounces"][p], ref, cls)
    print(a.config, rep)
    o = ref.rgb
    gg = g["rgb"][p].astype(np.float64)
    rel = (np.abs(gg - o) / (np.abs(o) + 1e-6)).max(1)
    order = np.argsort(-rel * cls.exact)
    for i in order[: a.top]:
        px, py = p[i] % sc.width, p[i] // sc.width
        print(f"pix ({px},{py}) exact={cls.exact[i]} margin={ref.margin[i].min():.3g} rel={rel[i]:.3g} "
              f"o={o[i]} g={gg[i]} ids_o={ref.hit_ids[i].tolist()} ids_g={g['ids'][p[i]].tolist()}")
        sr = po.render(sc, pixels=[p[i]], perturb=parity.PERTURB, perturb_seed=1)
        print(f"   replica rgb={sr.rgb[0]} spread={(np.abs(sr.rgb[0]-o[i])/(np.abs(o[i])+1e-6)).max():.3g}")
    d8 = np.abs(parity.tonemap8(gg) - parity.tonemap8(o)).max(1)
    for i in np.nonzero(d8 > 1)[0][: a.top]:
        px, py = p[i] % sc.width, p[i] // sc.width
        print(f"DIFF8 pix ({px},{py}) d8={d8[i]} exact={cls.exact[i]} margins={np.round(ref.margin[i], 6).tolist()} "
              f"o={np.round(o[i], 5)} g={np.round(gg[i], 5)}")
        for s_ in range(sc.spp):
            print(f"    s{s_}: ids_o={ref.hit_ids[i, s_].tolist()} ids_g={g['ids'][p[i], s_].tolist()} "
                  f"L_o={np.round(ref.sample_rgb[i, s_], 4).tolist()}")
    # histogram of relative errors for exact-class pixels
    ex = cls.exact
    for thr in (1e-7, 1e-6, 1e-5, 3e-5, 1e-4, 3e-4):
        print(f"  exact pixels with rel > {thr:g}: {(rel[ex] > thr).sum()}")


if __name__ == "__main__":
    main()
