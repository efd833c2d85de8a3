"""Debug aid for the NEXT-1/NEXT-2 modes: C0 (or a tiny random scene) with the global integrator
and area lights at a few frame sizes; prints the parity report and the 8-bit offenders with
their per-sample hit ids on both sides (test tooling, not product code)."""
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
    ap.add_argument("--sizes", default="56x42,80x60,128x96")
    ap.add_argument("--spp", type=int, default=2)
    ap.add_argument("--top", type=int, default=6)
    a = ap.parse_args()
    okw = dict(integrator=1, area_lights=1)
    for wh in a.sizes.split(","):
        W, H = map(int, wh.split("x"))
        sc = scenegen.get("C0").with_frame(width=W, height=H, spp=a.spp)
        g = gpu_render(sc, integrator="global", area_lights=True)
        ref = po.render(sc, **okw)
        cls = parity.classify(po, sc, ref, None, **okw)
        rep = parity.compare(g["rgb"], g["ids"], g["bounces"], ref, cls)
        print(f"C0 {W}x{H} spp{a.spp}: {rep}  margin_ok={cls.margin_ok.mean():.3f} cond_ok={cls.cond_ok.mean():.3f}")
        d8 = np.abs(parity.tonemap8(g["rgb"]) - parity.tonemap8(ref.rgb)).max(1)
        bad = np.nonzero(d8 > 1)[0]
        for i in bad[: a.top]:
            same = (g["ids"][i] == ref.hit_ids[i]).all(axis=1)
            print(f"  pix {i % W},{i // W} d8={d8[i]} margin={ref.margin[i].round(8).tolist()} cond={cls.cond_ok[i]} "
                  f"o={ref.rgb[i].round(4).tolist()} g={g['rgb'][i].round(4).tolist()} same_ids_per_sample={same.tolist()}")
            for s in np.nonzero(~same)[0]:
                print(f"     s{s}: o={ref.hit_ids[i, s].tolist()} g={g['ids'][i, s].tolist()}")


if __name__ == "__main__":
    main()
