"""Command line renderer (SPEC cli_main S:495-504):

    python -m paper_1504_03151_b200 --scene PATH [--width 640 --height 480] [--passes 64]
        [--mode global|local|whitted] [--depth 6] [--seed 0] [--out out.ppm]
        [--snapshot-every K] [--no-area-lights] [--exposure 1] [--gamma 2.2]

Parses the scene (rt_scene_load), renders progressive passes on the GPU (rt_render_passes into a
float64 device buffer), writes the tone-mapped mean image as a binary PPM (rt_write_ppm).
Modes: global = cosine-bounce global illumination (SPEC default), local = direct lighting only
(depth 0), whitted = the §8(a) hot path (mirror / refraction continuation to --depth).
--snapshot-every K writes PATH_passK.ppm after every K passes (the paper's Fig. 5 -> 6
progression); each snapshot is exactly the mean of the passes so far.
Exit codes: 0 ok, 1 usage error, 2 scene parse error, 3 I/O error, 4 device/runtime error.
SPEC's --workers / --bench / --oracle flags belong to its CPU program and are not provided
(the oracle is test infrastructure, never run by the product)."""
from __future__ import annotations

import argparse
import os
import sys

EXIT_OK, EXIT_USAGE, EXIT_PARSE, EXIT_IO, EXIT_RUNTIME = 0, 1, 2, 3, 4


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (argparse's default is 2 = parse error here)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def _args(argv):
    ap = _Parser(prog="python -m paper_1504_03151_b200", description=__doc__,
                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--scene", required=True, help="scene text file (grammar: include/rt.h)")
    ap.add_argument("--width", type=int, default=640)
    ap.add_argument("--height", type=int, default=480)
    ap.add_argument("--passes", type=int, default=64)
    ap.add_argument("--mode", choices=["global", "local", "whitted"], default="global")
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="out.ppm")
    ap.add_argument("--snapshot-every", type=int, default=0)
    ap.add_argument("--no-area-lights", action="store_true")
    ap.add_argument("--exposure", type=float, default=1.0)
    ap.add_argument("--gamma", type=float, default=2.2)
    a = ap.parse_args(argv)
    if a.width < 1 or a.height < 1 or a.passes < 1 or a.depth < 0 or a.snapshot_every < 0 or a.seed < 0:
        ap.error("width, height, passes must be >= 1; depth, snapshot-every, seed >= 0")
    if not (a.exposure > 0 and a.gamma > 0):
        ap.error("exposure and gamma must be > 0")
    return a


def main(argv=None) -> int:
    try:
        a = _args(sys.argv[1:] if argv is None else argv)
    except SystemExit as e:
        return int(e.code or 0)
    from paper_1504_03151_b200 import rt
    try:
        rt.scene_load(a.scene)               # parse + validate before any device work
    except rt.RtError as e:
        sys.stderr.write(f"{e}\n")
        return {-7: EXIT_PARSE, -8: EXIT_IO}.get(e.code, EXIT_RUNTIME)
    try:
        import torch
        if not torch.cuda.is_available():
            raise rt.RtError("cuda", -4, "no CUDA device (the B200 path has no CPU fallback)")
        W, H = a.width, a.height
        depth = 0 if a.mode == "local" else a.depth
        rt.set_seed(a.seed)
        rt.set_integrator("global" if a.mode == "global" else "whitted", not a.no_area_lights)
        accum = torch.zeros((H, W, 3), dtype=torch.float64, device="cuda")
        out = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
        step = a.snapshot_every if a.snapshot_every > 0 else a.passes
        done = 0
        base, ext = os.path.splitext(a.out)
        while done < a.passes:
            n = min(step, a.passes - done)
            rt.render_passes(W, H, depth, done, n, accum, out)
            done += n
            if a.snapshot_every and done < a.passes:
                rt.write_ppm(out, W, H, f"{base}_pass{done}{ext or '.ppm'}", a.exposure, a.gamma)
        rt.write_ppm(out, W, H, a.out, a.exposure, a.gamma)
        st = rt.stats()
        sys.stderr.write(f"rendered {W}x{H}, {a.passes} passes, mode {a.mode}: "
                         f"{st['primary'] + st['shadow'] + st['secondary']} rays in the last call -> {a.out}\n")
    except rt.RtError as e:
        sys.stderr.write(f"{e}\n")
        return EXIT_IO if e.code == -8 else EXIT_RUNTIME
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
