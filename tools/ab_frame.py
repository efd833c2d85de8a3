#!/usr/bin/env python
"""A/B of library builds on one box: per build, the median frame time of the benched
configuration (concurrent streams, graph replay, L2 flushed before every frame, CUDA events) and
the in-order per-kernel times (library events, rt_set_concurrency(0)).

    python tools/ab_frame.py [--config C4] [--frames 30] [--rounds 2] [--pipeline K] [--variant V] LIB.so [LIB2.so ...]

Each measurement runs in its own process (B200RT_LIB selects the build); builds alternate over
the rounds so clock drift hits every build alike. Tool only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, frames, pipeline=0, variant="auto"):
    sys.path.insert(0, ROOT)
    import torch
    import scenegen
    from paper_1504_03151_b200 import rt
    sc = scenegen.get(config)
    stream = torch.cuda.current_stream()
    rt.set_stream(stream)
    rt.load_scene(sc)
    if pipeline:
        rt.set_pipeline(pipeline)
    rt.set_variant(variant)
    out = torch.empty((sc.height, sc.width, 4), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    for _ in range(4):
        rt.render(W, H, D, S, out)
    ms = []
    for _ in range(frames):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rt.render(W, H, D, S, out)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    st = rt.stats()
    res = {"frame_ms": statistics.median(ms), "rays": st["primary"] + st["shadow"] + st["secondary"]}
    if st["variant"] == 1:
        rt.set_concurrency(False)
        acc = {}
        for i in range(3 + 10):
            flush.zero_()
            rt.render(W, H, D, S, out)
            f = rt.stats()
            if i < 3:
                continue
            for k in ("last_render_ms", "isect_eye_ms", "isect_closest_ms", "isect_shadow_ms", "shade_ms", "accumulate_ms"):
                acc[k] = acc.get(k, 0.0) + f[k] / 10
        acc["secondary_ms"] = acc["isect_closest_ms"] - acc["isect_eye_ms"]
        res.update(inorder=acc)
    print("RESULT " + json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--pipeline", type=int, default=0, help="rt_set_pipeline slots (0: the library default)")
    ap.add_argument("--variant", default="auto", help="auto | wavefront | megakernel")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return child(a.config, a.frames, a.pipeline, a.variant)
    libs = a.libs or [os.path.join(ROOT, "paper_1504_03151_b200", "libb200rt.so")]
    res = {lib: [] for lib in libs}
    for _ in range(a.rounds):
        for lib in libs:
            out = subprocess.run([sys.executable, __file__, "--child", "--config", a.config, "--frames", str(a.frames),
                                  "--pipeline", str(a.pipeline), "--variant", a.variant],
                                 env=dict(os.environ, B200RT_LIB=os.path.abspath(lib)), capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT ")]
            if not line:
                print(lib, "FAILED", out.stderr[-2000:])
                continue
            res[lib].append(json.loads(line[0][7:]))
    for lib, rs in res.items():
        if not rs:
            continue
        fr = [r["frame_ms"] for r in rs]
        msg = f"{os.path.basename(lib):28s} frame {min(fr):.3f} ms (runs {', '.join(f'{x:.3f}' for x in fr)})"
        if "inorder" in rs[0]:
            io = {k: min(r["inorder"][k] for r in rs) for k in rs[0]["inorder"]}
            msg += (f" | in-order {io['last_render_ms']:.3f}: eye {io['isect_eye_ms']:.3f} sec {io['secondary_ms']:.3f} "
                    f"shadow {io['isect_shadow_ms']:.3f} shade {io['shade_ms']:.3f} accum {io['accumulate_ms']:.3f}")
        print(msg, flush=True)


if __name__ == "__main__":
    sys.exit(main())
