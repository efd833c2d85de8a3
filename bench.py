#!/usr/bin/env python
"""Benchmark of the B200 ray-tracing hot path (arXiv 1504.03151) — prints ONE JSON line.

Metric (BASELINE.json): "Mrays/s (primary+shadow+secondary) and fps at 1080p depth 5, 1/2/4/8
B200". Workload: config C4 (BJ:10) — 1920x1080, 1000 random spheres, 8 point lights,
max_depth 5, 4 spp, tile-sharded across N GPUs (one process per GPU, NCCL all-gather of the
tile slabs to rank 0, which assembles the frame). A step = one full frame.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C4]
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: W untimed warm-up frames; K timed frames bracketed by barrier + synchronize; each frame
timed with CUDA events on the launch stream; L2 (126 MB) is flushed with a 256 MiB write before
every frame, outside the per-frame events; value = rays of all ranks / max-over-ranks time.
`--impl reference` times the CPU oracle (the plain C reference written from the paper) on the
host cores with the same metric, on a bounded pixel sample per step.

`--mode progressive` (auxiliary; 1 GPU): the paper-shaped Cornell
box C0 (640x480, depth 6) with the global integrator and its spherical area light, a step =
one rt_render_passes call of --passes passes accumulated into a device float64 buffer.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import scenegen  # noqa: E402

METRIC = "Mrays/s (primary+shadow+secondary) and fps at 1080p depth 5, 1/2/4/8 B200"
FLOP_SPHERE, FLOP_PLANE = 19, 12   # SURVEY.md §8(d).3 counted flops per test
PEAK_FALLBACK_MHZ = 1965.0


# ---------------------------------------------------------------------------------------------
def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.idx, self.period, self.proc, self.lines = gpu_index, period_ms, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 f"-lms", str(self.period), "-i", str(self.idx)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _measured_peak(key: str, fallback: float) -> float:
    """Driver-written MEASURED_PEAKS.json (this pool's B200s), else the profiling guide's figure."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))[key])
    except (OSError, ValueError, KeyError):
        return fallback


def measure_fp32_peak(gpu: int) -> dict:
    """The FFMA2 chain microbenchmark (tools/micro/ffma2_peak.cu) on this box right before the
    timed frames, with nvidia-smi sampling the SM clock under that FP32 load."""
    from paper_1504_03151_b200 import build as rtbuild
    try:
        exe = rtbuild.build_peak_tool()
        clk = ClockSampler(gpu, period_ms=20)
        clk.start()
        out = subprocess.run([exe, "40"], capture_output=True, text=True, timeout=120,
                             env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", str(gpu))))
        c = clk.stop()
        res = json.loads(out.stdout.strip().splitlines()[-1])
        res.update(sm_mhz_under_load=c.get("sm_mhz"), clock_reasons=c.get("reasons"))
        return res
    except Exception as ex:  # noqa: BLE001 - reported, the derived figure is used instead
        return {"error": f"{type(ex).__name__}: {ex}"}


def _load_profile(workload: str) -> dict:
    """The committed ncu --set full summary of one kernel class (profiles/ncu_render_kernel.json):
    DRAM bytes per launch, FMA-pipe and issue activity."""
    path = os.path.join(ROOT, "profiles", "ncu_render_kernel.json")
    try:
        return json.load(open(path)).get(workload) or {}
    except (OSError, ValueError):
        return {}


def _load_profile_traffic(workload: str):
    """dram bytes per launch of a kernel class from the committed ncu --set full summary."""
    v = _load_profile(workload).get("dram_bytes_per_launch")
    return float(v) if v else None


# ---------------------------------------------------------------------------------------------
_SCENES = {}


def _oracle_chunk(args):
    """Worker: oracle on a slice of pixels (runs in a separate process; scene cached)."""
    name, pixels, okw = args
    from oracle import pyoracle as po
    if name not in _SCENES:
        _SCENES[name] = scenegen.get(name)
    sc = _SCENES[name]
    if okw.get("spp"):
        sc = sc.with_frame(spp=okw["spp"])
    okw = {k: v for k, v in okw.items() if k != "spp"}
    _, counts = po.render_rgb_only(sc, pixels=np.asarray(pixels, np.int64), **okw)
    return counts


class OracleTimer:
    """The CPU oracle, as it stands, on all host cores (pixel slices across processes).
    okw: oracle mode arguments (progressive mode: integrator, area_lights, jitter, spp)."""

    def __init__(self, name: str, okw: dict | None = None):
        import concurrent.futures as cf
        from oracle import pyoracle as po
        po.build()
        self.name = name
        self.okw = dict(okw or {})
        self.cores = os.cpu_count() or 1
        self.pool = cf.ProcessPoolExecutor(max_workers=self.cores)
        list(self.pool.map(_oracle_chunk, [(name, [0], self.okw)] * self.cores))  # warm the workers

    def run(self, pixels: np.ndarray) -> tuple[float, dict]:
        chunks = [(self.name, c.tolist(), self.okw) for c in np.array_split(pixels, self.cores) if len(c)]
        t0 = time.perf_counter()
        res = list(self.pool.map(_oracle_chunk, chunks))
        dt = time.perf_counter() - t0
        tot = {k: sum(r[k] for r in res) for k in res[0]}
        return dt, tot

    def close(self):
        self.pool.shutdown()


def cpu_baseline(name: str, target_core_s: float = 20.0, seed: int = 7, okw: dict | None = None) -> dict:
    sc = scenegen.get(name)
    if okw and okw.get("spp"):
        sc = sc.with_frame(spp=okw["spp"])
    tm = OracleTimer(name, okw)
    rng = np.random.default_rng(seed)
    # calibrate: per-pixel cost on a small sample, then size the sample to ~target_core_s
    probe = rng.choice(sc.width * sc.height, 64 * tm.cores, replace=False)
    dt, _ = tm.run(probe)
    per_px_core = dt * tm.cores / len(probe)
    n = int(min(sc.width * sc.height, max(len(probe), target_core_s / max(per_px_core, 1e-9))))
    pix = rng.choice(sc.width * sc.height, n, replace=False)
    dt, cnt = tm.run(pix)
    # the same oracle single-threaded, on 1/cores of the sample
    sub = pix[: max(1, n // tm.cores)]
    t1 = time.perf_counter()
    c1 = _oracle_chunk((name, sub.tolist(), dict(okw or {})))
    dt1 = time.perf_counter() - t1
    tm.close()
    rays = cnt["primary"] + cnt["shadow"] + cnt["secondary"]
    rays1 = c1["primary"] + c1["shadow"] + c1["secondary"]
    frac = n / (sc.width * sc.height)
    what = f"all {sc.spp} spp" if not okw else f"{sc.spp} progressive passes, global integrator + area lights"
    return {"value": rays / dt / 1e6, "unit": "Mrays/s", "cores": tm.cores, "kind": "oracle",
            "sample": f"{n} random pixels of {name} ({what}, depth {sc.max_depth}) = {frac:.2%} of the frame, "
                      f"{dt:.2f} s wall on {tm.cores} processes",
            "fps_extrapolated": 1.0 / (dt / frac),
            "value_1thread": rays1 / dt1 / 1e6, "sample_1thread": f"{len(sub)} of those pixels in this process"}


# ---------------------------------------------------------------------------------------------
def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    name = args.config
    sc = scenegen.get(name)
    tm = OracleTimer(name)
    rng = np.random.default_rng(11)
    n_px = args.ref_pixels
    for _ in range(args.warmup):
        tm.run(rng.choice(sc.width * sc.height, n_px, replace=False))
    tot_t, tot_rays = 0.0, 0
    for _ in range(args.steps):
        dt, cnt = tm.run(rng.choice(sc.width * sc.height, n_px, replace=False))
        tot_t += dt
        tot_rays += cnt["primary"] + cnt["shadow"] + cnt["secondary"]
    tm.close()
    value = tot_rays / tot_t / 1e6
    frac = n_px / (sc.width * sc.height)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "fps": 1.0 / (tot_t / args.steps / frac),
        "config": dict(sc.describe(), workload=name, sample_pixels_per_step=n_px),
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": tm.cores, "kind": "oracle",
                         "sample": f"{n_px} random pixels of {name} per step ({frac:.3%} of the frame)"},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------------
def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_1504_03151_b200 import build as rtbuild
    from paper_1504_03151_b200 import rt
    from paper_1504_03151_b200.multigpu import CudaBackend, P2PRenderer, ShardedRenderer

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    # B200RT_DIST_BACKEND=gloo + B200RT_SHARE_GPU=1: every rank on cuda:0 with host barriers — a
    # smoke test of the multi-rank flow on a one-GPU box (the ranks' kernels never wait on each
    # other there); the benchmark itself is NCCL, one GPU per rank
    backend = os.environ.get("B200RT_DIST_BACKEND", "nccl")
    gpu = 0 if os.environ.get("B200RT_SHARE_GPU") == "1" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    rtbuild.build()  # no-op when the in-tree library is current
    stream = torch.cuda.current_stream()
    rt.set_stream(stream)

    sc = scenegen.get(args.config)
    W, H, D, S = sc.width, sc.height, sc.max_depth, sc.spp
    prims, mats, lights, env = rt.pack_scene(sc)
    rt.load_scene(sc)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    collective = None
    if world > 1:
        rend = None
        if args.collective == "p2p":  # fused render + gather: pixels stored into rank 0's frame over NVLink
            try:
                rend = P2PRenderer(W, H, D, S)
                collective = "p2p (resolve kernels store into rank 0's frame over NVLink peer memory)"

                def step():
                    rend.render(want_stats=False)  # stream-ordered barrier, no host sync
            except RuntimeError as ex:
                if rank == 0:
                    print(f"bench.py: {ex}; falling back to the NCCL all-gather", file=sys.stderr)
                rend = None
        if rend is None:
            rend = ShardedRenderer(CudaBackend(dev), W, H, D, S)
            step = rend.render
            collective = "allgather (NCCL all_gather_into_tensor of the tile slabs + rank-0 assembly)"
    else:
        out = torch.empty((H, W, 4), dtype=torch.float32, device=dev)
        step = lambda: rt.render(W, H, D, S, out)  # noqa: E731

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[gpu])
            else:
                torch.cuda.synchronize()
                dist.barrier()
        torch.cuda.synchronize()

    if world > 1:  # kernels per frame on this rank: the shard render (+ assembly or stats sum on rank 0)
        probe = torch.empty(rt.shard_layout(W, H, world)[1], dtype=torch.uint8, device=dev)
        rt.render_shard(W, H, D, S, rank, world, probe)  # same launches as the direct shard
        extra = (2 if isinstance(rend, ShardedRenderer) else 1) if rank == 0 else 0
        launches_per_step = rt.stats()["launches"] + extra
        del probe
    fp32 = measure_fp32_peak(gpu) if rank == 0 and not args.no_fp32_peak else None
    # warm-up (after the probe, so the frame's launch sequence is captured as a CUDA graph here)
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    barrier()
    clocks = ClockSampler(gpu)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    t_wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()                       # L2 flush, outside the frame events
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    barrier()
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    frame_ms = [a.elapsed_time(b) for a, b in evs]
    my_total = sum(frame_ms)
    st = rt.stats()  # last frame (rank 0 holds the all-rank sum after assembly)
    per_frame = [st]  # per-kernel event times of the last timed frame
    if world == 1:
        launches_per_step = st["launches"]
    t = torch.tensor([my_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    per_rank = None
    if world > 1:  # every rank's step time and its last shard render (imbalance)
        # this rank's shard render alone, once more after the timed region (rank 0's statistics
        # above are the assembly's, which times no render)
        probe = torch.empty(rt.shard_layout(W, H, world)[1], dtype=torch.uint8, device=dev)
        rt.render_shard(W, H, D, S, rank, world, probe)
        shard_ms = float(rt.stats()["last_render_ms"])
        del probe
        cdev = dev if backend == "nccl" else torch.device("cpu")
        mine = torch.tensor([my_total / args.steps, shard_ms], dtype=torch.float64, device=cdev)
        allt = torch.empty(2 * world, dtype=torch.float64, device=cdev)
        dist.all_gather_into_tensor(allt, mine)
        rows = allt.view(world, 2).tolist()
        per_rank = {"step_ms": [round(r[0], 4) for r in rows], "shard_render_ms": [round(r[1], 4) for r in rows],
                    "note": "step = shard render + the frame's collective (CUDA events, mean over the timed "
                            "steps); shard_render = the library's own events around one more render of this "
                            "rank's shard after the timed region"}

    # per-kernel times for the roofline: the same frames with every wavefront launch in order on
    # one stream (the timed frames overlap a depth's shadow scan with the next closest-hit scan,
    # so their per-launch events would share the GPU); CUDA events inside the library
    kt = None
    if world == 1 and st["variant"] == 1:
        rt.set_concurrency(False)
        ks = max(3, min(args.steps, 20))
        keys = (("closest", "isect_closest_ms"), ("shadow", "isect_shadow_ms"), ("eye", "isect_eye_ms"),
                ("shade", "shade_ms"), ("accumulate", "accumulate_ms"), ("frame", "last_render_ms"))
        acc = {k: 0.0 for k, _ in keys}
        for it in range(3 + ks):  # 3 warm-up frames: the in-order sequence is captured as a graph
            flush.zero_()
            step()
            f = rt.stats()
            if it < 3:
                continue
            for k, key in keys:
                acc[k] += f[key]
        rt.set_concurrency(True)
        kt = {k: v / ks for k, v in acc.items()}
        kt["frames"] = ks

    # e2e: the public C-ABI calls with host buffers: H2D of the step's inputs (the scene, on
    # every rank) and D2H of the step's result (the frame, on rank 0), wall clock, max over ranks
    host_out = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True) if rank == 0 else None
    h2d = (prims.nbytes + mats.nbytes + lights.nbytes + env.nbytes) * world
    d2h = H * W * 16 + 64
    ke = max(3, min(args.steps, 20))
    rays_e2e = 0
    for it in range(max(3, args.warmup) + ke):  # the first iterations are warm-up (untimed)
        if it == max(3, args.warmup):
            barrier()
            t0 = time.perf_counter()
            rays_e2e = 0
        rt.scene_upload(prims, mats, lights, env)
        rt.camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)
        if world == 1:
            rt.render(W, H, D, S, host_out)   # host pointer: returns after the D2H copy
            s2 = rt.stats()
        else:
            frame = rend.render()
            if rank == 0:
                host_out.copy_(frame.image.view(H, W, 4))
            torch.cuda.synchronize()
            if isinstance(rend, P2PRenderer):
                rend.release()
            s2 = frame.stats or {"primary": 0, "shadow": 0, "secondary": 0}
        rays_e2e += s2["primary"] + s2["shadow"] + s2["secondary"]
    dt = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    e2e = {"value": rays_e2e / dt / 1e6, "unit": "Mrays/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "steps": ke, "ms_per_step": 1e3 * dt / ke,
           "timing": "host wall clock (max over ranks) around rt_scene_upload + rt_camera_set + "
                     + ("rt_render(pinned host buffer)" if world == 1 else
                        ("rt_render_shard_direct (pixels stored into rank 0's frame over peer memory) + per-frame "
                         "barrier + D2H to pinned host" if isinstance(rend, P2PRenderer) else
                         "rt_render_shard + NCCL all-gather + rt_assemble_tiles + D2H to pinned host"))}

    if rank == 0:
        rays = st["primary"] + st["shadow"] + st["secondary"]
        ms_per_step = total_ms / args.steps
        value = rays / (ms_per_step * 1e-3) / 1e6
        # roofline of the dominant kernel (the largest share of the in-order frame):
        #  * scans: bound "alu"; achieved = EXECUTED FP32 flops (the FMAs the filter form needs per
        #    test: 3 FMA for camera rays and light-origin shadow rays (the tangent test of a shared
        #    origin), 7 FMA for secondary rays)
        #    per second of the kernel's own launches; peak = the FFMA2 microbenchmark measured on
        #    this box in this run; the counted figure (19 flops per test) beside it;
        #  * wf_shade / wf_accumulate: bound "hbm"; achieved = algorithmic bytes /
        #    time; peak = MEASURED_PEAKS.json hbm_gbs.
        props = torch.cuda.get_device_properties(dev)
        sms = props.multi_processor_count
        sm_max = clk.get("sm_max_mhz") or PEAK_FALLBACK_MHZ
        derived = sms * 128 * 2 * sm_max * 1e6 / 1e12
        peak, peak_basis = derived, f"{sms} SMs x 128 FP32 lanes x 2 flop x {sm_max:.0f} MHz (derived; measurement failed)"
        if fp32 and fp32.get("tflops"):
            peak = fp32["tflops"]
            peak_basis = (f"measured in this run: FFMA2 dependent chains on all SMs (tools/micro/ffma2_peak.cu), "
                          f"best of {fp32.get('reps')}, SM clock {fp32.get('sm_mhz_under_load')} MHz under that load "
                          f"(derived {derived:.2f} at {sm_max:.0f} MHz)")
        hbm_peak = _measured_peak("hbm_gbs", 6549.1)
        traffic = _load_profile_traffic(args.config) if world == 1 else None
        extra = {}
        if kt is not None:
            n_closest = st["closest_sphere_tests"]
            n_eye = st["primary"] * sc.n_spheres
            n_shadow = st["sphere_tests"] - n_closest
            sh_fma = 3 if 0 < sc.n_lights <= 30 else 7  # light-origin scans for <= 30 point lights
            prim, sec, shd = st["primary"], st["secondary"], st["shadow"]
            cands = {
                "shadow": {"kernel": "wf_isect_lt (shadow rays to point lights, scanned from the light; FP32 FFMA2, "
                                     "early exit at a certain occluder)", "bound": "alu",
                           "ms": kt["shadow"], "tests": n_shadow, "fma_per_test": sh_fma},
                "camera": {"kernel": "wf_isect_eye2 (camera rays, shared-origin FP32 FFMA2 scan)", "bound": "alu",
                           "ms": kt["eye"], "tests": n_eye, "fma_per_test": 3},
                "secondary": {"kernel": "wf_isect<closest> (secondary closest-hit rays, FP32 FFMA2 scan)", "bound": "alu",
                              "ms": kt["closest"] - kt["eye"], "tests": n_closest - n_eye, "fma_per_test": 7},
                # algorithmic bytes: per shaded path the ray state in (84 B at depth >= 1;
                # camera rays are implicit), its candidate count in (4 B) and its entry range and next
                # position out (12 B); per continuation the next state out (84 B); per ended path its
                # radiance (12 B); per shadow ray its scan record (24 B: float direction and t_max,
                # entry, skip), its contribution (12 B) and its slot (4 B) out (round 1 wrote the 56-B
                # FP64 ray instead of the record: 68 B per shadow ray)
                "shade": {"kernel": "wf_shade (FP64 nearest hit, shading, shadow-ray set-up, bounce)", "bound": "hbm",
                          "ms": kt["shade"],
                          "bytes": 84 * sec + 16 * (prim + sec) + 84 * sec + 12 * prim + 40 * shd},
                # per shadow ray its decision inputs (status 8 B) and contribution (12 B); per shading
                # path the entry range (8 B) and the radiance read and written (24 B)
                "accumulate": {"kernel": "wf_accumulate (FP64 occlusion decisions, radiance sums)", "bound": "hbm",
                               "ms": kt["accumulate"], "bytes": 20 * shd + 32 * (prim + sec)},
            }
            for k, v in cands.items():
                v["share_of_frame"] = v["ms"] / kt["frame"]
                prof = _load_profile(f"{args.config}:{k}")
                if prof:  # the committed ncu capture of this kernel class (one launch, cold, serialised)
                    v["ncu"] = {kk: prof.get(kk) for kk in ("fma_pipe_active_pct", "issue_active_pct",
                                                             "warp_efficiency_pct", "dram_bytes_per_launch", "source")}
                if v["bound"] == "alu":
                    v["achieved"] = 2 * v["fma_per_test"] * v["tests"] / (v["ms"] * 1e-3) / 1e12
                    v["achieved_counted"] = FLOP_SPHERE * v["tests"] / (v["ms"] * 1e-3) / 1e12
                    v["frac"] = v["achieved"] / peak
                    v["unit"] = "TFLOP/s"
                else:
                    v["achieved"] = v["bytes"] / (v["ms"] * 1e-3) / 1e9
                    v["frac"] = v["achieved"] / hbm_peak
                    v["unit"] = "GB/s"
            dom = max(cands, key=lambda k: cands[k]["ms"])
            d = cands[dom]
            achieved, bound, unit = d["achieved"], d["bound"], d["unit"]
            rpeak = peak if bound == "alu" else hbm_peak
            kernel = d["kernel"] + ", CUDA events per launch, launches in order on one stream"
            traffic = _load_profile_traffic(f"{args.config}:{dom}") or traffic
            extra = {"share_of_frame": d["share_of_frame"],
                     "kernels": {k: {kk: vv for kk, vv in v.items() if kk != "kernel"} for k, v in cands.items()},
                     "kernel_timing_pass": f"{kt['frames']} frames, frame {kt['frame']:.3f} ms in order vs "
                                           f"{ms_per_step:.3f} ms in the timed (concurrent) frames",
                     "whole_frame_counted_tflops": (FLOP_SPHERE * st["sphere_tests"] + FLOP_PLANE * st["plane_tests"])
                     / (ms_per_step * 1e-3) / 1e12}
            if bound == "alu":
                extra["achieved_counted"] = d["achieved_counted"]
        else:
            flops = FLOP_SPHERE * st["sphere_tests"] + FLOP_PLANE * st["plane_tests"]
            achieved = flops / world / (total_ms / args.steps * 1e-3) / 1e12
            bound, unit, rpeak = "alu", "TFLOP/s", peak
            kernel = ("render_kernel (megakernel), counted flops" if world == 1
                      else "whole shard frame incl. the gather, counted flops")
        roofline = {"bound": bound, "achieved": achieved, "peak": rpeak, "unit": unit, "frac": achieved / rpeak,
                    "traffic": traffic, "kernel": kernel, **extra,
                    "peak_basis": peak_basis if bound == "alu" else "MEASURED_PEAKS.json hbm_gbs (burst copy bandwidth)",
                    "fp32_peak_measured": fp32,
                    "flops_basis": "executed: 3 FMA per camera-ray / light-origin shadow test (tangent test), "
                                   "7 per secondary test; "
                                   "counted: 19 flops/sphere test + 12/plane test (SURVEY 8(d).3)"}
        line = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (FFMA2 filter) + f64 (candidate refinement, shading geometry)",
            "data": "synthetic (seeded scenegen C4 scene; no dataset)",
            "fps": 1e3 / ms_per_step,
            "config": dict(sc.describe(), workload=args.config, parallelism=f"tiles{world}", collective=collective,
                           l2="flushed (256 MiB write) before every frame, outside the frame events",
                           rays_per_frame=int(rays), primary=int(st["primary"]), shadow=int(st["shadow"]),
                           secondary=int(st["secondary"]), sphere_tests=int(st["sphere_tests"]),
                           plane_tests=int(st["plane_tests"]), wall_s=t_wall),
            "roofline": roofline,
            "clocks": clk,
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
        }
        if per_rank:
            line["per_rank"] = per_rank
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.config, target_core_s=args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()
    return 0


def run_progressive(args):
    """NEXT-1/NEXT-2 measurement: progressive passes of C0 with the global integrator and area
    lights. A step = one rt_render_passes call of args.passes passes (pass indices continue
    across steps, the float64 accumulation buffer stays on the device)."""
    import torch
    from paper_1504_03151_b200 import build as rtbuild
    from paper_1504_03151_b200 import rt
    if _env_int("WORLD_SIZE", 1) != 1:
        raise SystemExit("--mode progressive runs on one GPU (rt_render_passes is a full-frame call)")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    rtbuild.build()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    rt.set_stream(stream)
    name = args.config if args.config != "C4" else "C0"
    sc = scenegen.get(name)
    W, H, D, P = sc.width, sc.height, sc.max_depth, args.passes
    prims, mats, lights, env = rt.pack_scene(sc)
    rt.load_scene(sc)
    rt.set_integrator("global", True)
    accum = torch.zeros((H, W, 3), dtype=torch.float64, device=dev)
    out = torch.empty((H, W, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    nxt = [0]

    def step():
        rt.render_passes(W, H, D, nxt[0], P, accum, out)
        nxt[0] += P

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    first = nxt[0]
    clocks = ClockSampler(0)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    st_last = rt.stats()
    # exact ray counts of the timed steps: replay the same pass indices (deterministic) untimed
    acc2 = torch.zeros_like(accum)
    rays = tests_c = tests_s = tests_p = 0
    n_closest = n_shadow = n_secondary = 0
    for i in range(args.steps):
        rt.render_passes(W, H, D, first + i * P, P, acc2, None)
        s2 = rt.stats()
        rays += s2["primary"] + s2["shadow"] + s2["secondary"]
        tests_c += s2["closest_sphere_tests"]
        tests_s += s2["sphere_tests"] - s2["closest_sphere_tests"]
        tests_p += s2["plane_tests"]
        n_closest += s2["primary"] + s2["secondary"]
        n_shadow += s2["shadow"]
        n_secondary += s2["secondary"]
    ms_per_step = total_ms / args.steps
    value = rays / (total_ms * 1e-3) / 1e6
    props = torch.cuda.get_device_properties(dev)
    sm_max = clk.get("sm_max_mhz") or PEAK_FALLBACK_MHZ
    peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12
    whole = (FLOP_SPHERE * (tests_c + tests_s) + FLOP_PLANE * tests_p) / (total_ms * 1e-3) / 1e12
    tc = st_last["isect_closest_ms"]
    # dominant kernel here: wf_shade (profiles/r01_launches_c0_progressive_summary.txt). Its
    # algorithmic HBM bytes: 124 B per shaded path (queue id, ray, candidate count,
    # skip, depth, T, L in; T, L, shadow offset/count, exit sphere out) + 44 B per shadow entry
    # (path, light, contribution, sampled emitter point; C0 has no point lights) + 60 B per
    # continuation (ray, depth, skip, queue slot). Timed per launch with CUDA events in the library.
    shade_ms = st_last["shade_ms"]
    last_closest = st_last["primary"] + st_last["secondary"]
    shade_bytes = 124 * last_closest + 44 * st_last["shadow"] + 60 * st_last["secondary"]
    hbm_peak = _measured_peak("hbm_gbs", 6549.1)
    shade_gbs = shade_bytes / (shade_ms * 1e-3) / 1e9 if shade_ms > 0 else 0.0
    # e2e through the public API with host buffers: scene H2D, P passes, mean frame D2H
    host_out = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
    ke = max(3, min(args.steps, 10))
    acc3 = torch.zeros_like(accum)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rays_e2e = 0
    for i in range(ke):
        rt.scene_upload(prims, mats, lights, env)
        rt.camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)
        rt.render_passes(W, H, D, i * P, P, acc3, host_out)
        s3 = rt.stats()
        rays_e2e += s3["primary"] + s3["shadow"] + s3["secondary"]
    dt = time.perf_counter() - t0
    rt.set_integrator("whitted", False)
    line = {
        "metric": "Mrays/s (primary+shadow+secondary), progressive passes, global illumination + area light",
        "value": value, "unit": "Mrays/s", "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (FFMA2 filter, radiance) + f64 (decisions, geometry, accumulation)",
        "data": f"synthetic (seeded scenegen {name} Cornell box; no dataset)",
        "passes_per_s": P / (ms_per_step * 1e-3),
        "config": dict(sc.describe(), workload=name, mode="progressive", integrator="global", area_lights=True,
                       passes_per_step=P, l2="flushed (256 MiB write) before every step, outside the events",
                       rays_per_step=int(rays / args.steps)),
        "roofline": {"bound": "hbm", "achieved": shade_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": shade_gbs / hbm_peak, "traffic": _load_profile_traffic("C0"),
                     "kernel": "wf_shade (FP64 nearest hit + shading + light sampling + bounce), per-launch CUDA "
                               "events of the last timed step; algorithmic bytes per DESIGN.md §7",
                     "share_of_step": shade_ms / ms_per_step,
                     "peak_basis": "MEASURED_PEAKS.json hbm_gbs (burst copy bandwidth)",
                     "closest_scan": {"bound": "alu", "share_of_step": tc / ms_per_step},
                     "whole_step_test_flops_tflops": whole, "alu_peak_tflops": peak},
        "clocks": clk,
        "gpu_launches": st_last["launches"] * args.steps,
        "e2e": {"value": rays_e2e / dt / 1e6, "unit": "Mrays/s",
                "h2d_bytes_per_step": int(prims.nbytes + mats.nbytes + lights.nbytes + env.nbytes),
                "d2h_bytes_per_step": H * W * 16, "steps": ke, "ms_per_step": 1e3 * dt / ke,
                "timing": "host wall clock around rt_scene_upload + rt_camera_set + rt_render_passes(pinned host out)"},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name, target_core_s=args.cpu_seconds,
                                            okw=dict(integrator=1, area_lights=1, jitter=1, spp=P))
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="C4", choices=sorted(scenegen.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32-peak", action="store_true", help="skip the in-run FFMA2 peak measurement "
                    "(e.g. under ncu, which would profile the microbenchmark too); the derived peak is used")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="core-seconds of oracle work")
    ap.add_argument("--ref-pixels", type=int, default=4096, help="--impl reference: pixels per step")
    ap.add_argument("--strict", action="store_true", default=True)
    ap.add_argument("--mode", choices=["hot", "progressive"], default="hot",
                    help="hot: the §8(a) path on C4 (default); progressive: NEXT-1/2 passes on C0")
    ap.add_argument("--passes", type=int, default=16, help="--mode progressive: passes per step")
    ap.add_argument("--collective", choices=["allgather", "p2p"], default="allgather",
                    help="N>1: the NCCL all-gather of the tile slabs + rank-0 assembly (default, north_star's one "
                         "collective) or the ablation: render+gather fused into rank 0's frame over peer memory")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "progressive":
        return run_progressive(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
