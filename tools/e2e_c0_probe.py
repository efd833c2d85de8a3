import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, scenegen
from paper_1504_03151_b200 import rt
sc = scenegen.get("C0"); W,H,D = sc.width, sc.height, sc.max_depth
prims, mats, lights, env = rt.pack_scene(sc)
rt.set_stream(torch.cuda.current_stream())
rt.load_scene(sc); rt.set_integrator("global", True)
host = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
dev = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
acc = torch.zeros((H, W, 3), dtype=torch.float64, device="cuda")
for k in range(3): rt.render_passes(W, H, D, 0, 16, acc, host)
for mode in ["host", "dev"]:
    t = time.perf_counter()
    for i in range(5):
        rt.render_passes(W, H, D, 16*i, 16, acc, host if mode == "host" else dev)
        st = rt.stats()
    torch.cuda.synchronize()
    print(mode, (time.perf_counter()-t)/5*1e3, "ms", st["last_render_ms"], st["variant"], st["launches"])
acc3 = torch.zeros_like(acc)
torch.cuda.synchronize()
for i in range(6):
    t0 = time.perf_counter()
    rt.scene_upload(prims, mats, lights, env)
    t1 = time.perf_counter()
    rt.camera_set(sc.eye, sc.look_at, sc.up, sc.vfov)
    rt.render_passes(W, H, D, i * 16, 16, acc3, host)
    s3 = rt.stats()
    t2 = time.perf_counter()
    print("e2e step", i, round((t1 - t0) * 1e3, 3), round((t2 - t1) * 1e3, 3), s3["launches"])
