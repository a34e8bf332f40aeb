"""Per-wave live-mode time of a frame (CUDA events), several repeats:
python tools/live_waves.py <config> [mode]"""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
mode = sys.argv[2] if len(sys.argv) > 2 else "live"
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, waves = bench.make_workload_device(args)
tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY) for c in (True, False)}
def frame(times=None):
    for t in tabs.values(): t.clear()
    for name, kind, closest, O, D, a, c in waves:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hb.trace_wave(b, tabs[closest], mode, O, D, a, c, closest)
        e1.record()
        if times is not None: times.append((name, e0, e1))
for _ in range(2): frame()
acc = {}
for _ in range(4):
    T = []
    frame(T); torch.cuda.synchronize()
    for n, e0, e1 in T: acc.setdefault(n, []).append(e0.elapsed_time(e1))
res = {n: round(sorted(v)[len(v) // 2], 3) for n, v in acc.items()}
print(json.dumps({"cfg": cfg, "mode": mode, "total": round(sum(res.values()), 3), "waves": res}))
