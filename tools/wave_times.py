"""per-wave GPU time of baseline (full traversal) and live mode."""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, waves = bench.make_workload(args, lambda bv, O, D, a, c: hb.intersect_closest_batch(bv, O, D, a, c))
dev = torch.device("cuda")
dw = [(w[0], w[2], *(torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in w[3:])) for w in waves]
tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY) for c in (True, False)}
def frame(mode, times=None):
    for t in tabs.values(): t.clear()
    for name, closest, O, D, a, c in dw:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, st = hb.trace_wave(b, tabs[closest] if mode != "baseline" else None, mode, O, D, a, c, closest)
        e1.record()
        if times is not None: times.append((name, e0, e1, st.copy()))
for mode in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("baseline", "live", "fast")):
    for _ in range(2): frame(mode)
    T = []
    frame(mode, T); torch.cuda.synchronize()
    for name, e0, e1, st in T:
        print(json.dumps({"mode": mode, "wave": name, "ms": round(e0.elapsed_time(e1), 3), "rays": int(st[0]), "tp": int(st[1]), "bb": int(st[4]), "ob": int(st[6])}))
