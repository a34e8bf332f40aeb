"""Exact live mode on each wave of a frame under different speculation
policies (hrpp_set_live_rounds R: R exact suspend/trace/resume rounds,
then one speculative round; R = 0 traces every non-TP ray up front)."""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, waves = bench.make_workload_device(args)
tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY) for c in (True, False)}
def frame(rounds_of, times=None):
    for t in tabs.values(): t.clear()
    for name, kind, closest, O, D, a, c in waves:
        hb.set_live_rounds(rounds_of(name))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, st = hb.trace_wave(b, tabs[closest], "live", O, D, a, c, closest)
        e1.record()
        if times is not None: times.append((name, e0, e1, st.copy()))
    hb.set_live_rounds(0)
for R in (0, 1, 2, 3):
    pol = lambda name: R if name == "primary" else 0
    for _ in range(2): frame(pol)
    T = []
    frame(pol, T); torch.cuda.synchronize()
    print(json.dumps({"R": R, "waves": {n: round(e0.elapsed_time(e1), 3) for n, e0, e1, st in T},
                      "primary_bb": int(T[0][3][4])}), flush=True)
