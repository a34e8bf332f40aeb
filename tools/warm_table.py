"""Live mode on tables kept from the previous frame: frame 0 trains the
tables, frame 1 (the same camera, re-jittered rays and light / bounce
samples) is traced on them.  Prints per-wave GPU time, TPs and traced box
tests of frame 1 in baseline mode, live on fresh tables and live on the
warm tables.  python tools/warm_table.py <config>"""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, w0 = bench.make_workload_device(args)
_, _, w1 = bench.make_workload_device(args, seed=1, scene_bvh=(sc, b))
tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY) for c in (True, False)}
def frame(waves, mode, times=None):
    for name, kind, closest, O, D, a, c in waves:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, st = hb.trace_wave(b, tabs[closest] if mode != "baseline" else None, mode, O, D, a, c, closest)
        e1.record()
        if times is not None: times.append((name, e0, e1, st.copy()))
def clear():
    for t in tabs.values(): t.clear()
def run(label, prep, mode):
    for _ in range(2):
        prep(); frame(w1, mode)
    prep()
    T = []
    frame(w1, mode, T); torch.cuda.synchronize()
    rows = {n: {"ms": round(e0.elapsed_time(e1), 3), "tp": int(st[1]), "bb": int(st[4])} for n, e0, e1, st in T}
    print(json.dumps({"cfg": cfg, "run": label, "total_ms": round(sum(r["ms"] for r in rows.values()), 3),
                      "rays": int(sum(int(st[0]) for _, _, _, st in T)), "waves": rows}), flush=True)
def warm():
    clear(); frame(w0, "live")
run("frame1 baseline", clear, "baseline")
run("frame1 live, fresh tables", clear, "live")
run("frame1 live, tables trained by frame0", warm, "live")
