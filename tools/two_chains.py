"""a live frame with the closest-hit and hit-any chains on two
streams (host threads) vs sequential."""
import sys, json, threading
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
b.ancestor_lut(0)
streams = {True: torch.cuda.Stream(), False: torch.cuda.Stream()}
def chain(closest, mode):
    with torch.cuda.stream(streams[closest]):
        tabs[closest].clear()
        for name, c, O, D, a, t1 in dw:
            if c == closest:
                hb.trace_wave(b, tabs[closest], mode, O, D, a, t1, c)
def frame_seq(mode):
    for t in tabs.values(): t.clear()
    for name, c, O, D, a, t1 in dw:
        hb.trace_wave(b, tabs[c], mode, O, D, a, t1, c)
def frame_par(mode):
    ths = [threading.Thread(target=chain, args=(c, mode)) for c in (True, False)]
    for t in ths: t.start()
    for t in ths: t.join()
import time
for mode in ("baseline", "live", "fast"):
    for name, fn in (("seq", frame_seq), ("par", frame_par)):
        for _ in range(2): fn(mode)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5): fn(mode)
        torch.cuda.synchronize()
        print(json.dumps({"mode": mode, "sched": name, "ms": round((time.perf_counter() - t0) / 5 * 1e3, 3)}), flush=True)
