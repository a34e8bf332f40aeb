"""GPU idle gaps inside one live frame (bench --config), from a CUPTI kernel timeline
(torch.profiler): every interval where no kernel or memcpy/memset runs, with
the activities on either side.  Usage: python tools/gap_timeline.py [bench args]"""
import sys
from pathlib import Path
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1910_01304_b200 as hb  # noqa: E402

TL = "--timeline" in sys.argv
MODE = "fast" if "--fast" in sys.argv else "live"
WARM = "--warm" in sys.argv  # profile a re-jittered frame on the tables the frame left
sys.argv = [a for a in sys.argv if a not in ("--timeline", "--fast", "--warm")]
args = bench.parse()
sc, bvh, waves = bench.make_workload_device(args)
dw = [(w[2], *w[3:]) for w in waves]
cfg = hb.HashConfig(args.precision)
tables = {c: hb.PredictorTable(cfg, args.go_up, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
          for c in (True, False)}


def frame():
    for t in tables.values():
        t.clear()
    for closest, O, D, t0, t1 in dw:
        hb.trace_wave(bvh, tables[closest], MODE, O, D, t0, t1, closest)


for _ in range(3):
    frame()
torch.cuda.synchronize()
if WARM:
    _, _, waves1 = bench.make_workload_device(args, seed=1, scene_bvh=(sc, bvh))
    dw1 = [(w[2], *w[3:]) for w in waves1]

    def frame1():
        for closest, O, D, t0, t1 in dw1:
            hb.trace_wave(bvh, tables[closest], MODE, O, D, t0, t1, closest)

    for _ in range(2):
        frame()
        frame1()
    frame()
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    (frame1 if WARM else frame)()
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        ev.append((e.time_range.start, e.time_range.end, e.name[:60]))
ev.sort()
t0, t1 = ev[0][0], max(e[1] for e in ev)
busy_end = ev[0][1]
gaps = []
prev = ev[0]
for s, e, n in ev[1:]:
    if s > busy_end:
        gaps.append((s - busy_end, prev[2], n))
    if e > busy_end:
        busy_end, prev = e, (s, e, n)
tot = sum(g[0] for g in gaps)
print(f"frame span {(t1 - t0) / 1e3:.3f} ms, {len(ev)} activities, idle {tot / 1e3:.3f} ms in {len(gaps)} gaps")
for g in sorted(gaps, reverse=True)[:25]:
    print(f"{g[0]:8.1f} us  after {g[1]:60s} before {g[2]}")

if TL:
    print("\n# start_us  dur_us  kernel (one frame, all streams)")
    for s, e, n in ev:
        d = (e - s)
        if d >= 15:
            print(f"{(s - t0):9.1f} {d:8.1f}  {n}")
