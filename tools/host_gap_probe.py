"""Where the gaps between device stages go: wall time per live c2 frame vs
time inside the C call (hrpp_trace_wave) vs the Python around it."""
import sys
import time
from argparse import Namespace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1910_01304_b200 as hb  # noqa: E402
from paper_1910_01304_b200 import _lib  # noqa: E402

args = Namespace(config="c2", res=None, spp=None, precision=6, go_up=0)
sc, bvh, waves = bench.make_workload(args, lambda b, O, D, t0, t1:
                                     hb.intersect_closest_batch(b, O, D, t0, t1))
cfg = hb.HashConfig(6)
tables = {True: hb.PredictorTable(cfg, 0, hb.RayKind.CLOSEST_HIT),
          False: hb.PredictorTable(cfg, 0, hb.RayKind.HIT_ANY)}
dev = [(w[2], *(torch.from_numpy(a).cuda() for a in w[3:])) for w in waves]
orig = _lib.lib
real = orig.hrpp_trace_wave
acc = {"c": 0.0}


def timed(*a):
    t = time.perf_counter()
    r = real(*a)
    acc["c"] += time.perf_counter() - t
    return r


class Shim:
    def __getattr__(self, k):
        return timed if k == "hrpp_trace_wave" else getattr(orig, k)


def frame():
    for t in tables.values():
        t.clear()
    for c, O, D, t0, t1 in dev:
        hb.trace_wave(bvh, tables[c], "live", O, D, t0, t1, c)


for _ in range(3):
    frame()
torch.cuda.synchronize()
_lib.lib = Shim()
import paper_1910_01304_b200.tracer as tr  # noqa: E402
tr._lib.lib = _lib.lib
N = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
e0.record()
for _ in range(N):
    frame()
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / N * 1e3
print(f"wall {wall:.2f} ms/frame, device {e0.elapsed_time(e1) / N:.2f}, inside C "
      f"{acc['c'] / N * 1e3:.2f}, python around it {wall - acc['c'] / N * 1e3:.2f}")
