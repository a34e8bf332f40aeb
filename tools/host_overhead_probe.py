"""Host time per wave: Python wrapper around hrpp_trace_wave vs the C call
itself (which includes the GPU work up to the end-of-wave sync), and the C
call's time before its first GPU work (tiny wave).  c2 live frame."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1910_01304_b200 as hb  # noqa: E402
from paper_1910_01304_b200 import _lib  # noqa: E402

args = bench.parse()
sc, bvh, waves = bench.make_workload(args, trace_closest=lambda b, O, D, t0, t1:
                                     hb.intersect_closest_batch(b, O, D, t0, t1))
dev = torch.device("cuda")
dw = [(w[2], *(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in w[3:])) for w in waves]
cfg = hb.HashConfig(args.precision)
tables = {c: hb.PredictorTable(cfg, args.go_up, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
          for c in (True, False)}
real = _lib.lib.hrpp_trace_wave
acc = {"c": 0.0}


def timed_call(*a):
    t = time.perf_counter()
    r = real(*a)
    acc["c"] += time.perf_counter() - t
    return r


class Shim:
    def __getattr__(self, k):
        return timed_call if k == "hrpp_trace_wave" else getattr(_lib.lib, k)


import paper_1910_01304_b200.tracer as tr  # noqa: E402
tr._lib = type("L", (), {})()
for k in dir(_lib):
    if not k.startswith("__"):
        setattr(tr._lib, k, getattr(_lib, k))
tr._lib.lib = Shim()
outs = [{"found": torch.empty(w[1].shape[0], dtype=torch.bool, device=dev),
         "t": torch.empty(w[1].shape[0], dtype=torch.float64, device=dev),
         "slot": torch.empty(w[1].shape[0], dtype=torch.int32, device=dev),
         "leaf": torch.empty(w[1].shape[0], dtype=torch.int32, device=dev)} for w in dw]
for pre in (False, True):
    for rep in range(5):
        for t in tables.values():
            t.clear()
        torch.cuda.synchronize()
        acc["c"] = 0.0
        tw = 0.0
        for j, (closest, O, D, t0, t1) in enumerate(dw):
            t = time.perf_counter()
            hb.trace_wave(bvh, tables[closest], "live", O, D, t0, t1, closest,
                          outputs=outs[j] if pre else None)
            tw += time.perf_counter() - t
    print("prealloc" if pre else "alloc", "wrapper-only %.1f us per wave" % (1e6 * (tw - acc["c"]) / 3))
# C call overhead on a 1-ray wave (no GPU work to speak of)
O, D = dw[0][1][:1].contiguous(), dw[0][2][:1].contiguous()
t0, t1 = dw[0][3][:1].contiguous(), dw[0][4][:1].contiguous()
for _ in range(5):
    tables[True].clear()
    hb.trace_wave(bvh, tables[True], "live", O, D, t0, t1, True)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    tables[True].clear()
    torch.cuda.synchronize()
    acc["c"] = 0.0
    hb.trace_wave(bvh, tables[True], "live", O, D, t0, t1, True)
    ts.append(acc["c"])
print("1-ray wave: C call %.1f us (median)" % (1e6 * float(np.median(ts))))
