"""Host overhead per wave: host wall time of each trace_wave call vs the GPU
time between events recorded just before and after it (c2 live frame)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1910_01304_b200 as hb  # noqa: E402

args = bench.parse()
args.res = None
sc, bvh, waves = bench.make_workload(args, trace_closest=lambda b, O, D, t0, t1:
                                     hb.intersect_closest_batch(b, O, D, t0, t1))
dev = torch.device("cuda")
dw = [(w[2], *(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in w[3:])) for w in waves]
cfg = hb.HashConfig(6)
tables = {c: hb.PredictorTable(cfg, 0, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
          for c in (True, False)}
outs = [{"found": torch.empty(w[1].shape[0], dtype=torch.bool, device=dev),
         "t": torch.empty(w[1].shape[0], dtype=torch.float64, device=dev),
         "slot": torch.empty(w[1].shape[0], dtype=torch.int32, device=dev),
         "leaf": torch.empty(w[1].shape[0], dtype=torch.int32, device=dev)} for w in dw]
for pre in (False, True):
    for rep in range(4):
        for t in tables.values():
            t.clear()
        torch.cuda.synchronize()
        rows = []
        f0 = time.perf_counter()
        for j, (closest, O, D, t0, t1) in enumerate(dw):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0 = time.perf_counter()
            e0.record()
            hb.trace_wave(bvh, tables[closest], "live", O, D, t0, t1, closest,
                          outputs=outs[j] if pre else None)
            e1.record()
            h1 = time.perf_counter()
            torch.cuda.synchronize()
            rows.append((1e3 * (h1 - h0), e0.elapsed_time(e1)))
        f1 = time.perf_counter()
        if rep == 3:
            print("prealloc" if pre else "alloc", "frame wall %.3f ms" % (1e3 * (f1 - f0)),
                  " ".join("host %.3f gpu %.3f" % r for r in rows))
