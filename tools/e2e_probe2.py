"""Host-side timing of the double-buffered e2e pipeline (bench.run_e2e):
time blocked in trace_wave, in the upload and download enqueues."""
import os
import sys
import time
from argparse import Namespace
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1910_01304_b200 as hb  # noqa: E402

args = Namespace(config="c2", res=None, spp=None, precision=6, go_up=0)
sc, bvh, waves = bench.make_workload(args, lambda b, O, D, t0, t1:
                                     hb.intersect_closest_batch(b, O, D, t0, t1))
dev = torch.device("cuda")
cfg = hb.HashConfig(6)
tables = {True: hb.PredictorTable(cfg, 0, hb.RayKind.CLOSEST_HIT),
          False: hb.PredictorTable(cfg, 0, hb.RayKind.HIT_ANY)}
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
h_in = [[pin(a) for a in w[3:]] for w in waves]
h_out = []
for w in waves:
    n = w[3].shape[0]
    mk = lambda dt: torch.empty(n, dtype=dt).pin_memory()  # noqa: E731
    h_out.append({"found": mk(torch.bool), "t": mk(torch.float64), "slot": mk(torch.int32),
                  "leaf": mk(torch.int32)})
d_in = [[[torch.empty_like(t, device=dev) for t in h] for h in h_in] for _ in range(2)]
d_out = [[{k: torch.empty_like(v, device=dev) for k, v in h.items()} for h in h_out]
         for _ in range(2)]
copy, copy_back = torch.cuda.Stream(), torch.cuda.Stream()
stream = torch.cuda.current_stream()
W = len(waves)
gpu = []
mode = sys.argv[1] if len(sys.argv) > 1 else "default"


def run(frames):
    items = [(f, j) for f in range(frames) for j in range(W)]
    ev_up = [torch.cuda.Event() for _ in items]
    ev_comp = [torch.cuda.Event() for _ in items]
    ev_down = [torch.cuda.Event() for _ in items]
    tt = {"trace": 0.0, "up": 0.0, "down": 0.0}
    gpu.clear()

    def upload(i):
        a = time.perf_counter()
        f, j = items[i]
        with torch.cuda.stream(copy):
            if i >= 2 * W:
                copy.wait_event(ev_comp[i - 2 * W])
            for d_, h_ in zip(d_in[f % 2][j], h_in[j]):
                d_.copy_(h_, non_blocking=True)
            ev_up[i].record(copy)
        tt["up"] += time.perf_counter() - a

    for i in range(W):
        upload(i)
    for i, (f, j) in enumerate(items):
        if j == 0:
            for t in tables.values():
                t.clear()
        if i + W < len(items):
            upload(i + W)
        stream.wait_event(ev_up[i])
        if i >= 2 * W:
            stream.wait_event(ev_down[i - 2 * W])
        ca = torch.cuda.Event(enable_timing=True)
        cb = torch.cuda.Event(enable_timing=True)
        ua = torch.cuda.Event(enable_timing=True)
        ua.record(stream)
        stream.wait_event(ev_up[i])
        ca.record(stream)
        gpu.append((ua, ca, cb))
        a = time.perf_counter()
        hb.trace_wave(bvh, tables[waves[j][2]], "live", *d_in[f % 2][j], waves[j][2],
                      outputs=d_out[f % 2][j])
        tt["trace"] += time.perf_counter() - a
        cb.record(stream)
        ev_comp[i].record(stream)
        a = time.perf_counter()
        s_ = stream if mode == "same" else copy_back
        s_.wait_event(ev_comp[i])
        with torch.cuda.stream(s_):
            if mode == "one":  # one packed download per wave
                pass
            for k in h_out[j]:
                h_out[j][k].copy_(d_out[f % 2][j][k], non_blocking=True)
            ev_down[i].record(s_)
        tt["down"] += time.perf_counter() - a
    copy.synchronize()
    copy_back.synchronize()
    torch.cuda.synchronize()
    return tt


run(1)
t0 = time.perf_counter()
tt = run(10)
dt = time.perf_counter() - t0
comp = sum(c.elapsed_time(b) for _, c, b in gpu) / 10
wait = sum(u.elapsed_time(c) for u, c, _ in gpu) / 10
print(mode, f"{dt / 10 * 1e3:.2f} ms/frame", {k: round(v / 10 * 1e3, 2) for k, v in tt.items()},
      f"device compute {comp:.2f} ms/frame, compute stream waiting for uploads {wait:.2f}")
