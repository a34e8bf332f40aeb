"""Where the e2e frame time goes: uploads alone, device-resident compute
alone, and the pipelined host-buffer loop with per-wave host timestamps."""
import sys
import time
from argparse import Namespace
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1910_01304_b200 as hb  # noqa: E402


def main():
    args = Namespace(config="c2", res=None, spp=None, precision=6, go_up=0)
    sc, bvh, waves = bench.make_workload(args, lambda b, O, D, t0, t1:
                                         hb.intersect_closest_batch(b, O, D, t0, t1))
    dev = torch.device("cuda")
    cfg = hb.HashConfig(6)
    tables = {True: hb.PredictorTable(cfg, 0, hb.RayKind.CLOSEST_HIT),
              False: hb.PredictorTable(cfg, 0, hb.RayKind.HIT_ANY)}
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h_in = [[pin(a) for a in w[3:]] for w in waves]
    d_in = [[torch.empty_like(t, device=dev) for t in h] for h in h_in]
    copy = torch.cuda.Stream()
    stream = torch.cuda.current_stream()

    def uploads(frames):
        for _ in range(frames):
            for j in range(len(waves)):
                with torch.cuda.stream(copy):
                    for d_, h_ in zip(d_in[j], h_in[j]):
                        d_.copy_(h_, non_blocking=True)
        copy.synchronize()

    def compute(frames):
        for _ in range(frames):
            for t in tables.values():
                t.clear()
            for j, w in enumerate(waves):
                hb.trace_wave(bvh, tables[w[2]], "live", *d_in[j], w[2])
        torch.cuda.synchronize()

    for name, fn in (("uploads", uploads), ("compute", compute)):
        fn(1)
        t0 = time.perf_counter()
        fn(3)
        print(f"{name}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms/frame")

    # pipelined like bench.run_e2e, with host timestamps
    n_fr = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    with_d2h = len(sys.argv) > 2 and sys.argv[2] == "d2h"
    copy_back = torch.cuda.Stream()
    h_out, d_out = [], []
    for w in waves:
        n = w[3].shape[0]
        h_out.append({"found": torch.empty(n, dtype=torch.bool).pin_memory(),
                      "t": torch.empty(n, dtype=torch.float64).pin_memory(),
                      "slot": torch.empty(n, dtype=torch.int32).pin_memory(),
                      "leaf": torch.empty(n, dtype=torch.int32).pin_memory()})
        d_out.append({k: torch.empty_like(v, device=dev) for k, v in h_out[-1].items()})
    items = [(f, j) for f in range(n_fr) for j in range(len(waves))]
    ev_in = [torch.cuda.Event() for _ in items]

    def upload(i):
        _, j = items[i]
        with torch.cuda.stream(copy):
            for d_, h_ in zip(d_in[j], h_in[j]):
                d_.copy_(h_, non_blocking=True)
            ev_in[i].record(copy)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    upload(0)
    marks = []
    for i, (f, j) in enumerate(items):
        if j == 0:
            for t in tables.values():
                t.clear()
        if i + 1 < len(items):
            upload(i + 1)
        a = time.perf_counter()
        stream.wait_event(ev_in[i])
        hb.trace_wave(bvh, tables[waves[j][2]], "live", *d_in[j], waves[j][2],
                      outputs=d_out[j])
        if with_d2h:
            done = torch.cuda.Event()
            done.record(stream)
            copy_back.wait_event(done)
            with torch.cuda.stream(copy_back):
                for k in h_out[j]:
                    h_out[j][k].copy_(d_out[j][k], non_blocking=True)
        marks.append((f, waves[j][0], round((a - t0) * 1e3, 2),
                      round((time.perf_counter() - t0) * 1e3, 2)))
    torch.cuda.synchronize()
    copy_back.synchronize()
    tot = time.perf_counter() - t0
    for m in marks[-6:]:
        print("frame %d %-10s host start %7.2f ms  returned %7.2f ms" % m)
    print(f"pipelined ({n_fr} frames, d2h={with_d2h}): {tot / n_fr * 1e3:.2f} ms/frame")


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "copies"):
    main()


def copies_only():
    """uploads and downloads of the same sizes, no compute, both engines."""
    args = Namespace(config="c2", res=None, spp=None, precision=6, go_up=0)
    _, _, waves = bench.make_workload(args, lambda b, O, D, t0, t1:
                                      hb.intersect_closest_batch(b, O, D, t0, t1))
    dev = torch.device("cuda")
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h_in = [[pin(a) for a in w[3:]] for w in waves]
    d_in = [[torch.empty_like(t, device=dev) for t in h] for h in h_in]
    h_out = [torch.empty(w[3].shape[0] * 17, dtype=torch.uint8).pin_memory() for w in waves]
    d_out = [torch.empty_like(h, device=dev) for h in h_out]
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    for mode in ("up", "down", "both"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            for j in range(len(waves)):
                if mode in ("up", "both"):
                    with torch.cuda.stream(up):
                        for d_, h_ in zip(d_in[j], h_in[j]):
                            d_.copy_(h_, non_blocking=True)
                if mode in ("down", "both"):
                    with torch.cuda.stream(down):
                        h_out[j].copy_(d_out[j], non_blocking=True)
        torch.cuda.synchronize()
        print(f"copies {mode}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms/frame")


if len(sys.argv) > 1 and sys.argv[1] == "copies":
    copies_only()
