"""Micro-benchmark of the full-traversal kernel on the c2 primary wave.

    HRPP_LIB=exp/x/libhrpp_b200.so python tools/trace_bench.py [--config c2]

Prints ms per 8.4M-ray closest-hit batch and per shadow (hit-any) batch,
CUDA-event timed on device-resident inputs (median of 7 after 3 warm-ups).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1910_01304_b200 as hb  # noqa: E402
from paper_1910_01304_b200 import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--res", default=None)
    a = ap.parse_args()
    res = tuple(int(x) for x in a.res.split("x")) if a.res else None
    sc = scenes.make_scene(a.config, resolution=res)
    b = hb.build_bvh_from_arrays(sc.v0, sc.v1, sc.v2, median_split=sc.builder == "median")
    O, D = scenes.primary_rays(sc.camera, sc.spp, seed=0)
    n = O.shape[0]
    dev = torch.device("cuda")
    Ot, Dt = torch.from_numpy(O).to(dev), torch.from_numpy(D).to(dev)
    t0 = torch.zeros(n, dtype=torch.float64, device=dev)
    t1 = torch.full((n,), float("inf"), dtype=torch.float64, device=dev)
    base = hb.intersect_closest_batch(b, O, D, np.zeros(n), np.full(n, np.inf))
    _, P, N = scenes.hit_frames(O, D, base["found"], base["t"], base["slot"],
                                scenes.slot_normals(b.tv0, b.tv1, b.tv2))
    lp = (scenes.area_light_samples(P.shape[0], *sc.area_light, seed=0) if sc.area_light
          else np.broadcast_to(np.asarray(sc.point_lights[0]), P.shape))
    so, sd, s0, s1 = scenes.shadow_rays(P, lp)
    S = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (so, sd, s0, s1)]
    bo, bd, b0, b1 = scenes.cosine_bounce(P, N, seed=0)
    B = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (bo, bd, b0, b1)]

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    ms_c = timeit(lambda: hb.intersect_closest_batch(b, Ot, Dt, t0, t1))
    import hashlib

    def digest(res):
        m = hashlib.md5()
        for k in sorted(res):
            v = res[k]
            v = v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)
            m.update(k.encode())
            m.update(np.ascontiguousarray(v).tobytes())
        return m.hexdigest()[:10]

    dig = "-".join(digest(f()) for f in (
        lambda: hb.intersect_closest_batch(b, Ot, Dt, t0, t1),
        lambda: hb.intersect_any_batch(b, *S), lambda: hb.intersect_closest_batch(b, *B)))
    ms_a = timeit(lambda: hb.intersect_any_batch(b, *S))
    ms_b = timeit(lambda: hb.intersect_closest_batch(b, *B))
    print(json.dumps({"closest_ms": round(ms_c, 4), "closest_mrays_s": round(n / ms_c / 1e3, 1),
                      "any_ms": round(ms_a, 4), "any_mrays_s": round(len(so) / ms_a / 1e3, 1),
                      "bounce_ms": round(ms_b, 4), "bounce_mrays_s": round(len(bo) / ms_b / 1e3, 1),
                      "mean_box": float(base["box"].mean()), "n": n, "digest": dig}))


if __name__ == "__main__":
    main()
