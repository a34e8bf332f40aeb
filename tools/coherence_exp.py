"""Experiment: does sorting secondary rays by a coherence key speed up traversal?"""
import json, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1910_01304_b200 as hb
from paper_1910_01304_b200 import scenes


def part1by2(x):
    x = x.astype(np.uint64) & np.uint64(0x3FF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x30000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x300F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x30C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x9249249)
    return x


def key(O, D, obits, dbits):
    lo, hi = O.min(0), O.max(0)
    q = ((O - lo) / np.maximum(hi - lo, 1e-9) * (2 ** obits - 1)).astype(np.uint64)
    morton = part1by2(q[:, 0]) | (part1by2(q[:, 1]) << np.uint64(1)) | (part1by2(q[:, 2]) << np.uint64(2))
    dq = ((D + 1.0) * 0.5 * (2 ** dbits - 1)).astype(np.uint64)
    dm = part1by2(dq[:, 0]) | (part1by2(dq[:, 1]) << np.uint64(1)) | (part1by2(dq[:, 2]) << np.uint64(2))
    octant = (D[:, 0] < 0).astype(np.uint64) | ((D[:, 1] < 0).astype(np.uint64) << np.uint64(1)) | ((D[:, 2] < 0).astype(np.uint64) << np.uint64(2))
    return (octant << np.uint64(60)) | (dm << np.uint64(3 * obits)) | morton


def main():
    sc = scenes.make_scene("c2")
    b = hb.build_bvh_from_arrays(sc.v0, sc.v1, sc.v2)
    O, D = scenes.primary_rays(sc.camera, sc.spp, seed=0)
    n = O.shape[0]
    base = hb.intersect_closest_batch(b, O, D, np.zeros(n), np.full(n, np.inf))
    _, P, N = scenes.hit_frames(O, D, base["found"], base["t"], base["slot"], scenes.slot_normals(b.tv0, b.tv1, b.tv2))
    lp = scenes.area_light_samples(P.shape[0], *sc.area_light, seed=0)
    waves = {"shadow": (False, *scenes.shadow_rays(P, lp)), "bounce": (True, *scenes.cosine_bounce(P, N, seed=0))}
    dev = torch.device("cuda")
    out = {}
    for name, (closest, Ow, Dw, t0, t1) in waves.items():
        for label, order in [("ray_order", np.arange(len(Ow)))] + [
                (f"o{ob}_d{db}", np.argsort(key(Ow, Dw, ob, db), kind="stable")) for ob, db in ((10, 0), (6, 3), (5, 5), (4, 6))]:
            T = [torch.from_numpy(np.ascontiguousarray(x[order])).to(dev) for x in (Ow, Dw, t0, t1)]
            fn = (lambda: hb.intersect_closest_batch(b, *T)) if closest else (lambda: hb.intersect_any_batch(b, *T))
            for _ in range(3): fn()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            out[f"{name}_{label}"] = round(float(np.median(ts)), 3)
    print(json.dumps(out))


main()
