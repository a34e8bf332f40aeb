"""does reordering a wave for coherence speed up full traversal?"""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, waves = bench.make_workload(args, lambda bv, O, D, a, c: hb.intersect_closest_batch(bv, O, D, a, c))
dev = torch.device("cuda")
lo = torch.tensor(b.bmin[0], device=dev, dtype=torch.float32); hi = torch.tensor(b.bmax[0], device=dev, dtype=torch.float32)
def part1by2(x):
    x = x & 0x3FF
    x = (x | (x << 16)) & 0x030000FF
    x = (x | (x << 8)) & 0x0300F00F
    x = (x | (x << 4)) & 0x030C30C3
    x = (x | (x << 2)) & 0x09249249
    return x
def keys(O, D, mode):
    q = ((O - lo) / (hi - lo)).clamp(0, 1)
    qi = (q * 1023).long()
    morton = part1by2(qi[:, 0]) | (part1by2(qi[:, 1]) << 1) | (part1by2(qi[:, 2]) << 2)
    octant = ((D[:, 0] < 0).long()) | ((D[:, 1] < 0).long() << 1) | ((D[:, 2] < 0).long() << 2)
    dq = (((D + 1) * 0.5).clamp(0, 1) * 15).long()
    dk = dq[:, 0] | (dq[:, 1] << 4) | (dq[:, 2] << 8)
    if mode == "octant": return octant
    if mode == "morton": return morton
    if mode == "oct_morton": return (octant << 30) | morton
    if mode == "dir_morton": return (dk << 30) | morton
    if mode == "oct_dir": return (octant << 12) | dk
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for name, kind, closest, O, D, t0, t1 in waves:
    Od, Dd = torch.from_numpy(O).to(dev), torch.from_numpy(D).to(dev)
    a, c = torch.from_numpy(t0).to(dev), torch.from_numpy(t1).to(dev)
    f = hb.intersect_closest_batch if closest else hb.intersect_any_batch
    res = {"wave": name, "orig": round(timeit(lambda: f(b, Od, Dd, a, c)), 3)}
    for mode in ("octant", "morton", "oct_morton", "dir_morton", "oct_dir"):
        k = keys(Od, Dd, mode)
        perm = torch.sort(k, stable=True).indices
        Op, Dp, ap, cp = Od[perm].contiguous(), Dd[perm].contiguous(), a[perm].contiguous(), c[perm].contiguous()
        res[mode] = round(timeit(lambda: f(b, Op, Dp, ap, cp)), 3)
    print(json.dumps(res), flush=True)
