"""traversal time of the rays each key owner would hold (N ranks,
owner = (mix64(key) >> 32) % N, ray order kept) against contiguous blocks of
the same sizes, on one GPU (the coherence cost of exact key sharding)."""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_1910_01304_b200 as hb
from paper_1910_01304_b200.parallel import partition_by_owner
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, waves = bench.make_workload(args, lambda bv, O, D, a, c: hb.intersect_closest_batch(bv, O, D, a, c))
dev = torch.device("cuda")
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for name, kind, closest, O, D, t0, t1 in waves[:3]:
    Od, Dd = torch.from_numpy(O).to(dev), torch.from_numpy(D).to(dev)
    a, c = torch.from_numpy(t0).to(dev), torch.from_numpy(t1).to(dev)
    f = hb.intersect_closest_batch if closest else hb.intersect_any_batch
    keys = hb.hash_rays(Od, Dd, hb.HashConfig(6))
    perm, counts = partition_by_owner(keys, N)
    perm = perm.long()
    sizes = counts.tolist()
    own, blk = [], []
    start = 0
    n = Od.shape[0]
    for r, m in enumerate(sizes):
        idx = perm[start:start + m]; start += m
        Oo, Do, ao, co = Od[idx].contiguous(), Dd[idx].contiguous(), a[idx].contiguous(), c[idx].contiguous()
        own.append(timeit(lambda: f(b, Oo, Do, ao, co)))
        lo = (n * r) // N; hi = lo + m
        Ob, Db, ab, cb = Od[lo:hi].contiguous(), Dd[lo:hi].contiguous(), a[lo:hi].contiguous(), c[lo:hi].contiguous()
        blk.append(timeit(lambda: f(b, Ob, Db, ab, cb)))
    print(json.dumps({"wave": name, "N": N, "owner_ms_sum": round(sum(own), 3), "block_ms_sum": round(sum(blk), 3),
                      "owner_max": round(max(own), 3), "block_max": round(max(blk), 3),
                      "full_ms": round(timeit(lambda: f(b, Od, Dd, a, c)), 3), "sizes": sizes}), flush=True)
