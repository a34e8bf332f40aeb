"""Which key bits vary within each wave of a frame (the grouping sort only
needs those): python tools/key_bits.py <config> [precision]"""
import sys, json
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 6
args = Namespace(config=cfg, res=None, spp=None, precision=p, go_up=0)
sc, b, waves = bench.make_workload_device(args)
for name, kind, closest, O, D, a, c in waves:
    k = hb.hash_rays(O, D, hb.HashConfig(p)).view(torch.int64)
    o = a_ = None
    kk = k.cpu().numpy().view("uint64")
    import numpy as np
    o = int(np.bitwise_or.reduce(kk)); an = int(np.bitwise_and.reduce(kk))
    vary = o & ~an
    lanes = [(vary >> s) & 0xFFFF for s in (0, 16, 32)]
    print(json.dumps({"cfg": cfg, "wave": name, "n": int(kk.size), "distinct": int(np.unique(kk).size),
                      "varying_bits": bin(vary).count("1"),
                      "lanes": [format(x, "013b") for x in lanes]}), flush=True)
