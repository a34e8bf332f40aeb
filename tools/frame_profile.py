"""a few c2 frames in a given mode (for ncu launch lists)."""
import sys
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_1910_01304_b200 as hb
cfg = sys.argv[1]; mode = sys.argv[2]; frames = int(sys.argv[3]) if len(sys.argv) > 3 else 2
args = Namespace(config=cfg, res=None, spp=None, precision=6, go_up=0)
sc, b, waves = bench.make_workload(args, lambda bv, O, D, a, c: hb.intersect_closest_batch(bv, O, D, a, c))
dev = torch.device("cuda")
dw = [(w[0], w[2], *(torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in w[3:])) for w in waves]
tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY) for c in (True, False)}
for f in range(frames):
    for t in tabs.values(): t.clear()
    for name, closest, O, D, a, c in dw:
        hb.trace_wave(b, tabs[closest] if mode != "baseline" else None, mode, O, D, a, c, closest)
torch.cuda.synchronize()
print("done")
