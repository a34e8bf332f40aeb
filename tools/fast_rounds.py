import sys, time
import numpy as np
from argparse import Namespace
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import bench
from oracle import oracle
cfg = sys.argv[1]; p = int(sys.argv[2]) if len(sys.argv) > 2 else 6
rounds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2, 4, 8, 1000]
args = Namespace(config=cfg, res=None, spp=None, precision=p, go_up=0)
sc, ob, waves = bench.make_workload(args, lambda b, O, D, a, c: b.trace_batch(True, O, D, a, c, threads=0), build=oracle.build_bvh)
def run(mode):
    tabs = {c: oracle.OracleTable(p, 0, c) for c in (True, False)}
    tot = {}; outs = []
    for name, kind, closest, O, D, a, b in waves:
        rc, out, st = oracle.trace_wave(ob, tabs[closest], mode, closest, O, D, a, b, threads=1)
        tot[kind] = tot.get(kind, 0) + st; outs.append(out)
    return tot, {c: tabs[c].dump_lines() for c in tabs}, outs
ref = run("live")
for R in rounds:
    oracle.set_fast_rounds(R, int(sys.argv[4]) if len(sys.argv) > 4 else 32)
    t0 = time.time(); got = run("fast"); dt = time.time() - t0
    same = all(np.array_equal(got[0][k], ref[0][k]) for k in ref[0]) and got[1] == ref[1]
    msg = []
    for k in ref[0]:
        a, b = ref[0][k], got[0][k]
        msg.append(f"{k}: tp {b[1]}/{a[1]} ({100*(b[1]-a[1])/max(a[1],1):+.2f}%) bb {100*(b[4]-a[4])/max(a[4],1):+.2f}%")
    print(f"R={R} exact={same} {dt:.1f}s | " + " | ".join(msg), flush=True)
oracle.set_fast_rounds(1000, 0)
got = run("fast")
for k in ref[0]:
    print(k, ref[0][k], got[0][k])
for c in (True, False):
    a, b = ref[1][c], got[1][c]
    d = [(x, y) for x, y in zip(a, b) if x != y]
    print(c, len(a), len(b), d[:3])
for w, (x, y) in enumerate(zip(ref[2], got[2])):
    for k in ("found", "t", "slot", "leaf"):
        if not np.array_equal(x[k], y[k]): print("wave", w, k, np.flatnonzero(x[k] != y[k])[:5])
