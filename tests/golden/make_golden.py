"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``hrpp`` from /root/reference/pkg/src (read-only; numba's cache is
redirected to /tmp so nothing is written into the reference tree) and writes
compressed ``.npz`` fixtures next to this script.  The fixtures are committed;
the GPU box never reads /root/reference.

Fixtures:

* ``hash.npz``      -- hrpp/rayhash.py:99-115 keys for p = 1..7 over random
  and edge-case floats (signed zeros, denormals, huge values).
* ``bvh_<name>.npz`` -- BVH arrays from the reference SAH builder
  (hrpp/bvh.py:184-276) for: ``strip8`` (8 separated tris, leaf size 1),
  ``soup256`` (tests/helpers.py random_soup(256, seed=7)), ``spheres``
  (bundled scene) and ``ico1282`` (this repo's c1 icosphere generator;
  checks the native builder).
* ``trace_<name>.npz`` -- intersect_{closest,any}_batch outputs
  (hrpp/bvh.py:398-442).
* ``wave_<tag>.npz`` -- _trace_wave (hrpp/tracer.py:343-371) in limit mode
  with the OutcomeLog captured, and in live mode, for a primary ->
  shadow -> reflection wave sequence at several (p, go_up) settings,
  plus RayKindStats and PredictorTable.dump_lines after every wave.
* ``predict.npz``  -- PredictorTable.predict (hrpp/predictor.py:167-192)
  against a frozen trained table.
* ``record.npz``   -- PredictorTable.record sequence semantics.
"""

from __future__ import annotations

import dataclasses
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hrpp_numba_cache")
sys.dont_write_bytecode = True  # never write __pycache__ into /root/reference
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, "/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import hrpp  # noqa: E402
from hrpp import HashConfig, PredictorTable, RayKind, RenderConfig, RenderMode  # noqa: E402
from hrpp.bvh import (build_bvh, build_bvh_from_arrays, intersect_any_batch,  # noqa: E402
                      intersect_closest_batch)
from hrpp.metrics import RayKindStats  # noqa: E402
from hrpp.scene_io import load_bundled_scene  # noqa: E402
from hrpp.tracer import _trace_wave, generate_primary_rays  # noqa: E402
from helpers import random_rays, random_soup, separated_strip  # noqa: E402

OUT = Path(__file__).resolve().parent
STATS_FIELDS = [f.name for f in dataclasses.fields(RayKindStats)]


def bvh_dict(b):
    return dict(bmin=b.bmin, bmax=b.bmax, left=b.left, right=b.right, axis=b.axis,
                first=b.first, count=b.count, parent=b.parent, depth=b.depth, tv0=b.tv0,
                tv1=b.tv1, tv2=b.tv2, tri_ids=b.tri_ids, max_depth=np.int64(b.max_depth))


def save(name, **arrays):
    np.savez_compressed(OUT / name, **arrays)
    print("wrote", name, sum(np.asarray(a).nbytes for a in arrays.values()), "bytes raw")


def make_hash():
    rng = np.random.default_rng(1234)
    n = 4096
    O = rng.uniform(-100, 100, (n, 3)).astype(np.float32)
    D = rng.normal(size=(n, 3))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    D = D.astype(np.float32)
    # edge cases: signed zeros, denormals, huge and tiny magnitudes
    special = np.array([0.0, -0.0, 1e-40, -1e-40, 1.0, -1.0, 3.4e38, -3.4e38, 1e-30, 2.0 ** -126,
                        0.5, -0.5, 65504.0, 1.0 + 2 ** -23, 7.0, -7.25], np.float32)
    m = 512
    O[:m] = special[rng.integers(0, len(special), (m, 3))]
    D[m:2 * m] = special[rng.integers(0, len(special), (m, 3))]
    keys = np.stack([hrpp.hash_rays(O, D, HashConfig(p)) for p in range(1, 8)])
    scal = np.array([[hrpp.map_float_to_hash(f, HashConfig(p)) for f in special]
                     for p in range(1, 8)], np.int64)
    save("hash.npz", O=O, D=D, keys=keys, special=special, special_hash=scal)


def make_bvhs():
    out = {}
    strip = build_bvh(separated_strip(8), max_leaf_size=1)
    out["strip8"] = strip
    soup = build_bvh(random_soup(256, seed=7), max_leaf_size=4)
    out["soup256"] = soup
    sc = load_bundled_scene("spheres")
    out["spheres"] = build_bvh_from_arrays(sc.v0, sc.v1, sc.v2)
    from paper_1910_01304_b200.scenes import make_scene
    ico = make_scene("c1")
    out["ico1282"] = build_bvh_from_arrays(ico.v0, ico.v1, ico.v2, max_leaf_size=4)
    for k, b in out.items():
        hrpp.bvh.validate(b)
        d = bvh_dict(b)
        if k == "ico1282":
            d.update(in_v0=ico.v0, in_v1=ico.v1, in_v2=ico.v2)
        save(f"bvh_{k}.npz", **d)
    return out, sc


def make_trace(bvhs):
    soup = bvhs["soup256"]
    O, D = random_rays(3000, seed=21)
    n = O.shape[0]
    tmax_any = np.random.default_rng(5).uniform(2.0, 14.0, n)
    c = intersect_closest_batch(soup, O, D, np.zeros(n), np.full(n, np.inf))
    a = intersect_any_batch(soup, O, D, np.zeros(n), tmax_any)
    # start at a non-root node too
    c7 = intersect_closest_batch(soup, O, D, np.zeros(n), np.full(n, np.inf), start=7)
    save("trace_soup256.npz", O=O, D=D, tmax_any=tmax_any,
         **{f"c_{k}": v for k, v in c.items()}, **{f"a_{k}": v for k, v in a.items()},
         **{f"c7_{k}": v for k, v in c7.items()})
    # axis-aligned rays hit the zero-direction (signed-inf reciprocal) path
    strip = bvhs["strip8"]
    Oa = np.array([[2.0 * i + 0.25, 0.25, -5.0] for i in range(8)] +
                  [[0.0, 0.0, -5.0], [1.0, 0.0, -5.0], [0.0, 1.0, -5.0], [16.0, 0.5, -1.0],
                   [0.5, 0.25, 5.0], [-1.0, 0.25, 0.0]], np.float32)
    Da = np.array([[0, 0, 1]] * 8 + [[0, 0, 1]] * 3 + [[-1, 0, 0], [0, 0, -1], [1, 0, 0]],
                  np.float32)
    Da[-1] = [1.0, -0.0, 0.0]
    m = Oa.shape[0]
    c = intersect_closest_batch(strip, Oa, Da, np.zeros(m), np.full(m, np.inf))
    a = intersect_any_batch(strip, Oa, Da, np.zeros(m), np.full(m, 100.0))
    save("trace_strip8.npz", O=Oa, D=Da, **{f"c_{k}": v for k, v in c.items()},
         **{f"a_{k}": v for k, v in a.items()})


def spawn_shadow(bvh, O, D, base, light):
    """Shadow rays exactly as hrpp/tracer.py:442-464 spawns them."""
    hit = base["found"]
    ho = O[hit].astype(np.float64)
    hd = D[hit].astype(np.float64)
    P = ho + base["t"][hit][:, None] * hd
    N = bvh.slot_normals()[base["slot"][hit]]
    facing = np.einsum("ij,ij->i", N, hd)
    N = np.where(facing[:, None] > 0.0, -N, N)
    offset_P = P + 1e-4 * N
    lvec = np.asarray(light, np.float64)[None, :] - offset_P
    dist = np.maximum(np.linalg.norm(lvec, axis=1), 1e-9)
    ldir = lvec / dist[:, None]
    so = offset_P.astype(np.float32)
    sd = ldir.astype(np.float32)
    stmax = np.maximum(dist - 1e-4, 1e-6)
    # mirror bounce (hrpp/tracer.py:488-492), every hit reflects here
    rdot = np.einsum("ij,ij->i", hd, N)
    rdir = hd - 2.0 * rdot[:, None] * N
    rdir /= np.linalg.norm(rdir, axis=1, keepdims=True)
    return so, sd, stmax, offset_P.astype(np.float32), rdir.astype(np.float32)


def make_waves(bvhs, scene):
    bvh = bvhs["spheres"]
    cam = dataclasses.replace(scene.camera, resolution=(48, 48))
    O, D = generate_primary_rays(cam, RenderConfig(spp=4, rng_seed=0))
    n = O.shape[0]
    base = intersect_closest_batch(bvh, O, D, np.zeros(n), np.full(n, np.inf))
    so, sd, stmax, ro, rd = spawn_shadow(bvh, O, D, base, scene.lights[0].position)
    waves = [("primary", True, O, D, np.zeros(n), np.full(n, np.inf)),
             ("shadow", False, so, sd, np.zeros(len(so)), stmax),
             ("reflection", True, ro, rd, np.zeros(len(ro)), np.full(len(ro), np.inf))]
    arrays = {}
    for wname, closest, Ow, Dw, t0, t1 in waves:
        arrays[f"{wname}_O"] = Ow
        arrays[f"{wname}_D"] = Dw
        arrays[f"{wname}_tmin"] = t0
        arrays[f"{wname}_tmax"] = t1
    save("wave_inputs.npz", **arrays)

    for (p, g) in ((6, 0), (3, 0), (4, 2), (7, 1)):
        for mode in (RenderMode.LIMIT, RenderMode.LIVE):
            cfg = HashConfig(p)
            tables = {True: PredictorTable(cfg, g, kind=RayKind.CLOSEST_HIT),
                      False: PredictorTable(cfg, g, kind=RayKind.HIT_ANY)}
            res = {}
            for wname, closest, Ow, Dw, t0, t1 in waves:
                stats = RayKindStats()
                ll = ({"cls": [], "eval_box": [], "base_box": [], "pred_t": [], "pred_slot": [],
                       "keys": []} if mode is RenderMode.LIMIT else None)
                out = _trace_wave(bvh, tables[closest], None, mode, Ow, Dw, t0, t1, stats,
                                  closest=closest, log_lists=ll)
                for k, v in out.items():
                    res[f"{wname}_{k}"] = np.asarray(v)
                res[f"{wname}_stats"] = np.array([getattr(stats, f) for f in STATS_FIELDS],
                                                 np.int64)
                if ll is not None:
                    res[f"{wname}_log_cls"] = np.array(ll["cls"], np.int8)
                    res[f"{wname}_log_eval_box"] = np.array(ll["eval_box"], np.int64)
                    res[f"{wname}_log_base_box"] = np.array(ll["base_box"], np.int64)
                    res[f"{wname}_log_pred_t"] = np.array(ll["pred_t"], np.float64)
                    res[f"{wname}_log_pred_slot"] = np.array(ll["pred_slot"], np.int64)
                    res[f"{wname}_log_keys"] = np.array(ll["keys"], np.uint64)
                res[f"{wname}_dump"] = np.array(list(tables[closest].dump_lines()))
                ts = hrpp.table_stats(tables[closest])
                res[f"{wname}_tstats"] = np.array(
                    [ts.entries, ts.stored_nodes, ts.max_nodes_per_entry,
                     ts.memory.total_bytes], np.int64)
            save(f"wave_{mode.value}_p{p}_g{g}.npz", **res)


def make_predict(bvhs):
    soup = bvhs["soup256"]
    O, D = random_rays(1500, seed=77)
    n = O.shape[0]
    res = intersect_closest_batch(soup, O, D, np.zeros(n), np.full(n, np.inf))
    out = {}
    for kind, closest in ((RayKind.CLOSEST_HIT, True), (RayKind.HIT_ANY, False)):
        t = PredictorTable(HashConfig(4), 1 if closest else 0, kind=kind)
        keys = hrpp.hash_rays(O, D, t.cfg)
        lut = soup.ancestor_lut(t.go_up_level)
        # train on the first half, predict on everything (frozen table)
        for i in range(n // 2):
            if res["found"][i]:
                t.record(int(keys[i]), int(lut[res["leaf"][i]]))
        cls, tt, tri_id, leaf, box, est = [], [], [], [], [], []
        for i in range(n):
            r = hrpp.Ray(O[i], D[i], kind=kind, t_max=(np.inf if closest else 6.0))
            o = t.predict(soup, r)
            cls.append({"true_positive": 0, "false_positive": 1,
                        "negative": 2}[o.classification.value])
            tt.append(o.hit.t if o.hit else np.inf)
            tri_id.append(o.hit.triangle_id if o.hit else -1)
            leaf.append(o.hit.leaf_node if o.hit else -1)
            box.append(o.overhead.box_tests)
            est.append(o.skipped_box_tests)
        pre = "c" if closest else "a"
        out.update({f"{pre}_cls": np.array(cls, np.int8), f"{pre}_t": np.array(tt),
                    f"{pre}_tri_id": np.array(tri_id, np.int64),
                    f"{pre}_leaf": np.array(leaf, np.int64), f"{pre}_box": np.array(box, np.int64),
                    f"{pre}_est": np.array(est, np.int64),
                    f"{pre}_dump": np.array(list(t.dump_lines()))})
    save("predict.npz", O=O, D=D, **out)


def make_record():
    rng = np.random.default_rng(99)
    keys = rng.integers(0, 40, 600).astype(np.uint64) * np.uint64(0x10001)
    nodes = rng.integers(0, 25, 600).astype(np.int32)
    t = PredictorTable(HashConfig(6), 0)
    ins = np.array([t.record(int(k), int(v)) for k, v in zip(keys, nodes)], np.bool_)
    ts = hrpp.table_stats(t)
    save("record.npz", keys=keys, nodes=nodes, inserted=ins, dump=np.array(list(t.dump_lines())),
         tstats=np.array([ts.entries, ts.stored_nodes, ts.max_nodes_per_entry,
                          ts.memory.total_bytes], np.int64))


if __name__ == "__main__":
    make_hash()
    bvhs, scene = make_bvhs()
    make_trace(bvhs)
    make_waves(bvhs, scene)
    make_predict(bvhs)
    make_record()
