"""Pin the C oracle (oracle/hrpp_oracle.c) to the real reference.

Every fixture under tests/golden/ was produced by running the reference
package itself (tests/golden/make_golden.py).  CPU only.
"""
import numpy as np
import pytest

from conftest import load_golden

WAVES = ("primary", "shadow", "reflection")
SETTINGS = ((6, 0), (3, 0), (4, 2), (7, 1))


def obvh(oracle_mod, name):
    return oracle_mod.OracleBvh.from_dict(load_golden(f"bvh_{name}.npz"))


def test_hash_matches_reference(oracle_mod):
    g = load_golden("hash.npz")
    for p in range(1, 8):
        assert np.array_equal(oracle_mod.hash_rays(g["O"], g["D"], p), g["keys"][p - 1])
        assert np.array_equal(oracle_mod.hash_rays_np(g["O"], g["D"], p), g["keys"][p - 1])


def test_hash_nonfinite(oracle_mod):
    O = np.zeros((2, 3), np.float32)
    D = np.array([[0, 0, 1], [0, np.nan, 1]], np.float32)
    assert oracle_mod.hash_rays(O, D, 3) is None
    D[1, 1] = np.inf
    assert oracle_mod.hash_rays(O, D, 3) is None


@pytest.mark.parametrize("threads", [1, 4])
def test_trace_batch_matches_reference(oracle_mod, threads):
    g = load_golden("trace_soup256.npz")
    b = obvh(oracle_mod, "soup256")
    n = g["O"].shape[0]
    c = b.trace_batch(True, g["O"], g["D"], np.zeros(n), np.full(n, np.inf), threads=threads)
    for k, v in c.items():
        assert np.array_equal(v, g[f"c_{k}"]), k
    a = b.trace_batch(False, g["O"], g["D"], np.zeros(n), g["tmax_any"], threads=threads)
    for k, v in a.items():
        assert np.array_equal(v, g[f"a_{k}"]), k
    c7 = b.trace_batch(True, g["O"], g["D"], np.zeros(n), np.full(n, np.inf), start=7)
    for k, v in c7.items():
        assert np.array_equal(v, g[f"c7_{k}"]), k


def test_trace_axis_aligned_rays(oracle_mod):
    g = load_golden("trace_strip8.npz")
    b = obvh(oracle_mod, "strip8")
    n = g["O"].shape[0]
    c = b.trace_batch(True, g["O"], g["D"], np.zeros(n), np.full(n, np.inf))
    for k, v in c.items():
        assert np.array_equal(v, g[f"c_{k}"]), k
    a = b.trace_batch(False, g["O"], g["D"], np.zeros(n), np.full(n, 100.0))
    for k, v in a.items():
        assert np.array_equal(v, g[f"a_{k}"]), k


@pytest.mark.parametrize("p,g_", SETTINGS)
@pytest.mark.parametrize("mode", ["limit", "live"])
def test_wave_sequence_matches_reference(oracle_mod, p, g_, mode):
    inp = load_golden("wave_inputs.npz")
    ref = load_golden(f"wave_{mode}_p{p}_g{g_}.npz")
    b = obvh(oracle_mod, "spheres")
    tables = {True: oracle_mod.OracleTable(p, g_, True), False: oracle_mod.OracleTable(p, g_, False)}
    for w in WAVES:
        closest = w != "shadow"
        rc, out, stats = oracle_mod.trace_wave(
            b, tables[closest], mode, closest, inp[f"{w}_O"], inp[f"{w}_D"], inp[f"{w}_tmin"],
            inp[f"{w}_tmax"], capture=True)
        assert rc == 0
        assert np.array_equal(stats, ref[f"{w}_stats"]), (w, stats, ref[f"{w}_stats"])
        for k in ("found", "t", "slot", "leaf"):
            assert np.array_equal(out[k], ref[f"{w}_{k}"]), (w, k)
        if mode == "limit":
            for k in ("u", "v", "box", "tri", "visited"):
                if f"{w}_{k}" in ref:
                    assert np.array_equal(out[k], ref[f"{w}_{k}"]), (w, k)
            log = out["log"]
            assert np.array_equal(log["cls"], ref[f"{w}_log_cls"])
            assert np.array_equal(log["eval_box"], ref[f"{w}_log_eval_box"])
            assert np.array_equal(log["pred_t"], ref[f"{w}_log_pred_t"])
            assert np.array_equal(log["pred_slot"], ref[f"{w}_log_pred_slot"])
            assert np.array_equal(out["keys"], ref[f"{w}_log_keys"])
        assert tables[closest].dump_lines() == list(ref[f"{w}_dump"])
        e, s, m = tables[closest].info()
        assert [e, s, m, 16 * e + 4 * s] == list(ref[f"{w}_tstats"])


def test_predict_matches_reference(oracle_mod):
    g = load_golden("predict.npz")
    b = obvh(oracle_mod, "soup256")
    O, D = g["O"], g["D"]
    n = O.shape[0]
    for pre, closest, go_up in (("c", True, 1), ("a", False, 0)):
        t = oracle_mod.OracleTable(4, go_up, closest)
        keys = oracle_mod.hash_rays(O, D, 4)
        base = b.trace_batch(True, O, D, np.zeros(n), np.full(n, np.inf))
        lut = b.ancestor_lut(go_up)
        half = np.arange(n // 2)
        sel = half[base["found"][half]]
        t.record_batch(keys[sel], lut[base["leaf"][sel]])
        assert t.dump_lines() == list(g[f"{pre}_dump"])
        tmax = np.full(n, np.inf) if closest else np.full(n, 6.0)
        out = oracle_mod.predict_batch(b, t, closest, keys, O, D, np.zeros(n), tmax)
        assert np.array_equal(out["cls"], g[f"{pre}_cls"])
        tp = out["cls"] == 0
        assert np.array_equal(out["t"][tp], g[f"{pre}_t"][tp])
        assert np.array_equal(b.tri_ids[out["slot"][tp]], g[f"{pre}_tri_id"][tp])
        assert np.array_equal(out["leaf"][tp], g[f"{pre}_leaf"][tp])
        assert np.array_equal(out["box"], g[f"{pre}_box"])
        assert np.array_equal(out["est"], g[f"{pre}_est"])


def test_record_sequence_matches_reference(oracle_mod):
    g = load_golden("record.npz")
    t = oracle_mod.OracleTable(6, 0, True)
    rc, ins = t.record_batch(g["keys"], g["nodes"])
    assert rc == 0
    assert np.array_equal(ins, g["inserted"])
    assert t.dump_lines() == list(g["dump"])


def test_capacity(oracle_mod):
    t = oracle_mod.OracleTable(6, 0, True, max_entries=2)
    rc, _ = t.record_batch(np.array([1, 2, 1], np.uint64), np.array([0, 0, 5], np.int32))
    assert rc == 0
    rc, _ = t.record_batch(np.array([3], np.uint64), np.array([0], np.int32))
    assert rc == oracle_mod.CAPACITY


def _tris_from_bvh(g):
    order = np.argsort(g["tri_ids"], kind="stable")
    return g["tv0"][order], g["tv1"][order], g["tv2"][order], g["tri_ids"][order]


@pytest.mark.parametrize("name,leaf", [("strip8", 1), ("soup256", 4), ("spheres", 4),
                                       ("ico1282", 4)])
def test_oracle_builder_matches_reference(oracle_mod, name, leaf):
    """The oracle's C restatement of the SAH builder (hrpp/bvh.py:184-357)
    reproduces the reference-built golden BVHs array for array."""
    g = load_golden(f"bvh_{name}.npz")
    if "in_v0" in g:
        v0, v1, v2, ids = g["in_v0"], g["in_v1"], g["in_v2"], None
    else:
        v0, v1, v2, ids = _tris_from_bvh(g)
    b = oracle_mod.build_bvh(v0, v1, v2, ids=ids, max_leaf_size=leaf)
    for k in ("bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth",
              "tv0", "tv1", "tv2", "tri_ids"):
        assert np.array_equal(getattr(b, k), g[k]), k
    assert b.max_depth == int(g["max_depth"])


def test_oracle_builder_edge_cases(oracle_mod):
    with pytest.raises(ValueError):  # every triangle degenerate (bvh.py:195-201)
        oracle_mod.build_bvh(np.zeros((2, 3)), np.ones((2, 3)), 2 * np.ones((2, 3)))
    t = np.array([[0, 0, 0]], np.float32), np.array([[1, 0, 0]], np.float32), \
        np.array([[0, 1, 0]], np.float32)
    b = oracle_mod.build_bvh(*(np.repeat(a, 3, axis=0) for a in t), max_leaf_size=1)
    assert b.node_count == 1 and int(b.count[0]) == 3  # coincident centroids: one leaf


@pytest.mark.parametrize("median", [False, True])
def test_oracle_builder_matches_native_builder(oracle_mod, median):
    """Same arrays as the product's native builder on a BASELINE c1 scene
    (the median-split option has no reference counterpart: both builders
    implement the reference's forced split at every oversized node)."""
    import paper_1910_01304_b200 as hb
    from paper_1910_01304_b200.scenes import make_scene
    sc = make_scene("c1")
    a = oracle_mod.build_bvh(sc.v0, sc.v1, sc.v2, median_split=median)
    b = hb.build_bvh_from_arrays(sc.v0, sc.v1, sc.v2, median_split=median)
    for k in ("bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth",
              "tv0", "tv1", "tv2", "tri_ids"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.max_depth == b.max_depth


@pytest.mark.parametrize("p,g_", ((6, 0), (3, 0), (4, 2)))
@pytest.mark.parametrize("mode", ["limit", "live"])
@pytest.mark.parametrize("shards", [2, 5])
def test_sharded_oracle_equals_reference(oracle_mod, p, g_, mode, shards):
    """The key-sharded multi-threaded consult (the CPU baseline's) gives the
    reference's hits, statistics and table (union of the shards)."""
    inp = load_golden("wave_inputs.npz")
    ref = load_golden(f"wave_{mode}_p{p}_g{g_}.npz")
    b = obvh(oracle_mod, "spheres")
    tables = {c: oracle_mod.ShardedTable(p, g_, c, shards=shards) for c in (True, False)}
    for w in WAVES:
        closest = w != "shadow"
        rc, out, stats = oracle_mod.trace_wave(b, tables[closest], mode, closest, inp[f"{w}_O"],
                                               inp[f"{w}_D"], inp[f"{w}_tmin"],
                                               inp[f"{w}_tmax"])
        assert rc == 0
        assert np.array_equal(stats, ref[f"{w}_stats"]), (w, stats, ref[f"{w}_stats"])
        for k in ("found", "t", "slot", "leaf"):
            assert np.array_equal(out[k], ref[f"{w}_{k}"]), (w, k)
        assert tables[closest].dump_lines() == list(ref[f"{w}_dump"])


@pytest.mark.parametrize("p,g_", SETTINGS)
def test_fast_mode_many_rounds_matches_reference_live(oracle_mod, p, g_):
    """Fast mode's speculation rounds replay the live loop: with enough
    rounds every ray sees exactly the appends of the rays before it, so the
    classification, traversal counters, occlusion hits and table equal the
    reference's live mode (hrpp/tracer.py:295-331); closest-hit TPs may
    skip nodes appended between their own round and their turn, which only
    moves the overhead/est counters (and t on a closer later node)."""
    inp = load_golden("wave_inputs.npz")
    ref = load_golden(f"wave_live_p{p}_g{g_}.npz")
    b = obvh(oracle_mod, "spheres")
    oracle_mod.set_fast_rounds(100000, 0)
    try:
        tables = {c: oracle_mod.OracleTable(p, g_, c) for c in (True, False)}
        for w in WAVES:
            closest = w != "shadow"
            rc, out, st = oracle_mod.trace_wave(b, tables[closest], "fast", closest,
                                                inp[f"{w}_O"], inp[f"{w}_D"], inp[f"{w}_tmin"],
                                                inp[f"{w}_tmax"])
            assert rc == 0
            want = ref[f"{w}_stats"]
            same = [0, 1, 2, 3, 4, 5] if closest else list(range(11))
            assert np.array_equal(st[same], want[same]), (w, st, want)
            assert np.array_equal(out["found"], ref[f"{w}_found"])
            if not closest:
                for k in ("t", "slot", "leaf"):
                    assert np.array_equal(out[k], ref[f"{w}_{k}"]), (w, k)
            assert tables[closest].dump_lines() == list(ref[f"{w}_dump"]), w
    finally:
        oracle_mod.set_fast_rounds()
