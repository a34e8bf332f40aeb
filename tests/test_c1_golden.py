"""BASELINE config c1 pinned to the reference itself.

tests/golden/make_golden_c1.py ran the reference's ``_trace_wave``
(hrpp/tracer.py:343-371) over the c1 frame (primary, point-light shadow,
diffuse bounce; median-split BVH injected through ``Bvh(...)``) in limit and
live mode, and its ``report_row`` / ``render_csv`` / ``write_json``
(hrpp/metrics.py:140-218) over the frame's statistics.  Here: the oracle
(CPU), the report writers (CPU) and the GPU wave (GPU) against those bytes.
"""
import hashlib
import sys
import tempfile
from argparse import Namespace
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, load_golden

sys.path.insert(0, str(ROOT))

SETTINGS = ((6, 0), (5, 1))
MODES = ("limit", "live")


def _digest(waves):
    h = hashlib.sha256()
    for w in waves:
        for a in w[3:]:
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def c1(oracle_mod):
    """The c1 frame's waves (regenerated bit for bit: digest-checked) and the
    oracle's BVH."""
    import bench
    args = Namespace(config="c1", res=None, spp=None, precision=6, go_up=0)
    sc, ob, waves = bench.make_workload(
        args, lambda b, O, D, t0, t1: b.trace_batch(True, O, D, t0, t1, threads=0),
        build=oracle_mod.build_bvh)
    assert _digest(waves) == str(load_golden("c1_frame_live_p6_g0.npz")["digest"])
    return ob, waves


def _tstats(dump):
    import paper_1910_01304_b200 as hb
    sizes = [len(ln.split("[")[1].rstrip("]").split(",")) if not ln.endswith("[]") else 0
             for ln in dump]
    e, s = len(sizes), sum(sizes)
    return hb.TableStats(entries=e, stored_nodes=s, avg_nodes_per_entry=s / e if e else 0.0,
                         max_nodes_per_entry=max(sizes) if sizes else 0,
                         memory=hb.MemoryEstimate(entry_bytes=16 * e, node_ref_bytes=4 * s))


def _reports(g, kind_stats, tstats, mode, p, g_):
    """Our report rows / CSV / JSON bytes for the frame."""
    import paper_1910_01304_b200 as hb
    rows = [hb.report_row("c1", mode, k, p, g_, 1, "256x256", 0, kind_stats[k],
                          tstats[k != "shadow"]) for k in [str(x) for x in g["kinds"]]]
    rows.append(hb.failed_row("c1", mode, "primary", p, g_, 1, "256x256", 0, "example failure"))
    csv = hb.render_csv(rows, timestamp=False)
    with tempfile.TemporaryDirectory() as d:
        hb.write_json(rows, Path(d) / "r.json")
        js = (Path(d) / "r.json").read_text()
    return csv, js


def _kind_stats(waves, stats_of):
    import paper_1910_01304_b200 as hb
    ks = {}
    for name, kind, *_ in waves:
        ks.setdefault(kind, hb.RayKindStats()).add_array(stats_of(name))
    return ks


@pytest.mark.parametrize("p,g_", SETTINGS)
@pytest.mark.parametrize("mode", MODES)
def test_oracle_c1_frame_matches_reference(c1, oracle_mod, p, g_, mode):
    ob, waves = c1
    g = load_golden(f"c1_frame_{mode}_p{p}_g{g_}.npz")
    tabs = {c: oracle_mod.OracleTable(p, g_, c) for c in (True, False)}
    for name, kind, closest, O, D, t0, t1 in waves:
        rc, out, st = oracle_mod.trace_wave(ob, tabs[closest], mode, closest, O, D, t0, t1,
                                            capture=True)
        assert rc == 0
        assert np.array_equal(st, g[f"{name}_stats"]), (name, st, g[f"{name}_stats"])
        for k in ("found", "t", "slot", "leaf"):
            assert np.array_equal(out[k], g[f"{name}_{k}"]), (name, k)
        if mode == "limit":
            for k in ("cls", "eval_box", "pred_t", "pred_slot"):
                assert np.array_equal(out["log"][k], g[f"{name}_log_{k}"]), (name, k)
        assert tabs[closest].dump_lines() == list(g[f"{name}_dump"]), name


@pytest.mark.parametrize("p,g_", SETTINGS)
@pytest.mark.parametrize("mode", MODES)
def test_reports_match_reference_bytes(c1, p, g_, mode):
    """report_row / render_csv / write_json over the reference's own frame
    statistics reproduce its CSV and JSON bytes (hrpp/metrics.py:121-218)."""
    ob, waves = c1
    g = load_golden(f"c1_frame_{mode}_p{p}_g{g_}.npz")
    ks = _kind_stats(waves, lambda name: g[f"{name}_stats"])
    last = {c: [w[0] for w in waves if w[2] == c][-1] for c in (True, False)}
    ts = {c: _tstats(list(g[f"{last[c]}_dump"])) for c in (True, False)}
    csv, js = _reports(g, ks, ts, mode, p, g_)
    assert csv == str(g["csv"])
    assert js == str(g["json"])


@pytest.mark.gpu
@pytest.mark.parametrize("p,g_", SETTINGS)
@pytest.mark.parametrize("mode", MODES)
def test_gpu_c1_frame_matches_reference(c1, p, g_, mode):
    """The GPU wave on the c1 frame equals the reference's: hits, statistics,
    OutcomeLog, tables after every wave, and the frame's report bytes."""
    import paper_1910_01304_b200 as hb
    ob, waves = c1
    g = load_golden(f"c1_frame_{mode}_p{p}_g{g_}.npz")
    b = hb.Bvh(ob.bmin, ob.bmax, ob.left, ob.right, ob.axis, ob.first, ob.count, ob.parent,
               ob.depth, ob.tv0, ob.tv1, ob.tv2, ob.tri_ids, ob.max_depth)
    tabs = {c: hb.PredictorTable(hb.HashConfig(p), g_,
                                 hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
            for c in (True, False)}
    stats = {}
    for name, kind, closest, O, D, t0, t1 in waves:
        out, st = hb.trace_wave(b, tabs[closest], mode, O, D, t0, t1, closest,
                                capture_outcomes=True)
        stats[name] = st
        assert np.array_equal(st, g[f"{name}_stats"]), (name, st, g[f"{name}_stats"])
        for k in ("found", "t", "slot", "leaf"):
            assert np.array_equal(out[k], g[f"{name}_{k}"]), (name, k)
        if mode == "limit":
            for k in ("cls", "eval_box", "pred_t", "pred_slot"):
                assert np.array_equal(out[f"log_{k}"], g[f"{name}_log_{k}"]), (name, k)
        assert list(tabs[closest].dump_lines()) == list(g[f"{name}_dump"]), name
    ks = _kind_stats(waves, lambda name: stats[name])
    ts = {c: hb.table_stats(tabs[c]) for c in (True, False)}
    csv, js = _reports(g, ks, ts, mode, p, g_)
    assert csv == str(g["csv"])
    assert js == str(g["json"])
