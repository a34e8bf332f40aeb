"""The drop-in boundary driven by the reference's own types and renderer.

* ``_trace_wave`` (hrpp/tracer.py:343-371) must accept the reference's
  ``RenderMode`` members and add into its ``RayKindStats``
  (hrpp/metrics.py:38-68); stand-ins shaped exactly like them are used when
  the reference is not importable.
* With the reference installed (``baseline/_ref``, git-ignored; it travels to
  the GPU box with the snapshot), ``hrpp.tracer.render`` is run twice on the
  same scene: once stock, once with ``_trace_wave`` monkeypatched to this
  package's and this package's BVH / tables -- the INTEGRATION.md two-line
  patch.  Image, per-kind statistics and table statistics must be identical.
"""

import dataclasses
import enum
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


class StandInMode(enum.Enum):  # shaped like hrpp.tracer.RenderMode (tracer.py:58-61)
    BASELINE = "baseline"
    LIMIT = "limit"
    LIVE = "live"


@dataclasses.dataclass
class StandInStats:  # shaped like hrpp.metrics.RayKindStats (metrics.py:38-51), no add_array
    rays: int = 0
    tp: int = 0
    fp: int = 0
    neg: int = 0
    baseline_box_tests: int = 0
    baseline_tri_tests: int = 0
    overhead_box_tests: int = 0
    overhead_tri_tests: int = 0
    skipped_box_tests: int = 0
    skipped_box_tests_estimated: int = 0
    wrong_closest: int = 0


def test_mode_and_stats_conversion():
    """Host-side conversion (no GPU): enum members of another class and
    strings map by value; counters are added by field name."""
    from paper_1910_01304_b200 import tracer
    assert tracer.as_mode(StandInMode.LIVE) is tracer.RenderMode.LIVE
    assert tracer.as_mode("limit") is tracer.RenderMode.LIMIT
    assert tracer.as_mode(tracer.RenderMode.BASELINE) is tracer.RenderMode.BASELINE
    with pytest.raises(ValueError):
        tracer.as_mode("fastest")
    s = StandInStats(rays=3)
    tracer.add_stats(s, np.arange(11, dtype=np.int64))
    assert dataclasses.astuple(s) == (3, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10)


def test_table_accepts_foreign_kind_enum():
    from paper_1910_01304_b200 import HashConfig, PredictorTable

    class Kind(enum.Enum):  # shaped like hrpp.geom.RayKind
        HIT_ANY = "hit_any"
        CLOSEST_HIT = "closest_hit"

    t = PredictorTable(HashConfig(6), 0, Kind.HIT_ANY)
    assert t.kind is Kind.HIT_ANY and not t.closest
    assert PredictorTable(HashConfig(6), 0, Kind.CLOSEST_HIT).closest
    with pytest.raises(ValueError):
        PredictorTable(HashConfig(6), 0, "sideways")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", list(StandInMode))
def test_trace_wave_with_reference_shaped_types(mode):
    """_trace_wave with stand-ins of the reference's RenderMode/RayKindStats
    equals trace_wave with this package's own types (c1 primary wave)."""
    import paper_1910_01304_b200 as hb
    from paper_1910_01304_b200 import scenes
    sc = scenes.make_scene("c1", resolution=(64, 64))
    b = hb.build_bvh_from_arrays(sc.v0, sc.v1, sc.v2, median_split=True)
    O, D = scenes.primary_rays(sc.camera, 2, seed=1)
    n = O.shape[0]
    t0, t1 = np.zeros(n), np.full(n, np.inf)
    results = []
    for m, stats in ((mode, StandInStats()), (hb.RenderMode(mode.value), hb.RayKindStats())):
        table = hb.PredictorTable(hb.HashConfig(6), 0, hb.RayKind.CLOSEST_HIT)
        logs = ({k: [] for k in ("cls", "eval_box", "base_box", "pred_t", "pred_slot", "keys")}
                if mode is StandInMode.LIMIT else None)
        for _ in range(2):  # a second wave consults the trained table
            eff = hb._trace_wave(b, table, None, m, O, D, t0, t1, stats, True, logs)
        results.append((eff, dataclasses.astuple(stats), list(table.dump_lines()), logs))
    (e1, s1, d1, l1), (e2, s2, d2, l2) = results
    assert s1 == s2 and s1[0] == 2 * n
    assert d1 == d2
    for k in e2:
        assert np.array_equal(e1[k], e2[k]), k
    assert l1 == l2


def _import_reference():
    if not (REF / "hrpp").is_dir():
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hrpp")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    try:
        import hrpp  # noqa: F401
        import hrpp.tracer  # noqa: F401
    except Exception as e:  # numba missing on the box, ...
        pytest.skip(f"reference not importable: {e}")
    return sys.modules["hrpp"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["limit", "live"])
def test_reference_render_with_dropin(mode, monkeypatch):
    """hrpp.tracer.render (hrpp/tracer.py:377-524) through this package's
    _trace_wave, BVH and tables == the stock reference render: image bytes,
    per-kind RayKindStats, table stats.  Bundled 'spheres' scene (mirror
    floor: primary, shadow and reflection waves), 64x64, 4 spp."""
    hrpp = _import_reference()
    import hrpp.scene_io as rio
    import hrpp.tracer as rtr
    import paper_1910_01304_b200 as hb

    scene = rio.load_bundled_scene("spheres")
    scene = dataclasses.replace(scene, camera=dataclasses.replace(scene.camera,
                                                                  resolution=(64, 64)))
    rbvh = hrpp.bvh.build_bvh_from_arrays(scene.v0, scene.v1, scene.v2)
    cfg = rtr.RenderConfig(spp=4, max_reflection_depth=2, mode=rtr.RenderMode(mode))

    def ref_tables(mk):
        return {"closest": mk(hrpp.HashConfig(6), 0, hrpp.RayKind.CLOSEST_HIT),
                "hit_any": mk(hrpp.HashConfig(6), 0, hrpp.RayKind.HIT_ANY)}

    want = rtr.render(scene, rbvh, ref_tables(hrpp.PredictorTable), cfg)

    ours_bvh = hb.Bvh(rbvh.bmin, rbvh.bmax, rbvh.left, rbvh.right, rbvh.axis, rbvh.first,
                      rbvh.count, rbvh.parent, rbvh.depth, rbvh.tv0, rbvh.tv1, rbvh.tv2,
                      rbvh.tri_ids, rbvh.max_depth)
    monkeypatch.setattr(rtr, "_trace_wave", hb._trace_wave)  # the INTEGRATION.md patch
    got = rtr.render(scene, ours_bvh, ref_tables(hb.PredictorTable), cfg)

    assert np.array_equal(got.image, want.image)
    for k in want.stats:
        assert dataclasses.astuple(got.stats[k]) == dataclasses.astuple(want.stats[k]), k
    for k in ("closest", "hit_any"):
        g, w = got.table_stats[k], want.table_stats[k]
        assert (g.entries, g.stored_nodes, g.max_nodes_per_entry) == \
            (w.entries, w.stored_nodes, w.max_nodes_per_entry), k
        assert g.memory.total_bytes == w.memory.total_bytes
    assert want.stats["primary"].rays > 0 and want.stats["reflection"].rays > 0
