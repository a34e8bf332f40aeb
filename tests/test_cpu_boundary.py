"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, host logic (native builder, API surface, metrics, generators)."""
import re
from pathlib import Path

import numpy as np
import pytest

from bvh_checks import check_bvh
from conftest import ROOT, load_golden

import paper_1910_01304_b200 as hb
from paper_1910_01304_b200 import _lib


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "hrpp_b200.h").read_text()
    declared = set(re.findall(r"\b(hrpp_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(_lib.lib, name), f"{name} declared in hrpp_b200.h but not exported"
    assert set(_lib.EXPORTED) <= declared
    assert _lib.lib.hrpp_version() == 1


def test_library_is_sm100a():
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                       text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


def _tris_from_bvh(g):
    order = np.argsort(g["tri_ids"], kind="stable")
    return g["tv0"][order], g["tv1"][order], g["tv2"][order], g["tri_ids"][order]


@pytest.mark.parametrize("name,leaf", [("strip8", 1), ("soup256", 4), ("spheres", 4),
                                       ("ico1282", 4)])
def test_native_builder_matches_reference(name, leaf):
    g = load_golden(f"bvh_{name}.npz")
    if "in_v0" in g:
        v0, v1, v2, ids = g["in_v0"], g["in_v1"], g["in_v2"], None
    else:
        v0, v1, v2, ids = _tris_from_bvh(g)
    b = hb.build_bvh_from_arrays(v0, v1, v2, ids=ids, max_leaf_size=leaf)
    for k in ("bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth",
              "tv0", "tv1", "tv2", "tri_ids"):
        assert np.array_equal(getattr(b, k), g[k]), k
    assert b.max_depth == int(g["max_depth"])
    check_bvh(b)


def test_builder_edge_cases():
    with pytest.raises(hb.EmptyScene):
        hb.build_bvh([])
    degenerate = [hb.Triangle(hb.vec3(0, 0, 0), hb.vec3(1, 0, 0), hb.vec3(2, 0, 0))]
    with pytest.raises(hb.EmptyScene):
        hb.build_bvh(degenerate)
    tris = [hb.Triangle(hb.vec3(0, 0, 0), hb.vec3(1, 0, 0), hb.vec3(0, 1, 0), id=i)
            for i in range(2)]
    b = hb.build_bvh(tris, max_leaf_size=1)
    assert b.node_count == 1 and int(b.count[0]) == 2  # coincident -> oversized leaf
    one = hb.build_bvh([hb.Triangle(hb.vec3(0, 0, 0), hb.vec3(1, 0, 0), hb.vec3(0, 1, 0))])
    assert one.node_count == 1 and one.max_depth == 0


def test_median_split_builder():
    from paper_1910_01304_b200.scenes import make_scene
    sc = make_scene("c1")
    b = hb.build_bvh_from_arrays(sc.v0, sc.v1, sc.v2, median_split=True)
    check_bvh(b)
    assert int(b.count[b.left < 0].max()) <= 4


def test_hash_config_and_key_utils():
    with pytest.raises(ValueError):
        hb.HashConfig(0)
    with pytest.raises(ValueError):
        hb.HashConfig(8)
    assert hb.HashConfig(6).bits_per_float == 13
    assert hb.key_hex(0) == "000000000000"
    assert hb.key_hex((1 << 48) - 1) == "ffffffffffff"
    with pytest.raises(ValueError):
        hb.coarsen_key(5, 1)  # argument check precedes the device


def test_table_capacity_env(monkeypatch):
    monkeypatch.setenv("HRPP_MAX_TABLE_ENTRIES", "3")
    t = hb.PredictorTable(hb.HashConfig(6))
    assert t.max_entries == 3
    monkeypatch.setenv("HRPP_MAX_TABLE_ENTRIES", "bogus")
    with pytest.raises(ValueError):
        hb.PredictorTable(hb.HashConfig(6))
    monkeypatch.setenv("HRPP_MAX_TABLE_ENTRIES", "0")
    with pytest.raises(ValueError):
        hb.PredictorTable(hb.HashConfig(6))
    with pytest.raises(ValueError):
        hb.PredictorTable(hb.HashConfig(6), go_up_level=-1)


def test_empty_table_host_views():
    t = hb.PredictorTable(hb.HashConfig(6))
    assert t.entry_count == 0 and t.stored_node_count == 0
    assert t.lookup(123) is None
    assert t.memory_estimate().total_bytes == 0
    assert list(t.dump_lines()) == []


def test_metrics_formulas():
    s = hb.RayKindStats(rays=10, tp=4, fp=1, neg=5, baseline_box_tests=100,
                        skipped_box_tests=40, overhead_box_tests=5, overhead_tri_tests=3,
                        wrong_closest=1)
    assert hb.savings_percent(s) == pytest.approx(40.0)
    assert hb.net_savings_percent(s) == pytest.approx(32.0)
    assert hb.fully_skipped_percent(s) == pytest.approx(40.0)
    assert hb.wrong_closest_rate(s) == pytest.approx(0.25)
    with pytest.raises(hb.NoBaseline):
        hb.savings_percent(hb.RayKindStats())
    a = hb.RayKindStats(*range(11))
    assert (a + hb.RayKindStats()) == a
    assert np.array_equal(a.as_array(), np.arange(11))


def test_primary_ray_generator_matches_reference():
    # wave_inputs.npz primaries came from the reference's generate_primary_rays
    # (hrpp/tracer.py:173-211) on the bundled spheres camera at 48x48, spp 4.
    from paper_1910_01304_b200.scenes import Camera, primary_rays
    cam = Camera((7.0, 5.5, 9.5), (0.0, 0.6, 0.0), (0.0, 1.0, 0.0), 42.0, (48, 48))
    O, D = primary_rays(cam, 4, seed=0)
    g = load_golden("wave_inputs.npz")
    assert np.array_equal(O, g["primary_O"])
    assert np.array_equal(D, g["primary_D"])


def test_scene_sizes():
    from paper_1910_01304_b200.scenes import icosphere, make_scene
    for s, f in ((0, 20), (1, 80), (3, 1280)):
        assert icosphere(s)[1].shape[0] == f
    c1 = make_scene("c1")
    assert c1.n_tris == 1282


def test_report_rows_match_reference_format(tmp_path):
    s = hb.RayKindStats(rays=10, tp=3, fp=2, neg=5, baseline_box_tests=50, baseline_tri_tests=9,
                        overhead_box_tests=4, overhead_tri_tests=3, skipped_box_tests=20)
    ts = hb.TableStats(entries=1, stored_nodes=1, avg_nodes_per_entry=1.0,
                       max_nodes_per_entry=1,
                       memory=hb.MemoryEstimate(entry_bytes=16, node_ref_bytes=4))
    row = hb.report_row("demo", "limit", "primary", 6, 0, 8, "64x64", 0, s, ts)
    assert set(hb.REPORT_COLUMNS) == set(row)
    assert row["savings_percent"] == pytest.approx(40.0) and row["consulted"] == 10
    text = hb.render_csv([row], timestamp=False)
    assert text.splitlines()[0] == ",".join(hb.REPORT_COLUMNS)
    assert "40.000000" in text.splitlines()[1]
    assert hb.render_csv([row]).startswith("# generated ")
    hb.write_json([row], tmp_path / "r.json")
    import json
    assert json.loads((tmp_path / "r.json").read_text())[0]["tp"] == 3
    f = hb.failed_row("demo", "limit", "primary", 6, 0, 8, "64x64", 0, "boom")
    assert f["status"] == "failed: boom" and f["rays"] == 0
