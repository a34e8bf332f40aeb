"""Parity at the larger BASELINE configs, where the BVH leaves L2 (c4, c5)
and the hash is coarse (c3 p = 3) or wide (c3 p = 7).

The GPU wave (hrpp_trace_wave) against the oracle's restatement of the
reference's wave (hrpp/tracer.py:343-371) on the same rays: every hit,
every statistic and both tables.  The oracle runs its key-sharded consult
on all host cores (exact: tests/test_oracle_golden.py pins it to the
reference); its traversal batches use all cores too.
"""
import sys
from argparse import Namespace

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def _workload(config, res=None, spp=None, precision=6, go_up=0):
    import bench
    import paper_1910_01304_b200 as hb
    args = Namespace(config=config, res=res, spp=spp, precision=precision, go_up=go_up)
    return bench.make_workload(args, lambda bv, O, D, t0, t1:
                               hb.intersect_closest_batch(bv, O, D, t0, t1))


def _obvh(oracle_mod, b):
    return oracle_mod.OracleBvh(b.bmin, b.bmax, b.left, b.right, b.axis, b.first, b.count,
                                b.parent, b.depth, b.tv0, b.tv1, b.tv2, b.tri_ids)


def _check_waves(oracle_mod, b, waves, mode, p, g_):
    import paper_1910_01304_b200 as hb
    ob = _obvh(oracle_mod, b)
    cfg = hb.HashConfig(p)
    tabs = {c: hb.PredictorTable(cfg, g_, hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
            for c in (True, False)}
    otabs = {c: oracle_mod.ShardedTable(p, g_, c) for c in (True, False)}
    for name, kind, closest, O, D, t0, t1 in waves:
        out, st = hb.trace_wave(b, tabs[closest], mode, O, D, t0, t1, closest)
        rc, ref, rst = oracle_mod.trace_wave(ob, otabs[closest], mode, closest, O, D, t0, t1)
        assert rc == 0
        assert np.array_equal(st, rst), (name, mode, st, rst)
        for k in ("found", "t", "slot", "leaf"):
            assert np.array_equal(out[k], ref[k]), (name, mode, k)
    for c in (True, False):
        for x, y in zip(tabs[c].export(), otabs[c].export()):
            assert np.array_equal(x, y), (mode, c)


@pytest.fixture(scope="module")
def c5():
    """BASELINE c5 (53.2 M triangles, 69 M nodes, 1024 x 1024 x 8): the
    primary wave, its area-light shadow wave and the first diffuse bounce."""
    sc, b, waves = _workload("c5")
    return b, waves[:3]


@pytest.mark.parametrize("mode", ["limit", "live"])
def test_c5_waves_vs_oracle(c5, oracle_mod, mode):
    b, waves = c5
    assert b.node_count > 60_000_000 and [w[0] for w in waves] == ["primary", "shadow0_0",
                                                                   "bounce1"]
    _check_waves(oracle_mod, b, waves, mode, 6, 0)


@pytest.mark.parametrize("p,res,spp", [(3, "256x256", 8), (7, "1024x1024", 1)])
@pytest.mark.parametrize("mode", ["limit", "live"])
def test_c3_precision_sweep_vs_oracle(oracle_mod, p, res, spp, mode):
    """c3's sweep end points on its primary wave and first shadow waves:
    p = 3 (a few hundred keys, entries of hundreds of nodes, block replay)
    and p = 7 at 2^20 rays (3 x 15 key bits + 20 index bits > 64: the
    generic 64-bit grouping sort)."""
    sc, b, waves = _workload("c3", res=res, spp=spp, precision=p)
    _check_waves(oracle_mod, b, waves[:3], mode, p, 0)


@pytest.mark.parametrize("mode", ["limit", "live"])
def test_c4_go_up_2_vs_oracle(oracle_mod, mode):
    """c4 (1 M triangles, BVH about L2-sized) at go-up level 2: the ancestor
    LUT (hrpp/bvh.py:140-151) on the full 1024 x 1024 x 8 primary wave and
    its shadow wave."""
    sc, b, waves = _workload("c4", precision=6, go_up=2)
    _check_waves(oracle_mod, b, waves[:2], mode, 6, 2)
