"""Multi-rank host logic on CPU (gloo, world_size 2): contiguous ray blocks,
variable-length all-gather of deferred predictor records and their merge in
global ray order, so every rank ends a wave with the identical table."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1910_01304_b200.parallel import block_range, merge_records


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeTable:
    """pending_records/record_batch stand-in backed by the C oracle table."""

    def __init__(self, oracle_mod, keys, nodes, rays):
        self.t = oracle_mod.OracleTable(6, 0, True)
        self._p = (keys, nodes, rays)

    def pending_records(self, device=False):
        return self._p

    def record_batch(self, k, n):
        rc, ins = self.t.record_batch(k, n)
        assert rc == 0
        return ins


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import oracle
    from paper_1910_01304_b200.parallel import merge_wave_records
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        n = 1000
        keys_all = rng.integers(0, 50, n).astype(np.uint64) * np.uint64(0x10001)
        nodes_all = rng.integers(0, 30, n).astype(np.int32)
        lo, hi = block_range(n, rank, world)
        sel = np.arange(lo, hi)
        sel = sel[rng.random(sel.shape[0]) < 0.3 + 0.4 * rank]  # ragged per rank
        local_rays = (sel - lo).astype(np.int32)
        tab = FakeTable(oracle, keys_all[sel], nodes_all[sel], local_rays)
        m = merge_wave_records(tab, dist, ray_offset=lo)
        q.put((rank, m, tab.t.dump_lines()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_record_merge_two_ranks(world, oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical tables on every rank, equal to a sequential replay
    assert res[0][2] == res[1][2]
    assert res[0][1] == res[1][1]


def test_merge_records_orders_by_global_ray():
    k = [np.array([5, 6], np.uint64), np.array([7], np.uint64)]
    n = [np.array([1, 2], np.int32), np.array([3], np.int32)]
    r = [np.array([3, 1], np.int32), np.array([0], np.int32)]
    mk, mn = merge_records(k, n, r, [0, 2])
    assert mk.tolist() == [6, 7, 5] and mn.tolist() == [2, 3, 1]


def test_block_range_contiguous_cover():
    for n in (0, 1, 7, 1000):
        for w in (1, 2, 3, 8):
            spans = [block_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _sharded_worker(rank, world, port, q):
    """Key-sharded waves (primary, shadow, reflection) with the C oracle as
    each owner's engine; hits, summed stats and table union vs one process."""
    import torch
    import torch.distributed as dist
    from conftest import load_golden
    from oracle import oracle
    from paper_1910_01304_b200.parallel import block_range, key_sharded_wave
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bvh = oracle.OracleBvh.from_dict(load_golden("bvh_spheres.npz"))
        g = load_golden("wave_inputs.npz")
        res = []
        for mode in ("limit", "live"):
            tabs = {c: oracle.OracleTable(6, 0, c) for c in (True, False)}
            for name, closest in (("primary", True), ("shadow", False), ("reflection", True)):
                arrs = [g[f"{name}_{k}"] for k in ("O", "D", "tmin", "tmax")]
                lo, hi = block_range(arrs[0].shape[0], rank, world)
                mine = [torch.from_numpy(np.ascontiguousarray(a[lo:hi])) for a in arrs]

                def trace_fn(O, D, t0, t1, closest=closest):
                    rc, out, st = oracle.trace_wave(bvh, tabs[closest], mode, closest, O.numpy(),
                                                    D.numpy(), t0.numpy(), t1.numpy())
                    assert rc == 0
                    return {k: torch.from_numpy(np.ascontiguousarray(out[k]))
                            for k in ("found", "t", "slot", "leaf")}, st

                out, st = key_sharded_wave(
                    dist, trace_fn, lambda O, D: oracle.hash_rays_np(O.numpy(), D.numpy(), 6),
                    oracle.partition_by_owner_np, *mine)
                res.append((mode, name, lo, {k: v.numpy() for k, v in out.items()},
                            np.asarray(st)))
            res.append((mode, "tables", {c: t.dump_lines() for c, t in tabs.items()}))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_key_sharded_waves_equal_single_process(oracle_mod):
    from conftest import load_golden
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    bvh = oracle_mod.OracleBvh.from_dict(load_golden("bvh_spheres.npz"))
    g = load_golden("wave_inputs.npz")
    i = 0
    for mode in ("limit", "live"):
        tabs = {c: oracle_mod.OracleTable(6, 0, c) for c in (True, False)}
        for name, closest in (("primary", True), ("shadow", False), ("reflection", True)):
            rc, ref, rst = oracle_mod.trace_wave(bvh, tabs[closest], mode, closest,
                                                 *(g[f"{name}_{k}"] for k in
                                                   ("O", "D", "tmin", "tmax")))
            assert rc == 0
            parts = [got[r][i] for r in range(world)]
            assert all(p[0] == mode and p[1] == name for p in parts)
            for k in ("found", "t", "slot", "leaf"):
                assert np.array_equal(np.concatenate([p[3][k] for p in parts]), ref[k]), \
                    (mode, name, k)
            assert np.array_equal(sum(p[4] for p in parts), rst), (mode, name)
            i += 1
        tables = [got[r][i][2] for r in range(world)]
        for c in (True, False):
            union = sorted(tables[0][c] + tables[1][c])
            assert union == tabs[c].dump_lines(), (mode, c)
            assert not set(tables[0][c]) & set(tables[1][c])  # disjoint partitions
        i += 1


def test_partition_by_owner_np_stable():
    from oracle import oracle
    keys = np.arange(1000, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15 % (1 << 48))
    perm, counts = oracle.partition_by_owner_np(keys, 3)
    assert counts.sum() == 1000 and counts.min() > 250
    assert sorted(perm.tolist()) == list(range(1000))
    start = 0
    for c in counts:  # ray order kept within each owner
        seg = perm[start:start + c]
        assert np.all(np.diff(seg) > 0)
        start += c
