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

    def pending_records(self):
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
