"""The multi-GPU data plane's device-tensor branches at world size 2 on one
GPU: both ranks use cuda:0 and their collectives cross a gloo group through
host copies (``HostStagedDist``), so no kernel of one rank ever waits for the
other (on a multi-GPU box NCCL takes this role; only one GPU is available
here).  Covers the CUDA pack/all-to-all/unpack path of exact key sharding
(parallel.key_sharded_wave) and the device-resident record all-gather of
ray blocks (parallel.merge_wave_records)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KEYS = ("bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth", "tv0",
        "tv1", "tv2", "tri_ids")
WAVES = (("primary", True), ("shadow", False), ("reflection", True))


class HostStagedDist:
    """torch.distributed facade whose collectives on CUDA tensors run on the
    gloo group through host copies; it reports the "nccl" backend so the
    data plane takes its device-tensor branches."""

    def __init__(self, dist):
        self._d = dist

    def get_world_size(self, group=None):
        return self._d.get_world_size(group)

    def get_rank(self, group=None):
        return self._d.get_rank(group)

    def get_backend(self, group=None):
        return "nccl"

    def barrier(self, group=None):
        self._d.barrier(group=group)

    def all_gather(self, outs, t, group=None):
        host = [torch.empty(o.shape, dtype=o.dtype) for o in outs]
        self._d.all_gather(host, t.cpu(), group=group)
        for o, h in zip(outs, host):
            o.copy_(h)

    def all_to_all_single(self, out, inp, out_split_sizes=None, in_split_sizes=None,
                          group=None):
        h = torch.empty(out.shape, dtype=out.dtype)
        self._d.all_to_all_single(h, inp.cpu(), out_split_sizes, in_split_sizes, group=group)
        out.copy_(h)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def _setup(rank, world, port):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    return dist


def _key_sharded_worker(rank, world, port, q):
    from conftest import load_golden
    import paper_1910_01304_b200 as hb
    from paper_1910_01304_b200.parallel import block_range, key_sharded_wave, partition_by_owner
    dist = _setup(rank, world, port)
    try:
        staged = HostStagedDist(dist)
        g = load_golden("bvh_spheres.npz")
        b = hb.Bvh(*(g[k] for k in KEYS), int(g["max_depth"]))
        inp = load_golden("wave_inputs.npz")
        dev = torch.device("cuda", 0)
        res = []
        for mode in ("limit", "live"):
            tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0,
                                         hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
                    for c in (True, False)}
            for name, closest in WAVES:
                arrs = [inp[f"{name}_{k}"] for k in ("O", "D", "tmin", "tmax")]
                lo, hi = block_range(arrs[0].shape[0], rank, world)
                mine = [torch.from_numpy(np.ascontiguousarray(a[lo:hi])).to(dev) for a in arrs]

                def trace_fn(O, D, t0, t1, closest=closest):
                    return hb.trace_wave(b, tabs[closest], mode, O, D, t0, t1, closest)

                out, st = key_sharded_wave(
                    staged, trace_fn, lambda O, D: hb.hash_rays(O, D, hb.HashConfig(6)),
                    lambda k, w: partition_by_owner(k, w, device_counts=True), *mine)
                assert all(v.is_cuda for v in out.values())
                res.append((mode, name, {k: v.cpu().numpy() for k, v in out.items()},
                            np.asarray(st)))
            res.append((mode, "tables", {c: list(t.dump_lines()) for c, t in tabs.items()}))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_key_sharding_device_branch_two_ranks(oracle_mod):
    """CUDA pack -> all-to-all -> owner wave -> pack hits -> all-to-all ->
    unpack, two ranks: hits, summed statistics and the union of the table
    partitions equal one process (the oracle)."""
    from conftest import load_golden
    got = _spawn(_key_sharded_worker)
    bvh = oracle_mod.OracleBvh.from_dict(load_golden("bvh_spheres.npz"))
    inp = load_golden("wave_inputs.npz")
    i = 0
    for mode in ("limit", "live"):
        tabs = {c: oracle_mod.OracleTable(6, 0, c) for c in (True, False)}
        for name, closest in WAVES:
            rc, ref, rst = oracle_mod.trace_wave(bvh, tabs[closest], mode, closest,
                                                 *(inp[f"{name}_{k}"] for k in
                                                   ("O", "D", "tmin", "tmax")))
            assert rc == 0
            parts = [got[r][i] for r in range(2)]
            for k in ("found", "t", "slot", "leaf"):
                assert np.array_equal(np.concatenate([p[2][k] for p in parts]), ref[k]), \
                    (mode, name, k)
            assert np.array_equal(parts[0][3] + parts[1][3], rst), (mode, name)
            i += 1
        for c in (True, False):
            union = sorted(got[0][i][2][c] + got[1][i][2][c])
            assert union == tabs[c].dump_lines(), (mode, c)
        i += 1


def _blocks_worker(rank, world, port, q):
    from conftest import load_golden
    import paper_1910_01304_b200 as hb
    from paper_1910_01304_b200.parallel import block_range, merge_wave_records
    dist = _setup(rank, world, port)
    try:
        staged = HostStagedDist(dist)
        g = load_golden("bvh_spheres.npz")
        b = hb.Bvh(*(g[k] for k in KEYS), int(g["max_depth"]))
        inp = load_golden("wave_inputs.npz")
        dev = torch.device("cuda", 0)
        tabs = {c: hb.PredictorTable(hb.HashConfig(6), 0,
                                     hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
                for c in (True, False)}
        merged = []
        for name, closest in WAVES:
            arrs = [inp[f"{name}_{k}"] for k in ("O", "D", "tmin", "tmax")]
            lo, hi = block_range(arrs[0].shape[0], rank, world)
            mine = [torch.from_numpy(np.ascontiguousarray(a[lo:hi])).to(dev) for a in arrs]
            hb.trace_wave(b, tabs[closest], "live", *mine, closest, defer_commit=True)
            merged.append(merge_wave_records(tabs[closest], staged, ray_offset=lo))
        q.put((rank, (merged, {c: list(t.dump_lines()) for c, t in tabs.items()})))
    finally:
        dist.destroy_process_group()


def test_block_records_device_merge_two_ranks():
    """Ray blocks with deferred commits: the device records of both ranks are
    all-gathered and applied in global ray order, leaving identical tables
    that equal the one-process two-block emulation."""
    import paper_1910_01304_b200 as hb
    from conftest import load_golden
    from paper_1910_01304_b200.parallel import block_range
    got = _spawn(_blocks_worker)
    assert got[0] == got[1]
    g = load_golden("bvh_spheres.npz")
    b = hb.Bvh(*(g[k] for k in KEYS), int(g["max_depth"]))
    inp = load_golden("wave_inputs.npz")
    # one process: each wave's two blocks against the same wave-start table
    ref = {c: hb.PredictorTable(hb.HashConfig(6), 0,
                                hb.RayKind.CLOSEST_HIT if c else hb.RayKind.HIT_ANY)
           for c in (True, False)}
    for name, closest in WAVES:
        arrs = [inp[f"{name}_{k}"] for k in ("O", "D", "tmin", "tmax")]
        n = arrs[0].shape[0]
        recs = []
        for rank in range(2):
            lo, hi = block_range(n, rank, 2)
            hb.trace_wave(b, ref[closest], "live", *(a[lo:hi] for a in arrs), closest,
                          defer_commit=True)
            k, nd, _ = ref[closest].pending_records()
            recs.append((k, nd))
        ref[closest].set_deferred(False)
        ref[closest].record_batch(np.concatenate([r[0] for r in recs]),
                                  np.concatenate([r[1] for r in recs]))
    assert got[0][1] == {c: list(t.dump_lines()) for c, t in ref.items()}
