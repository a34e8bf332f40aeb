"""Multi-GPU waves: exact key sharding, or ray blocks with a record exchange.

Key sharding (``key_sharded_wave``, exact at any world size):
the owner of key k is (mix64(k) >> 32) % world.  Each rank partitions its
contiguous block of a wave by owner (stable, ``partition_by_owner`` on the
device), one all-to-all moves every ray to the owner of its key, the owner
runs the wave on its table partition, and a second all-to-all returns the
hits.  Source blocks arrive in rank order, so each owner sees all rays of
its keys in global ray order; a key's consult touches only its own entry
(hrpp/tracer.py:233-267, 295-331), hence every hit, every statistic (summed
over ranks) and the union of the table partitions equal one GPU's.

Ray blocks (``merge_wave_records``, approximate): every rank holds the whole BVH
and a local predictor table, and takes a CONTIGUOUS block of every wave
(interleaving destroys within-wave training).  A rank consults its block in
ray order against its table in deferred mode, so the table is not modified
and the wave's append records (key, node, ray index) are kept.  Between
waves the records of all ranks are all-gathered (NCCL over NVLink on GPUs;
gloo in the CPU tests), ordered by global ray index and applied with the
sequential-semantics ``record_batch``: every rank ends the wave with the
identical table T_prev + records-in-ray-order.  With one rank this is
exactly the direct commit.  Within a wave, a rank does not see the other
ranks' inserts; that is the only difference from the single-GPU replay and
costs < 0.5 pp of savings at 8 ranks (SURVEY 8(e) probe).
"""

from __future__ import annotations

import numpy as np

from . import _lib


def block_range(n: int, rank: int, world: int):
    """[lo, hi) of this rank's contiguous block of an n-ray wave."""
    return (n * rank) // world, (n * (rank + 1)) // world


def _backend_device(dist, group=None):
    import torch
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_varlen(dist, t, group=None) -> list:
    """All-gather 1-D tensors of different lengths (padded to the longest):
    the list of every rank's tensor, in rank order, on the backend's
    device (NCCL: device-resident, nothing passes through the host)."""
    import torch
    dev = _backend_device(dist, group)
    world = dist.get_world_size(group)
    t = torch.as_tensor(t).to(dev)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(max(sizes), 1)
    buf = torch.zeros(m, dtype=t.dtype, device=dev)
    buf[:t.shape[0]] = t
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return [o[:s] for o, s in zip(outs, sizes)]


def merge_records(parts_keys, parts_nodes, parts_rays, offsets):
    """Host restatement of the merge (tests): concatenate per-rank records
    and order them by global ray index."""
    if not parts_keys:
        return np.zeros(0, np.uint64), np.zeros(0, np.int32)
    keys = np.concatenate(parts_keys).astype(np.uint64)
    nodes = np.concatenate(parts_nodes).astype(np.int32)
    rays = np.concatenate([r.astype(np.int64) + int(o) for r, o in zip(parts_rays, offsets)])
    order = np.argsort(rays, kind="stable")
    return keys[order], nodes[order]


def merge_wave_records(table, dist, ray_offset: int = 0, group=None):
    """Exchange the last deferred wave's records and apply them in global ray
    order on every rank (the collective step between waves).

    Every rank holds a contiguous block of the wave, blocks in rank order,
    and its records are sorted by ray index within the block, so the ranks'
    records concatenated in rank order ARE the wave's records in global ray
    order: one all-gather (NCCL over NVLink: device tensors end to end) and
    one sequential-semantics ``record_batch`` on the device.  ``ray_offset``
    (this block's first global ray) is checked to be non-decreasing in rank
    order."""
    import torch
    dev = _backend_device(dist, group)
    keys, nodes, _ = table.pending_records(device=dev.type == "cuda")
    if isinstance(keys, np.ndarray):
        keys, nodes = torch.from_numpy(keys.view(np.int64)), torch.from_numpy(nodes)
    else:
        keys = keys.view(torch.int64)
    offs = [int(o.item()) for o in all_gather_varlen(
        dist, torch.tensor([ray_offset], dtype=torch.int64), group)]
    if any(b < a for a, b in zip(offs, offs[1:])):
        raise ValueError("ray blocks must be in rank order")
    mk = torch.cat(all_gather_varlen(dist, keys, group))
    mn = torch.cat(all_gather_varlen(dist, nodes, group))
    if mk.shape[0]:
        if dev.type == "cuda":
            table.record_batch(mk.view(torch.uint64), mn)
        else:
            table.record_batch(mk.numpy().view(np.uint64), mn.numpy())
    return int(mk.shape[0])


# ---------------------------------------------------------------------------
# exact key sharding
# ---------------------------------------------------------------------------

def partition_by_owner(keys, world: int, device_counts: bool = False):
    """(perm, counts): this rank's rays grouped by key owner, ray order kept
    within each owner (hrpp_partition_by_owner).  ``keys`` is a CUDA uint64
    tensor; perm is a CUDA int32 tensor; counts a host int64[world], or with
    ``device_counts`` a CUDA int64 tensor (no host round trip)."""
    if not (_lib.is_torch(keys) and keys.is_cuda):
        raise ValueError("partition_by_owner needs device keys (a CUDA tensor)")
    n = int(keys.shape[0])
    perm = _lib.empty(n, np.int32, like=keys)
    if device_counts:
        counts = _lib.empty(int(world), np.int64, like=keys) if world > 0 else None
        cptr = _lib.ptr(counts)
    else:
        counts = np.zeros(max(int(world), 0), np.int64)
        cptr = counts.ctypes.data_as(_lib.C.c_void_p)
    rc = _lib.lib.hrpp_partition_by_owner(_lib.ptr(keys), n, int(world), _lib.ptr(perm), cptr,
                                          _lib.stream_of(keys))
    _lib.check(rc, "partition_by_owner")
    return perm, counts


def _a2a(dist, x, send_counts, recv_counts, group=None):
    """all_to_all_single of the leading dimension with uneven splits."""
    import torch
    shape = (int(sum(recv_counts)),) + tuple(x.shape[1:])
    flat = x.view(torch.uint8) if x.dtype == torch.bool else x
    out = torch.empty(shape, dtype=flat.dtype, device=x.device)
    dist.all_to_all_single(out, flat.contiguous(), [int(c) for c in recv_counts],
                           [int(c) for c in send_counts], group=group)
    return out.view(torch.bool) if x.dtype == torch.bool else out


HIT_FIELDS = ("found", "t", "slot", "leaf")


def key_sharded_wave(dist, trace_fn, key_fn, partition_fn, O, D, tmins, tmaxs, outputs=None,
                     group=None):
    """One wave over all ranks by key ownership (exact at any world size).

    O, D (n,3) float32, tmins/tmaxs (n,) float64: this rank's CONTIGUOUS
    block of the wave, blocks in rank order (``block_range``), as torch
    tensors on the collective backend's device.  ``key_fn(O, D)`` hashes
    (hrpp_hash_rays), ``partition_fn(keys, world)`` groups by owner
    (``partition_by_owner``) and ``trace_fn(O, D, tmins, tmaxs)`` runs this
    rank's table partition on the rays it owns (``trace_wave``) and returns
    (hits dict, stats).  Returns (hits in this rank's ray order for
    HIT_FIELDS, this rank's stats): the stats of all ranks sum to the
    single-GPU stats.
    """
    import torch
    world = dist.get_world_size(group)
    keys = key_fn(O, D)
    perm, counts = partition_fn(keys, world)
    perm32 = torch.as_tensor(perm, device=O.device).to(torch.int32).contiguous()
    perm = perm32.long()
    dev = O.device
    send = torch.as_tensor(counts, device=dev).to(torch.int64)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    both = torch.cat([send, recv]).cpu().tolist()  # the one host round trip
    send_counts = [int(c) for c in both[:world]]
    recv_counts = [int(c) for c in both[world:]]
    n = int(O.shape[0])
    out = dict(outputs) if outputs else {}
    if dev.type == "cuda":  # one all-to-all each way, rows packed on the device
        parts = _exchange_rays(dist, perm32, O, D, tmins, tmaxs, send_counts, recv_counts,
                               group)
        hits, stats = trace_fn(*parts)
        _exchange_hits(dist, hits, perm32, n, out, recv_counts, send_counts, group)
        return out, stats
    # host tensors (the gloo tests): the same exchange, one field at a time
    parts = [_a2a(dist, x.index_select(0, perm), send_counts, recv_counts, group)
             for x in (O, D, tmins, tmaxs)]
    hits, stats = trace_fn(*parts)
    for k in HIT_FIELDS:
        back = _a2a(dist, torch.as_tensor(hits[k], device=dev), recv_counts, send_counts, group)
        if k not in out:
            out[k] = torch.empty(n, dtype=back.dtype, device=dev)
        out[k].index_copy_(0, perm, back.to(out[k].dtype))
    return out, stats


def _exchange_rays(dist, perm32, O, D, tmins, tmaxs, send_counts, recv_counts, group):
    """Gather this rank's rays in owner order into 40-byte rows
    (hrpp_pack_rays), all-to-all them, unpack the received rows."""
    import torch
    dev = O.device
    st = _lib.stream_of(O)
    n = int(O.shape[0])
    O = O.reshape(-1, 3).to(torch.float32).contiguous()
    D = D.reshape(-1, 3).to(torch.float32).contiguous()
    t0 = tmins.reshape(-1).to(torch.float64).contiguous()
    t1 = tmaxs.reshape(-1).to(torch.float64).contiguous()
    rows = torch.empty((n, 40), dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib.hrpp_pack_rays(_lib.ptr(perm32), n, _lib.ptr(O), _lib.ptr(D),
                                       _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(rows), st),
               "pack_rays")
    got = _a2a(dist, rows, send_counts, recv_counts, group)
    m = int(got.shape[0])
    Or = torch.empty((m, 3), dtype=torch.float32, device=dev)
    Dr = torch.empty((m, 3), dtype=torch.float32, device=dev)
    t0r = torch.empty(m, dtype=torch.float64, device=dev)
    t1r = torch.empty(m, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib.hrpp_unpack_rays(_lib.ptr(got), m, _lib.ptr(Or), _lib.ptr(Dr),
                                         _lib.ptr(t0r), _lib.ptr(t1r), st), "unpack_rays")
    return Or, Dr, t0r, t1r


def _exchange_hits(dist, hits, perm32, n, out, send_counts, recv_counts, group):
    """Pack the owner's hits into 24-byte rows (hrpp_pack_hits), send them
    back, and scatter them to this rank's ray order (hrpp_unpack_hits)."""
    import torch
    f = hits["found"]
    dev = f.device
    st = _lib.stream_of(f)
    m = int(f.shape[0])
    cols = [torch.as_tensor(hits[k], device=dev).to(dt).contiguous()
            for k, dt in zip(HIT_FIELDS, (torch.bool, torch.float64, torch.int32, torch.int32))]
    rows = torch.empty((m, 24), dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib.hrpp_pack_hits(m, *(_lib.ptr(c) for c in cols), _lib.ptr(rows), st),
               "pack_hits")
    back = _a2a(dist, rows, send_counts, recv_counts, group)
    for k, dt in zip(HIT_FIELDS, (torch.bool, torch.float64, torch.int32, torch.int32)):
        if k not in out or out[k].dtype != dt or not out[k].is_contiguous():
            out[k] = torch.empty(n, dtype=dt, device=dev)
    _lib.check(_lib.lib.hrpp_unpack_hits(_lib.ptr(back), _lib.ptr(perm32), n,
                                         *(_lib.ptr(out[k]) for k in HIT_FIELDS), st),
               "unpack_hits")
