"""Predictor table in HBM (reference API: hrpp/predictor.py:117-211).

The reference keeps a Python dict of key -> insertion-ordered, de-duplicated
node lists.  Here the table lives on the GPU behind a C-ABI handle
(csrc/k_table.cu): an open-addressed hash index (atomicCAS inserts) over
48-bit keys, entry records {key, arena offset, length} and contiguous node
lists in an int32 arena.  The same semantics hold: ``record`` is an
idempotent append that raises ``CapacityExceeded`` only when a NEW key would
exceed ``max_entries`` (default 2^26, env ``HRPP_MAX_TABLE_ENTRIES``);
lookups never mutate; ``dump_lines`` is sorted by key.  One table serves one
ray kind.

Differences, by design: ``entries()`` iterates in key order (the reference
iterates in insertion order; no consumer depends on it), and a batch whose
new keys would exceed the cap leaves the table unchanged (the reference
stops half-way through its loop).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from enum import Enum
from typing import Iterator, Optional

import numpy as np

from . import _lib
from .bvh import Bvh, TraversalCounters, ancestor_at
from .geom import HitRecord, Ray, RayKind
from .rayhash import HashConfig, hash_ray, key_hex

DEFAULT_MAX_ENTRIES = 1 << 26
CAPACITY_ENV_VAR = "HRPP_MAX_TABLE_ENTRIES"
ENTRY_OVERHEAD_BYTES = 16
NODE_REF_BYTES = 4


class PredictionClass(Enum):
    TRUE_POSITIVE = "true_positive"
    FALSE_POSITIVE = "false_positive"
    NEGATIVE = "negative"


_CLS = {0: PredictionClass.TRUE_POSITIVE, 1: PredictionClass.FALSE_POSITIVE,
        2: PredictionClass.NEGATIVE}


@dataclass
class PredictionOutcome:
    classification: PredictionClass
    hit: Optional[HitRecord]
    overhead: TraversalCounters
    skipped_box_tests: int = 0


@dataclass
class MemoryEstimate:
    entry_bytes: int
    node_ref_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.entry_bytes + self.node_ref_bytes


class PredictorEntry:
    """Read-only snapshot of one entry's node list (insertion order)."""

    __slots__ = ("_nodes",)

    def __init__(self, nodes: np.ndarray):
        self._nodes = np.asarray(nodes, dtype=np.int32)

    @property
    def nodes(self) -> np.ndarray:
        return self._nodes

    def __len__(self) -> int:
        return int(self._nodes.shape[0])

    def __contains__(self, node) -> bool:
        return bool(np.any(self._nodes == node))


def _capacity_from_env(default: int) -> int:
    raw = os.environ.get(CAPACITY_ENV_VAR)
    if raw is None:
        return default
    try:
        cap = int(raw)
    except ValueError:
        raise ValueError(f"{CAPACITY_ENV_VAR} must be an integer, got {raw!r}")
    if cap < 1:
        raise ValueError(f"{CAPACITY_ENV_VAR} must be >= 1")
    return cap


class PredictorTable:
    """Device-resident mapping from 48-bit ray keys to predicted node lists."""

    def __init__(self, cfg: HashConfig, go_up_level: int = 0,
                 kind: RayKind = RayKind.CLOSEST_HIT, max_entries: Optional[int] = None,
                 device: Optional[int] = None):
        if go_up_level < 0:
            raise ValueError("go_up_level must be >= 0")
        if getattr(kind, "value", kind) not in (RayKind.CLOSEST_HIT.value, RayKind.HIT_ANY.value):
            raise ValueError(f"unknown ray kind {kind!r}")
        self.cfg = cfg
        self.go_up_level = int(go_up_level)
        self.kind = kind
        self.max_entries = (_capacity_from_env(DEFAULT_MAX_ENTRIES) if max_entries is None
                            else int(max_entries))
        self._device = device
        self._handle = None

    # -- handle ------------------------------------------------------------------

    @property
    def handle(self):
        if self._handle is None:
            dev = _lib.device_index() if self._device is None else int(self._device)
            h = C.c_void_p()
            rc = _lib.lib.hrpp_table_create(
                int(self.cfg.precision_bits), self.go_up_level,
                _lib.CLOSEST_HIT if self.closest else _lib.HIT_ANY,
                int(self.max_entries), dev, C.byref(h))
            _lib.check(rc, "table_create")
            self._handle = h
            self._device = dev
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                _lib.lib.hrpp_table_destroy(h)
            except Exception:
                pass
            self._handle = None

    @property
    def closest(self) -> bool:
        # by value: ``kind`` may be the reference's own RayKind member
        # (hrpp/geom.py), kept as given so its renderer's identity checks
        # (hrpp/tracer.py:384-387) hold
        return getattr(self.kind, "value", self.kind) == RayKind.CLOSEST_HIT.value

    def _info(self, with_max=False):
        if self._handle is None:
            return 0, 0, 0
        e, s, m = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib.hrpp_table_info(self._handle, C.byref(e), C.byref(s),
                                            C.byref(m) if with_max else None), "table_info")
        return e.value, s.value, m.value

    # -- core mapping (predictor.py:135-160) -------------------------------------------

    @property
    def entry_count(self) -> int:
        return self._info()[0]

    @property
    def stored_node_count(self) -> int:
        return self._info()[1]

    @property
    def max_nodes_per_entry(self) -> int:
        return self._info(with_max=True)[2]

    def lookup(self, key: int) -> Optional[PredictorEntry]:
        if self._handle is None:
            return None
        n = C.c_int64()
        _lib.check(_lib.lib.hrpp_table_lookup(self._handle, int(key), None, 0, C.byref(n)),
                   "lookup")
        if n.value == 0:
            return None
        buf = np.empty(n.value, np.int32)
        _lib.check(_lib.lib.hrpp_table_lookup(self._handle, int(key), _lib.ptr(buf), n.value,
                                              C.byref(n)), "lookup")
        return PredictorEntry(buf)

    def record_batch(self, keys, nodes):
        """Sequential-semantics batch of ``record`` calls; returns the per-record
        'entry grew' flags."""
        keys = _lib.as_array(keys, np.uint64)
        nodes = _lib.as_array(nodes, np.int32)
        n = int(keys.shape[0])
        ins = _lib.empty(n, np.bool_, like=keys)
        rc = _lib.lib.hrpp_table_record(self.handle, _lib.ptr(keys), _lib.ptr(nodes), n,
                                        _lib.ptr(ins), _lib.stream_of(keys))
        _lib.check(rc, "record")
        return ins

    def record(self, key: int, node: int) -> bool:
        """Idempotent set insertion; returns whether the entry grew."""
        return bool(self.record_batch(np.array([int(key)], np.uint64),
                                      np.array([int(node)], np.int32))[0])

    def export(self):
        """(keys sorted ascending, CSR offsets, nodes) copied to the host."""
        e, s, _ = self._info()
        keys = np.zeros(e, np.uint64)
        offs = np.zeros(e + 1, np.int64)
        nodes = np.zeros(max(s, 1), np.int32)
        if e:
            _lib.check(_lib.lib.hrpp_table_export(self._handle, _lib.ptr(keys), _lib.ptr(offs),
                                                  _lib.ptr(nodes)), "export")
        return keys, offs, nodes[:s]

    def entries(self) -> Iterator[tuple[int, PredictorEntry]]:
        keys, offs, nodes = self.export()
        for i, k in enumerate(keys):
            yield int(k), PredictorEntry(nodes[offs[i]:offs[i + 1]])

    # -- multi-GPU record exchange -------------------------------

    def set_deferred(self, on: bool):
        """In deferred mode a wave leaves the table unchanged and keeps its
        append records for ``pending_records`` (see parallel.py)."""
        on = bool(on)
        if getattr(self, "_deferred", False) != on:
            _lib.check(_lib.lib.hrpp_table_set_deferred(self.handle, int(on)), "set_deferred")
            self._deferred = on

    def pending_records(self, device: bool = False):
        """(keys u64, nodes i32, ray indices i32) of the last deferred wave,
        sorted by ray index within the wave: numpy arrays, or with ``device``
        CUDA tensors on the table's device (a device-to-device copy)."""
        cnt = C.c_int64()
        _lib.check(_lib.lib.hrpp_table_pending(self.handle, None, None, None, 0, C.byref(cnt)),
                   "pending")
        m = cnt.value
        if device:
            import torch
            dev = torch.device("cuda", self._device)
            keys = torch.empty(m, dtype=torch.uint64, device=dev)
            nodes = torch.empty(m, dtype=torch.int32, device=dev)
            rays = torch.empty(m, dtype=torch.int32, device=dev)
        else:
            keys = np.empty(m, np.uint64)
            nodes = np.empty(m, np.int32)
            rays = np.empty(m, np.int32)
        if m:
            _lib.check(_lib.lib.hrpp_table_pending(self.handle, _lib.ptr(keys), _lib.ptr(nodes),
                                                   _lib.ptr(rays), m, C.byref(cnt)), "pending")
        return keys, nodes, rays

    def clear(self, stream=None):
        """Empty the table (capacity kept).  Stream-ordered on ``stream`` (a
        torch stream or raw handle; default: torch's current stream when a
        device is in use), so the host does not wait."""
        if self._handle is not None:
            st = (_lib.current_stream_handle(self._device) if stream is None
                  else C.c_void_p(getattr(stream, "cuda_stream", stream)))
            _lib.check(_lib.lib.hrpp_table_clear_async(self._handle, st), "clear")

    # -- prediction (predictor.py:167-197) ---------------------------------------------

    def predict_batch(self, bvh: Bvh, O, D, tmins, tmaxs, keys=None):
        """predict() for a batch of rays against the frozen table."""
        O = _lib.as_array(O, np.float32, shape=(-1, 3))
        D = _lib.as_array(D, np.float32, shape=(-1, 3))
        n = int(O.shape[0])
        if keys is None:
            from .rayhash import hash_rays
            keys = hash_rays(O, D, self.cfg)
        keys = _lib.as_array(keys, np.uint64)
        t0 = _lib.as_array(tmins, np.float64)
        t1 = _lib.as_array(tmaxs, np.float64)
        spec = (("cls", np.int8), ("t", np.float64), ("slot", np.int32), ("leaf", np.int32),
                ("u", np.float64), ("v", np.float64), ("box", np.int64), ("tri", np.int64),
                ("visited", np.int64), ("est", np.int64))
        out = {k: _lib.empty(n, dt, like=O) for k, dt in spec}
        rc = _lib.lib.hrpp_predict_batch(bvh.handle, self.handle, _lib.ptr(keys), _lib.ptr(O),
                                         _lib.ptr(D), _lib.ptr(t0), _lib.ptr(t1), n,
                                         *(_lib.ptr(out[k]) for k, _ in spec),
                                         _lib.stream_of(O))
        _lib.check(rc, "predict")
        return out

    def predict(self, bvh: Bvh, ray: Ray) -> PredictionOutcome:
        """Consult the table for ``ray``; never mutates the table."""
        if getattr(ray.kind, "value", ray.kind) != getattr(self.kind, "value", self.kind):
            raise ValueError(
                f"table holds {self.kind.value} entries, got a {ray.kind.value} ray")
        key = hash_ray(ray, self.cfg)
        r = self.predict_batch(bvh, ray.origin[None, :], ray.direction[None, :],
                               np.array([ray.t_min]), np.array([ray.t_max]),
                               keys=np.array([key], np.uint64))
        overhead = TraversalCounters()
        overhead.add(r["box"][0], r["tri"][0], r["visited"][0])
        cls = _CLS[int(r["cls"][0])]
        if cls is not PredictionClass.TRUE_POSITIVE:
            return PredictionOutcome(cls, None, overhead)
        hit = HitRecord(t=float(r["t"][0]), triangle_id=int(bvh.tri_ids[r["slot"][0]]),
                        leaf_node=int(r["leaf"][0]), u=float(r["u"][0]), v=float(r["v"][0]))
        return PredictionOutcome(cls, hit, overhead, skipped_box_tests=int(r["est"][0]))

    def train_from_traversal(self, bvh: Bvh, key: int, hit: HitRecord) -> bool:
        """Record the go-up-level ancestor of a full traversal's hit leaf."""
        return self.record(key, ancestor_at(bvh, hit.leaf_node, self.go_up_level))

    # -- reporting (predictor.py:201-211) ----------------------------------------------

    def memory_estimate(self) -> MemoryEstimate:
        e, s, _ = self._info()
        return MemoryEstimate(entry_bytes=e * ENTRY_OVERHEAD_BYTES,
                              node_ref_bytes=s * NODE_REF_BYTES)

    def dump_lines(self) -> Iterator[str]:
        keys, offs, nodes = self.export()
        for i, k in enumerate(keys):
            body = ",".join(map(str, nodes[offs[i]:offs[i + 1]].tolist()))
            yield f"{key_hex(int(k))} -> [{body}]"


def memory_estimate(table: PredictorTable) -> MemoryEstimate:
    return table.memory_estimate()
