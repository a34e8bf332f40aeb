"""BVH handle, native builder and batch traversal (reference: hrpp/bvh.py).

``Bvh`` takes the reference's flat arrays (hrpp/bvh.py:75-92: bmin/bmax
(N,3) f32, left/right i32, axis i8, first/count i32, parent/depth i32,
tv0/tv1/tv2 (M,3) f32, tri_ids i32) and mirrors them once into the HBM
layout of csrc/hrpp_device.cuh (32-B float32 nodes, 96-B triangle records:
float64 v0 and edges plus the leaf).  Traversal
(``intersect_*``) runs the sm_100a float64 kernel; results are bit-identical
to hrpp/kernels.py.  ``build_bvh_from_arrays`` calls the native builder
(csrc/bvh_build.cpp), which reproduces the reference SAH builder's arrays.

Rays are float32, as everywhere on the reference's wave path (the hash
reads their bits, hrpp/geom.py:97-99); float64 inputs are rounded to
float32.  numpy arrays in -> numpy arrays out; CUDA tensors in -> CUDA
tensors out (zero-copy).
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .errors import EmptyScene
from .geom import HitRecord, Ray, RayKind, Triangle

log = logging.getLogger(__name__)

SAH_BINS = 16
DEFAULT_MAX_LEAF_SIZE = 4
MAX_STACK = 512


@dataclass
class TraversalCounters:
    """Per-run tallies (hrpp/bvh.py:37-51)."""

    box_tests: int = 0
    tri_tests: int = 0
    nodes_visited: int = 0

    def add(self, box_tests=0, tri_tests=0, nodes_visited=0):
        self.box_tests += int(box_tests)
        self.tri_tests += int(tri_tests)
        self.nodes_visited += int(nodes_visited)

    def merge(self, other: "TraversalCounters"):
        self.add(other.box_tests, other.tri_tests, other.nodes_visited)


@dataclass(frozen=True)
class BvhNode:
    index: int
    bmin: np.ndarray
    bmax: np.ndarray
    parent: Optional[int]
    depth: int
    left: Optional[int] = None
    right: Optional[int] = None
    first_prim: Optional[int] = None
    prim_count: Optional[int] = None

    @property
    def is_leaf(self) -> bool:
        return self.first_prim is not None


class Bvh:
    """Flat binary BVH; the device copy is created on first traversal."""

    def __init__(self, bmin, bmax, left, right, axis, first, count, parent, depth, tv0, tv1,
                 tv2, tri_ids, max_depth, device: Optional[int] = None):
        f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32).reshape(-1, 3)  # noqa: E731
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
        self.bmin, self.bmax = f32(bmin), f32(bmax)
        self.left, self.right = i32(left), i32(right)
        self.axis = np.ascontiguousarray(axis, dtype=np.int8)
        self.first, self.count = i32(first), i32(count)
        self.parent, self.depth = i32(parent), i32(depth)
        self.tv0, self.tv1, self.tv2 = f32(tv0), f32(tv1), f32(tv2)
        self.tri_ids = i32(tri_ids)
        self.max_depth = int(max_depth)
        self._device = device
        self._handle = None
        self._luts: dict[int, np.ndarray] = {}

    # -- device handle ---------------------------------------------------------

    @property
    def handle(self):
        if self._handle is None:
            dev = _lib.device_index() if self._device is None else int(self._device)
            h = C.c_void_p()
            rc = _lib.lib.hrpp_bvh_create(
                *(_lib.ptr(a) for a in (self.bmin, self.bmax, self.left, self.right, self.axis,
                                        self.first, self.count, self.parent, self.depth,
                                        self.tv0, self.tv1, self.tv2, self.tri_ids)),
                self.node_count, self.triangle_count, dev, C.byref(h))
            _lib.check(rc, "bvh_create")
            self._handle = h
            self._device = dev
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                _lib.lib.hrpp_bvh_destroy(h)
            except Exception:
                pass
            self._handle = None

    # -- structure ---------------------------------------------------------------

    @property
    def node_count(self) -> int:
        return self.bmin.shape[0]

    @property
    def triangle_count(self) -> int:
        return self.tv0.shape[0]

    @property
    def prim_order(self) -> np.ndarray:
        return self.tri_ids

    def is_leaf(self, i: int) -> bool:
        return self.left[i] < 0

    def node(self, i: int) -> BvhNode:
        par = int(self.parent[i])
        par = None if par < 0 else par
        if self.is_leaf(i):
            return BvhNode(i, self.bmin[i].copy(), self.bmax[i].copy(), par, int(self.depth[i]),
                           first_prim=int(self.first[i]), prim_count=int(self.count[i]))
        return BvhNode(i, self.bmin[i].copy(), self.bmax[i].copy(), par, int(self.depth[i]),
                       left=int(self.left[i]), right=int(self.right[i]))

    def leaf_indices(self) -> np.ndarray:
        return np.flatnonzero(self.left < 0).astype(np.int32)

    def _arrays(self):
        return (self.bmin, self.bmax, self.left, self.right, self.axis, self.first, self.count,
                self.tv0, self.tv1, self.tv2)

    def slot_normals(self) -> np.ndarray:
        e1 = self.tv1.astype(np.float64) - self.tv0.astype(np.float64)
        e2 = self.tv2.astype(np.float64) - self.tv0.astype(np.float64)
        nrm = np.cross(e1, e2)
        return nrm / np.linalg.norm(nrm, axis=1, keepdims=True)

    def ancestor_lut(self, go_up_level: int) -> np.ndarray:
        """node -> ancestor ``go_up_level`` steps up, clamped at the root
        (hrpp/bvh.py:140-151), computed by a device kernel and cached."""
        if go_up_level < 0:
            raise ValueError("go_up_level must be >= 0")
        lut = self._luts.get(go_up_level)
        if lut is None:
            lut = np.empty(self.node_count, np.int32)
            _lib.check(_lib.lib.hrpp_bvh_ancestor_lut(self.handle, int(go_up_level),
                                                      _lib.ptr(lut)), "ancestor_lut")
            self._luts[go_up_level] = lut
        return lut


def ancestor_at(bvh: Bvh, leaf: int, go_up_level: int) -> int:
    """The node ``go_up_level`` parent links above ``leaf``, clamped at the
    root (hrpp/bvh.py:154-166): an index into the device-built LUT."""
    if not (0 <= leaf < bvh.node_count):
        raise ValueError(f"node index {leaf} out of range")
    return int(bvh.ancestor_lut(go_up_level)[leaf])


# -- build ---------------------------------------------------------------------------


def build_bvh(triangles: Sequence[Triangle], max_leaf_size: int = DEFAULT_MAX_LEAF_SIZE) -> Bvh:
    if len(triangles) == 0:
        raise EmptyScene("no triangles supplied")
    v0 = np.array([t.v0 for t in triangles], dtype=np.float32).reshape(-1, 3)
    v1 = np.array([t.v1 for t in triangles], dtype=np.float32).reshape(-1, 3)
    v2 = np.array([t.v2 for t in triangles], dtype=np.float32).reshape(-1, 3)
    ids = np.array([t.id for t in triangles], dtype=np.int32)
    return build_bvh_from_arrays(v0, v1, v2, ids=ids, max_leaf_size=max_leaf_size)


def build_bvh_from_arrays(v0, v1, v2, ids=None, max_leaf_size: int = DEFAULT_MAX_LEAF_SIZE,
                          median_split: bool = False, device: Optional[int] = None) -> Bvh:
    """Native builder restating hrpp/bvh.py:184-357 (binned SAH, 16 bins);
    ``median_split=True`` builds the median-split tree of BASELINE config c1."""
    if max_leaf_size < 1:
        raise ValueError("max_leaf_size must be >= 1")
    v0 = np.ascontiguousarray(v0, dtype=np.float32).reshape(-1, 3)
    v1 = np.ascontiguousarray(v1, dtype=np.float32).reshape(-1, 3)
    v2 = np.ascontiguousarray(v2, dtype=np.float32).reshape(-1, 3)
    m = v0.shape[0]
    ids = (np.arange(m, dtype=np.int32) if ids is None
           else np.ascontiguousarray(ids, dtype=np.int32))
    cap = max(2 * m, 1)
    o = dict(bmin=np.zeros((cap, 3), np.float32), bmax=np.zeros((cap, 3), np.float32),
             left=np.zeros(cap, np.int32), right=np.zeros(cap, np.int32),
             axis=np.zeros(cap, np.int8), first=np.zeros(cap, np.int32),
             count=np.zeros(cap, np.int32), parent=np.zeros(cap, np.int32),
             depth=np.zeros(cap, np.int32), tv0=np.zeros((max(m, 1), 3), np.float32),
             tv1=np.zeros((max(m, 1), 3), np.float32), tv2=np.zeros((max(m, 1), 3), np.float32),
             tri_ids=np.zeros(max(m, 1), np.int32))
    nn, nt, md = C.c_int64(), C.c_int64(), C.c_int32()
    rc = _lib.lib.hrpp_build_bvh(
        _lib.ptr(v0), _lib.ptr(v1), _lib.ptr(v2), _lib.ptr(ids), m, int(max_leaf_size),
        int(bool(median_split)), *(_lib.ptr(o[k]) for k in (
            "bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth", "tv0",
            "tv1", "tv2", "tri_ids")), C.byref(nn), C.byref(nt), C.byref(md))
    if rc == _lib.INVALID_ARG and nt.value == 0:
        raise EmptyScene("no valid triangles remain after filtering")
    if rc != _lib.OK:
        raise RuntimeError(f"BVH build failed (status {rc}): depth limit exceeded?")
    if nt.value < m:
        log.warning("dropped %d degenerate triangle(s) before BVH build", m - nt.value)
    n, t = nn.value, nt.value
    return Bvh(o["bmin"][:n], o["bmax"][:n], o["left"][:n], o["right"][:n], o["axis"][:n],
               o["first"][:n], o["count"][:n], o["parent"][:n], o["depth"][:n], o["tv0"][:t],
               o["tv1"][:t], o["tv2"][:t], o["tri_ids"][:t], md.value, device=device)


# -- traversal -----------------------------------------------------------------------


def _batch(bvh: Bvh, closest: bool, O, D, tmins, tmaxs, start: int):
    if not (0 <= start < bvh.node_count):
        raise ValueError(f"start node {start} out of range")
    O = _lib.as_array(O, np.float32, shape=(-1, 3))
    D = _lib.as_array(D, np.float32, shape=(-1, 3))
    n = int(O.shape[0])
    t0 = _lib.as_array(tmins, np.float64)
    t1 = _lib.as_array(tmaxs, np.float64)
    out = {"found": _lib.empty(n, np.bool_, like=O), "t": _lib.empty(n, np.float64, like=O),
           "slot": _lib.empty(n, np.int32, like=O), "leaf": _lib.empty(n, np.int32, like=O)}
    if closest:
        out["u"] = _lib.empty(n, np.float64, like=O)
        out["v"] = _lib.empty(n, np.float64, like=O)
    out["box"] = _lib.empty(n, np.int64, like=O)
    out["tri"] = _lib.empty(n, np.int64, like=O)
    out["visited"] = _lib.empty(n, np.int64, like=O)
    w = _lib.WaveOut(*(_lib.ptr(out.get(k)) for k in ("found", "t", "slot", "leaf", "u", "v",
                                                       "box", "tri", "visited")), None)
    rc = _lib.lib.hrpp_trace_batch(bvh.handle, _lib.CLOSEST_HIT if closest else _lib.HIT_ANY,
                                   _lib.ptr(O), _lib.ptr(D), _lib.ptr(t0), _lib.ptr(t1),
                                   int(start), n, C.byref(w), _lib.stream_of(O))
    _lib.check(rc, "trace_batch")
    return out


def intersect_closest_batch(bvh: Bvh, O, D, tmins, tmaxs, start: int = 0):
    """hrpp/bvh.py:398-420: dict of found/t/slot/leaf/u/v/box/tri/visited."""
    return _batch(bvh, True, O, D, tmins, tmaxs, start)


def intersect_any_batch(bvh: Bvh, O, D, tmins, tmaxs, start: int = 0):
    """hrpp/bvh.py:423-442: dict of found/t/slot/leaf/box/tri/visited."""
    return _batch(bvh, False, O, D, tmins, tmaxs, start)


def intersect_from_node(bvh: Bvh, start: int, ray: Ray,
                        counters: TraversalCounters) -> Optional[HitRecord]:
    """Traversal restricted to the subtree rooted at ``start`` (bvh.py:379-395)."""
    closest = ray.kind is not RayKind.HIT_ANY
    r = _batch(bvh, closest, ray.origin[None, :], ray.direction[None, :],
               np.array([ray.t_min], np.float64), np.array([ray.t_max], np.float64), start)
    counters.add(r["box"][0], r["tri"][0], r["visited"][0])
    if not r["found"][0]:
        return None
    return HitRecord(t=float(r["t"][0]), triangle_id=int(bvh.tri_ids[r["slot"][0]]),
                     leaf_node=int(r["leaf"][0]), u=float(r["u"][0]) if closest else 0.0,
                     v=float(r["v"][0]) if closest else 0.0)


def intersect_closest(bvh: Bvh, ray: Ray, counters: TraversalCounters) -> Optional[HitRecord]:
    if ray.kind is not RayKind.CLOSEST_HIT:
        raise ValueError("intersect_closest requires a CLOSEST_HIT ray")
    return intersect_from_node(bvh, 0, ray, counters)


def intersect_any(bvh: Bvh, ray: Ray, counters: TraversalCounters) -> Optional[HitRecord]:
    if ray.kind is not RayKind.HIT_ANY:
        raise ValueError("intersect_any requires a HIT_ANY ray")
    return intersect_from_node(bvh, 0, ray, counters)
