"""ctypes front-end of the C oracle (TEST INFRASTRUCTURE ONLY).

Restates the reference HRPP path (``hrpp`` 0.1.0) on the CPU so that the
CUDA product path can be checked against it on the GPU box, where the
reference itself is absent.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline / ``--impl reference``) may import this module.

Parity of this oracle with the real reference is pinned by
``tests/test_oracle_golden.py`` against vectors that
``tests/golden/make_golden.py`` produced by running the reference.

Entry points and the reference code each one restates:

=======================  ==========================================
``hash_rays_np``         hrpp/rayhash.py:99-122 (numpy restatement)
``hash_rays``            same, C (or_hash_rays)
``OracleBvh.trace_batch`` hrpp/kernels.py:209-248, hrpp/bvh.py:398-442
``OracleTable``          hrpp/predictor.py:117-211
``trace_wave``           hrpp/tracer.py:217-371 (_consult_limit,
                         _consult_live, _trace_wave)
``predict_batch``        hrpp/predictor.py:167-192
=======================  ==========================================
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libhrpp_oracle.so"

OK, NONFINITE, CAPACITY, INVALID = 0, 1, 2, 3
STATS_FIELDS = ("rays", "tp", "fp", "neg", "baseline_box_tests", "baseline_tri_tests",
                "overhead_box_tests", "overhead_tri_tests", "skipped_box_tests",
                "skipped_box_tests_estimated", "wrong_closest")


class OracleError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"oracle {what} failed with status {code}")


SOURCES = ("hrpp_oracle.c", "hrpp_oracle_bvh.c")


def build(force: bool = False) -> Path:
    """Compile the C oracle with gcc (OpenMP if available)."""
    srcs = [HERE / s for s in SOURCES]
    if LIB_PATH.exists() and not force and all(LIB_PATH.stat().st_mtime >= s.stat().st_mtime
                                               for s in srcs):
        return LIB_PATH
    LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    base = ["gcc", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
            "-shared", "-o", str(LIB_PATH), *map(str, srcs), "-lm"]
    try:
        subprocess.run(base[:1] + ["-fopenmp"] + base[1:], check=True, capture_output=True)
    except subprocess.CalledProcessError:
        subprocess.run(base, check=True, capture_output=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        # idle OpenMP workers sleep instead of spinning: the sharded consult
        # and the traversal batches alternate with serial work (measured: a
        # spinning team slowed small sharded waves ~40x)
        os.environ.setdefault("OMP_WAIT_POLICY", "passive")
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32


def _declare(L):
    L.or_hash_rays.argtypes = [P, P, I64, C.c_int, P]
    L.or_hash_rays.restype = C.c_int
    bvh = [P] * 11 + [I64, I64]
    L.or_trace_batch.argtypes = bvh + [C.c_int, P, P, P, P, I32, I64] + [P] * 9 + [C.c_int]
    L.or_trace_batch.restype = C.c_int
    L.or_table_create.argtypes = [I64]
    L.or_table_create.restype = P
    L.or_table_destroy.argtypes = [P]
    L.or_table_destroy.restype = None
    L.or_table_record.argtypes = [P, P, P, I64, P]
    L.or_table_record.restype = C.c_int
    L.or_table_lookup.argtypes = [P, C.c_uint64, P, I64]
    L.or_table_lookup.restype = I64
    L.or_table_info.argtypes = [P, P, P, P]
    L.or_table_info.restype = None
    L.or_table_export.argtypes = [P, P, P, P]
    L.or_table_export.restype = None
    L.or_trace_wave.argtypes = (bvh + [P, P, C.c_int, C.c_int, C.c_int, P, P, P, P, I64]
                                + [P] * 9 + [P, P] + [P] * 4 + [C.c_int])
    L.or_trace_wave.restype = C.c_int
    L.or_predict_batch.argtypes = bvh + [P, C.c_int, P, P, P, P, P, I64] + [P] * 10
    L.or_predict_batch.restype = C.c_int
    L.or_max_threads.argtypes = []
    L.or_max_threads.restype = C.c_int
    L.or_trace_wave_sharded.argtypes = (bvh + [P, P, C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                                               P, P, I64] + [P] * 9 + [P, P])
    L.or_trace_wave_sharded.restype = C.c_int
    L.or_build_bvh.argtypes = [P, P, P, P, I64, C.c_int, C.c_int] + [P] * 13 + [P, P, P]
    L.or_build_bvh.restype = C.c_int
    L.or_set_fast_rounds.argtypes = [C.c_int, C.c_int]
    L.or_set_fast_rounds.restype = None


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# --------------------------------------------------------------------------
# hash
# --------------------------------------------------------------------------

def _lane_hash_np(bits, p):
    # hrpp/rayhash.py:118-122
    sign = bits >> np.uint32(31)
    exp_top = ((bits >> np.uint32(23)) & np.uint32(0xFF)) >> np.uint32(8 - p)
    man_top = (bits & np.uint32(0x7FFFFF)) >> np.uint32(23 - p)
    return (sign << np.uint32(2 * p)) | (exp_top << np.uint32(p)) | man_top


def partition_by_owner_np(keys, world):
    """CPU restatement of hrpp_partition_by_owner (k_shard.cu), the checker of
    the key-sharded multi-GPU mode: owner = (mix64(key) >> 32) % world;
    returns (stable permutation grouping rays by owner, counts per owner)."""
    x = np.asarray(keys, np.uint64).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xff51afd7ed558ccd)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xc4ceb9fe1a85ec53)
        x ^= x >> np.uint64(33)
    owner = ((x >> np.uint64(32)) % np.uint64(world)).astype(np.int64)
    perm = np.argsort(owner, kind="stable").astype(np.int32)
    return perm, np.bincount(owner, minlength=world).astype(np.int64)


def hash_rays_np(O, D, p):
    """numpy restatement of hrpp/rayhash.py:99-115; None on non-finite input."""
    bo = _c(O, np.float32).view(np.uint32).reshape(-1, 3)
    bd = _c(D, np.float32).view(np.uint32).reshape(-1, 3)
    if (((bo >> 23) & 0xFF) == 0xFF).any() or (((bd >> 23) & 0xFF) == 0xFF).any():
        return None
    key = np.zeros(bo.shape[0], np.uint64)
    for lane, (oi, di) in enumerate(((0, 2), (1, 1), (2, 0))):
        v = _lane_hash_np(bo[:, oi], p) ^ _lane_hash_np(bd[:, di], p)
        key |= v.astype(np.uint64) << np.uint64(16 * lane)
    return key


def hash_rays(O, D, p):
    O = _c(O, np.float32).reshape(-1, 3)
    D = _c(D, np.float32).reshape(-1, 3)
    n = O.shape[0]
    keys = np.zeros(n, np.uint64)
    rc = lib().or_hash_rays(_p(O), _p(D), n, p, _p(keys))
    if rc == NONFINITE:
        return None
    if rc != OK:
        raise OracleError(rc, "hash_rays")
    return keys


# --------------------------------------------------------------------------
# BVH
# --------------------------------------------------------------------------

class OracleBvh:
    """Holds the reference's flat BVH arrays (hrpp/bvh.py:75-92)."""

    def __init__(self, bmin, bmax, left, right, axis, first, count, parent, depth,
                 tv0, tv1, tv2, tri_ids=None, max_depth=None):
        self.bmin = _c(bmin, np.float32).reshape(-1, 3)
        self.bmax = _c(bmax, np.float32).reshape(-1, 3)
        self.left = _c(left, np.int32)
        self.right = _c(right, np.int32)
        self.axis = _c(axis, np.int8)
        self.first = _c(first, np.int32)
        self.count = _c(count, np.int32)
        self.parent = _c(parent, np.int32)
        self.depth = _c(depth, np.int32)
        self.tv0 = _c(tv0, np.float32).reshape(-1, 3)
        self.tv1 = _c(tv1, np.float32).reshape(-1, 3)
        self.tv2 = _c(tv2, np.float32).reshape(-1, 3)
        self.tri_ids = (np.arange(self.tv0.shape[0], dtype=np.int32) if tri_ids is None
                        else _c(tri_ids, np.int32))
        self._luts = {}

    @classmethod
    def from_dict(cls, d):
        keys = ("bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth",
                "tv0", "tv1", "tv2", "tri_ids")
        return cls(*(d[k] for k in keys))

    @property
    def node_count(self):
        return self.bmin.shape[0]

    def _args(self):
        return [_p(self.bmin), _p(self.bmax), _p(self.left), _p(self.right), _p(self.axis),
                _p(self.first), _p(self.count), _p(self.tv0), _p(self.tv1), _p(self.tv2),
                _p(self.depth), self.node_count, self.tv0.shape[0]]

    def ancestor_lut(self, g):
        # hrpp/bvh.py:140-151
        lut = self._luts.get(g)
        if lut is None:
            lut = np.arange(self.node_count, dtype=np.int32)
            for _ in range(g):
                up = self.parent[lut]
                lut = np.where(up < 0, lut, up).astype(np.int32)
            self._luts[g] = lut
        return lut

    def trace_batch(self, closest, O, D, tmins, tmaxs, start=0, threads=0):
        O = _c(O, np.float32).reshape(-1, 3)
        D = _c(D, np.float32).reshape(-1, 3)
        n = O.shape[0]
        out = {"found": np.zeros(n, np.bool_), "t": np.zeros(n), "slot": np.zeros(n, np.int32),
               "leaf": np.zeros(n, np.int32)}
        if closest:
            out["u"] = np.zeros(n)
            out["v"] = np.zeros(n)
        out.update(box=np.zeros(n, np.int64), tri=np.zeros(n, np.int64),
                   visited=np.zeros(n, np.int64))
        rc = lib().or_trace_batch(
            *self._args(), int(bool(closest)), _p(O), _p(D), _p(_c(tmins, np.float64)),
            _p(_c(tmaxs, np.float64)), int(start), n, _p(out["found"]), _p(out["t"]),
            _p(out["slot"]), _p(out["leaf"]), _p(out.get("u")), _p(out.get("v")),
            _p(out["box"]), _p(out["tri"]), _p(out["visited"]), int(threads))
        if rc != OK:
            raise OracleError(rc, "trace_batch")
        return out


def build_bvh(v0, v1, v2, ids=None, max_leaf_size=4, median_split=False):
    """hrpp/bvh.py:184-357 restated in C (oracle/hrpp_oracle_bvh.c): the
    reference builder's arrays, as an OracleBvh (+ ``max_depth``).  Raises
    ValueError when no triangle survives the degenerate filter."""
    v0, v1, v2 = (_c(a, np.float32).reshape(-1, 3) for a in (v0, v1, v2))
    m = v0.shape[0]
    ids = None if ids is None else _c(ids, np.int32)
    cap = max(2 * m, 1)
    o = {k: np.zeros((cap, 3), np.float32) for k in ("bmin", "bmax")}
    o.update({k: np.zeros(cap, np.int32) for k in ("left", "right", "first", "count", "parent",
                                                    "depth")})
    o["axis"] = np.zeros(cap, np.int8)
    o.update({k: np.zeros((max(m, 1), 3), np.float32) for k in ("tv0", "tv1", "tv2")})
    o["tri_ids"] = np.zeros(max(m, 1), np.int32)
    nn, nt, md = I64(), I64(), I32()
    order = ("bmin", "bmax", "left", "right", "axis", "first", "count", "parent", "depth", "tv0",
             "tv1", "tv2", "tri_ids")
    rc = lib().or_build_bvh(_p(v0), _p(v1), _p(v2), _p(ids), m, int(max_leaf_size),
                            int(bool(median_split)), *(_p(o[k]) for k in order), C.byref(nn),
                            C.byref(nt), C.byref(md))
    if rc == INVALID:
        raise ValueError("no valid triangles remain after filtering")
    if rc != OK:
        raise OracleError(rc, "build_bvh")
    n, t = nn.value, nt.value
    b = OracleBvh(*(o[k][:n] for k in order[:9]), *(o[k][:t] for k in order[9:]))
    b.max_depth = md.value
    return b


# --------------------------------------------------------------------------
# predictor table + wave
# --------------------------------------------------------------------------

class OracleTable:
    def __init__(self, p=6, go_up_level=0, closest=True, max_entries=1 << 26):
        self.p = int(p)
        self.go_up_level = int(go_up_level)
        self.closest = bool(closest)
        self.max_entries = int(max_entries)
        self._h = lib().or_table_create(self.max_entries)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.or_table_destroy(h)
            self._h = None

    def record_batch(self, keys, nodes):
        keys = _c(keys, np.uint64)
        nodes = _c(nodes, np.int32)
        ins = np.zeros(keys.shape[0], np.uint8)
        rc = lib().or_table_record(self._h, _p(keys), _p(nodes), keys.shape[0], _p(ins))
        return rc, ins.astype(bool)

    def lookup(self, key):
        n = lib().or_table_lookup(self._h, int(key), None, 0)
        if n == 0:
            return None
        out = np.zeros(n, np.int32)
        lib().or_table_lookup(self._h, int(key), _p(out), n)
        return out

    def info(self):
        e, s, m = I64(), I64(), I64()
        lib().or_table_info(self._h, C.byref(e), C.byref(s), C.byref(m))
        return e.value, s.value, m.value

    def export(self):
        e, s, _ = self.info()
        keys = np.zeros(e, np.uint64)
        offs = np.zeros(e + 1, np.int64)
        nodes = np.zeros(max(s, 1), np.int32)
        lib().or_table_export(self._h, _p(keys), _p(offs), _p(nodes))
        return keys, offs, nodes[:s]

    def dump_lines(self):
        keys, offs, nodes = self.export()
        return [f"{int(k):012x} -> [" + ",".join(str(int(x)) for x in nodes[offs[i]:offs[i + 1]])
                + "]" for i, k in enumerate(keys)]


class ShardedTable:
    """One logical predictor table held as ``shards`` key-disjoint tables,
    one per host thread (see or_trace_wave_sharded): trace_wave consults
    each shard's keys on its own thread, in ray order.  export() and
    dump_lines() give the union, sorted by key -- the single table's."""

    def __init__(self, p=6, go_up_level=0, closest=True, shards=None, max_entries=1 << 26):
        self.p = int(p)
        self.go_up_level = int(go_up_level)
        self.closest = bool(closest)
        self.shards = [OracleTable(p, go_up_level, closest, max_entries)
                       for _ in range(int(shards or os.cpu_count() or 1))]
        self._arr = (C.c_void_p * len(self.shards))(*(s._h for s in self.shards))

    def info(self):
        e = [s.info() for s in self.shards]
        return sum(x[0] for x in e), sum(x[1] for x in e), max(x[2] for x in e)

    def export(self):
        parts = [s.export() for s in self.shards]
        keys = np.concatenate([k for k, _, _ in parts])
        lists = [nd[o[i]:o[i + 1]] for _, o, nd in parts for i in range(len(o) - 1)]
        order = np.argsort(keys, kind="stable")
        lens = np.array([len(lists[i]) for i in order], np.int64)
        offs = np.zeros(len(order) + 1, np.int64)
        np.cumsum(lens, out=offs[1:])
        nodes = (np.concatenate([lists[i] for i in order]) if len(order)
                 else np.zeros(0, np.int32))
        return keys[order], offs, nodes.astype(np.int32)

    def dump_lines(self):
        keys, offs, nodes = self.export()
        return [f"{int(k):012x} -> [" + ",".join(str(int(x)) for x in nodes[offs[i]:offs[i + 1]])
                + "]" for i, k in enumerate(keys)]


MODES = {"baseline": 0, "limit": 1, "live": 2, "fast": 3}


def trace_wave(bvh: OracleBvh, table, mode, closest, O, D, tmins, tmaxs, stats=None,
               capture=False, threads=0):
    """hrpp/tracer.py:343-371.  Returns (status, out dict, stats int64[11])."""
    O = _c(O, np.float32).reshape(-1, 3)
    D = _c(D, np.float32).reshape(-1, 3)
    n = O.shape[0]
    m = MODES[mode] if isinstance(mode, str) else int(mode)
    stats = np.zeros(11, np.int64) if stats is None else stats
    out = {"found": np.zeros(n, np.bool_), "t": np.zeros(n), "slot": np.zeros(n, np.int32),
           "leaf": np.zeros(n, np.int32)}
    if m in (0, 1):
        if closest:
            out["u"] = np.zeros(n)
            out["v"] = np.zeros(n)
        out.update(box=np.zeros(n, np.int64), tri=np.zeros(n, np.int64),
                   visited=np.zeros(n, np.int64))
    keys = np.zeros(n, np.uint64) if m != 0 else None
    log = None
    if capture and m == 1:
        log = {"cls": np.zeros(n, np.int8), "eval_box": np.zeros(n, np.int64),
               "pred_t": np.zeros(n), "pred_slot": np.zeros(n, np.int64)}
    anc = bvh.ancestor_lut(table.go_up_level) if table is not None else None
    if isinstance(table, ShardedTable) and m != 0:
        rc = lib().or_trace_wave_sharded(
            *bvh._args(), _p(anc), table._arr, len(table.shards), table.p, m,
            int(bool(closest)), _p(O), _p(D), _p(_c(tmins, np.float64)),
            _p(_c(tmaxs, np.float64)), n, _p(out["found"]), _p(out["t"]), _p(out["slot"]),
            _p(out["leaf"]), _p(out.get("u")), _p(out.get("v")), _p(out.get("box")),
            _p(out.get("tri")), _p(out.get("visited")), _p(keys), _p(stats))
        if keys is not None:
            out["keys"] = keys
        return rc, out, stats
    rc = lib().or_trace_wave(
        *bvh._args(), _p(anc), None if table is None else table._h,
        0 if table is None else table.p, m, int(bool(closest)), _p(O), _p(D),
        _p(_c(tmins, np.float64)), _p(_c(tmaxs, np.float64)), n, _p(out["found"]), _p(out["t"]),
        _p(out["slot"]), _p(out["leaf"]), _p(out.get("u")), _p(out.get("v")), _p(out.get("box")),
        _p(out.get("tri")), _p(out.get("visited")), _p(keys), _p(stats),
        *([_p(log[k]) for k in ("cls", "eval_box", "pred_t", "pred_slot")] if log
          else [None] * 4), int(threads))
    if keys is not None:
        out["keys"] = keys
    if log is not None:
        out["log"] = log
    return rc, out, stats


def predict_batch(bvh: OracleBvh, table: OracleTable, closest, keys, O, D, tmins, tmaxs):
    O = _c(O, np.float32).reshape(-1, 3)
    D = _c(D, np.float32).reshape(-1, 3)
    n = O.shape[0]
    out = {"cls": np.zeros(n, np.int8), "t": np.zeros(n), "slot": np.zeros(n, np.int32),
           "leaf": np.zeros(n, np.int32), "u": np.zeros(n), "v": np.zeros(n),
           "box": np.zeros(n, np.int64), "tri": np.zeros(n, np.int64),
           "visited": np.zeros(n, np.int64), "est": np.zeros(n, np.int64)}
    rc = lib().or_predict_batch(
        *bvh._args(), table._h, int(bool(closest)), _p(_c(keys, np.uint64)), _p(O), _p(D),
        _p(_c(tmins, np.float64)), _p(_c(tmaxs, np.float64)), n,
        *[_p(out[k]) for k in ("cls", "t", "slot", "leaf", "u", "v", "box", "tri", "visited",
                               "est")])
    if rc != OK:
        raise OracleError(rc, "predict_batch")
    return out


def set_fast_rounds(rounds: int = 8, stop_div: int = 32):
    """Fast mode's speculation policy (oracle/hrpp_oracle.c fast_wave)."""
    lib().or_set_fast_rounds(int(rounds), int(stop_div))


def max_threads():
    return int(lib().or_max_threads())
