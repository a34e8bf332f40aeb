"""The wave: hash -> (full traversal) -> ray-ordered predictor consult.

Reference: ``_trace_wave`` (hrpp/tracer.py:343-371) with ``_consult_limit``
(:217-275) and ``_consult_live`` (:278-340).  One C-ABI call
(``hrpp_trace_wave``) runs the whole wave on the GPU:

* baseline -- full traversal of every ray; counters fill the denominators;
* limit -- full traversal + the exact per-key consult/train replay; the
  returned hits are the full-traversal hits, statistics are exact;
* live -- the reference's predict-or-traverse loop, exact: every ray that
  is not a true positive at its turn gets its full traversal (from the
  root) and trains the table in ray order.  On a table that is empty at
  the wave start every ray is traced up front (overlapping the grouping
  sort), since no TP is known before the wave's first appends; TPs then
  take their entry's result.  See DESIGN.md section 6;
* fast -- live mode as sort-free key-parallel speculation rounds, within a
  stated tolerance of exact.

``_trace_wave`` keeps the reference's signature so the reference renderer's
loop can call it unchanged; ``trace_wave`` is the array-level API used by
bench.py (numpy in/out, or CUDA tensors zero-copy).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum
from typing import Optional

import numpy as np

from . import _lib
from .bvh import Bvh
from .metrics import RayKindStats
from .predictor import PredictorTable

SHADOW_OFFSET = 1e-4
WRONG_CLOSEST_EPS = 1e-9
RAY_KIND_LABELS = ("primary", "shadow", "reflection")


class RenderMode(Enum):
    BASELINE = "baseline"
    LIMIT = "limit"
    LIVE = "live"
    # extension (no reference counterpart): live mode without the grouping
    # sort, as R key-parallel speculation rounds
    FAST = "fast"


_MODE = {RenderMode.BASELINE: _lib.MODE_BASELINE, RenderMode.LIMIT: _lib.MODE_LIMIT,
         RenderMode.LIVE: _lib.MODE_LIVE, RenderMode.FAST: _lib.MODE_FAST}

# RayKindStats field order (hrpp/metrics.py:38-51) = the C ABI's stats order
STATS_FIELDS = ("rays", "tp", "fp", "neg", "baseline_box_tests", "baseline_tri_tests",
                "overhead_box_tests", "overhead_tri_tests", "skipped_box_tests",
                "skipped_box_tests_estimated", "wrong_closest")


def as_mode(mode) -> RenderMode:
    """This package's RenderMode for any enum member or string whose value is
    baseline / limit / live -- the reference's own ``hrpp.tracer.RenderMode``
    (hrpp/tracer.py:58-61) included, so its renderer can pass its members."""
    if isinstance(mode, RenderMode):
        return mode
    return RenderMode(getattr(mode, "value", mode))


def add_stats(stats, raw) -> None:
    """Add the int64[11] counters into any object with the RayKindStats
    attributes (hrpp/metrics.py:38-51), by field name."""
    for name, v in zip(STATS_FIELDS, np.asarray(raw).tolist()):
        setattr(stats, name, getattr(stats, name) + int(v))


@dataclass
class OutcomeLog:
    """Per-consulted-ray records in limit mode (hrpp/tracer.py:144-153)."""

    classification: np.ndarray
    eval_box_tests: np.ndarray
    baseline_box_tests: np.ndarray
    predicted_t: np.ndarray
    predicted_slot: np.ndarray
    keys: np.ndarray


def set_live_rounds(rounds: int):
    """Exact consult rounds before the speculative round (speed only)."""
    _lib.check(_lib.lib.hrpp_set_live_rounds(int(rounds)), "set_live_rounds")


FAST_ROUNDS, FAST_STOP_DIV = 8, 32  # the library's defaults


def set_fast_rounds(rounds: int = FAST_ROUNDS, stop_div: int = FAST_STOP_DIV):
    """Fast mode's speculation policy: at most ``rounds`` rounds, none after
    a round that resolved fewer than n / stop_div rays (0: never stop early).
    Moves statistics within the stated tolerance, never found flags."""
    _lib.check(_lib.lib.hrpp_set_fast_rounds(int(rounds), int(stop_div)), "set_fast_rounds")


def set_consult_short(length: int):
    """Key segments with <= length rays are replayed per lane (speed only)."""
    _lib.check(_lib.lib.hrpp_set_consult_short(int(length)), "set_consult_short")


def trace_wave(bvh: Bvh, table: Optional[PredictorTable], mode: RenderMode, O, D, tmins,
               tmaxs, closest: bool, stats: Optional[np.ndarray] = None,
               capture_outcomes: bool = False, want_keys: bool = False, outputs=None,
               defer_commit: bool = False):
    """Run one wave.  Returns (result dict, stats int64[11]).

    Result keys: found, t, slot, leaf (+ u, v (closest), box, tri, visited in
    baseline/limit mode), keys (if requested or captured) and, with
    ``capture_outcomes`` in limit mode, log_cls / log_eval_box / log_pred_t /
    log_pred_slot.  ``outputs`` may pre-supply result arrays (reused buffers).
    """
    mode = as_mode(mode)
    if mode is not RenderMode.BASELINE:
        if table is None:
            raise ValueError(f"{mode.value} mode needs a predictor table")
        if table.closest != bool(closest):
            raise ValueError("table kind does not match the wave's ray kind")
    if table is not None and mode is not RenderMode.BASELINE:
        table.set_deferred(defer_commit)
    O = _lib.as_array(O, np.float32, shape=(-1, 3))
    D = _lib.as_array(D, np.float32, shape=(-1, 3))
    n = int(O.shape[0])
    t0 = _lib.as_array(tmins, np.float64)
    t1 = _lib.as_array(tmaxs, np.float64)
    if stats is None:
        stats = np.zeros(_lib.STATS_LEN, np.int64)
    out = dict(outputs) if outputs else {}

    def want(k, dt):
        if k not in out:
            out[k] = _lib.empty(n, dt, like=O)

    for k, dt in (("found", np.bool_), ("t", np.float64), ("slot", np.int32),
                  ("leaf", np.int32)):
        want(k, dt)
    if mode not in (RenderMode.LIVE, RenderMode.FAST):
        if closest:
            want("u", np.float64)
            want("v", np.float64)
        for k in ("box", "tri", "visited"):
            want(k, np.int64)
    if mode is not RenderMode.BASELINE and (want_keys or capture_outcomes):
        want("keys", np.uint64)
    log = None
    if capture_outcomes and mode is RenderMode.LIMIT:
        for k, dt in (("log_cls", np.int8), ("log_eval_box", np.int64),
                      ("log_pred_t", np.float64), ("log_pred_slot", np.int64)):
            want(k, dt)
        log = _lib.OutcomeLogC(*(_lib.ptr(out[k]) for k in ("log_cls", "log_eval_box",
                                                             "log_pred_t", "log_pred_slot")))
    w = _lib.WaveOut(*(_lib.ptr(out.get(k)) for k in ("found", "t", "slot", "leaf", "u", "v",
                                                       "box", "tri", "visited", "keys")))
    rc = _lib.lib.hrpp_trace_wave(
        bvh.handle, None if table is None else table.handle, _MODE[mode], int(bool(closest)),
        _lib.ptr(O), _lib.ptr(D), _lib.ptr(t0), _lib.ptr(t1), n, C.byref(w),
        C.byref(log) if log is not None else None, stats.ctypes.data_as(C.c_void_p),
        _lib.stream_of(O))
    _lib.check(rc, "trace_wave")
    return out, stats


def _trace_wave(bvh, table, cfg, mode, O32, D32, tmins, tmaxs, stats: RayKindStats,
                closest: bool, log_lists):
    """Drop-in for hrpp/tracer.py:343-371 (same arguments, same effects):
    adds into ``stats`` (this package's or the reference's RayKindStats, by
    field name), extends ``log_lists`` in limit mode, mutates ``table`` and
    returns the hits shading should use.  ``mode`` may be the reference's
    RenderMode member (converted by value)."""
    mode = as_mode(mode)
    capture = log_lists is not None and mode is RenderMode.LIMIT
    raw = np.zeros(_lib.STATS_LEN, np.int64)
    try:
        out, raw = trace_wave(bvh, table, mode, O32, D32, tmins, tmaxs, closest, stats=raw,
                              capture_outcomes=capture)
    finally:
        add_stats(stats, raw)
    if capture:
        log_lists["cls"].extend(out["log_cls"].tolist())
        log_lists["eval_box"].extend(out["log_eval_box"].tolist())
        log_lists["base_box"].extend(out["box"].tolist())
        log_lists["pred_t"].extend(out["log_pred_t"].tolist())
        log_lists["pred_slot"].extend(out["log_pred_slot"].tolist())
        log_lists["keys"].extend(out["keys"].tolist())
    return {k: v for k, v in out.items() if not k.startswith("log_") and k != "keys"}
