#!/usr/bin/env python
"""HRPP hot-path benchmark (BASELINE.json metric, config c2 by default).

A step is one frame of BASELINE config c2 through the HRPP hot path in live
mode (predict first, full traversal only for rays that are not true
positives, train in ray order): the 1024x1024x8 primary wave (hit-all),
one area-light shadow ray per primary hit (hit-any) and one cosine-weighted
diffuse bounce per primary hit (hit-all), with fresh predictor tables per
frame.  Inputs (float32 origins/directions, float64 tmin/tmax; 335 MB for the
primary wave alone, larger than the 126 MB L2) are resident in HBM before the
timed region; scenes and waves are seeded synthetic stand-ins.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Rank 0 prints one JSON line.  Multi-GPU: one process per GPU (torchrun);
each rank takes a contiguous block of every wave and its own predictor
tables; new (key, node) records are all-gathered between waves and merged in
ray order.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mrays/s with HRPP prediction vs full traversal; % BVH node visits skipped"
KINDS = ("primary", "shadow", "bounce")
STATS_NAMES = ("rays", "tp", "fp", "neg", "baseline_box_tests", "baseline_tri_tests",
               "overhead_box_tests", "overhead_tri_tests", "skipped_box_tests",
               "skipped_box_tests_estimated", "wrong_closest")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--res", default=None, help="override resolution WxH (testing)")
    ap.add_argument("--spp", type=int, default=None)
    ap.add_argument("--precision", type=int, default=6)
    ap.add_argument("--go-up", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-warm", action="store_true", help="skip the warm-table block")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the distributed wave path (NCCL collectives) even at N = 1 (testing)")
    ap.add_argument("--shard", default="keys", choices=["keys", "blocks"],
                    help="N > 1: exact key sharding (all-to-all) or ray blocks + record merge")
    ap.add_argument("--live-rounds", type=int, default=None)
    ap.add_argument("--consult-short", type=int, default=None)
    ap.add_argument("--profile-only", action="store_true",
                    help="setup + a few live frames, no extras (for ncu)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def make_workload_device(args, seed=0, scene_bvh=None):
    """The same frame generated on the GPU (our arm): primary rays by
    k_gen_primary, full-traversal hits on the device, shadow and bounce
    waves by k_spawn, so the waves never leave HBM.  Bit-identical to
    make_workload's numpy waves (tests/test_gpu_parity.py
    test_device_waves_equal_host_waves).  Returns the same triple with CUDA
    tensors in the waves.  ``seed`` re-jitters the frame (0: the bench's and
    the tests' frame); ``scene_bvh`` reuses an already built (scene, bvh)."""
    import paper_1910_01304_b200 as hb
    from paper_1910_01304_b200 import scenes, waves as dwaves
    if scene_bvh is not None:
        sc, bvh = scene_bvh
    else:
        res = tuple(int(x) for x in args.res.split("x")) if args.res else None
        sc = scenes.make_scene(args.config, resolution=res, spp=args.spp)
        bvh = hb.build_bvh_from_arrays(sc.v0, sc.v1, sc.v2, median_split=sc.builder == "median")
    O, D = dwaves.generate_primary_rays(sc.camera, sc.spp, seed=seed)
    n = O.shape[0]
    t0 = torch_zeros(n, O.device)
    waves = [("primary", "primary", True, O, D, t0, torch_inf(n, O.device))]
    cur = waves[0]
    for level in range(sc.bounces + 1):
        _, _, _, Oc, Dc, a, b = cur
        base = hb.intersect_closest_batch(bvh, Oc, Dc, a, b)
        lights = ([("area", sc.area_light[0], sc.area_light[1])] if sc.area_light is not None
                  else [("point", lp) for lp in sc.point_lights])
        shadow = level < sc.bounces or level == 0
        bounce = "diffuse" if level < sc.bounces else None
        for li, light in enumerate(lights if shadow else [None]):
            sp = dwaves.spawn_secondary(bvh, Oc, Dc, base, shadow=light,
                                        bounce=bounce if li == 0 else None,
                                        seed=level + 1000 * seed)
            if light is not None:
                waves.append((f"shadow{level}_{li}", "shadow", False, *sp["shadow"]))
            if li == 0 and bounce:
                nxt = (f"bounce{level + 1}", "bounce", True, *sp["bounce"])
        if level < sc.bounces:
            cur = nxt
            waves.append(cur)
    return sc, bvh, waves


def torch_zeros(n, dev):
    import torch
    return torch.zeros(n, dtype=torch.float64, device=dev)


def torch_inf(n, dev):
    import torch
    return torch.full((n,), float("inf"), dtype=torch.float64, device=dev)


def make_workload(args, trace_closest=None, build=None):
    """Scene, BVH and the ordered waves of one frame (host numpy).

    Waves: the primary wave; shadow rays (one wave per light) from its hits;
    then for every diffuse bounce b = 1..B the bounce wave spawned from the
    previous closest-hit wave, followed by its shadow waves except after the
    last bounce.  `build` makes the BVH (the native builder in our arm, the
    oracle's restatement of the reference builder in the reference arm) and
    `trace_closest` gives the full-traversal hits used for spawning (GPU in
    our arm, the oracle in the reference arm); both pairs are bit-identical.
    Returns (scene, bvh, [(name, kind, closest, O, D, tmin, tmax), ...])."""
    from paper_1910_01304_b200 import scenes  # numpy only: loads no native library
    res = tuple(int(x) for x in args.res.split("x")) if args.res else None
    sc = scenes.make_scene(args.config, resolution=res, spp=args.spp)
    if build is None:
        import paper_1910_01304_b200 as hb
        build = hb.build_bvh_from_arrays
    bvh = build(sc.v0, sc.v1, sc.v2, median_split=sc.builder == "median")
    normals = scenes.slot_normals(bvh.tv0, bvh.tv1, bvh.tv2)
    O, D = scenes.primary_rays(sc.camera, sc.spp, seed=0)
    n = O.shape[0]
    waves = [("primary", "primary", True, O, D, np.zeros(n), np.full(n, np.inf))]
    cur = waves[0]
    for level in range(sc.bounces + 1):
        _, _, _, Oc, Dc, t0, t1 = cur
        base = trace_closest(bvh, Oc, Dc, t0, t1)
        _, P, N = scenes.hit_frames(Oc, Dc, base["found"], base["t"], base["slot"], normals)
        if level < sc.bounces or level == 0:
            if sc.area_light is not None:
                lps = [scenes.area_light_samples(P.shape[0], sc.area_light[0], sc.area_light[1],
                                                 seed=level)]
            else:
                lps = [np.broadcast_to(np.asarray(lp, np.float64), P.shape)
                       for lp in sc.point_lights]
            for li, lp in enumerate(lps):
                waves.append((f"shadow{level}_{li}", "shadow", False, *scenes.shadow_rays(P, lp)))
        if level < sc.bounces:
            cur = (f"bounce{level + 1}", "bounce", True, *scenes.cosine_bounce(P, N, seed=level))
            waves.append(cur)
    return sc, bvh, waves


def shard(wave, rank, world):
    """Contiguous ray block of this rank (never interleave: SURVEY 8(e))."""
    name, kind, closest, O, D, t0, t1 = wave
    n = O.shape[0]
    lo, hi = (n * rank) // world, (n * (rank + 1)) // world
    return name, kind, closest, O[lo:hi], D[lo:hi], t0[lo:hi], t1[lo:hi]


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock and clock-event reasons sampled during the timed region: NVML
    every 2 ms from a thread (a timed region of a few frames is < 100 ms, too
    short for nvidia-smi's polling); nvidia-smi -lms as the fallback."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.proc = None
        self.lines = []
        self.device = device
        self.nv = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = (("hw_slowdown", nv.nvmlClocksEventReasonHwSlowdown),
                    ("hw_thermal_slowdown", nv.nvmlClocksEventReasonHwThermalSlowdown),
                    ("sw_thermal_slowdown", nv.nvmlClocksEventReasonSwThermalSlowdown),
                    ("sw_power_cap", nv.nvmlClocksEventReasonSwPowerCap))

            def poll():
                while not self.stop.is_set():
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    flags = ["Active" if r & b else "Not Active" for _, b in bits]
                    self.lines.append(", ".join([str(sm), str(mx), "0", hex(r)] + flags))
                    time.sleep(0.002)

            self.nv = nv
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1910_01304_b200 as hb
    from paper_1910_01304_b200 import _lib
    from paper_1910_01304_b200.parallel import (key_sharded_wave, merge_wave_records,
                                                partition_by_owner)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    multi = world > 1 or args.force_dist  # distributed wave paths (collectives)
    if args.live_rounds is not None:
        hb.set_live_rounds(args.live_rounds)
    if args.consult_short is not None:
        hb.set_consult_short(args.consult_short)

    # the frame's waves generated on the device (never leave HBM); host copies
    # (outside any timed region) feed the e2e leg and the CPU baseline
    sc, bvh, gen_waves = make_workload_device(args)
    waves = [(*w[:3], *(a.cpu().numpy() for a in w[3:])) for w in gen_waves]
    cfg = hb.HashConfig(args.precision)
    tables = {True: hb.PredictorTable(cfg, args.go_up, hb.RayKind.CLOSEST_HIT, device=local_rank),
              False: hb.PredictorTable(cfg, args.go_up, hb.RayKind.HIT_ANY, device=local_rank)}
    my = [shard(w, rank, world) for w in waves]
    offsets = [(w[3].shape[0] * rank) // world for w in waves]
    dwaves = [(w[2], *(a.contiguous() for a in w[3:]))
              for w in (shard(g, rank, world) for g in gen_waves)]
    n_local = sum(w[1].shape[0] for w in dwaves)
    n_total = sum(w[3].shape[0] for w in waves)
    kinds = sorted({w[1] for w in waves}, key=KINDS.index)
    stream = torch.cuda.current_stream()

    keyed = multi and args.shard == "keys"

    def run_wave(j, mode, O, D, t0, t1, stats=None, outputs=None):
        """One wave of this rank: key-sharded (exact), or its ray block with
        the deferred-record exchange, or (N = 1) the plain call."""
        closest = waves[j][2]
        table = tables[closest] if mode != "baseline" else None
        if keyed and mode != "baseline":
            def trace_fn(Oo, Do, a, b):
                return hb.trace_wave(bvh, table, mode, Oo, Do, a, b, closest, stats=stats)
            return key_sharded_wave(dist, trace_fn, lambda Oo, Do: hb.hash_rays(Oo, Do, cfg),
                                    lambda k, w: partition_by_owner(k, w, device_counts=True),
                                    O, D, t0, t1, outputs=outputs)[0]
        out, _ = hb.trace_wave(bvh, table, mode, O, D, t0, t1, closest, stats=stats,
                               outputs=outputs, defer_commit=multi and mode != "baseline")
        if multi and mode != "baseline":
            merge_wave_records(table, dist, ray_offset=offsets[j])
        return out

    # output buffers reused frame to frame (trace_wave(outputs=...)), as a
    # renderer would; live mode writes found/t/slot/leaf
    wave_out = [{"found": torch.empty(w[1].shape[0], dtype=torch.bool, device=dev),
                 "t": torch.empty(w[1].shape[0], dtype=torch.float64, device=dev),
                 "slot": torch.empty(w[1].shape[0], dtype=torch.int32, device=dev),
                 "leaf": torch.empty(w[1].shape[0], dtype=torch.int32, device=dev)}
                for w in dwaves]

    def frame(mode, stats=None):
        for t in tables.values():
            t.clear()  # stream-ordered (hrpp_table_clear_async)
        for j, (closest, O, D, t0, t1) in enumerate(dwaves):
            run_wave(j, mode, O, D, t0, t1, stats=stats[waves[j][1]] if stats is not None else None,
                     outputs=wave_out[j] if mode == "live" and not keyed else None)

    def barrier():
        if multi:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1)
        if multi:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    if args.profile_only:
        for _ in range(max(1, args.warmup)):
            frame("live")
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"profile_only": True, "rays": n_total}))
        return

    # ---- headline: live frames --------------------------------------------------------
    for _ in range(args.warmup):
        frame("live")
    # Stage breakdown from an untimed pass with every stage bracketed by events
    # (~60 event pairs a frame cost ~4 % of the frame); the timed region then
    # records only the dominant stage, for the roofline's launch durations.
    _lib.profile_enable(True)
    _lib.profile_read(reset=True)
    for _ in range(args.steps):
        frame("live")
    prof = _lib.profile_read(reset=True)
    dom_stage = max(("hash", "trace_queue", "consult"), key=lambda k: prof[k][0])
    _lib.profile_enable(True, stages=[dom_stage])
    launches0 = _lib.launch_count()
    with ClockSampler(local_rank) as clk:
        ms_live = timed(lambda: frame("live"), args.steps)
    prof_timed = _lib.profile_read(reset=True)
    _lib.profile_enable(False)
    launches = _lib.launch_count() - launches0
    value = n_total * args.steps / (ms_live * 1e-3) / 1e6

    # stats of one live frame (identical every frame: fresh tables, same rays)
    live_stats = {k: np.zeros(11, np.int64) for k in kinds}
    frame("live", stats=live_stats)
    stored_live = sum(int(t.stored_node_count) for t in tables.values())

    # ---- full traversal (baseline mode) and exact savings (limit mode) ---------------
    for _ in range(2):
        frame("baseline")
    ms_base = timed(lambda: frame("baseline"), args.steps)
    base_value = n_total * args.steps / (ms_base * 1e-3) / 1e6

    # ---- fast mode (sort-free speculation rounds) -------------
    fast = None
    if not multi:
        for _ in range(2):
            frame("fast")
        ms_fast = timed(lambda: frame("fast"), args.steps)
        fast_stats = {k: np.zeros(11, np.int64) for k in kinds}
        frame("fast", stats=fast_stats)
        fast = {"mrays_s": round(n_total * args.steps / (ms_fast * 1e-3) / 1e6, 3),
                "ms_per_step": round(ms_fast / args.steps, 4),
                "speedup_vs_full_traversal": round(ms_base / ms_fast, 4),
                "policy": {"max_rounds": hb.tracer.FAST_ROUNDS,
                           "stop_div": hb.tracer.FAST_STOP_DIV},
                "stats": {k: dict(zip(STATS_NAMES, map(int, fast_stats[k]))) for k in kinds},
                "tp_rel_vs_exact_live": {
                    k: round((int(fast_stats[k][1]) - int(live_stats[k][1]))
                             / max(1, int(live_stats[k][1])), 4) for k in kinds},
                "note": "statistics within the stated tolerance of exact live mode "
                        "(tests/test_fast_mode.py); found flags and table_entries exact"}
    # ---- tables kept from the previous frame (extra, N = 1) -----------------------------
    # The reference renders one frame on fresh tables, and so does the headline.
    # A renderer that keeps its tables sees wave-start TPs: frame 0 trains the
    # tables, frame 1 (same camera, re-jittered rays, light and bounce samples)
    # is traced on them, wave by wave against its own full traversal.
    warm = None
    if not multi and not args.no_warm:
        _, _, gen1 = make_workload_device(args, seed=1, scene_bvh=(sc, bvh))
        w1 = [(w[0], w[1], w[2], *(a.contiguous() for a in w[3:])) for w in gen1]

        def frame1(mode, acc, st_acc=None):
            for name, kind, closest, O, D, t0, t1 in w1:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _, st = hb.trace_wave(bvh, tables[closest] if mode != "baseline" else None, mode,
                                      O, D, t0, t1, closest)
                e1.record(stream)
                acc.setdefault(name, []).append((e0, e1))
                if st_acc is not None:
                    st_acc[name] = st

        t_base, t_warm, st_warm = {}, {}, {}
        for rep in range(4):
            frame1("baseline", t_base if rep else {})
            frame("live")  # frame 0 on fresh tables: trains them
            frame1("live", t_warm if rep else {}, st_warm)
        torch.cuda.synchronize()
        med = lambda ev: float(np.median([a.elapsed_time(b) for a, b in ev]))  # noqa: E731
        wb = {k: med(v) for k, v in t_base.items()}
        ww = {k: med(v) for k, v in t_warm.items()}
        mixed = ww["primary"] + sum(v for k, v in wb.items() if k != "primary")
        warm = {
            "what": "frame 1 (re-jittered) traced on the tables frame 0 left, against frame 1's "
                    "own full traversal; per-wave CUDA events, median of 3",
            "frame_ms": {"full_traversal": round(sum(wb.values()), 3),
                         "live_warm": round(sum(ww.values()), 3)},
            "waves_ms": {k: {"full_traversal": round(wb[k], 3), "live_warm": round(ww[k], 3)}
                         for k in wb},
            "primary": {"tp_percent": round(100.0 * int(st_warm["primary"][1])
                                            / max(1, int(st_warm["primary"][0])), 2),
                        "traced_box_tests": int(st_warm["primary"][4]),
                        "speedup_vs_full_traversal": round(wb["primary"] / ww["primary"], 4)},
            "hrpp_on_primary_rays_only": {
                "frame_ms": round(mixed, 3),
                "speedup_vs_full_traversal": round(sum(wb.values()) / mixed, 4),
                "note": "live mode on the primary wave, baseline mode on the others"},
        }
        del gen1, w1
    lim_stats = {k: np.zeros(11, np.int64) for k in kinds}
    frame("limit", stats=lim_stats)
    tstats = {}
    for c, t in tables.items():
        ts = hb.table_stats(t)
        if keyed:  # disjoint key partitions: the union's stats
            v = torch.tensor([ts.entries, ts.stored_nodes, ts.memory.entry_bytes,
                              ts.memory.node_ref_bytes], dtype=torch.int64, device=dev)
            mx = torch.tensor([ts.max_nodes_per_entry], dtype=torch.int64, device=dev)
            dist.all_reduce(v)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            e, sn, eb, nb = (int(x) for x in v.tolist())
            ts = hb.TableStats(entries=e, stored_nodes=sn,
                               avg_nodes_per_entry=sn / e if e else 0.0,
                               max_nodes_per_entry=int(mx.item()),
                               memory=hb.MemoryEstimate(entry_bytes=eb, node_ref_bytes=nb))
        tstats["closest" if c else "hit_any"] = ts
    if multi:
        for d_ in (lim_stats, live_stats):
            for k in kinds:
                t = torch.from_numpy(d_[k]).to(dev)
                dist.all_reduce(t)
                d_[k] = t.cpu().numpy()

    def pct(a, b):
        return 100.0 * a / b if b else 0.0

    savings = {k: round(pct(lim_stats[k][8], lim_stats[k][4]), 4) for k in kinds}
    base_boxes = sum(int(lim_stats[k][4]) for k in kinds)
    live_boxes = sum(int(live_stats[k][4] + live_stats[k][6]) for k in kinds)
    visit_reduction = 100.0 * (1.0 - live_boxes / base_boxes) if base_boxes else 0.0

    # ---- roofline of the dominant stage -------------------------------------------------
    steps = args.steps
    per_frame = {k: (v[0] / steps, v[1] / steps) for k, v in prof.items()}
    s_live = {i: sum(int(live_stats[k][i]) for k in kinds) // world for i in range(11)}
    n_fallback = s_live[2] + s_live[3]
    alg = {  # algorithmic bytes per frame
        "hash": 32 * n_local,
        "trace_queue": 64 * n_fallback + 32 * s_live[4] + 36 * s_live[5],
        "consult": 72 * n_local + 32 * s_live[6] + 36 * s_live[7] + 32 * stored_live,
    }
    peak = (json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
            if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0)
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (measured copy)"
                if (ROOT / "MEASURED_PEAKS.json").exists() else "fallback 6650 GB/s")
    stages = {}
    for k, (ms, cnt) in per_frame.items():
        if cnt == 0:
            continue
        ent = {"ms_per_frame": round(ms, 4), "launches_per_frame": cnt,
               "share": round(ms / (ms_live / steps), 4)}
        if k in alg and ms > 0:
            ent["achieved_gbs"] = round(alg[k] / (ms * 1e-3) / 1e9, 2)
            ent["frac_of_hbm_peak"] = round(alg[k] / (ms * 1e-3) / 1e9 / peak, 4)
        stages[k] = ent
    dom = dom_stage
    tq = prof_timed[dom]  # (ms, launches) of the dominant stage inside the timed region
    d_ms = tq[0] / max(1, tq[1])  # average launch duration
    d_bytes = alg[dom] / max(1, tq[1] / steps)
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():  # ncu DRAM bytes per launch of the stage, by config
        traffic = json.loads(tp.read_text()).get(args.config, {}).get(dom)
    achieved = d_bytes / (d_ms * 1e-3) / 1e9
    roofline = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": peak_src,
                "achieved_note": "algorithmic bytes (SURVEY 8(d): 32 B/box test, 36 B/tri test, "
                                 "64 B/ray I/O) per launch / mean launch time"}
    if traffic:
        dram = traffic / (d_ms * 1e-3) / 1e9
        roofline.update(dram_achieved=round(dram, 2), dram_frac=round(dram / peak, 4))
    if dom.startswith("trace"):
        roofline["bound_note"] = (
            "the traversal's node/triangle reads mostly hit L1/L2 (c5: 56 % L2, 61 % L1 "
            "hit rate; profiles/r2_c5_trace_full.md): it is bound by dependent-load latency "
            "and SIMT divergence (~10 of 32 lanes active), not by DRAM bandwidth; dram_frac "
            "is the HBM share actually used")

    # ---- e2e: host buffers through the public API ------------------------------------
    # Every step copies each wave's inputs from pinned host memory and its hits
    # back.  The copies run on a side stream, overlapped with the previous /
    # next wave's compute (waves still run in order: the tables chain them).
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        h_in, h_out = [], []
        h2d = d2h = 0
        for w in my:
            n = w[3].shape[0]
            h_in.append([pin(a) for a in w[3:]])
            mk = lambda dt: torch.empty(n, dtype=dt).pin_memory()  # noqa: E731
            h_out.append({"found": mk(torch.bool), "t": mk(torch.float64),
                          "slot": mk(torch.int32), "leaf": mk(torch.int32)})
            h2d += sum(t.numel() * t.element_size() for t in h_in[-1])
            d2h += sum(t.numel() * t.element_size() for t in h_out[-1].values())
        # device buffers double-buffered by frame parity, so the uploads of
        # frame f+1 run while frame f computes
        d_in = [[[torch.empty_like(t, device=dev) for t in h] for h in h_in] for _ in range(2)]
        d_out = [[{k: torch.empty_like(v, device=dev) for k, v in h.items()} for h in h_out]
                 for _ in range(2)]
        copy = torch.cuda.Stream(device=dev)   # uploads
        copy_back = torch.cuda.Stream(device=dev)  # downloads (the other copy engine)
        W = len(my)

        def run_e2e(frames):
            """`frames` frames back to back as one (frame, wave) pipeline:
            uploads run a whole frame ahead on one copy engine, downloads on
            the other, the waves in order on the compute stream."""
            items = [(f, j) for f in range(frames) for j in range(W)]
            ev_up = [torch.cuda.Event() for _ in items]
            ev_comp = [torch.cuda.Event() for _ in items]
            ev_down = [torch.cuda.Event() for _ in items]

            skip = os.environ.get("HRPP_E2E_DIAG_SKIP", "")  # diagnosis only: up|down

            def upload(i):
                f, j = items[i]
                if skip == "up" and i >= W:
                    ev_up[i].record(copy)
                    return
                with torch.cuda.stream(copy):
                    if i >= 2 * W:  # buffer last read by item i - 2W
                        copy.wait_event(ev_comp[i - 2 * W])
                    for d_, h_ in zip(d_in[f % 2][j], h_in[j]):
                        d_.copy_(h_, non_blocking=True)
                    ev_up[i].record(copy)

            for i in range(min(W, len(items))):
                upload(i)
            for i, (f, j) in enumerate(items):
                if j == 0:
                    for t in tables.values():
                        t.clear()
                if i + W < len(items):
                    upload(i + W)
                stream.wait_event(ev_up[i])
                if i >= 2 * W:  # output buffer last downloaded by item i - 2W
                    stream.wait_event(ev_down[i - 2 * W])
                run_wave(j, "live", *d_in[f % 2][j], outputs=d_out[f % 2][j])
                ev_comp[i].record(stream)
                copy_back.wait_event(ev_comp[i])
                with torch.cuda.stream(copy_back):
                    if skip != "down":
                        for k in h_out[j]:
                            h_out[j][k].copy_(d_out[f % 2][j][k], non_blocking=True)
                    ev_down[i].record(copy_back)
            copy.synchronize()
            copy_back.synchronize()

        run_e2e(1)
        barrier()
        t0w = time.perf_counter()
        e_steps = args.steps
        run_e2e(e_steps)
        barrier()
        dt = time.perf_counter() - t0w
        if multi:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(n_total * e_steps / dt / 1e6, 3), "unit": "Mrays/s",
               "h2d_bytes_per_step": int(h2d * world), "d2h_bytes_per_step": int(d2h * world),
               "how": "pinned host inputs -> trace_wave (public API) -> pinned host hits every "
                      "step; uploads one frame ahead (double-buffered) and downloads on the two "
                      "copy engines, overlapped with compute; K frames back to back; wall "
                      "clock"}

    # ---- CPU baseline (oracle port, rank 0, N=1 only) ---------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, n_cpu, threads = cpu_reference_frame(_oracle_bvh(bvh), waves, args)
        cpu = {"value": round(n_cpu / dt / 1e6, 4), "unit": "Mrays/s", "cores": threads,
               "kind": "port", "sample": cpu_sample_desc(n_cpu, threads),
               "seconds": round(dt, 3)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_live / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded displaced icosphere scene + generated ray waves)",
            "config": dict(workload_config(args, sc, bvh, waves),
                           parallelism=(f"key sharding x{world} (exact; all-to-all of rays "
                                        "to key owners)" if keyed else
                                        f"contiguous ray blocks x{world}")),
            "full_traversal_mrays_s": round(base_value, 3),
            "speedup_vs_full_traversal": round(value / base_value, 4),
            "nodes_skipped_percent": savings,
            "live_node_visit_reduction_percent": round(visit_reduction, 3),
            "table_stats": {k: {"entries": v.entries, "stored_nodes": v.stored_nodes,
                                "avg_nodes_per_entry": round(v.avg_nodes_per_entry, 4),
                                "max_nodes_per_entry": v.max_nodes_per_entry,
                                "memory_bytes": v.memory.total_bytes}
                            for k, v in tstats.items()},
            "limit_stats": {k: dict(zip(STATS_NAMES, map(int, lim_stats[k]))) for k in kinds},
            "live_stats": {k: dict(zip(STATS_NAMES, map(int, live_stats[k]))) for k in kinds},
            "stages": stages,
            "stages_note": "per-stage CUDA events in a separate untimed pass of the same frames; "
                           "a live wave on an empty table (the first wave of each ray kind) "
                           "traces on a side stream while its grouping is queued beside it "
                           "(the group stage's events span that wait), so group and "
                           "trace_queue overlap and the stages sum past the frame; "
                           "the roofline stage alone is event-timed inside the timed region",
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "fast_mode": fast,
            "warm_tables": warm,
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line))


# ---------------------------------------------------------------------------
# CPU reference (the oracle port; reference arm and cpu_baseline)
# ---------------------------------------------------------------------------

def workload_config(args, sc, bvh, waves):
    """The line's `config`, identical in both arms (same scene, BVH, waves)."""
    res = sc.camera.resolution
    return {"workload": f"{args.config}: {sc.n_tris} tris, {res[0]}x{res[1]} spp{sc.spp}, "
                        f"{len(waves)} waves (" + ", ".join(w[0] for w in waves) + ")",
            "mode": "live (predict, else full traversal, train in ray order)",
            "rays_per_step": int(sum(w[3].shape[0] for w in waves)),
            "rays_per_wave": {w[0]: int(w[3].shape[0]) for w in waves},
            "bvh_nodes": int(bvh.node_count), "bvh_max_depth": int(bvh.max_depth),
            "precision": args.precision, "go_up": args.go_up,
            "l2": "inputs > L2 (335 MB primary wave); no flush needed"}


def _oracle_bvh(bvh):
    from oracle import oracle
    oracle.build()
    return oracle.OracleBvh(bvh.bmin, bvh.bmax, bvh.left, bvh.right, bvh.axis, bvh.first,
                            bvh.count, bvh.parent, bvh.depth, bvh.tv0, bvh.tv1, bvh.tv2,
                            bvh.tri_ids)


def cpu_reference_frame(ob, waves, args):
    """One live-mode frame (every ray of every wave, fresh tables) through the
    oracle: the reference's sequential consult loop (hrpp/tracer.py:278-340
    restated in C) on every host core, each core running it for the keys it
    owns (exact: a key's entry is read and written only by its own rays).
    Returns (seconds, rays, threads)."""
    from oracle import oracle
    threads = os.cpu_count() or 1
    tabs = {c: oracle.ShardedTable(args.precision, args.go_up, c, shards=threads)
            for c in (True, False)}
    n = 0
    t0 = time.perf_counter()
    for _, _, closest, O, D, a, b in waves:
        rc, _, _ = oracle.trace_wave(ob, tabs[closest], "live", closest, O, D, a, b)
        assert rc == 0
        n += O.shape[0]
    return time.perf_counter() - t0, n, threads


def cpu_sample_desc(n, threads):
    return (f"one full live-mode frame ({n} rays, every wave, fresh tables); C oracle "
            f"(oracle/hrpp_oracle.c, the reference's consult loop restated) on {threads} host "
            f"threads, keys sharded across threads (exact); host has {os.cpu_count()} cores")


def run_reference(args, rank, world):
    """The reference algorithm on the host cores for the same frame: scene
    and waves from the same generators, the BVH from the oracle's own
    restatement of the reference builder, full-traversal spawning and the
    timed frames through the oracle.  Never loads the product library."""
    if rank != 0:
        return
    from oracle import oracle
    oracle.build()

    def cpu_trace(b, O, D, t0, t1):
        return b.trace_batch(True, O, D, t0, t1, threads=0)

    sc, ob, waves = make_workload(args, cpu_trace, build=oracle.build_bvh)
    frames = []
    for _ in range(args.warmup):
        cpu_reference_frame(ob, waves, args)
    for _ in range(args.steps):
        dt, n, threads = cpu_reference_frame(ob, waves, args)
        frames.append(dt)
    total = sum(frames)
    value = round(n * len(frames) / total / 1e6, 4)
    line = {"metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * total / len(frames), 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same seeded scene and waves as our arm)", "impl": "reference",
            "config": dict(workload_config(args, sc, ob, waves),
                           parallelism=f"host threads x{threads}"),
            "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads,
                             "kind": "port", "sample": cpu_sample_desc(n, threads)},
            "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    multi = world > 1 or args.force_dist
    if multi:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank),
                                rank=rank, world_size=world)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if multi:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
