"""Ray waves generated and spawned on the GPU (csrc/k_spawn.cu).

* ``generate_primary_rays`` -- the reference's ``generate_primary_rays``
  (hrpp/tracer.py:173-211, counter RNG hrpp/rng.py:15-31), bit-identical,
  returned as CUDA tensors (or numpy with ``to_host=True``).
* ``spawn_secondary`` -- from a closest-hit wave's hits: shadow rays to a
  point light (bit-identical to hrpp/tracer.py:442-464) or an area light,
  and mirror (bit-identical to hrpp/tracer.py:488-492) or cosine-weighted
  diffuse bounces.  Hits are compacted in ray order, as the renderer does.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib


def _stratum_grid(spp):
    sx = max(1, int(math.sqrt(spp)))
    while spp % sx:
        sx -= 1
    return sx, spp // sx


def camera_basis(position, look_at, up):
    """hrpp/tracer.py:84-97 (float64, numpy, once per camera)."""
    pos = np.asarray(position, np.float32).astype(np.float64)
    fwd = np.asarray(look_at, np.float32).astype(np.float64) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float32).astype(np.float64))
    right /= np.linalg.norm(right)
    return fwd, right, np.cross(right, fwd)


def generate_primary_rays(camera, spp: int, seed: int = 0, jitter: bool = True,
                          to_host: bool = False):
    import torch
    w, h = camera.resolution
    n = w * h * spp
    fwd, right, up = camera_basis(camera.position, camera.look_at, camera.up)
    basis = np.ascontiguousarray(np.concatenate([fwd, right, up]), np.float64)
    pos = np.asarray(camera.position, np.float32)
    sx, sy = _stratum_grid(spp)
    dev = torch.device("cuda", _lib.device_index())
    O = torch.empty((n, 3), dtype=torch.float32, device=dev)
    D = torch.empty((n, 3), dtype=torch.float32, device=dev)
    _lib.check(_lib.lib.hrpp_gen_primary(
        _lib.ptr(pos), _lib.ptr(basis), math.tan(math.radians(camera.vertical_fov) / 2.0), w / h,
        w, h, spp, sx, sy, int(seed) & 0xFFFFFFFFFFFFFFFF, int(bool(jitter)), _lib.ptr(O),
        _lib.ptr(D), _lib.stream_of(O)), "gen_primary")
    if to_host:
        return O.cpu().numpy(), D.cpu().numpy()
    return O, D


def spawn_secondary(bvh, O, D, hits, shadow=None, bounce=None, seed: int = 0):
    """Secondary waves from ``hits`` (dict with found/t/slot of a closest-hit
    wave).  shadow: ("point", xyz) | ("area", center_xyz, half); bounce:
    "mirror" | "diffuse" | None.  Returns {"shadow": (O, D, tmin, tmax),
    "bounce": (...), "count": hits} as CUDA tensors."""
    import torch
    dev = torch.device("cuda", _lib.device_index())
    to_dev = lambda a, dt: torch.as_tensor(np.asarray(a) if not _lib.is_torch(a) else a,  # noqa
                                           dtype=dt).to(dev).contiguous()
    Ot, Dt = to_dev(O, torch.float32).reshape(-1, 3), to_dev(D, torch.float32).reshape(-1, 3)
    found = to_dev(hits["found"], torch.bool)
    t = to_dev(hits["t"], torch.float64)
    slot = to_dev(hits["slot"], torch.int32)
    n = Ot.shape[0]
    sk, light, half = 0, np.zeros(3), 0.0
    if shadow is not None:
        if shadow[0] == "point":
            sk, light = 1, np.asarray(shadow[1], np.float32).astype(np.float64)
        elif shadow[0] == "area":
            sk, light, half = 2, np.asarray(shadow[1], np.float64), float(shadow[2])
        else:
            raise ValueError(f"unknown shadow kind {shadow[0]!r}")
    bk = {None: 0, "mirror": 1, "diffuse": 2}[bounce]
    light = np.ascontiguousarray(light, np.float64)
    f32 = lambda shp: torch.empty(shp, dtype=torch.float32, device=dev)  # noqa: E731
    f64 = lambda shp: torch.empty(shp, dtype=torch.float64, device=dev)  # noqa: E731
    so, sd, s0, s1 = f32((n, 3)), f32((n, 3)), f64(n), f64(n)
    bo, bd, b0, b1 = f32((n, 3)), f32((n, 3)), f64(n), f64(n)
    import ctypes as C
    m = C.c_int64()
    _lib.check(_lib.lib.hrpp_spawn(
        bvh.handle, _lib.ptr(Ot), _lib.ptr(Dt), _lib.ptr(found), _lib.ptr(t), _lib.ptr(slot), n,
        sk, _lib.ptr(light), half, bk, int(seed) & 0xFFFFFFFFFFFFFFFF, _lib.ptr(so), _lib.ptr(sd),
        _lib.ptr(s0), _lib.ptr(s1), _lib.ptr(bo), _lib.ptr(bd), _lib.ptr(b0), _lib.ptr(b1),
        C.byref(m), _lib.stream_of(Ot)), "spawn")
    k = m.value
    out = {"count": k}
    if sk:
        out["shadow"] = (so[:k], sd[:k], s0[:k], s1[:k])
    if bk:
        out["bounce"] = (bo[:k], bd[:k], b0[:k], b1[:k])
    return out
