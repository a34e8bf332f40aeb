"""Seeded synthetic scenes and ray waves for BASELINE.json configs c1..c5.

The paper's PBRT scenes (Teapot, Killeroo, Buddha, Sportscar) are not
available, and the reference ships no icosphere/noise/instancing generator
(hrpp/scene_io.py:106-223 has grid, UV spheres and Menger only).  These
generators are stand-ins at the configs' triangle counts: displaced
icospheres (value noise / fBm radial displacement), seeded face trimming,
instancing, and a ground quad, all float32.

Ray waves follow the reference conventions:

* primary rays -- ``generate_primary_rays`` semantics (hrpp/tracer.py:173-211):
  pixel-major / sample-minor order, stratified jitter from the counter RNG
  ``unit_floats`` (hrpp/rng.py:15-31), float32 unit directions;
* shadow rays (hit-any) -- origin offset 1e-4 along the geometric normal
  flipped to face the incoming ray, tmax = max(dist - 1e-4, 1e-6)
  (hrpp/tracer.py:449-464), toward a point light or a uniform sample on a
  1x1 area light;
* diffuse bounces (hit-all) -- cosine-weighted about the facing normal,
  tmin 0, tmax inf (absent from the reference renderer; BASELINE configs).

This module is input generation (host numpy), not the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_U = np.uint64
_M1 = _U(0xBF58476D1CE4E5B9)
_M2 = _U(0x94D049BB133111EB)
_GOLDEN = _U(0x9E3779B97F4A7C15)


# ---------------------------------------------------------------------------
# counter RNG (restates hrpp/rng.py:15-31 so primary rays match bit for bit)
# ---------------------------------------------------------------------------

def _mix(x):
    x = x ^ (x >> _U(30))
    x = x * _M1
    x = x ^ (x >> _U(27))
    x = x * _M2
    return x ^ (x >> _U(31))


def unit_floats(seed: int, pixel, sample, dim: int):
    pixel = np.asarray(pixel, dtype=np.uint64)
    sample = np.asarray(sample, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix(_U(seed & 0xFFFFFFFFFFFFFFFF) + _GOLDEN)
        h = _mix(h ^ (pixel * _GOLDEN + _U(1)))
        h = _mix(h ^ (sample * _M1 + _U(dim) * _M2 + _U(1)))
    return (h >> _U(11)).astype(np.float64) * (2.0 ** -53)


# ---------------------------------------------------------------------------
# geometry generators
# ---------------------------------------------------------------------------

def icosphere(subdiv: int):
    """Unit icosphere: (V,3) float64 vertices, (F,3) int64 faces; F = 20*4^s."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)
    for _ in range(subdiv):
        nv = v.shape[0]
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        e.sort(axis=1)
        code = e[:, 0] * nv + e[:, 1]
        uniq, inv = np.unique(code, return_inverse=True)
        a, b = uniq // nv, uniq % nv
        mid = v[a] + v[b]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = nv + inv.reshape(3, -1)
        v = np.concatenate([v, mid])
        m01, m12, m20 = m[0], m[1], m[2]
        f = np.concatenate([
            np.stack([f[:, 0], m01, m20], 1), np.stack([f[:, 1], m12, m01], 1),
            np.stack([f[:, 2], m20, m12], 1), np.stack([m01, m12, m20], 1)])
    return v, f


def _lattice(ix, iy, iz, seed):
    with np.errstate(over="ignore"):
        h = (ix.astype(np.int64).astype(np.uint64) * _U(0x8DA6B343)
             ^ iy.astype(np.int64).astype(np.uint64) * _U(0xD8163841)
             ^ iz.astype(np.int64).astype(np.uint64) * _U(0xCB1AB31F)
             ^ (_U(seed) * _GOLDEN))
        h = _mix(h)
    return (h >> _U(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def value_noise(p, seed: int):
    """Trilinear, smoothstep-faded value noise in [-1, 1] at points p (n,3)."""
    fl = np.floor(p)
    fr = p - fl
    w = fr * fr * (3.0 - 2.0 * fr)
    i = fl.astype(np.int64)
    out = np.zeros(p.shape[0])
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                c = _lattice(i[:, 0] + dx, i[:, 1] + dy, i[:, 2] + dz, seed)
                wx = w[:, 0] if dx else 1.0 - w[:, 0]
                wy = w[:, 1] if dy else 1.0 - w[:, 1]
                wz = w[:, 2] if dz else 1.0 - w[:, 2]
                out += c * wx * wy * wz
    return out


def fbm(p, seed: int, octaves: int, lacunarity=2.0, gain=0.5):
    out = np.zeros(p.shape[0])
    amp, freq, norm = 1.0, 1.0, 0.0
    for o in range(octaves):
        out += amp * value_noise(p * freq, seed + 7919 * o)
        norm += amp
        amp *= gain
        freq *= lacunarity
    return out / norm


def displaced_icosphere(subdiv, seed, amplitude, octaves=1, frequency=2.5):
    v, f = icosphere(subdiv)
    n = fbm(v * frequency, seed, octaves) if octaves > 1 else value_noise(v * frequency, seed)
    v = v * (1.0 + amplitude * n)[:, None]
    return v, f


def trim_faces(f, target, seed):
    if target >= f.shape[0]:
        return f
    rng = np.random.default_rng(seed)
    keep = np.sort(rng.choice(f.shape[0], size=target, replace=False))
    return f[keep]


def ground_quad(y, half):
    a, b, c, d = [(-half, y, -half), (half, y, -half), (half, y, half), (-half, y, half)]
    v0 = np.array([a, a], np.float32)
    v1 = np.array([c, d], np.float32)
    v2 = np.array([b, c], np.float32)
    return v0, v1, v2


def _rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


# ---------------------------------------------------------------------------
# configs
# ---------------------------------------------------------------------------

@dataclass
class Camera:
    position: tuple
    look_at: tuple
    up: tuple
    vertical_fov: float
    resolution: tuple


@dataclass
class SceneSpec:
    name: str
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    camera: Camera
    point_lights: list = field(default_factory=list)
    area_light: tuple | None = None   # (center xyz, half extent) of a y-facing quad
    spp: int = 8
    bounces: int = 1
    builder: str = "sah"
    precision: int = 6
    go_up: int = 0

    @property
    def n_tris(self):
        return self.v0.shape[0]


def _mesh_tris(v, f):
    v = v.astype(np.float32)
    return v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]


def make_scene(name: str, resolution=None, spp=None) -> SceneSpec:
    """Seeded scene for config ``name`` in {c1, c2, c3, c4, c5, tiny}."""
    if name in ("c1", "tiny"):
        v, f = displaced_icosphere(3, seed=1, amplitude=0.15)
        m0, m1, m2 = _mesh_tris(v, f)
        g0, g1, g2 = ground_quad(-1.2, 6.0)
        res = (256, 256) if name == "c1" else (32, 32)
        cam = Camera((0.0, 0.3, 3.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, res)
        sc = SceneSpec(name, np.concatenate([m0, g0]), np.concatenate([m1, g1]),
                       np.concatenate([m2, g2]), cam, point_lights=[(2.0, 4.0, 2.0)], spp=1,
                       bounces=1, builder="median")
    elif name == "c2":
        v, f = displaced_icosphere(6, seed=2, amplitude=0.15)
        f = trim_faces(f, 60_000, seed=2)
        m0, m1, m2 = _mesh_tris(v, f)
        g0, g1, g2 = ground_quad(-1.2, 6.0)
        cam = Camera((0.0, 0.3, 3.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, (1024, 1024))
        sc = SceneSpec(name, np.concatenate([m0, g0]), np.concatenate([m1, g1]),
                       np.concatenate([m2, g2]), cam, area_light=((0.0, 4.0, 0.0), 0.5),
                       spp=8, bounces=1)
    elif name == "c3":
        rng = np.random.default_rng(3)
        base_v, base_f = displaced_icosphere(5, seed=3, amplitude=0.15)
        parts = []
        for i in range(64):
            f = trim_faces(base_f, 7_812, seed=100 + i)
            R = _rotation(rng)
            s = rng.uniform(0.2, 0.8)
            pos = rng.uniform(-4.0, 4.0, 3)
            parts.append(_mesh_tris((base_v @ R.T) * s + pos, f))
        cam = Camera((0.0, 0.3, 12.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, (1024, 1024))
        sc = SceneSpec(name, *(np.concatenate([p[k] for p in parts]) for k in range(3)), cam,
                       point_lights=[(6.0, 8.0, 6.0), (-6.0, 8.0, 6.0), (6.0, 8.0, -6.0),
                                     (-6.0, 8.0, -6.0)], spp=8, bounces=2)
    elif name == "c4":
        v, f = displaced_icosphere(8, seed=4, amplitude=0.2, octaves=4, frequency=4.0)
        f = trim_faces(f, 1_000_000, seed=4)
        m0, m1, m2 = _mesh_tris(v, f)
        cam = Camera((0.0, 0.3, 3.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, (1024, 1024))
        sc = SceneSpec(name, m0, m1, m2, cam, point_lights=[(2.0, 4.0, 2.0)], spp=8, bounces=1)
    elif name == "c5":
        # 4096 seeded instances (64 x 64 grid, jittered, random rotation and
        # scale) of a 13k-triangle displaced mesh, flattened, plus a ground plane
        rng = np.random.default_rng(5)
        base_v, base_f = displaced_icosphere(5, seed=5, amplitude=0.2, octaves=2)
        base_f = trim_faces(base_f, 13_000, seed=5)
        bv = base_v.astype(np.float64)
        inst = []
        for i in range(4096):
            gx, gz = i % 64, i // 64
            R = _rotation(rng)
            sc_ = rng.uniform(0.3, 0.7)
            pos = np.array([(gx - 31.5) * 1.6 + rng.uniform(-0.3, 0.3), rng.uniform(0.0, 0.6),
                            (gz - 31.5) * 1.6 + rng.uniform(-0.3, 0.3)])
            inst.append(((bv @ R.T) * sc_ + pos).astype(np.float32))
        verts = np.stack(inst)  # (4096, V, 3)
        m0 = verts[:, base_f[:, 0]].reshape(-1, 3)
        m1 = verts[:, base_f[:, 1]].reshape(-1, 3)
        m2 = verts[:, base_f[:, 2]].reshape(-1, 3)
        g0, g1, g2 = ground_quad(-0.8, 60.0)
        cam = Camera((0.0, 14.0, 40.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, (1024, 1024))
        sc = SceneSpec(name, np.concatenate([m0, g0]), np.concatenate([m1, g1]),
                       np.concatenate([m2, g2]), cam, area_light=((0.0, 30.0, 0.0), 5.0),
                       spp=8, bounces=3)
    else:
        raise ValueError(f"unknown scene config {name!r}")
    if resolution is not None:
        sc.camera.resolution = tuple(resolution)
    if spp is not None:
        sc.spp = int(spp)
    return sc


# ---------------------------------------------------------------------------
# ray waves
# ---------------------------------------------------------------------------

def _stratum_grid(spp):
    sx = max(1, int(math.sqrt(spp)))
    while spp % sx:
        sx -= 1
    return sx, spp // sx


def primary_rays(cam: Camera, spp: int, seed: int = 0, jitter: bool = True):
    """hrpp/tracer.py:173-211 semantics: float32 (n,3) origins and unit dirs."""
    w, h = cam.resolution
    n = w * h * spp
    ray_idx = np.arange(n, dtype=np.uint64)
    pixel = ray_idx // np.uint64(spp)
    sample = ray_idx % np.uint64(spp)
    px = (pixel % np.uint64(w)).astype(np.float64)
    py = (pixel // np.uint64(w)).astype(np.float64)
    if jitter:
        sx, sy = _stratum_grid(spp)
        six = (sample % np.uint64(sx)).astype(np.float64)
        siy = (sample // np.uint64(sx)).astype(np.float64)
        offx = (six + unit_floats(seed, pixel, sample, 0)) / sx
        offy = (siy + unit_floats(seed, pixel, sample, 1)) / sy
    else:
        offx = np.full(n, 0.5)
        offy = np.full(n, 0.5)
    pos = np.asarray(cam.position, np.float32).astype(np.float64)
    fwd = np.asarray(cam.look_at, np.float32).astype(np.float64) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(cam.up, np.float32).astype(np.float64))
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    tan_half = math.tan(math.radians(cam.vertical_fov) / 2.0)
    aspect = w / h
    ndc_x = ((px + offx) / w) * 2.0 - 1.0
    ndc_y = 1.0 - ((py + offy) / h) * 2.0
    d = (fwd[None, :] + ndc_x[:, None] * (tan_half * aspect) * right[None, :]
         + ndc_y[:, None] * tan_half * up[None, :])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    origins = np.broadcast_to(np.asarray(cam.position, np.float32), (n, 3)).copy()
    return origins, d.astype(np.float32)


def slot_normals(tv0, tv1, tv2):
    e1 = tv1.astype(np.float64) - tv0.astype(np.float64)
    e2 = tv2.astype(np.float64) - tv0.astype(np.float64)
    nrm = np.cross(e1, e2)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return nrm


def hit_frames(O, D, found, t, slot, normals):
    """Hit points offset 1e-4 along the facing normal (hrpp/tracer.py:442-453)."""
    hit = np.asarray(found, bool)
    ho = O[hit].astype(np.float64)
    hd = D[hit].astype(np.float64)
    P = ho + np.asarray(t)[hit][:, None] * hd
    N = normals[np.asarray(slot)[hit]]
    facing = np.einsum("ij,ij->i", N, hd)
    N = np.where(facing[:, None] > 0.0, -N, N)
    return hit, P + 1e-4 * N, N


def shadow_rays(offset_P, light_points):
    """hrpp/tracer.py:456-464 for per-ray light sample points (n,3)."""
    lvec = np.asarray(light_points, np.float64) - offset_P
    dist = np.maximum(np.linalg.norm(lvec, axis=1), 1e-9)
    ldir = lvec / dist[:, None]
    stmax = np.maximum(dist - 1e-4, 1e-6)
    return offset_P.astype(np.float32), ldir.astype(np.float32), np.zeros(len(stmax)), stmax


def area_light_samples(n, center, half, seed, dim0=10):
    idx = np.arange(n, dtype=np.uint64)
    u = unit_floats(seed, idx, np.zeros(n, np.uint64), dim0)
    v = unit_floats(seed, idx, np.zeros(n, np.uint64), dim0 + 1)
    c = np.asarray(center, np.float64)
    return np.stack([c[0] + (2 * u - 1) * half, np.full(n, c[1]), c[2] + (2 * v - 1) * half], 1)


# Taylor coefficients of sin and cos on [0, pi/2] (truncation error < 5e-14)
_SIN_C = (-1.0 / 6, 1.0 / 120, -1.0 / 5040, 1.0 / 362880, -1.0 / 39916800, 1.0 / 6227020800,
          -1.0 / 1307674368000, 1.0 / 355687428096000)
_COS_C = (-1.0 / 2, 1.0 / 24, -1.0 / 720, 1.0 / 40320, -1.0 / 3628800, 1.0 / 479001600,
          -1.0 / 87178291200, 1.0 / 20922789888000)
_HALF_PI = 1.5707963267948966


def cos_sin_turn(u):
    """(cos, sin) of 2 pi u for u in [0, 1): quarter-turn reduction and
    Horner polynomials in plain float64 operations, so the device spawn
    (csrc/k_spawn.cu, built without FMA) reproduces it bit for bit."""
    x = 4.0 * np.asarray(u, np.float64)
    q = np.floor(x)
    t = (x - q) * _HALF_PI
    t2 = t * t
    s = _SIN_C[-1]
    for k in _SIN_C[-2::-1]:
        s = k + t2 * s
    s = t * (1.0 + t2 * s)
    c = _COS_C[-1]
    for k in _COS_C[-2::-1]:
        c = k + t2 * c
    c = 1.0 + t2 * c
    qi = q.astype(np.int64) & 3
    cos = np.select([qi == 0, qi == 1, qi == 2], [c, -s, -c], s)
    sin = np.select([qi == 0, qi == 1, qi == 2], [s, c, -s], -c)
    return cos, sin


def cosine_bounce(offset_P, N, seed, dim0=20):
    n = offset_P.shape[0]
    idx = np.arange(n, dtype=np.uint64)
    u1 = unit_floats(seed, idx, np.zeros(n, np.uint64), dim0)
    u2 = unit_floats(seed, idx, np.zeros(n, np.uint64), dim0 + 1)
    r = np.sqrt(u1)
    cphi, sphi = cos_sin_turn(u2)
    lx, ly, lz = r * cphi, r * sphi, np.sqrt(np.maximum(0.0, 1.0 - u1))
    a = np.where(np.abs(N[:, 0:1]) > 0.9, np.array([[0.0, 1.0, 0.0]]), np.array([[1.0, 0, 0]]))
    tx = np.cross(N, a)
    tx /= np.linalg.norm(tx, axis=1, keepdims=True)
    ty = np.cross(N, tx)
    d = lx[:, None] * tx + ly[:, None] * ty + lz[:, None] * N
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return (offset_P.astype(np.float32), d.astype(np.float32), np.zeros(n),
            np.full(n, np.inf))
