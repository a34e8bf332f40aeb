"""Ray/hit value types of the reference API (hrpp/geom.py:71-169).

Only the types the hot-path API exchanges are provided: ``RayKind``,
``Ray`` (float32 origin/direction whose bits feed the hash, unit direction
within 1e-4, t_min >= 0, t_max > t_min), ``HitRecord``, ``Triangle`` and
``vec3``.  The reference's pure-Python intersection predicates
(``ray_aabb_intersect``, ``ray_triangle_intersect``) are the semantic spec
that the CUDA kernels restate; they are not a product path here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import NonFiniteInput

DET_EPS = 1e-9
DEGENERATE_AREA_EPS = 1e-12
DIRECTION_NORM_TOL = 1e-4


class RayKind(Enum):
    HIT_ANY = "hit_any"
    CLOSEST_HIT = "closest_hit"


def vec3(x, y, z) -> np.ndarray:
    v = np.array([x, y, z], dtype=np.float32)
    if not np.all(np.isfinite(v)):
        raise NonFiniteInput(f"non-finite vector component in ({x}, {y}, {z})")
    return v


def _as_vec3(v) -> np.ndarray:
    a = np.asarray(v, dtype=np.float32)
    if a.shape != (3,):
        raise ValueError(f"expected a 3-vector, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise NonFiniteInput("non-finite vector component")
    return a


@dataclass(frozen=True)
class Ray:
    origin: np.ndarray
    direction: np.ndarray
    t_min: float = 0.0
    t_max: float = math.inf
    kind: RayKind = RayKind.CLOSEST_HIT

    def __post_init__(self):
        object.__setattr__(self, "origin", _as_vec3(self.origin))
        object.__setattr__(self, "direction", _as_vec3(self.direction))
        n = float(np.linalg.norm(self.direction.astype(np.float64)))
        if abs(n - 1.0) > DIRECTION_NORM_TOL:
            raise ValueError(f"direction must be unit length, |d| = {n}")
        if self.t_min < 0.0:
            raise ValueError("t_min must be >= 0")
        if not self.t_max > self.t_min:
            raise ValueError("t_max must be > t_min")


@dataclass(frozen=True)
class Triangle:
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    id: int = 0

    def __post_init__(self):
        object.__setattr__(self, "v0", _as_vec3(self.v0))
        object.__setattr__(self, "v1", _as_vec3(self.v1))
        object.__setattr__(self, "v2", _as_vec3(self.v2))


@dataclass
class HitRecord:
    t: float
    triangle_id: int
    leaf_node: int = -1
    u: float = 0.0
    v: float = 0.0
