"""Oracle: DPP parameters, manufactured solutions, boundary specification.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference problem.py:26-45 (parameters and validation), :78-83 (eta),
:100-144 (2D / 3D closed-form fields, paper Eq. 44 / 46 with the k2 micro
scale), :160-172 (constant patch fields) and :176-215 (boundary partition).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np


@dataclass(frozen=True)
class Params:
    mu: float = 1.0
    beta: float = 1.0
    k1: float = 1.0
    k2: float = 0.1
    eta_u: float = 10.0
    eta_p: float = 10.0
    gamma_b: tuple = (0.0, 0.0)
    L: float = 1.0

    def __post_init__(self):
        if self.mu <= 0 or self.k1 <= 0 or self.k2 <= 0:
            raise ValueError("mu, k1, k2 must be positive")
        if self.beta < 0:
            raise ValueError("beta must be nonnegative")
        if self.eta_u < 0 or self.eta_p < 0:
            raise ValueError("penalty numbers must be nonnegative")


def paper_2d_parameters():
    return Params(gamma_b=(0.0, 0.0))


def paper_3d_parameters():
    return Params(gamma_b=(0.0, 0.0, 0.0))


def eta(p: Params) -> float:
    return math.sqrt(p.beta * (p.k1 + p.k2) / (p.k1 * p.k2))


@dataclass(frozen=True)
class Fields:
    dim: int
    u1: Callable
    p1: Callable
    u2: Callable
    p2: Callable

    def field(self, name):
        return getattr(self, name)


def _exact(pts, p: Params, scale="k2"):
    pts = np.asarray(pts, dtype=float)
    et = eta(p)
    x = pts[..., 0]
    ex = np.exp(np.pi * x)
    if pts.shape[-1] == 2:
        y = pts[..., 1]
        s, c, ey = np.sin(np.pi * y), np.cos(np.pi * y), np.exp(et * y)
        u1 = -p.k1 * np.stack([ex * s, ex * c - et / (p.beta * p.k1) * ey], axis=-1)
        p1 = p.mu / np.pi * ex * s - p.mu / (p.beta * p.k1) * ey
        u2 = -p.k2 * np.stack([ex * s, ex * c + et / (p.beta * p.k2) * ey], axis=-1)
        p2 = p.mu / np.pi * ex * s + p.mu / (p.beta * p.k2) * ey
        return u1, p1, u2, p2
    y, z = pts[..., 1], pts[..., 2]
    sy, cy, sz, cz = np.sin(np.pi * y), np.cos(np.pi * y), np.sin(np.pi * z), np.cos(np.pi * z)
    ey, ez = np.exp(et * y), np.exp(et * z)
    u1 = -p.k1 * np.stack([ex * (sy + sz), ex * cy - et / (p.beta * p.k1) * ey,
                           ex * cz - et / (p.beta * p.k1) * ez], axis=-1)
    p1 = p.mu / np.pi * ex * (sy + sz) - p.mu / (p.beta * p.k1) * (ey + ez)
    u2 = -p.k2 * np.stack([ex * (sy + sz), ex * cy + et / (p.beta * p.k2) * ey,
                           ex * cz + et / (p.beta * p.k2) * ez], axis=-1)
    kp = p.k2 if scale == "k2" else p.k1
    p2 = p.mu / np.pi * ex * (sy + sz) + p.mu / (p.beta * kp) * (ey + ez)
    return u1, p1, u2, p2


def mms(dim: int, p: Params) -> Fields:
    def pick(i):
        return lambda pts: _exact(pts, p)[i]
    return Fields(dim, pick(0), pick(1), pick(2), pick(3))


def constant_mms(dim: int, value: float) -> Fields:
    def zu(pts):
        pts = np.asarray(pts)
        return np.zeros(pts.shape[:-1] + (dim,))

    def cp(pts):
        pts = np.asarray(pts)
        return np.full(pts.shape[:-1], float(value))
    return Fields(dim, zu, cp, zu, cp)


@dataclass(frozen=True)
class BoundarySpec:
    p_data: tuple
    un_data: tuple | None = None
    velocity_facets: tuple = (frozenset(), frozenset())

    def is_velocity_facet(self, net, f):
        return f in self.velocity_facets[net - 1]


def boundary_data(fields: Fields, mesh, velocity_facets=(frozenset(), frozenset())):
    if fields.dim != mesh.dim:
        raise ValueError("dimension mismatch")

    def flux(fn):
        return lambda pts, normal: fn(pts) @ normal
    return BoundarySpec((fields.p1, fields.p2), (flux(fields.u1), flux(fields.u2)),
                        (frozenset(velocity_facets[0]), frozenset(velocity_facets[1])))
