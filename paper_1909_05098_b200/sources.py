"""Volumetric heat sources and convective (Robin) boundaries.

Extensions required by BASELINE.json configs 1-5 that the reference lacks
(parity unpinned except where a source is static and is fed
identically to the oracle).  Lumping follows the reference's metabolic term
(precompute.py:47): a volumetric density Q(x) becomes the nodal power
Q(x_i) * v_i.

* `GaussianSource`: Q = amp * exp(-|x - c(t)|^2 / (2 sigma^2)), c(t) = x0 + vel * t,
  active while t0 <= t < t1 (t = step start time, like heat_loads).
* `RFSource`: Q = min(P / (4 pi r^2), cap), r = |x - tip| (cap at r = 0).
* `RobinSpec`: h (W/m^2/K) and T_inf on a node set; the face areas of the
  boundary faces lying in the set are lumped equally to their corners, and a
  node i gets rate += hA_i T_inf - hA_i T_i.  Dirichlet wins on shared nodes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError


@dataclass(frozen=True)
class GaussianSource:
    amp: float
    sigma: float
    x0: tuple = (0.0, 0.0, 0.0)
    vel: tuple = (0.0, 0.0, 0.0)
    t0: float = -math.inf
    t1: float = math.inf

    @property
    def is_static(self) -> bool:
        return all(v == 0.0 for v in self.vel) and self.t0 == -math.inf and self.t1 == math.inf

    def density(self, xyz, t=0.0):
        c = np.asarray(self.x0, float) + np.asarray(self.vel, float) * t
        d = np.asarray(xyz, float) - c
        r2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        return self.amp * np.exp(-r2 / (2.0 * self.sigma * self.sigma))

    def as_dict(self):
        return {"kind": "gauss", "amp": self.amp, "sigma": self.sigma, "cap": math.inf, "x0": self.x0,
                "vel": self.vel, "t0": self.t0, "t1": self.t1}


@dataclass(frozen=True)
class RFSource:
    power: float
    tip: tuple
    cap: float = 1.0e8
    t0: float = -math.inf
    t1: float = math.inf

    @property
    def is_static(self) -> bool:
        return self.t0 == -math.inf and self.t1 == math.inf

    def density(self, xyz, t=0.0):
        d = np.asarray(xyz, float) - np.asarray(self.tip, float)
        r2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        with np.errstate(divide="ignore"):
            q = np.where(r2 > 0.0, self.power / (4.0 * math.pi * r2), self.cap)
        return np.minimum(q, self.cap)

    def as_dict(self):
        return {"kind": "rf", "amp": self.power, "sigma": 1.0, "cap": self.cap, "x0": self.tip,
                "vel": (0.0, 0.0, 0.0), "t0": self.t0, "t1": self.t1}


@dataclass(frozen=True)
class RobinSpec:
    nodeset: str
    h: float
    t_inf: float


def static_nodal_power(sources, nodes, node_volumes) -> np.ndarray | None:
    """Sum of the static sources lumped as Q(x_i) * v_i (W per node)."""
    q = None
    for s in sources:
        if not s.is_static:
            continue
        term = s.density(nodes) * node_volumes
        q = term if q is None else q + term
    return q


def _boundary_faces(mesh, members):
    """Faces with every corner in ``members`` that belong to exactly one element.

    Only faces inside the node set can be its boundary faces, so the
    multiplicity count runs on that (small) subset."""
    tet_faces = np.array([[0, 1, 2], [0, 1, 3], [0, 2, 3], [1, 2, 3]])
    hex_faces = np.array([[0, 1, 2, 3], [4, 5, 6, 7], [0, 1, 5, 4], [1, 2, 6, 5], [2, 3, 7, 6], [3, 0, 4, 7]])
    out = []
    for conn, faces in ((mesh.tets, tet_faces), (mesh.hexes, hex_faces)):
        if conn.size == 0:
            continue
        cand = conn[members[conn].sum(axis=1) >= faces.shape[1]]
        f = cand[:, faces].reshape(-1, faces.shape[1])
        f = f[members[f].all(axis=1)]
        if f.size == 0:
            continue
        key = np.sort(f, axis=1)
        _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
        out.append(f[cnt[inv.ravel()] == 1])
    return out


def robin_lumps(mesh, spec: RobinSpec, exclude=None):
    """(nodes, hA, hA*T_inf) for a Robin condition on node set ``spec.nodeset``.

    Boundary faces whose corners all lie in the set contribute area/n_corners
    to each corner (triangles: exact area; quads: sum of the two triangles of
    the 0-2 diagonal).  Nodes in ``exclude`` (Dirichlet) are dropped.
    """
    if spec.nodeset not in mesh.node_sets:
        raise ConfigError(f"mesh has no node set {spec.nodeset!r}")
    members = np.zeros(mesh.n_nodes, bool)
    members[mesh.node_sets[spec.nodeset]] = True
    area = np.zeros(mesh.n_nodes)
    for faces in _boundary_faces(mesh, members):
        p = mesh.nodes[faces]
        if faces.shape[1] == 3:
            a = 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)
        else:
            a = 0.5 * (np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)
                       + np.linalg.norm(np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]), axis=1))
        np.add.at(area, faces.ravel(), np.repeat(a / faces.shape[1], faces.shape[1]))
    nodes = np.nonzero(area > 0.0)[0]
    if exclude is not None and len(exclude):
        nodes = np.setdiff1d(nodes, np.asarray(exclude, np.int64))
    hA = spec.h * area[nodes]
    return nodes.astype(np.int64), hA, hA * spec.t_inf
