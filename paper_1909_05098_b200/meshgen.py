"""Deterministic synthetic meshes.

`generate_cube_mesh` reproduces /root/reference/pkg/src/fedheat/meshgen.py:59-116
bit for bit (node coordinates, connectivity and node sets): nodes x-fastest,
cells z-fastest, six Kuhn tets per cell (one per axis permutation, odd
permutations with their middle vertices swapped so every tet is positively
oriented), all tets of a cell adjacent in element order; node sets x0..z1 and
``center`` (the node nearest the centroid, lowest index on ties).

The BASELINE.json generators that the reference lacks are
builder-defined and seeded: `jittered_cube_mesh` (config 3) and
`voxel_ellipsoid_mesh` (config 5).
"""

from __future__ import annotations

from itertools import permutations

import numpy as np

from .element import ElemKind
from .errors import ConfigError
from .mesh import Mesh


def _kuhn_patterns() -> np.ndarray:
    pats = []
    for perm in permutations(range(3)):
        corners = [np.zeros(3, dtype=np.int64)]
        for ax in perm:
            step = corners[-1].copy()
            step[ax] += 1
            corners.append(step)
        parity = sum(1 for a in range(3) for b in range(a + 1, 3) if perm[a] > perm[b]) % 2
        if parity:
            corners[1], corners[2] = corners[2], corners[1]
        pats.append(np.stack(corners))
    return np.stack(pats)  # (6, 4, 3)


KUHN_PATTERNS = _kuhn_patterns()
HEX_CORNER_OFFSETS = np.array(
    [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]],
    dtype=np.int64)


def _kind(kind) -> ElemKind:
    if isinstance(kind, ElemKind):
        return kind
    aliases = {"tet": ElemKind.TET4, "tet4": ElemKind.TET4, "hex": ElemKind.HEX8, "hex8": ElemKind.HEX8}
    if kind not in aliases:
        raise ConfigError(f"unknown element kind {kind!r} (use 'tet' or 'hex')")
    return aliases[kind]


def cube_arrays(kind, divisions: int, size: float):
    """Raw arrays of the structured cube: (nodes, tets, hexes, node_sets)."""
    kind = _kind(kind)
    div = int(divisions)
    if div < 1:
        raise ConfigError(f"divisions must be >= 1, got {divisions}")
    size = float(size)
    if not (size > 0.0 and np.isfinite(size)):
        raise ConfigError(f"size must be positive and finite, got {size}")
    n = div + 1
    ticks = np.linspace(0.0, size, n)
    gz, gy, gx = np.meshgrid(ticks, ticks, ticks, indexing="ij")
    nodes = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)

    # cell (i, j, k) with k fastest; node id = i + n*(j + n*k)
    cell = np.arange(div, dtype=np.int64)
    ci = np.repeat(cell, div * div)
    cj = np.tile(np.repeat(cell, div), div)
    ck = np.tile(cell, div * div)
    base = ci + n * (cj + n * ck)
    stride = np.array([1, n, n * n], dtype=np.int64)

    tets = np.empty((0, 4), dtype=np.int64)
    hexes = np.empty((0, 8), dtype=np.int64)
    if kind is ElemKind.TET4:
        offs = KUHN_PATTERNS @ stride  # (6, 4)
        tets = (base[:, None, None] + offs[None]).reshape(-1, 4)
    else:
        hexes = base[:, None] + (HEX_CORNER_OFFSETS @ stride)[None]

    ids = np.arange(n ** 3, dtype=np.int64).reshape(n, n, n)  # [k, j, i]
    sets = {
        "x0": ids[:, :, 0].ravel(), "x1": ids[:, :, -1].ravel(),
        "y0": ids[:, 0, :].ravel(), "y1": ids[:, -1, :].ravel(),
        "z0": ids[0, :, :].ravel(), "z1": ids[-1, :, :].ravel(),
    }
    d2 = ((nodes - size / 2.0) ** 2).sum(axis=1)
    sets["center"] = np.array([int(np.argmin(d2))], dtype=np.int64)
    return nodes, tets, hexes, sets


def generate_cube_mesh(kind, divisions: int, size: float) -> Mesh:
    nodes, tets, hexes, sets = cube_arrays(kind, divisions, size)
    return Mesh(nodes=nodes, tets=tets, hexes=hexes, node_sets=sets)


def jittered_cube_mesh(kind, divisions: int, size: float, jitter: float = 0.2,
                       seed: int = 0) -> Mesh:
    """Config-3 mesh: cube numbering, interior nodes moved by U(-jitter*h, +jitter*h)
    per axis (seeded ``np.random.default_rng(seed)``), boundary nodes fixed so
    the face node sets stay planar."""
    nodes, tets, hexes, sets = cube_arrays(kind, divisions, size)
    h = float(size) / int(divisions)
    rng = np.random.default_rng(seed)
    delta = rng.uniform(-jitter, jitter, nodes.shape) * h
    on_face = np.zeros(nodes.shape[0], dtype=bool)
    for name in ("x0", "x1", "y0", "y1", "z0", "z1"):
        on_face[sets[name]] = True
    delta[on_face] = 0.0
    return Mesh(nodes=nodes + delta, tets=tets, hexes=hexes, node_sets=sets)
