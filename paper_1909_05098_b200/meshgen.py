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


def voxel_ellipsoid_mesh(dims=(512, 384, 320), h: float = 0.3 / 512, semi=(0.15, 0.10, 0.08),
                         split_fraction: float = 0.1, seed: int = 5):
    """Config-5 mesh: voxels of a (nx, ny, nz) grid of spacing h whose centre
    lies inside the ellipsoid (semi-axes ``semi``, centred in the grid) become
    hex8 elements; a seeded ``split_fraction`` of the boundary voxels (active
    voxels with an inactive face neighbour) are split into 6 Kuhn tets.
    Node set ``surface``: nodes on faces shared with an inactive voxel.
    Returns (mesh, centre)."""
    nx, ny, nz = (int(d) for d in dims)
    centre = np.array([nx * h / 2.0, ny * h / 2.0, nz * h / 2.0])
    xs = (((np.arange(nx) + 0.5) * h - centre[0]) / semi[0]) ** 2
    ys = (((np.arange(ny) + 0.5) * h - centre[1]) / semi[1]) ** 2
    zs = (((np.arange(nz) + 0.5) * h - centre[2]) / semi[2]) ** 2
    active = (zs[:, None, None] + ys[None, :, None] + xs[None, None, :]) <= 1.0  # [k, j, i]
    pad = np.pad(active, 1)
    exposed = []  # per direction: active cells whose neighbour is inactive
    for axis in range(3):
        for step in (-1, 1):
            nb = np.roll(pad, -step, axis=axis)[1:-1, 1:-1, 1:-1]
            exposed.append(active & ~nb)
    boundary = np.logical_or.reduce(exposed)
    kb, jb, ib = np.nonzero(boundary)
    rng = np.random.default_rng(seed)
    n_split = int(round(split_fraction * kb.size))
    pick = np.sort(rng.choice(kb.size, size=n_split, replace=False))
    split = np.zeros_like(active)
    split[kb[pick], jb[pick], ib[pick]] = True
    # grid points used by active voxels -> compact node ids (x fastest)
    gx, gy = nx + 1, ny + 1
    used = np.zeros((nz + 1, ny + 1, nx + 1), dtype=bool)
    for dk in (0, 1):
        for dj in (0, 1):
            for di in (0, 1):
                used[dk:dk + nz, dj:dj + ny, di:di + nx] |= active
    flat_used = used.ravel()
    node_id = np.cumsum(flat_used, dtype=np.int64) - 1
    gidx = np.nonzero(flat_used)[0]
    k_, rem = np.divmod(gidx, gx * gy)
    j_, i_ = np.divmod(rem, gx)
    nodes = np.stack([i_ * h, j_ * h, k_ * h], axis=1).astype(np.float64)
    stride = np.array([1, gx, gx * gy], dtype=np.int64)

    def cells(mask):
        k, j, i = np.nonzero(mask)
        return i + gx * (j + gy * k)

    hex_base = cells(active & ~split)
    hexes = node_id[hex_base[:, None] + (HEX_CORNER_OFFSETS @ stride)[None]]
    tet_base = cells(split)
    tets = node_id[(tet_base[:, None, None] + (KUHN_PATTERNS @ stride)[None])].reshape(-1, 4)
    surf = np.zeros(flat_used.size, dtype=bool)
    faces = {(0, -1): [0, 3, 4, 7], (0, 1): [1, 2, 5, 6], (1, -1): [0, 1, 4, 5], (1, 1): [2, 3, 6, 7],
             (2, -1): [0, 1, 2, 3], (2, 1): [4, 5, 6, 7]}
    q = 0
    for axis in range(3):
        for step in (-1, 1):
            base = cells(exposed[q])
            q += 1
            axis_map = {0: 2, 1: 1, 2: 0}  # exposed[] axes are (k, j, i) -> (z, y, x)
            corners = faces[(axis_map[axis], step)]
            for c in corners:
                surf[base + HEX_CORNER_OFFSETS[c] @ stride] = True
    sets = {"surface": node_id[np.nonzero(surf)[0]]}
    return Mesh(nodes=nodes, tets=tets, hexes=hexes, node_sets=sets), centre


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
