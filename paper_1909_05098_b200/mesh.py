"""Unstructured tet4/hex8 mesh with named node sets.

Data model of /root/reference/pkg/src/fedheat/mesh.py:38-150: a frozen
container of read-only arrays (nodes float64 (V,3); tets int64 (Et,4); hexes
int64 (Eh,8); node sets as sorted unique int64 arrays).  The global element
order is all tets, then all hexes.  Construction validates index ranges,
repeated nodes, positive orientation and node-set names.

Validation runs in blocks of `_BLOCK` elements so 25 M-element meshes do not
need tens of GB of numpy temporaries.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np

from .element import ElemKind, HEX_VERTEX_SIGNS, _cofactor_inverse, _seq_matmul
from .errors import DegenerateElementError, MeshFormatError

_NAME_RE = re.compile(r"^[A-Za-z_][A-Za-z0-9_.-]*$")
_BLOCK = 1 << 20


def _det_tet(p):
    edges = p[:, 1:, :] - p[:, :1, :]
    return _cofactor_inverse(np.swapaxes(edges, -1, -2))[1]


def _det_hex(p):
    jac = _seq_matmul(np.swapaxes(p, -1, -2), HEX_VERTEX_SIGNS / 8.0)
    return _cofactor_inverse(jac)[1]


@dataclass(frozen=True)
class Mesh:
    nodes: np.ndarray
    tets: np.ndarray
    hexes: np.ndarray
    node_sets: dict = field(default_factory=dict)

    def __post_init__(self):
        nodes = np.ascontiguousarray(np.asarray(self.nodes, dtype=np.float64))
        tets = np.ascontiguousarray(np.asarray(self.tets, dtype=np.int64).reshape(-1, 4))
        hexes = np.ascontiguousarray(np.asarray(self.hexes, dtype=np.int64).reshape(-1, 8))
        sets = {str(k): np.unique(np.asarray(v, dtype=np.int64)) for k, v in self.node_sets.items()}
        for arr in (nodes, tets, hexes, *sets.values()):
            arr.setflags(write=False)
        object.__setattr__(self, "nodes", nodes)
        object.__setattr__(self, "tets", tets)
        object.__setattr__(self, "hexes", hexes)
        object.__setattr__(self, "node_sets", sets)
        self.validate()

    @property
    def n_nodes(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def n_elements(self) -> int:
        return int(self.tets.shape[0] + self.hexes.shape[0])

    def iter_elements(self) -> Iterator[tuple[ElemKind, np.ndarray]]:
        for row in self.tets:
            yield ElemKind.TET4, row
        for row in self.hexes:
            yield ElemKind.HEX8, row

    def element(self, index: int):
        nt = self.tets.shape[0]
        if 0 <= index < nt:
            return ElemKind.TET4, self.tets[index]
        if nt <= index < self.n_elements:
            return ElemKind.HEX8, self.hexes[index - nt]
        raise IndexError(f"element index {index} out of range [0, {self.n_elements})")

    def validate(self) -> None:
        if self.nodes.ndim != 2 or self.nodes.shape[1] != 3:
            raise MeshFormatError(f"nodes must be (n, 3), got {self.nodes.shape}")
        if self.n_nodes == 0:
            raise MeshFormatError("mesh has no nodes")
        finite = np.isfinite(self.nodes).all(axis=1)
        if not finite.all():
            raise MeshFormatError(f"node {int(np.argmin(finite))} has non-finite coordinates")
        if self.n_elements == 0:
            raise MeshFormatError("mesh has no elements")
        for kind, conn, offset, det_fn in (
            (ElemKind.TET4, self.tets, 0, _det_tet),
            (ElemKind.HEX8, self.hexes, self.tets.shape[0], _det_hex),
        ):
            if conn.size == 0:
                continue
            bad_idx = (conn < 0) | (conn >= self.n_nodes)
            if bad_idx.any():
                e = int(np.argmax(bad_idx.any(axis=1)))
                raise MeshFormatError(
                    f"element {offset + e} references a node outside [0, {self.n_nodes})")
            srt = np.sort(conn, axis=1)
            dup = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
            if dup.any():
                raise MeshFormatError(f"element {offset + int(np.argmax(dup))} repeats a node")
            for lo in range(0, conn.shape[0], _BLOCK):
                det = det_fn(self.nodes[conn[lo:lo + _BLOCK]])
                bad = det <= 0.0
                if bad.any():
                    e = int(np.argmax(bad))
                    what = ("tet has non-positive volume (6V" if kind is ElemKind.TET4
                            else "hex has non-positive Jacobian (det J")
                    raise DegenerateElementError(f"{what} = {det[e]:.6g})", element=offset + lo + e)
        for name, ids in self.node_sets.items():
            if not _NAME_RE.match(name):
                raise MeshFormatError(f"invalid node-set name {name!r}")
            if ids.size and (ids[0] < 0 or ids[-1] >= self.n_nodes):
                raise MeshFormatError(
                    f"node set {name!r} references a node outside [0, {self.n_nodes})")


def element_volume_shares(mesh: Mesh):
    """(node index, share) pairs: each element gives V_e / n_e to each corner."""
    idx, val = [], []
    if mesh.tets.size:
        vol = np.concatenate([_det_tet(mesh.nodes[mesh.tets[lo:lo + _BLOCK]]) / 6.0
                              for lo in range(0, mesh.tets.shape[0], _BLOCK)])
        idx.append(mesh.tets.ravel())
        val.append(np.repeat(vol / 4.0, 4))
    if mesh.hexes.size:
        det = np.concatenate([_det_hex(mesh.nodes[mesh.hexes[lo:lo + _BLOCK]])
                              for lo in range(0, mesh.hexes.shape[0], _BLOCK)])
        idx.append(mesh.hexes.ravel())
        val.append(np.repeat(8.0 * det / 8.0, 8))
    return np.concatenate(idx), np.concatenate(val)


def node_volume_shares(mesh: Mesh) -> np.ndarray:
    """Lumped nodal volume v_i = sum of V_e/n_e over elements touching i.

    Order independent (reference mesh.py:128-150): each node's shares are
    added from 0.0 in ascending value order, so any element permutation gives
    the same bits.  The device precompute reproduces this exact order.
    """
    idx, val = element_volume_shares(mesh)
    order = np.lexsort((val, idx))
    out = np.zeros(mesh.n_nodes)
    np.add.at(out, idx[order], val[order])
    return out
