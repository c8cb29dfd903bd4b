"""Element geometry for tet4 / hex8 (host-side API helpers).

Behaviour follows /root/reference/pkg/src/fedheat/element.py:99-184: a tet4
has constant shape gradients and ``A = V * B^T B``; a hex8 uses one-point
integration at the reference-cube centre, ``A = 8 det(J) * B^T B`` and the
stored "volume" is ``8 det(J)``.  Every element's conduction operator is
``kbar_e * A_e``.

These numpy helpers are the *API surface* of the reference (``tet_geometry``,
``build_precomp``...).  The engine never calls them on its step path: the
device precompute (csrc/fh_precompute.cu) recomputes the same quantities on
the GPU in the same floating-point operation order (sequential sums, no FMA),
which is what makes the exact mode bitwise equal to the reference.

The factorisation the fast path relies on: with D the
(n_nodes x 3) matrix of reference-space gradients, ``B = J^-T D^T`` so
``A = D G D^T`` with the symmetric 3x3 ``G = w J^-1 J^-T`` -- six numbers per
element instead of n_nodes^2.  `metric_tensor` returns G.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import DegenerateElementError


class ElemKind(Enum):
    TET4 = "tet4"
    HEX8 = "hex8"

    @property
    def n_nodes(self) -> int:
        return 8 if self is ElemKind.HEX8 else 4


# (xi, eta, zeta) signs of the 8 hex corners: bottom face counter-clockwise
# seen from +z, then the top face in the same order.
HEX_VERTEX_SIGNS = np.array(
    [[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
     [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)
HEX_VERTEX_SIGNS.setflags(write=False)

# reference-space gradients of the tet4 shape functions (rows = nodes)
TET_REF_GRADS = np.array([[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
TET_REF_GRADS.setflags(write=False)


@dataclass(frozen=True)
class ElementPrecomp:
    kind: ElemKind
    node_ids: np.ndarray
    unit_conductance: np.ndarray
    volume: float


def _cofactor_inverse(m):
    """Inverse and determinant of stacked 3x3 matrices via cofactors.

    Operation order matches the reference's ``_inv3`` (element.py:69-96):
    minors as two products and a difference, det = (a*C00 + b*C01) + c*C02,
    then every cofactor divided by det.
    """
    a, b, c = m[..., 0, 0], m[..., 0, 1], m[..., 0, 2]
    d, e, f = m[..., 1, 0], m[..., 1, 1], m[..., 1, 2]
    g, h, i = m[..., 2, 0], m[..., 2, 1], m[..., 2, 2]
    c00 = e * i - f * h
    c01 = f * g - d * i
    c02 = d * h - e * g
    det = a * c00 + b * c01 + c * c02
    adj = np.stack([
        np.stack([c00, c * h - b * i, b * f - c * e], axis=-1),
        np.stack([c01, a * i - c * g, c * d - a * f], axis=-1),
        np.stack([c02, b * g - a * h, a * e - b * d], axis=-1),
    ], axis=-2)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = adj / det[..., None, None]
    return inv, det


def _seq_matmul(x, y):
    """(..., n, k) @ (k, m) with a strictly sequential k-sum (no BLAS)."""
    out = np.zeros(x.shape[:-1] + (y.shape[1],))
    for col in range(y.shape[1]):
        acc = np.zeros(x.shape[:-1])
        for kk in range(x.shape[-1]):
            acc = acc + x[..., kk] * y[kk, col]
        out[..., col] = acc
    return out


def batch_tet_geometry(coords):
    """(E,4,3) corners -> (B (E,3,4), volume (E,)); raises on volume <= 0."""
    p = np.asarray(coords, dtype=np.float64)
    edges = p[..., 1:, :] - p[..., :1, :]
    inv, det = _cofactor_inverse(np.swapaxes(edges, -1, -2))
    if (det <= 0.0).any():
        bad = int(np.argmax(det <= 0.0))
        raise DegenerateElementError(
            f"tet has non-positive volume (6V = {det.ravel()[bad]:.6g})", element=bad)
    grads = np.empty(p.shape[:-2] + (3, 4))
    grads[..., 1:] = np.swapaxes(inv, -1, -2)
    grads[..., 0] = -(grads[..., 1] + grads[..., 2] + grads[..., 3])
    return grads, det / 6.0


def batch_hex_geometry(coords):
    """(E,8,3) corners -> (B (E,3,8) at the centre, det J (E,)); raises on det <= 0."""
    p = np.asarray(coords, dtype=np.float64)
    dn = HEX_VERTEX_SIGNS / 8.0
    jac = _seq_matmul(np.swapaxes(p, -1, -2), dn)
    inv, det = _cofactor_inverse(jac)
    if (det <= 0.0).any():
        bad = int(np.argmax(det <= 0.0))
        raise DegenerateElementError(
            f"hex has non-positive Jacobian (det J = {det.ravel()[bad]:.6g})", element=bad)
    grads = _seq_matmul(np.swapaxes(inv, -1, -2), dn.T)
    return grads, det


def tet_geometry(coords):
    b, vol = batch_tet_geometry(np.asarray(coords, dtype=np.float64)[None])
    return b[0], float(vol[0])


def hex_geometry(coords):
    b, det = batch_hex_geometry(np.asarray(coords, dtype=np.float64)[None])
    return b[0], float(det[0])


def _gram(grads, weight):
    n = grads.shape[-1]
    a = np.empty(grads.shape[:-2] + (n, n))
    for r in range(n):
        for s in range(n):
            a[..., r, s] = (grads[..., 0, r] * grads[..., 0, s]
                            + grads[..., 1, r] * grads[..., 1, s]) + grads[..., 2, r] * grads[..., 2, s]
    return a * weight[..., None, None]


def batch_precompute(kind: ElemKind, coords):
    """(A (E,n,n), volume (E,)) for one element kind; A exactly symmetric."""
    if kind is ElemKind.TET4:
        b, vol = batch_tet_geometry(coords)
        return _gram(b, vol), vol
    b, det = batch_hex_geometry(coords)
    w = 8.0 * det
    return _gram(b, w), w


def metric_tensor(kind: ElemKind, coords):
    """G = w J^-1 J^-T (E,3,3), so that A = D G D^T (D = reference gradients)."""
    p = np.asarray(coords, dtype=np.float64)
    if kind is ElemKind.TET4:
        jac = np.swapaxes(p[..., 1:, :] - p[..., :1, :], -1, -2)
        inv, det = _cofactor_inverse(jac)
        w = det / 6.0
    else:
        jac = _seq_matmul(np.swapaxes(p, -1, -2), HEX_VERTEX_SIGNS / 8.0)
        inv, det = _cofactor_inverse(jac)
        w = 8.0 * det
    return np.einsum("...ik,...jk->...ij", inv, inv) * w[..., None, None]


def build_precomp(kind: ElemKind, node_ids, coords) -> ElementPrecomp:
    ids = np.asarray(node_ids, dtype=np.int64)
    if ids.shape != (kind.n_nodes,):
        raise ValueError(f"{kind.value} needs {kind.n_nodes} node ids, got shape {ids.shape}")
    a, vol = batch_precompute(kind, np.asarray(coords, dtype=np.float64)[None])
    return ElementPrecomp(kind=kind, node_ids=ids, unit_conductance=a[0], volume=float(vol[0]))
