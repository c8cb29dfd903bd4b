"""Lumped nodal quantities (API of /root/reference/pkg/src/fedheat/precompute.py:22-62).

``build_lumped`` / ``lumped_mass`` are the reference's host-side helpers.  The
engine does not use them on its step path: ExplicitEngine computes the lumped
volumes on the GPU (fh_create) and exposes them as ``engine.lumped`` with the
same bits (kb = (w_b c_b) v, qb = kb * T_a, qm = Q_m v).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .material import TissueMaterial, eval_property
from .mesh import Mesh, node_volume_shares


@dataclass(frozen=True)
class LumpedSystem:
    node_volumes: np.ndarray
    perfusion_conductance: np.ndarray
    perfusion_heat: np.ndarray
    metabolic_heat: np.ndarray

    def __post_init__(self):
        for arr in (self.node_volumes, self.perfusion_conductance, self.perfusion_heat, self.metabolic_heat):
            arr.setflags(write=False)

    @property
    def n_nodes(self) -> int:
        return int(self.node_volumes.shape[0])


def lumped_from_volumes(vols: np.ndarray, material: TissueMaterial) -> LumpedSystem:
    vols = np.array(vols, dtype=np.float64)
    kb = material.perfusion_rate * material.blood_specific_heat * vols
    return LumpedSystem(node_volumes=vols, perfusion_conductance=kb,
                        perfusion_heat=kb * material.arterial_temperature,
                        metabolic_heat=material.metabolic_rate * vols)


def build_lumped(mesh: Mesh, material: TissueMaterial) -> LumpedSystem:
    return lumped_from_volumes(node_volume_shares(mesh), material)


def lumped_mass(material: TissueMaterial, node_volumes, temperature) -> np.ndarray:
    """Diagonal heat capacity rho(T) c(T) v per node (J/K)."""
    return eval_property(material.density, temperature) * eval_property(material.specific_heat, temperature) \
        * node_volumes
