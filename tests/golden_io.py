"""Helpers that turn the golden .npz fixtures (tests/golden/make_golden.py)
back into inputs for the oracle and the engine."""

from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def curve(d, name, prefix="mat_"):
    return SimpleNamespace(temperatures=d[f"{prefix}{name}_x"], values=d[f"{prefix}{name}_y"])


def material_ns(d, prefix="mat_"):
    """Duck-typed TissueMaterial (works for the oracle)."""
    dens, cap, cond = (curve(d, n, prefix) for n in ("density", "specific_heat", "conductivity"))
    is_const = all(np.all(c.values == c.values[0]) for c in (dens, cap, cond))
    return SimpleNamespace(
        density=dens, specific_heat=cap, conductivity=cond,
        perfusion_rate=float(d[f"{prefix}perfusion_rate"]),
        blood_specific_heat=float(d[f"{prefix}blood_specific_heat"]),
        arterial_temperature=float(d[f"{prefix}arterial_temperature"]),
        metabolic_rate=float(d[f"{prefix}metabolic_rate"]),
        perfusion_curve=None, is_constant=is_const)


def material(d, prefix="mat_"):
    """A real paper_1909_05098_b200 TissueMaterial."""
    from paper_1909_05098_b200.material import PropertyCurve, TissueMaterial
    return TissueMaterial(
        density=PropertyCurve(d[f"{prefix}density_x"], d[f"{prefix}density_y"]),
        specific_heat=PropertyCurve(d[f"{prefix}specific_heat_x"], d[f"{prefix}specific_heat_y"]),
        conductivity=PropertyCurve(d[f"{prefix}conductivity_x"], d[f"{prefix}conductivity_y"]),
        perfusion_rate=float(d[f"{prefix}perfusion_rate"]),
        blood_specific_heat=float(d[f"{prefix}blood_specific_heat"]),
        arterial_temperature=float(d[f"{prefix}arterial_temperature"]),
        metabolic_rate=float(d[f"{prefix}metabolic_rate"]))


def mesh_ns(d, prefix=""):
    return SimpleNamespace(nodes=d[f"{prefix}nodes"], tets=d[f"{prefix}tets"].reshape(-1, 4),
                           hexes=d[f"{prefix}hexes"].reshape(-1, 8))


def loads(d):
    offs = d["load_offs"]
    return [(d["load_nodes"][offs[i]:offs[i + 1]], float(d["load_power"][i]), float(d["load_t0"][i]),
             float(d["load_t1"][i])) for i in range(len(offs) - 1)]


RUNS = ["scen_conduction", "scen_perfusion", "scen_metabolic", "scen_twostage", "scen_td", "cfg1", "cfg2"]
PRECOMP = ["mixed3", "mixed5", "tet4j", "hex4j"]
