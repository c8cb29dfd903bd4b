"""The BASELINE.json workloads as seeded synthetic problems.

Builder decisions for the parameters BASELINE leaves open are documented in
DESIGN.md "Open parameters"; everything is seeded so the GPU engine, the oracle
and the CPU baseline see identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .material import TissueMaterial, linear_law, make_constant
from .meshgen import generate_cube_mesh, jittered_cube_mesh
from .solver import BoundarySpec
from .sources import GaussianSource, RFSource, RobinSpec

FACES = ("x0", "x1", "y0", "y1", "z0", "z1")
PERFUSION_SLOPE = 0.002  # 1/K, open parameter


@dataclass
class Problem:
    name: str
    mesh: object
    material: TissueMaterial
    boundary: BoundarySpec
    steps: int
    precision: int
    td_mode: bool
    sources: tuple = ()
    robin: tuple = ()
    kfactor: np.ndarray | None = None
    auto_dt_safety: float = 0.9
    notes: dict = field(default_factory=dict)
    materials: list | None = None
    element_region: np.ndarray | None = None

    def engine_kwargs(self):
        kw = dict(td_mode=self.td_mode, precision=self.precision, sources=self.sources, robin=self.robin,
                  kfactor=self.kfactor)
        if self.materials is not None:
            kw.update(materials=self.materials, element_region=self.element_region)
        return kw


def pennes_constant() -> TissueMaterial:
    # BASELINE cfg1: rho 1060, c 3600, k 0.5; w_b = 0.5e-3 1/s * rho_b 1050 -> 0.525 kg/(m^3 s)
    return TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5, perfusion_rate=0.525,
                                   blood_specific_heat=3640.0, arterial_temperature=37.0, metabolic_rate=420.0)


def pennes_td(perfusion_td: bool = True, k0: float = 0.5, wb0: float = 0.525) -> TissueMaterial:
    # BASELINE cfg2 laws: k = 0.5 (1 + 0.0013 (T-37)), c = 3600 (1 - 0.0005 (T-37)), rho const,
    # perfusion linear in T (slope = PERFUSION_SLOPE, open parameter)
    return TissueMaterial(
        density=make_constant(1060.0), specific_heat=linear_law(3600.0, -0.0005, 37.0),
        conductivity=linear_law(k0, 0.0013, 37.0), perfusion_rate=wb0, blood_specific_heat=3640.0,
        arterial_temperature=37.0, metabolic_rate=420.0,
        perfusion_curve=linear_law(wb0, PERFUSION_SLOPE, 37.0) if perfusion_td else None)


def cfg1(divisions: int = 20) -> Problem:
    mesh = generate_cube_mesh("hex", divisions, 0.1)
    src = GaussianSource(amp=5.0e6, sigma=0.005, x0=(0.05, 0.05, 0.05))
    return Problem("cfg1", mesh, pennes_constant(), BoundarySpec(dirichlet=tuple((f, 37.0) for f in FACES)),
                   steps=1000, precision=64, td_mode=False, sources=(src,))


def cfg2(divisions: int = 20, precision: int = 64) -> Problem:
    mesh = generate_cube_mesh("hex", divisions, 0.1)
    src = GaussianSource(amp=2.0e7, sigma=0.005, x0=(0.05, 0.05, 0.05))
    return Problem("cfg2", mesh, pennes_td(), BoundarySpec(dirichlet=tuple((f, 37.0) for f in FACES)),
                   steps=2000, precision=precision, td_mode=True, sources=(src,))


def cfg3(divisions: int = 100, precision: int = 32, seed: int = 3) -> Problem:
    mesh = jittered_cube_mesh("tet", divisions, 0.1, 0.2, seed=seed)
    rng = np.random.default_rng(seed + 1000)
    centres = rng.uniform(0.025, 0.075, (3, 3))
    srcs = tuple(GaussianSource(amp=5.0e6, sigma=0.005, x0=tuple(c)) for c in centres)
    bnd = BoundarySpec(dirichlet=tuple((f, 37.0) for f in FACES if f != "z1"))
    return Problem("cfg3", mesh, pennes_td(), bnd, steps=500, precision=precision, td_mode=True, sources=srcs,
                   robin=(RobinSpec("z1", 10.0, 25.0),))


def cfg5(scale: int = 1, seed: int = 5) -> Problem:
    """Organ-like domain: ellipsoid (0.15 x 0.10 x 0.08 m) voxel-masked from a
    512 x 384 x 320 grid (h = 0.3/512 m; ``scale`` divides the grid for tests),
    10 % of boundary voxels split into tets, tumour sphere r = 15 mm (k 0.55,
    w_b 0.2e-3 1/s) in healthy tissue (k 0.5, w_b 0.6e-3 1/s), cfg2 laws, RF
    source at the tumour centre (P = 5 W, capped 1e8 W/m^3), Dirichlet 37 C on
    the organ surface (open parameters)."""
    from .meshgen import voxel_ellipsoid_mesh

    dims = (512 // scale, 384 // scale, 320 // scale)
    h = 0.3 / 512 * scale
    mesh, centre = voxel_ellipsoid_mesh(dims, h, seed=seed)
    rng = np.random.default_rng(seed + 1)
    # tumour centre: seeded, at least r = 15 mm inside the ellipsoid
    inner = np.array([0.15, 0.10, 0.08]) - 0.02
    while True:
        off = rng.uniform(-1.0, 1.0, 3) * inner
        if ((off / inner) ** 2).sum() <= 1.0:
            break
    tumour = centre + off
    conn = [mesh.tets, mesh.hexes]
    cent = np.concatenate([mesh.nodes[c].mean(axis=1) for c in conn if c.size])
    region = (np.linalg.norm(cent - tumour, axis=1) < 0.015).astype(np.int32)
    healthy = pennes_td(k0=0.5, wb0=0.6e-3 * 1050.0)
    tumour_mat = pennes_td(k0=0.55, wb0=0.2e-3 * 1050.0)
    src = RFSource(power=5.0, tip=tuple(tumour), cap=1.0e8)
    bnd = BoundarySpec(dirichlet=(("surface", 37.0),))
    prob = Problem("cfg5", mesh, healthy, bnd, steps=500, precision=32, td_mode=True, sources=(src,),
                   notes={"tumour_centre": tumour.tolist(), "regions": region})
    prob.materials = [healthy, tumour_mat]
    prob.element_region = region
    return prob


def cfg4(divisions: int = 256, seed: int = 4) -> Problem:
    mesh = generate_cube_mesh("hex", divisions, 0.1)
    rng = np.random.default_rng(seed)
    # per-element log-normal conductivity factor, sigma 0.2, median 1 (open parameter: normalisation)
    kf = np.exp(0.2 * rng.standard_normal(mesh.n_elements))
    a, b = rng.uniform(0.03, 0.07, 3), rng.uniform(0.03, 0.07, 3)
    steps = 200
    # moving source: straight segment a -> b traversed over the run at constant speed
    vel = tuple((b - a) / (steps * 1.0))  # m/s for dt = 1 s; rescaled in the bench to the actual dt
    src = GaussianSource(amp=5.0e6, sigma=0.005, x0=tuple(a), vel=vel)
    bnd = BoundarySpec(dirichlet=tuple((f, 37.0) for f in FACES))
    return Problem("cfg4", mesh, pennes_td(), bnd, steps=steps, precision=32, td_mode=True, sources=(src,),
                   kfactor=kf, notes={"path": (a.tolist(), b.tolist())})
