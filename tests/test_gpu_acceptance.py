"""The reference's acceptance guarantees (/root/reference/pkg/tests/
test_acceptance.py:190-450), restated against this package and run on the GPU
engine in both step implementations:

  04  uniform adiabatic field is a bitwise no-op; adiabatic conduction keeps
      the heat content sum C_i T_i to 1e-9 over 1e4 steps (TILED fp64 too);
  05  at 0.9x the Gershgorin step the field stays inside its initial envelope
      for 1e4 steps; at 2x the exact stability limit it blows up;
  06  the Gershgorin step is never optimistic (estimate >= exact eigenvalue);
  09  the explicit scheme converges to first order in dt.

Meshes are seeded, small (<= 300 nodes), so the dense generalised eigenvalue
problem of (K + K_b, C) is cheap on the host.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")

PAPER = dict(density=1060.0, specific_heat=3700.0, conductivity=0.518)
MODES = [("exact", 64), ("tiled", 64)]


def dense_lambda_max(mesh, mat, eng):
    """Largest eigenvalue of C^-1 (K + K_b) for constant properties."""
    K = np.zeros((mesh.n_nodes, mesh.n_nodes))
    for kind, ids in mesh.iter_elements():
        pre = fh.build_precomp(kind, ids, mesh.nodes[ids])
        K[np.ix_(ids, ids)] += mat.conductivity.values[0] * pre.unit_conductance
    v = fh.node_volume_shares(mesh)
    cap = mat.density.values[0] * mat.specific_heat.values[0] * v
    kb = mat.perfusion_rate * mat.blood_specific_heat * v
    K[np.diag_indices_from(K)] += kb
    s = 1.0 / np.sqrt(cap)
    return float(np.linalg.eigvalsh(s[:, None] * K * s[None, :]).max())


@pytest.mark.parametrize("assembly,prec", MODES)
def test_04_conservation_and_equilibrium(assembly, prec):
    mat = fh.TissueMaterial.constant(**PAPER)
    mesh = fh.generate_cube_mesh("tet", 4, 0.1)
    rng = np.random.default_rng(404)
    kw = dict(assembly=assembly, precision=prec, part_nodes=40)
    eng = fh.ExplicitEngine(mesh, mat, **kw)
    res = eng.run(37.25, steps=1000, dt=1.0)
    assert np.all(res.state.temperatures == 37.25)
    T0 = 37.0 + rng.uniform(-1.0, 1.0, mesh.n_nodes)
    st = eng.initial_state(T0)
    cap = fh.lumped_mass(mat, eng.lumped.node_volumes, st.temperatures)
    total0 = float(cap @ st.temperatures)
    dt = 0.5 * eng.critical_dt(st.temperatures)
    T = eng.run(T0, steps=10_000, dt=dt).state.temperatures
    assert abs(float(cap @ T) - total0) / abs(total0) <= 1e-9
    perf = fh.TissueMaterial.constant(**PAPER, perfusion_rate=26.6, arterial_temperature=39.0)
    T = fh.ExplicitEngine(mesh, perf, **kw).run(39.0, steps=1000, dt=0.05).state.temperatures
    assert np.abs(T - 39.0).max() <= 1e-12


@pytest.mark.parametrize("assembly,prec", MODES)
def test_05_stability_boundary(assembly, prec):
    rng = np.random.default_rng(505)
    for case in range(4):
        mesh = fh.generate_cube_mesh("tet", int(rng.integers(2, 5)), float(10.0 ** rng.uniform(-2.0, 0.0)))
        wb = 0.0 if case % 2 == 0 else float(rng.uniform(1.0, 30.0))
        mat = fh.TissueMaterial.constant(density=float(rng.uniform(800, 1200)),
                                         specific_heat=float(rng.uniform(1000, 4200)),
                                         conductivity=float(rng.uniform(0.2, 2.0)), perfusion_rate=wb,
                                         arterial_temperature=37.0)
        T0 = rng.uniform(20.0, 60.0, mesh.n_nodes)
        eng = fh.ExplicitEngine(mesh, mat, assembly=assembly, precision=prec, part_nodes=40)
        dt = 0.9 * eng.critical_dt(T0)
        centre = 37.0 if wb > 0 else 0.5 * (T0.min() + T0.max())
        bound = float(np.abs(T0 - centre).max())
        peak, T = bound, T0.copy()
        for _ in range(100):  # 1e4 steps, the envelope checked every 100
            T = eng.run(T, steps=100, dt=dt).state.temperatures
            peak = max(peak, float(np.abs(T - centre).max()))
        assert np.all(np.isfinite(T))
        assert (peak - bound) / bound <= 1e-9
        lam = dense_lambda_max(mesh, mat, eng)
        big = fh.ExplicitEngine(mesh, mat, assembly=assembly, precision=prec, part_nodes=40, runaway_limit=1e290)
        T = big.run(T0.copy(), steps=100, dt=2.0 * (2.0 / lam)).state.temperatures
        assert float(np.abs(T).max()) / float(np.abs(T0).max()) > 10.0


def test_06_safe_step_never_optimistic():
    rng = np.random.default_rng(606)
    for case in range(12):
        kind = "tet" if case % 2 else "hex"
        mesh = fh.generate_cube_mesh(kind, int(rng.integers(2, 5)), float(rng.uniform(0.02, 1.0)))
        mat = fh.TissueMaterial.constant(density=float(rng.uniform(800, 1200)),
                                         specific_heat=float(rng.uniform(1000, 4200)),
                                         conductivity=float(rng.uniform(0.2, 2.0)),
                                         perfusion_rate=float(rng.uniform(0.0, 30.0)))
        eng = fh.ExplicitEngine(mesh, mat)
        T = rng.uniform(20.0, 60.0, mesh.n_nodes)
        assert 2.0 / eng.critical_dt(T) >= dense_lambda_max(mesh, mat, eng) * (1.0 - 1e-12)


@pytest.mark.parametrize("assembly,prec", MODES)
def test_09_first_order_convergence_in_dt(assembly, prec):
    mesh = fh.generate_cube_mesh("tet", 6, 0.1)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0),), heat_loads=(("center", 0.5, 0.0, 1.0e9),))
    eng = fh.ExplicitEngine(mesh, fh.TissueMaterial.constant(**PAPER), bnd, assembly=assembly, precision=prec,
                            part_nodes=60)
    dt0 = 0.5 * eng.critical_dt(37.0)
    f = {d: eng.run(37.0, steps=64 * d, dt=dt0 / d).state.temperatures.copy() for d in (1, 2, 32)}
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b - 37.0))  # noqa: E731
    ratio = rel(f[1], f[32]) / rel(f[2], f[32])
    assert 1.7 <= ratio <= 2.3
