"""Failure and boundary semantics of the GPU step (reference solver.py:348-382).

* A runaway step on a mesh several launch waves large: every CTA of the failing
  step must still write its tile, so the reported step, node and field are the
  reference's (the oracle's) -- EXACT bitwise, TILED fp64 to 1e-10.
* Dirichlet values are re-imposed on the device in TILED mode, whatever the
  host state holds at those nodes (solver.py:364-365).
* A Dirichlet value beyond the runaway limit fails the first step (the
  reference checks max |T| over every node, solver.py:369-370).
* state.inflow after ExplicitEngine.step in TILED mode is the step's F.
* fh_step_host_async / fh_host_wait: a failure rolls the clock back, clears
  the flag and refuses further async calls until a field is set.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import _native as N  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def unstable_problem(div=100, seed=7):
    """A 100^3 hex cube (1.03 M nodes: ~3.5 waves of EXACT node blocks, and
    with 256-node tiles ~7 waves of TILED CTAs) with a rough initial field and
    dt = 3x the critical step: the highest modes grow ~5x per step."""
    mesh = fh.generate_cube_mesh("hex", div, 0.1)
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
    rng = np.random.default_rng(seed)
    T0 = 37.0 + rng.uniform(-1.0, 1.0, mesh.n_nodes)
    return mesh, mat, T0


def oracle_failure(mesh, mat, T0, dt):
    ora = orc.OracleModel(mesh, mat, td_mode=False)
    ora.initial_state(T0)
    with pytest.raises(orc.InstabilityInOracle) as err:
        ora.step(dt, 200)
    return err.value.step, err.value.node, ora.T


@pytest.mark.parametrize("assembly,prec", [("exact", 64), ("tiled", 64)])
def test_multiwave_instability_matches_oracle(assembly, prec):
    mesh, mat, T0 = unstable_problem()
    eng = fh.ExplicitEngine(mesh, mat, assembly=assembly, precision=prec, part_nodes=256)
    dt = 3.0 * eng.critical_dt(T0)
    fs, fn, T_ref = oracle_failure(mesh, mat, T0, dt)
    assert fs > 3  # several clean steps first
    with pytest.raises(fh.InstabilityError) as err:
        eng.run(T0, steps=200, dt=dt)
    assert err.value.step == fs
    assert err.value.node == fn
    T = eng.temperature()
    if assembly == "exact":
        assert np.array_equal(T, T_ref)
    else:
        assert np.abs(T - T_ref).max() <= 1e-10 * np.abs(T_ref).max()
    # the engine is reusable afterwards
    eng.run(37.0, steps=2, dt=dt / 10.0)


@pytest.mark.parametrize("prec", [64, 32])
def test_tiled_step_reimposes_dirichlet(prec):
    mesh = fh.generate_cube_mesh("hex", 12, 0.1)
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
    bnd = fh.BoundarySpec(dirichlet=(("x0", 30.0), ("x1", 45.0)))
    eng = fh.ExplicitEngine(mesh, mat, bnd, assembly="tiled", precision=prec, part_nodes=128)
    ref = fh.ExplicitEngine(mesh, mat, bnd)
    dt = 0.5 * ref.critical_dt(37.0)
    # a state NOT built by initial_state: wrong values at the Dirichlet nodes
    st = fh.SimState(temperatures=np.full(mesh.n_nodes, 37.0))
    st_ref = fh.SimState(temperatures=np.full(mesh.n_nodes, 37.0))
    for _ in range(5):
        eng.step(st, dt)
        ref.step(st_ref, dt)
    d = eng.boundary.dirichlet_nodes
    assert np.array_equal(st.temperatures[d], eng.boundary.dirichlet_values)
    tol = 1e-10 if prec == 64 else 1e-5
    assert np.abs(st.temperatures - st_ref.temperatures).max() <= tol * 45.0


@pytest.mark.parametrize("assembly", ["exact", "tiled"])
def test_dirichlet_beyond_runaway_fails_first_step(assembly):
    mesh = fh.generate_cube_mesh("hex", 4, 0.1)
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
    bnd = fh.BoundarySpec(dirichlet=(("x0", 2.0e6),))
    eng = fh.ExplicitEngine(mesh, mat, bnd, assembly=assembly)
    with pytest.raises(fh.InstabilityError) as err:
        eng.run(37.0, steps=5, dt=1.0)
    assert err.value.step == 1
    assert err.value.node == int(eng.boundary.dirichlet_nodes[0])


@pytest.mark.parametrize("prec", [64, 32])
def test_tiled_step_fills_inflow(prec):
    mesh = fh.generate_cube_mesh("tet", 8, 0.1)
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 30.0),))
    eng = fh.ExplicitEngine(mesh, mat, bnd, assembly="tiled", precision=prec, part_nodes=96)
    ex = fh.ExplicitEngine(mesh, mat, bnd)
    rng = np.random.default_rng(3)
    st = eng.initial_state(37.0 + rng.uniform(-2, 2, mesh.n_nodes))
    st_ex = fh.SimState(temperatures=st.temperatures.copy())
    eng.step(st, 1.0)
    ex.step(st_ex, 1.0)
    free = np.ones(mesh.n_nodes, bool)
    free[eng.boundary.dirichlet_nodes] = False
    scale = np.abs(st_ex.inflow[free]).max()
    tol = 1e-10 if prec == 64 else 1e-4
    assert np.abs(st.inflow[free] - st_ex.inflow[free]).max() <= tol * scale
    assert np.all(st.inflow[~free] == 0.0)


def test_async_failure_resets_and_refuses():
    mesh, mat, T0 = unstable_problem(div=24)
    eng = fh.ExplicitEngine(mesh, mat, assembly="tiled", precision=64, part_nodes=256)
    dt = 3.0 * eng.critical_dt(T0)
    fs, _, _ = oracle_failure(mesh, mat, T0, dt)
    L, h = eng._L, eng._h
    Tin = N.f64(T0)
    Tout = np.empty_like(Tin)
    N.check(L.fh_set_temperature(h, N.ptr(Tin), Tin.size, 0, 0.0))
    N.check(L.fh_step_host_async(h, N.ptr(Tin), N.ptr(Tout), Tin.size, 200, dt, 0))
    rep = N.FhReport()
    rc = L.fh_host_wait(h, 0, C.byref(rep))
    assert rc == 2 and rep.fail_step == fs and rep.step_index == fs
    assert L.fh_step_host_async(h, N.ptr(Tin), N.ptr(Tout), Tin.size, 1, dt, 1) == 1  # refused
    N.check(L.fh_set_temperature(h, N.ptr(Tin), Tin.size, 0, 0.0))
    N.check(L.fh_step_host_async(h, N.ptr(Tin), N.ptr(Tout), Tin.size, 1, dt / 10.0, 1))
    N.check(L.fh_host_wait(h, 1, C.byref(rep)))


def test_async_failure_on_the_resident_exact_kernel_stops_at_the_failing_step():
    """A multi-step asynchronous call cannot replay a runaway, so it keeps the
    resident kernel's grid barrier: the field that comes back is the one right
    after the failing step, exactly what the synchronous call reports."""
    mesh, mat, T0 = unstable_problem(div=12)
    dt = None
    fields = []
    for mode in ("sync", "async"):
        eng = fh.ExplicitEngine(mesh, mat)  # EXACT fp64, resident kernel (stamped halo words by default)
        assert eng.layout()["kernels_per_step"] == 0
        dt = dt or 3.0 * eng.critical_dt(T0)
        L, h = eng._L, eng._h
        Tin = N.f64(T0)
        Tout = np.empty_like(Tin)
        rep = N.FhReport()
        if mode == "sync":
            assert L.fh_step_host(h, N.ptr(Tin), N.ptr(Tout), Tin.size, 300, dt, C.byref(rep)) == 2
        else:
            N.check(L.fh_set_temperature(h, N.ptr(Tin), Tin.size, 0, 0.0))
            N.check(L.fh_step_host_async(h, N.ptr(Tin), N.ptr(Tout), Tin.size, 300, dt, 0))
            assert L.fh_host_wait(h, 0, C.byref(rep)) == 2
        fields.append((rep.fail_step, eng.temperature()))
    assert fields[0][0] == fields[1][0] > 1
    assert np.array_equal(fields[0][1], fields[1][1], equal_nan=True)
