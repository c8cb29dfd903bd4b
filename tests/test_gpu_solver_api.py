"""The reference's solver test cases (/root/reference/pkg/tests/test_solver.py),
restated against this package's API and run on the GPU engine.

Same scenarios, same known answers (hand values, closed forms, exact
invariants), so a fedheat user sees the same behaviour after switching.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")

UNIT_TET = fh.Mesh(nodes=np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]), tets=np.array([[0, 1, 2, 3]]),
                   hexes=np.empty((0, 8)), node_sets={"all": np.arange(4), "first": np.array([0])})
CONST = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518)


def td_material(**kw):
    return fh.TissueMaterial(density=fh.PropertyCurve([37.0, 65.0], [1040.0, 1000.0]),
                             specific_heat=fh.PropertyCurve([37.0, 65.0], [3600.0, 3800.0]),
                             conductivity=fh.PropertyCurve([37.0, 65.0], [0.53, 0.57]), **kw)


def mixed_mesh(rng, div=3):
    from paper_1909_05098_b200.meshgen import HEX_CORNER_OFFSETS, KUHN_PATTERNS
    n = div + 1
    size = float(rng.uniform(0.02, 1.5))
    ax = np.linspace(0.0, size, n)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    nodes = np.column_stack([xx.ravel(), yy.ravel(), zz.ravel()]) + rng.uniform(-0.12, 0.12, (n ** 3, 3)) * size / div
    idx = lambda i, j, k: i + n * (j + n * k)  # noqa: E731
    tets, hexes = [], []
    for i in range(div):
        for j in range(div):
            for k in range(div):
                b = np.array([i, j, k])
                if rng.random() < 0.5:
                    tets += [[idx(*(b + o)) for o in p] for p in KUHN_PATTERNS]
                else:
                    hexes.append([idx(*(b + o)) for o in HEX_CORNER_OFFSETS])
    return fh.Mesh(nodes=nodes, tets=np.array(tets, np.int64).reshape(-1, 4),
                   hexes=np.array(hexes, np.int64).reshape(-1, 8), node_sets={"all": np.arange(n ** 3)})


def dense_k(mesh, kval):
    K = np.zeros((mesh.n_nodes, mesh.n_nodes))
    for kind, ids in mesh.iter_elements():
        pre = fh.build_precomp(kind, ids, mesh.nodes[ids])
        K[np.ix_(ids, ids)] += kval * pre.unit_conductance
    return K


@pytest.mark.parametrize("assembly", ["exact", "tiled"])
def test_scatter_matches_dense_assembly(rng, assembly):
    """scatter == -K T to 1e-12 (reference test_solver.py:76-87), via one explicit step."""
    for _ in range(3):
        mesh = mixed_mesh(rng)
        T = rng.uniform(20.0, 60.0, mesh.n_nodes)
        expected = -(dense_k(mesh, 0.518) @ T)
        if assembly == "exact":
            packed = fh.PackedElements(mesh)
            got = fh.scatter_loads(packed, np.full(packed.n_elements, 0.518), T)
        else:  # F = C (T' - T) / dt on an adiabatic constant-property step
            eng = fh.ExplicitEngine(mesh, CONST, assembly="tiled", precision=64, part_nodes=40)
            st = eng.initial_state(T)
            C = fh.lumped_mass(CONST, eng.lumped.node_volumes, T)
            dt = 100.0 / np.abs(expected / C).max()  # one (unstable but exact) step with O(100) increments
            eng.step(st, dt)
            got = (st.temperatures - T) * C / dt
            assert np.abs(got - expected).max() <= 1e-11 * np.abs(expected).max()
            continue
        assert np.abs(got - expected).max() <= 1e-12 * max(np.abs(expected).max(), 1e-30)


def test_uniform_field_bitwise_zero(rng):
    mesh = mixed_mesh(rng)
    packed = fh.PackedElements(mesh)
    out = fh.scatter_loads(packed, rng.uniform(0.3, 0.8, packed.n_elements), np.full(mesh.n_nodes, 38.25))
    assert np.array_equal(out, np.zeros(mesh.n_nodes))


@pytest.mark.parametrize("assembly,prec", [("exact", 64), ("tiled", 64), ("tiled", 32)])
def test_uniform_adiabatic_bitwise_constant(rng, assembly, prec):
    mesh = mixed_mesh(rng)
    eng = fh.ExplicitEngine(mesh, CONST, assembly=assembly, precision=prec, part_nodes=40)
    st = eng.initial_state(37.25)
    ref = st.temperatures.copy()
    for _ in range(50):
        eng.step(st, 1.0)
    assert np.array_equal(st.temperatures, ref)


def test_perfusion_single_step_hand_value():
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518, perfusion_rate=26.6,
                                     blood_specific_heat=3617.0, arterial_temperature=39.0)
    eng = fh.ExplicitEngine(UNIT_TET, mat)
    st = eng.initial_state(37.0)
    eng.step(st, 0.01)
    expected = 37.0 + 0.01 * (26.6 * 3617.0) * 2.0 / (1060.0 * 3700.0)
    assert np.allclose(st.temperatures, expected, rtol=1e-14)
    assert st.temperatures[0] == pytest.approx(37.000490628, abs=1e-8)


def test_perfusion_trajectory_discrete_closed_form():
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518, perfusion_rate=26.6,
                                     blood_specific_heat=3617.0, arterial_temperature=39.0)
    eng = fh.ExplicitEngine(fh.generate_cube_mesh("tet", 2, 0.05), mat)
    res = eng.run(37.0, steps=500, dt=0.01)
    ratio = 26.6 * 3617.0 / (1060.0 * 3700.0)
    assert np.allclose(res.state.temperatures, 39.0 - 2.0 * (1.0 - 0.01 * ratio) ** 500, rtol=1e-12)


def test_metabolic_rise_exactly_linear():
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518, metabolic_rate=33800.0)
    eng = fh.ExplicitEngine(fh.generate_cube_mesh("hex", 2, 0.04), mat)
    res = eng.run(37.0, steps=400, dt=0.01)
    assert np.allclose(res.state.temperatures, 37.0 + 400 * 0.01 * 33800.0 / (1060.0 * 3700.0), rtol=1e-12)


def test_dirichlet_held_exactly_and_half_open_load_window():
    mesh = fh.generate_cube_mesh("tet", 3, 0.1)
    eng = fh.ExplicitEngine(mesh, CONST, fh.BoundarySpec(dirichlet=(("z0", 36.0), ("z1", 40.0))))
    st = eng.initial_state(37.0)
    for _ in range(20):
        eng.step(st, 50.0)
        assert np.all(st.temperatures[mesh.node_sets["z0"]] == 36.0)
        assert np.all(st.temperatures[mesh.node_sets["z1"]] == 40.0)
    mat = fh.TissueMaterial.constant(density=1000.0, specific_heat=1000.0, conductivity=0.5)
    eng = fh.ExplicitEngine(UNIT_TET, mat, fh.BoundarySpec(heat_loads=(("all", 2.0, 0.0, 0.5),)))
    st = eng.initial_state(37.0)
    per = 0.25 * 2.0 / (1000.0 * 1000.0 * (1.0 / 6.0) / 4.0)
    eng.step(st, 0.25)
    assert np.allclose(st.temperatures, 37.0 + per, rtol=1e-12)
    eng.step(st, 0.25)
    frozen = st.temperatures.copy()
    eng.step(st, 0.25)  # t = 0.5: closed end of [0, 0.5)
    assert np.array_equal(st.temperatures, frozen)


def test_critical_dt_closed_form_and_scaling():
    eng = fh.ExplicitEngine(UNIT_TET, CONST)
    assert eng.critical_dt(37.0) == pytest.approx(1060.0 * 3700.0 / (12.0 * 0.518), rel=1e-12)
    mat2 = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=1.036)
    assert fh.ExplicitEngine(UNIT_TET, mat2).critical_dt(37.0) == pytest.approx(eng.critical_dt(37.0) / 2, rel=1e-12)


@pytest.mark.parametrize("assembly,prec", [("exact", 64), ("tiled", 32)])
def test_instability_and_runaway(assembly, prec):
    mesh = fh.generate_cube_mesh("tet", 3, 0.01)
    eng = fh.ExplicitEngine(mesh, CONST, assembly=assembly, precision=prec, part_nodes=30)
    dt_cr = eng.critical_dt(37.0)
    st = eng.initial_state(37.0 + 0.01 * np.sin(np.arange(mesh.n_nodes)))
    with pytest.raises(fh.InstabilityError):
        for _ in range(2000):
            eng.step(st, 10.0 * dt_cr)
    mat = fh.TissueMaterial.constant(density=1000.0, specific_heat=1000.0, conductivity=0.5, metabolic_rate=1e9)
    eng = fh.ExplicitEngine(UNIT_TET, mat, runaway_limit=50.0, assembly=assembly, precision=prec)
    st = eng.initial_state(37.0)
    with pytest.raises(fh.InstabilityError, match="node"):
        for _ in range(10_000):
            eng.step(st, 1.0)


def test_run_probes_auto_dt_and_argument_checks():
    mesh = fh.generate_cube_mesh("tet", 3, 0.1)
    eng = fh.ExplicitEngine(mesh, CONST, fh.BoundarySpec(dirichlet=(("z0", 38.0),)))
    res = eng.run(37.0, steps=10, dt=2.0, probes=mesh.node_sets["center"], probe_interval=2)
    assert res.probe_values.shape == (6, 1)
    assert np.allclose(res.probe_times, [0.0, 4.0, 8.0, 12.0, 16.0, 20.0])
    res = fh.ExplicitEngine(UNIT_TET, CONST).run(37.0, steps=3, auto_dt_safety=0.5)
    assert res.dt == pytest.approx(0.5 * res.dt_critical, rel=1e-12)
    with pytest.raises(fh.ConfigError, match="exactly one"):
        fh.ExplicitEngine(UNIT_TET, CONST).run(37.0, steps=3, dt=0.1, auto_dt_safety=0.5)


def test_ti_mode_freezes_initial_properties():
    mat = fh.TissueMaterial(density=fh.make_constant(1000.0), specific_heat=fh.make_constant(1000.0),
                            conductivity=fh.PropertyCurve([37.0, 40.0], [0.5, 1.0]))
    mesh = fh.generate_cube_mesh("tet", 2, 0.1)
    hot = fh.BoundarySpec(dirichlet=(("z0", 60.0),))
    for assembly, prec in (("exact", 64), ("tiled", 64)):
        r_ti = fh.ExplicitEngine(mesh, mat, hot, td_mode=False, assembly=assembly, precision=prec).run(
            37.0, steps=200, dt=100.0)
        r_td = fh.ExplicitEngine(mesh, mat, hot, td_mode=True, assembly=assembly, precision=prec).run(
            37.0, steps=200, dt=100.0)
        assert not np.allclose(r_ti.state.temperatures, r_td.state.temperatures, rtol=1e-6)


def test_orphan_node_rules():
    nodes = np.vstack([UNIT_TET.nodes, [5.0, 5.0, 5.0]])
    mesh = fh.Mesh(nodes=nodes, tets=UNIT_TET.tets, hexes=np.empty((0, 8)), node_sets={"orphan": np.array([4])})
    with pytest.raises(fh.ConfigError, match="capacity"):
        fh.ExplicitEngine(mesh, CONST).initial_state(37.0)
    eng = fh.ExplicitEngine(mesh, CONST, fh.BoundarySpec(dirichlet=(("orphan", 37.0),)))
    st = eng.initial_state(37.0)
    eng.step(st, 1.0)
    assert st.temperatures[4] == 37.0


@pytest.mark.parametrize("assembly,prec", [("exact", 64), ("tiled", 32)])
def test_full_runs_bitwise_repeatable(assembly, prec):
    mesh = fh.generate_cube_mesh("tet", 5, 0.1)
    mat = td_material(perfusion_rate=26.6, arterial_temperature=37.0, metabolic_rate=33800.0)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0),), heat_loads=(("center", 2.0, 0.0, 1.0),))
    eng = fh.ExplicitEngine(mesh, mat, bnd, assembly=assembly, precision=prec, part_nodes=50)
    a = eng.run(37.0, steps=60, dt=0.01).state.temperatures
    b = eng.run(37.0, steps=60, dt=0.01).state.temperatures
    assert np.array_equal(a, b)


@pytest.mark.parametrize("assembly,prec", [("exact", 64), ("tiled", 32)])
def test_step_host_async_matches_sync(assembly, prec):
    """fh_step_host_async (double-buffered host I/O) == fh_step_host, bitwise,
    for alternating slots; misuse (slot still in flight) is a ConfigError."""
    import ctypes as C

    import torch

    from paper_1909_05098_b200 import _native as N

    mesh = fh.generate_cube_mesh("hex", 8, 0.1)
    mat = fh.TissueMaterial(density=fh.make_constant(1060.0), specific_heat=fh.linear_law(3600.0, -0.0005, 37.0),
                            conductivity=fh.linear_law(0.5, 0.0013, 37.0), perfusion_rate=0.525,
                            blood_specific_heat=3640.0, metabolic_rate=420.0)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0),), heat_loads=(("center", 0.5, 0.0, 1e9),))
    eng = fh.ExplicitEngine(mesh, mat, bnd, assembly=assembly, precision=prec)
    dt = 0.9 * eng.critical_dt(37.0)
    L, h, V = eng._L, eng._h, mesh.n_nodes
    rng = np.random.default_rng(7)
    fields = [37.0 + rng.random(V) for _ in range(4)]
    rep = N.FhReport()
    ref = []
    for f in fields:
        out = np.empty(V)
        N.check(L.fh_step_host(h, N.ptr(np.ascontiguousarray(f)), N.ptr(out), V, 3, dt, C.byref(rep)))
        ref.append(out)
    pins = [torch.empty(V, dtype=torch.float64, pin_memory=True) for _ in range(4)]
    outs = [torch.empty(V, dtype=torch.float64, pin_memory=True) for _ in range(4)]
    ptr = lambda t: C.cast(C.c_void_p(t.data_ptr()), N.f64p)  # noqa: E731
    for k, f in enumerate(fields):
        pins[k].numpy()[:] = f
        N.check(L.fh_step_host_async(h, ptr(pins[k]), ptr(outs[k]), V, 3, dt, k % 2))
        if k >= 1:
            N.check(L.fh_host_wait(h, (k - 1) % 2, C.byref(rep)))
    N.check(L.fh_host_wait(h, 1, C.byref(rep)))
    for k in range(4):
        assert np.array_equal(outs[k].numpy(), ref[k])
    N.check(L.fh_step_host_async(h, ptr(pins[0]), ptr(outs[0]), V, 1, dt, 0))
    with pytest.raises(fh.ConfigError):
        N.check(L.fh_step_host_async(h, ptr(pins[1]), ptr(outs[1]), V, 1, dt, 0))
    N.check(L.fh_host_wait(h, 0, C.byref(rep)))
