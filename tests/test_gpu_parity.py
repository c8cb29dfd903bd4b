"""GPU parity: the CUDA engine vs the reference golden vectors and the oracle.

EXACT mode (fp64, reference operation order) must be bit-identical to the
reference; TILED mode (fused single kernel, G-form) must agree with the
oracle within rel 1e-10 (fp64) / 1e-4 (fp32), the tolerances of north_star.
"""

import numpy as np
import pytest

from golden_io import PRECOMP, RUNS, load, loads, material, mesh_ns

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from oracle import oracle as orc  # noqa: E402

TOL = {64: 1e-10, 32: 1e-4}


def golden_problem(d):
    """Mesh + BoundarySpec reproducing a golden run's resolved boundary."""
    sets = {}
    dirichlet = []
    for k, v in enumerate(np.unique(d["dir_vals"])):
        sets[f"dir{k}"] = d["dir_nodes"][d["dir_vals"] == v]
        dirichlet.append((f"dir{k}", float(v)))
    heat = []
    for i, (nodes, p, a, b) in enumerate(loads(d)):
        sets[f"load{i}"] = nodes
        heat.append((f"load{i}", p, a, b))
    mesh = fh.Mesh(nodes=d["nodes"], tets=d["tets"], hexes=d["hexes"], node_sets=sets)
    return mesh, fh.BoundarySpec(dirichlet=tuple(dirichlet), heat_loads=tuple(heat))


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("tag", RUNS)
def test_exact_runs_bitwise_vs_reference(tag):
    d = load(f"run_{tag}.npz")
    mesh, bnd = golden_problem(d)
    eng = fh.ExplicitEngine(mesh, material(d), bnd, td_mode=bool(d["td_mode"]))
    res = eng.run(d["T0"], steps=int(d["steps"]), dt=float(d["dt"]), probes=d["probes"],
                  probe_interval=int(d["interval"]))
    assert np.array_equal(res.state.temperatures, d["T_final"])
    assert np.array_equal(res.probe_values, d["probe_values"])
    assert np.array_equal(res.probe_times, d["probe_times"])
    assert res.state.time == float(d["time_final"])


def test_exact_cfg1_auto_dt_bitwise():
    d = load("run_cfg1.npz")
    mesh, bnd = golden_problem(d)
    eng = fh.ExplicitEngine(mesh, material(d), bnd)
    res = eng.run(37.0, steps=int(d["steps"]), auto_dt_safety=0.9, probes=d["probes"])
    assert res.dt == float(d["dt"]) and res.dt_critical == float(d["dt_critical"])
    assert np.array_equal(res.state.temperatures, d["T_final"])


def test_exact_step_api_bitwise():
    d = load("run_scen_twostage.npz")
    mesh, bnd = golden_problem(d)
    eng = fh.ExplicitEngine(mesh, material(d), bnd)
    st = eng.initial_state(d["T0"])
    for _ in range(int(d["steps"])):
        eng.step(st, float(d["dt"]))
    assert np.array_equal(st.temperatures, d["T_final"])
    assert st.step_index == int(d["steps"])


@pytest.mark.parametrize("tag", PRECOMP)
def test_device_precompute_bitwise(tag):
    d = load(f"precompute_{tag}.npz")
    mesh = fh.Mesh(nodes=d["nodes"], tets=d["tets"], hexes=d["hexes"])
    eng = fh.ExplicitEngine(mesh, material(d))
    assert np.array_equal(eng.lumped.node_volumes, d["node_volumes"])
    assert np.array_equal(eng.lumped.perfusion_conductance, d["perfusion_conductance"])
    assert np.array_equal(eng.lumped.perfusion_heat, d["perfusion_heat"])


def test_scatter_bitwise_engine_and_operator():
    d = load("scatter_tet12.npz")
    mesh = fh.Mesh(nodes=d["nodes"], tets=d["tets"], hexes=d["hexes"])
    packed = fh.PackedElements(mesh)
    for r in range(3):
        out = fh.scatter_loads(packed, d[f"kbar{r}"], d[f"T{r}"])
        assert np.array_equal(out, d[f"inflow{r}"])


def test_critical_dt_bitwise():
    d = load("critical_dt.npz")
    mat = material(d)
    for case in range(6):
        mesh = fh.Mesh(nodes=d[f"c{case}_nodes"], tets=d[f"c{case}_tets"], hexes=d[f"c{case}_hexes"])
        assert fh.ExplicitEngine(mesh, mat).critical_dt(d[f"c{case}_T"]) == float(d[f"c{case}_dt"])


def test_instability_step_node_field():
    d = load("instability.npz")
    mesh = fh.Mesh(nodes=d["nodes"], tets=d["tets"], hexes=d["hexes"])
    for assembly, prec in (("exact", 64), ("tiled", 64)):
        eng = fh.ExplicitEngine(mesh, material(d), assembly=assembly, precision=prec)
        st = eng.initial_state(d["T0"])
        with pytest.raises(fh.InstabilityError) as err:
            for _ in range(2000):
                eng.step(st, float(d["dt"]))
        if assembly == "exact":
            assert err.value.step == int(d["fail_step"]) and err.value.node == int(d["fail_node"])
            assert np.array_equal(st.temperatures, d["T_fail"])
        else:
            assert abs(err.value.step - int(d["fail_step"])) <= 1


def test_operator_layer_bitwise(rng):
    from paper_1909_05098_b200 import kernels as K
    xs, ys = np.array([37.0, 50.0, 65.0]), np.array([0.53, 0.55, 0.57])
    T = rng.uniform(20.0, 80.0, 5000)
    out = np.empty_like(T)
    K.eval_curve_nodes(xs, ys, T, out)
    assert np.array_equal(out, np.interp(T, xs, ys))
    v = rng.uniform(1e-6, 1e-5, T.size)
    K.lumped_capacity_nodes(xs, ys * 2e3, xs, ys * 7e3, T, v, out)
    assert np.array_equal(out, np.interp(T, xs, ys * 2e3) * np.interp(T, xs, ys * 7e3) * v)
    arrs = [rng.uniform(-1, 1, T.size) for _ in range(6)]
    arrs[1] = rng.uniform(1, 2, T.size)
    got = T.copy()
    K.nodal_update(got, *arrs, 0.3)
    F, Cp, kb, qb, qm, qr = arrs
    assert np.array_equal(got, T + 0.3 * (F - kb * T + qb + qm + qr) / Cp)


# ---------------------------------------------------------------------------
# TILED (fused) mode vs the oracle


def oracle_for(eng, d=None, mesh=None, mat=None):
    rb = eng.boundary
    return orc.OracleModel(mesh or eng.mesh, mat or eng.material, dirichlet=(rb.dirichlet_nodes, rb.dirichlet_values),
                           loads=[(n, p, a, b) for n, p, a, b in rb.loads], td_mode=eng.td_mode)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("tag", ["scen_td", "scen_twostage", "cfg1"])
def test_tiled_vs_oracle(tag, prec):
    d = load(f"run_{tag}.npz")
    mesh, bnd = golden_problem(d)
    steps = min(int(d["steps"]), 400)
    eng = fh.ExplicitEngine(mesh, material(d), bnd, td_mode=bool(d["td_mode"]), assembly="tiled",
                            precision=prec, part_nodes=512)
    res = eng.run(d["T0"], steps=steps, dt=float(d["dt"]))
    ora = oracle_for(eng, mat=material(d))
    T_ref, _ = ora.run(d["T0"], steps, float(d["dt"]))
    assert rel_err(res.state.temperatures, T_ref) <= TOL[prec]


@pytest.mark.parametrize("prec", [64, 32])
def test_tiled_deterministic_and_invariants(prec):
    mesh = fh.generate_cube_mesh("tet", 6, 0.1)
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518,
                                     perfusion_rate=26.6, arterial_temperature=39.0)
    eng = fh.ExplicitEngine(mesh, mat, assembly="tiled", precision=prec, part_nodes=96)
    st = eng.initial_state(39.0)
    ref = st.temperatures.copy()
    for _ in range(20):
        eng.step(st, 0.05)
    assert np.array_equal(st.temperatures, ref)  # arterial fixed point, bitwise
    mat2 = fh.TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518)
    eng2 = fh.ExplicitEngine(mesh, mat2, fh.BoundarySpec(dirichlet=(("z0", 30.0),)), assembly="tiled",
                             precision=prec, part_nodes=96)
    a = eng2.run(37.0, steps=50, dt=20.0).state.temperatures
    b = eng2.run(37.0, steps=50, dt=20.0).state.temperatures
    assert np.array_equal(a, b)
