"""The resident small-mesh EXACT path (csrc/fh_resident.cu): many steps per
cooperative launch; the CTAs synchronise through stamped halo words (the
default, ``resident_sync=0``) or a grid barrier per step (``resident_sync=1``).

It must be bit-identical to the two-launch EXACT path (and so to the
reference): every run below is done twice, once with the resident kernel
(the default on meshes whose per-CTA working set fits shared memory) and once
with ``tuning={"exact_resident": 1}`` (k_exact_elem + k_exact_node per step),
and fields, probes, inflow and failure reports are compared bit for bit.  The
golden reference runs (tests/test_gpu_parity.py) already go through the
resident kernel by default; these cases add the extensions, load windows that
split a call into several launches, probe records across calls, TI freezing,
instability and the step() API.  Every case runs in both synchronisation
modes (the ``sync`` fixture).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import configs  # noqa: E402

from golden_io import load, material  # noqa: E402


@pytest.fixture(params=[0, 1], ids=["stamped", "barrier"], autouse=True)
def sync(request):
    global SYNC
    SYNC = request.param
    return request.param


SYNC = 0


def engines(mesh, mat, bnd=None, **kw):
    res = fh.ExplicitEngine(mesh, mat, bnd, tuning={"resident_sync": SYNC}, **kw)
    two = fh.ExplicitEngine(mesh, mat, bnd, tuning={"exact_resident": 1}, **kw)
    assert res.layout()["resident_ctas"] > 0 and res.layout()["kernels_per_step"] == 0
    assert two.layout()["resident_ctas"] == 0 and two.layout()["kernels_per_step"] == 2
    return res, two


def same_run(a, b):
    assert np.array_equal(a.state.temperatures, b.state.temperatures)
    assert np.array_equal(a.probe_values, b.probe_values)
    assert np.array_equal(a.probe_times, b.probe_times)
    assert a.state.time == b.state.time and a.state.step_index == b.state.step_index


def test_golden_cfg2_resident_bitwise():
    d = load("run_cfg2.npz")
    from test_gpu_parity import golden_problem

    mesh, bnd = golden_problem(d)
    eng = fh.ExplicitEngine(mesh, material(d), bnd, td_mode=bool(d["td_mode"]),
                            tuning={"exact_resident": 2, "resident_sync": SYNC})
    res = eng.run(d["T0"], steps=int(d["steps"]), dt=float(d["dt"]), probes=d["probes"],
                  probe_interval=int(d["interval"]))
    assert np.array_equal(res.state.temperatures, d["T_final"])
    assert np.array_equal(res.probe_values, d["probe_values"])


def test_load_windows_split_launches():
    """Heat loads switching on and off mid-call: each window edge starts a new
    launch with the new q_r (solver.py:307-318, start-of-step time)."""
    mesh = fh.generate_cube_mesh("hex", 8, 0.04)
    mat = configs.pennes_td()
    bnd = fh.BoundarySpec(dirichlet=(("x0", 37.0), ("x1", 37.0)),
                          heat_loads=(("center", 0.4, 0.0, 30.0), ("z1", 0.01, 20.0, 55.0), ("y0", 0.02, 41.0, 1e9)))
    a, b = engines(mesh, mat, bnd)
    dt = 0.8 * a.critical_dt(37.0)
    probes = np.array([0, 5, mesh.node_sets["center"][0], mesh.n_nodes - 1])
    ra = a.run(37.0, steps=97, dt=dt, probes=probes, probe_interval=3)
    rb = b.run(37.0, steps=97, dt=dt, probes=probes, probe_interval=3)
    same_run(ra, rb)
    assert ra.state.temperatures.max() > 37.001


@pytest.mark.parametrize("td", [True, False])
def test_extensions_bitwise(td):
    """cfg3 family: jittered tets, three Gaussians, Robin top face."""
    prob = configs.cfg3(divisions=7, precision=64)
    kw = dict(td_mode=td, sources=prob.sources, robin=prob.robin)
    a, b = engines(prob.mesh, prob.material, prob.boundary, **kw)
    dt = 0.9 * a.critical_dt(37.0)
    same_run(a.run(37.0, steps=60, dt=dt, probes=[0, 17, 99]), b.run(37.0, steps=60, dt=dt, probes=[0, 17, 99]))


def test_regions_kfactor_moving_source_bitwise():
    """Two materials (k(T) interpolated per element corner, not staged),
    per-element conductivity factor, a moving Gaussian (per-step start time)."""
    mesh = fh.generate_cube_mesh("hex", 9, 0.1)
    centroids = mesh.nodes[mesh.hexes].mean(axis=1)
    region = (np.linalg.norm(centroids - 0.05, axis=1) < 0.025).astype(np.int32)
    mats = [configs.pennes_td(k0=0.5, wb0=0.6e-3 * 1050.0), configs.pennes_td(k0=0.55, wb0=0.2e-3 * 1050.0)]
    kf = np.exp(0.2 * np.random.default_rng(5).standard_normal(mesh.n_elements))
    src = fh.GaussianSource(amp=2e5, sigma=0.01, x0=(0.03, 0.04, 0.05), vel=(1e-5, 0.0, 2e-6), t0=0.0)
    bnd = fh.BoundarySpec(dirichlet=tuple((f, 37.0) for f in configs.FACES))
    kw = dict(materials=mats, element_region=region, kfactor=kf, sources=(src,))
    a, b = engines(mesh, mats[0], bnd, **kw)
    dt = 0.9 * a.critical_dt(37.0)
    same_run(a.run(37.0, steps=45, dt=dt, probes=[1, 500]), b.run(37.0, steps=45, dt=dt, probes=[1, 500]))


def test_calls_continue_and_step_api():
    """Probe records and the clock continue across run segments; step() (one
    step per call) and inflow match the two-launch path."""
    mesh = fh.generate_cube_mesh("tet", 6, 0.05)
    mat = configs.pennes_td()
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0),), heat_loads=(("center", 0.3, 0.0, 1e9),))
    a, b = engines(mesh, mat, bnd)
    sa, sb = a.initial_state(36.5), b.initial_state(36.5)
    for k in range(7):
        a.step(sa, 0.7)
        b.step(sb, 0.7)
        assert np.array_equal(sa.temperatures, sb.temperatures), k
        assert np.array_equal(sa.inflow, sb.inflow), k
    T0 = np.linspace(36.0, 39.0, mesh.n_nodes)
    ra = a.run(T0, steps=31, dt=0.9, probes=[3, 4], probe_interval=4)
    rb = b.run(T0, steps=31, dt=0.9, probes=[3, 4], probe_interval=4)
    same_run(ra, rb)


@pytest.mark.parametrize("td", [False, True])
def test_instability_report_bitwise(td):
    mesh = fh.generate_cube_mesh("hex", 12, 0.1)
    mat = configs.pennes_td() if td else fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0,
                                                                    conductivity=0.5)
    T0 = 37.0 + np.random.default_rng(3).uniform(-1.0, 1.0, mesh.n_nodes)
    a, b = engines(mesh, mat, td_mode=td)
    dt = 3.0 * a.critical_dt(T0)
    errs = []
    for eng in (a, b):
        with pytest.raises(fh.InstabilityError) as err:
            eng.run(T0, steps=400, dt=dt, probes=[0, 7], probe_interval=2)
        errs.append(err.value)
    assert errs[0].step == errs[1].step > 2
    assert errs[0].node == errs[1].node
    assert np.array_equal(a.temperature(), b.temperature())
    # the engines stay usable: the same call fails the same way again, and a stable run follows
    with pytest.raises(fh.InstabilityError) as again:
        a.run(T0, steps=400, dt=dt)
    assert again.value.step == errs[0].step and again.value.node == errs[0].node
    ok_dt = 0.5 * a.critical_dt(T0)
    same_run(a.run(T0, steps=30, dt=ok_dt), b.run(T0, steps=30, dt=ok_dt))


def test_many_short_calls_keep_stamps_apart():
    """Stamps never repeat across launches: many 1- and 2-step calls with state
    resets in between (the step index restarts at 0 each time) stay bitwise."""
    mesh = fh.generate_cube_mesh("hex", 10, 0.1)
    mat = configs.pennes_td()
    bnd = fh.BoundarySpec(dirichlet=(("x0", 37.0),), heat_loads=(("center", 0.5, 0.0, 1e9),))
    a, b = engines(mesh, mat, bnd)
    dt = 0.9 * a.critical_dt(37.0)
    rng = np.random.default_rng(11)
    for k in range(12):
        T0 = 37.0 + rng.uniform(-0.5, 0.5, mesh.n_nodes)
        n = 1 + k % 3
        same_run(a.run(T0, steps=n, dt=dt), b.run(T0, steps=n, dt=dt))
