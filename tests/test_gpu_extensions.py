"""Extensions the BASELINE configs need but the reference lacks:
volumetric sources (static / moving Gaussian, RF), Robin convection,
T-dependent perfusion, per-element conductivity factor, material regions.

Their parity is unpinned by the reference (it has no such features); they
are checked against the oracle's restatement (oracle/fh_oracle.c) of the
extended step defined in DESIGN.md: EXACT mode bit for bit (static terms) or
to 1e-13 (time-dependent sources: CUDA exp vs glibc exp), TILED within the
north_star tolerances 1e-10 (fp64) / 1e-4 (fp32).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import configs  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def oracle_of(eng, prob_sources, kfactor=None, materials=None, element_region=None):
    rb = eng.boundary
    dyn = [s.as_dict() for s in prob_sources if not s.is_static]
    return orc.OracleModel(eng.mesh, materials or eng.material, dirichlet=(rb.dirichlet_nodes, rb.dirichlet_values),
                           loads=[(n, p, a, b) for n, p, a, b in rb.loads], q_static=eng.q_static, sources=dyn,
                           robin=eng.robin, kfactor=kfactor, elem_region=element_region, td_mode=eng.td_mode)


def run_pair(prob, steps, assembly, precision, **extra):
    kw = dict(td_mode=prob.td_mode, precision=precision, sources=prob.sources, robin=prob.robin,
              kfactor=prob.kfactor, **extra)
    eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly=assembly, **kw)
    dt = 0.9 * eng.critical_dt(37.0)
    res = eng.run(37.0, steps=steps, dt=dt)
    ora = oracle_of(eng, prob.sources, kfactor=prob.kfactor, materials=extra.get("materials"),
                    element_region=extra.get("element_region"))
    T_ref, _ = ora.run(37.0, steps, dt)
    return res.state.temperatures, T_ref, eng, ora, dt


def test_cfg3_family_exact_bitwise():
    prob = configs.cfg3(divisions=8, precision=64)
    T, T_ref, eng, ora, dt = run_pair(prob, 60, "exact", 64)
    assert eng.robin is not None and len(eng.robin[0]) > 0
    assert np.array_equal(T, T_ref)
    assert eng.critical_dt(37.0) == ora.critical_dt(np.full(prob.mesh.n_nodes, 37.0))


@pytest.mark.parametrize("prec", [64, 32])
def test_cfg3_family_tiled(prec):
    prob = configs.cfg3(divisions=10, precision=prec)
    T, T_ref, *_ = run_pair(prob, 80, "tiled", prec, part_nodes=300)
    assert rel(T, T_ref) <= (1e-10 if prec == 64 else 1e-4)


def moving_cfg4(div):
    prob = configs.cfg4(divisions=div)
    a, b = (np.asarray(v) for v in prob.notes["path"])
    prob.sources = (fh.GaussianSource(amp=5e7, sigma=0.01, x0=tuple(a), vel=tuple((b - a) / 40.0), t0=0.0),)
    return prob


def test_cfg4_family_exact_moving_source():
    prob = moving_cfg4(10)
    T, T_ref, *_ = run_pair(prob, 50, "exact", 64)
    assert rel(T, T_ref) <= 1e-13
    assert T.max() > 37.5  # the source did heat


@pytest.mark.parametrize("prec", [64, 32])
def test_cfg4_family_tiled(prec):
    prob = moving_cfg4(12)
    T, T_ref, *_ = run_pair(prob, 60, "tiled", prec, part_nodes=256, n_domains=8, slab_axis=2)
    assert rel(T, T_ref) <= (1e-10 if prec == 64 else 1e-4)


def regions_problem(div=10):
    mesh = fh.generate_cube_mesh("hex", div, 0.1)
    centroids = mesh.nodes[mesh.hexes].mean(axis=1)
    region = (np.linalg.norm(centroids - 0.05, axis=1) < 0.02).astype(np.int32)
    healthy = configs.pennes_td(k0=0.5, wb0=0.6e-3 * 1050.0)
    tumour = configs.pennes_td(k0=0.55, wb0=0.2e-3 * 1050.0)
    src = fh.RFSource(power=0.01, tip=(0.05, 0.05, 0.05), cap=2e5)
    bnd = fh.BoundarySpec(dirichlet=tuple((f, 37.0) for f in configs.FACES))
    return mesh, [healthy, tumour], region, src, bnd


@pytest.mark.parametrize("assembly,prec,tol", [("exact", 64, 0.0), ("tiled", 64, 1e-10), ("tiled", 32, 1e-4)])
def test_regions_rf_source(assembly, prec, tol):
    mesh, mats, region, src, bnd = regions_problem()
    eng = fh.ExplicitEngine(mesh, mats[0], bnd, materials=mats, element_region=region, sources=(src,),
                            assembly=assembly, precision=prec, part_nodes=300)
    dt = 0.9 * eng.critical_dt(37.0)
    res = eng.run(37.0, steps=50, dt=dt)
    ora = oracle_of(eng, (src,), materials=mats, element_region=region)
    T_ref, _ = ora.run(37.0, 50, dt)
    if tol == 0.0:
        assert np.array_equal(res.state.temperatures, T_ref)
    else:
        assert rel(res.state.temperatures, T_ref) <= tol


def test_td_perfusion_fixed_point_bitwise():
    """T == T_a stays a bitwise fixed point with T-dependent perfusion too."""
    mesh = fh.generate_cube_mesh("tet", 4, 0.05)
    mat = configs.pennes_td()
    mat = mat.with_updates(metabolic_rate=0.0)
    for assembly, prec in (("exact", 64), ("tiled", 64), ("tiled", 32)):
        eng = fh.ExplicitEngine(mesh, mat, assembly=assembly, precision=prec, part_nodes=64)
        st = eng.initial_state(37.0)
        for _ in range(10):
            eng.step(st, 1.0)
        assert np.all(st.temperatures == 37.0), assembly


@pytest.mark.parametrize("assembly,prec,tol", [("exact", 64, 0.0), ("tiled", 64, 1e-10), ("tiled", 32, 1e-4)])
def test_cfg5_family_mixed_voxel_regions(assembly, prec, tol):
    """Voxel ellipsoid (hexes + split boundary tets), two regions, RF source."""
    prob = configs.cfg5(scale=16)
    assert prob.mesh.tets.shape[0] > 0 and prob.element_region.sum() > 0
    eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly=assembly, precision=prec,
                            part_nodes=400, **{k: v for k, v in prob.engine_kwargs().items() if k != "precision"})
    dt = 0.9 * eng.critical_dt(37.0)
    res = eng.run(37.0, steps=40, dt=dt)
    ora = oracle_of(eng, prob.sources, materials=prob.materials, element_region=prob.element_region)
    T_ref, _ = ora.run(37.0, 40, dt)
    assert T_ref.max() > 37.01
    if tol == 0.0:
        assert np.array_equal(res.state.temperatures, T_ref)
    else:
        assert rel(res.state.temperatures, T_ref) <= tol


def clamped_material():
    """Two-knot laws whose knots lie INSIDE the temperatures of the run: part
    of the field is interpolated, part is clamped (np.interp semantics)."""
    from paper_1909_05098_b200.material import linear_law, make_constant

    return fh.TissueMaterial(
        density=make_constant(1060.0), specific_heat=linear_law(3600.0, -0.0005, 37.0, t_lo=36.6, t_hi=37.8),
        conductivity=linear_law(0.5, 0.02, 37.0, t_lo=36.8, t_hi=37.6), perfusion_rate=0.525,
        blood_specific_heat=3640.0, arterial_temperature=37.0, metabolic_rate=420.0,
        perfusion_curve=linear_law(0.525, configs.PERFUSION_SLOPE, 37.0, t_lo=36.9, t_hi=37.4))


@pytest.mark.parametrize("kind", ["hex", "tet", "mixed"])
@pytest.mark.parametrize("prec,tol", [(64, 1e-10), (32, 1e-4)])
def test_tiled_two_knot_laws_clamp_outside_their_knots(kind, prec, tol):
    """The fused step stages T alone for two-knot laws and takes k(mean T) per
    slot; tiles holding a temperature outside the conductivity knots must fall
    back to per-corner clamped interpolation (fh_tiled.cu kbar_lin).  A field
    that straddles both knots, in tiles of all three kinds, against the oracle;
    the LEAN loops and the general kernel agree bit for bit."""
    if kind == "mixed":
        mesh = configs.cfg5(scale=16).mesh
    else:
        mesh = fh.jittered_cube_mesh(kind, 10, 0.1, 0.15, seed=5)
    mat = clamped_material()
    rng = np.random.default_rng(8)
    # a smooth ramp from 36.2 to 38.4 C across x plus noise: some tiles entirely
    # between the knots, some entirely outside, some straddling them
    x = mesh.nodes[:, 0]
    T0 = 36.2 + 2.2 * (x - x.min()) / (x.max() - x.min()) + rng.uniform(-0.05, 0.05, mesh.n_nodes)
    fields = []
    for lean in (0, 1):
        eng = fh.ExplicitEngine(mesh, mat, assembly="tiled", precision=prec, part_nodes=200,
                                tuning={"lean_kernels": lean})
        dt = 0.8 * eng.critical_dt(T0)
        fields.append(eng.run(T0, steps=40, dt=dt).state.temperatures)
    assert np.array_equal(fields[0], fields[1])
    ora = orc.OracleModel(mesh, mat, td_mode=True)
    T_ref, _ = ora.run(T0, 40, dt)
    assert np.abs(T_ref - T0).max() > 1e-3
    assert float(np.abs(fields[0] - T_ref).max() / np.abs(T_ref - T0).max()) <= tol
    assert rel(fields[0], T_ref) <= tol


def test_hex_mesh_with_regions_runs_lean_tiles_bitwise():
    """A hex-only mesh with two materials: the tiles whose elements all belong
    to material 0 run the LEAN 2 batch loop beside the general kernel's tiles
    (two launches per step); the field equals the general kernel's bit for bit."""
    mesh, mats, region, src, bnd = regions_problem(div=14)
    fields = []
    for lean in (0, 1):
        eng = fh.ExplicitEngine(mesh, mats[0], bnd, materials=mats, element_region=region, sources=(src,),
                                assembly="tiled", precision=32, part_nodes=200, tuning={"lean_kernels": lean})
        assert eng.layout()["kernels_per_step"] == (2 if lean == 0 else 1)
        dt = 0.9 * eng.critical_dt(37.0)
        fields.append(eng.run(37.0, steps=40, dt=dt).state.temperatures)
    assert np.array_equal(fields[0], fields[1])
    assert fields[0].max() > 37.001
