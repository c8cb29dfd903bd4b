"""Parity at the BASELINE sizes and step counts against the CPU oracle.

north_star: "nodal temperature histories must match the reference's CPU
implementation on identical seeded meshes within rel. 1e-10 (fp64) / 1e-4
(fp32) after N steps".  Here N is each config's BASELINE step count and the
mesh is the full BASELINE mesh:

  cfg3  6.0 M jittered tets, TD, 3 Gaussians, Robin   fp32 + fp64  500 steps
  cfg4  16.8 M hexes, TD, k-field, moving Gaussian    fp32         200 steps
  cfg5  25.2 M hex + tet organ, 2 regions, RF source  fp32         500 steps
  cfg2  20^3 hexes, TD incl. perfusion, Gaussian      fp32 + fp64 2000 steps
  cfg1  20^3 hexes vs the REFERENCE's own golden run  fp32 + fp64 1000 steps

The oracle (oracle/fh_oracle.c: the reference's operation order, O(E)
memory, OpenMP over the host cores) runs the same problem in fp64 on the GPU
box's CPU.  Both the final field and the probe histories (recorded every
step by the TILED engine, solver.py:458-460,486-487) are compared, each with
two norms:

  rel_T    = max|T - T_ref| / max|T_ref|          (north_star's relative error)
  rel_rise = max|T - T_ref| / max|T_ref - T0|     (relative to the computed change)

Both norms are gated at the north_star tolerance, 1e-10 (fp64) / 1e-4
(fp32): the rise-normalised norm is the stricter one (the rise is 3-40x
smaller than max |T| over these runs).  With FH_PARITY_JSON set, every measured norm is appended to
that file (profiles/r2_parity_fullsize.json holds the GPU box's numbers).
"""

from __future__ import annotations

import json
import os
import time

import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import configs  # noqa: E402
from paper_1909_05098_b200.sources import robin_lumps  # noqa: E402
from oracle import oracle as orc  # noqa: E402

TOL_T = {64: 1e-10, 32: 1e-4}
TOL_RISE = {64: 1e-10, 32: 1e-4}
T0 = 37.0


def norms(T, T_ref):
    d = float(np.abs(T - T_ref).max())
    return {"max_abs": d, "rel_T": d / float(np.abs(T_ref).max()),
            "rel_rise": d / max(float(np.abs(T_ref - T0).max()), 1e-300)}


def record(entry):
    path = os.environ.get("FH_PARITY_JSON")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(entry) + "\n")


def probe_nodes(prob, n_random=24, seed=11):
    """Seeded interior nodes plus the node nearest each source position."""
    mesh = prob.mesh
    rng = np.random.default_rng(seed)
    picks = list(rng.choice(mesh.n_nodes, n_random, replace=False))
    pts = []
    for s in prob.sources:
        d = s.as_dict()
        pts.append(np.asarray(d["x0"]))
    if prob.name == "cfg4":
        a, b = (np.asarray(v) for v in prob.notes["path"])
        pts += [a, 0.5 * (a + b), b]
    for p in pts:
        picks.append(int(np.argmin(((mesh.nodes - p) ** 2).sum(axis=1))))
    return np.unique(np.asarray(picks, dtype=np.int64))


def problem(name, precision):
    if name == "cfg3":
        prob = configs.cfg3(precision=precision)
    elif name == "cfg2":
        prob = configs.cfg2(precision=precision)
    else:
        prob = getattr(configs, name)()
    prob.precision = precision
    return prob


def with_dt(prob, dt):
    """cfg4: the moving source covers its seeded segment over the run (bench.py)."""
    if prob.name == "cfg4":
        a, b = (np.asarray(v) for v in prob.notes["path"])
        prob.sources = (fh.GaussianSource(amp=5.0e6, sigma=0.005, x0=tuple(a),
                                          vel=tuple((b - a) / (prob.steps * dt)), t0=0.0),)
    return prob


_ORACLE = {}


def oracle_run(name, prob, eng, dt, probes):
    """One fp64 oracle run per config, shared by the precisions."""
    if name in _ORACLE:
        return _ORACLE[name]
    rb = eng.boundary
    robin = robin_lumps(prob.mesh, prob.robin[0], exclude=rb.dirichlet_nodes) if prob.robin else None
    dyn = [s.as_dict() for s in prob.sources if not s.is_static]
    ora = orc.OracleModel(prob.mesh, prob.materials or prob.material,
                          dirichlet=(rb.dirichlet_nodes, rb.dirichlet_values), q_static=eng.q_static, sources=dyn,
                          robin=robin, kfactor=prob.kfactor, elem_region=prob.element_region, td_mode=prob.td_mode)
    t = time.perf_counter()
    T_ref, hist = ora.run(T0, prob.steps, dt, probes=probes, interval=1)
    out = (T_ref, hist, time.perf_counter() - t, orc.max_threads())
    del ora
    _ORACLE.clear()
    _ORACLE[name] = out
    return out


CASES = [("cfg2", 32), ("cfg2", 64), ("cfg3", 32), ("cfg3", 64), ("cfg4", 32), ("cfg5", 32)]


@pytest.mark.parametrize("name,prec", CASES, ids=[f"{n}-fp{p}" for n, p in CASES])
def test_tiled_full_size_vs_oracle(name, prec):
    prob = problem(name, prec)
    kw = prob.engine_kwargs()
    kw["precision"] = prec
    extra = dict(n_domains=8, slab_axis=2) if name == "cfg4" else {}  # the bench's tiles
    # dt from the reference-order Gershgorin bound (EXACT path of the engine)
    probe = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="tiled", **kw, **extra)
    dt = 0.9 * probe.critical_dt(T0)
    prob = with_dt(prob, dt)
    if name == "cfg4":
        probe.set_sources(prob.sources)
    eng = probe
    probes = probe_nodes(prob)
    t = time.perf_counter()
    res = eng.run(T0, steps=prob.steps, dt=dt, probes=probes)
    gpu_s = time.perf_counter() - t
    T_ref, hist_ref, cpu_s, threads = oracle_run(name, prob, eng, dt, probes)
    del eng, probe
    fin = norms(res.state.temperatures, T_ref)
    his = norms(res.probe_values, hist_ref)
    record({"config": name, "precision": prec, "steps": prob.steps, "elements": prob.mesh.n_elements,
            "nodes": prob.mesh.n_nodes, "dt": dt, "final": fin, "probes": his, "n_probes": int(probes.size),
            "max_rise_K": float(np.abs(T_ref - T0).max()), "oracle_s": cpu_s, "oracle_threads": threads,
            "gpu_run_s": gpu_s})
    assert res.probe_values.shape == hist_ref.shape
    assert np.abs(T_ref - T0).max() > 0.1  # the sources did heat
    for n in (fin, his):
        assert n["rel_T"] <= TOL_T[prec], (name, prec, n)
        assert n["rel_rise"] <= TOL_RISE[prec], (name, prec, n)


@pytest.mark.parametrize("prec", [64, 32])
def test_tiled_cfg1_full_run_vs_reference_golden(prec):
    """cfg1 (1000 steps, auto dt) against the reference's own run (golden)."""
    from test_gpu_parity import golden_problem
    from golden_io import material

    d = load("run_cfg1.npz")
    mesh, bnd = golden_problem(d)
    eng = fh.ExplicitEngine(mesh, material(d), bnd, assembly="tiled", precision=prec)
    res = eng.run(37.0, steps=int(d["steps"]), auto_dt_safety=0.9, probes=d["probes"])
    assert res.dt == float(d["dt"])
    fin = norms(res.state.temperatures, d["T_final"])
    his = norms(res.probe_values, d["probe_values"])
    record({"config": "cfg1-golden", "precision": prec, "steps": int(d["steps"]), "final": fin, "probes": his})
    for n in (fin, his):
        assert n["rel_T"] <= TOL_T[prec], n
        assert n["rel_rise"] <= TOL_RISE[prec], n


@pytest.fixture(scope="module", params=["cfg3", "cfg4", "cfg5"])
def big(request):
    return problem(request.param, 32)


def test_tiled_deterministic_full_size(big):
    kw = big.engine_kwargs()
    eng = fh.ExplicitEngine(big.mesh, big.material, big.boundary, assembly="tiled", **kw)
    dt = 0.9 * eng.critical_dt(T0)
    a = eng.run(T0, steps=20, dt=dt).state.temperatures
    b = eng.run(T0, steps=20, dt=dt).state.temperatures
    assert np.array_equal(a, b)


def test_arterial_fixed_point_full_size(big):
    import dataclasses

    mats = big.materials or [big.material]
    quiet = [dataclasses.replace(m, metabolic_rate=0.0) for m in mats]
    kw = dict(td_mode=big.td_mode, precision=32, kfactor=big.kfactor)
    if big.materials is not None:
        kw.update(materials=quiet, element_region=big.element_region)
    bnd = fh.BoundarySpec(dirichlet=big.boundary.dirichlet)
    eng = fh.ExplicitEngine(big.mesh, quiet[0], bnd, assembly="tiled", **kw)
    Ta = quiet[0].arterial_temperature
    dt = 0.9 * eng.critical_dt(Ta)
    T = eng.run(Ta, steps=20, dt=dt).state.temperatures
    assert np.all(T == Ta)
