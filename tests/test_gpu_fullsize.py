"""Parity at the full BASELINE sizes (cfg3 6.0 M tets, cfg4 16.8 M hexes,
cfg5 25.2 M mixed elements).

The CPU oracle cannot run these sizes inside a test, so parity is carried by
two things that do not depend on size:

* the EXACT engine: fp64, reference operation order, bitwise equal to the
  reference / oracle on every golden and family case (test_gpu_parity.py,
  test_gpu_extensions.py) and the same code at any size.  The fused TILED
  step must agree with it within the north_star tolerances (1e-10 fp64,
  1e-4 fp32) after 20 steps at full size;
* properties: two TILED runs are bitwise identical, and a uniform arterial
  field without heat sources stays bitwise at T_a (F = 0 exactly, k_b T and
  q_b round identically).
"""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import configs  # noqa: E402

STEPS = 20
TOL = {64: 1e-10, 32: 1e-4}


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.fixture(scope="module", params=["cfg3", "cfg4", "cfg5"])
def prob(request):
    return {"cfg3": configs.cfg3, "cfg4": configs.cfg4, "cfg5": configs.cfg5}[request.param]()


def engine(prob, assembly, precision, **over):
    kw = prob.engine_kwargs()
    kw.update(precision=precision, **over)
    return fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly=assembly, **kw)


def test_tiled_matches_exact_full_size(prob):
    exact = engine(prob, "exact", 64)
    dt = 0.9 * exact.critical_dt(37.0)
    T_ex = exact.run(37.0, steps=STEPS, dt=dt).state.temperatures
    del exact
    assert T_ex.max() > 37.0 + 1e-6  # the sources did heat
    for prec in (64, 32):
        tiled = engine(prob, "tiled", prec)
        T = tiled.run(37.0, steps=STEPS, dt=dt).state.temperatures
        assert rel(T, T_ex) <= TOL[prec], (prob.name, prec)
        if prec == 32:  # determinism: a second run is bitwise identical
            T2 = tiled.run(37.0, steps=STEPS, dt=dt).state.temperatures
            assert np.array_equal(T, T2)
        del tiled


def test_arterial_fixed_point_full_size(prob):
    mats = prob.materials or [prob.material]
    quiet = [dataclasses.replace(m, metabolic_rate=0.0) for m in mats]
    kw = dict(td_mode=prob.td_mode, precision=32, kfactor=prob.kfactor)
    if prob.materials is not None:
        kw.update(materials=quiet, element_region=prob.element_region)
    bnd = fh.BoundarySpec(dirichlet=prob.boundary.dirichlet)
    eng = fh.ExplicitEngine(prob.mesh, quiet[0], bnd, assembly="tiled", **kw)
    Ta = quiet[0].arterial_temperature
    dt = 0.9 * eng.critical_dt(Ta)
    T = eng.run(Ta, steps=STEPS, dt=dt).state.temperatures
    assert np.all(T == Ta)
