"""ATOMIC assembly (csrc/fh_atomic.cu): element loads scattered with
warp-aggregated global atomics, then a node kernel -- the alternative
north_star (iii) names, kept for the measured comparison with the TILED
gather.  Its per-node summation order follows atomic
arrival, so it is checked against the oracle within the north_star
tolerances only (rel 1e-10 fp64, 1e-4 fp32, normalised by max |T| and by the
rise max |T - T0|)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import configs  # noqa: E402
from oracle import oracle as orc  # noqa: E402

TOL = {64: 1e-10, 32: 1e-4}


def oracle_run(eng, prob, steps, dt, srcs):
    rb = eng.boundary
    ora = orc.OracleModel(prob.mesh, prob.material, dirichlet=(rb.dirichlet_nodes, rb.dirichlet_values),
                          sources=[s.as_dict() for s in srcs], robin=eng.robin, kfactor=prob.kfactor,
                          td_mode=True)
    T, _ = ora.run(37.0, steps, dt)
    return T


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("cfg", ["cfg4", "cfg3"])
def test_atomic_vs_oracle(cfg, prec):
    if cfg == "cfg4":
        prob = configs.cfg4(divisions=12)
        a, b = (np.asarray(v) for v in prob.notes["path"])
        srcs = (fh.GaussianSource(amp=5e6, sigma=0.01, x0=tuple(a), vel=tuple((b - a) / 3000.0), t0=0.0),)
    else:
        prob = configs.cfg3(divisions=9, precision=prec)
        srcs = prob.sources
    kw = dict(td_mode=True, precision=prec, sources=srcs, robin=prob.robin, kfactor=prob.kfactor)
    eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="atomic", **kw)
    lay = eng.layout()
    assert lay["kernels_per_step"] == 2
    dt = 0.9 * eng.critical_dt(37.0)
    res = eng.run(37.0, steps=60, dt=dt)
    T_ref = oracle_run(eng, prob, 60, dt, srcs)
    d = np.abs(res.state.temperatures - T_ref).max()
    assert T_ref.max() > 37.01
    assert d / np.abs(T_ref).max() <= TOL[prec]
    assert d / np.abs(T_ref - 37.0).max() <= 10 * TOL[prec]


def test_atomic_refuses_what_it_does_not_cover():
    mesh = fh.generate_cube_mesh("hex", 4, 0.1)
    with pytest.raises(fh.ConfigError):  # TI runs freeze kbar: TILED / EXACT only
        fh.ExplicitEngine(mesh, configs.pennes_constant(), assembly="atomic", precision=32, td_mode=False)
    region = np.zeros(mesh.n_elements, np.int32)
    region[:5] = 1
    with pytest.raises(fh.ConfigError):
        fh.ExplicitEngine(mesh, configs.pennes_td(), assembly="atomic", precision=32,
                          materials=[configs.pennes_td(), configs.pennes_td(k0=0.6)], element_region=region)
