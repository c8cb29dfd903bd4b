"""Schedule invariance of the step kernels -- the race evidence this GPU pool
allows (compute-sanitizer is closed on it; scripts/build_variant.sh checked
builds the device bounds checks).

Every value a kernel computes has a fixed operation order, so the fields must
not change with anything that only moves work in time:
* TILED: the TMA ring depth (1-4 batches in flight: when each stage buffer is
  refilled relative to the threads still reading it) and the tile launch order
  (RCB order vs longest tiles first);
* resident EXACT: the number of CTAs (which nodes share a CTA, a barrier and
  the staging loads).
A missing barrier or an early refill would show up as a field difference that
depends on timing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import configs  # noqa: E402


def problem(kind):
    if kind == "hex":
        return configs.cfg4(divisions=14)
    if kind == "tet":
        return configs.cfg3(divisions=10, precision=32)
    return configs.cfg5(scale=16)


def field(prob, prec, **kw):
    k = prob.engine_kwargs()
    k["precision"] = prec
    eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="tiled", part_nodes=300, **k, **kw)
    dt = 0.9 * eng.critical_dt(37.0)
    T0 = 37.0 + np.sin(60 * prob.mesh.nodes[:, 0]) * np.cos(50 * prob.mesh.nodes[:, 2])
    return eng.run(T0, steps=40, dt=dt).state.temperatures


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("kind", ["hex", "tet", "mixed"])
def test_tiled_ring_depth_and_launch_order_invariant(kind, prec):
    prob = problem(kind)
    ref = field(prob, prec)
    assert np.isfinite(ref).all() and np.abs(ref - 37.0).max() > 0.01
    # (lean_kernels=1: the general kernel instead of the LEAN 1 / 2 / 3 batch loops -- same bits)
    for tuning in ({"tile_stages": 1}, {"tile_stages": 3}, {"tile_stages": 4}, {"launch_order": 1},
                   {"launch_order": 2}, {"lean_kernels": 1}):
        assert np.array_equal(field(prob, prec, tuning=tuning), ref), tuning


def test_resident_cta_count_invariant():
    prob = configs.cfg2(divisions=14)
    out = []
    for ctas in (0, 37, 96, 296):
        eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, tuning={"resident_ctas": ctas},
                                **prob.engine_kwargs())
        assert eng.layout()["resident_ctas"] > 0
        out.append(eng.run(37.0, steps=300, dt=0.9 * eng.critical_dt(37.0)).state.temperatures)
    for T in out[1:]:
        assert np.array_equal(T, out[0])
