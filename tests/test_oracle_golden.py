"""Pin the CPU oracle (oracle/fh_oracle.c) bit for bit to the reference.

The golden vectors were produced by running the reference package itself
(tests/golden/make_golden.py).  Every comparison here is np.array_equal:
the oracle restates the reference's floating-point operation order exactly.
"""

import numpy as np
import pytest

from golden_io import PRECOMP, RUNS, load, loads, material_ns, mesh_ns
from oracle import oracle as orc


@pytest.mark.parametrize("tag", PRECOMP)
def test_precompute_bitwise(tag):
    d = load(f"precompute_{tag}.npz")
    m = orc.OracleModel(mesh_ns(d), material_ns(d))
    pre = m.precompute()
    assert np.array_equal(pre["mat_data"], d["mat_data"])
    assert np.array_equal(pre["volumes"], d["volumes"])
    assert np.array_equal(pre["row_abs"], d["row_abs"])
    assert np.array_equal(pre["node_volumes"], d["node_volumes"])


def test_scatter_chunked_bitwise():
    d = load("scatter_tet12.npz")
    m = orc.OracleModel(mesh_ns(d), material_ns(load("precompute_mixed3.npz")))
    assert m.E > 2 * orc.CHUNK
    for r in range(3):
        out = m.scatter(d[f"kbar{r}"], d[f"T{r}"])
        assert np.array_equal(out, d[f"inflow{r}"])


def test_scatter_thread_count_invariant():
    d = load("scatter_tet12.npz")
    m = orc.OracleModel(mesh_ns(d), material_ns(load("precompute_mixed3.npz")))
    outs = []
    for n in (1, 2, 3, 8):
        orc.set_threads(n)
        outs.append(m.scatter(d["kbar0"], d["T0"]))
    orc.set_threads(orc.max_threads())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_critical_dt_bitwise():
    d = load("critical_dt.npz")
    mat = material_ns(d)
    mat.is_constant = False
    for case in range(6):
        m = orc.OracleModel(mesh_ns(d, f"c{case}_"), mat)
        assert m.critical_dt(d[f"c{case}_T"]) == float(d[f"c{case}_dt"])


def test_instability_step_and_node():
    d = load("instability.npz")
    m = orc.OracleModel(mesh_ns(d), material_ns(d))
    m.initial_state(d["T0"])
    with pytest.raises(orc.InstabilityInOracle) as err:
        m.step(float(d["dt"]), 2000)
    assert err.value.step == int(d["fail_step"])
    assert err.value.node == int(d["fail_node"])
    assert np.array_equal(m.T, d["T_fail"])


@pytest.mark.parametrize("tag", RUNS)
def test_runs_bitwise(tag):
    d = load(f"run_{tag}.npz")
    m = orc.OracleModel(mesh_ns(d), material_ns(d), dirichlet=(d["dir_nodes"], d["dir_vals"]),
                        loads=loads(d), td_mode=bool(d["td_mode"]))
    if tag == "cfg1":
        assert m.critical_dt(np.full(m.V, 37.0)) == float(d["dt_critical"])
    T, hist = m.run(d["T0"], int(d["steps"]), float(d["dt"]), d["probes"], int(d["interval"]))
    assert np.array_equal(T, d["T_final"])
    assert np.array_equal(hist, d["probe_values"])


def test_cfg1_static_source_equals_loads():
    """Static per-node power through q_static == the reference's one-node heat loads."""
    d = load("run_cfg1.npz")
    m = orc.OracleModel(mesh_ns(d), material_ns(d), dirichlet=(d["dir_nodes"], d["dir_vals"]),
                        q_static=d["q_static"])
    T, _ = m.run(d["T0"], 200, float(d["dt"]))
    m2 = orc.OracleModel(mesh_ns(d), material_ns(d), dirichlet=(d["dir_nodes"], d["dir_vals"]),
                         loads=loads(d))
    T2, _ = m2.run(d["T0"], 200, float(d["dt"]))
    assert np.array_equal(T, T2)
