"""Measured selection of the assembly (north_star (iii)): device ms per step
of the TILED gather and the ATOMIC warp-aggregated scatter on the same
workload, same box, plus their field difference.  python scripts/atomic_vs_tiled.py cfg4 cfg3"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import _native as N  # noqa: E402

for cfg in sys.argv[1:] or ["cfg4"]:
    prob = bench.make_problem(cfg, 0, 32)
    res = {}
    for rep in range(2):
        for asm in ("tiled", "atomic"):
            kw = prob.engine_kwargs()
            eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly=asm, n_domains=8,
                                    slab_axis=2 if cfg == "cfg4" else -1, **kw)
            dt = 0.9 * eng.critical_dt(37.0)
            if cfg == "cfg4":
                eng.set_sources(bench.run_sources(prob, dt))
            st = eng.initial_state(37.0)
            L, h = eng._L, eng._h
            N.check(L.fh_set_temperature(h, N.ptr(st.temperatures), st.temperatures.size, 0, 0.0))
            r, el = N.FhReport(), C.c_float()
            N.check(L.fh_step_timed(h, 5, dt, C.byref(r), C.byref(el)))
            N.check(L.fh_step_timed(h, 100, dt, C.byref(r), C.byref(el)))
            res[asm] = (el.value / 100, eng.temperature().copy(), eng.layout())
            del eng
        T0, T1 = res["tiled"][1], res["atomic"][1]
        print(json.dumps({"cfg": cfg, "rep": rep, "ms_tiled": round(res["tiled"][0], 4),
                          "ms_atomic": round(res["atomic"][0], 4),
                          "frac_tiled": res["tiled"][2]["canonical_bytes"] / (res["tiled"][0] / 1e3) / 1e9 / bench.peaks()[0],
                          "frac_atomic": res["atomic"][2]["canonical_bytes"] / (res["atomic"][0] / 1e3) / 1e9 / bench.peaks()[0],
                          "max_rel_diff": float(np.abs(T1 - T0).max() / np.abs(T0).max()),
                          "max_rise_rel_diff": float(np.abs(T1 - T0).max() / np.abs(T0 - 37.0).max())}), flush=True)
