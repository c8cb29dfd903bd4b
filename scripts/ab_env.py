"""Same-box A/B of an engine tuning knob (fh_options): python scripts/ab_env.py KNOB v0 v1 cfg...
Device ms per step for each value (2 reps) and a bitwise comparison of the fields."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import _native as N  # noqa: E402

var, vals, cfgs = sys.argv[1], sys.argv[2:4], sys.argv[4:]
for spec in cfgs:  # "cfg3" or "cfg3:64"
    cfg, _, prec = spec.partition(":")
    prob = bench.make_problem(cfg, 0, int(prec or 32))
    for rep in range(2):
        res = {}
        for v in vals:
            eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="tiled", n_domains=8,
                                    slab_axis=2 if cfg == "cfg4" else -1, tuning={var: int(v)},
                                    **prob.engine_kwargs())
            dt = 0.9 * eng.critical_dt(37.0)
            if cfg == "cfg4":
                eng.set_sources(bench.run_sources(prob, dt))
            st = eng.initial_state(37.0)
            L, h = eng._L, eng._h
            N.check(L.fh_set_temperature(h, N.ptr(st.temperatures), st.temperatures.size, 0, 0.0))
            r, el = N.FhReport(), C.c_float()
            N.check(L.fh_step_timed(h, 5, dt, C.byref(r), C.byref(el)))
            N.check(L.fh_step_timed(h, 100, dt, C.byref(r), C.byref(el)))
            res[v] = (el.value / 100, eng.temperature().copy())
            del eng
        print(json.dumps({"cfg": spec, "rep": rep, **{f"ms_{var}={v}": round(res[v][0], 4) for v in vals},
                          "bitwise_equal": bool(np.array_equal(res[vals[0]][1], res[vals[1]][1]))}), flush=True)
