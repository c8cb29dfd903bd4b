"""Same-box A/B of the tile-kind split on a mixed mesh (cfg5): device time per
step with tuning kind_split=1 (one launch) / 0 (split, default) and a bitwise comparison of the fields."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import _native as N  # noqa: E402

prob = bench.make_problem(sys.argv[1] if len(sys.argv) > 1 else "cfg5", 0, 32)
out = {}
for rep in range(2):
    for split in ("0", "1"):
        eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="tiled", n_domains=8,
                                tuning={"kind_split": 1 if split == "0" else 0}, **prob.engine_kwargs())
        dt = 0.9 * eng.critical_dt(37.0)
        st = eng.initial_state(37.0)
        L, h = eng._L, eng._h
        N.check(L.fh_set_temperature(h, N.ptr(st.temperatures), st.temperatures.size, 0, 0.0))
        r, el = N.FhReport(), C.c_float()
        N.check(L.fh_step_timed(h, 5, dt, C.byref(r), C.byref(el)))
        N.check(L.fh_step_timed(h, 100, dt, C.byref(r), C.byref(el)))
        out[split] = (el.value / 100, eng.temperature().copy(), eng.layout()["kernels_per_step"])
        del eng
    print(json.dumps({"rep": rep, "ms_nosplit": out["0"][0], "ms_split": out["1"][0], "launches": out["1"][2],
                      "bitwise_equal": bool(np.array_equal(out["0"][1], out["1"][1]))}), flush=True)
