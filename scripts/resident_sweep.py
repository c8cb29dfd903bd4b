"""Resident small-mesh EXACT path (GPU): device time per step of cfg1 / cfg2
for several CTA counts, against the two-launch EXACT path, with a bitwise
comparison of the fields.  python scripts/resident_sweep.py [cfg1|cfg2] [steps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
prob = bench.make_problem(cfg, 0, 64)
scratch = torch.empty(2 * 126 * 2**20, dtype=torch.uint8, device="cuda")
ref = None
for tun in ({"exact_resident": 1}, {}, {"resident_sync": 1}, {"resident_ctas": 148}, {"resident_ctas": 222},
            {"resident_ctas": 296}, {"resident_ctas": 444}, {"resident_ctas": 592}):
    kw = prob.engine_kwargs()
    kw["precision"] = 64
    try:
        eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="exact", tuning=tun, **kw)
    except Exception as ex:  # noqa: BLE001
        print(json.dumps({"tuning": tun, "error": str(ex)}), flush=True)
        continue
    dt = 0.9 * eng.critical_dt(37.0)
    st = eng.initial_state(37.0)
    L, h = eng._L, eng._h
    T = st.temperatures
    res = []
    for rep in range(3):
        N.check(L.fh_set_temperature(h, N.ptr(T), T.size, 0, 0.0))
        scratch.fill_(rep)
        torch.cuda.synchronize()
        r, el = N.FhReport(), C.c_float()
        N.check(L.fh_step_timed(h, steps, dt, C.byref(r), C.byref(el)))
        res.append(el.value / steps * 1e3)
    Tf = eng.temperature()
    if ref is None:
        ref = Tf
    lay = eng.layout()
    print(json.dumps({"cfg": cfg, "tuning": tun, "us_per_step": [round(x, 3) for x in res],
                      "resident_ctas": lay["resident_ctas"], "threads": lay["resident_threads"],
                      "bitwise_equal_to_two_launch": bool(np.array_equal(Tf, ref))}), flush=True)
    del eng
