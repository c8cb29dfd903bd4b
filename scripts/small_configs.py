"""Time the latency-bound small configs (cfg1, cfg2) through the public API:
ms/step of a full `run` (device-resident steps) in EXACT fp64 and TILED
fp64/fp32 modes, plus parity of TILED against the EXACT field."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import configs  # noqa: E402

for name in ("cfg1", "cfg2"):
    prob = getattr(configs, name)()
    ref = None
    for assembly, prec in (("exact", 64), ("tiled", 64), ("tiled", 32)):
        eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly=assembly, precision=prec,
                                td_mode=prob.td_mode, sources=prob.sources)
        dt = 0.9 * eng.critical_dt(37.0)
        eng.run(37.0, steps=20, dt=dt)  # warm-up
        t0 = time.perf_counter()
        res = eng.run(37.0, steps=prob.steps, dt=dt)
        el = time.perf_counter() - t0
        T = res.state.temperatures
        if ref is None:
            ref = T
        line = {"config": name, "assembly": assembly, "precision": prec, "steps": prob.steps,
                "ms_per_step": 1e3 * el / prob.steps, "elem_steps_per_s": prob.mesh.n_elements * prob.steps / el,
                "centre_T": float(T[prob.mesh.node_sets["center"][0]]),
                "rel_vs_exact": float(np.abs(T - ref).max() / np.abs(ref).max())}
        print(json.dumps(line), flush=True)
