"""Small runs of every step kernel for compute-sanitizer (racecheck /
synccheck / memcheck): TILED hex (two-row corner phases) and tet (colour
phases, 4 rows) fp32 + fp64, mixed hex+tet with regions, the resident EXACT
kernel, the two-launch EXACT path and the ATOMIC assembly."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import configs  # noqa: E402

steps = 3
hexm = configs.cfg4(divisions=10)
tet = configs.cfg3(divisions=8, precision=32)
mixed = configs.cfg5(scale=20)
for prob, asm, prec, extra in ((hexm, "tiled", 32, {}), (hexm, "tiled", 64, {}), (tet, "tiled", 32, {}),
                               (tet, "tiled", 64, {}), (mixed, "tiled", 32, {}), (hexm, "atomic", 32, {}),
                               (hexm, "exact", 64, {}), (hexm, "exact", 64, {"tuning": {"exact_resident": 1}})):
    kw = prob.engine_kwargs()
    kw["precision"] = prec
    eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly=asm,
                            part_nodes=0 if asm == "exact" else 200, **kw, **extra)
    dt = 0.9 * eng.critical_dt(37.0)
    res = eng.run(37.0, steps=steps, dt=dt)
    print(prob.name, asm, prec, extra, eng.layout()["kernels_per_step"], float(res.state.temperatures.max()), flush=True)
