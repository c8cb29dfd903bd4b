"""Tuning sweep of the fused step on one workload (GPU): tile size x
accumulation mode x TMA ring depth (fh_options tuning knobs; --tuning adds
more, e.g. --tuning first_touch=1,hex_color=1).  The mesh is built once; each
variant gets its own engine.  Prints one line per variant.  Mode ids are the
kernel's (0 ranked, 1 corner phases, 3 colour phases, 4 shared atomics, 5 two-row
corner phases); mode -1 = the engine default."""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1909_05098_b200 as fh  # noqa: E402
from paper_1909_05098_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--divisions", type=int, default=0)
ap.add_argument("--precision", type=int, default=0)
ap.add_argument("--parts", default="768,1024")
ap.add_argument("--modes", default="1,2")
ap.add_argument("--stages", default="2,3")
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--tuning", default="")
ap.add_argument("--bench-layout", action="store_true", help="bench.py's domains (8; cfg4: z-slabs)")
ap.add_argument("--check", action="store_true", help="compare each variant's field with the first one's")
args = ap.parse_args()

prob = bench.make_problem(args.config, args.divisions, args.precision)
peak, _ = bench.peaks()
t0 = time.time()
ref = None
for pn in [int(x) for x in args.parts.split(",")]:
    for mode in [int(x) for x in args.modes.split(",")]:
        for stg in [int(x) for x in args.stages.split(",")]:
            tuning = {"tile_mode": mode + 1, "tile_stages": stg}
            tuning.update({k: int(v) for k, v in (kv.split("=") for kv in args.tuning.split(",") if kv)})
            if mode == 4:
                tuning["allow_nondeterministic"] = 1
            lay_kw = dict(n_domains=8, slab_axis=2 if args.config == "cfg4" else -1) if args.bench_layout else {}
            eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="tiled", part_nodes=pn,
                                    tuning=tuning, **lay_kw, **prob.engine_kwargs())
            dt = 0.9 * eng.critical_dt(37.0)
            if args.config == "cfg4":
                eng.set_sources(bench.run_sources(prob, dt))
            st = eng.initial_state(37.0)
            L, h = eng._L, eng._h
            N.check(L.fh_set_temperature(h, N.ptr(st.temperatures), st.temperatures.size, 0, 0.0))
            rep = N.FhReport()
            el = C.c_float()
            N.check(L.fh_step_timed(h, 5, dt, C.byref(rep), C.byref(el)))
            N.check(L.fh_step_timed(h, args.steps, dt, C.byref(rep), C.byref(el)))
            ms = el.value / args.steps
            lay = eng.layout()
            frac = lay["canonical_bytes"] / (ms / 1e3) / 1e9 / peak
            rec = {"part_nodes": pn, "mode": mode, "stages": stg, "ms": round(ms, 4),
                   "frac": round(frac, 4), "parts": lay["n_parts"], "slots": lay["n_slots"]}
            if args.check:
                T = eng.temperature()
                if ref is None:
                    ref = T
                rec["max_rel_diff_vs_first"] = float(np.max(np.abs(T - ref) / np.maximum(np.abs(ref), 1e-30)))
                rec["max_abs_diff_vs_first"] = float(np.max(np.abs(T - ref)))
            print(json.dumps(rec), flush=True)
            del eng
print("sweep wall", time.time() - t0)
