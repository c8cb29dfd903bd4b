"""Per-rank device working set and halo overhead of the multi-GPU layout at
W = 1/2/4/8 (host bookkeeping only, no GPU): python scripts/plan_scaling.py cfg4 [cfg5]
Writes profiles/r2_plan_scaling.json.  The tile decomposition does not depend
on W, so the slot duplication (slots per element) is the same for every W and
the only multi-GPU cost is the halo temperature exchange (n_recv values per
rank per step)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1909_05098_b200.dist import Plan  # noqa: E402

out = {}
for cfg in sys.argv[1:] or ["cfg4"]:
    prob = bench.make_problem(cfg)
    E = prob.mesh.n_elements
    rows = []
    for W in (1, 2, 4, 8):
        t0 = time.time()
        ranks = []
        for r in range(W):
            p = Plan(prob.mesh, prob.material, prob.boundary, world=W, rank=r, n_domains=8,
                     slab_axis=2 if cfg == "cfg4" else -1, precision=32, robin=prob.robin)
            ranks.append({k: p.info[k] for k in ("rank_real_slots", "rank_local_nodes", "rank_owned_nodes",
                                                 "rank_step_bytes", "rank_device_bytes", "n_send", "n_recv",
                                                 "n_peers")})
            del p
        rows.append({"W": W, "slots_per_element": sum(x["rank_real_slots"] for x in ranks) / E,
                     "max_rank_device_bytes": max(x["rank_device_bytes"] for x in ranks),
                     "max_rank_step_bytes": max(x["rank_step_bytes"] for x in ranks),
                     "max_halo_recv_values": max(x["n_recv"] for x in ranks),
                     "halo_bytes_per_step_fp32": 4 * max(x["n_recv"] for x in ranks),
                     "ranks": ranks, "plan_s": round(time.time() - t0, 1)})
        print(cfg, {k: v for k, v in rows[-1].items() if k != "ranks"}, flush=True)
    out[cfg] = {"elements": E, "nodes": prob.mesh.n_nodes, "rows": rows}
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "r2_plan_scaling.json"), "w") as f:
    json.dump(out, f, indent=1)
