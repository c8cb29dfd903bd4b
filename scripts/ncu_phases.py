"""Split a step-kernel ncu capture (SASS page) into its phases by the
BAR.SYNC layout: staging (before the first batch), batches, node update.
Usage: ncu_phases.py report.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]; ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
blocks = []
for r in data:
    c = f(r, "Instructions Executed")
    if not blocks or blocks[-1]["c"] != c:
        blocks.append({"c": c, "rows": []})
    blocks[-1]["rows"].append(r)
st = lambda b: sum(f(r, "Warp Stall Sampling (All Samples)") for r in b["rows"])
w = lambda b: b["c"] * len(b["rows"])
tot_i = sum(w(b) for b in blocks); tot_s = sum(st(b) for b in blocks)
# the batch loop: blocks containing SYNCS.PHASECHK (mbarrier wait) start it; the
# node update starts after the last BAR.SYNC that follows the loop
first_wait = next(k for k, b in enumerate(blocks) if any("SYNCS.PHASECHK" in r[1] for r in b["rows"]))
loop_exec = blocks[first_wait]["c"]
last_loop = max(k for k, b in enumerate(blocks) if b["c"] >= 0.5 * loop_exec and k >= first_wait)
phases = {"staging": blocks[:first_wait], "batches": blocks[first_wait:last_loop + 1], "node update": blocks[last_loop + 1:]}
print(f"total {tot_i/1e6:.1f}M warp-instr")
for name, bs in phases.items():
    print(f"{name:12s} instr {sum(w(b) for b in bs)/1e6:6.1f}M ({100*sum(w(b) for b in bs)/tot_i:4.1f}%)  stall samples {100*sum(st(b) for b in bs)/tot_s:4.1f}%")
