"""Per-block stall reasons from an ncu report's SASS page (hot regions only)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
ts = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
blocks = []
for r in data:
    c = f(r, "Instructions Executed")
    if not blocks or blocks[-1]["c"] != c:
        blocks.append({"c": c, "n": 0, "ops": {}, "st": {k: 0.0 for k in stall_cols}, "tot": 0.0, "first": r[1].strip()})
    b = blocks[-1]
    b["n"] += 1
    s = r[1].strip(); op = (s.split()[1] if s.startswith('@') else s.split()[0]).split('.')[0]
    b["ops"][op] = b["ops"].get(op, 0) + 1
    b["tot"] += f(r, "Warp Stall Sampling (All Samples)")
    for k in stall_cols: b["st"][k] += f(r, k)
for b in sorted(blocks, key=lambda b: -b["tot"])[:12]:
    top = sorted(b["st"].items(), key=lambda x: -x[1])[:4]
    print(f"{100*b['tot']/ts:5.1f}%  exec {b['c']/1e6:5.2f}M x{b['n']:3d}  "
          + ", ".join(f"{k[6:]} {100*v/max(b['tot'],1):.0f}%" for k, v in top)
          + "  | " + str(dict(sorted(b['ops'].items(), key=lambda x: -x[1])[:6])))
