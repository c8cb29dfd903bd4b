"""Group the SASS of an ncu report into equal-execution-count blocks (hot regions)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
ti = sum(f(r, "Instructions Executed") for r in data)
ts = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
blocks = []
for r in data:
    c = f(r, "Instructions Executed")
    if blocks and blocks[-1][0] == c:
        blocks[-1][1].append(r[1].strip()); blocks[-1][2] += f(r, "Warp Stall Sampling (All Samples)")
    else:
        blocks.append([c, [r[1].strip()], f(r, "Warp Stall Sampling (All Samples)")])
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for c, ins, st in blocks:
    if c * len(ins) / ti > thr or st / ts > thr:
        ops = {}
        for s in ins:
            op = s.split()[1] if s.startswith('@') else s.split()[0]
            op = op.split('.')[0]; ops[op] = ops.get(op, 0) + 1
        print(f"{c/1e6:6.2f}M x {len(ins):3d} = inst {100*c*len(ins)/ti:5.1f}% stall {100*st/ts:5.1f}%  "
              f"{dict(sorted(ops.items(), key=lambda x: -x[1])[:9])}")
