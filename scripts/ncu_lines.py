"""Instructions executed and stall samples per CUDA source line of a step-kernel
capture (cuda,sass correlated view; needs -lineinfo).  Usage: ncu_lines.py rep [n]"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]; ix = {}
for i, h in enumerate(hdr):
    ix.setdefault(h, i)
line_src, stats, cur, fname = {}, {}, None, ""
for r in rows[hi + 1:]:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]; cur = None
        continue
    if r[0] in ("Function Name", "Line No", "File Name"):
        continue
    if r[0] not in ("", "-"):
        cur = (fname, int(r[0])); line_src[cur] = r[1]
    if cur is None:
        continue
    try:
        ins = float(r[ix["Instructions Executed"]]); smp = float(r[ix["Warp Stall Sampling (All Samples)"]])
    except (ValueError, IndexError):
        continue
    s = stats.setdefault(cur, [0.0, 0.0]); s[0] += ins; s[1] += smp
ti = sum(v[0] for v in stats.values()) or 1; ts = sum(v[1] for v in stats.values()) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total {ti/1e6:.1f}M warp-instr")
for ln, (ins, smp) in sorted(stats.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100*ins/ti:5.1f}% instr {100*smp/ts:5.1f}% stalls  {ln[0][:12]}:{ln[1]:<4d} {line_src.get(ln, '').strip()[:90]}")
