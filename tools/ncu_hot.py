"""Per-loop breakdown of an ncu source page (SASS): groups instructions by
execution count and prints instruction / stall-sample shares with the opcode
mix.  python tools/ncu_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = rows[2:]
ia, isrc, iss = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot_i = sum(int(r[ia]) for r in data if r[ia].isdigit())
tot_s = sum(int(r[iss]) for r in data if r[iss].isdigit())
g = defaultdict(lambda: [0, 0, Counter()])
for r in data:
    if not r[ia].isdigit():
        continue
    c = int(r[ia])
    g[c][0] += 1
    g[c][1] += int(r[iss]) if r[iss].isdigit() else 0
    op = r[isrc].strip().split()
    op = op[1] if op[0].startswith("@") else op[0]
    g[c][2][op.split(".")[0]] += 1
print(f"warp instructions {tot_i:.4g}, stall samples {tot_s}")
for c, (k, smp, ops) in sorted(g.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"exec {c:>9} x {k:>5} instr  inst {100 * c * k / tot_i:5.1f}%  samples {100 * smp / tot_s:5.1f}%  ",
          ops.most_common(7))
