"""Per-source-line warp-stall samples from an ncu report (needs -lineinfo builds).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep <kernel-regex> [--top 30]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[h]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
per = defaultdict(float)
src = {}
why = defaultdict(lambda: defaultdict(float))
for r in rows[h + 1:]:
    if len(r) != len(hdr) or not r[0]:
        continue
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    per[r[0]] += v
    src[r[0]] = r[1]
    for i in stall_cols:
        try:
            why[r[0]][hdr[i][6:]] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(per.values()) or 1.0
for line, v in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
    w = sorted(why[line].items(), key=lambda kv: -kv[1])[:2]
    print(f"{100 * v / tot:5.1f}% L{line:>4} {src[line].strip()[:80]:80s} " + " ".join(f"{k}:{int(x)}" for k, x in w))
