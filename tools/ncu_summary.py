"""Summarise an ncu report: per-kernel stall breakdown and hottest SASS lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-regex] [--top 25]
"""
import csv
import io
import subprocess
import sys


def page(rep, kernel, what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--launch-count", "1", "--print-source", what], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    kernel = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "k_"
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    rows = page(rep, kernel, "sass")
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = {hdr[i]: sum(f(r[i]) for r in data) for i in stall_cols}
    s = sum(tot.values()) or 1.0
    print("stall breakdown (% of samples):")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {k:28s} {100 * v / s:5.1f}")
    order = sorted(range(len(data)), key=lambda j: -f(data[j][si]))
    allsamp = sum(f(r[si]) for r in data) or 1.0
    print(f"top {top} SASS by samples (idx: instruction index in kernel):")
    for j in order[:top]:
        r = data[j]
        stalls = sorted(((hdr[i][6:], f(r[i])) for i in stall_cols), key=lambda kv: -kv[1])[:3]
        print(f"  {100 * f(r[si]) / allsamp:5.1f}%  [{j:4d}] {r[1][:58]:58s} " + " ".join(f"{k}:{int(v)}" for k, v in stalls))


if __name__ == "__main__":
    main()
