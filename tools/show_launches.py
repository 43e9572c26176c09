import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ks = [(r[ki].split("(")[0], float(r[vi]) / 1e3) for r in rows]
# last build = last len/3 launches: print the final build's kernels
n = len(ks)
start = max(i for i, (k, _) in enumerate(ks) if k == "k_boxes_count")
tot = 0
for k, t in ks[start:]:
    tot += t
    print(f"  {k:32s} {t:8.1f} us")
print(f"  {'total':32s} {tot:8.1f} us")
