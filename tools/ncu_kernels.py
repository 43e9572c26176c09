"""Per-kernel summary of an ncu --set full report -> JSON lines (profiles/rNN_ncu_full_*.json).

    python tools/ncu_kernels.py gpurun_out/r1b_full.ncu-rep > profiles/r1b_ncu_full_cfg3.json
Fields: time_us, DRAM read/write bytes, DRAM % of peak, SM %, warps active %, registers, grid,
block, executed warp instructions."""
import csv
import io
import json
import subprocess
import sys

METRICS = {"gpu__time_duration.sum": "time_us", "dram__bytes_read.sum": "dram_read_bytes",
           "dram__bytes_write.sum": "dram_write_bytes",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
           "launch__registers_per_thread": "regs", "launch__grid_size": "grid", "launch__block_size": "block",
           "smsp__inst_executed.sum": "warp_instructions",
           "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct"}
SCALE = {"time_us": {"ns": 1e-3, "us": 1.0, "ms": 1e3}, "dram_read_bytes": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "dram_write_bytes": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}}

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
    for m, name in METRICS.items():
        i = hdr.index(m)
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        v *= SCALE.get(name, {}).get(units[i], 1.0)
        rec[name] = round(v, 3)
    print(json.dumps(rec))
