"""Summary of an ncu --set full report as the bench's JSON (profiles/rN_ncu_full_top_kernels.json):
one dict per kernel launch with [value, unit] pairs of the metrics the bench and DESIGN cite.
usage: python tools/ncu_json.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = {"Kernel Name": [r[hdr.index("Kernel Name")], ""]}
    for k in KEYS:
        if k in hdr:
            d[k] = [r[hdr.index(k)], units[hdr.index(k)]]
    out.append(d)
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(len(out), "kernels")
