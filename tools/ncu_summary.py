"""Summarise an ncu --set full report into profiles/<name>.json (+ print).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_scd_async_c2.json [regex]
traffic_bytes = DRAM read + write of the scd_async launch (else the first kernel).
"""
import csv
import io
import json
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.sum", "lts__t_requests_srcunit_tex_op_read.sum",
        "lts__t_requests_srcunit_tex_op_red.sum", "lts__t_requests_srcunit_ltcfabric.sum",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_op_read_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard"]
kernels = []
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    rec = {"kernel": name, "id": r[h.index("ID")]}
    for k in want:
        if k in h:
            v = r[h.index(k)].replace(",", "")
            try:
                rec[k] = float(v)
            except ValueError:
                rec[k] = v
            rec[k + ".unit"] = units[h.index(k)]
    kernels.append(rec)
summary = {"report": rep, "kernels": kernels}
if kernels:
    # traffic of the epoch kernel when the report has one (bench.py reads it)
    k0 = next((k for k in kernels if "scd_async" in k["kernel"]), kernels[0])
    def to_bytes(key):
        v, u = k0.get(key), k0.get(key + ".unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return v * scale if isinstance(v, float) else None
    rb, wb = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
    summary["traffic_bytes"] = (rb or 0) + (wb or 0)
json.dump(summary, open(out, "w"), indent=1)
for k in kernels:
    print(k["kernel"][:60])
    for key in want:
        if key in k:
            print(f"   {key:70s} {k[key]} {k.get(key + '.unit', '')}")
print("traffic_bytes", summary.get("traffic_bytes"))
