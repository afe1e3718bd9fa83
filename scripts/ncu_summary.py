"""Readable summary of one `ncu --set full` capture (key sections, pipe
utilisation, stall reasons, DRAM bytes).  Usage:
  python scripts/ncu_summary.py gpurun_out/x.ncu-rep "title" > profiles/<tag>_sweep_ncu.txt"""
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(det.splitlines()))
hdr = rows[0]
print(title)
print(f"report: {rep}\n")
keep = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Occupancy",
        "Launch Statistics", "Warp State Statistics", "Memory Workload Analysis")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Section Name") in keep and d.get("Metric Name"):
        print(f"{d['Section Name'][:28]:28s} {d['Metric Name'][:44]:44s} "
              f"{d['Metric Value']:>16s} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(raw.splitlines()))
d = dict(zip(r[0], r[2]))
u = dict(zip(r[0], r[1]))
print("\npipe utilisation (% of peak, active cycles):")
for k in ["fp64", "lsu", "alu", "fma", "tensor_subpipe_dmma", "tmem", "xu", "uniform"]:
    key = f"sm__inst_executed_pipe_{k}.avg.pct_of_peak_sustained_active"
    if key in d:
        print(f"  {k:24s} {float(d[key]):6.1f}")
print("warp stall reasons (cycles per issued instruction):")
for k in sorted(d):
    if k.startswith("smsp__average_warps_issue_stalled_") and \
            k.endswith("_per_issue_active.ratio") and float(d[k]) > 0.05:
        print(f"  {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s}"
              f" {float(d[k]):5.2f}")
rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
print(f"DRAM read {rd:.1f} {u['dram__bytes_read.sum']}, write {wr:.1f} {u['dram__bytes_write.sum']}")
print(f"instructions executed: {d['smsp__inst_executed.sum']}")
