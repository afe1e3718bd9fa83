"""Turn the raw ncu/bench outputs in gpurun_out/ into the committed profiles/.

  python scripts/summarize_profiles.py r01
writes profiles/<tag>_launches.csv        (ncu launch list, per-launch device time + DRAM bytes)
       profiles/<tag>_launch_summary.txt  (readable table of the second frame)
       profiles/<tag>_sweep_ncu.txt        (key metrics + stall reasons of the full sweep capture)
       profiles/<tag>_bench.json           (bench line(s))
       profiles/sweep_dram_traffic.json    (DRAM bytes of the finest-level sweep launch, read by bench.py)
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    iK, iM, iV, iI = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[iI]), r[iK].split("(")[0])
        d.setdefault(key, {})[r[iM]] = float(r[iV].replace(",", ""))
    return sorted(d.items())


def ncu_details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    keep = ["Duration", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
            "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
            "Executed Instructions", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate",
            "L1/TEX Hit Rate", "Compute (SM) Throughput", "Grid Size", "Block Size",
            "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
    res = []
    for r in rows[1:]:
        if len(r) > 4 and r[-4] in keep:
            res.append(f"{r[-4]:40s} {r[-3]:14s} {r[-2]}")
    return res


def ncu_raw(rep, prefixes):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    res = {}
    for i, k in enumerate(h):
        if any(k.startswith(p) for p in prefixes):
            try:
                res[k] = float(v[i].replace(",", ""))
            except ValueError:
                pass
    return res


def main(tag):
    os.makedirs(OUT, exist_ok=True)
    lp = os.path.join(RAW, "launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(OUT, f"{tag}_launches.csv"))
        items = launches(lp)
        second = items[len(items) // 2:]
        lines = [f"{'id':>4} {'kernel':58s} {'us':>9} {'DRAM R MB':>10} {'DRAM W MB':>10} {'GB/s':>7}"]
        tot = 0.0
        finest = None
        for (i, k), m in second:
            t = m["gpu__time_duration.sum"] / 1e3
            rb, wb = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6
            tot += t
            lines.append(f"{i:>4} {k:58s} {t:9.1f} {rb:10.1f} {wb:10.1f} {(rb + wb) / t * 1e3 if t else 0:7.0f}")
            if "oras_sweep" in k and finest is None and t > 1000:
                finest = (i, k, m)
        lines.append(f"total device time of one 4K frame (serialised, cold caches): {tot:.1f} us")
        open(os.path.join(OUT, f"{tag}_launch_summary.txt"), "w").write("\n".join(lines) + "\n")
        if finest:
            i, k, m = finest
            n = 3840 * 2160
            json.dump({"kernel": k, "launch_id": i,
                       "launch": "first finest-level sweep of the second frame (4K RGB, fp64)",
                       "dram_bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                       "algorithmic_bytes_per_launch": n * (2 * 3 * 8 + 1),
                       "device_us": m["gpu__time_duration.sum"] / 1e3,
                       "source": f"profiles/{tag}_launches.csv"},
                      open(os.path.join(OUT, "sweep_dram_traffic.json"), "w"), indent=1)
    rp = os.path.join(RAW, "sweep_full.ncu-rep")
    if os.path.exists(rp):
        det = ncu_details(rp)
        raw = ncu_raw(rp, ["smsp__average_warps_issue_stalled", "sm__pipe_fp64_cycles_active",
                           "sm__inst_executed_pipe_fp64", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
                           "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active"])
        stalls = sorted(((v, k.replace("smsp__average_warps_issue_stalled_", "")
                          .replace("_per_issue_active.ratio", ""))
                         for k, v in raw.items() if "issue_stalled" in k and
                         k.endswith("per_issue_active.ratio")), reverse=True)[:8]
        pipes = {k: v for k, v in raw.items() if "pct_of_peak_sustained_active" in k and
                 ("fp64" in k or "shared" in k) and ".avg." in k}
        txt = [f"ncu --set full capture of oras_sweep_kernel (finest level, 4K RGB fp64): {rp}", ""]
        txt += det + ["", "pipe utilisation (% of peak, active cycles):"]
        txt += [f"  {k:70s} {v:6.1f}" for k, v in sorted(pipes.items())]
        txt += ["", "warp stall reasons (cycles per issued instruction):"]
        txt += [f"  {k:30s} {v:6.2f}" for v, k in stalls]
        open(os.path.join(OUT, f"{tag}_sweep_ncu.txt"), "w").write("\n".join(txt) + "\n")
        # the on-chip bound of the sweep, next to its DRAM traffic (bench.py)
        tp = os.path.join(OUT, "sweep_dram_traffic.json")
        if os.path.exists(tp):
            tj = json.load(open(tp))
            fp64 = [v for k, v in pipes.items() if k.startswith("sm__pipe_fp64_cycles_active")]
            if fp64:
                tj["fp64_pipe_pct_of_peak"] = fp64[0]
            tj["ncu_full_capture"] = f"profiles/{tag}_sweep_ncu.txt"
            json.dump(tj, open(tp, "w"), indent=1)
    bench = []
    for name in ("bench.json", "bench_fp32.json", "bench_mixed.json"):
        p = os.path.join(RAW, name)
        if os.path.exists(p):
            for line in open(p):
                line = line.strip()
                if line.startswith("{"):
                    bench.append(json.loads(line))
    if bench:
        json.dump(bench, open(os.path.join(OUT, f"{tag}_bench.json"), "w"), indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
