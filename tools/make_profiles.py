"""Summarize ncu outputs from gpurun_out/ into profiles/ (committed evidence).

usage: python tools/make_profiles.py ROUND_TAG WORKLOAD launches.csv|- report.ncu-rep
Writes:
  profiles/<tag>_launches_<workload>.csv   per-kernel totals of the launch list (share of the step)
  profiles/<tag>_ncu_<workload>.txt        key metrics + per-line stall summary of the top kernel
  profiles/ncu_traffic.json                DRAM bytes per launch of the top kernel (read by bench.py)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        name = r[ki].split("(")[0].replace("void ", "").strip()
        agg[name].append(v * scale)
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, v, u in zip(hdr, r, units)})
    return res


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    tag, workload, lcsv, rep = sys.argv[1:5]
    os.makedirs(PROF, exist_ok=True)
    if lcsv != "-":
        agg = launches(lcsv)
        tot = sum(sum(v) for v in agg.values())
        with open(os.path.join(PROF, f"{tag}_launches_{workload}.csv"), "w") as fh:
            fh.write("kernel,launches,total_us,avg_us,share\n")
            for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
                fh.write(f"{k},{len(v)},{sum(v):.1f},{sum(v) / len(v):.2f},{sum(v) / tot:.4f}\n")
    mets = raw_metrics(rep)
    lines = []
    traffic = None
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__block_size",
            "launch__grid_size", "launch__cluster_dim_x", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__cycles_active.avg",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg",
            "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors.sum"]
    extra = {}
    for m in mets:
        name = m.get("Kernel Name", ("?", ""))[0]
        lines.append(f"kernel: {name}")
        for w in want:
            if w in m:
                v, u = m[w]
                lines.append(f"  {w:60s} {v} {u}")
        if "greedy" in name and traffic is None:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rv, ru = m.get("dram__bytes_read.sum", ("nan", "byte"))
            wv, wu = m.get("dram__bytes_write.sum", ("nan", "byte"))
            traffic = num(rv) * scale.get(ru, 1) + num(wv) * scale.get(wu, 1)
            wf = num(m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", ("nan", ""))[0])
            cyc = num(m.get("sm__cycles_elapsed.avg", ("nan", ""))[0])
            n_sm = 148
            extra = {"smem_pipe_frac": wf / (cyc * n_sm) if cyc == cyc and wf == wf else None,
                     "issue_active_pct": num(m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", ("nan", ""))[0]),
                     "warps_active_pct": num(m.get("sm__warps_active.avg.pct_of_peak_sustained_active", ("nan", ""))[0]),
                     "kernel_ms": num(m.get("gpu__time_duration.sum", ("nan", ""))[0])}
    src = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25"], capture_output=True,
                         text=True).stdout
    with open(os.path.join(PROF, f"{tag}_ncu_{workload}.txt"), "w") as fh:
        fh.write(f"# ncu --set full --clock-control none --import-source on, {workload}\n")
        fh.write("\n".join(lines) + "\n\n# per source line (instructions, warp stall samples)\n" + src)
    tj = os.path.join(PROF, "ncu_traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    if traffic is not None:
        data[workload] = dict({"kernel": "greedy_kernel", "dram_bytes_per_launch": traffic,
                               "source": f"{tag}_ncu_{workload}.txt"}, **extra)
    json.dump(data, open(tj, "w"), indent=1)
    if lcsv != "-":
        print(open(os.path.join(PROF, f"{tag}_launches_{workload}.csv")).read())
    print("\n".join(lines))
    print("traffic", traffic)


if __name__ == "__main__":
    main()
