"""Aggregate an ncu source page by line ranges of greedy_kernel.cuh (phases) and by
stall reason.  usage: python tools/ncu_regions.py report.ncu-rep "PA:180-260,PM:300-700,..." """
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ranges = [(nm, int(a), int(b)) for nm, ab in (x.split(":") for x in sys.argv[2].split(",")) for a, b in [ab.split("-")]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
fname = ""
acc = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))
    reg = fname
    if fname == "greedy_kernel.cuh":
        reg = "other"
        for nm, a, b in ranges:
            if a <= ln <= b:
                reg = nm
    for k, v in d.items():
        if k.startswith("stall_") or k in ("Instructions Executed", "Warp Stall Sampling (All Samples)"):
            try:
                acc[reg][k] += float(v)
            except ValueError:
                pass
tot = sum(c["Warp Stall Sampling (All Samples)"] for c in acc.values()) or 1
for reg, c in sorted(acc.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"]):
    ss = c["Warp Stall Sampling (All Samples)"]
    top = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:5]
    print(f"{reg:28s} stall {100 * ss / tot:5.1f}%  instr {c['Instructions Executed']:.3g}  " +
          " ".join(f"{n}:{v:.0f}" for v, n in top))
