"""Summarize an ncu report per CUDA source line (instructions executed, warp
stall samples and the top stall reasons).  Usage:
    python tools/ncu_lines.py report.ncu-rep [top_n]
Needs a report captured with --import-source on and a -lineinfo build."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    fname = ""
    lines = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or r[0] in ("", "Function Name", "File Path"):
            continue
        try:
            int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr, r))
        lines.append((fname, int(r[0]), r[1], d))
    ie = "Instructions Executed"
    ss = "Warp Stall Sampling (All Samples)"

    def num(d, k):
        try:
            return float(d.get(k, "0"))
        except ValueError:
            return 0.0

    tot_i = sum(num(d, ie) for *_, d in lines) or 1
    tot_s = sum(num(d, ss) for *_, d in lines) or 1
    stall_cols = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
    print(f"total instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    for f, ln, src, d in sorted(lines, key=lambda x: -num(x[3], ss))[:top]:
        st = sorted(((num(d, c), c[6:]) for c in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
        print(f"{f}:{ln:<5d} instr {100 * num(d, ie) / tot_i:5.1f}%  stall {100 * num(d, ss) / tot_s:5.1f}%  "
              f"[{sts}]  {src.strip()[:70]}")


if __name__ == "__main__":
    main()
