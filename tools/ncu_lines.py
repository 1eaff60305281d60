"""Per-source-line warp-stall samples of an ncu --set full report (the
cuda,sass source page), to find where a kernel's time goes.
Usage: python tools/ncu_lines.py REP [--top 30]"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, line, src = "?", None, ""
    tot = defaultdict(float)
    text = {}
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0].strip().isdigit():  # a source line (with its own aggregated columns)
            line = (fname, int(r[0]))
            text[line] = r[1][:90]
            try:
                tot[line] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:args.top]:
        print(f"{100 * v / s:6.2f}%  {k[0]}:{k[1]}  {text.get(k, '')}")


if __name__ == "__main__":
    main()
