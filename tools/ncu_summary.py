"""Summarise ncu captures into profiles/ (tracked): key metrics of a --set full
report, top stall lines of its source page, and the kernel shares of a launch
list. Usage:
  python tools/ncu_summary.py --rep gpurun_out/prof_lamb.ncu-rep --name r01_lamb [--traffic-key lamb_kernel]
  python tools/ncu_summary.py --launches gpurun_out/launches.csv --name r01_bench_launches
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize_rep(rep: Path, top: int = 15):
    rows = ncu_csv(["-i", str(rep), "--page", "raw"])
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in METRICS:
        if k in hdr:
            i = hdr.index(k)
            m[k] = {"value": vals[i], "unit": units[i]}
    # per-launch DRAM traffic in bytes
    def to_bytes(k):
        v = float(m[k]["value"].replace(",", ""))
        u = m[k]["unit"]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    if "dram__bytes_read.sum" in m:
        m["dram_bytes_per_launch"] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    src = ncu_csv(["-i", str(rep), "--page", "source", "--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        ia, isrc, iw = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = src[2:]
        tot = sum(float(r[iw] or 0) for r in data) or 1.0
        m["top_stall_sass"] = [{"pct": round(float(r[iw] or 0) / tot * 100, 2), "sass": r[isrc].strip()}
                               for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:top]]
    return m


def summarize_launches(path: Path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iu = hdr.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            v = float(r[iv].replace(",", ""))
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[iu]]
            per[r[ik]].append(v * scale)
    total = sum(sum(v) for v in per.values()) or 1.0
    return {"total_us": total, "kernels": sorted(
        [{"kernel": k[:160], "launches": len(v), "us_total": sum(v), "us_avg": sum(v) / len(v),
          "share": sum(v) / total} for k, v in per.items()], key=lambda x: -x["share"])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--name", required=True)
    ap.add_argument("--traffic-key")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    if a.rep:
        s = summarize_rep(Path(a.rep))
        (PROF / f"{a.name}.json").write_text(json.dumps(s, indent=1))
        if a.traffic_key and "dram_bytes_per_launch" in s:
            tp = PROF / "ncu_traffic.json"
            t = json.loads(tp.read_text()) if tp.exists() else {}
            t[a.traffic_key] = {"dram_bytes_per_launch": s["dram_bytes_per_launch"], "source": f"profiles/{a.name}.json",
                                "kernel": s["kernel"]}
            tp.write_text(json.dumps(t, indent=1))
    if a.launches:
        (PROF / f"{a.name}.json").write_text(json.dumps(summarize_launches(Path(a.launches)), indent=1))
    print("wrote", PROF / f"{a.name}.json")


if __name__ == "__main__":
    main()
