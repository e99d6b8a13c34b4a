"""Summarise ncu outputs into profiles/: a launch-list CSV (gpu__time_duration
+ dram bytes per launch) and a --set full report (key counters per kernel).

    python tools/ncu_summary.py --launches gpurun_out/r1_launches.csv \
        --full gpurun_out/r1_full.ncu-rep --out profiles/r1 [--steps 2]
"""

import argparse
import csv
import io
import json
import subprocess
from collections import OrderedDict, defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
]


def short(name: str) -> str:
    name = name.replace("moe::", "")
    return name.split("(")[0][:70]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per, names = defaultdict(dict), {}
    for r in rows[1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = short(r[ki])
    return per, names


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = OrderedDict(kernel=short(r[hdr.index("Kernel Name")]))
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    lines = []
    if a.launches:
        per, names = launches(a.launches)
        agg = OrderedDict()
        for i in sorted(per):
            m = per[i]
            lines.append(f"{i:4d} {names[i]:70s} {m.get('gpu__time_duration.sum', 0) / 1e3:10.1f} us"
                         f"  rd {m.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB"
                         f"  wr {m.get('dram__bytes_write.sum', 0) / 1e6:9.1f} MB")
            a_ = agg.setdefault(names[i], [0, 0.0, 0.0, 0.0])
            a_[0] += 1
            a_[1] += m.get("gpu__time_duration.sum", 0)
            a_[2] += m.get("dram__bytes_read.sum", 0)
            a_[3] += m.get("dram__bytes_write.sum", 0)
        tot = sum(v[1] for v in agg.values())
        lines.append("")
        lines.append("per kernel: launches, mean us, share of device time, mean DRAM MB (rd+wr)")
        for k, (n, t, rd, wr) in agg.items():
            lines.append(f"  {k:70s} {n:3d} {t / n / 1e3:9.1f} us {100 * t / tot:5.1f}%"
                         f"  {(rd + wr) / n / 1e6:9.1f} MB")
        open(a.out + "_launches.txt", "w").write("\n".join(lines) + "\n")
    if a.full:
        res = full(a.full)
        with open(a.out + "_full.txt", "w") as f:
            for d in res:
                f.write(f"== {d['kernel']}\n")
                for k, v in d.items():
                    if k != "kernel":
                        f.write(f"   {k:70s} {v}\n")
        json.dump(res, open(a.out + "_full.json", "w"), indent=1)
    print("\n".join(lines[-12:]))


if __name__ == "__main__":
    main()
