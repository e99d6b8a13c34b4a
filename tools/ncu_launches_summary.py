"""Summarise ncu --csv launch lists (tools/ncu_r2_job.sh) into a table and
profiles/traffic.json: DRAM bytes (read + write) of the grouped-GEMM launches of
ONE layer step per workload, the roofline's `traffic` field in bench.py.
python tools/ncu_launches_summary.py <tag> <csv>..."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    hdr, data = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
                 "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "hz": 1, "Ghz": 1e9,
                 "Mhz": 1e6, "sector": 1, "%": 1}.get(unit, 1)
        data.setdefault(key, {})[d["Metric Name"]] = v * scale
    return data


def main():
    tag, paths = sys.argv[1], sys.argv[2:]
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic = {k: v for k, v in traffic.items() if isinstance(v, dict)}
    lines = []
    for p in paths:
        wl = os.path.basename(p).split("launches_")[1].rsplit(".", 1)[0]
        data = parse(p)
        gemm_bytes = 0.0
        lines.append(f"== {wl} ({os.path.basename(p)})")
        for (i, name), m in data.items():
            short = name.split("(")[0].replace("void ", "")
            rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
            t = m.get("gpu__time_duration.sum", 0)
            l2 = m.get("lts__t_sectors_srcunit_tex_op_read.sum", 0) * 32
            clk = m.get("sm__cycles_elapsed.avg.per_second", 0)
            tens = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0)
            lines.append(f"{i:2d} {short:55s} {t * 1e6:9.1f} us  DRAM r {rd / 1e9:7.3f} GB w "
                         f"{wr / 1e9:6.3f} GB  L2->SM rd {l2 / 1e9:6.2f} GB  tensor {tens:5.1f}%  "
                         f"{clk / 1e9:5.2f} GHz")
            if "gemm_bf16_tc_kernel" in name and not name.split("<")[1].startswith(("32,", "64,", "128,")):
                gemm_bytes += rd + wr
            elif "gemm_bf16_tc_kernel" in name and wl in ("c3",) and not name.split("<")[1].startswith("128,"):
                gemm_bytes += rd + wr
        traffic[f"{wl}_n1"] = {"grouped_gemm_bytes_per_step": gemm_bytes,
                               "source": f"profiles/{tag}_launches_{wl}.csv (ncu, one step, "
                                         f"cold-cache serialised launches)"}
        lines.append(f"   grouped-GEMM DRAM bytes per step: {gemm_bytes / 1e9:.3f} GB")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
