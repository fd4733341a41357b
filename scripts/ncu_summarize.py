"""Summarise an ncu capture into profiles/: selected per-kernel metrics (CSV + markdown rows).

    python scripts/ncu_summarize.py gpurun_out/prof_r1i.ncu-rep profiles/r1_ncu_full.csv
    python scripts/ncu_summarize.py --launches gpurun_out/launches_r1i.csv profiles/r1_launches.csv
"""
import csv
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum",
]


def full(rep, out):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel"] + [f"{m} [{units[idx[m]]}]" for m in METRICS if m in idx])
        for r in rows[2:]:
            name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
            w.writerow([name] + [r[idx[m]] for m in METRICS if m in idx])
    print(open(out).read())


def launches(src, out):
    rows = list(csv.reader(open(src)))
    start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[start]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["launch", "kernel", "gpu__time_duration_us"])
        for r in rows[start + 1:]:
            if len(r) <= iV:
                continue
            name = r[iN].split("(")[0].replace("void ", "")
            us = float(r[iV].replace(",", "")) / 1e3
            agg[name].append(us)
            w.writerow([r[0], name, f"{us:.1f}"])
    tot = sum(sum(v) for v in agg.values())
    for k, v in agg.items():
        print(f"{k:45s} n={len(v):3d} mean={sum(v)/len(v):9.1f} us share={sum(v)/tot:6.1%}")


def traffic(csv_path, config, tag):
    """profiles/ncu_traffic.json[config]: DRAM bytes (read + write) per launch of the kernels
    gesr_tasa_score launches in a bench capture (-k attn_pair|proj_kernel|hma_kernel, in launch
    order hma, K/V projection, [Q projection], attention): bench.py's roofline.traffic."""
    import json
    import os
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[0]
    ir = [i for i, h in enumerate(hdr) if h.startswith("dram__bytes_read.sum")][0]
    iw = [i for i, h in enumerate(hdr) if h.startswith("dram__bytes_write.sum")][0]
    def scale(h):
        return 1e9 if "Gbyte" in h else (1e6 if "Mbyte" in h else (1e3 if "Kbyte" in h else 1.0))
    kern = {}
    projs = 0
    for r in rows[1:]:
        name = r[0]
        b = float(r[ir]) * scale(hdr[ir]) + float(r[iw]) * scale(hdr[iw])
        if "proj_kernel" in name:
            projs += 1
            if projs == 2:
                kern["proj_kernel (q projection)"] = b
        elif "attn" in name:
            kern[name] = b
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "ncu_traffic.json")
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[config] = {"tasa_bytes_per_launch": sum(kern.values()), "kernels": kern,
                 "source": f"{csv_path} (ncu --set full, dram__bytes_read.sum + "
                           f"dram__bytes_write.sum; capture {tag})"}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d[config], indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[1], sys.argv[2])
