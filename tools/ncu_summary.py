#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: the per-kernel launch list (share of
the step) and the key counters of one `--set full` capture.

    python tools/ncu_summary.py --launches gpurun_out/launches_c2.csv \
        --rep gpurun_out/prof_c2.ncu-rep --out profiles/r01_c2.md
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__sectors_read.sum", "dram__sectors_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_lookup_miss.sum", "lts__t_sectors_srcunit_tex_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
    "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    return agg


def rep_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        m = {h: (row[i], units[i]) for i, h in enumerate(hdr)}
        res.append(m)
    stalls = []
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        agg = launches(a.launches)
        tot = sum(sum(v) for v in agg.values())
        lines += ["## Launch list (ncu gpu__time_duration.sum, cold/serialised)", "",
                  "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/len(v)/1e3:.1f} | "
                         f"{sum(v)/tot*100:.1f}% |")
        lines.append("")
    if a.rep:
        for m in rep_metrics(a.rep):
            name = m.get("Kernel Name", ("?", ""))[0]
            lines += [f"## `{name[:120]}`", "", "| metric | value | unit |", "|---|---|---|"]
            for k in KEYS:
                if k in m:
                    lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
            st = []
            for k, (v, u) in m.items():
                if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                    try:
                        st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""),
                                   float(v.replace(",", ""))))
                    except ValueError:
                        pass
            st.sort(key=lambda x: -x[1])
            tot = sum(v for _, v in st) or 1
            lines += ["", "Top stall reasons (pc sampling):", ""]
            lines += [f"- {k}: {v/tot*100:.1f}%" for k, v in st[:8]]
            lines.append("")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print(open(a.out).read())


if __name__ == "__main__":
    main()
