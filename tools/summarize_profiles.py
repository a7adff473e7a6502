#!/usr/bin/env python
"""Summarise a gpurun evidence directory into profiles/: ncu --set full
captures (key metrics + stall mix), DRAM traffic per launch, launch list.

usage: tools/summarize_profiles.py <run dir> <round tag> name=report.ncu-rep|report.raw.csv ...
"""
import collections
import csv
import json
import os
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    if rep.endswith(".csv"):  # a `--page raw --csv` export of the report
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def main():
    run, tag = sys.argv[1], sys.argv[2]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = os.path.join(root, "profiles")
    summ, traffic = {}, {}
    tpath = os.path.join(prof, "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for arg in sys.argv[3:]:
        name, rep = arg.split("=", 1)
        d = raw(os.path.join(run, rep))
        m = {k: d[k][0] + (" " + d[k][1] if d[k][1] else "") for k in KEYS if k in d}
        st = {}
        for h, (v, _) in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        m["stall_top_pct"] = {k: round(100 * v / tot, 1)
                              for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]}
        summ[name] = m
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = d[k]
            b += float(v.replace(",", "")) * SCALE.get(u, 1)
        traffic[name] = int(b)
    json.dump(summ, open(os.path.join(prof, f"{tag}_ncu_summary.json"), "w"), indent=1)
    json.dump(traffic, open(tpath, "w"), indent=1)
    lc = os.path.join(run, "launches.csv")
    if os.path.exists(lc):
        rows = [r for r in csv.reader(open(lc)) if len(r) > 10]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = collections.OrderedDict()
        for r in rows[1:]:
            agg.setdefault(r[ki].split("(")[0][:90], []).append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        with open(os.path.join(prof, f"{tag}_launches_cfg2.txt"), "w") as fh:
            fh.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, "
                     "serialised) of\n  python bench.py --steps 2 --warmup 3 --no-cpu-baseline "
                     "--no-e2e --load-seconds 0\n(torch kernels = untimed data generation and the "
                     "L2 flush; one recover launch per step)\n\n")
            for k, v in agg.items():
                fh.write(f"{len(v):4d} launches  mean {sum(v) / len(v) / 1e3:9.1f} us  total "
                         f"{sum(v) / 1e3:10.1f} us  {100 * sum(v) / tot:5.1f}%  {k}\n")
        subprocess.run(["cp", lc, os.path.join(prof, f"{tag}_launches_cfg2.csv")])
    print(json.dumps(summ, indent=1)[:1500])


if __name__ == "__main__":
    main()
