#!/usr/bin/env python3
"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked evidence).

usage: ncu_summary.py launches <launches.csv> <out.txt>
       ncu_summary.py full <report.ncu-rep> <out.txt> [traffic_key]
The 'full' mode also records dram bytes per launch into profiles/ncu_traffic.json
under traffic_key (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= mi:
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("dcsc_cuda::", "")
        v = float(r[mi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"# ncu launch list ({sum(cnt.values())} launches, gpu__time_duration.sum, --clock-control none;",
             "# cold-cache serialised: compare shares, not absolutes)",
             f"{'total_ms':>10} {'share':>7} {'launches':>8} {'avg_us':>10}  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{v / 1e6:10.3f} {100 * v / T:6.2f}% {cnt[k]:8d} {v / cnt[k] / 1e3:10.1f}  {k}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def full(path, out, key=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    lines = [f"# ncu --set full summary of {os.path.basename(path)}"]
    traffic = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        lines.append(f"## kernel: {re.sub(r'[(].*', '', d.get('Kernel Name', '?'))}")
        for w in WANT:
            if w in d:
                lines.append(f"{w:70s} {d[w]:>20s} {u.get(w, '')}")
        stalls = []
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(d[h]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        lines.append("top stall reasons (warp cycles per issued instruction):")
        for v, h in sorted(stalls, reverse=True)[:8]:
            lines.append(f"   {h:30s} {v:.3f}")

        def gb(name):
            v = float(d[name].replace(",", ""))
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u.get(name, "byte"), 1.0)

        try:
            traffic.append(gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum"))
        except Exception:
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if key and traffic:
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        data = json.load(open(tpath)) if os.path.exists(tpath) else {}
        data[key] = sum(traffic) / len(traffic)
        json.dump(data, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
