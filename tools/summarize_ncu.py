"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

    python tools/summarize_ncu.py --tag r01 [--rep gpurun_out/prof_fused.ncu-rep]
                                  [--launches gpurun_out/launches.csv]

Writes profiles/<tag>_launches.txt (per-kernel share of the launch list),
profiles/<tag>_ncu_<kernel>.txt (the counters SURVEY.md 8(d) asks for: DRAM
throughput, bytes, sectors/request, warp-stall breakdown, pipe utilisation,
top source lines by stall samples) and updates profiles/ncu_summary.json
(dram bytes per launch, read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu_csv(rep, *args):
    r = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def short(name):
    n = name.split("(")[0]
    for pre in ("void ", "adamas_dev::", "at::native::", "at::"):
        n = n.replace(pre, "")
    return n[:70]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    d = defaultdict(list)
    for r in rows[1:]:
        d[short(r[h.index("Kernel Name")])].append(float(r[h.index("Metric Value")].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
             f"# source: {os.path.basename(path)}", f"{'kernel':72s} {'n':>5s} {'mean_us':>9s} {'share':>7s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:72s} {len(v):5d} {sum(v) / len(v) / 1000:9.2f} {sum(v) / tot:7.1%}")
    open(out, "w").write("\n".join(lines) + "\n")
    return d


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__cluster_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_op_read.sum", "lts__t_bytes.sum",
]


def full(rep, out, tag):
    raw = ncu_csv(rep, "--page", "raw")
    h, units = raw[0], raw[1]
    summary = {}
    lines = [f"# ncu --set full --clock-control none: {os.path.basename(rep)} ({tag})"]
    for row in raw[2:]:
        kname = short(row[h.index("Kernel Name")])
        lines.append(f"\n## {kname}")
        vals = {n: (row[i], units[i]) for i, n in enumerate(h)}
        for n in WANT:
            if n in vals:
                lines.append(f"{n:60s} {vals[n][0]:>16s} {vals[n][1]}")
        try:
            sec = float(vals["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"][0].replace(",", ""))
            req = float(vals["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"][0].replace(",", ""))
            lines.append(f"{'sectors/request (global ld)':60s} {sec / max(req, 1):16.2f}")
        except (KeyError, ValueError):
            pass
        stalls = []
        for n, (v, u) in vals.items():
            if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".ratio") is False \
                    and "pct" not in n:
                try:
                    stalls.append((float(v.replace(",", "")), n.replace("smsp__average_warp_latency_issue_stalled_", "")))
                except ValueError:
                    pass
        if not stalls:
            for n, (v, u) in vals.items():
                if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                    try:
                        stalls.append((float(v.replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
        if stalls:
            lines.append("warp-stall breakdown (top 10):")
            tot = sum(s for s, _ in stalls) or 1.0
            for s, n in sorted(stalls, reverse=True)[:10]:
                lines.append(f"  {n:50s} {s:12.1f} {s / tot:7.1%}")
        pipes = []
        for n, (v, u) in vals.items():
            if n.startswith("sm__inst_executed_pipe_") and n.endswith("pct_of_peak_sustained_active"):
                try:
                    pipes.append((float(v.replace(",", "")), n))
                except ValueError:
                    pass
        if pipes:
            lines.append("pipe utilisation (% of peak, active cycles; top 8):")
            for s, n in sorted(pipes, reverse=True)[:8]:
                lines.append(f"  {n.replace('sm__inst_executed_pipe_', ''):60s} {s:7.2f}")
        try:
            b = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * (1e6 if vals["dram__bytes_read.sum"][1] == "Mbyte" else 1e3 if vals["dram__bytes_read.sum"][1] == "Kbyte" else 1)
            w = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * (1e6 if vals["dram__bytes_write.sum"][1] == "Mbyte" else 1e3 if vals["dram__bytes_write.sum"][1] == "Kbyte" else 1)
            t = float(vals["gpu__time_duration.sum"][0].replace(",", ""))
            summary.setdefault(kname.split("<")[0], {"dram_bytes_per_launch": b + w, "duration_us": t,
                                                     "source": f"profiles/{os.path.basename(out)}"})
        except (KeyError, ValueError):
            pass
    # top source lines by stall samples
    src = ncu_csv(rep, "--page", "source", "--print-source", "cuda,sass")
    hdr, cur, rows = None, None, []
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6 or r[0] == "":
            continue
        try:
            rows.append((int(r[4]), cur, r[0], r[1].strip()[:80]))
        except ValueError:
            pass
    if rows:
        tot = sum(x[0] for x in rows) or 1
        lines.append("\ntop source lines by warp-stall samples:")
        for s, f, ln, txt in sorted(rows, reverse=True)[:20]:
            lines.append(f"  {s / tot:6.1%} {f}:{ln}  {txt}")
    open(out, "w").write("\n".join(lines) + "\n")
    return summary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof_fused.ncu-rep"))
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--name", default="fused")
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "profiles"),
                    help="where the summaries go (on a GPU box: under gpurun_out/, merged back)")
    a = ap.parse_args()
    prof = a.out_dir
    os.makedirs(prof, exist_ok=True)
    if os.path.exists(a.launches):
        launches(a.launches, os.path.join(prof, f"{a.tag}_launches.txt"))
    if os.path.exists(a.rep):
        s = full(a.rep, os.path.join(prof, f"{a.tag}_ncu_{a.name}.txt"), a.tag)
        p = os.path.join(prof, "ncu_summary.json")
        cur = json.load(open(p)) if os.path.exists(p) else {}
        cur.update(s)
        json.dump(cur, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
