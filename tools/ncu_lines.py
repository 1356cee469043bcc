"""Summarize an ncu report's warp-stall samples per CUDA source line.

    python tools/ncu_lines.py report.ncu-rep [top_n]
Uses `ncu --page source --print-source cuda,sass --csv` (needs -lineinfo).
"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname, seen_fn = None, "?", 0
res = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Function Name":
        seen_fn += 1
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        samples = int(float(r[4] or 0))
    except ValueError:
        continue
    stalls = {}
    for i, k in enumerate(hdr):
        if k.startswith("stall_") and "Not Issued" not in k and i < len(r):
            try:
                v = int(float(r[i] or 0))
            except ValueError:
                v = 0
            if v:
                stalls[k[6:]] = stalls.get(k[6:], 0) + v
    res.append((samples, fname, r[0], r[1], stalls))
tot = sum(x[0] for x in res) or 1
print(f"total samples {tot} over {seen_fn} function blocks")
for s, f, ln, src, st in sorted(res, key=lambda x: -x[0])[:top]:
    stt = " ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{s:6d} {100 * s / tot:5.1f}% {f}:{ln:<5} {src.strip()[:60]:60s} {stt}")
