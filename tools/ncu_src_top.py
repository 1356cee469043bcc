"""Top source lines by warp-stall samples from an ncu report (source page).
    python tools/ncu_src_top.py <report.ncu-rep> [N] [file-filter]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = {n: i for i, n in enumerate(hdr)}
        continue
    if hdr is None or len(r) < 6 or r[0] == "":
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    st = {n[6:]: int(r[si[n]]) for n in hdr if n.startswith("stall_") and "Not Issued" not in n
          and r[si[n]].isdigit() and int(r[si[n]]) > 0}
    out.append((cur, int(r[0]), r[1].strip(), s, st))
tot = sum(o[3] for o in out) or 1
print("total samples", tot)
for o in sorted(out, key=lambda o: -o[3]):
    if filt and filt not in o[0]:
        continue
    if N == 0:
        break
    N -= 1
    st = sorted(o[4].items(), key=lambda kv: -kv[1])[:3]
    print(f"{o[3]:6d} {o[3] / tot:6.1%} {o[0]}:{o[1]:<4d} {o[2][:58]:58s} {st}")
