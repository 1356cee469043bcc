"""Opcode summary of every kernel instance in the production library.

    python tools/sass_summary.py [lib.so] > profiles/<round>_sass_summary.txt

Per instance: registers / shared / stack (cuobjdump -res-usage), SASS size,
and counts of the opcodes that show what the kernel is built from: bulk
copies (UBLKCP), mbarrier ops (SYNCS), cluster shared stores (STAS), POPC /
LOP3 (the scan), shared atomics (ATOMS), barriers, and the global-load
flavours (LDG ... CONSTANT is the non-coherent path: it must not appear on
buffers a peer writes while the kernel runs).
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2510_18413_b200/libadamas_b200.so"
KEYS = ["UBLKCP", "UTMALDG", "SYNCS", "STAS", "POPC", "LOP3", "ATOMS", "BAR", "UCGABAR", "LDS", "STS",
        "LDG", "LDG.CONSTANT", "LDG.STRONG.SYS", "STG", "STG.STRONG.SYS", "CCTL", "SHFL", "DADD", "DMUL", "MUFU"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    usage = {}
    fn = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", line)
        if m and fn:
            usage[fn] = tuple(int(x) for x in m.groups())
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            op = m.group(1)
            c = funcs[cur]
            c["_n"] += 1
            base = op.split(".")[0]
            c[base] += 1
            if base == "LDG":
                if ".CONSTANT" in op:
                    c["LDG.CONSTANT"] += 1
                if ".STRONG.SYS" in op:
                    c["LDG.STRONG.SYS"] += 1
            if base == "STG" and ".STRONG.SYS" in op:
                c["STG.STRONG.SYS"] += 1
    names = demangle(list(funcs))
    print(f"# SASS opcode summary of {LIB} (cuobjdump -sass / -res-usage, sm_100a)")
    print("# columns: regs stack smem_static instrs | " + " ".join(KEYS))
    for f, c in funcs.items():
        r = usage.get(f, (0, 0, 0))
        name = names[f].replace("adamas_dev::", "").replace("(adamas_dev::FusedParams)", "")
        name = re.sub(r"\(.*\)$", "", name)
        cols = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
        print(f"{name}\n    regs={r[0]} stack={r[1]} smem={r[2]} instrs={c['_n']} | {cols}")


if __name__ == "__main__":
    main()
