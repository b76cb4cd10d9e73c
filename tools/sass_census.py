#!/usr/bin/env python
"""Per-kernel SASS instruction census of libb2moe.so (cuobjdump -sass): the tcgen05 / TMEM / TMA
instructions that prove the GEMMs run on the 5th-generation tensor cores, plus the registers,
stack and local memory of every kernel (cuobjdump -res-usage).

  python tools/sass_census.py > profiles/r02_sass_census.md
"""
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2604_00785_b200", "libb2moe.so")
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
# mnemonic prefixes of interest: tcgen05 MMA (UTCHMMA / UTCQMMA), TMEM load/store/alloc
# (LDTM / STTM / UTCATOMSWS...), TMA (UTMALDG / UTMASTG / UTMAPF / UBLKCP), mbarriers (SYNCS),
# FP64 (DFMA / DMUL / DADD / MUFU.RSQ64H), the f32x2 FMA (FFMA2), async copies (LDGSTS)
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTCATOM", "UTMALDG", "UTMASTG", "UTMAPF",
        "UBLKCP", "UBLKRED", "SYNCS", "FFMA2", "FFMA", "DFMA", "DMUL", "DADD", "MUFU", "LDGSTS", "LDG", "STG",
        "LDS", "STS"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    sass = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run([CUOBJDUMP, "-res-usage", LIB], capture_output=True, text=True).stdout
    counts = defaultdict(Counter)
    cur = None
    for line in sass.split("\n"):
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            op, mod = m.group(2), m.group(3) or ""
            for k in KEYS:
                if op == k:
                    counts[cur][k + (mod if k in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM") else "")] += 1
    usage = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", res):
        usage[m.group(1)] = tuple(int(x) for x in m.group(2, 3, 4, 5))
    names = sorted(set(counts) | set(usage))
    dm = demangle(names)
    print(f"# SASS census of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass / -res-usage, sm_100a)\n")
    print("| kernel | regs | stack | static smem | local | key instructions |")
    print("|---|---|---|---|---|---|")
    for n in sorted(names, key=lambda x: dm[x]):
        r = usage.get(n, ("?",) * 4)
        c = ", ".join(f"{k} {v}" for k, v in sorted(counts[n].items()))
        short = re.sub(r"\([^()]*\)$", "", dm[n]).replace("b2::", "").replace("sm100::", "") or n
        print(f"| `{short}` | {r[0]} | {r[1]} | {r[2]} | {r[3]} | {c} |")
    tot = Counter()
    for n in names:
        tot.update(counts[n])
    print("\nTotals: " + ", ".join(f"{k} {v}" for k, v in sorted(tot.items())))


if __name__ == "__main__":
    main()
