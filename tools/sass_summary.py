#!/usr/bin/env python3
"""Per-kernel SASS opcode counts of the built library's objects (cuobjdump
-sass), highlighting the instructions that prove the sm_100a paths:
UTCHMMA / UTCQMMA / UTCIMMA (tcgen05.mma kind::f16 / f8f6f4 / i8), UTMALDG / UTMASTG (TMA), LDTM / STTM
(tcgen05.ld / st), UTCBAR (tcgen05.commit), SYNCS (mbarrier), MUFU (ex2).

    python tools/sass_summary.py > profiles/r02_sass_summary.md
"""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "IMMA", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "UTCBAR", "SYNCS", "MUFU",
       "FFMA", "HMMA"]


def kernels(obj):
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    cur, out = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            out[cur][m.group(1)] += 1
    return out


def short(name):
    try:
        dm = subprocess.run(["cu++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        dm = name
    m = re.search(r"(\w+_kernel)(<[^>]*>)?\(", dm)
    return (m.group(1) + (m.group(2) or "").replace("(int)", "").replace("(bool)", "")) if m else name[:60]


def main():
    objs = sorted(glob.glob(os.path.join(ROOT, "paper_2602_01077_b200", "lib", "obj", "*.o")))
    print("# SASS opcode summary (cuobjdump -sass of paper_2602_01077_b200/lib/obj/*.o, sm_100a)\n")
    print("| object | kernel | " + " | ".join(KEY) + " | total |")
    print("|---" * (len(KEY) + 3) + "|")
    for o in objs:
        for k, c in kernels(o).items():
            print(f"| {os.path.basename(o)} | `{short(k)}` | " + " | ".join(str(c.get(x, 0)) for x in KEY)
                  + f" | {sum(c.values())} |")
    return 0


if __name__ == "__main__":
    sys.exit(main())
