"""Opcode histogram of a SASS address range (cuobjdump -sass output), optionally skipping ranges.

    python tools/sass_hist.py file.sass 0x5c90 0x7830 [--skip 0x6120:0x6bb0 ...]
"""
import re
import sys
from collections import Counter


def main():
    path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
    skips = []
    if "--skip" in sys.argv:
        for s in sys.argv[sys.argv.index("--skip") + 1:]:
            a, b = s.split(":")
            skips.append((int(a, 16), int(b, 16)))
    c, n = Counter(), 0
    for line in open(path):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if not m:
            continue
        addr = int(m.group(1), 16)
        if not lo <= addr < hi or any(a <= addr < b for a, b in skips):
            continue
        op = m.group(3).split(".")[0]
        c[op] += 1
        n += 1
    for op, k in c.most_common():
        print(f"{op:12s} {k}")
    print(f"{'TOTAL':12s} {n}")


if __name__ == "__main__":
    main()
