"""Opcode evidence from the built library: counts of the Blackwell-specific opcodes over all kernels
and the opcode histogram of the table walk's step loop (found through the back branch after the last
IDP.2A) for the main kernel variants.

    cuobjdump -sass paper_2601_03332_b200/liblutkan_b200.so > /tmp/all.sass
    python tools/sass_loops.py /tmp/all.sass > profiles/<round>/sass_hist.txt
"""
import collections
import re
import sys

KERNELS = {
    "C2 layer 0 walk (BAL, XB=2, IDP, in-kernel coordinates; static count: the exact-coordinate fallback "
    "(DFMA/F2F/CALL) sits inside the loop and is rarely executed, ~227 executed per step)":
        "Li2ELi16ELb0ELb1ELb0ELb0ELb0ELi1ELb0ELb1ELi2ELb0ELi2ELb0ELi0E",
    "C4/C3 REC walk (XT, TMEM f64)": "Li2ELi16ELb0ELb1ELb0ELb1ELb0ELi1ELb0ELb0ELi1ELb1ELi2ELb1ELi0E",
    "C5 REC walk on pair entries (GC, asym, zero_spline)": "Li2ELi16ELb1ELb1ELb1ELb1ELb0ELi1ELb1ELb0ELi1ELb1ELi3ELb1ELi0E",
    "small-batch walk (R=1, 4 stages; static count incl. the fallback)":
        "Li1ELi16ELb0ELb1ELb0ELb0ELb0ELi1ELb0ELb1ELi1ELb0ELi2ELb0ELi4E",
}


def main():
    funcs, cur = {}, None
    for line in open(sys.argv[1]):
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", line)
        if m and cur:
            funcs[cur].append((int(m.group(1), 16), m.group(3), m.group(4)))
    tot = collections.Counter(op.split(".")[0] for ins in funcs.values() for _, op, _ in ins)
    print("# liblutkan_b200.so (sm_100a), cuobjdump -sass: opcode evidence (tools/sass_loops.py)")
    print(f"# Blackwell-specific and hot opcodes over all {len(funcs)} kernels")
    for k in ("UTMALDG", "UBLKCP", "SYNCS", "LDTM", "STTM", "UTCHMMA", "UTCBAR", "IDP", "LDGSTS", "FFMA2", "FADD2",
              "DADD", "MUFU", "LDG", "LDS", "PRMT"):
        if tot.get(k):
            print(f"{k:10s} {tot[k]}")
    for title, sub in KERNELS.items():
        f = next((f for f in funcs if sub in f), None)
        if not f:
            print(f"\n# {title}: kernel not found")
            continue
        ins = funcs[f]
        idp = [i for i, (_, op, _) in enumerate(ins) if op.startswith("IDP.2A")]
        lo_a = ins[idp[0]][0]
        start = end = None
        for i in range(idp[-1], len(ins)):
            a, op, rest = ins[i]
            m = re.search(r"0x([0-9a-f]+)", rest) if op.startswith("BRA") else None
            if m and int(m.group(1), 16) <= lo_a:
                start, end = int(m.group(1), 16), a
                break
        body = [op for a, op, _ in ins if start <= a <= end]
        c = collections.Counter(op.split(".")[0] for op in body)
        print(f"\n# {title}\n#   step loop 0x{start:x}-0x{end:x}: {len(body)} instructions per warp-step")
        print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
