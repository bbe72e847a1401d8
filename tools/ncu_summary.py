"""Summarise an `ncu --set full --import-source on` report for profiles/: headline metrics of the
first captured kernel, warp-stall reasons (share of samples), and stall samples aggregated by
SASS opcode. Usage: python tools/ncu_summary.py <report.ncu-rep> [header line]"""
import collections
import csv
import io
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
STALLS = ["stall_math", "stall_wait", "stall_dispatch", "stall_short_sb", "stall_not_selected", "stall_selected",
          "stall_lg", "stall_barrier", "stall_long_sb", "stall_mio", "stall_branch_resolving", "stall_no_inst",
          "stall_sleep", "stall_misc", "stall_membar", "stall_drain", "stall_tex"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    rep = sys.argv[1]
    out = [f"# {sys.argv[2]}" if len(sys.argv) > 2 else f"# ncu summary of {rep}", "# metric | value | unit"]
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, first = raw[0], raw[1], raw[2]
    ix = {h: i for i, h in enumerate(hdr)}
    out.append(f"Kernel Name | {first[ix['Kernel Name']]} |")
    for m in METRICS:
        if m in ix:
            out.append(f"{m} | {first[ix[m]]} | {units[ix[m]]}")
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sh, data = src[1], src[2:]
    si = {h: i for i, h in enumerate(sh)}

    def val(r, c):
        try:
            return int(r[si[c]] or 0)
        except (KeyError, ValueError, IndexError):
            return 0
    total = sum(val(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
    out.append("# warp-stall samples by reason (share of all samples)")
    for s in sorted(STALLS, key=lambda c: -sum(val(r, c) for r in data)):
        v = sum(val(r, s) for r in data)
        if v / total >= 0.005:
            out.append(f"{s} | {v / total:.3f}")
    out.append("# stall samples by SASS opcode: share | instructions executed | top reasons")
    agg = collections.defaultdict(collections.Counter)
    for r in data:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[si["Source"]].strip()).split()
        if not op:
            continue
        for c in STALLS + ["Warp Stall Sampling (All Samples)", "Instructions Executed"]:
            agg[op[0]][c] += val(r, c)
    for op, a in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:16]:
        s = a["Warp Stall Sampling (All Samples)"]
        top = sorted(((a[c], c) for c in STALLS), reverse=True)[:3]
        out.append(f"{op} | {s / total:.3f} | {a['Instructions Executed']} | " +
                   " ".join(f"{c[6:]}={v / total:.3f}" for v, c in top if v))
    # shared-memory excess wavefronts (bank conflicts) by SASS line, where the source page has them
    exc = [c for c in sh if "Shared Excessive" in c or ("Excessive" in c and "Shared" in c)]
    for c in exc[:2]:
        rows = sorted(data, key=lambda r: -val(r, c))[:8]
        if rows and val(rows[0], c):
            out.append(f"# top SASS lines by '{c}': address | value | source")
            for r in rows:
                if val(r, c):
                    out.append(f"{r[si.get('Address', 0)]} | {val(r, c)} | {r[si['Source']].strip()[:90]}")
    print("\n".join(out))


if __name__ == "__main__":
    main()
