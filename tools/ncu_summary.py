"""Summarise an ncu capture exported by tools/ncu_capture.sh (details/raw/source CSVs).

usage: python tools/ncu_summary.py gpurun_out/<name> [--frames F] [--top N]
Prints the speed-of-light, occupancy and issue numbers, stall reasons, DRAM traffic, the
instruction mix and, from the cuda,sass source view, where the samples land per source line
(decoder.cuh template / generated code line).
"""
import argparse
import csv
import gzip
import io
import re
from collections import Counter, defaultdict

KEEP = ["Duration", "SM Frequency", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "Theoretical Active Warps per SM",
        "Achieved Active Warps Per SM", "Block Limit Registers", "Block Limit Shared Mem", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Shared Memory Configuration Size"]


def details(prefix):
    rows = list(csv.reader(open(prefix + "_details.csv")))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = {}
    for r in rows[1:]:
        if r[mi] in KEEP and r[mi] not in out:
            out[r[mi]] = f"{r[vi]} {r[ui]}"
    return out


def raw(prefix):
    rows = list(csv.reader(open(prefix + "_raw.csv")))
    h, v = rows[0], rows[2]
    d = {}
    for i, n in enumerate(h):
        try:
            d[n] = float(v[i].replace(",", ""))
        except ValueError:
            pass
    return d


def source(prefix, top):
    """Per CUDA line (file:line) samples and executed instructions from the cuda,sass view,
    the SASS opcode mix, and the generated-code op lines grouped by (op, N_v)."""
    with gzip.open(prefix + "_source.csv.gz", "rt") as f:
        rows = list(csv.reader(f))
    per_line = defaultdict(lambda: [0, 0])
    per_op, per_op_s = Counter(), Counter()
    gen_ops = defaultdict(lambda: [0, 0])
    cur = "?"
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 8:
            continue
        try:
            smp, n = int(r[6] or 0), int(r[7] or 0)
        except ValueError:
            continue
        if r[0]:
            key = (cur, r[0], r[1].strip()[:90])
            per_line[key][0] += smp
            per_line[key][1] += n
            m = re.match(r"(?:const uint32_t m\d+ = )?(w[A-Za-z0-9]+|c[A-Za-z0-9]+|if \(threadIdx.x < 32\) sub\d+)<(?:P, )?(?:T, )?(\d+)?", r[1].strip())
            if cur.startswith("code_") and m:
                g = gen_ops[(m.group(1), int(m.group(2) or 0))]
                g[0] += smp
                g[1] += n
        elif len(r) > 3 and r[2].startswith("0x"):
            t = r[3].split()
            op = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
            per_op[op.split(".")[0]] += n
            per_op_s[op.split(".")[0]] += smp
    tot = sum(v[0] for v in per_line.values()) or 1
    print(f"\n-- top source lines by samples (total {tot})")
    for (fn, ln, src), (smp, n) in sorted(per_line.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * smp / tot:5.1f}%  inst {n:>12}  {fn}:{ln}  {src}")
    if gen_ops:
        print("\n-- generated op lines grouped by (op, N_v): samples share, instructions")
        for (op, nv), (smp, n) in sorted(gen_ops.items(), key=lambda x: -x[1][0])[:top]:
            print(f"{100 * smp / tot:5.1f}%  inst {n:>12}  {op}<{nv}>")
    return per_op, per_op_s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("prefix")
    ap.add_argument("--frames", type=float, default=0)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    d = details(a.prefix)
    for k in KEEP:
        if k in d:
            print(f"{k:40s} {d[k]}")
    r = raw(a.prefix)
    inst = r.get("smsp__inst_executed.sum", 0)
    print(f"{'warp instructions executed':40s} {inst:.0f}" + (f"  ({inst / a.frames:.0f} per frame)" if a.frames else ""))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in r:
            print(f"{k:40s} {r[k]:.4g}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): v for k, v in r.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    print("stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    pipes = {k.split("pipe_")[1].split(".")[0]: v for k, v in r.items()
             if re.match(r"sm__inst_executed_pipe_[a-z0-9_]+\.avg\.pct_of_peak_sustained_active$", k)}
    print("pipes %: " + ", ".join(f"{k} {v:.1f}" for k, v in sorted(pipes.items(), key=lambda x: -x[1])[:8]))
    try:
        per_op, per_op_s = source(a.prefix, a.top)
        T = sum(per_op.values()) or 1
        print("\n-- SASS mix (share of executed warp instructions)")
        print(", ".join(f"{k} {100 * v / T:.1f}%" for k, v in per_op.most_common(22)))
    except FileNotFoundError:
        pass


if __name__ == "__main__":
    main()
