"""Attribute the executed warp instructions of an ncu cuda,sass source export to the
device function (decoder.cuh / kernels.cuh / xframe.cuh) whose body holds the source line.
usage: python tools/ncu_by_function.py gpurun_out/<name> [--frames F]"""
import argparse
import csv
import gzip
import os
import re
from collections import Counter

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1504_00353_b200", "csrc")
FN = re.compile(r"^\s*(?:template\s*<[^>]*>\s*)?(?:static\s+)?(?:PD_INLINE|__device__|__global__|__host__ __device__)[^(]*?\b(\w+)\s*\(")


def spans(path):
    """line -> enclosing function name (by the last function header above it)."""
    out, cur = {}, "?"
    for i, l in enumerate(open(path), 1):
        m = FN.match(l)
        if m:
            cur = m.group(1)
        out[i] = cur
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("prefix")
    ap.add_argument("--frames", type=float, default=1)
    a = ap.parse_args()
    maps = {f: spans(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".cuh", ".cu"))}
    per, cur, line = Counter(), "?", None
    samp = Counter()
    reasons = {}
    hdr, sidx = None, []
    total = 0
    by_addr = {}  # an inlined instruction is listed under every source line of its inline chain
    with gzip.open(a.prefix + "_source.csv.gz", "rt") as f:
        for r in csv.reader(f):
            if not r:
                continue
            if r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r[0] == "Line No":  # the stall-reason columns (all samples, not the not-issued copies)
                sidx = [i for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
                hdr = [r[i].replace("stall_", "") for i in sidx]
            if r[0] in ("Function Name", "Line No") or len(r) < 8:
                continue
            if r[0]:
                line = int(r[0]) if r[0].isdigit() else None
                continue
            if len(r) > 3 and r[2].startswith("0x"):
                try:
                    n = int(r[7] or 0)
                    smp = int(r[4] or 0)
                    why = [int(r[i] or 0) for i in sidx] if hdr else []
                except ValueError:
                    continue
                if cur in maps and line:
                    key = f"{cur}:{maps[cur].get(line, '?')}"
                elif cur.startswith("code_"):
                    key = "generated code"
                else:
                    key = cur
                by_addr.setdefault(r[2], [n, [], smp, why])[1].append(key)
    # attribute each instruction once, to the outermost caller that is not a small helper
    helpers = re.compile(r":(h2add|h2minxs|h2max|fminxs|vld|vst|ld|f|g|g0|hd|mag_key|add|acc|acc_neg|v|one|pair|gtid|"
                         r"lane_id|l2_policy|low_mask|smem_u32|unpack_raw|load_raw)$|intrinsics|_rt\.hpp|functions\.hpp")
    for n, keys, smp, why in by_addr.values():
        total += n
        good = [k for k in keys if not helpers.search(k)]
        k = (good or keys)[-1]
        per[k] += n
        samp[k] += smp
        acc = reasons.setdefault(k, Counter())
        for name, c in zip(hdr or [], why):
            acc[name] += c
    ts = max(1, sum(samp.values()))
    print(f"total warp instructions {total:.0f} ({total / a.frames:.0f} per frame); columns: share of instructions, "
          f"instructions per frame, share of warp-stall samples (where the time goes)")
    for k, v in per.most_common(40):
        top = ", ".join(f"{r} {100 * c / max(1, samp[k]):.0f}%" for r, c in reasons.get(k, Counter()).most_common(3))
        print(f"{100 * v / total:5.1f}%  {v / a.frames:9.0f}/frame  {100 * samp[k] / ts:5.1f}%  {k}  [{top}]")


if __name__ == "__main__":
    main()
