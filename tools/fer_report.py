"""Merge `fer_sweep.py ferfast` segments (JSON lines) into the FER-1e-8 report of SURVEY 8(f) N2:
the paper's claim that 8-bit LLRs lose < 0.025 dB against float at FER 1e-8 for (32768,27568)
(P:486).  The int8 and f32 runs decode the SAME seeded frames (frame index -> noise), so the
comparison is paired: on the frame range both profiles covered, count the error frames they
share and those only one of them got.
Usage: python tools/fer_report.py seg1.json [seg2.json ...] > report.md"""
import json
import math
import sys

from scipy.stats import beta as beta_dist, binomtest


def cp(k, n, a=0.05):
    lo = 0.0 if k == 0 else beta_dist.ppf(a / 2, k, n - k + 1)
    hi = 1.0 if k == n else beta_dist.ppf(1 - a / 2, k + 1, n - k)
    return lo, hi


def prefix(ranges):
    """End of the contiguous run of frame ranges that starts at frame 0."""
    end = 0
    for a, b in sorted(ranges):
        if a > end:
            break
        end = max(end, b)
    return end


def main(paths):
    segs = [json.loads(l) for p in paths for l in open(p) if l.strip().startswith("{")]
    by = {}
    for s in segs:
        key = (tuple(s["code"]), s["ebn0"], s["profile"])
        d = by.setdefault(key, {"ranges": [], "errors": set(), "frames": 0, "fe": 0, "be": 0, "checked": 0, "sec": 0.0})
        d["ranges"].append((s["first_frame"], s["first_frame"] + s["frames"]))
        d["errors"].update(s["error_frames"])
        d["frames"] += s["frames"]
        d["fe"] += s["frame_errors"]
        d["be"] += s["bit_errors"]
        d["checked"] += s["oracle_checked_frames"]
        d["sec"] += s["seconds"]
    print("| code | Eb/N0 | profile | frames | frame errors | FER | 95% CI | BER | oracle-checked | s |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for (code, e, prof), d in sorted(by.items()):
        lo, hi = cp(d["fe"], d["frames"])
        K = code[1]
        print(f"| {code} | {e} | {prof} | {d['frames']:,} | {d['fe']} | {d['fe'] / d['frames']:.3g} | "
              f"[{lo:.3g}, {hi:.3g}] | {d['be'] / (d['frames'] * K):.3g} | {d['checked']} | {d['sec']:.0f} |")
    # paired comparison on the common prefix [0, m)
    for (code, e, prof), d in sorted(by.items()):
        if prof != "i8" or (code, e, "f32") not in by:
            continue
        f = by[(code, e, "f32")]
        m = min(prefix(d["ranges"]), prefix(f["ranges"]))
        ei = {x for x in d["errors"] if x < m}
        ef = {x for x in f["errors"] if x < m}
        both, only_i, only_f = len(ei & ef), len(ei - ef), len(ef - ei)
        print()
        print(f"Paired on frames [0, {m:,}) of {code} at {e} dB: int8 errors {len(ei)}, f32 errors {len(ef)}, "
              f"shared {both}, int8 only {only_i}, f32 only {only_f}.")
        if only_i + only_f:
            p = binomtest(only_i, only_i + only_f, 0.5).pvalue
            print(f"Exact two-sided sign test on the discordant frames: p = {p:.3g}.")
        if len(ef):
            r = len(ei) / len(ef)
            print(f"FER ratio int8/f32 = {r:.3g}" + (f" (= {math.log10(r):+.3f} decades)" if r > 0 else "") + ".")


if __name__ == "__main__":
    main(sys.argv[1:])
