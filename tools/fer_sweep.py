"""FER / BER sweep (BASELINE config 4) and batch-size throughput sweep (config 5).

  python tools/fer_sweep.py fer   [--code 32768,27568 --design 4.0 --points 3.5,3.75,4.0,4.25 ...]
  python tools/fer_sweep.py batch [--code 2048,1723 --design 4.0 --max-log4 11]

fer: for each Eb/N0 point, decode seeded frames (device generator, mask fixed at the design
Eb/N0, reading C1) in chunks until `--errors` frame errors or `--max-frames`; every frame the GPU
decodes wrongly plus `--check` random frames per point are re-decoded by the CPU oracle (O2)
and must match bit for bit; prints FER/BER with Clopper-Pearson 95% intervals next to the GA
closed-form estimate 1 - prod(1 - Q(sqrt(m_i / 2))) over the information set (SURVEY 8(c) pin 9).
batch: info Gbps and frames/s of the int8 decoder for batches 4^0 .. 4^max (CUDA events).
Writes one JSON line per point to stdout.
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy.stats import beta as beta_dist  # noqa: E402

import oracle  # noqa: E402  (test/measurement infrastructure: the checker)
import paper_1504_00353_b200 as pb  # noqa: E402

SEED = 1504000353


# ------------------------------------------------------------------ checkpoint / resume
# Every finished point is one JSON line; with --out FILE the lines are also appended (and
# flushed) to FILE, and --resume skips the points FILE already holds, so a sweep cut off by a
# time limit (the FER-1e-8 points take GPU-hours) restarts where it stopped.
_OUT = None


def point_key(d):
    """Identity of a finished point: (code, design, Eb/N0, profile[, first frame, frame cap])."""
    k = (tuple(d["code"]), float(d["design_ebn0"]), float(d["ebn0"]), d["profile"])
    return k + ((int(d["first_frame"]), int(d.get("max_frames", d["frames"]))) if "first_frame" in d else ())


def completed(path):
    done = set()
    if path and os.path.exists(path):
        for line in open(path):
            line = line.strip()
            if line.startswith("{"):
                try:
                    done.add(point_key(json.loads(line)))
                except (KeyError, ValueError):
                    pass
    return done


def emit(d):
    line = json.dumps(d)
    print(line, flush=True)
    if _OUT:
        with open(_OUT, "a") as f:
            f.write(line + "\n")
            f.flush()
            os.fsync(f.fileno())


def clopper_pearson(k, n, a=0.05):
    lo = 0.0 if k == 0 else beta_dist.ppf(a / 2, k, n - k + 1)
    hi = 1.0 if k == n else beta_dist.ppf(1 - a / 2, k + 1, n - k)
    return lo, hi


def ga_fer(N, K, design, ebn0):
    mask = oracle.construct_ga(N, K, design)
    m = oracle.ga_means(N, K, ebn0)[mask == 0]
    q = 0.5 * np.array([math.erfc(math.sqrt(x / 2) / math.sqrt(2)) for x in m])
    return float(1.0 - np.prod(1.0 - q))


def fer(a):
    N, K = map(int, a.code.split(","))
    code = pb.PolarCode.ga(N, K, a.design)
    mask = code.mask()
    W = code.info_words
    chunk = a.chunk
    llr8 = torch.empty(chunk, N, dtype=torch.int8, device="cuda")
    llr32 = torch.empty(chunk, N, dtype=torch.float32, device="cuda") if a.f32 else None
    truth = torch.empty(chunk, W, dtype=torch.int32, device="cuda")
    out = torch.empty(chunk, W, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(7)
    done = completed(a.out) if a.resume else set()
    for e in [float(x) for x in a.points.split(",")]:
        for prof in (["i8", "f32"] if a.f32 else ["i8"]):
            if ((N, K), a.design, e, prof) in done:
                print(f"resume: skipping ({N},{K}) {e} dB {prof}", file=sys.stderr)
                continue
            frames = bit_err = frame_err = checked = 0
            first = 0
            t0 = time.time()
            while frame_err < a.errors and frames < a.max_frames:
                n = min(chunk, a.max_frames - frames)
                code.gen_bpsk_awgn(SEED, first, n, e, 4.0, llr_f32=llr32[:n] if prof == "f32" else None,
                                   llr_i8=llr8[:n] if prof == "i8" else None, info=truth[:n])
                x = llr8[:n] if prof == "i8" else llr32[:n]
                (code.decode_i8 if prof == "i8" else code.decode_f32)(x, out[:n])
                d = (out[:n] ^ truth[:n]).cpu().numpy().view(np.uint32)
                bad = np.flatnonzero(d.any(axis=1))
                frame_err += len(bad)
                bit_err += int(np.unpackbits(d.view(np.uint8)).sum())
                # oracle re-decode of the GPU's error frames and of a random sample
                idx = np.union1d(bad[: a.check], rng.choice(n, min(a.check, n), replace=False))
                sample = x[torch.from_numpy(idx).cuda()].cpu().numpy()
                want = oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, sample, threads=os.cpu_count())))
                got = out[:n][torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint32)
                if not np.array_equal(got, want):
                    raise SystemExit(f"PARITY FAILURE at {e} dB {prof}: {int((got != want).any(axis=1).sum())} frames")
                checked += len(idx)
                frames += n
                first += n
            lo, hi = clopper_pearson(frame_err, frames)
            emit({"code": [N, K], "design_ebn0": a.design, "ebn0": e, "profile": prof, "frames": frames,
                  "frame_errors": frame_err, "fer": frame_err / frames, "fer_ci95": [lo, hi],
                  "ber": bit_err / (frames * K), "ga_fer": ga_fer(N, K, a.design, e),
                  "oracle_checked_frames": checked, "seconds": round(time.time() - t0, 2)})


def ferfast(a):
    """FER segment for the FER-1e-8 regime: frames [first, first + max)
    at one Eb/N0, errors counted on the device (polar_count_errors); only error frames (and a few
    random ones) come back to the host, where the oracle re-decodes them bit for bit.  Segments
    over disjoint frame ranges are independent samples and add up."""
    N, K = map(int, a.code.split(","))
    code = pb.PolarCode.ga(N, K, a.design)
    mask = code.mask()
    W = code.info_words
    chunk = a.chunk
    e = float(a.points)
    prof = "f32" if a.f32 else "i8"
    if a.resume and ((N, K), a.design, e, prof, a.first_frame, a.max_frames) in completed(a.out):
        print(f"resume: segment ({N},{K}) {e} dB {prof} from frame {a.first_frame} already done", file=sys.stderr)
        return
    x = torch.empty(chunk, N, dtype=torch.float32 if a.f32 else torch.int8, device="cuda")
    truth = torch.empty(chunk, W, dtype=torch.int32, device="cuda")
    out = torch.empty(chunk, W, dtype=torch.int32, device="cuda")
    ctr = torch.zeros(3, dtype=torch.int64, device="cuda")
    rng = np.random.default_rng(a.first_frame + 11)
    frames = checked = 0
    err_frames = []
    t0 = time.time()
    dec = code.decode_f32 if a.f32 else code.decode_i8
    while frames < a.max_frames and time.time() - t0 < a.max_seconds:
        n = min(chunk, a.max_frames - frames)
        first = a.first_frame + frames
        code.gen_bpsk_awgn(SEED, first, n, e, 4.0, llr_f32=x[:n] if a.f32 else None,
                           llr_i8=None if a.f32 else x[:n], info=truth[:n])
        dec(x[:n], out[:n])
        before = int(ctr[2])
        code.count_errors(out[:n], truth[:n], ctr)
        nerr = int(ctr[2]) - before
        idx = []
        if nerr:
            bad = (out[:n] != truth[:n]).any(dim=1).nonzero().flatten().cpu().numpy()
            err_frames += [int(first + i) for i in bad]
            idx = list(bad[: a.check])
        if (frames // chunk) % 64 == 0:
            idx += list(rng.choice(n, 2, replace=False))
        if idx:
            idx = np.unique(np.array(idx, dtype=np.int64))
            sample = x[torch.from_numpy(idx).cuda()].cpu().numpy()
            want = oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, sample, threads=os.cpu_count())))
            got = out[:n][torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint32)
            if not np.array_equal(got, want):
                raise SystemExit(f"PARITY FAILURE at {e} dB {prof} frames {idx.tolist()}")
            checked += len(idx)
        frames += n
    torch.cuda.synchronize()
    f_, be, fe = ctr.tolist()
    emit({"code": [N, K], "design_ebn0": a.design, "ebn0": e, "profile": prof,
          "first_frame": a.first_frame, "frames": f_, "max_frames": a.max_frames, "frame_errors": fe, "bit_errors": be,
          "error_frames": err_frames, "oracle_checked_frames": checked, "seconds": round(time.time() - t0, 1)})


def batch(a):
    N, K = map(int, a.code.split(","))
    code = pb.PolarCode.ga(N, K, a.design)
    W = code.info_words
    nmax = 4 ** a.max_log4
    llr = torch.empty(nmax, N, dtype=torch.int8, device="cuda")
    code.gen_bpsk_awgn(SEED, 0, nmax, a.design, 4.0, llr_i8=llr)
    out = torch.empty(nmax, W, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    for k in range(a.max_log4 + 1):
        n = 4 ** k
        for _ in range(3):
            code.decode_i8(llr[:n], out[:n])
        reps = max(3, min(200, (1 << 22) // n))
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        for _ in range(reps):
            code.decode_i8(llr[:n], out[:n])
        ev1.record(s)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / reps
        print(json.dumps({"code": [N, K], "batch": n, "ms": ms, "frames_per_s": n / (ms * 1e-3),
                          "info_gbps": n * K / (ms * 1e-3) / 1e9,
                          "variant": "latency" if n <= torch.cuda.get_device_properties(0).multi_processor_count else "throughput"}),
              flush=True)


def idud(a):
    """Instruction-based (generic, interpreted) vs unrolled (specialised) decoder on the same
    code -- the GPU analogue of the paper's tab:impl:tp:algo-unroll."""
    N, K = map(int, a.code.split(","))
    code = pb.PolarCode.ga(N, K, a.design)
    W = code.info_words
    s = torch.cuda.current_stream()
    for batch in (1, a.batch):
        llr = torch.empty(batch, N, dtype=torch.int8, device="cuda")
        code.gen_bpsk_awgn(SEED, 0, batch, a.design, 4.0, llr_i8=llr)
        out = torch.empty(batch, W, dtype=torch.int32, device="cuda")
        ref = None
        for variant in ("auto", "generic"):
            code.set_variant(variant)
            for _ in range(3):
                code.decode_i8(llr, out)
            reps = 50 if batch == 1 else 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                code.decode_i8(llr, out)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), "generic and unrolled decoders disagree"
            print(json.dumps({"code": [N, K], "decoder": "unrolled" if variant == "auto" else "instruction-based",
                              "batch": batch, "us": ms * 1e3, "info_gbps": batch * K / (ms * 1e-3) / 1e9}), flush=True)
    code.set_variant("auto")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["fer", "ferfast", "batch", "idud"])
    ap.add_argument("--first-frame", type=int, default=0)
    ap.add_argument("--max-seconds", type=float, default=1e9)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--code", default="32768,27568")
    ap.add_argument("--design", type=float, default=4.0)
    ap.add_argument("--points", default="3.5,3.75,4.0,4.25")
    ap.add_argument("--errors", type=int, default=100)
    ap.add_argument("--max-frames", type=int, default=20_000_000)
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--check", type=int, default=64)
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--max-log4", type=int, default=8)
    ap.add_argument("--out", default=None, help="also append every finished point to this JSON-lines file")
    ap.add_argument("--resume", action="store_true", help="skip the points --out already holds")
    a = ap.parse_args()
    _OUT = a.out
    {"fer": fer, "ferfast": ferfast, "batch": batch, "idud": idud}[a.mode](a)
