"""Small decodes for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):
each registered code family and kernel variant (throughput, latency, generic, frame-interleaved,
and the batch-1 mailbox) on a few
frames, checked against the oracle.   usage: compute-sanitizer --tool X python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1504_00353_b200 as pb  # noqa: E402
from seeded_inputs import random_llr_i8, random_mask  # noqa: E402

CASES = [(8, 5, None), (1024, 512, 2.5), (2048, 1723, 4.0), (4096, 2048, 2.5), (8192, 6000, 3.5), (32768, 29492, 4.5)]
bad = 0
for N, K, e in CASES:
    mask = np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8) if e is None else oracle.construct_ga(N, K, e)
    code = pb.PolarCode(N, K, mask)
    n = 7 if N >= 8192 else 37
    x = random_llr_i8(N + 1, (n, N), -60, 60)
    xs = {"i8": x, "f32": x.astype(np.float32)}
    want = {p: oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, v))) for p, v in xs.items()}
    for variant in ("throughput", "latency", "generic", "xframe"):
        code.set_variant(variant)
        for prof in ("i8", "f32"):
            t = torch.from_numpy(xs[prof]).cuda()
            out = (code.decode_i8(t) if prof == "i8" else code.decode_f32(t)).cpu().numpy().view(np.uint32)
            ok = np.array_equal(out, want[prof])
            bad += not ok
            print(f"({N},{K}) {variant:10s} {prof}: {'ok' if ok else 'MISMATCH'}", flush=True)
m = random_mask(5, 256, 100)
os.environ["POLAR_JIT"] = "0"  # the generic decoder itself
code = pb.PolarCode(256, 100, m)
del os.environ["POLAR_JIT"]
x = random_llr_i8(9, (5, 256))
ok = np.array_equal(code.decode_i8(torch.from_numpy(x).cuda()).cpu().numpy().view(np.uint32),
                    oracle.pack_bits(oracle.info_bits(m, oracle.fastssc_decode(m, x))))
bad += not ok
print("generic random mask:", "ok" if ok else "MISMATCH")
# round 2: non-systematic output, a run-time specialised code, a long code (N > 32768)
for N, K, e in [(2048, 1723, 4.0), (32768, 29492, 4.5)]:
    mask = oracle.construct_ga(N, K, e)
    code = pb.PolarCode(N, K, mask)
    code.set_output("nonsystematic")
    x = random_llr_i8(N + 3, (5, N), -60, 60)
    want = oracle.pack_bits(oracle.info_bits(mask, oracle.encode(oracle.fastssc_decode(mask, x))))
    for variant in ("throughput", "latency", "generic"):
        code.set_variant(variant)
        ok = np.array_equal(code.decode_i8(torch.from_numpy(x).cuda()).cpu().numpy().view(np.uint32), want)
        bad += not ok
        print(f"({N},{K}) {variant:10s} non-systematic: {'ok' if ok else 'MISMATCH'}", flush=True)
for N, K, e in [(4096, 2048, 3.0), (65536, 58982, 4.5)]:
    mask = oracle.construct_ga(N, K, e)
    code = pb.PolarCode(N, K, mask)
    x = random_llr_i8(N + 5, (3, N), -60, 60)
    for prof, v in (("i8", x), ("f32", x.astype(np.float32))):
        want = oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, v)))  # per profile (int8 saturates)
        t = torch.from_numpy(v).cuda()
        ok = np.array_equal((code.decode_i8(t) if prof == "i8" else code.decode_f32(t)).cpu().numpy().view(np.uint32), want)
        bad += not ok
        kind = "run-time specialised" if code.run_time_specialised else "long-code generic"
        print(f"({N},{K}) {kind} {prof}: {'ok' if ok else 'MISMATCH'}", flush=True)
# batch-1 mailbox (persistent kernel on host-mapped memory)
for N, K, e in [(2048, 1723, 4.0), (32768, 29492, 4.5)]:
    mask = oracle.construct_ga(N, K, e)
    code = pb.PolarCode(N, K, mask)
    x = random_llr_i8(N + 7, (2, N), -60, 60)
    want = oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, x)))
    code.mailbox_open(idle_seconds=120.0)
    for i in range(2):
        out = np.zeros(code.info_words, np.uint32)
        code.mailbox_decode_i8(np.ascontiguousarray(x[i]), out, timeout_seconds=60.0)
        ok = np.array_equal(out, want[i])
        bad += not ok
        print(f"({N},{K}) mailbox: {'ok' if ok else 'MISMATCH'}", flush=True)
    code.mailbox_close()
sys.exit(1 if bad else 0)
