"""Frame-interleaved variant: equality with the warp-cooperative throughput variant on every
registered code (both are parity-tested against the oracle in tests/), and CUDA-event timing
of both on the bench workloads.  Usage (GPU box): python tools/xf_check.py [--time-only]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_00353_b200 as pb  # noqa: E402


def frames(code, n, ebn0, seed=7):
    llr = torch.empty(n, code.N, dtype=torch.int8, device="cuda")
    info = torch.empty(n, code.info_words, dtype=torch.int32, device="cuda")
    try:
        code.gen_bpsk_awgn(seed, 0, n, ebn0, 4.0, llr_i8=llr, info=info)
    except pb.PolarError:  # not superset-closed (random masks): noisy all-zero codeword
        g = torch.Generator(device="cuda").manual_seed(seed)
        llr = (12 + 12 * torch.randn(n, code.N, generator=g, device="cuda")).round().clamp(-128, 127).to(torch.int8)
    return llr, info


def timed(code, llr, reps=5):
    out = torch.empty(llr.shape[0], code.info_words, dtype=torch.int32, device="cuda")
    for _ in range(2):
        code.decode_i8(llr, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        code.decode_i8(llr, out=out)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    time_only = "--time-only" in sys.argv
    if not time_only:
        bad = 0
        for N, K, m in pb.registry():
            code = pb.PolarCode(N, K, m)
            n = 4099 if N <= 4096 else 1000
            for e in (1.0, 3.0, 5.0):
                llr, _ = frames(code, n, e)
                # adversarial: full int8 range incl. -128 on a slice
                g = torch.Generator(device="cuda").manual_seed(N + K)
                llr[: n // 8] = torch.randint(-128, 128, (n // 8, N), generator=g, device="cuda", dtype=torch.int32).to(torch.int8)
                llr[n // 8 : n // 4] = torch.randint(-2, 3, (n // 4 - n // 8, N), generator=g, device="cuda", dtype=torch.int32).to(torch.int8)
                code.set_variant("throughput")
                a = code.decode_i8(llr)
                code.set_variant("xframe")
                b = code.decode_i8(llr)
                torch.cuda.synchronize()
                d = (a != b).any(dim=1).nonzero().flatten()
                if d.numel():
                    bad += 1
                    print(f"MISMATCH ({N},{K}) ebn0={e}: {d.numel()} frames differ, first {d[:8].tolist()}")
            print(f"({N},{K}) checked", flush=True)
        print("xf equality:", "FAIL" if bad else "ok")
    for (N, K, e, n) in [(2048, 1723, 4.0, 1 << 20), (32768, 29492, 4.5, 16384), (32768, 29492, 4.5, 65536),
                         (1024, 512, 2.5, 1 << 20)]:
        code = pb.PolarCode.ga(N, K, e)
        llr, _ = frames(code, n, e)
        r = {"code": [N, K], "n": n}
        for v in ("throughput", "xframe"):
            code.set_variant(v)
            ms = timed(code, llr)
            r[v] = {"ms": ms, "gbps": n * K / ms / 1e6}
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
