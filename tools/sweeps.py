"""The paper's two GPU design sweeps re-run on B200 (tools/variant_build.sh builds, one library
per configuration; every configuration oracle-checked on a sample):

* threads per frame (fig:gpu_threads: (1024,922), "more than 128 threads per block
  negatively affects performance"): the one-CTA-per-frame variant with T threads per CTA and
  CTA-wide ops above a 256-element warp subtree (thr_<T>), at batches of 148 x 4^k frames;
* shared vs global memory (fig:gpu_mem_type: shared memory wins at few blocks,
  global at many): (32768,29492) warp-per-frame variant with the stages of size >= GS in global
  (L2) scratch, the rest in shared memory (mem_<GS>; 65536 = all in shared memory), same batches.

Prints one JSON line per (configuration, batch)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1504_00353_b200 as pb  # noqa: E402


def rate(code, llr, out, reps=5):
    code.decode_i8(llr, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        code.decode_i8(llr, out)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def sweep(tag, lib, N, K, e, variant, batches):
    mask = oracle.construct_ga(N, K, e)
    code = pb.PolarCode(N, K, mask, library=lib)
    code.set_variant(variant)
    nmax = max(batches)
    llr = torch.empty(nmax, N, dtype=torch.int8, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, nmax, e, 4.0, llr_i8=llr)
    out = torch.empty(nmax, code.info_words, dtype=torch.int32, device="cuda")
    idx = np.linspace(0, nmax - 1, 64).astype(np.int64)
    for B in batches:
        ms = rate(code, llr[:B], out[:B])
        print(json.dumps({"config": tag, "code": [N, K], "variant": variant, "batch": B, "ms": ms,
                          "info_gbps": B * K / (ms * 1e-3) / 1e9, "smem_per_cta": code.smem_bytes}), flush=True)
    got = out[idx].cpu().numpy().view(np.uint32)  # the largest batch's output
    want = oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, llr[idx].cpu().numpy(), threads=os.cpu_count())))
    bad = int((got != want).any(axis=1).sum())
    print(json.dumps({"config": tag, "parity_frames_differ": bad, "checked": len(idx)}), flush=True)
    return bad


if __name__ == "__main__":
    bad = 0
    B = [148 * 4 ** k for k in range(6)]  # 148 .. 151,552
    for T in (32, 64, 128, 256, 512):
        bad += sweep(f"thr_{T}", pb._load(os.path.abspath(f"vlibs/thr_{T}.so")), 1024, 922, 4.5, "latency", B)
    for G in (65536, 16384, 8192, 4096, 1024):
        bad += sweep(f"mem_{G}", pb._load(os.path.abspath(f"vlibs/mem_{G}.so")), 32768, 29492, 4.5, "throughput", B[:5])
    sys.exit(1 if bad else 0)
