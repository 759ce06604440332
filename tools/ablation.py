"""The paper's algorithm ablation on B200 (tab:impl:tp:algo-unroll): the same
unrolled-decoder generator restricted to node sets (plain SC, SSC, Fast-SSC without SPC -- the
paper's GPU set, P:1134-1136 -- and Fast-SSC), each built into its own library
(tools/variant_build.sh ab_<set> variants/specs/ab_<set>.txt), plus the program-interpreted
decoder (the paper's instruction-based decoder).  For each: oracle parity on 2,000
frames (oracle.nodeset_decode, the same node set), int8/f32 throughput on 1M frames and
batch-1 device latency (CUDA graph of 100 single-frame launches).  One JSON line per decoder."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1504_00353_b200 as pb  # noqa: E402

N, K, E = 2048, 1707, 4.51
mask = oracle.construct_ga(N, K, E)


def timed(fn, reps=5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def graph_us(code, x, out, reps=100):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            code.decode_i8(x, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            code.decode_i8(x, out)
    return timed(g.replay) * 1e3 / reps


def run(tag, node_set, lib, variant="auto"):
    code = pb.PolarCode(N, K, mask, library=lib)
    code.set_variant(variant)
    n = 1 << 20
    llr = torch.empty(n, N, dtype=torch.int8, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, n, E, 4.0, llr_i8=llr)
    out = torch.empty(n, code.info_words, dtype=torch.int32, device="cuda")
    ms = timed(lambda: code.decode_i8(llr, out))
    res = {"decoder": tag, "node_set": node_set, "n_ops": code.n_ops, "i8_gbps": n * K / ms / 1e6}
    got = out[:2000].cpu().numpy().view(np.uint32)
    x = llr[:2000].cpu().numpy()
    want = oracle.pack_bits(oracle.info_bits(mask, oracle.nodeset_decode(mask, x, node_set, threads=os.cpu_count())))
    res["parity_i8_frames_differ"] = int((got != want).any(axis=1).sum())
    del llr
    n32 = 1 << 18
    l32 = torch.empty(n32, N, dtype=torch.float32, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, n32, E, 4.0, llr_f32=l32)
    o32 = torch.empty(n32, code.info_words, dtype=torch.int32, device="cuda")
    ms = timed(lambda: code.decode_f32(l32, o32))
    res["f32_gbps"] = n32 * K / ms / 1e6
    got = o32[:2000].cpu().numpy().view(np.uint32)
    want = oracle.pack_bits(oracle.info_bits(mask, oracle.nodeset_decode(mask, l32[:2000].cpu().numpy(), node_set,
                                                                          threads=os.cpu_count())))
    res["parity_f32_frames_differ"] = int((got != want).any(axis=1).sum())
    del l32
    x1 = torch.empty(1, N, dtype=torch.int8, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, 1, E, 4.0, llr_i8=x1)
    o1 = torch.empty(1, code.info_words, dtype=torch.int32, device="cuda")
    res["batch1_graph_us_i8"] = graph_us(code, x1, o1)
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    bad = 0
    for s in ("sc", "ssc", "nospc", "fastssc"):
        r = run(f"unrolled ({s})", s, pb._load(os.path.abspath(f"vlibs/ab_{s}.so")))
        bad += r["parity_i8_frames_differ"] + r["parity_f32_frames_differ"]
    r = run("instruction-based (generic)", "fastssc", pb.lib(), variant="generic")
    bad += r["parity_i8_frames_differ"] + r["parity_f32_frames_differ"]
    sys.exit(1 if bad else 0)
