"""Batch-1 device latency without host submission gaps: 100 single-frame decode calls
captured into one CUDA graph, replayed; CUDA events around the replay / 100.
python tools/lat_graph.py N K ebn0 [variant ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1504_00353_b200 as pb  # noqa: E402


def graph_latency(code, fn, x, out, reps=100, rounds=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(5):
            fn(x, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn(x, out)
    g.replay()
    torch.cuda.synchronize()
    best = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best.append(a.elapsed_time(b) * 1e3 / reps)
    best.sort()
    return best[len(best) // 2]


if __name__ == "__main__":
    N, K, e = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
    variants = sys.argv[4:] or ["latency", "throughput"]
    code = pb.PolarCode.ga(N, K, e)
    llr = torch.empty(1, N, dtype=torch.int8, device="cuda")
    llr32 = torch.empty(1, N, dtype=torch.float32, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, 1, e, 4.0, llr_f32=llr32, llr_i8=llr)
    out = torch.empty(1, code.info_words, dtype=torch.int32, device="cuda")
    res = {"code": [N, K]}
    for v in variants:
        code.set_variant(v)
        for prof, x, fn in (("i8", llr, code.decode_i8), ("f32", llr32, code.decode_f32)):
            res[f"{v}_{prof}_us"] = round(graph_latency(code, fn, x, out), 2)
    print(json.dumps(res), flush=True)
