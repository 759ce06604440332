"""Throughput of one code alone (for experiment builds holding a subset of the codes):
python tools/tp_bench.py N K ebn0 batch [prof]   -> one JSON line, info Gbps (median of 5 runs
of 5 launches, CUDA events, inputs resident in HBM, generated once)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1504_00353_b200 as pb  # noqa: E402

N, K, e, B = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
prof = sys.argv[5] if len(sys.argv) > 5 else "i8"
code = pb.PolarCode.ga(N, K, e)
llr = torch.empty(B, N, dtype=torch.int8 if prof == "i8" else torch.float32, device="cuda")
code.gen_bpsk_awgn(1504000353, 0, B, e, 4.0, **({"llr_i8": llr} if prof == "i8" else {"llr_f32": llr}))
fn = code.decode_i8 if prof == "i8" else code.decode_f32
out = fn(llr)
for _ in range(3):
    fn(llr, out)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn(llr, out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 5)
ms = sorted(ts)[2]
print(json.dumps({"code": [N, K], "prof": prof, "batch": B, "ms": ms, "info_gbps": B * K / ms / 1e6}))
