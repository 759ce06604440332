"""Batch-1 device latency of every kernel variant of a code (CUDA events over back-to-back
launches).  python tools/lat_variants.py [N K ebn0]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1504_00353_b200 as pb  # noqa: E402

N, K, e = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (2048, 1723, 4.0)
code = pb.PolarCode.ga(N, K, e)
llr = torch.empty(1, N, dtype=torch.int8, device="cuda")
llr32 = torch.empty(1, N, dtype=torch.float32, device="cuda")
code.gen_bpsk_awgn(1504000353, 0, 1, e, 4.0, llr_f32=llr32, llr_i8=llr)
out = torch.empty(1, code.info_words, dtype=torch.int32, device="cuda")
res = {"code": [N, K]}
ref = None
for v in ("latency", "throughput", "xframe", "generic"):
    code.set_variant(v)
    for prof, x, fn in (("i8", llr, code.decode_i8), ("f32", llr32, code.decode_f32)):
        for _ in range(20):
            fn(x, out)
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(200):
            fn(x, out)
        t.record()
        torch.cuda.synchronize()
        res[f"{v}_{prof}_us"] = round(s.elapsed_time(t) / 200 * 1e3, 2)
        ref = out.clone() if ref is None else ref
        assert torch.equal(out, ref), v
print(json.dumps(res))
