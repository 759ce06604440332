"""Host-observed batch-1 latency through the mailbox (wall clock per call, p50 of 2000)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1504_00353_b200 as pb
res = {"wc": os.environ.get("POLAR_MAILBOX_WC", "1")}
for (N, K, e) in [(2048, 1723, 4.0), (32768, 29492, 4.5)]:
    code = pb.PolarCode.ga(N, K, e)
    llr = torch.empty(1, N, dtype=torch.int8, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, 1, e, 4.0, llr_i8=llr)
    hx = llr.cpu().numpy().reshape(-1).copy()
    out = np.zeros(code.info_words, np.uint32)
    code.mailbox_open(idle_seconds=30)
    for _ in range(100):
        code.mailbox_decode_i8(hx, out)
    t = []
    for _ in range(2000):
        t0 = time.perf_counter_ns()
        code.mailbox_decode_i8(hx, out)
        t.append((time.perf_counter_ns() - t0) / 1e3)
    code.mailbox_close()
    res[f"{N}_{K}_p50_us"] = round(float(np.median(t)), 2)
print(json.dumps(res))
