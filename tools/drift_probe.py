import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_1504_00353_b200 as pb
N, K, e = 32768, 29492, 4.5
code = pb.PolarCode.ga(N, K, e)
n = 1 << 20
llr = torch.empty(n, N, dtype=torch.int8, device="cuda")
for c in range(0, n, 1 << 17):
    code.gen_bpsk_awgn(1504000353, c, 1 << 17, e, 4.0, llr_i8=llr[c:c + (1 << 17)])
out = torch.empty(n, code.info_words, dtype=torch.int32, device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
one = t(lambda: code.decode_i8(llr, out))
def chunks(m):
    for c in range(0, n, m): code.decode_i8(llr[c:c + m], out[c:c + m])
res = {"one_launch_gbps": n * K / one / 1e6}
for m in (16384, 65536, 262144):
    res[f"chunks_{m}_gbps"] = n * K / t(lambda: chunks(m)) / 1e6
# the same 16K frames repeatedly (small address window)
res["same16k_gbps"] = 16384 * K / t(lambda: code.decode_i8(llr[:16384], out[:16384]), reps=20) / 1e6
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
