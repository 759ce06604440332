"""Run a few decode launches of one code (for ncu captures; not a benchmark)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1504_00353_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=32768)
ap.add_argument("--K", type=int, default=29492)
ap.add_argument("--ebn0", type=float, default=4.5)
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--prof", default="i8", choices=["i8", "f32"])
ap.add_argument("--variant", default="auto", choices=["auto", "throughput", "latency", "generic", "xframe"])
a = ap.parse_args()
code = pb.PolarCode.ga(a.N, a.K, a.ebn0)
code.set_variant(a.variant)
dt = torch.int8 if a.prof == "i8" else torch.float32
llr = torch.empty(a.batch, a.N, dtype=dt, device="cuda")
code.gen_bpsk_awgn(1504000353, 0, a.batch, a.ebn0, 4.0, **({"llr_i8": llr} if a.prof == "i8" else {"llr_f32": llr}))
fn = code.decode_i8 if a.prof == "i8" else code.decode_f32
out = fn(llr)
for _ in range(a.iters):
    fn(llr, out)
torch.cuda.synchronize()
print("done", a.N, a.K, a.prof, a.batch)
