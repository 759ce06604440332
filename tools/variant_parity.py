"""Parity of an experiment library (POLAR_LIB=...) against the oracle on one code:
python tools/variant_parity.py N K ebn0 n_frames [variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1504_00353_b200 as pb  # noqa: E402

N, K, e, n = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
variant = sys.argv[5] if len(sys.argv) > 5 else "throughput"
mask = oracle.construct_ga(N, K, e)
code = pb.PolarCode(N, K, mask)
code.set_variant(variant)
bad = 0
for prof in ("i8", "f32"):
    llr = torch.empty(n, N, dtype=torch.int8 if prof == "i8" else torch.float32, device="cuda")
    code.gen_bpsk_awgn(99, 0, n, e - 0.5, 4.0, **({"llr_i8": llr} if prof == "i8" else {"llr_f32": llr}))
    out = (code.decode_i8 if prof == "i8" else code.decode_f32)(llr).cpu().numpy().view(np.uint32)
    x = llr.cpu().numpy()
    want = oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, x, threads=os.cpu_count())))
    b = int((out != want).any(axis=1).sum())
    bad += b
    print(f"{os.environ.get('POLAR_LIB', 'libpolar.so')} ({N},{K}) {prof} {variant}: {b} of {n} frames differ")
sys.exit(1 if bad else 0)
