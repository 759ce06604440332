"""Per-op latency breakdown of the batch-1 decode (latency variant) from a POLAR_TRACE build.

usage: POLAR_LIB=variants/T/libpolar.so python tools/trace_latency.py --labels variants/T/build/gen/trace_c32768_29492.txt
Runs a few warm batch-1 decodes, reads the clock64() stamps recorded after each op of frame 0
and prints the time per op kind / node size and per tree level (the north star's "latency
per tree level").  Stamps are SM clocks of block 0, thread 0.
"""
import argparse
import os
import re
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_00353_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--labels", required=True)
ap.add_argument("--N", type=int, default=32768)
ap.add_argument("--K", type=int, default=29492)
ap.add_argument("--ebn0", type=float, default=4.5)
ap.add_argument("--prof", default="i8")
a = ap.parse_args()
labels = [l.rstrip("\n") for l in open(a.labels)]
code = pb.PolarCode.ga(a.N, a.K, a.ebn0)
code.set_variant("latency")
dt = torch.int8 if a.prof == "i8" else torch.float32
llr = torch.empty(1, a.N, dtype=dt, device="cuda")
code.gen_bpsk_awgn(1504000353, 0, 1, a.ebn0, 4.0, **({"llr_i8": llr} if a.prof == "i8" else {"llr_f32": llr}))
fn = code.decode_i8 if a.prof == "i8" else code.decode_f32
out = fn(llr)
for _ in range(20):
    fn(llr, out)
torch.cuda.synchronize()
st = code.trace(len(labels)).astype(np.int64)
d = np.diff(st)
total = st[-1] - st[0]
print(f"code ({a.N},{a.K}) {a.prof}: {len(labels)} marks, {total} cycles from first to last op stamp")
kind = defaultdict(lambda: [0, 0])
level = defaultdict(lambda: [0, 0])
for i in range(1, len(labels)):
    lab = labels[i]
    m = re.match(r"(cta:)?([A-Za-z_0-9]+)(?:<(?:P, T, )?(\d+))?", lab)
    k = (("cta " if m.group(1) else "warp ") + m.group(2), int(m.group(3) or 0))
    kind[k][0] += int(d[i - 1])
    kind[k][1] += 1
    lv = k[1]
    level[lv][0] += int(d[i - 1])
    level[lv][1] += 1
print(f"{'op':24s} {'N_v':>6s} {'count':>6s} {'cycles':>9s} {'share':>6s} {'cyc/op':>7s}")
for (op, nv), (cy, c) in sorted(kind.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{op:24s} {nv:6d} {c:6d} {cy:9d} {100 * cy / total:5.1f}% {cy / c:7.1f}")
print("\nper node size (tree level):")
for nv, (cy, c) in sorted(level.items()):
    print(f"  N_v={nv:6d}: {c:5d} ops {cy:9d} cycles {100 * cy / total:5.1f}%")
