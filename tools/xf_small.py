import json, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1504_00353_b200 as pb
sys.path.insert(0, "tools")
from xf_check import frames, timed
for (N, K, e) in [(1024, 922, 4.5), (1024, 512, 2.5), (512, 400, 3.5), (256, 128, 2.0), (64, 32, 2.0)]:
    code = pb.PolarCode.ga(N, K, e)
    n = (1 << 26) // N
    llr, _ = frames(code, n, e)
    r = {"code": [N, K], "n": n}
    for v in ("throughput", "xframe"):
        code.set_variant(v)
        ms = timed(code, llr)
        r[v] = round(n * K / ms / 1e6, 1)
    print(json.dumps(r), flush=True)
