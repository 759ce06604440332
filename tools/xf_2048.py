"""(2048,1723) int8, 1M frames: warp-per-frame vs frame-interleaved, Gbps (CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1504_00353_b200 as pb  # noqa: E402
from xf_check import frames, timed  # noqa: E402
code = pb.PolarCode.ga(2048, 1723, 4.0)
n = 1 << 20
llr, _ = frames(code, n, 4.0)
r = {}
for v in ("throughput", "xframe", "throughput", "xframe"):
    code.set_variant(v)
    r.setdefault(v, []).append(round(n * 1723 / timed(code, llr, reps=10) / 1e6, 1))
print(json.dumps(r))
