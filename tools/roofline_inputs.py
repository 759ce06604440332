"""Per-frame SM work of a decode kernel from one ncu --set full capture (tools/ncu_capture.sh),
merged into profiles/roofline_inputs.json under <key>: warp instructions, ALU-pipe warp
instructions, shared-memory wavefronts and DRAM bytes per frame.  bench.py multiplies them by
the frames/s it measures live and divides by the measured SM ceilings (profiles/peaks_sm.json).

usage: python tools/roofline_inputs.py gpurun_out/<capture> <frames> <key>"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prefix, frames, key = sys.argv[1], float(sys.argv[2]), sys.argv[3]
rows = list(csv.reader(open(prefix + "_raw.csv")))
h, u, v = rows[0], rows[1], rows[2]
r = {}
for i, n in enumerate(h):
    try:
        r[n] = (float(v[i].replace(",", "")), u[i])
    except ValueError:
        pass


def val(name, scale_units=True):
    x, unit = r[name]
    if scale_units:
        x *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(unit, 1.0)
    return x


cyc = val("sm__cycles_active.sum")
out = {
    "capture": os.path.basename(prefix),
    "frames": frames,
    "warp_inst_per_frame": val("smsp__inst_executed.sum") / frames,
    # ncu's ALU-pipe peak is 0.5 warp instructions / cycle / SMSP = 2 per SM per cycle
    "alu_warp_inst_per_frame": val("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") / 100 * 2 * cyc / frames,
    "smem_wavefronts_per_frame": val("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / frames,
    "dram_bytes_per_frame": (val("dram__bytes_read.sum") + val("dram__bytes_write.sum")) / frames,
    "issue_active_pct": 100 * val("smsp__issue_active.avg.per_cycle_active"),
    "alu_pipe_pct": val("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
}
path = os.path.join(ROOT, "profiles", "roofline_inputs.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[key] = out
json.dump(d, open(path, "w"), indent=1, sort_keys=True)
print(key, json.dumps(out))
