"""Benchmark of the B200 Fast-SSC polar decoder (the driver's bench contract).

One step = one polar_decode_i8 call over a batch of B frames of the (32768,29492) code
(BASELINE.json's metric code; int8 profile), LLRs resident in HBM (B*N bytes > L2, so no
flush is needed).  value = information bits decoded per second over all ranks (Gbps).

Also reported on the same line:
  e2e            the same metric through polar_decode_i8_host (pinned host LLRs -> device ->
                 host info bits, copies inside the timed region);
  latency        batch-1 single-frame decode time (config 3), kernel-only (CUDA events);
  roofline       the decode kernel against the ALU issue ceiling;
  cpu_baseline   the CPU oracle (oracle/, plain C) on a bounded sample, rank 0 only;
  extra          the (2048,1723) int8 throughput (config 2) and FER/BER of the timed frames.

--impl reference times the CPU oracle instead (the reference arm of this tier).
Multi-GPU: torchrun, one rank per GPU, frames sharded (weak scaling), NCCL all-reduce of
the error counters and MAX of the elapsed time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 1504000353
CODE = (32768, 29492, 4.5)       # config 3/5 code, design = operating Eb/N0 (reading C1)
CODE2 = (2048, 1723, 4.0)        # config 2 code
BATCH = 16384                    # frames per step per GPU for N=32768 (512 MiB of int8 LLRs)
BATCH2 = 1 << 20                 # frames per step per GPU for N=2048 (2 GiB)


def _relaunch(argv, n):
    """`python bench.py --gpus N` outside torchrun: start N ranks under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the NCCL log shows every rank and the transport
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr, so stdout keeps one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """Samples SM clocks and throttle reasons during the timed region: NVML in-process every
    1 ms (the timed region is tens of ms), nvidia-smi as a fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._nv = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._masks = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                           pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _poll(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((float(sm), float(self._max), [bool(r & m) for m in self._masks]))
            except Exception:
                pass
            time.sleep(0.001)

    def _read_smi(self):
        for line in self._p.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) == 6 and f[0].replace(".", "").isdigit():
                self.rows.append((float(f[0]), float(f[1]), [x.lower() == "active" for x in f[2:6]]))

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        self._p = None
        try:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read_smi, daemon=True)
            self._t.start()
        except FileNotFoundError:
            pass
        return self

    def __exit__(self, *a):
        if self._nv is not None:
            self._stop.set()
            self._t.join()
        elif self._p:
            time.sleep(0.15)
            self._p.terminate()
            self._p.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2][i]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nv is not None else "nvidia-smi"}


def cpu_oracle_rate(N, K, e, sample_frames, threads, min_seconds=0.0):
    """Oracle O2 (plain C Fast-SSC) on host cores: info bits/s over a bounded sample -- a tile
    of `sample_frames` frames (64 seeded AWGN frames repeated), decoded repeatedly until at
    least `min_seconds` have elapsed."""
    import oracle
    from seeded_inputs import bpsk_awgn_llr, draw, quantize_i8

    mask = oracle.construct_ga(N, K, e)
    base = 64
    bits, noise = draw(SEED, 0, base, K, N)
    q = quantize_i8(bpsk_awgn_llr(oracle.encode_systematic(mask, bits), noise, e, K))
    reps = max(1, sample_frames // base)
    llr = np.ascontiguousarray(np.tile(q, (reps, 1)))
    n = 0
    t0 = time.perf_counter()
    while True:
        oracle.fastssc_decode(mask, llr, threads=threads)
        n += llr.shape[0]
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return n * K / dt, n, dt


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    N, K, e = CODE
    cores = os.cpu_count() or 1
    samples = []
    for _ in range(args.warmup):
        cpu_oracle_rate(N, K, e, 256, cores)
    for _ in range(args.steps):
        r, n, dt = cpu_oracle_rate(N, K, e, 512, cores)
        samples.append((r, n, dt))
    rate = sum(s[1] for s in samples) * K / sum(s[2] for s in samples)
    v = rate / 1e9
    ms = 1e3 * float(np.mean([s[2] for s in samples]))
    line = {"impl": "reference", "metric": "info_gbps", "value": v, "unit": "Gbps", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": f"({N},{K}) int8 Fast-SSC, CPU oracle, 512-frame sample per step",
                       "code": [N, K], "ebn0_db": e, "global_batch": 512, "parallelism": "host threads"},
            "cpu_baseline": {"value": v, "unit": "Gbps", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} x 512 frames of ({N},{K}) int8 (64 seeded AWGN frames tiled)"},
            "e2e": {"value": v, "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-extra", action="store_true", help="skip the (2048,1723) and latency legs")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: exercise the multi-rank path on one GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(sys.argv[1:], args.gpus))
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1504_00353_b200 as pb
    from paper_1504_00353_b200.shard import allreduce_counters, frame_range

    ws, rank, local = _dist()
    if ws != args.gpus:
        print(f"bench: WORLD_SIZE={ws} but --gpus {args.gpus}; reporting the {ws} ranks that run", file=sys.stderr)
    # one rank per GPU; with fewer GPUs than ranks (the gloo check on a 1-GPU lease) ranks share
    ndev = torch.cuda.device_count()
    local = local % max(1, ndev)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    def barrier():
        if ws > 1:
            dist.barrier()

    from paper_1504_00353_b200.shard import max_over_ranks as _mor

    def max_over_ranks(x: float) -> float:
        return _mor(x, dev if args.backend == "nccl" else None)

    def throughput(code_t, B, steps, warmup, with_e2e, prof="i8"):
        N, K, e = code_t
        code = pb.PolarCode.ga(N, K, e)
        llr = torch.empty(B, N, dtype=torch.int8 if prof == "i8" else torch.float32, device=dev)
        truth = torch.empty(B, code.info_words, dtype=torch.int32, device=dev)
        out = torch.empty(B, code.info_words, dtype=torch.int32, device=dev)
        first, _ = frame_range(rank, ws, B)  # weak scaling: disjoint global frame ranges
        code.gen_bpsk_awgn(SEED, first, B, e, 4.0, llr_i8=llr if prof == "i8" else None,
                           llr_f32=llr if prof == "f32" else None, info=truth)
        decode = code.decode_i8 if prof == "i8" else code.decode_f32
        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            decode(llr, out)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        with Clocks(local) as clk:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for i in range(steps):
                ev[i][0].record(stream)
                decode(llr, out)
                ev[i][1].record(stream)
            t1.record(stream)
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        total_ms = max_over_ranks(t0.elapsed_time(t1))
        per_launch_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        ctr = torch.zeros(3, dtype=torch.int64, device=dev)
        code.count_errors(out, truth, ctr)
        if args.backend == "gloo":
            ctr = ctr.cpu()
        allreduce_counters(ctr)  # the one collective of the path
        frames, bit_err, frame_err = ctr.tolist()
        assert frames == ws * B, f"all-reduced frame count {frames} != {ws} ranks x {B}"
        res = {"code": code, "N": N, "K": K, "B": B, "frames": frames, "total_ms": total_ms, "ms_per_step": total_ms / steps,
               "launch_ms": per_launch_ms, "gbps": ws * B * K * steps / (total_ms * 1e-3) / 1e9,
               "fer": frame_err / max(frames, 1), "ber": bit_err / max(frames * K, 1), "clocks": clk.summary()}
        if with_e2e:
            host = llr.cpu().pin_memory()
            hout = torch.empty(B, code.info_words, dtype=torch.int32).pin_memory()
            code.decode_host(host, hout)
            barrier()
            e2e_steps = max(1, min(steps, 5))
            t = time.perf_counter()
            for _ in range(e2e_steps):
                code.decode_host(host, hout)
            dt = max_over_ranks(time.perf_counter() - t)
            assert torch.equal(hout, out.cpu()), "host path disagrees with the device path"
            res["e2e"] = {"value": ws * B * K * e2e_steps / dt / 1e9, "unit": "Gbps",
                          "h2d_bytes_per_step": B * N, "d2h_bytes_per_step": B * code.info_words * 4}
            del host, hout
        del llr, truth, out
        torch.cuda.empty_cache()
        return res

    def graph_latency_us(fn, x, out, reps=100):
        """Device latency without host submission gaps: `reps` single-frame decode calls in one
        CUDA graph (each still one full kernel launch), replayed; median of 5 replays / reps."""
        stream = torch.cuda.current_stream()
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            for _ in range(3):
                fn(x, out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(reps):
                fn(x, out)
        g.replay()
        torch.cuda.synchronize()
        t = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            t.append(a.elapsed_time(b) * 1e3 / reps)
        return float(np.median(t))

    def latency_batch1(code_t, iters=300):
        N, K, e = code_t
        code = pb.PolarCode.ga(N, K, e)
        llr = torch.empty(1, N, dtype=torch.int8, device=dev)
        out = torch.empty(1, code.info_words, dtype=torch.int32, device=dev)
        llr32 = torch.empty(1, N, dtype=torch.float32, device=dev)
        code.gen_bpsk_awgn(SEED, 0, 1, e, 4.0, llr_f32=llr32, llr_i8=llr)
        stream = torch.cuda.current_stream()
        res = {}
        for prof, x, fn in (("i8", llr, code.decode_i8), ("f32", llr32, code.decode_f32)):
            for _ in range(20):
                fn(x, out)
            torch.cuda.synchronize()
            ts = []
            for _ in range(iters):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn(x, out)
                b.record(stream)
                ts.append((a, b))
            torch.cuda.synchronize()
            us = np.array([a.elapsed_time(b) * 1e3 for a, b in ts])
            res[prof] = {"p50_us": float(np.median(us)), "p99_us": float(np.percentile(us, 99))}
            try:  # auxiliary legs never cost the bench line: an error is recorded instead
                res[prof]["graph_us"] = graph_latency_us(fn, x, out)
            except Exception as exc:
                res[prof]["graph_us"] = None
                res[prof]["graph_error"] = str(exc)[:200]
        res["n_ops"] = code.n_ops
        # host-observed end to end (the paper's definition, copies included):
        # host int8 frame -> info bits in host memory, wall clock per call
        hx = llr.cpu().numpy().reshape(-1).copy()
        hout = np.zeros(code.info_words, np.uint32)
        hin_t = torch.from_numpy(llr.cpu().numpy()).pin_memory()
        hout_t = torch.zeros(1, code.info_words, dtype=torch.int32).pin_memory()

        def wall(fn, n=iters):
            for _ in range(20):
                fn()
            t = []
            for _ in range(n):
                t0 = time.perf_counter_ns()
                fn()
                t.append((time.perf_counter_ns() - t0) / 1e3)
            return {"p50_us": float(np.median(t)), "p99_us": float(np.percentile(t, 99))}

        try:
            res["e2e_host_path_i8"] = wall(lambda: code.decode_host(hin_t, hout_t))
        except Exception as exc:
            res["e2e_host_path_i8"] = {"error": str(exc)[:200]}
        try:
            code.mailbox_open(idle_seconds=60.0)
            try:
                res["e2e_mailbox_i8"] = wall(lambda: code.mailbox_decode_i8(hx, hout))
            finally:
                code.mailbox_close()
            if not np.array_equal(hout, hout_t.numpy().view(np.uint32)[0]):
                res["e2e_mailbox_i8"]["error"] = "mailbox and host path disagree"
        except Exception as exc:
            res["e2e_mailbox_i8"] = {"error": str(exc)[:200]}
        return res

    def long_code_leg():
        N, K = 1 << 20, 1 << 19
        # Bhattacharyya parameters of BEC(0.5) (Arikan's construction, natural index order)
        z = np.array([0.5])
        while z.size < N:
            z = np.stack([2 * z - z * z, z * z], axis=1).reshape(-1)
        mask = np.zeros(N, np.uint8)
        mask[np.argsort(-z, kind="stable")[: N - K]] = 1
        code = pb.PolarCode(N, K, mask)
        B = 2 * torch.cuda.get_device_properties(dev).multi_processor_count
        llr = torch.empty(B, N, dtype=torch.int8, device=dev)
        code.gen_bpsk_awgn(SEED, 0, B, 2.5, 4.0, llr_i8=llr)
        out = code.decode_i8(llr)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            code.decode_i8(llr, out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        return {"info_gbps": B * K / (ms * 1e-3) / 1e9, "frames_per_launch": B, "ms_per_launch": ms, "n_ops": code.n_ops,
                "decoder": "program-interpreted, one CTA per frame (k_generic_big)"}

    main_r = throughput(CODE, args.batch, args.steps, args.warmup, with_e2e=True)
    extra = {}
    if not args.no_extra:
        r2 = throughput(CODE2, BATCH2, max(3, args.steps // 2), args.warmup, with_e2e=False)
        extra["c2048_1723_i8"] = {"info_gbps": r2["gbps"], "frames_per_s": ws * r2["B"] / (r2["ms_per_step"] * 1e-3),
                                  "batch_per_gpu": r2["B"], "ms_per_step": r2["ms_per_step"], "fer": r2["fer"]}
        # f32 profile throughput of both codes (same frames as LLR floats)
        for tag, code_t, B in (("c32768_29492_f32", CODE, args.batch // 2), ("c2048_1723_f32", CODE2, BATCH2 // 4)):
            r3 = throughput(code_t, B, max(3, args.steps // 2), args.warmup, with_e2e=False, prof="f32")
            extra[tag] = {"info_gbps": r3["gbps"], "frames_per_s": ws * r3["B"] / (r3["ms_per_step"] * 1e-3),
                          "batch_per_gpu": r3["B"], "ms_per_step": r3["ms_per_step"], "fer": r3["fer"]}
        # a code too long to unroll (the paper's instruction-based regime, N up to 2^24):
        # (2^20, 2^19), Bhattacharyya construction, program-interpreted decoder, 2 frames per SM
        try:
            extra["c1048576_524288_i8_generic"] = long_code_leg()
        except Exception as exc:  # an auxiliary leg never costs the bench line
            extra["c1048576_524288_i8_generic"] = {"error": str(exc)[:200]}
        extra["latency_batch1_32768_29492"] = latency_batch1(CODE)
        extra["latency_batch1_2048_1723"] = latency_batch1(CODE2)
    N, K = main_r["N"], main_r["K"]
    B = main_r["B"]
    # Roofline.  Headline: HBM -- algorithmic bytes per frame (the channel
    # LLRs read once + the packed information bits written once) x frames / the decode launch's
    # average CUDA-event duration, against MEASURED_PEAKS.json's copy bandwidth.  The kernel is
    # bound inside the SM, so the same line carries its fractions of the measured SM ceilings
    # (profiles/peaks_sm.json, tools/sm_peaks.cu): ALU pipe, issue slots and shared memory, each
    # = the ncu-counted work per frame of this kernel (profiles/roofline_inputs.json, from the
    # capture named there) x the frames/s measured here / the ceiling at the SM clock sampled
    # during the timed region.
    frames_per_s = B / (main_r["launch_ms"] * 1e-3)
    hbm_bytes_frame = N + 4 * code_words(K)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6.65 TB/s"
    hbm_ach = hbm_bytes_frame * frames_per_s / 1e9
    sm_clk = (main_r["clocks"].get("sm_mhz") or 1965.0) * 1e6
    ri, psm = {}, {}
    try:
        ri = json.load(open(os.path.join(ROOT, "profiles", "roofline_inputs.json")))["c32768_29492_i8_tp"]
        psm = json.load(open(os.path.join(ROOT, "profiles", "peaks_sm.json")))["pipes"]
    except (OSError, KeyError, ValueError):
        pass
    ceilings = {}
    if ri and psm:
        nsm = 148
        alu_peak = psm["LOP3"]["warp_inst_per_clk_per_sm"] * nsm * sm_clk
        ceilings["alu_pipe"] = {"achieved": ri["alu_warp_inst_per_frame"] * frames_per_s, "peak": alu_peak,
                                "unit": "warp inst/s", "frac": ri["alu_warp_inst_per_frame"] * frames_per_s / alu_peak}
        iss_peak = 4 * nsm * sm_clk
        ceilings["issue"] = {"achieved": ri["warp_inst_per_frame"] * frames_per_s, "peak": iss_peak,
                             "unit": "warp inst/s", "frac": ri["warp_inst_per_frame"] * frames_per_s / iss_peak}
        smem_peak = psm["LDS128"]["per_clk_per_sm"] * nsm * sm_clk / 128.0  # 128-byte wavefronts/s
        ceilings["smem"] = {"achieved": ri["smem_wavefronts_per_frame"] * frames_per_s, "peak": smem_peak,
                            "unit": "wavefronts/s", "frac": ri["smem_wavefronts_per_frame"] * frames_per_s / smem_peak}
        ceilings["source"] = (f"per-frame work: ncu capture {ri['capture']} (profiles/roofline_inputs.json); "
                              "ceilings: profiles/peaks_sm.json (tools/sm_peaks.cu) at the sampled SM clock")
    traffic = ri.get("dram_bytes_per_frame", 0) * B if ri else None
    line = {
        "metric": "info_gbps", "value": main_r["gbps"], "unit": "Gbps", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main_r["ms_per_step"], "higher_is_better": True,
        "ranks": {"world_size": ws, "backend": args.backend if ws > 1 else None, "devices": min(ws, ndev),
                  "frames_allreduced_per_step": main_r["frames"]},
        "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": {"workload": f"({N},{K}) systematic polar, int8 Fast-SSC, BPSK-AWGN {CODE[2]} dB, "
                               f"{B} frames/GPU per step resident in HBM",
                   "code": [N, K], "ebn0_db": CODE[2], "global_batch": B * ws, "batch_per_gpu": B,
                   "l2_flush": "inputs larger than L2 (512 MiB int8 LLRs per GPU)", "parallelism": f"dp{ws}"},
        "e2e": main_r["e2e"],
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": hbm_ach, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_ach / hbm_peak,
                     "traffic": traffic, "peak_source": hbm_src,
                     "algorithmic_bytes_per_frame": hbm_bytes_frame,
                     "traffic_source": "ncu dram__bytes_read+write per frame (profiles/roofline_inputs.json) x frames per launch",
                     "sm_ceilings": ceilings},
        "clocks": main_r["clocks"],
        "fer": main_r["fer"], "ber": main_r["ber"],
        "extra": extra,
    }
    if rank == 0 and ws == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        r, n, dt = cpu_oracle_rate(N, K, CODE[2], 2048, cores, min_seconds=10.0)
        line["cpu_baseline"] = {"value": r / 1e9, "unit": "Gbps", "cores": cores, "kind": "oracle",
                                "sample": f"{n} frame decodes of ({N},{K}) int8 (a 2048-frame tile of 64 seeded "
                                          f"AWGN frames, repeated for >= 10 s), {dt:.1f} s on {cores} threads"}
        # the paper's one-core protocol: the same oracle on one thread
        r1, n1, dt1 = cpu_oracle_rate(N, K, CODE[2], 64, 1, min_seconds=4.0)
        model = ""
        try:
            model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
        except (OSError, StopIteration):
            pass
        line["cpu_baseline"]["single_thread"] = {"value": r1 / 1e9, "unit": "Gbps", "us_per_frame": dt1 / n1 * 1e6,
                                                 "frames": n1, "seconds": round(dt1, 1)}
        line["cpu_baseline"]["cpu_model"] = model
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def code_words(K):
    return (K + 31) // 32


if __name__ == "__main__":
    main()
