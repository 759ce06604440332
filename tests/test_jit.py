"""Run-time specialisation: polar_code_create generates and NVRTC-compiles the
unrolled decoder of a frozen set that has no build-time decoder (the paper generates one per
code).  CPU: the generator's output compiles for sm_100a.  GPU: run-time specialised
handles decode exactly like the oracle (AWGN and adversarial frames, both kernel variants),
and the same code specialised at build and at run time decodes identically and about as fast."""
import os
import time

import numpy as np
import pytest

import oracle
import paper_1504_00353_b200 as pb
from seeded_inputs import bpsk_awgn_llr, draw, quantize_i8, random_llr_f32, random_llr_i8, random_mask


def test_generated_source_compiles_with_nvrtc(tmp_path, monkeypatch):
    monkeypatch.setenv("POLAR_JIT_CACHE", str(tmp_path))
    tag = pb.jit_compile(64, 30, random_mask(5, 64, 30))
    assert tag.startswith("compiled polar_64_30_")
    assert any(p.suffix == ".cubin" for p in tmp_path.iterdir())
    assert pb.jit_compile(64, 30, random_mask(5, 64, 30)) == tag  # cache hit, same tag


def _expected(mask, x):
    return oracle.pack_bits(oracle.info_bits(mask, oracle.fastssc_decode(mask, x, threads=os.cpu_count() or 1)))


# ga_32768_32000: ceil(K/32) = 1000 output words = 32 groups of the gather's piece table, so the
# gather takes its per-group path with a header load past the first 32 groups (decoder.cuh
# gather_info) in both kernel variants
JIT_CODES = [("random_1024_600", 1024, 600, None, 2.5), ("ga_4096_2048_at_3dB", 4096, 2048, 3.0, 3.0),
             ("ga_32768_29492_at_4dB", 32768, 29492, 4.0, 4.5), ("ga_32768_32000_at_6dB", 32768, 32000, 6.0, 6.5)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,K,design,ebn0", JIT_CODES, ids=[c[0] for c in JIT_CODES])
def test_run_time_specialised_decoder_equals_oracle(name, N, K, design, ebn0):
    torch = pytest.importorskip("torch")
    mask = random_mask(308, N, K) if design is None else oracle.construct_ga(N, K, design)
    code = pb.PolarCode(N, K, mask)
    assert code.run_time_specialised, pb.lib().polar_last_error().decode()
    n = 64 if N <= 4096 else 24
    bits, noise = draw(77, 0, n, K, N)
    llr = bpsk_awgn_llr(oracle.encode_systematic(mask, bits), noise, ebn0 - 1.0, K)
    cases = {"f32": llr, "i8": quantize_i8(llr), "i8_full_range": random_llr_i8(3, (n, N), -128, 127),
             "f32_ties": random_llr_f32(4, (n, N), 1.0).round()}
    for variant in ("throughput", "latency"):
        code.set_variant(variant)
        for what, x in cases.items():
            t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
            got = (code.decode_i8(t) if x.dtype == np.int8 else code.decode_f32(t)).cpu().numpy().view(np.uint32)
            want = _expected(mask, x)
            bad = np.flatnonzero((got != want).any(axis=1))
            assert bad.size == 0, f"{name} {variant} {what}: {bad.size} frames differ"


@pytest.mark.gpu
def test_build_time_and_run_time_specialisation_agree(monkeypatch):
    """(2048,1723): the registered code and the same code forced through NVRTC
    (POLAR_JIT_FORCE=1) decode 256K frames identically; the run-time kernel runs at >= 90% of
    the build-time kernel's throughput (same generated source, same compiler back end)."""
    torch = pytest.importorskip("torch")
    N, K, e = 2048, 1723, 4.0
    mask = oracle.construct_ga(N, K, e)
    aot = pb.PolarCode(N, K, mask)
    monkeypatch.setenv("POLAR_JIT_FORCE", "1")
    jit = pb.PolarCode(N, K, mask)
    monkeypatch.delenv("POLAR_JIT_FORCE")
    assert aot.specialised and not aot.run_time_specialised and jit.run_time_specialised
    n = 1 << 18
    llr = torch.empty(n, N, dtype=torch.int8, device="cuda")
    aot.gen_bpsk_awgn(11, 0, n, e, 4.0, llr_i8=llr)
    rates = {}
    outs = {}
    for tag, c in (("aot", aot), ("jit", jit)):
        out = c.decode_i8(llr)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            c.decode_i8(llr, out)
        torch.cuda.synchronize()
        rates[tag] = 5 * n / (time.perf_counter() - t)
        outs[tag] = out
    assert torch.equal(outs["aot"], outs["jit"])
    assert rates["jit"] >= 0.9 * rates["aot"], rates
