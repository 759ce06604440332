"""GPU parity: the sm_100a Fast-SSC kernels (through the C ABI) against the CPU oracle.

Bar (north star): int8 bit-exact; f32 decision-exact -- the kernels use the oracle's op
order with one IEEE add per g and no FMA, so f32 is compared bit-exactly as well.  Inputs
are seeded synthetic frames (random information bits -> oracle systematic encoder -> BPSK
-> AWGN, seeded_inputs) plus adversarial LLRs (ties, saturation, -128, huge magnitudes).
"""
import os

import numpy as np
import pytest

import oracle
import paper_1504_00353_b200 as pb
from seeded_inputs import bpsk_awgn_llr, draw, quantize_i8, random_llr_f32, random_llr_i8

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = min(16, os.cpu_count() or 1)


def _design():
    """code name -> (N, K, mask, operating Eb/N0) for every specialised code."""
    spec = {}
    for fn in ("codes.txt", "codes_random.txt"):
        for line in open(os.path.join(ROOT, "paper_1504_00353_b200", fn)):
            f = line.split("#")[0].split()
            if len(f) >= 5:
                spec[(int(f[1]), int(f[2]), f[4] if f[3] == "mask" else None)] = (f[0], float(f[4]) if f[3] == "ga" else 2.0)
    out = []
    for N, K, m in pb.registry():
        key = (N, K, "".join(str(int(b)) for b in m))
        name, e = spec.get(key, spec.get((N, K, None), ("?", 2.0)))
        out.append((name, N, K, m, e))
    return out


CODES = _design()


def _n_frames(N):
    return 400 if N <= 256 else 200 if N <= 2048 else 48 if N <= 8192 else 12


def frames(mask, K, n, ebn0, seed, first=0):
    N = mask.shape[0]
    bits, noise = draw(seed, first, n, K, N)
    x = oracle.encode_systematic(mask, bits)
    llr = bpsk_awgn_llr(x, noise, ebn0, K)
    return bits, llr, quantize_i8(llr)


def expected(mask, llr):
    x = oracle.fastssc_decode(mask, llr, threads=THREADS)
    return oracle.pack_bits(oracle.info_bits(mask, x))


def gpu_decode(code, llr):
    t = torch.from_numpy(np.ascontiguousarray(llr)).cuda()
    out = code.decode_i8(t) if llr.dtype == np.int8 else code.decode_f32(t)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32)


def assert_same(got, want, what):
    bad = np.flatnonzero((got != want).any(axis=1))
    assert bad.size == 0, f"{what}: {bad.size} of {len(want)} frames differ (first {bad[:8]})"


@pytest.mark.parametrize("name,N,K,mask,ebn0", CODES, ids=[c[0] for c in CODES])
@pytest.mark.parametrize("prof", ["f32", "i8"])
@pytest.mark.parametrize("variant", ["throughput", "latency", "xframe"])
def test_parity_awgn_frames(name, N, K, mask, ebn0, prof, variant):
    if variant == "xframe" and prof == "f32":
        pytest.skip("the frame-interleaved variant is int8 only (f32 runs the throughput kernel)")
    code = pb.PolarCode(N, K, mask)
    code.set_variant(variant)
    n = _n_frames(N)
    for k, e in enumerate((ebn0, ebn0 - 1.5)):  # operating point and a noisy point
        _, llr, q = frames(mask, K, n, e, seed=1000 + k)
        x = q if prof == "i8" else llr
        assert_same(gpu_decode(code, x), expected(mask, x), f"{name} {prof} {variant} {e} dB")


@pytest.mark.parametrize("name,N,K,mask,ebn0", CODES, ids=[c[0] for c in CODES])
@pytest.mark.parametrize("variant", ["throughput", "latency", "xframe"])
def test_parity_adversarial_llrs(name, N, K, mask, ebn0, variant):
    code = pb.PolarCode(N, K, mask)
    code.set_variant(variant)
    n = max(8, _n_frames(N) // 4)
    cases = {
        "i8_uniform_full_range": random_llr_i8(7, (n, N), -128, 127),
        "i8_small_ties": random_llr_i8(8, (n, N), -2, 2),
        "i8_saturating": np.where(random_llr_i8(10, (n, N), 0, 1) > 0, 127, -128).astype(np.int8),
        "i8_zero": np.zeros((2, N), np.int8),
        "f32_gauss": random_llr_f32(11, (n, N), 3.0),
        "f32_zero": np.zeros((2, N), np.float32),
        "f32_huge": random_llr_f32(12, (n, N), 1e20),
        "f32_ints_ties": random_llr_f32(13, (n, N), 1.0).round().astype(np.float32),
    }
    for what, x in cases.items():
        assert_same(gpu_decode(code, x), expected(mask, x), f"{name} {what}")


@pytest.mark.parametrize("name,N,K,mask,ebn0", [c for c in CODES if c[1] <= 4096], ids=[c[0] for c in CODES if c[1] <= 4096])
def test_f32_equals_plain_sc(name, N, K, mask, ebn0):
    """Pin 5: on f32 frames without exact-zero decisions, Fast-SSC == plain SC."""
    code = pb.PolarCode(N, K, mask)
    _, llr, _ = frames(mask, K, 64, ebn0 - 1.0, seed=77)
    xs, _, zd = oracle.sc_decode(mask, llr, with_stats=True)
    keep = zd == 0
    want = oracle.pack_bits(oracle.info_bits(mask, xs))
    assert_same(gpu_decode(code, llr)[keep], want[keep], name)


GENERIC = [(2, 1, 301), (4, 2, 302), (8, 3, 303), (16, 9, 304), (32, 20, 305), (64, 30, 306), (256, 100, 307),
           (1024, 600, 308), (4096, 3000, 309), (32768, 20000, 310)]


@pytest.mark.parametrize("N,K,seed", GENERIC, ids=[f"{n}_{k}" for n, k, _ in GENERIC])
def test_generic_decoder_random_masks(N, K, seed, monkeypatch):
    """N1: frozen sets without a specialised decoder use the interpreted decoder (run-time
    specialisation off: tests/test_jit.py covers it)."""
    from seeded_inputs import random_mask

    monkeypatch.setenv("POLAR_JIT", "0")
    mask = random_mask(seed, N, K)
    code = pb.PolarCode(N, K, mask)
    assert not code.specialised
    n = 2 if N >= 32768 else 24 if N >= 4096 else 200
    cases = {"i8": random_llr_i8(seed, (n, N), -128, 127), "i8_ties": random_llr_i8(seed + 1, (n, N), -2, 2),
             "f32": random_llr_f32(seed, (n, N), 3.0), "f32_ints": random_llr_f32(seed + 2, (n, N), 1.0).round()}
    for what, x in cases.items():
        assert_same(gpu_decode(code, x.astype(x.dtype)), expected(mask, x), f"generic ({N},{K}) {what}")


@pytest.mark.parametrize("name,N,K,mask,ebn0", [c for c in CODES if c[1] in (8, 1024, 2048, 32768)],
                         ids=[c[0] for c in CODES if c[1] in (8, 1024, 2048, 32768)])
def test_generic_variant_equals_oracle_on_registered_codes(name, N, K, mask, ebn0):
    code = pb.PolarCode(N, K, mask)
    code.set_variant("generic")
    _, llr, q = frames(mask, K, 8 if N >= 32768 else 100, ebn0 - 1.0, seed=55)
    for x in (llr, q):
        assert_same(gpu_decode(code, x), expected(mask, x), f"{name} generic {x.dtype}")


@pytest.mark.parametrize("variant", ["auto", "xframe"])
def test_ragged_batches_and_grid_striding(variant):
    """Frame counts that are not multiples of the CTA's (or warp's 32) frames and exceed one
    resident wave."""
    for (N, K, e) in [(64, 32, 2.0), (1024, 512, 2.5), (4096, 2048, 2.5)]:
        mask = oracle.construct_ga(N, K, e)
        code = pb.PolarCode(N, K, mask)
        code.set_variant(variant)
        n = {64: 40013, 1024: 6007 if variant == "auto" else 20011, 4096: 1201}[N]
        x = random_llr_i8(21, (n, N), -40, 40)
        assert_same(gpu_decode(code, x), expected(mask, x), f"({N},{K}) x{n} {variant}")


def test_zero_frames_is_noop_and_bad_pointers_rejected():
    mask = oracle.construct_ga(1024, 512, 2.5)
    code = pb.PolarCode(1024, 512, mask)
    out = torch.full((1, 16), 7, dtype=torch.int32, device="cuda")
    code.decode_f32(torch.zeros(0, 1024, device="cuda"), out[:0])
    torch.cuda.synchronize()
    assert int(out[0, 0]) == 7
    llr = torch.zeros(2 * 1024 + 1, device="cuda")
    with pytest.raises(pb.PolarError) as e:
        pb.lib()  # noqa
        pb._check(pb.lib().polar_decode_f32(code._h, llr.data_ptr() + 4, 1, out.data_ptr(), None))
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT


def test_batch1_and_full_size_32768():
    """Batch-1 (config 3) and a throughput batch in the bench's launch configuration,
    checked on every frame the oracle can afford."""
    for K, e in [(29492, 4.5), (27568, 4.0)]:
        mask = oracle.construct_ga(32768, K, e)
        code = pb.PolarCode(32768, K, mask)
        _, llr, q = frames(mask, K, 1, e, seed=5)
        for x in (llr, q):
            assert_same(gpu_decode(code, x), expected(mask, x), f"batch-1 {K} {x.dtype}")
    code = pb.PolarCode(32768, 29492, oracle.construct_ga(32768, 29492, 4.5))
    n = 4096
    llr = torch.empty(n, 32768, dtype=torch.int8, device="cuda")
    truth = torch.empty(n, code.info_words, dtype=torch.int32, device="cuda")
    code.gen_bpsk_awgn(123, 0, n, 4.5, 4.0, llr_i8=llr, info=truth)
    out = code.decode_i8(llr)
    torch.cuda.synchronize()
    idx = np.random.default_rng(0).choice(n, 48, replace=False)
    sample = llr[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert_same(out.cpu().numpy().view(np.uint32)[idx], expected(code.mask(), sample), "32768 sampled")


def test_full_size_2048_1723_one_million_frames():
    """Config 2 at full size (1M frames) in the bench's launch configuration: a sample of
    frames against the oracle, and the frame-error rate against the truth bits."""
    mask = oracle.construct_ga(2048, 1723, 4.0)
    code = pb.PolarCode(2048, 1723, mask)
    n = 1 << 20
    llr = torch.empty(n, 2048, dtype=torch.int8, device="cuda")
    truth = torch.empty(n, code.info_words, dtype=torch.int32, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, n, 4.0, 4.0, llr_i8=llr, info=truth)
    out = code.decode_i8(llr)
    ctr = torch.zeros(3, dtype=torch.int64, device="cuda")
    code.count_errors(out, truth, ctr)
    torch.cuda.synchronize()
    idx = np.random.default_rng(1).choice(n, 3000, replace=False)
    idx.sort()
    sample = llr[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert_same(out.cpu().numpy().view(np.uint32)[idx], expected(mask, sample), "1M sampled")
    frames_, bit_err, frame_err = ctr.tolist()
    assert frames_ == n
    fer = frame_err / n
    assert 0.005 < fer < 0.05, fer  # MC 1.9e-2 at 4.0 dB
    assert bit_err >= frame_err


def test_encoder_and_generator_against_oracle():
    for N, K, e in [(8, 5, None), (1024, 512, 2.5), (2048, 1723, 4.0), (32768, 29492, 4.5)]:
        mask = np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8) if e is None else oracle.construct_ga(N, K, e)
        code = pb.PolarCode(N, K, mask)
        bits, _ = draw(3, 0, 16, K, N)
        info = torch.from_numpy(oracle.pack_bits(bits).view(np.int32)).cuda()
        cw = code.encode_systematic(info)
        torch.cuda.synchronize()
        want = oracle.pack_bits(oracle.encode_systematic(mask, bits))
        np.testing.assert_array_equal(cw.cpu().numpy().view(np.uint32), want)
        # generator: determinism across batching, the truth it reports is what it encoded
        n = 64
        l1 = torch.empty(n, N, device="cuda")
        t1 = torch.empty(n, code.info_words, dtype=torch.int32, device="cuda")
        code.gen_bpsk_awgn(9, 100, n, 3.0, 4.0, llr_f32=l1, info=t1)
        l2 = torch.empty(n - 10, N, device="cuda")
        code.gen_bpsk_awgn(9, 110, n - 10, 3.0, 4.0, llr_f32=l2)
        q = torch.empty(n, N, dtype=torch.int8, device="cuda")
        code.gen_bpsk_awgn(9, 100, n, 3.0, 4.0, llr_i8=q)
        torch.cuda.synchronize()
        assert torch.equal(l1[10:], l2)
        np.testing.assert_array_equal(q.cpu().numpy(), quantize_i8(l1.cpu().numpy()))
        tb = oracle.unpack_bits(t1.cpu().numpy().view(np.uint32), K)
        x = oracle.encode_systematic(mask, tb).astype(np.float64)
        s = 1.0 - 2.0 * x
        s2 = 1.0 / (2 * (K / N) * 10 ** 0.3)
        y = l1.cpu().numpy().astype(np.float64) * s2 / 2.0
        noise = (y - s) / np.sqrt(s2)
        m = noise.size  # 5-sigma bounds for the sample mean and standard deviation
        assert abs(noise.mean()) < 5 / np.sqrt(m) and abs(noise.std() - 1.0) < 5 / np.sqrt(2 * m)


def test_count_errors_matches_numpy():
    code = pb.PolarCode(1024, 512, oracle.construct_ga(1024, 512, 2.5))
    rng = np.random.default_rng(4)
    a = rng.integers(0, 2**32, size=(1000, 16), dtype=np.uint64).astype(np.uint32)
    b = a.copy()
    flip = rng.random((1000, 16)) < 0.05
    b[flip] ^= rng.integers(1, 2**32, size=int(flip.sum()), dtype=np.uint64).astype(np.uint32)
    ctr = torch.zeros(3, dtype=torch.int64, device="cuda")
    code.count_errors(torch.from_numpy(a.view(np.int32)).cuda(), torch.from_numpy(b.view(np.int32)).cuda(), ctr)
    torch.cuda.synchronize()
    bits = int(np.unpackbits((a ^ b).view(np.uint8)).sum())
    fr = int(((a ^ b) != 0).any(axis=1).sum())
    assert ctr.tolist() == [1000, bits, fr]


def test_host_buffer_path_equals_device_path():
    mask = oracle.construct_ga(2048, 1723, 4.0)
    code = pb.PolarCode(2048, 1723, mask)
    _, llr, q = frames(mask, 1723, 300, 3.5, seed=31)
    for x in (llr, q):
        host_out = np.zeros((300, code.info_words), np.uint32)
        code.decode_host(np.ascontiguousarray(x), host_out)
        assert_same(host_out, expected(mask, x), f"host-buffer path {x.dtype}")
        pinned = torch.from_numpy(x).pin_memory()
        pout = torch.zeros(300, code.info_words, dtype=torch.int32).pin_memory()
        code.decode_host(pinned, pout)
        np.testing.assert_array_equal(pout.numpy().view(np.uint32), host_out)


def test_mailbox_batch1_equals_oracle_and_error_paths():
    """Batch-1 mailbox (persistent kernel on host-mapped memory): every frame
    bit-identical to the oracle, -128 clamped, clean close, and the documented errors."""
    import time
    for (N, K, e) in [(2048, 1723, 4.0), (32768, 29492, 4.5)]:
        mask = oracle.construct_ga(N, K, e)
        code = pb.PolarCode(N, K, mask)
        _, _, q = frames(mask, K, 5, e - 0.5, seed=77)
        q[0, :7] = -128
        q[1] = random_llr_i8(78, (1, N), -2, 2)[0]  # ties
        want = expected(mask, q)
        out = np.zeros(code.info_words, np.uint32)
        with pytest.raises(pb.PolarError):  # not open
            code.mailbox_decode_i8(np.ascontiguousarray(q[0]), out)
        code.mailbox_open(idle_seconds=30.0)
        try:
            with pytest.raises(pb.PolarError):  # second open
                code.mailbox_open()
            for _ in range(2):
                for i in range(len(q)):
                    out[:] = 0
                    code.mailbox_decode_i8(np.ascontiguousarray(q[i]), out)
                    assert np.array_equal(out, want[i]), f"mailbox ({N},{K}) frame {i}"
        finally:
            code.mailbox_close()
        code.mailbox_close()  # closing twice is a no-op
    # idle self-exit: the kernel leaves on its own; the next request times out; close still works
    code.mailbox_open(idle_seconds=0.2)
    time.sleep(0.6)
    with pytest.raises(pb.PolarError) as err:
        code.mailbox_decode_i8(np.ascontiguousarray(q[0]), out, timeout_seconds=0.2)
    assert err.value.status == pb.POLAR_ERR_CUDA
    code.mailbox_close()
    other = pb.PolarCode(1024, 512, oracle.construct_ga(1024, 512, 2.5))
    with pytest.raises(pb.PolarError) as err:
        other.mailbox_open()
    assert err.value.status == pb.POLAR_ERR_UNSUPPORTED_CODE


def test_concurrent_streams_share_a_handle():
    """Two streams decode different frames on ONE handle at the same time; small launches so
    both kernels are resident together. The variants with per-handle global stage scratch
    (N = 32768 throughput, frame-interleaved) must still be exact."""
    for (N, K, e, n, variant) in [(32768, 29492, 4.5, 300, "throughput"), (2048, 1723, 4.0, 4096, "xframe")]:
        mask = oracle.construct_ga(N, K, e)
        code = pb.PolarCode(N, K, mask)
        code.set_variant(variant)
        xs = [torch.from_numpy(random_llr_i8(90 + k, (n, N), -30, 30)).cuda() for k in range(2)]
        want = [code.decode_i8(x) for x in xs]
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream() for _ in range(2)]
        outs = [torch.empty_like(w) for w in want]
        for _ in range(20):
            for k in range(2):
                with torch.cuda.stream(streams[k]):
                    code.decode_i8(xs[k], outs[k], stream=streams[k])
            torch.cuda.synchronize()
            for k in range(2):
                assert torch.equal(outs[k], want[k]), f"({N},{K}) {variant} stream {k}"
        sample = xs[0][:8].cpu().numpy()
        assert_same(want[0][:8].cpu().numpy().view(np.uint32), expected(mask, sample), f"({N},{K}) {variant}")


def test_dynamic_frame_scheduling_many_rounds():
    """The throughput variant of N = 32768 hands out frame groups with an atomic counter
    (kernels.cuh DYN): ~8 rounds of the persistent grid, a ragged last group, and a second
    launch on the same handle (the counter is re-zeroed) must equal the latency variant (no
    dynamic scheduling) on every frame; a sample is checked against the oracle."""
    mask = oracle.construct_ga(32768, 29492, 4.5)
    code = pb.PolarCode(32768, 29492, mask)
    n = 20011
    llr = torch.empty(n, 32768, dtype=torch.int8, device="cuda")
    code.gen_bpsk_awgn(4242, 0, n, 4.0, 4.0, llr_i8=llr)
    code.set_variant("throughput")
    a = code.decode_i8(llr)
    b = code.decode_i8(llr[: n - 5000])
    code.set_variant("latency")
    c = code.decode_i8(llr)
    torch.cuda.synchronize()
    assert torch.equal(a, c), int((a != c).any(dim=1).sum())
    assert torch.equal(b, c[: n - 5000])
    idx = np.array([0, 1, 2665, 5329, n - 1])
    sample = llr[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert_same(a.cpu().numpy().view(np.uint32)[idx], expected(mask, sample), "dynamic scheduling")


@pytest.mark.parametrize("N,K,e,prof,n", [(32768, 29492, 4.5, "f32", 8192), (32768, 29492, 4.5, "i8", 16384),
                                         (2048, 1723, 4.0, "f32", 262144)],
                         ids=["32768_f32_8192", "32768_i8_16384", "2048_f32_262144"])
def test_bench_batches_every_frame_against_oracle(N, K, e, prof, n):
    """The launch configurations bench.py times, every frame against the oracle: f32 at
    N = 32768 runs ~3 rounds of the persistent grid with dynamic frame-group hand-out, f32 at
    (2048,1723) fills both TMA ingest buffers of every warp many times."""
    mask = oracle.construct_ga(N, K, e)
    code = pb.PolarCode(N, K, mask)
    llr = torch.empty(n, N, dtype=torch.float32 if prof == "f32" else torch.int8, device="cuda")
    code.gen_bpsk_awgn(1504000353, 0, n, e, 4.0, **({"llr_f32": llr} if prof == "f32" else {"llr_i8": llr}))
    out = code.decode_f32(llr) if prof == "f32" else code.decode_i8(llr)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    x = llr.cpu().numpy()
    del llr
    assert_same(got, expected(mask, x), f"({N},{K}) {prof} x {n}")


NONSYS = [c for c in CODES if c[1] in (8, 64, 1024, 2048, 4096, 32768)]


@pytest.mark.parametrize("name,N,K,mask,ebn0", NONSYS, ids=[c[0] for c in NONSYS])
@pytest.mark.parametrize("variant", ["throughput", "latency", "generic"])
def test_nonsystematic_output_equals_oracle(name, N, K, mask, ebn0, variant):
    """Non-systematic output mode (reading C4): u_hat[A] with u_hat = x_hat G_N.
    Frames of the non-systematic code x = u G_N (u[A] = d, u[F] = 0); every frame
    against the oracle's x_hat G_N, and noiseless frames return d exactly."""
    code = pb.PolarCode(N, K, mask)
    code.set_variant(variant)
    code.set_output("nonsystematic")
    n = _n_frames(N)
    bits, noise = draw(4321, 0, n, K, N)
    u = np.zeros((n, N), np.uint8)
    u[:, mask == 0] = bits
    x = oracle.encode(u)
    llr = bpsk_awgn_llr(x, noise, ebn0 - 1.0, K)
    for y in (llr, quantize_i8(llr)):
        xh = oracle.fastssc_decode(mask, y, threads=THREADS)
        want = oracle.pack_bits(oracle.info_bits(mask, oracle.encode(xh)))
        assert_same(gpu_decode(code, y), want, f"{name} non-systematic {variant} {y.dtype}")
    clean = np.where(x == 0, 8.0, -8.0).astype(np.float32)
    np.testing.assert_array_equal(gpu_decode(code, clean), oracle.pack_bits(bits))
    code.set_output("systematic")
    assert_same(gpu_decode(code, clean), oracle.pack_bits(oracle.info_bits(mask, x)), f"{name} back to systematic")
