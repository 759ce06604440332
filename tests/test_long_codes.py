"""Codes longer than the unrolled decoders (N up to 2^20): the program-interpreted decoder in
its one-CTA-per-frame form (generic.cu k_generic_big; the paper's instruction-based decoder is
its answer for N up to 2^24).  Frozen sets: GA at N = 65536; a Bhattacharyya (BEC)
construction at N = 2^20 (GA's bisection is too slow for a test there; any frozen set is valid
input to the decoder)."""
import os

import numpy as np
import pytest

import oracle
import paper_1504_00353_b200 as pb
from seeded_inputs import bpsk_awgn_llr, draw, quantize_i8, random_llr_i8


def bec_mask(N, K, z0):
    z = oracle.bhattacharyya_bec(N, z0)
    m = np.zeros(N, np.uint8)
    m[np.argsort(-z, kind="stable")[: N - K]] = 1
    return m


def test_long_code_handle_without_gpu():
    """polar_code_create accepts N up to 2^20 (program-interpreted decoder); the schedule is the
    oracle's; N = 2^21 is refused."""
    m = bec_mask(1 << 17, 1 << 16, 0.5)
    c = pb.PolarCode(1 << 17, 1 << 16, m)
    assert not c.specialised and c.n_ops == len(oracle.fastssc_trace(m))
    with pytest.raises(pb.PolarError):
        pb.PolarCode(1 << 21, 1 << 20, bec_mask(1 << 21, 1 << 20, 0.5))


LONG = [("ga_65536", 1 << 16, 58982, "ga", 4.5), ("bec_1M", 1 << 20, 1 << 19, "bec", 2.5)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,K,how,ebn0", LONG, ids=[c[0] for c in LONG])
def test_long_code_decoder_equals_oracle(name, N, K, how, ebn0):
    torch = pytest.importorskip("torch")
    mask = oracle.construct_ga(N, K, ebn0) if how == "ga" else bec_mask(N, K, 0.5)
    code = pb.PolarCode(N, K, mask)
    n = 6
    bits, noise = draw(515, 0, n, K, N)
    llr = bpsk_awgn_llr(oracle.encode_systematic(mask, bits), noise, ebn0, K)
    cases = {"f32": llr, "i8": quantize_i8(llr), "i8_full_range": random_llr_i8(2, (2, N), -128, 127)}
    threads = os.cpu_count() or 1
    for what, x in cases.items():
        t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        for mode in ("systematic", "nonsystematic"):
            code.set_output(mode)
            got = (code.decode_i8(t) if x.dtype == np.int8 else code.decode_f32(t)).cpu().numpy().view(np.uint32)
            xh = oracle.fastssc_decode(mask, x, threads=threads)
            if mode == "nonsystematic":
                xh = oracle.encode(xh)
            want = oracle.pack_bits(oracle.info_bits(mask, xh))
            bad = np.flatnonzero((got != want).any(axis=1))
            assert bad.size == 0, f"{name} {what} {mode}: frames {bad} differ"
    code.set_output("systematic")
    # the generator and encoder handle long codes too: encode(info) is the oracle's codeword
    info = torch.from_numpy(oracle.pack_bits(bits[:2]).view(np.int32)).cuda()
    cw = code.encode_systematic(info).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(cw, oracle.pack_bits(oracle.encode_systematic(mask, bits[:2])))
