"""Intermediate-LLR parity (north star: "for float must match on decisions with intermediate
LLRs within 1e-5 relative (same op order, no FMA contraction)"): libpolar_dump.so is the
product's kernels built with POLAR_DEBUG_DUMP, which append every F / G / G_0R output vector
(eq:f P:295-302, eq:g P:304-315) in op order (Listing 1); the oracle's O2 records the
same vectors (oracle.fastssc_alpha_dump).  Compared for the throughput and the latency variant,
f32 and int8, on AWGN and adversarial frames: exactly (signed zeros equal), which implies the
1e-5 relative bar; the max relative error is asserted too."""
import numpy as np
import pytest

import oracle
import paper_1504_00353_b200 as pb
from seeded_inputs import bpsk_awgn_llr, draw, quantize_i8, random_llr_f32, random_llr_i8

CODES = [(8, 5, None, 2.0), (1024, 512, 2.5, 2.5), (2048, 1723, 4.0, 4.0), (32768, 29492, 4.5, 4.5)]


def _mask(N, K, design):
    return np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8) if design is None else oracle.construct_ga(N, K, design)


def test_dump_library_exports_the_abi():
    L = pb.dump_lib()
    for name in pb.EXPORTS:
        assert hasattr(L, name), name


@pytest.mark.gpu
@pytest.mark.parametrize("N,K,design,ebn0", CODES, ids=[f"{c[0]}_{c[1]}" for c in CODES])
@pytest.mark.parametrize("variant", ["throughput", "latency"])
def test_alpha_stages_equal_oracle(N, K, design, ebn0, variant):
    torch = pytest.importorskip("torch")
    mask = _mask(N, K, design)
    code = pb.PolarCode(N, K, mask, library=pb.dump_lib())
    assert code.specialised
    code.set_variant(variant)
    n = 4
    bits, noise = draw(2024, 0, n, K, N)
    llr = bpsk_awgn_llr(oracle.encode_systematic(mask, bits), noise, ebn0 - 1.0, K)
    cases = {"f32_awgn": llr, "i8_awgn": quantize_i8(llr), "f32_gauss": random_llr_f32(5, (n, N), 3.0),
             "i8_full_range": random_llr_i8(6, (n, N), -128, 127), "f32_ties": random_llr_f32(7, (n, N), 1.0).round(),
             "i8_saturating": np.where(random_llr_i8(8, (n, N), 0, 1) > 0, 127, -128).astype(np.int8)}
    for what, x in cases.items():
        x = np.ascontiguousarray(x)
        t = torch.from_numpy(x).cuda()
        (code.decode_i8 if x.dtype == np.int8 else code.decode_f32)(t)
        torch.cuda.synchronize()
        got = code.alpha_dump(n)
        for k in range(n):
            want = oracle.fastssc_alpha_dump(mask, x[k]).astype(np.float32)
            g = got[k, : want.size]
            assert np.isnan(got[k, want.size:]).all(), f"{what} frame {k}: more values than the oracle's ops"
            assert not np.isnan(g).any(), f"{what} frame {k}: fewer values than the oracle's ops"
            rel = np.abs(g.astype(np.float64) - want) / np.maximum(np.abs(want.astype(np.float64)), 1e-30)
            assert rel.max(initial=0.0) <= 1e-5, f"{what} frame {k}: max rel err {rel.max()}"
            bad = np.flatnonzero(g != want)
            assert bad.size == 0, f"{what} frame {k}: {bad.size} of {want.size} alpha values differ, first at {bad[:5]}"
