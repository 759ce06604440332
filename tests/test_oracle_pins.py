"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage (PAPER.md line, "P:n") or the mathematical fact it relies on.
None of them re-types the oracle's own formula: they use printed values (tests/golden/),
closed forms, brute force on tiny inputs, invariants, or a second, independent algorithm.
"""
import itertools
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line)
    return rows


# ------------------------------------------------------------------ primitives (hand values)
def test_f_g_hand_values():
    """eq:f P:295-302 / eq:g P:304-315; hand-evaluated examples."""
    assert oracle.f_f32(2.0, -3.0) == -2.0
    assert oracle.f_f32(0.0, 7.0) == 0.0
    assert [oracle.f_f32(5, -3), oracle.f_f32(2, -7)] == [-3.0, -2.0]
    assert oracle.g_f32(2.0, 3.0, 0) == 5.0
    assert oracle.g_f32(2.0, 3.0, 1) == 1.0
    # G_0R = g with beta_l = 0: g_0r([7,-2,3,9]) -> [10, 7]
    assert [oracle.g_f32(7, 3, 0), oracle.g_f32(-2, 9, 0)] == [10.0, 7.0]
    # int8: saturating adders, range [-127,127] (Listing 4's max(-127))
    assert oracle.g_i8(100, 100, 0) == 127
    assert oracle.g_i8(100, -100, 1) == -127
    assert oracle.g_i8(-127, -127, 0) == -127
    assert oracle.g_i8(127, -127, 1) == -127
    assert oracle.f_i8(-127, 5) == -5
    assert oracle.f_i8(-127, -127) == 127


def test_rep_spc_hand_values():
    """Repetition P:431-440 (sum >= 0 -> 0), SPC P:442-459 (flip argmin |alpha|)."""
    assert list(oracle.rep_node(np.array([-1, 2, -3, 1], np.float32))) == [1, 1, 1, 1]
    assert list(oracle.rep_node(np.array([0, 0], np.float32))) == [0, 0]
    assert list(oracle.rep_node(np.array([5, -1], np.int8))) == [0, 0]
    assert list(oracle.spc_node(np.array([2, -1, 3, 4], np.float32))) == [0, 0, 0, 0]
    assert list(oracle.spc_node(np.array([1, 1], np.float32))) == [0, 0]
    # N_v = 4 tie: all |alpha| equal, lowest index flipped (reading C10)
    assert list(oracle.spc_node(np.array([-1, -1, -1, 1], np.float32))) == [0, 1, 1, 0]
    assert list(oracle.spc_node(np.array([-1, -1, -1, 1], np.int8))) == [0, 1, 1, 0]


# ------------------------------------------------------------------ encoder
def test_g4_matches_paper():
    """G_4 printed at P:142-151: row i of G is the encoding of the unit vector e_i."""
    rows = _read_golden("g4_paper.txt")
    for i in range(4):
        e = np.zeros(4, np.uint8); e[i] = 1
        assert "".join(map(str, oracle.encode_matrix(e))) == rows[i]
        assert "".join(map(str, oracle.encode(e[None])[0])) == rows[i]


@pytest.mark.parametrize("N", [2, 4, 8, 16, 64, 256])
def test_encode_block_form_equals_kronecker_definition(N):
    """Block recursion G_N = [G 0; G G] equals the Kronecker definition."""
    rng = np.random.default_rng(N)
    for _ in range(8):
        u = rng.integers(0, 2, N, dtype=np.uint8)
        assert np.array_equal(oracle.encode(u[None])[0], oracle.encode_matrix(u))


@pytest.mark.parametrize("N", [8, 128, 2048])
def test_encode_is_involution(N):
    """F_2^{(x)n} squared is the identity over GF(2) (F_2^2 = I)."""
    rng = np.random.default_rng(1 + N)
    u = rng.integers(0, 2, (4, N), dtype=np.uint8)
    assert np.array_equal(oracle.encode(oracle.encode(u)), u)


@pytest.mark.parametrize("N,K,ebn0", [(8, 5, 2.0), (64, 32, 2.0), (1024, 512, 2.5), (2048, 1723, 4.0)])
def test_systematic_encoder(N, K, ebn0):
    """Systematic codeword: x[A] = d, and u = x G has u[F] = 0 (x is a codeword)."""
    frozen = oracle.construct_ga(N, K, ebn0)
    bits, _ = si.draw(7, 0, 6, K, N)
    x = oracle.encode_systematic(frozen, bits)
    assert np.array_equal(x[:, frozen == 0], bits)
    u = oracle.encode(x)
    assert not u[:, frozen == 1].any()


def test_systematic_encoder_arbitrary_mask():
    """The oracle's systematic encoder is exact for any frozen set (not only
    superset-closed ones)."""
    for seed in range(6):
        frozen = si.random_mask(seed, 32, 13)
        bits, _ = si.draw(seed, 0, 3, 13, 32)
        x = oracle.encode_systematic(frozen, bits)
        assert np.array_equal(x[:, frozen == 0], bits)
        assert not oracle.encode(x)[:, frozen == 1].any()


# ------------------------------------------------------------------ Listing 1 and the worked frame
def test_listing1_op_sequence():
    """O2's op sequence on the (8,5) frozen={0,1,4} code is Listing 1."""
    rows = _read_golden("listing1_8_5.txt")
    frozen = np.array([int(c) for c in rows[0]], np.uint8)
    assert oracle.fastssc_trace(frozen) == rows[1:]


def test_worked_8_5_frame():
    """Hand-worked f32 frame (golden/worked_8_5_f32.txt): Fast-SSC and plain SC give the
    traced codeword; SC's leaf decisions u_hat are x_hat G."""
    g = {r.split()[0]: r.split()[1:] for r in _read_golden("worked_8_5_f32.txt")}
    frozen = np.array(g["frozen"], np.uint8)
    a = np.array(g["alpha_c"], np.float32)[None]
    xhat = np.array(g["xhat"], np.uint8)
    assert np.array_equal(oracle.fastssc_decode(frozen, a)[0], xhat)
    xs, us, zd = oracle.sc_decode(frozen, a, with_stats=True)
    assert np.array_equal(xs[0], xhat)
    assert np.array_equal(us[0], np.array(g["uhat"], np.uint8))
    assert np.array_equal(oracle.info_bits(frozen, xs[0]), np.array(g["info"], np.uint8))
    # intermediate values of the hand trace
    f8 = [oracle.f_f32(a[0, i], a[0, i + 4]) for i in range(4)]
    assert f8 == [float(v) for v in g["f8"]]
    g0r = [oracle.g_f32(f8[i], f8[i + 2], 0) for i in range(2)]
    assert g0r == [float(v) for v in g["g0r4"]]
    g8 = [oracle.g_f32(a[0, i], a[0, i + 4], 1) for i in range(4)]
    assert g8 == [float(v) for v in g["g8"]]
    # the oracle's alpha dump (the reference side of the GPU alpha-stage parity test) records
    # exactly the hand trace's F<8>, G_0R<4>, G<8> outputs in Listing-1 order
    want = [float(v) for k in ("f8", "g0r4", "g8") for v in g[k]]
    assert oracle.fastssc_alpha_dump(frozen, a[0]).tolist() == want
    assert oracle.fastssc_alpha_dump(frozen, np.rint(4 * a[0]).astype(np.int8)).tolist() == [4 * v for v in want]


# ------------------------------------------------------------------ node decoders are ML (brute force)
def _ml_over(words, alpha):
    """Brute-force correlation metric of every codeword (rows of `words`)."""
    metric = (1.0 - 2.0 * words.astype(np.float64)) @ alpha.astype(np.float64)
    return metric.max(), metric


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_rep_and_spc_nodes_are_ml(n):
    """The Repetition and SPC rules return an ML codeword of their node code
    (brute force over all codewords; exact for continuous inputs, and an ML member of the
    optimal set for int8 ties)."""
    rng = np.random.default_rng(100 + n)
    rep_words = np.stack([np.zeros(n, np.uint8), np.ones(n, np.uint8)])
    allw = np.array(list(itertools.product([0, 1], repeat=n)), np.uint8)
    spc_words = allw[allw.sum(axis=1) % 2 == 0]
    for trial in range(300):
        a = rng.standard_normal(n).astype(np.float32)
        for words, fn in ((rep_words, oracle.rep_node), (spc_words, oracle.spc_node)):
            out = fn(a)
            best, metric = _ml_over(words, a)
            winners = np.flatnonzero(metric == best)
            assert len(winners) == 1 and np.array_equal(out, words[winners[0]])
        q = rng.integers(-6, 7, n).astype(np.int8)
        for words, fn in ((rep_words, oracle.rep_node), (spc_words, oracle.spc_node)):
            out = fn(q)
            best, metric = _ml_over(words, q)
            assert (words == out).all(axis=1).any()
            assert float(np.sum((1.0 - 2.0 * out) * q.astype(np.float64))) == best


def _all_masks(N):
    for bits in itertools.product([0, 1], repeat=N):
        if 0 < N - sum(bits) <= N:
            yield np.array(bits, np.uint8)


def test_fastssc_is_ml_when_root_is_a_special_node():
    """For N <= 8 codes whose root is Rate-1 / Rep / SPC, Fast-SSC = brute-force ML (O3);
    for every other mask O3's metric bounds Fast-SSC's and the output is a codeword."""
    rng = np.random.default_rng(5)
    for N in (2, 4, 8):
        for frozen in _all_masks(N):
            a = rng.standard_normal((20, N)).astype(np.float32)
            ml = oracle.ml_decode(frozen, a)
            fs = oracle.fastssc_decode(frozen, a)
            kind = oracle.classify(frozen)
            mm = np.sum((1.0 - 2.0 * ml) * a, axis=1)
            mf = np.sum((1.0 - 2.0 * fs) * a, axis=1)
            assert np.all(mf <= mm + 1e-5)
            assert not oracle.encode(fs)[:, frozen == 1].any()
            if kind in ("Rate1", "Rep", "SPC"):
                assert np.array_equal(ml, fs)


# ------------------------------------------------------------------ SC == Fast-SSC (two algorithms)
def _frames(N, K, ebn0, n, seed, i8=False):
    frozen = oracle.construct_ga(N, K, ebn0)
    bits, noise = si.draw(seed, 0, n, K, N)
    x = oracle.encode_systematic(frozen, bits)
    llr = si.bpsk_awgn_llr(x, noise, ebn0, K)
    if i8:
        llr = si.quantize_i8(llr)
    return frozen, bits, x, llr


@pytest.mark.parametrize("N,K,ebn0", [(64, 32, 1.5), (256, 128, 2.0), (1024, 512, 2.5), (2048, 1723, 4.0)])
def test_sc_equals_fastssc_f32(N, K, ebn0):
    """f32: plain SC (O1) and Fast-SSC (O2) take identical decisions on every frame with no
    exactly-zero hard decision (SURVEY 8(c) pin 5; Rate-1 proof in Appendix A; Rep and
    SPC agree with SC under reading C13 / because SC on an SPC node is the Wagner rule)."""
    frozen, bits, x, llr = _frames(N, K, ebn0, 400, 11)
    xs, _, zd = oracle.sc_decode(frozen, llr, with_stats=True)
    xf = oracle.fastssc_decode(frozen, llr)
    clean = zd == 0
    assert clean.mean() > 0.95
    assert np.array_equal(xs[clean], xf[clean])


@pytest.mark.parametrize("N,K,ebn0", [(256, 128, 2.0), (1024, 512, 2.5), (2048, 1723, 4.0)])
def test_sc_equals_fastssc_i8(N, K, ebn0):
    """int8: O1 == O2 on frames where SC took no decision on an exact zero (pin 6)."""
    frozen, bits, x, llr = _frames(N, K, ebn0, 400, 12, i8=True)
    xs, _, zd = oracle.sc_decode(frozen, llr, with_stats=True)
    xf = oracle.fastssc_decode(frozen, llr)
    clean = zd == 0
    assert clean.mean() > 0.5
    assert np.array_equal(xs[clean], xf[clean])


def test_sc_equals_fastssc_random_masks():
    """Same agreement on arbitrary (non-constructed) frozen sets, f32."""
    for seed in range(10):
        N = [16, 32, 64, 128][seed % 4]
        K = 1 + (seed * 37) % (N - 1)
        frozen = si.random_mask(seed, N, K)
        llr = si.random_llr_f32(seed, (50, N))
        xs, _, zd = oracle.sc_decode(frozen, llr, with_stats=True)
        xf = oracle.fastssc_decode(frozen, llr)
        clean = zd == 0
        assert np.array_equal(xs[clean], xf[clean])


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("i8", [False, True])
def test_outputs_are_codewords_and_noiseless_roundtrip(i8):
    """Every decoder output is a codeword ((xhat G)[F] = 0), and a noiseless frame
    decodes to the transmitted codeword (x[A] = d)."""
    N, K = 1024, 512
    frozen, bits, x, llr = _frames(N, K, 2.5, 200, 13, i8=i8)
    for dec in (oracle.fastssc_decode, oracle.sc_decode):
        xh = dec(frozen, llr)
        assert not oracle.encode(xh)[:, frozen == 1].any()
    clean = (1.0 - 2.0 * x).astype(np.float32) * 8.0
    if i8:
        clean = si.quantize_i8(clean)
    for dec in (oracle.fastssc_decode, oracle.sc_decode):
        xh = dec(frozen, clean)
        assert np.array_equal(xh, x)
        assert np.array_equal(oracle.info_bits(frozen, xh), bits)


def test_int8_minus128_is_clamped():
    """-128 is outside the symmetric range (reading C8): decoded as -127."""
    frozen = oracle.construct_ga(64, 32, 2.0)
    a = si.random_llr_i8(3, (40, 64))
    a[:, ::3] = -128
    b = a.copy(); b[b == -128] = -127
    assert np.array_equal(oracle.fastssc_decode(frozen, a), oracle.fastssc_decode(frozen, b))
    assert np.array_equal(oracle.sc_decode(frozen, a), oracle.sc_decode(frozen, b))


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    b = rng.integers(0, 2, (5, 77), dtype=np.uint8)
    w = oracle.pack_bits(b)
    assert w.shape == (5, 3) and w.dtype == np.uint32
    assert np.array_equal(oracle.unpack_bits(w, 77), b)
    assert int(oracle.pack_bits(np.array([[1, 0, 1]], np.uint8))[0, 0]) == 5


# ------------------------------------------------------------------ construction
def test_bhattacharyya_closed_forms():
    """BEC(z0): the all-minus channel has z = 1 - (1 - z0)^N and the all-plus z0^N."""
    z = oracle.bhattacharyya_bec(8, 0.5)
    assert z[0] == pytest.approx(1 - 0.5 ** 8)
    assert z[7] == pytest.approx(0.5 ** 8)
    # capacity is conserved on the BEC: sum of (1 - z_i) = N (1 - z0)
    for N in (8, 64, 1024):
        assert np.sum(1 - oracle.bhattacharyya_bec(N, 0.3)) == pytest.approx(N * 0.7)


def test_ga_ordering_n8_matches_bhattacharyya():
    """For N = 8 the GA ranks bit channels 0,1,2,4,3,5,6,7 (least reliable first) at every
    design SNR from -3 to 10 dB, the same order as the textbook BEC(0.5) recursion
    (SURVEY 0.1 fact 3).  Hence no reliability construction yields P:187-194's {0,1,4}."""
    zorder = list(np.argsort(-oracle.bhattacharyya_bec(8, 0.5), kind="stable"))
    assert zorder == [0, 1, 2, 4, 3, 5, 6, 7]
    for snr in np.arange(-3.0, 10.5, 0.5):
        m = oracle.ga_means(8, 4, float(snr))
        assert list(np.argsort(m, kind="stable")) == zorder
        assert set(np.flatnonzero(oracle.construct_ga(8, 5, float(snr)))) == {0, 1, 2}


@pytest.mark.parametrize("N,K,ebn0", [(64, 32, 1.0), (1024, 512, 2.5), (2048, 1723, 4.0), (32768, 29492, 4.5)])
def test_ga_respects_bit_dominance(N, K, ebn0):
    """Universal partial order: if the bits of i are a subset of the bits of j, channel j is
    at least as reliable (a theorem for any symmetric channel).  So the GA means are
    monotone under bit dominance and the information set is superset-closed."""
    m = oracle.ga_means(N, K, ebn0)
    n = N.bit_length() - 1
    for b in range(n):
        i = np.arange(N)
        lo = i[(i >> b) & 1 == 0]
        assert np.all(m[lo | (1 << b)] >= m[lo] * (1 - 1e-12))
    frozen = oracle.construct_ga(N, K, ebn0)
    assert frozen.sum() == N - K
    info = np.flatnonzero(frozen == 0)
    for b in range(n):
        assert np.all(frozen[info | (1 << b)] == 0)


def test_phi_inverse():
    for x in (0.01, 0.5, 3.0, 9.9, 10.5, 40.0, 500.0, 1e5):
        y = oracle.lib().or_log_phi(x)
        assert oracle.lib().or_inv_log_phi(y) == pytest.approx(x, rel=1e-9)


def test_phi_against_its_definition():
    """Chung's two-piece phi (or_log_phi) against phi's definition as an integral,
    phi(x) = 1 - (4 pi x)^-1/2 * int tanh(u/2) exp(-(u - x)^2 / (4x)) du (Chung et al. 2001,
    the function the GA recursion m- = phi^-1(1 - (1 - phi(m))^2) is written in), evaluated by
    quadrature: the approximation is within 3.5% of the exact value over [0.05, 80]; a wrong
    constant (0.4527, 0.86, 0.0218, or the x >= 10 tail) moves it by 10% or more."""
    from scipy.integrate import quad

    def exact(x):
        r = 40.0 * np.sqrt(x) + 5.0
        v, _ = quad(lambda u: np.tanh(u / 2.0) * np.exp(-(u - x) ** 2 / (4.0 * x)), x - r, x + r, limit=400)
        return 1.0 - v / np.sqrt(4.0 * np.pi * x)

    for x in (0.05, 0.1, 0.3, 1.0, 2.0, 5.0, 9.9, 10.1, 15.0, 20.0, 40.0, 80.0):
        assert np.exp(oracle.lib().or_log_phi(x)) / exact(x) == pytest.approx(1.0, abs=0.035), x


# Op and element counts of the unfused Listing-1 schedule for the GA masks, as written by the
# committed oracle-only script tools/gen_op_counts.py into tests/golden/op_counts.txt (they
# reproduce SURVEY section 8's table; a mismatch means a different mask or schedule).
def _op_counts():
    rows = []
    for line in open(os.path.join(GOLD, "op_counts.txt")):
        if line.strip() and not line.startswith("#"):
            N, K, e, ops, f, g, leaf = line.split()
            rows.append(((int(N), int(K), float(e)), (int(ops), int(f), int(g), int(leaf))))
    return rows


@pytest.mark.parametrize("code,counts", _op_counts())
def test_op_counts_match_golden(code, counts):
    import re

    N, K, ebn0 = code
    ops = oracle.fastssc_trace(oracle.construct_ga(N, K, ebn0))
    f = sum(int(n) // 2 for o, n in (re.match(r"(\w+)<(\d+)>", x).groups() for x in ops) if o == "F")
    assert (len(ops), f) == counts[:2]


# ------------------------------------------------------------------ statistics (weak pins)
def _q(x):
    from math import erfc, sqrt
    return 0.5 * erfc(x / sqrt(2.0))


@pytest.mark.slow
def test_fer_close_to_ga_prediction_and_int8_loss_small():
    """FER of (1024,512) at 2.5 dB vs the GA union/product estimate
    1 - prod_{i in A} (1 - Q(sqrt(m_i / 2))) (SURVEY 8(c) pin 9, weak), and the 8-bit
    profile costs little error-correction performance."""
    N, K, ebn0, n = 1024, 512, 2.5, 3000
    frozen, bits, x, llr = _frames(N, K, ebn0, n, 21)
    m = oracle.ga_means(N, K, ebn0)
    pred = 1.0 - np.prod([1.0 - _q(np.sqrt(m[i] / 2.0)) for i in np.flatnonzero(frozen == 0)])
    fer = np.mean(np.any(oracle.fastssc_decode(frozen, llr) != x, axis=1))
    assert 0.4 * pred < fer < 2.5 * pred
    fer8 = np.mean(np.any(oracle.fastssc_decode(frozen, si.quantize_i8(llr)) != x, axis=1))
    assert fer8 < 1.5 * fer + 10.0 / n


def _alpha_bytes(N, elem, align):
    """alpha memory of the paper's layout: log2(N)+1 contiguous stages of N, N/2, ..., 1
    values, each stage aligned to the SIMD width (16 B SSE / 32 B AVX)."""
    total, m = 0, N
    while m >= 1:
        total += -(-m * elem // align) * align
        m //= 2
    return total


def test_paper_memory_closed_forms():
    """SURVEY 8(c) pin 8: the memory figures the paper prints follow from its stated layout."""
    # N = 32768 float decoder with AVX: 262,208 bytes including a 68-byte overhead
    packed = (2 * 32768 - 1) * 4
    assert _alpha_bytes(32768, 4, 32) == 262208
    assert _alpha_bytes(32768, 4, 32) - packed == 68
    # P:929-932 (tab:impl:tp_vs_gal): int8 AVX2 footprints 6 kB (N = 2048) and 98 kB (N = 32768):
    # alpha (32-byte aligned int8 stages) + beta as one byte per codeword bit (decimal kB, as
    # the 3,408 kB below): 6,272 B and 98,432 B
    assert round((_alpha_bytes(2048, 1, 32) + 2048) / 1000) == 6
    assert round((_alpha_bytes(32768, 1, 32) + 32768) / 1000) == 98
    # P:1242 (tab:impl:power_vs_gal): 3,408 kB per stream on the K20c for 208 frames of the
    # (2048,1707) float decoder = 208 x (N input LLRs + N output values) x 4 bytes
    assert round(208 * (2048 + 2048) * 4 / 1000) == 3408


@pytest.mark.parametrize("N,K,ebn0", [(16, 8, 2.0), (256, 128, 2.0), (1024, 512, 2.5)])
def test_nonsystematic_information_is_uhat_on_a(N, K, ebn0):
    """Non-systematic reading (C4): for x = u G_N with u[A] = d, u[F] = 0
    (P:138-155), the decoded codeword mapped back by G_N (its own inverse) gives u_hat with
    u_hat[A] = d and u_hat[F] = 0 on noiseless frames; SC's leaf decisions are that u_hat."""
    frozen = oracle.construct_ga(N, K, ebn0)
    bits, _ = si.draw(9, 0, 16, K, N)
    u = np.zeros((16, N), np.uint8)
    u[:, frozen == 0] = bits
    x = oracle.encode(u)
    llr = np.where(x == 0, 6.0, -6.0).astype(np.float32)
    uh = oracle.encode(oracle.fastssc_decode(frozen, llr))
    assert np.array_equal(uh[:, frozen == 0], bits) and not uh[:, frozen == 1].any()
    _, us, _ = oracle.sc_decode(frozen, llr, with_stats=True)
    assert np.array_equal(us, uh)


@pytest.mark.parametrize("N,K,ebn0", [(64, 32, 2.0), (256, 128, 2.0), (1024, 700, 3.0)])
def test_node_sets_of_the_ablation(N, K, ebn0):
    """The ablation's node sets against what fixes them: the plain-SC
    set reproduces O1 (recursive SC) exactly, int8 and f32, and visits every
    bit (N leaves); on f32 frames without an exact-zero decision every set equals O1 (the
    special-node rules are ML for their constituent codes, pin 5); the Fast-SSC set is O2."""
    frozen = oracle.construct_ga(N, K, ebn0)
    bits, noise = si.draw(21, 0, 48, K, N)
    llr = si.bpsk_awgn_llr(oracle.encode_systematic(frozen, bits), noise, ebn0 - 1.5, K)
    q = si.quantize_i8(llr)
    assert np.array_equal(oracle.nodeset_decode(frozen, q, "sc"), oracle.sc_decode(frozen, q))
    assert np.array_equal(oracle.nodeset_decode(frozen, llr, "sc"), oracle.sc_decode(frozen, llr))
    assert np.array_equal(oracle.nodeset_decode(frozen, q, "fastssc"), oracle.fastssc_decode(frozen, q))
    xs, _, zd = oracle.sc_decode(frozen, llr, with_stats=True)
    keep = zd == 0
    for s in ("nospc", "ssc"):
        assert np.array_equal(oracle.nodeset_decode(frozen, llr, s)[keep], xs[keep]), s
    tr = oracle.nodeset_trace(frozen, "sc")
    assert sum(1 for t in tr if t == "Info<1>") == K  # every information bit is its own leaf
    n_ops = [len(oracle.nodeset_trace(frozen, s)) for s in ("sc", "ssc", "nospc", "fastssc")]
    assert n_ops == sorted(n_ops, reverse=True) and n_ops[-1] == len(oracle.fastssc_trace(frozen))
