"""C-ABI library checks that need no GPU: the library loads, exports every symbol of
include/polar.h, creates handles for its specialised codes, and its host-side logic (GA
construction, Fast-SSC tree and op schedule) agrees with the oracle and the paper."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_1504_00353_b200 as pb
from seeded_inputs import random_mask

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "polar.h")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(polar_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = pb.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(pb.EXPORTS) == declared


def test_status_strings():
    L = pb.lib()
    for s in range(5):
        assert L.polar_status_string(s).decode()


def _codes_spec():
    """(name, N, K, how, arg) of every line of codes.txt / codes_random.txt."""
    out = []
    for fn in ("codes.txt", "codes_random.txt"):
        for line in open(os.path.join(ROOT, "paper_1504_00353_b200", fn)):
            line = line.split("#")[0].split()
            if len(line) >= 5:
                out.append((line[0], int(line[1]), int(line[2]), line[3], line[4]))
    return out


def test_registry_matches_spec_and_oracle_construction():
    reg = pb.registry()
    spec = _codes_spec()
    assert len(reg) == len(spec)
    for (N, K, m), (name, sN, sK, how, arg) in zip(reg, spec):
        assert (N, K) == (sN, sK), name
        assert int(m.sum()) == N - K
        if how == "ga":
            # product GA (csrc/construct.cpp) == oracle GA (oracle/polar_oracle.c), reading C1
            np.testing.assert_array_equal(m, oracle.construct_ga(N, K, float(arg)), err_msg=name)
        else:
            np.testing.assert_array_equal(m, np.array([c == "1" for c in arg], np.uint8), err_msg=name)


def test_construct_ga_matches_oracle_off_registry():
    for N, K, e in [(64, 20, 1.0), (512, 300, 2.0), (4096, 1000, 0.5), (16384, 15000, 5.0)]:
        np.testing.assert_array_equal(pb.construct_ga(N, K, e), oracle.construct_ga(N, K, e))


def test_listing1_schedule_from_the_library():
    """Listing 1 reproduced by the product's own schedule for the (8,5) code."""
    lines = [l.strip() for l in open(os.path.join(GOLDEN, "listing1_8_5.txt")) if not l.startswith("#")]
    mask = np.array([int(c) for c in lines[0]], np.uint8)
    code = pb.PolarCode(8, 5, mask)
    assert code.schedule() == [l for l in lines[1:] if l]
    assert code.n_ops == 7


def test_schedules_equal_oracle_traces():
    for N, K, m in pb.registry():
        code = pb.PolarCode(N, K, m)
        assert code.schedule() == oracle.fastssc_trace(m), (N, K)


@pytest.mark.parametrize("N,K,ops", [(1024, 512, 299), (2048, 1723, 371), (32768, 29492, 2607),
                                     (32768, 27568, 3577)])
def test_survey_op_counts(N, K, ops):
    design = {1024: 2.5, 2048: 4.0, 29492: 4.5, 27568: 4.0}[N if N < 32768 else K]
    assert pb.PolarCode.ga(N, K, design).n_ops == ops


def test_create_validation():
    m = pb.construct_ga(64, 32, 2.0)
    with pytest.raises(pb.PolarError) as e:
        pb.PolarCode(64, 33, m)  # popcount != N - K
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT
    with pytest.raises(ValueError):
        pb.PolarCode(64, 32, m[:32])
    bad = np.zeros(48, np.uint8)
    bad[:16] = 1
    with pytest.raises(pb.PolarError) as e:
        pb.PolarCode(48, 32, bad)  # N not a power of two
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT
    # a frozen set no decoder was specialised for gets the generic (interpreted) decoder when
    # run-time specialisation is off (tests/test_jit.py covers it)
    os.environ["POLAR_JIT"] = "0"
    try:
        g = pb.PolarCode(64, 32, random_mask(999, 64, 32))
    finally:
        del os.environ["POLAR_JIT"]
    assert not g.specialised
    assert g.schedule() == oracle.fastssc_trace(random_mask(999, 64, 32))
    assert pb.PolarCode(8, 5, np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8)).specialised


def test_handle_roundtrip_and_query():
    for N, K, m in pb.registry():
        c = pb.PolarCode(N, K, m)
        np.testing.assert_array_equal(c.mask(), m)
        assert c.N == N and c.K == K and c.smem_bytes > 0
        assert c.warp_root <= min(N, 2048) and c.warp_root & (c.warp_root - 1) == 0
        c.close()


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = pb.PolarCode(8, 5, np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8))
    llr = torch.zeros(1, 8)
    out = torch.zeros(1, 1, dtype=torch.int32)
    with pytest.raises(ValueError):  # the binding refuses host tensors for the device call
        c.decode_f32(llr, out, stream=0)
    with pytest.raises(pb.PolarError) as e:  # the library itself has no CPU path
        pb._check(pb.lib().polar_decode_f32(c._h, llr.data_ptr(), 1, out.data_ptr(), None))
    assert e.value.status == pb.POLAR_ERR_CUDA


def test_binding_rejects_bad_tensors():
    """The C ABI takes raw pointers; the binding checks dtype, device, contiguity, the frame
    length and the output size before passing them."""
    torch = pytest.importorskip("torch")
    c = pb.PolarCode(8, 5, np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8))
    ok = torch.zeros(4, 8, dtype=torch.int8)
    for bad in (torch.zeros(4, 8), torch.zeros(4, 16, dtype=torch.int8), torch.zeros(8, 8, dtype=torch.int8)[::2],
                torch.zeros(3, dtype=torch.int8)):
        with pytest.raises(ValueError):
            c.decode_host(bad if bad.dtype == torch.int8 else bad.to(torch.float64), torch.zeros(4, 1, dtype=torch.int32))
    for out in (torch.zeros(3, 1, dtype=torch.int32), torch.zeros(4, 1, dtype=torch.int64), np.zeros((4, 1), np.uint8)):
        with pytest.raises(ValueError):
            c.decode_host(ok, out)
    with pytest.raises(ValueError):
        c.decode_i8(ok)  # host tensor given to the device call


def test_variant_and_mailbox_argument_checks_without_gpu():
    """Variant selection accepts 0..4 (4 = frame-interleaved) and rejects the rest; the batch-1
    mailbox reports a missing device or a code built without it, and never falls back to the CPU."""
    torch = pytest.importorskip("torch")
    c = pb.PolarCode(8, 5, np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8))
    for v in ("auto", "throughput", "latency", "generic", "xframe"):
        c.set_variant(v)
    with pytest.raises(pb.PolarError) as e:
        pb._check(pb.lib().polar_code_set_variant(c._h, 5))
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT
    out = np.zeros(1, np.uint32)
    with pytest.raises(pb.PolarError) as e:  # not open
        c.mailbox_decode_i8(np.zeros(8, np.int8), out)
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT
    with pytest.raises(pb.PolarError) as e:
        pb._check(pb.lib().polar_mailbox_open(c._h, 0.0))  # idle_seconds must be > 0
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT
    c.mailbox_close()  # closing a mailbox that is not open is a no-op
    if not torch.cuda.is_available():
        for code in (c, pb.PolarCode.ga(2048, 1723, 4.0)):
            with pytest.raises(pb.PolarError) as e:
                code.mailbox_open()
            assert e.value.status == pb.POLAR_ERR_CUDA


def test_output_mode_argument_checks():
    c = pb.PolarCode(8, 5, np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8))
    c.set_output("nonsystematic")
    c.set_output("systematic")
    with pytest.raises(pb.PolarError) as e:
        pb._check(pb.lib().polar_code_set_output(c._h, 2))
    assert e.value.status == pb.POLAR_ERR_INVALID_ARGUMENT
