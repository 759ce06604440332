"""CPU oracle for Fast-SSC polar decoding -- TEST INFRASTRUCTURE ONLY.

Thin ctypes/numpy wrapper over ``oracle/polar_oracle.c`` (plain C, built with
``-fno-fast-math -ffp-contract=off``).  See the C file's header for what each function
follows in the paper (arXiv:1504.00353, PAPER.md line citations).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference
legs may import this package.  The product (``paper_1504_00353_b200``) never does; the two
share no code.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "polar_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=gnu11", "-fPIC", "-shared", "-fno-fast-math", "-ffp-contract=off"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        _i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
        _f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        _f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        _i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        L = _lib
        L.or_f_f32.argtypes = [C.c_float, C.c_float]; L.or_f_f32.restype = C.c_float
        L.or_g_f32.argtypes = [C.c_float, C.c_float, C.c_int]; L.or_g_f32.restype = C.c_float
        L.or_f_i8.argtypes = [C.c_int, C.c_int]; L.or_f_i8.restype = C.c_int
        L.or_g_i8.argtypes = [C.c_int, C.c_int, C.c_int]; L.or_g_i8.restype = C.c_int
        L.or_encode.argtypes = [C.c_int, _u8p, _u8p]
        L.or_encode_matrix.argtypes = [C.c_int, _u8p, _u8p]
        L.or_encode_systematic.argtypes = [C.c_int, _u8p, _u8p, _u8p]
        L.or_sc_decode_f32.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_sc_decode_i8.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_fastssc_decode_f32.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_long, C.c_void_p]
        L.or_fastssc_decode_i8.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_long, C.c_void_p]
        L.or_fastssc_trace.argtypes = [C.c_int, _u8p, C.c_char_p, C.c_int]; L.or_fastssc_trace.restype = C.c_int
        L.or_fastssc_dump_f32.argtypes = [C.c_int, _u8p, _f32p, _u8p, _f32p, C.c_long]
        L.or_fastssc_dump_f32.restype = C.c_long
        L.or_fastssc_dump_i8.argtypes = [C.c_int, _u8p, _i8p, _u8p, _i32p, C.c_long]
        L.or_fastssc_dump_i8.restype = C.c_long
        L.or_nodeset_decode_f32.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_long, C.c_void_p, C.c_int]
        L.or_nodeset_decode_i8.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_long, C.c_void_p, C.c_int]
        L.or_nodeset_trace.argtypes = [C.c_int, _u8p, C.c_int, C.c_char_p, C.c_int]
        L.or_nodeset_trace.restype = C.c_int
        L.or_ml_decode_f32.argtypes = [C.c_int, _u8p, _f32p, C.c_long, _u8p]
        L.or_rep_f32.argtypes = [C.c_int, _f32p, _u8p]
        L.or_spc_f32.argtypes = [C.c_int, _f32p, _u8p]
        L.or_rep_i8_bytes.argtypes = [C.c_int, _i8p, _u8p]
        L.or_spc_i8_bytes.argtypes = [C.c_int, _i8p, _u8p]
        L.or_classify.argtypes = [C.c_int, _u8p]; L.or_classify.restype = C.c_int
        L.or_log_phi.argtypes = [C.c_double]; L.or_log_phi.restype = C.c_double
        L.or_inv_log_phi.argtypes = [C.c_double]; L.or_inv_log_phi.restype = C.c_double
        L.or_ga_means.argtypes = [C.c_int, C.c_int, C.c_double, _f64p]
        L.or_construct_ga.argtypes = [C.c_int, C.c_int, C.c_double, _u8p]
        L.or_bhattacharyya_bec.argtypes = [C.c_int, C.c_double, _f64p]
        _ = (_i32p,)
    return _lib


# ---------------------------------------------------------------- scalar primitives
def f_f32(a: float, b: float) -> float:
    return lib().or_f_f32(a, b)


def g_f32(a: float, b: float, beta: int) -> float:
    return lib().or_g_f32(a, b, beta)


def f_i8(a: int, b: int) -> int:
    return lib().or_f_i8(a, b)


def g_i8(a: int, b: int, beta: int) -> int:
    return lib().or_g_i8(a, b, beta)


# ---------------------------------------------------------------- construction / encoding
def construct_ga(N: int, K: int, design_ebn0_db: float) -> np.ndarray:
    """Frozen mask (uint8[N], 1 = frozen), GA construction (reading C1)."""
    m = np.zeros(N, np.uint8)
    lib().or_construct_ga(N, K, design_ebn0_db, m)
    return m


def ga_means(N: int, K: int, design_ebn0_db: float) -> np.ndarray:
    m = np.zeros(N, np.float64)
    lib().or_ga_means(N, K, design_ebn0_db, m)
    return m


def bhattacharyya_bec(N: int, z0: float) -> np.ndarray:
    z = np.zeros(N, np.float64)
    lib().or_bhattacharyya_bec(N, z0, z)
    return z


def encode(u: np.ndarray) -> np.ndarray:
    """x = u G_N (block recursion). u: uint8[..., N]."""
    u = np.ascontiguousarray(u, np.uint8)
    N = u.shape[-1]
    flat = u.reshape(-1, N)
    out = np.empty_like(flat)
    for r in range(flat.shape[0]):
        row = np.ascontiguousarray(flat[r]); o = np.empty(N, np.uint8)
        lib().or_encode(N, row, o)
        out[r] = o
    return out.reshape(u.shape)


def encode_matrix(u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, np.uint8)
    N = u.shape[-1]
    o = np.empty(N, np.uint8)
    lib().or_encode_matrix(N, u, o)
    return o


def encode_systematic(frozen: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Systematic codewords x with x[A] = d (reading C4). d: uint8[n, K] -> uint8[n, N]."""
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    d = np.ascontiguousarray(d, np.uint8)
    d2 = d.reshape(-1, d.shape[-1])
    out = np.empty((d2.shape[0], N), np.uint8)
    for r in range(d2.shape[0]):
        o = np.empty(N, np.uint8)
        lib().or_encode_systematic(N, frozen, np.ascontiguousarray(d2[r]), o)
        out[r] = o
    return out


# ---------------------------------------------------------------- decoders
def _frames(llr: np.ndarray, N: int, dtype) -> np.ndarray:
    a = np.ascontiguousarray(llr, dtype)
    assert a.size % N == 0
    return a.reshape(-1, N)


def sc_decode(frozen: np.ndarray, llr: np.ndarray, with_stats: bool = False):
    """O1 plain SC. llr float32 or int8, shape [n, N]. Returns xhat uint8[n, N]
    (and uhat, zero-decision counts when with_stats)."""
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    is_i8 = np.asarray(llr).dtype == np.int8
    a = _frames(llr, N, np.int8 if is_i8 else np.float32)
    n = a.shape[0]
    xhat = np.empty((n, N), np.uint8)
    uhat = np.empty((n, N), np.uint8)
    zd = np.zeros(n, np.int32)
    fn = lib().or_sc_decode_i8 if is_i8 else lib().or_sc_decode_f32
    fn(N, frozen, a.ctypes.data, n, xhat.ctypes.data, uhat.ctypes.data, zd.ctypes.data)
    if with_stats:
        return xhat, uhat, zd
    return xhat


def fastssc_decode(frozen: np.ndarray, llr: np.ndarray, threads: int = 1) -> np.ndarray:
    """O2 straightforward Fast-SSC. llr float32 or int8 [n, N] -> xhat uint8[n, N].
    threads > 1 splits frames over Python threads (ctypes releases the GIL)."""
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    is_i8 = np.asarray(llr).dtype == np.int8
    a = _frames(llr, N, np.int8 if is_i8 else np.float32)
    n = a.shape[0]
    xhat = np.empty((n, N), np.uint8)
    fn = lib().or_fastssc_decode_i8 if is_i8 else lib().or_fastssc_decode_f32
    if threads <= 1 or n < 2:
        fn(N, frozen, a.ctypes.data, n, xhat.ctypes.data)
        return xhat
    bounds = np.linspace(0, n, threads + 1).astype(np.int64)

    def run(t):
        lo, hi = int(bounds[t]), int(bounds[t + 1])
        if hi > lo:
            fn(N, frozen, a[lo:hi].ctypes.data, hi - lo, xhat[lo:hi].ctypes.data)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(threads)))
    return xhat


NODE_SETS = {"fastssc": 0, "nospc": 1, "ssc": 2, "sc": 3}


def nodeset_decode(frozen: np.ndarray, llr: np.ndarray, node_set: str, threads: int = 1) -> np.ndarray:
    """O2's traversal restricted to a node set ('fastssc', 'nospc', 'ssc', 'sc'; the paper's
    algorithm ablation): xhat uint8[n, N]."""
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    is_i8 = np.asarray(llr).dtype == np.int8
    a = _frames(llr, N, np.int8 if is_i8 else np.float32)
    n = a.shape[0]
    xhat = np.empty((n, N), np.uint8)
    fn = lib().or_nodeset_decode_i8 if is_i8 else lib().or_nodeset_decode_f32
    bounds = np.linspace(0, n, max(1, threads) + 1).astype(np.int64)

    def run(t):
        lo, hi = int(bounds[t]), int(bounds[t + 1])
        if hi > lo:
            fn(N, frozen, a[lo:hi].ctypes.data, hi - lo, xhat[lo:hi].ctypes.data, NODE_SETS[node_set])

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(run, range(max(1, threads))))
    return xhat


def nodeset_trace(frozen: np.ndarray, node_set: str) -> list[str]:
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    cap = 64 * N + 64
    buf = C.create_string_buffer(cap)
    lib().or_nodeset_trace(N, frozen, NODE_SETS[node_set], buf, cap)
    return [t for t in buf.value.decode().split(";") if t]


def fastssc_trace(frozen: np.ndarray) -> list[str]:
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    cap = 64 * N + 64
    buf = C.create_string_buffer(cap)
    lib().or_fastssc_trace(N, frozen, buf, cap)
    s = buf.value.decode()
    return [t for t in s.split(";") if t]


def fastssc_alpha_dump(frozen: np.ndarray, llr: np.ndarray) -> np.ndarray:
    """O2 on ONE frame; every F / G / G_0R output vector in op order, concatenated (float32 for
    f32 input, int32 for int8 input): the intermediate LLRs of the decoder."""
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    x = np.ascontiguousarray(llr).reshape(N)
    cap = N * max(1, int(np.log2(N)))
    xhat = np.zeros(N, np.uint8)
    if x.dtype == np.int8:
        out = np.zeros(cap, np.int32)
        n = lib().or_fastssc_dump_i8(N, frozen, x, xhat, out, cap)
    else:
        out = np.zeros(cap, np.float32)
        n = lib().or_fastssc_dump_f32(N, frozen, x.astype(np.float32), xhat, out, cap)
    return out[:n]


def ml_decode(frozen: np.ndarray, llr: np.ndarray) -> np.ndarray:
    """O3 brute-force ML, N <= 16, float32 llr [n, N]."""
    frozen = np.ascontiguousarray(frozen, np.uint8)
    N = frozen.shape[0]
    assert N <= 16
    a = _frames(llr, N, np.float32)
    xhat = np.empty((a.shape[0], N), np.uint8)
    lib().or_ml_decode_f32(N, frozen, a, a.shape[0], xhat)
    return xhat


def rep_node(alpha: np.ndarray) -> np.ndarray:
    alpha = np.ascontiguousarray(alpha)
    out = np.empty(alpha.shape[0], np.uint8)
    if alpha.dtype == np.int8:
        lib().or_rep_i8_bytes(alpha.shape[0], alpha, out)
    else:
        lib().or_rep_f32(alpha.shape[0], np.ascontiguousarray(alpha, np.float32), out)
    return out


def spc_node(alpha: np.ndarray) -> np.ndarray:
    alpha = np.ascontiguousarray(alpha)
    out = np.empty(alpha.shape[0], np.uint8)
    if alpha.dtype == np.int8:
        lib().or_spc_i8_bytes(alpha.shape[0], alpha, out)
    else:
        lib().or_spc_f32(alpha.shape[0], np.ascontiguousarray(alpha, np.float32), out)
    return out


def classify(frozen: np.ndarray) -> str:
    k = lib().or_classify(len(frozen), np.ascontiguousarray(frozen, np.uint8))
    return ["Rate0", "Rate1", "Rep", "SPC", "Split"][k]


# ---------------------------------------------------------------- helpers used by tests/bench
def info_bits(frozen: np.ndarray, xhat: np.ndarray) -> np.ndarray:
    """Systematic information bits x[A], A ascending (reading C5)."""
    return xhat[..., np.flatnonzero(np.asarray(frozen) == 0)]


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """uint8 bits [n, K] -> uint32 words [n, ceil(K/32)], LSB-first (reading C5)."""
    bits = np.asarray(bits, np.uint8)
    n, K = bits.shape
    W = (K + 31) // 32
    pad = np.zeros((n, W * 32), np.uint64)
    pad[:, :K] = bits
    pad = pad.reshape(n, W, 32)
    words = (pad << np.arange(32, dtype=np.uint64)).sum(axis=2)
    return words.astype(np.uint32)


def unpack_bits(words: np.ndarray, K: int) -> np.ndarray:
    words = np.asarray(words, np.uint32)
    n, W = words.shape
    bits = (words[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(n, W * 32)[:, :K].astype(np.uint8)
