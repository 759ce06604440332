"""B200-native Fast-SSC polar decoding (Giard et al., arXiv:1504.00353).

Thin ctypes binding over ``libpolar.so`` (C ABI declared in ``include/polar.h``): argument
marshalling only.  Every step of the decode runs in the library's sm_100a kernels; torch is
used for device memory and streams.  There is no CPU fallback: if the library is missing
the import of ``lib()`` raises, and without a GPU every device call raises ``PolarError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# POLAR_LIB selects an experiment build (tools/variant_build.sh); default: the in-tree library.
LIB_PATH = os.environ.get("POLAR_LIB", os.path.join(_HERE, "libpolar.so"))

POLAR_OK = 0
POLAR_ERR_INVALID_ARGUMENT = 1
POLAR_ERR_UNSUPPORTED_CODE = 2
POLAR_ERR_CUDA = 3
POLAR_ERR_OUT_OF_MEMORY = 4

# Every symbol include/polar.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "polar_status_string", "polar_last_error", "polar_code_create", "polar_code_destroy",
    "polar_code_query", "polar_code_schedule", "polar_code_mask", "polar_code_set_variant",
    "polar_code_is_specialised", "polar_code_set_output", "polar_decode_f32",
    "polar_decode_i8", "polar_decode_f32_host", "polar_decode_i8_host", "polar_mailbox_open",
    "polar_mailbox_decode_i8", "polar_mailbox_close", "polar_construct_ga",
    "polar_encode_systematic", "polar_gen_bpsk_awgn", "polar_count_errors",
    "polar_registry_size", "polar_registry_entry", "polar_trace_fetch", "polar_debug_dump_stride",
    "polar_debug_dump_fetch", "polar_jit_compile",
]


class PolarError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_libs: dict[str, C.CDLL] = {}
DUMP_LIB_PATH = os.path.join(_HERE, "libpolar_dump.so")


def lib() -> C.CDLL:
    """Load libpolar.so (built by ``build()``); raises if it is absent."""
    return _load(LIB_PATH)


def dump_lib() -> C.CDLL:
    """libpolar_dump.so: the POLAR_DEBUG_DUMP build (test infrastructure: alpha-stage dumps)."""
    return _load(DUMP_LIB_PATH)


def _load(path: str) -> C.CDLL:
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run paper_1504_00353_b200.build.build() first")
    L = C.CDLL(path)
    vp, u8p, u32p, i64p = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_int64)
    sig = {
        "polar_status_string": (C.c_char_p, [C.c_int]),
        "polar_last_error": (C.c_char_p, []),
        "polar_code_create": (C.c_int, [C.c_uint32, C.c_uint32, vp, C.POINTER(vp)]),
        "polar_code_destroy": (None, [vp]),
        "polar_code_query": (C.c_int, [vp, u32p, u32p, u32p, u32p, u32p]),
        "polar_code_schedule": (C.c_int, [vp, C.c_char_p, C.c_uint32, u32p]),
        "polar_code_mask": (C.c_int, [vp, vp]),
        "polar_code_set_variant": (C.c_int, [vp, C.c_int]),
        "polar_code_set_output": (C.c_int, [vp, C.c_int]),
        "polar_code_is_specialised": (C.c_int, [vp, C.POINTER(C.c_int)]),
        "polar_decode_f32": (C.c_int, [vp, vp, C.c_int64, vp, vp]),
        "polar_decode_i8": (C.c_int, [vp, vp, C.c_int64, vp, vp]),
        "polar_decode_f32_host": (C.c_int, [vp, vp, C.c_int64, vp]),
        "polar_decode_i8_host": (C.c_int, [vp, vp, C.c_int64, vp]),
        "polar_mailbox_open": (C.c_int, [vp, C.c_double]),
        "polar_mailbox_decode_i8": (C.c_int, [vp, vp, vp, C.c_double]),
        "polar_mailbox_close": (C.c_int, [vp]),
        "polar_construct_ga": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, vp]),
        "polar_encode_systematic": (C.c_int, [vp, vp, C.c_int64, vp, vp]),
        "polar_gen_bpsk_awgn": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_float,
                                          vp, vp, vp, vp]),
        "polar_count_errors": (C.c_int, [vp, vp, vp, C.c_int64, vp, vp]),
        "polar_registry_size": (C.c_uint32, []),
        "polar_trace_fetch": (C.c_int, [vp, vp, C.c_uint32]),
        "polar_debug_dump_stride": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
        "polar_debug_dump_fetch": (C.c_int, [vp, vp, C.c_uint64]),
        "polar_jit_compile": (C.c_int, [C.c_uint32, C.c_uint32, vp, C.c_char_p, C.c_uint32]),
        "polar_registry_entry": (C.c_int, [C.c_uint32, u32p, u32p, vp]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(L, name):  # an older experiment build (tools/variant_build.sh); tests check the product's
            continue
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _ = (u8p, i64p)
    _libs[path] = L
    return L


def _check(status: int, L: C.CDLL | None = None) -> None:
    if status != POLAR_OK:
        L = L or lib()
        raise PolarError(status, f"{L.polar_status_string(status).decode()}: {L.polar_last_error().decode()}")


def _ptr(t) -> int | None:
    """Device/host address of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def construct_ga(N: int, K: int, design_ebn0_db: float) -> np.ndarray:
    """Frozen mask (uint8[N], 1 = frozen) of the GA construction (reading C1)."""
    m = np.zeros(N, np.uint8)
    _check(lib().polar_construct_ga(N, K, float(design_ebn0_db), m.ctypes.data))
    return m


def jit_compile(N: int, K: int, frozen_mask: np.ndarray) -> str:
    """Generate and NVRTC-compile the unrolled decoder of a frozen set (no device needed);
    returns the cache tag, raises PolarError with NVRTC's log on failure."""
    m = np.ascontiguousarray(np.asarray(frozen_mask, np.uint8))
    buf = C.create_string_buffer(4096)
    _check(lib().polar_jit_compile(N, K, m.ctypes.data, buf, 4096))
    return buf.value.decode()


def registry() -> list[tuple[int, int, np.ndarray]]:
    """(N, K, frozen mask) of every code specialised into this build."""
    L = lib()
    out = []
    for i in range(L.polar_registry_size()):
        n, k = C.c_uint32(), C.c_uint32()
        _check(L.polar_registry_entry(i, C.byref(n), C.byref(k), None))
        m = np.zeros(n.value, np.uint8)
        _check(L.polar_registry_entry(i, None, None, m.ctypes.data))
        out.append((n.value, k.value, m))
    return out


class PolarCode:
    """Handle of one (N, K, frozen set) code: ``polar_code_create`` / ``polar_code_destroy``."""

    def __init__(self, N: int, K: int, frozen_mask: np.ndarray, library: C.CDLL | None = None):
        self._L = library or lib()
        m = np.ascontiguousarray(np.asarray(frozen_mask, np.uint8))
        if m.shape != (N,):
            raise ValueError("frozen mask must have N entries")
        h = C.c_void_p()
        self._chk(self._L.polar_code_create(N, K, m.ctypes.data, C.byref(h)))
        self._h = h
        n, k, ops, smem, wr = (C.c_uint32() for _ in range(5))
        self._chk(self._L.polar_code_query(h, C.byref(n), C.byref(k), C.byref(ops), C.byref(smem), C.byref(wr)))
        self.N, self.K, self.n_ops, self.smem_bytes, self.warp_root = n.value, k.value, ops.value, smem.value, wr.value
        self.info_words = (self.K + 31) // 32
        sp = C.c_int()
        self._chk(self._L.polar_code_is_specialised(h, C.byref(sp)))
        self.specialised = bool(sp.value)
        self.run_time_specialised = sp.value == 2

    def _chk(self, status: int) -> None:
        _check(status, self._L)

    def alpha_dump(self, n_frames: int) -> np.ndarray:
        """POLAR_DEBUG_DUMP builds: float32 [n_frames, N log2 N], every F/G/G_0R output of the
        last decode in op order (NaN after the last one)."""
        st = C.c_uint64()
        self._chk(self._L.polar_debug_dump_stride(self._h, C.byref(st)))
        out = np.empty((n_frames, st.value), np.float32)
        self._chk(self._L.polar_debug_dump_fetch(self._h, out.ctypes.data, out.size))
        return out

    @classmethod
    def ga(cls, N: int, K: int, design_ebn0_db: float) -> "PolarCode":
        return cls(N, K, construct_ga(N, K, design_ebn0_db))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.polar_code_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_variant(self, variant: str) -> None:
        """'auto' | 'throughput' | 'latency' | 'generic' (all decode identically)."""
        self._chk(self._L.polar_code_set_variant(self._h, {"auto": 0, "throughput": 1, "latency": 2, "generic": 3, "xframe": 4}[variant]))

    def set_output(self, mode: str) -> None:
        """'systematic' (x_hat[A], default) | 'nonsystematic' (u_hat[A], u_hat = x_hat G_N)."""
        self._chk(self._L.polar_code_set_output(self._h, {"systematic": 0, "nonsystematic": 1}[mode]))

    def mask(self) -> np.ndarray:
        m = np.zeros(self.N, np.uint8)
        self._chk(self._L.polar_code_mask(self._h, m.ctypes.data))
        return m

    def schedule(self) -> list[str]:
        need = C.c_uint32()
        self._chk(self._L.polar_code_schedule(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        self._chk(self._L.polar_code_schedule(self._h, buf, need.value, None))
        return [s for s in buf.value.decode().split(";") if s]

    # ----------------------------------------------------------------- hot path
    # The C ABI takes raw pointers and cannot see a tensor's dtype, device, layout or size, so
    # the binding checks them (a strided slice or a wrong dtype would make the kernels read or
    # write past the buffers).
    def _frames(self, llr, dtype, on_cuda: bool) -> int:
        import torch
        if isinstance(llr, np.ndarray) and not on_cuda:  # host buffers may be numpy arrays
            if llr.dtype != np.dtype(str(dtype).replace("torch.", "")) or not llr.flags.c_contiguous:
                raise ValueError(f"llr must be a contiguous {dtype} array")
            llr = torch.from_numpy(llr)
        if not isinstance(llr, torch.Tensor):
            raise ValueError("llr must be a torch tensor")
        if llr.dtype != dtype:
            raise ValueError(f"llr must be {dtype}, got {llr.dtype}")
        if llr.is_cuda != on_cuda:
            raise ValueError(f"llr must be a {'CUDA' if on_cuda else 'host'} tensor")
        if not llr.is_contiguous():
            raise ValueError("llr must be contiguous")
        if llr.dim() == 2:
            if llr.shape[1] != self.N:
                raise ValueError(f"llr must be [n, {self.N}], got {tuple(llr.shape)}")
            return llr.shape[0]
        if llr.dim() == 1 and llr.numel() % self.N == 0:
            return llr.numel() // self.N
        raise ValueError(f"llr must be [n, {self.N}] (or a flat multiple of N), got {tuple(llr.shape)}")

    def _out(self, n: int, out, device):
        import torch
        if isinstance(out, np.ndarray) and device.type == "cpu":
            if out.dtype not in (np.uint32, np.int32) or not out.flags.c_contiguous or out.size < n * self.info_words:
                raise ValueError(f"out must be a contiguous 32-bit array of [n={n}, {self.info_words}] words")
            return out
        if out is None:
            return torch.empty((n, self.info_words), dtype=torch.int32, device=device)
        if not isinstance(out, torch.Tensor) or out.dtype != torch.int32 or not out.is_contiguous():
            raise ValueError("out must be a contiguous int32 tensor")
        if out.device != device:
            raise ValueError(f"out must be on {device}, got {out.device}")
        if out.numel() < n * self.info_words:
            raise ValueError(f"out must hold [n={n}, {self.info_words}] words, got {tuple(out.shape)}")
        return out

    def decode_f32(self, llr, out=None, stream=None):
        """Fast-SSC decode of float32 LLRs [n, N] (device) -> packed info bits [n, ceil(K/32)]."""
        import torch
        n = self._frames(llr, torch.float32, True)
        out = self._out(n, out, llr.device)
        self._chk(self._L.polar_decode_f32(self._h, _ptr(llr), n, _ptr(out), _stream(stream)))
        return out

    def decode_i8(self, llr, out=None, stream=None):
        """Fast-SSC decode of int8 LLRs [n, N] (device) -> packed info bits [n, ceil(K/32)]."""
        import torch
        n = self._frames(llr, torch.int8, True)
        out = self._out(n, out, llr.device)
        self._chk(self._L.polar_decode_i8(self._h, _ptr(llr), n, _ptr(out), _stream(stream)))
        return out

    def decode_host(self, llr, out):
        """End-to-end decode of HOST LLRs (float32 or int8 [n, N]) into HOST out [n, words]."""
        import torch
        is_i8 = str(llr.dtype).endswith("int8")
        n = self._frames(llr, torch.int8 if is_i8 else torch.float32, False)
        self._out(n, out, torch.device("cpu"))
        fn = self._L.polar_decode_i8_host if is_i8 else self._L.polar_decode_f32_host
        self._chk(fn(self._h, _ptr(llr), n, _ptr(out)))
        return out

    # ------------------------------------------------------------ batch-1 mailbox (N3)
    def mailbox_open(self, idle_seconds: float = 30.0) -> None:
        """Start the persistent batch-1 decoder (polar_mailbox_open): one SM, until mailbox_close."""
        self._chk(self._L.polar_mailbox_open(self._h, float(idle_seconds)))

    def mailbox_decode_i8(self, llr, out, timeout_seconds: float = 1.0):
        """One frame: host int8 LLRs [N] (numpy or CPU tensor) -> host packed info bits [words]."""
        self._chk(self._L.polar_mailbox_decode_i8(self._h, _ptr(llr), _ptr(out), float(timeout_seconds)))
        return out

    def mailbox_close(self) -> None:
        self._chk(self._L.polar_mailbox_close(self._h))

    # ----------------------------------------------------------------- non-hot helpers
    def encode_systematic(self, info, out=None, stream=None):
        import torch
        n = info.shape[0]
        if out is None:
            out = torch.empty((n, max(1, self.N // 32)), dtype=torch.int32, device=info.device)
        self._chk(self._L.polar_encode_systematic(self._h, _ptr(info), n, _ptr(out), _stream(stream)))
        return out

    def gen_bpsk_awgn(self, seed: int, first_frame: int, n: int, ebn0_db: float, q_scale: float = 4.0,
                      llr_f32=None, llr_i8=None, info=None, stream=None):
        self._chk(self._L.polar_gen_bpsk_awgn(self._h, seed, first_frame, n, float(ebn0_db), float(q_scale),
                                         _ptr(llr_f32), _ptr(llr_i8), _ptr(info), _stream(stream)))

    def trace(self, n: int) -> np.ndarray:
        """clock64 stamps of the latency variant's last frame (POLAR_TRACE builds only)."""
        out = np.zeros(n, np.uint64)
        self._chk(self._L.polar_trace_fetch(self._h, out.ctypes.data, n))
        return out

    def count_errors(self, decoded, truth, counters, stream=None):
        n = decoded.shape[0]
        self._chk(self._L.polar_count_errors(self._h, _ptr(decoded), _ptr(truth), n, _ptr(counters), _stream(stream)))
