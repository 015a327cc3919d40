"""B200-native certified interval-FFT multiplication (arXiv 1006.0405).

Thin ctypes binding over ``libivm.so`` (include/ivm.h).  Argument marshalling
only: every step of the multiply runs in the library's sm_100a kernels.
PyTorch provides device memory and streams.  There is no CPU fallback: if the
library is missing or no device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["lib", "Context", "IvmError", "F64", "F32", "fft_length", "max_digits",
           "twiddle_table", "EXPORTS"]

F64, F32 = 0, 1
_HERE = os.path.dirname(os.path.abspath(__file__))
# IVM_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("IVM_LIB") or os.path.join(_HERE, "libivm.so")

# every symbol include/ivm.h declares
EXPORTS = ["ivm_version", "ivm_strerror", "ivm_max_digits", "ivm_fft_length", "ivm_create",
           "ivm_destroy", "ivm_reserve", "ivm_multiply", "ivm_multiply_batched",
           "ivm_multiply_batched_diag", "ivm_multiply_batched_host", "ivm_generate_digits",
           "ivm_peak_probe", "ivm_last_launch_count", "ivm_twiddle_table", "ivm_long_multiply_batched",
           "ivm_multiply_exact", "ivm_multiply_naive", "ivm_multiply_disc", "ivm_multi_create",
           "ivm_multi_multiply", "ivm_multi_summary", "ivm_multi_destroy"]


class IvmError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = lib().ivm_strerror(status).decode() if _lib is not None else str(status)
        super().__init__(f"{what}: {msg} ({status})")
        self.status = status


_lib = None


def lib():
    """Load libivm.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1006_0405_b200.build` "
                              "(there is no fallback implementation)")
        L = ctypes.CDLL(LIB_PATH)
        P, S, I, U64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
        sig = {
            "ivm_version": (None, ctypes.c_char_p), "ivm_strerror": ([I], ctypes.c_char_p),
            "ivm_max_digits": ([I], S), "ivm_fft_length": ([S], S),
            "ivm_create": ([ctypes.POINTER(P), I], None), "ivm_destroy": ([P], None),
            "ivm_reserve": ([P, S, S, I], None), "ivm_multiply": ([P, P, P, S, P, P, I, P], None),
            "ivm_multiply_batched": ([P, P, P, S, S, P, P, I, P], None),
            "ivm_multiply_batched_diag": ([P, P, P, S, S, P, P, I, P, P, P, P, P, S, P], None),
            "ivm_multiply_batched_host": ([P, P, P, S, S, P, P, I, P], None),
            "ivm_generate_digits": ([P, P, S, S, U64, U64, I, I, P, P], None),
            "ivm_peak_probe": ([P, I, I, P, ctypes.POINTER(U64), P], None),
            "ivm_last_launch_count": ([P], None), "ivm_twiddle_table": ([I, I, P], None),
            "ivm_long_multiply_batched": ([P, P, P, S, S, P, P], None),
            "ivm_multiply_exact": ([P, P, P, S, S, P, P, I, P], None),
            "ivm_multiply_naive": ([P, P, P, S, S, P, I, P], None),
            "ivm_multiply_disc": ([P, P, P, S, S, P, P, P, P], None),
            "ivm_multi_create": ([ctypes.POINTER(P), I, P], None),
            "ivm_multi_multiply": ([P, P, P, S, S, P, P, I, I, P, P], None),
            "ivm_multi_summary": ([P, P, P, S, P, P], None),
            "ivm_multi_destroy": ([P], None),
        }
        # (an older build missing a symbol fails at that call, not at load:
        # tests/test_abi.py checks that this build exports every declared one)
        for name, (args, res) in sig.items():
            if hasattr(L, name):
                f = getattr(L, name)
                if args is not None:
                    f.argtypes = args
                if res is not None:
                    f.restype = res
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise IvmError(status, what)


def fft_length(n: int) -> int:
    return int(lib().ivm_fft_length(n))


def max_digits(prec: int = F64) -> int:
    return int(lib().ivm_max_digits(prec))


def twiddle_table(log2m: int, prec: int = F64):
    """The library's optimal twiddle enclosures, [m][4] (host, numpy)."""
    import numpy as np
    m = 1 << log2m
    out = np.zeros((m, 4), np.float64 if prec == F64 else np.float32)
    _check(lib().ivm_twiddle_table(log2m, prec, out.ctypes.data), "ivm_twiddle_table")
    return out


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_operands(a, b, on_device: bool, device: int | None = None):
    """Every wrapper's operand check: uint8, same shape [batch][n] (or [n]),
    contiguous, and on the context's CUDA device (on_device) or in host memory
    (the host entry point).  The C ABI reads a and b as dense [batch][n] rows,
    so anything else would multiply the wrong digits."""
    import torch
    for name, t in (("a", a), ("b", b)):
        if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8:
            raise TypeError(f"{name} must be a torch.uint8 tensor")
        if t.dim() not in (1, 2) or t.numel() == 0:
            raise ValueError(f"{name} must be a non-empty [batch][n] (or [n]) tensor")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous (row-major [batch][n])")
        if on_device:
            if not t.is_cuda or (device is not None and t.device.index != device):
                raise ValueError(f"{name} must be a CUDA tensor on cuda:{device}")
        elif t.is_cuda:
            raise ValueError(f"{name} must be a host tensor for the host entry point")
    if a.shape != b.shape:
        raise ValueError(f"operand shapes differ: {tuple(a.shape)} vs {tuple(b.shape)} "
                         "(zero-pad the shorter operand)")


def _check_out(t, shape, dtype, on_device: bool, name: str):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must be a {dtype} tensor of shape {tuple(shape)}")
    if not t.is_contiguous() or t.is_cuda != on_device:
        raise ValueError(f"{name} must be contiguous and {'on the device' if on_device else 'in host memory'}")


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Context:
    """One device context (twiddle tables + scratch).  Tensors are torch CUDA
    tensors on the context's device; results are valid after the stream syncs."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        _check(lib().ivm_create(ctypes.byref(h), device), "ivm_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().ivm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reserve(self, n: int, batch: int, prec: int = F64):
        _check(lib().ivm_reserve(self._h, n, batch, prec), "ivm_reserve")

    @property
    def last_launch_count(self) -> int:
        return int(lib().ivm_last_launch_count(self._h))

    def multiply(self, a, b, prec: int = F64, out=None, cert=None, stream=None):
        """Batched multiply of uint8 CUDA tensors a, b [batch][n] (or [n])."""
        import torch
        _check_operands(a, b, True, self.device)
        squeeze = a.dim() == 1
        if squeeze:
            a, b = a[None], b[None]
        B, n = a.shape
        if out is None:
            out = torch.empty((B, 2 * n), dtype=torch.uint8, device=a.device)
        if cert is None:
            cert = torch.empty((B,), dtype=torch.uint8, device=a.device)
        _check_out(out, (B, 2 * n), torch.uint8, True, "out")
        _check_out(cert, (B,), torch.uint8, True, "cert")
        _check(lib().ivm_multiply_batched(self._h, _ptr(a), _ptr(b), n, B, _ptr(out), _ptr(cert),
                                          prec, _stream(stream)), "ivm_multiply_batched")
        if squeeze:
            return out[0], cert[0]
        return out, cert

    def multiply_diag(self, a, b, prec: int = F64, dump_pairs=None, stream=None, coeffs=True):
        """Multiply with diagnostics: returns dict of CUDA tensors."""
        import torch
        _check_operands(a, b, True, self.device)
        if a.dim() == 1:
            a, b = a[None], b[None]
        B, n = a.shape
        dev = a.device
        m = fft_length(n)
        out = torch.empty((B, 2 * n), dtype=torch.uint8, device=dev)
        cert = torch.empty((B,), dtype=torch.uint8, device=dev)
        rad = torch.empty((B,), dtype=torch.float64, device=dev)
        bad = torch.empty((B,), dtype=torch.int32, device=dev)
        co = torch.empty((B, 2 * n - 1), dtype=torch.int64, device=dev) if coeffs else None
        dp, iv, nd = None, None, 0
        if dump_pairs is not None and len(dump_pairs):
            dp = torch.as_tensor(list(dump_pairs), dtype=torch.int32, device=dev)
            nd = dp.numel()
            iv = torch.empty((nd, m, 4), dtype=torch.float64, device=dev)
        _check(lib().ivm_multiply_batched_diag(self._h, _ptr(a), _ptr(b), n, B, _ptr(out),
                                               _ptr(cert), prec, _stream(stream), _ptr(rad),
                                               _ptr(bad), _ptr(co), _ptr(dp), nd, _ptr(iv)),
               "ivm_multiply_batched_diag")
        return {"prod": out, "cert": cert, "max_radius": rad, "first_bad": bad, "coeffs": co,
                "intervals": iv, "m": m}

    def multiply_naive(self, a, b, prec: int = F64, out=None, stream=None):
        """The paper's naive (punctual, round-to-nearest) SS: [B][2n] u8,
        NOT guaranteed correct."""
        import torch
        _check_operands(a, b, True, self.device)
        if a.dim() == 1:
            a, b = a[None], b[None]
        B, n = a.shape
        if out is None:
            out = torch.empty((B, 2 * n), dtype=torch.uint8, device=a.device)
        _check_out(out, (B, 2 * n), torch.uint8, True, "out")
        _check(lib().ivm_multiply_naive(self._h, _ptr(a), _ptr(b), n, B, _ptr(out), prec, _stream(stream)),
               "ivm_multiply_naive")
        return out

    def multiply_disc(self, a, b, out=None, cert=None, want_radius: bool = True, stream=None):
        """Circular containment sets (R15), fp64, n <= max_digits():
        (products [B][2n] u8, certified [B] u8, max disc radius [B] f64 or None)."""
        import torch
        _check_operands(a, b, True, self.device)
        if a.dim() == 1:
            a, b = a[None], b[None]
        B, n = a.shape
        if out is None:
            out = torch.empty((B, 2 * n), dtype=torch.uint8, device=a.device)
        if cert is None:
            cert = torch.empty((B,), dtype=torch.uint8, device=a.device)
        _check_out(out, (B, 2 * n), torch.uint8, True, "out")
        _check_out(cert, (B,), torch.uint8, True, "cert")
        rad = torch.empty((B,), dtype=torch.float64, device=a.device) if want_radius else None
        _check(lib().ivm_multiply_disc(self._h, _ptr(a), _ptr(b), n, B, _ptr(out), _ptr(cert), _ptr(rad),
                                       _stream(stream)), "ivm_multiply_disc")
        return out, cert, rad

    def long_multiply(self, a, b, out=None, stream=None):
        """Exact long multiplication on the device: [B][2n] u8."""
        import torch
        _check_operands(a, b, True, self.device)
        if a.dim() == 1:
            a, b = a[None], b[None]
        B, n = a.shape
        if out is None:
            out = torch.empty((B, 2 * n), dtype=torch.uint8, device=a.device)
        _check_out(out, (B, 2 * n), torch.uint8, True, "out")
        _check(lib().ivm_long_multiply_batched(self._h, _ptr(a), _ptr(b), n, B, _ptr(out), _stream(stream)),
               "ivm_long_multiply_batched")
        return out

    def multiply_exact(self, a, b, out=None, method=None, policy: int = 0, stream=None):
        """Exact products with the fp32 -> fp64 -> long-multiplication
        escalation (policy 1: long multiplication directly below
        m = 64); returns (products [B][2n] u8, method [B] u8:
        1 fp32 interval, 2 fp64 interval, 3 long multiplication)."""
        import torch
        _check_operands(a, b, True, self.device)
        if a.dim() == 1:
            a, b = a[None], b[None]
        B, n = a.shape
        if out is None:
            out = torch.empty((B, 2 * n), dtype=torch.uint8, device=a.device)
        if method is None:
            method = torch.empty((B,), dtype=torch.uint8, device=a.device)
        _check_out(out, (B, 2 * n), torch.uint8, True, "out")
        _check_out(method, (B,), torch.uint8, True, "method")
        _check(lib().ivm_multiply_exact(self._h, _ptr(a), _ptr(b), n, B, _ptr(out), _ptr(method), policy,
                                        _stream(stream)), "ivm_multiply_exact")
        return out, method

    def multiply_host(self, a, b, prec: int = F64, out=None, cert=None, stream=None):
        """End-to-end path: host uint8 tensors in (pinned for asynchronous
        copies; pageable memory works but is copied synchronously), host
        tensors out."""
        import torch
        _check_operands(a, b, False)
        if a.dim() == 1:
            a, b = a[None], b[None]
        B, n = a.shape
        if out is None:
            out = torch.empty((B, 2 * n), dtype=torch.uint8, pin_memory=True)
        if cert is None:
            cert = torch.empty((B,), dtype=torch.uint8, pin_memory=True)
        _check_out(out, (B, 2 * n), torch.uint8, False, "out")
        _check_out(cert, (B,), torch.uint8, False, "cert")
        _check(lib().ivm_multiply_batched_host(self._h, _ptr(a), _ptr(b), n, B, _ptr(out),
                                               _ptr(cert), prec, _stream(stream)),
               "ivm_multiply_batched_host")
        return out, cert

    def generate_digits(self, n: int, batch: int, seed: int, operand: int, kind=0, pair0: int = 0,
                        out=None, stream=None):
        """Seeded digits on the device (same bits as inputs.py).  kind: int or
        uint8 CUDA tensor of per-pair kinds."""
        import torch
        if out is None:
            out = torch.empty((batch, n), dtype=torch.uint8, device=f"cuda:{self.device}")
        kinds = None
        k = 0
        if isinstance(kind, int):
            k = kind
        else:
            kinds = kind
        _check(lib().ivm_generate_digits(self._h, _ptr(out), n, batch, seed & (2**64 - 1), pair0,
                                         operand, k, _ptr(kinds), _stream(stream)),
               "ivm_generate_digits")
        return out

    def peak_probe(self, prec: int, iters: int, sink, stream=None) -> int:
        cnt = ctypes.c_uint64()
        _check(lib().ivm_peak_probe(self._h, prec, iters, _ptr(sink), ctypes.byref(cnt),
                                    _stream(stream)), "ivm_peak_probe")
        return int(cnt.value)
