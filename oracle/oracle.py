"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/_build/liboracle_adamw.so.

Callers allowed: tests/, __graft_entry__.smoke(), bench.py (cpu_baseline and
--impl reference). The product never imports this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_BUILD = Path(__file__).resolve().parent / "_build"


def _has_avx512() -> bool:
    try:
        return " avx512f " in (" " + open("/proc/cpuinfo").read().replace("\n", " ") + " ")
    except OSError:
        return False


_SO = _BUILD / ("liboracle_adamw_avx512.so" if _has_avx512() and (_BUILD / "liboracle_adamw_avx512.so").exists()
                else "liboracle_adamw.so")
BF16, FP16, FP32 = 0, 1, 2


class Scalars(C.Structure):
    _fields_ = [(k, C.c_float) for k in (
        "beta1", "beta2", "one_minus_beta1", "one_minus_beta2", "bias_correction1",
        "bias_correction2", "step_size", "w_decay", "eps", "weight_decay")] + [("adamw_mode", C.c_int)]


class Counter(C.Structure):
    _fields_ = [("step", C.c_uint64), ("beta1", C.c_float), ("beta2", C.c_float),
                ("beta1_t", C.c_float), ("beta2_t", C.c_float)]


def _load():
    if not _SO.exists():
        raise ImportError(f"{_SO} missing; run `make -C oracle`")
    lib = C.CDLL(str(_SO))
    lib.oracle_adamw_scalars.argtypes = [C.c_float] * 5 + [C.c_uint64, C.c_int, C.c_int,
                                                           C.POINTER(Scalars)]
    lib.oracle_adamw_scalars.restype = None
    vp = C.c_void_p
    lib.oracle_adamw_scalars_bt.argtypes = [C.c_float] * 7 + [C.c_int, C.c_int, C.POINTER(Scalars)]
    lib.oracle_adamw_scalars_bt.restype = None
    lib.oracle_counter_init.argtypes = [C.POINTER(Counter), C.c_float, C.c_float]
    lib.oracle_counter_init.restype = None
    lib.oracle_counter_increment.argtypes = [C.POINTER(Counter), C.c_uint64, C.c_float, C.c_float,
                                             C.POINTER(C.c_float), C.POINTER(C.c_float)]
    lib.oracle_counter_increment.restype = None
    lib.oracle_adamw_step.argtypes = [vp, vp, vp, vp, C.c_int, vp, C.c_int, C.c_uint64,
                                      C.POINTER(Scalars), C.c_float, C.POINTER(C.c_double),
                                      C.POINTER(C.c_int)]
    lib.oracle_adamw_step.restype = None
    lib.oracle_adamw_step_omp.argtypes = [vp, vp, vp, vp, C.c_int, vp, C.c_int, C.c_uint64,
                                          C.POINTER(Scalars), C.c_float, C.c_int]
    lib.oracle_adamw_step_omp.restype = None
    lib.oracle_max_threads.restype = C.c_int
    lib.oracle_first_touch.argtypes = [vp, C.c_uint64, C.c_float, C.c_int]
    lib.oracle_fill_s8d.argtypes = [vp, C.c_uint64, C.c_int, C.c_uint64, C.c_int]
    lib.oracle_fill_s8d.restype = None
    lib.oracle_float_to_bf16.argtypes = [C.c_float]
    lib.oracle_float_to_bf16.restype = C.c_uint16
    lib.oracle_float_to_fp16.argtypes = [C.c_float]
    lib.oracle_float_to_fp16.restype = C.c_uint16
    lib.oracle_bf16_to_float.argtypes = [C.c_uint16]
    lib.oracle_bf16_to_float.restype = C.c_float
    lib.oracle_fp16_to_float.argtypes = [C.c_uint16]
    lib.oracle_fp16_to_float.restype = C.c_float
    return lib


LIB = _load()


def scalars(lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, step=10,
            adamw_mode=True, bias_correction=True) -> Scalars:
    s = Scalars()
    LIB.oracle_adamw_scalars(lr, beta1, beta2, eps, weight_decay, step, int(adamw_mode),
                             int(bias_correction), C.byref(s))
    return s


def scalars_bt(b1t: float, b2t: float, lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8,
               weight_decay=0.1, adamw_mode=True, bias_correction=True) -> Scalars:
    """update_state with explicit float beta1^t / beta2^t (a StepCounter's)."""
    s = Scalars()
    LIB.oracle_adamw_scalars_bt(lr, beta1, beta2, eps, weight_decay, b1t, b2t, int(adamw_mode),
                                int(bias_correction), C.byref(s))
    return s


class StepCounter:
    """DeepSpeed 0.9.3 Adam_Optimizer IncrementStep (oracle_counter_increment):
    call next() once per adam_update, i.e. once per chunk."""

    def __init__(self, beta1: float = 0.9, beta2: float = 0.95):
        self.c = Counter()
        LIB.oracle_counter_init(C.byref(self.c), beta1, beta2)

    def next(self, step: int, beta1: float = 0.9, beta2: float = 0.95):
        b1t, b2t = C.c_float(), C.c_float()
        LIB.oracle_counter_increment(C.byref(self.c), step, beta1, beta2, C.byref(b1t), C.byref(b2t))
        return b1t.value, b2t.value


def _p(a):
    return None if a is None else a.ctypes.data


def adamw_step(master: np.ndarray, m: np.ndarray, v: np.ndarray, grad: np.ndarray,
               grad_dtype: int, s: Scalars, grad_scale: float = 1.0, param_out=None,
               param_dtype: int = BF16):
    """In-place scalar oracle step on numpy arrays; grads/params as uint16 bit
    patterns for bf16/fp16 (float32 for FP32). Returns (grad_sq_sum, nonfinite)."""
    for a in (master, m, v):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    sq = C.c_double()
    bad = C.c_int(0)
    LIB.oracle_adamw_step(_p(master), _p(m), _p(v), _p(grad), grad_dtype, _p(param_out),
                          param_dtype, master.size, C.byref(s), grad_scale, C.byref(sq),
                          C.byref(bad))
    return sq.value, bad.value


def adamw_step_omp(master, m, v, grad, grad_dtype, s, grad_scale=1.0, param_out=None,
                   param_dtype=BF16, threads=0):
    LIB.oracle_adamw_step_omp(_p(master), _p(m), _p(v), _p(grad), grad_dtype, _p(param_out),
                              param_dtype, master.size, C.byref(s), grad_scale, threads)


def fill_s8d(master, m, v, grad_bits, seed: int = 20240817, threads: int = 0) -> None:
    """Parallel first-touch fill with SURVEY §8d's distributions (timing
    samples for the CPU baseline; see oracle_fill_s8d)."""
    for kind, a in enumerate((master, m, v, grad_bits)):
        LIB.oracle_fill_s8d(_p(a), a.size, kind, seed, threads)


def max_threads() -> int:
    return int(LIB.oracle_max_threads())


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    f = np.vectorize(LIB.oracle_float_to_bf16, otypes=[np.uint16])
    return f(x.astype(np.float32))


def f32_to_fp16_bits(x: np.ndarray) -> np.ndarray:
    f = np.vectorize(LIB.oracle_float_to_fp16, otypes=[np.uint16])
    return f(x.astype(np.float32))
