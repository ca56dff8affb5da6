"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end of the CPU oracle
(oracle/vocab_oracle.cpp, a restatement of /root/reference/proj/src/vocab_math.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module; the product path never does.
All matrices are row-major float64 numpy arrays; ids are int64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_LIB = None
_D = POINTER(c_double)
_F = POINTER(c_float)
_I = POINTER(c_int64)


def load():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    lib = ctypes.CDLL(LIB_PATH)
    lib.or_last_error.restype = c_char_p
    lib.or_num_threads.restype = c_int
    lib.or_set_num_threads.argtypes = [c_int]
    lib.or_random_instance.argtypes = [c_int64, c_int64, c_int64, c_uint64, _D, _D, _I]
    lib.or_oracle_output_layer.argtypes = [_D, _D, _I, c_int64, c_int64, c_int64, _D, _D, _D, _D, _D]
    lib.or_run.argtypes = [c_int, _D, _D, _I, c_int64, c_int64, c_int64, c_int, c_double, _D, _D, _D, _D]
    lib.or_local_stats.argtypes = [_D, _D, c_int64, c_int64, c_int64, c_int, c_int, _D, _D]
    lib.or_merge_max_sum.argtypes = [_D, _D, c_int, c_int64, _D, _D]
    lib.or_shard_check.argtypes = [c_int64, c_int]
    lib.or_input_forward.argtypes = [_I, c_int64, _D, c_int64, c_int64, c_int64, _D]
    lib.or_input_backward.argtypes = [_D, _I, c_int64, c_int64, c_int64, c_int64, _D]
    lib.or_input_backward_f32.argtypes = [_F, _I, c_int64, c_int64, c_int64, c_int64, _F, c_int]
    for name in ("or_oracle_output_layer", "or_run", "or_local_stats", "or_merge_max_sum", "or_shard_check",
                 "or_input_forward", "or_input_backward", "or_input_backward_f32"):
        getattr(lib, name).restype = c_int
    _LIB = lib
    return lib


class OracleError(ValueError):
    """std::invalid_argument raised by the restated reference."""


def _chk(rc):
    if rc == 0:
        return
    msg = (load().or_last_error() or b"").decode()
    if rc == 1:
        raise OracleError(msg)
    raise RuntimeError(msg)


def _d(a):
    return None if a is None else a.ctypes.data_as(_D)


def _i(a):
    return a.ctypes.data_as(_I)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    load().or_set_num_threads(int(n))


def num_threads() -> int:
    return int(load().or_num_threads())


def random_instance(n_tok: int, h: int, V: int, seed: int):
    """VM.cpp:253-270, bit-exact.  Returns (X [n,h], W [V,h], labels [n])."""
    X = np.empty((n_tok, h), np.float64)
    W = np.empty((V, h), np.float64)
    g = np.empty(n_tok, np.int64)
    load().or_random_instance(n_tok, h, V, seed, _d(X), _d(W), _i(g))
    return X, W, g


class Result:
    def __init__(self, softmax, loss, grad_x, grad_w):
        self.softmax, self.loss, self.grad_x, self.grad_w = softmax, loss, grad_x, grad_w


def oracle_output_layer(X, labels, W, logit_shift=None, want_softmax=True) -> Result:
    """VM.cpp:31-63."""
    X, W = _c64(X), _c64(W)
    labels = np.ascontiguousarray(labels, np.int64)
    n, h = X.shape
    V = W.shape[0]
    if W.shape[1] != h:  # VM.cpp:35-37 (the C entry takes one h for both)
        raise OracleError("oracle_output_layer: X/W hidden dim mismatch")
    sm = np.empty((n, V)) if want_softmax else None
    loss, gx, gw = np.empty(n), np.empty((n, h)), np.empty((V, h))
    shift = None if logit_shift is None else _c64(logit_shift)
    _chk(load().or_oracle_output_layer(_d(X), _d(W), _i(labels), n, h, V, _d(shift), _d(sm), _d(loss), _d(gx),
                                       _d(gw)))
    return Result(sm, loss, gx, gw)


def run(alg: str, X, labels, W, p: int, fault_scale: float = 1.0, want_softmax: bool = True) -> Result:
    """run_naive / run_alg1 / run_alg2 (VM.cpp:299-361)."""
    code = {"naive": 0, "alg1": 1, "alg2": 2}[alg]
    X, W = _c64(X), _c64(W)
    labels = np.ascontiguousarray(labels, np.int64)
    n, h = X.shape
    V = W.shape[0]
    sm = np.empty((n, V)) if (want_softmax or code == 0) else None
    loss, gx, gw = np.empty(n), np.empty((n, h)), np.empty((V, h))
    _chk(load().or_run(code, _d(X), _d(W), _i(labels), n, h, V, p, float(fault_scale), _d(sm), _d(loss), _d(gx),
                       _d(gw)))
    return Result(sm, loss, gx, gw)


def local_stats(X, W, p: int, k: int):
    """alg1_pass_S m_local / sum_local of shard k (VM.cpp:157-159)."""
    X, W = _c64(X), _c64(W)
    n, h = X.shape
    m, s = np.empty(n), np.empty(n)
    _chk(load().or_local_stats(_d(X), _d(W), n, h, W.shape[0], p, k, _d(m), _d(s)))
    return m, s


def merge_max_sum(ms, ss):
    """VM.cpp:82-101 over lists of per-part vectors."""
    p = len(ms)
    if p == 0:
        _chk(load().or_merge_max_sum(None, None, 0, 0, None, None))
    n = len(ms[0])
    if any(len(x) != n for x in list(ms) + list(ss)):
        raise OracleError("merge_max_sum: length mismatch")
    M, S = _c64(np.stack(ms)), _c64(np.stack(ss))
    m, s = np.empty(n), np.empty(n)
    _chk(load().or_merge_max_sum(_d(M), _d(S), p, n, _d(m), _d(s)))
    return m, s


def shard_check(V: int, p: int) -> None:
    _chk(load().or_shard_check(V, p))


def input_forward(tokens, Wk, row_begin: int):
    """VM.cpp:227-236 for one shard."""
    tokens = np.ascontiguousarray(tokens, np.int64)
    Wk = _c64(Wk)
    out = np.empty((len(tokens), Wk.shape[1]))
    _chk(load().or_input_forward(_i(tokens), len(tokens), _d(Wk), Wk.shape[0], Wk.shape[1], row_begin, _d(out)))
    return out


def input_backward(grad, tokens, rows: int, row_begin: int):
    """VM.cpp:238-251 for one shard (fp64)."""
    tokens = np.ascontiguousarray(tokens, np.int64)
    grad = _c64(grad)
    out = np.empty((rows, grad.shape[1]))
    _chk(load().or_input_backward(_d(grad), _i(tokens), len(tokens), grad.shape[1], rows, row_begin, _d(out)))
    return out


def input_backward_f32(grad, tokens, rows: int, row_begin: int, init=None):
    """Same scatter-add in fp32, ascending i — the bit-exact GPU target."""
    tokens = np.ascontiguousarray(tokens, np.int64)
    grad = np.ascontiguousarray(grad, np.float32)
    out = np.zeros((rows, grad.shape[1]), np.float32) if init is None else np.array(init, np.float32, copy=True)
    _chk(load().or_input_backward_f32(grad.ctypes.data_as(_F), _i(tokens), len(tokens), grad.shape[1], rows,
                                      row_begin, out.ctypes.data_as(_F), int(init is not None)))
    return out
