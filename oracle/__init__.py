"""fp64 CPU oracle for GLA (arXiv 2312.06635): the paper's recurrent form + hand backward.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The CUDA product path
(``paper_2312_06635_b200``) never imports it and shares no code with it.

What it computes (see ``gla_oracle.c`` for the passage-by-passage citations):
  * ``fwd``  -- S_t = diag(alpha_t) S_{t-1} + k_t^T v_t, o_t = q_t S_t   (beta == 1 per P:321)
  * ``bwd``  -- reverse-mode of the same recurrence (the paper gives none),
               pinned by central finite differences in tests/test_oracle.py
  * ``step`` -- one recurrence step (decode)
  * ``fwd_beta`` / ``bwd_beta`` / ``step_beta`` -- the same with the general outer-product gate
               G_t = alpha_t^T beta_t (``gla_beta_oracle.c``), gradients including d log beta

Parity pins (tests/test_oracle.py, all ``-m "not gpu"``): quadratic parallel / semiring form
(P:224-231), alpha == 1 -> (QK^T (.) M)V, alpha == gamma -> RetNet D-mask,
hand-evaluated scalar cases (tests/golden/), causality, finite differences, closed-form invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gla_oracle.c")
_SRC_BETA = os.path.join(_HERE, "gla_beta_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99 + pthreads, -O2, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_SRC_BETA))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC, _SRC_BETA,
                               "-lm", "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i = ctypes.c_int
        lib.oracle_fwd.argtypes = [i, i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, i]
        lib.oracle_bwd.argtypes = [i, i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                   _dp, _dp, _dp, _dp, _dp, i]
        lib.oracle_step.argtypes = [i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_fwd_beta.argtypes = [i, i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, i]
        lib.oracle_bwd_beta.argtypes = [i, i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                        _dp, _dp, _dp, _dp, _dp, _dp, i]
        lib.oracle_step_beta.argtypes = [i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        for f in (lib.oracle_fwd, lib.oracle_bwd, lib.oracle_step, lib.oracle_fwd_beta, lib.oracle_bwd_beta,
                  lib.oracle_step_beta):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _d(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _threads(n):
    return n if n else (os.cpu_count() or 1)


def fwd(q, k, v, log_alpha, h0=None, nthreads=0):
    """o [B,H,T,V], final_state [B,H,K,V] in fp64.  Inputs [B,H,T,K|V] (any float dtype)."""
    q, k, v, g = _d(q), _d(k), _d(v), _d(log_alpha)
    B, H, T, K = q.shape
    V = v.shape[-1]
    h0 = None if h0 is None else _d(h0)
    o = np.empty((B, H, T, V))
    fs = np.empty((B, H, K, V))
    rc = _load().oracle_fwd(B, H, T, K, V, _p(q), _p(k), _p(v), _p(g), _p(h0), _p(o), _p(fs),
                            _threads(nthreads))
    if rc:
        raise RuntimeError(f"oracle_fwd failed ({rc})")
    return o, fs


def bwd(q, k, v, log_alpha, d_out, h0=None, d_final=None, nthreads=0):
    """(dq, dk, dv, dlog_alpha, dh0) in fp64 for loss = <o, d_out> + <final_state, d_final>."""
    q, k, v, g, do = _d(q), _d(k), _d(v), _d(log_alpha), _d(d_out)
    B, H, T, K = q.shape
    V = v.shape[-1]
    h0 = None if h0 is None else _d(h0)
    d_final = None if d_final is None else _d(d_final)
    dq, dk, dg = (np.empty((B, H, T, K)) for _ in range(3))
    dv = np.empty((B, H, T, V))
    dh0 = np.empty((B, H, K, V))
    rc = _load().oracle_bwd(B, H, T, K, V, _p(q), _p(k), _p(v), _p(g), _p(h0), _p(do), _p(d_final),
                            _p(dq), _p(dk), _p(dv), _p(dg), _p(dh0), _threads(nthreads))
    if rc:
        raise RuntimeError(f"oracle_bwd failed ({rc})")
    return dq, dk, dv, dg, dh0


def step(q, k, v, log_alpha, state):
    """One decode step.  q,k,log_alpha [B,H,K]; v [B,H,V]; state [B,H,K,V] (updated copy returned)."""
    q, k, v, g = _d(q), _d(k), _d(v), _d(log_alpha)
    B, H, K = q.shape
    V = v.shape[-1]
    st = _d(state).copy()
    o = np.empty((B, H, V))
    rc = _load().oracle_step(B, H, K, V, _p(q), _p(k), _p(v), _p(g), _p(st), _p(o))
    if rc:
        raise RuntimeError(f"oracle_step failed ({rc})")
    return o, st


def fwd_beta(q, k, v, log_alpha, log_beta, h0=None, nthreads=0):
    """General gate G_t = alpha_t^T beta_t: o [B,H,T,V], final_state [B,H,K,V] in fp64.
    log_beta [B,H,T,V]."""
    q, k, v, g, gb = _d(q), _d(k), _d(v), _d(log_alpha), _d(log_beta)
    B, H, T, K = q.shape
    V = v.shape[-1]
    h0 = None if h0 is None else _d(h0)
    o = np.empty((B, H, T, V))
    fs = np.empty((B, H, K, V))
    rc = _load().oracle_fwd_beta(B, H, T, K, V, _p(q), _p(k), _p(v), _p(g), _p(gb), _p(h0), _p(o), _p(fs),
                                 _threads(nthreads))
    if rc:
        raise RuntimeError(f"oracle_fwd_beta failed ({rc})")
    return o, fs


def bwd_beta(q, k, v, log_alpha, log_beta, d_out, h0=None, d_final=None, nthreads=0):
    """(dq, dk, dv, dlog_alpha, dlog_beta, dh0) in fp64 for loss = <o, d_out> + <final_state, d_final>, general
    gate G_t = alpha_t^T beta_t."""
    q, k, v, g, gb, do = _d(q), _d(k), _d(v), _d(log_alpha), _d(log_beta), _d(d_out)
    B, H, T, K = q.shape
    V = v.shape[-1]
    h0 = None if h0 is None else _d(h0)
    d_final = None if d_final is None else _d(d_final)
    dq, dk, dga = (np.empty((B, H, T, K)) for _ in range(3))
    dv, dgb = np.empty((B, H, T, V)), np.empty((B, H, T, V))
    dh0 = np.empty((B, H, K, V))
    rc = _load().oracle_bwd_beta(B, H, T, K, V, _p(q), _p(k), _p(v), _p(g), _p(gb), _p(h0), _p(do), _p(d_final),
                                 _p(dq), _p(dk), _p(dv), _p(dga), _p(dgb), _p(dh0), _threads(nthreads))
    if rc:
        raise RuntimeError(f"oracle_bwd_beta failed ({rc})")
    return dq, dk, dv, dga, dgb, dh0


def step_beta(q, k, v, log_alpha, log_beta, state):
    """One decode step with both gates.  q,k,log_alpha [B,H,K]; v, log_beta [B,H,V]; state [B,H,K,V]."""
    q, k, v, g, gb = _d(q), _d(k), _d(v), _d(log_alpha), _d(log_beta)
    B, H, K = q.shape
    V = v.shape[-1]
    st = _d(state).copy()
    o = np.empty((B, H, V))
    rc = _load().oracle_step_beta(B, H, K, V, _p(q), _p(k), _p(v), _p(g), _p(gb), _p(st), _p(o))
    if rc:
        raise RuntimeError(f"oracle_step_beta failed ({rc})")
    return o, st
