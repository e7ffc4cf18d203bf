"""Thin Python binding over libgla.so (include/gla.h).  Argument marshalling only: every step of the
method runs in the library's CUDA kernels.  torch provides device memory and the current stream.

There is no CPU fallback: if libgla.so is missing or the tensors are not on a CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgla.so")

BF16, FP32 = 0, 1
PATHS = {"auto": 0, "simt": 1, "tc": 2}
_STATUS = {0: "ok", 1: "shape", 2: "plan", 3: "dtype", 4: "align", 5: "null", 6: "unsupported", 7: "cuda",
           8: "workspace"}


class GLAError(RuntimeError):
    def __init__(self, fn: str, status: int, lib):
        self.status = status
        msg = lib.gla_status_string(status).decode()
        if status == 7:
            msg += f" (cudaError {lib.gla_last_cuda_error()})"
        super().__init__(f"{fn}: {msg} [status {status}]")


class _Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("B", "H", "T", "K", "V", "chunk", "subchunk", "qkv_dtype", "gate_dtype", "path")]


_lib = None


def lib():
    """Load libgla.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libgla.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; "
                               f"g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, ip = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        dp = ctypes.POINTER(_Desc)
        L.gla_fwd_workspace_size.argtypes = [dp]
        L.gla_fwd_workspace_size.restype = sz
        L.gla_bwd_workspace_size.argtypes = [dp]
        L.gla_bwd_workspace_size.restype = sz
        L.gla_chunk_fwd.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.gla_chunk_bwd.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.gla_chunk_bwd_saved.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp]
        L.gla_recurrent_step.argtypes = [ip, ip, ip, ip, ip, ip, vp, vp, vp, vp, vp, vp, vp]
        L.gla_state_summary.argtypes = [dp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.gla_dstate_summary.argtypes = [dp, vp, vp, vp, vp, vp, sz, vp]
        L.gla_state_combine.argtypes = [ip, ip, ip, vp, vp, vp, vp, vp]
        L.gla_beta_workspace_size.argtypes = [dp]
        L.gla_beta_workspace_size.restype = sz
        L.gla_chunk_fwd_beta.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.gla_chunk_bwd_beta.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.gla_recurrent_step_beta.argtypes = [ip, ip, ip, ip, ip, ip, vp, vp, vp, vp, vp, vp, vp, vp]
        fl = ctypes.c_float
        L.gla_layer_bwd_workspace_size.argtypes = [ip, ip, ip, ip, ip]
        L.gla_layer_bwd_workspace_size.restype = sz
        L.gla_layer_prep.argtypes = [ip, ip, ip, ip, ip, fl, vp, ip, vp, vp, vp, vp, vp, vp, vp]
        L.gla_layer_out.argtypes = [ip, ip, ip, ip, vp, vp, ip, ip, vp, vp, vp, fl, vp, vp, vp, vp]
        L.gla_layer_out_bwd.argtypes = [ip, ip, ip, ip, vp, vp, vp, ip, ip, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                        vp, sz, vp]
        L.gla_layer_prep_bwd.argtypes = [ip, ip, ip, ip, ip, fl, vp, vp, vp, vp, vp, vp, vp, ip, vp, vp, vp, sz, vp]
        L.gla_status_string.argtypes = [ip]
        L.gla_status_string.restype = ctypes.c_char_p
        L.gla_resolve_path.argtypes = [dp]
        L.gla_profile_enable.argtypes = [ip]
        L.gla_profile_enable.restype = None
        L.gla_profile_reset.restype = None
        L.gla_profile_count.restype = ip
        L.gla_profile_get.argtypes = [ip, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ip)]
        L.gla_profile_get.restype = ip
        for f in (L.gla_chunk_fwd, L.gla_chunk_bwd, L.gla_recurrent_step, L.gla_state_summary,
                  L.gla_dstate_summary, L.gla_state_combine, L.gla_last_cuda_error, L.gla_version,
                  L.gla_resolve_path, L.gla_layer_prep, L.gla_layer_out, L.gla_layer_out_bwd, L.gla_layer_prep_bwd,
                  L.gla_chunk_fwd_beta, L.gla_chunk_bwd_beta, L.gla_recurrent_step_beta):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTS = ("gla_fwd_workspace_size", "gla_bwd_workspace_size", "gla_chunk_fwd", "gla_chunk_bwd", "gla_chunk_bwd_saved",
           "gla_recurrent_step", "gla_state_summary", "gla_dstate_summary", "gla_state_combine",
           "gla_status_string", "gla_last_cuda_error", "gla_resolve_path", "gla_version", "gla_profile_enable",
           "gla_profile_reset", "gla_profile_count", "gla_profile_get", "gla_layer_bwd_workspace_size",
           "gla_layer_prep", "gla_layer_out", "gla_layer_out_bwd", "gla_layer_prep_bwd", "gla_beta_workspace_size",
           "gla_chunk_fwd_beta", "gla_chunk_bwd_beta", "gla_recurrent_step_beta")


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return FP32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise RuntimeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise RuntimeError(f"{name} must be contiguous")


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _same_device(dev, named):
    for n, t in named:
        if t is not None and t.device != dev:
            raise RuntimeError(f"{n} is on {t.device}, expected {dev} (all tensors of one call share a device)")


def _shape(t, shape, name):
    if t is not None and tuple(t.shape) != tuple(shape):
        raise RuntimeError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _check_problem(q, k, v, log_alpha, d_out=None, initial_state=None, d_final_state=None, grads=None):
    """Shapes and devices of one call.  The C ABI receives only pointers and the descriptor built from q and v,
    so a mismatched tensor would make the kernels (and their TMA maps) read or write past its end: reject it
    here, before any launch."""
    if q.dim() != 4 or v.dim() != 4:
        raise RuntimeError(f"q and v must be [B,H,T,K] / [B,H,T,V] (got {tuple(q.shape)}, {tuple(v.shape)})")
    B, H, T, K = q.shape
    V = v.shape[-1]
    _shape(k, (B, H, T, K), "k")
    _shape(log_alpha, (B, H, T, K), "log_alpha")
    _shape(v, (B, H, T, V), "v")
    _shape(d_out, (B, H, T, V), "d_out")
    _shape(initial_state, (B, H, K, V), "initial_state")
    _shape(d_final_state, (B, H, K, V), "d_final_state")
    named = [("k", k), ("v", v), ("log_alpha", log_alpha), ("d_out", d_out), ("initial_state", initial_state),
             ("d_final_state", d_final_state)]
    if grads is not None:
        for n, t, shp in zip(("dq", "dk", "dv", "d_log_alpha", "d_initial_state"), grads,
                             ((B, H, T, K), (B, H, T, K), (B, H, T, V), (B, H, T, K), (B, H, K, V))):
            _shape(t, shp, n)
            named.append((n, t))
    for n, t in named:
        if t is not None:
            _check(t, n)
    for n, t in (("initial_state", initial_state), ("d_final_state", d_final_state)):
        if t is not None and t.dtype != torch.float32:
            raise RuntimeError(f"{n} must be fp32")
    _same_device(q.device, named)


def desc(q, v, log_alpha, chunk, subchunk, path) -> _Desc:
    B, H, T, K = q.shape
    return _Desc(B, H, T, K, v.shape[-1], chunk, subchunk, _dt(q), _dt(log_alpha), PATHS[path])


def resolve_path(q, v, log_alpha, chunk=64, subchunk=16, path="auto") -> str:
    r = lib().gla_resolve_path(ctypes.byref(desc(q, v, log_alpha, chunk, subchunk, path)))
    return {1: "simt", 2: "tc"}.get(r, f"error{r}")


def _call(fn, name, *args):
    s = fn(*args)
    if s != 0:
        raise GLAError(name, s, lib())


def fwd_workspace(q, v, log_alpha, chunk=64, subchunk=16, path="auto") -> torch.Tensor:
    n = lib().gla_fwd_workspace_size(ctypes.byref(desc(q, v, log_alpha, chunk, subchunk, path)))
    return torch.empty(max(n, 16), dtype=torch.uint8, device=q.device)


def bwd_workspace(q, v, log_alpha, chunk=64, subchunk=16, path="auto") -> torch.Tensor:
    n = lib().gla_bwd_workspace_size(ctypes.byref(desc(q, v, log_alpha, chunk, subchunk, path)))
    return torch.empty(max(n, 16), dtype=torch.uint8, device=q.device)


def chunk_fwd(q, k, v, log_alpha, chunk: int = 64, subchunk: int = 16, initial_state=None,
              output_final_state: bool = False, path: str = "auto", out=None, final_state=None, workspace=None):
    """o [B,H,T,V] (q's dtype) and final_state [B,H,K,V] fp32 (or None).  gla_chunk_fwd."""
    _check(q, "q")
    _check_problem(q, k, v, log_alpha, initial_state=initial_state)
    B, H, T, K = q.shape
    V = v.shape[-1]
    _shape(out, (B, H, T, V), "out")
    _shape(final_state, (B, H, K, V), "final_state")
    _same_device(q.device, [("out", out), ("final_state", final_state), ("workspace", workspace)])
    d = desc(q, v, log_alpha, chunk, subchunk, path)
    if out is None:
        out = torch.empty((B, H, T, V), dtype=q.dtype, device=q.device)
    if output_final_state and final_state is None:
        final_state = torch.empty((B, H, K, V), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = fwd_workspace(q, v, log_alpha, chunk, subchunk, path)
    with torch.cuda.device(q.device):
        _call(lib().gla_chunk_fwd, "gla_chunk_fwd", ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(log_alpha),
              _ptr(initial_state), _ptr(out), _ptr(final_state), _ptr(workspace), workspace.numel(),
              _stream(q.device))
    return out, final_state


def chunk_bwd(q, k, v, log_alpha, d_out, chunk: int = 64, subchunk: int = 16, initial_state=None,
              d_final_state=None, need_d_initial_state: bool = False, path: str = "auto", grads=None,
              workspace=None, fwd_workspace=None):
    """(dq, dk, dv, d_log_alpha fp32, d_initial_state fp32 or None).  gla_chunk_bwd, or gla_chunk_bwd_saved when
    ``fwd_workspace`` (the workspace a chunk_fwd call on the same q, k, log_alpha filled) is given."""
    _check(q, "q")
    _check_problem(q, k, v, log_alpha, d_out, initial_state, d_final_state, grads)
    B, H, T, K = q.shape
    d = desc(q, v, log_alpha, chunk, subchunk, path)
    if grads is None:
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        dg = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        dh0 = torch.empty((B, H, K, v.shape[-1]), dtype=torch.float32, device=q.device) \
            if need_d_initial_state else None
    else:
        dq, dk, dv, dg, dh0 = grads
    if workspace is None:
        workspace = bwd_workspace(q, v, log_alpha, chunk, subchunk, path)
    _same_device(q.device, [("workspace", workspace), ("fwd_workspace", fwd_workspace)])
    with torch.cuda.device(q.device):
        if fwd_workspace is not None:
            _check(fwd_workspace, "fwd_workspace")
            _call(lib().gla_chunk_bwd_saved, "gla_chunk_bwd_saved", ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v),
                  _ptr(log_alpha), _ptr(initial_state), _ptr(d_out), _ptr(d_final_state), _ptr(dq), _ptr(dk),
                  _ptr(dv), _ptr(dg), _ptr(dh0), _ptr(workspace), workspace.numel(), _ptr(fwd_workspace),
                  _stream(q.device))
            return dq, dk, dv, dg, dh0
        _call(lib().gla_chunk_bwd, "gla_chunk_bwd", ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(log_alpha),
              _ptr(initial_state), _ptr(d_out), _ptr(d_final_state), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dg),
              _ptr(dh0), _ptr(workspace), workspace.numel(), _stream(q.device))
    return dq, dk, dv, dg, dh0


def recurrent_step(q_t, k_t, v_t, log_alpha_t, state, out=None):
    """One decode step; ``state`` [B,H,K,V] fp32 is updated in place; returns o_t [B,H,V]."""
    for t, n in ((q_t, "q_t"), (k_t, "k_t"), (v_t, "v_t"), (log_alpha_t, "log_alpha_t"), (state, "state")):
        _check(t, n)
    B, H, K = q_t.shape
    V = v_t.shape[-1]
    _shape(k_t, (B, H, K), "k_t")
    _shape(log_alpha_t, (B, H, K), "log_alpha_t")
    _shape(v_t, (B, H, V), "v_t")
    _shape(state, (B, H, K, V), "state")
    if state.dtype != torch.float32:
        raise RuntimeError("state must be fp32")
    if out is None:
        out = torch.empty((B, H, V), dtype=q_t.dtype, device=q_t.device)
    _shape(out, (B, H, V), "out")
    _same_device(q_t.device, [("k_t", k_t), ("v_t", v_t), ("log_alpha_t", log_alpha_t), ("state", state),
                              ("out", out)])
    with torch.cuda.device(q_t.device):
        _call(lib().gla_recurrent_step, "gla_recurrent_step", B, H, K, V, _dt(q_t), _dt(log_alpha_t), _ptr(q_t),
              _ptr(k_t), _ptr(v_t), _ptr(log_alpha_t), _ptr(state), _ptr(out), _stream(q_t.device))
    return out


def state_summary(k, v, log_alpha, chunk: int = 64, subchunk: int = 16, path: str = "auto", workspace=None):
    """(S_loc [B,H,K,V] fp32, log_decay [B,H,K] fp32) of a segment with zero initial state (tensor cores when the
    descriptor resolves to the TC path; the workspace is then a forward workspace)."""
    _check(k, "k")
    _check_problem(k, k, v, log_alpha)
    B, H, T, K = k.shape
    V = v.shape[-1]
    d = desc(k, v, log_alpha, chunk, subchunk, path)
    S = torch.empty((B, H, K, V), dtype=torch.float32, device=k.device)
    D = torch.empty((B, H, K), dtype=torch.float32, device=k.device)
    if workspace is None:
        workspace = fwd_workspace(k, v, log_alpha, chunk, subchunk, path)
    with torch.cuda.device(k.device):
        _call(lib().gla_state_summary, "gla_state_summary", ctypes.byref(d), _ptr(k), _ptr(v), _ptr(log_alpha),
              _ptr(S), _ptr(D), _ptr(workspace), workspace.numel(), _stream(k.device))
    return S, D


def dstate_summary(q, d_out, log_alpha, chunk: int = 64, subchunk: int = 16, path: str = "auto", workspace=None):
    """dh0_loc [B,H,K,V] fp32 = d_initial_state of a segment when d_final_state = 0."""
    _check(q, "q")
    _check_problem(q, q, d_out, log_alpha)
    B, H, T, K = q.shape
    V = d_out.shape[-1]
    d = desc(q, d_out, log_alpha, chunk, subchunk, path)
    out = torch.empty((B, H, K, V), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = fwd_workspace(q, d_out, log_alpha, chunk, subchunk, path)
    with torch.cuda.device(q.device):
        _call(lib().gla_dstate_summary, "gla_dstate_summary", ctypes.byref(d), _ptr(q), _ptr(d_out),
              _ptr(log_alpha), _ptr(out), _ptr(workspace), workspace.numel(), _stream(q.device))
    return out


def state_combine(H_in, log_decay, S_loc, out=None):
    """H_out = diag(e^{log_decay}) H_in + S_loc (per (b,h) unit)."""
    B, H, K, V = H_in.shape
    _shape(log_decay, (B, H, K), "log_decay")
    _shape(S_loc, (B, H, K, V), "S_loc")
    for t, n in ((H_in, "H_in"), (log_decay, "log_decay"), (S_loc, "S_loc")):
        _check(t, n)
    if out is None:
        out = torch.empty_like(H_in)
    _same_device(H_in.device, [("log_decay", log_decay), ("S_loc", S_loc), ("out", out)])
    with torch.cuda.device(H_in.device):
        _call(lib().gla_state_combine, "gla_state_combine", B * H, K, V, _ptr(H_in), _ptr(log_decay), _ptr(S_loc),
              _ptr(out), _stream(H_in.device))
    return out


# ---- GLA layer stages (include/gla.h "GLA layer"; the module is paper_2312_06635_b200/layer.py) ------------------
def _need(t, name, dtype, shape=None):
    _check(t, name)
    if t.dtype != dtype:
        raise RuntimeError(f"{name} must be {dtype}")
    if shape is not None:
        _shape(t, shape, name)


def layer_prep(P, z_alpha, b_alpha, H: int, K: int, V: int, tau: float = 16.0):
    """q, k [B,H,T,K], v [B,H,T,V] (bf16) and log alpha [B,H,T,K] fp32 from the projection output P [B,T,ldP]
    (blocks q | k | v | r) and the low-rank gate pre-activation z_alpha [B,T,H*K] (gla_layer_prep)."""
    B, T, ldP = P.shape
    _need(P, "P", torch.bfloat16)
    _need(z_alpha, "z_alpha", torch.bfloat16, (B, T, H * K))
    _need(b_alpha, "b_alpha", torch.float32, (H * K,))
    dev = P.device
    q = torch.empty((B, H, T, K), dtype=torch.bfloat16, device=dev)
    k = torch.empty_like(q)
    v = torch.empty((B, H, T, V), dtype=torch.bfloat16, device=dev)
    g = torch.empty((B, H, T, K), dtype=torch.float32, device=dev)
    _same_device(dev, [("z_alpha", z_alpha), ("b_alpha", b_alpha)])
    with torch.cuda.device(dev):
        _call(lib().gla_layer_prep, "gla_layer_prep", B, T, H, K, V, float(tau), _ptr(P), ldP, _ptr(z_alpha),
              _ptr(b_alpha), _ptr(q), _ptr(k), _ptr(v), _ptr(g), _stream(dev))
    return q, k, v, g


def layer_out(O, P, r_off: int, b_r, ln_w, ln_b, eps: float = 1e-5):
    """Z [B,T,H*V] bf16 = concat_h(LN(O^h) ln_w + ln_b) (.) Swish(r + b_r), plus the LN mean / rstd (gla_layer_out)."""
    B, H, T, V = O.shape
    _need(O, "O", torch.bfloat16)
    _need(P, "P", torch.bfloat16)
    for t, n in ((b_r, "b_r"), (ln_w, "ln_w"), (ln_b, "ln_b")):
        _need(t, n, torch.float32, (H * V,))
    dev = O.device
    Z = torch.empty((B, T, H * V), dtype=torch.bfloat16, device=dev)
    mean = torch.empty((B, T, H), dtype=torch.float32, device=dev)
    rstd = torch.empty_like(mean)
    with torch.cuda.device(dev):
        _call(lib().gla_layer_out, "gla_layer_out", B, T, H, V, _ptr(O), _ptr(P), P.shape[-1], r_off, _ptr(b_r),
              _ptr(ln_w), _ptr(ln_b), float(eps), _ptr(Z), _ptr(mean), _ptr(rstd), _stream(dev))
    return Z, mean, rstd


def layer_bwd_workspace(B, T, H, K, V, device):
    n = lib().gla_layer_bwd_workspace_size(B, T, H, K, V)
    return torch.empty(max(n, 16), dtype=torch.uint8, device=device)


def layer_out_bwd(dZ, O, P, r_off: int, b_r, ln_w, ln_b, mean, rstd, dP, workspace=None):
    """dO [B,H,T,V] bf16 and (d ln_w, d ln_b, d b_r); d r is written into dP's r block (gla_layer_out_bwd)."""
    B, H, T, V = O.shape
    _need(dZ, "dZ", torch.bfloat16, (B, T, H * V))
    _need(dP, "dP", torch.bfloat16, P.shape)
    dev = O.device
    dO = torch.empty_like(O)
    dw, db, dbr = (torch.empty(H * V, dtype=torch.float32, device=dev) for _ in range(3))
    if workspace is None:
        workspace = layer_bwd_workspace(B, T, H, 8, V, dev)
    with torch.cuda.device(dev):
        _call(lib().gla_layer_out_bwd, "gla_layer_out_bwd", B, T, H, V, _ptr(dZ), _ptr(O), _ptr(P), P.shape[-1], r_off,
              _ptr(b_r), _ptr(ln_w), _ptr(ln_b), _ptr(mean), _ptr(rstd), _ptr(dO), _ptr(dP), _ptr(dw), _ptr(db),
              _ptr(dbr), _ptr(workspace), workspace.numel(), _stream(dev))
    return dO, dw, db, dbr


def layer_prep_bwd(dq, dk, dv, d_log_alpha, z_alpha, b_alpha, dP, tau: float = 16.0, workspace=None):
    """d z_alpha [B,T,H*K] bf16 and d b_alpha [H*K] fp32; dq, dk, dv go into dP's q | k | v blocks
    (gla_layer_prep_bwd)."""
    B, H, T, K = dq.shape
    V = dv.shape[-1]
    _need(d_log_alpha, "d_log_alpha", torch.float32, (B, H, T, K))
    _need(dP, "dP", torch.bfloat16)
    dev = dq.device
    dZa = torch.empty((B, T, H * K), dtype=torch.bfloat16, device=dev)
    dba = torch.empty(H * K, dtype=torch.float32, device=dev)
    if workspace is None:
        workspace = layer_bwd_workspace(B, T, H, K, V, dev)
    with torch.cuda.device(dev):
        _call(lib().gla_layer_prep_bwd, "gla_layer_prep_bwd", B, T, H, K, V, float(tau), _ptr(dq), _ptr(dk), _ptr(dv),
              _ptr(d_log_alpha), _ptr(z_alpha), _ptr(b_alpha), _ptr(dP), dP.shape[-1], _ptr(dZa), _ptr(dba),
              _ptr(workspace), workspace.numel(), _stream(dev))
    return dZa, dba


class GLAFunction(torch.autograd.Function):
    """Autograd wrapper: forward gla_chunk_fwd, backward gla_chunk_bwd_saved (the forward's workspace -- its
    per-chunk operands and anchor states -- is kept as the saved activation of the step)."""

    @staticmethod
    def forward(ctx, q, k, v, log_alpha, initial_state, chunk, subchunk, path):
        ws = fwd_workspace(q, v, log_alpha, chunk, subchunk, path)
        o, fs = chunk_fwd(q, k, v, log_alpha, chunk, subchunk, initial_state, True, path, workspace=ws)
        ctx.save_for_backward(q, k, v, log_alpha, initial_state)
        ctx.ws = ws
        ctx.cfg = (chunk, subchunk, path)
        return o, fs

    @staticmethod
    def backward(ctx, do, dfs):
        q, k, v, g, h0 = ctx.saved_tensors
        chunk, subchunk, path = ctx.cfg
        dq, dk, dv, dg, dh0 = chunk_bwd(q, k, v, g, do.contiguous(), chunk, subchunk, h0,
                                        None if dfs is None else dfs.contiguous(), h0 is not None, path,
                                        fwd_workspace=ctx.ws)
        ctx.ws = None
        return dq, dk, dv, dg.to(g.dtype), dh0, None, None, None


def gla(q, k, v, log_alpha, initial_state=None, chunk: int = 64, subchunk: int = 16, path: str = "auto"):
    """Differentiable chunk-wise GLA core: returns (o, final_state)."""
    return GLAFunction.apply(q, k, v, log_alpha, initial_state, chunk, subchunk, path)


def profile(enable: bool = True):
    """Turn the library's per-launch CUDA-event tracing on/off (resets the record)."""
    lib().gla_profile_reset()
    lib().gla_profile_enable(1 if enable else 0)


def profile_read():
    """{kernel name: (total_ms, launches)} for the launches recorded since profile(True)."""
    cap = 64
    names = ctypes.create_string_buffer(64 * cap)
    ms = (ctypes.c_float * cap)()
    n = (ctypes.c_int * cap)()
    cnt = lib().gla_profile_get(cap, names, ms, n)
    out = {}
    for i in range(min(cnt, cap)):
        nm = names.raw[64 * i: 64 * i + 64].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(n[i]))
    return out


# ---- the general outer-product gate G_t = alpha_t^T beta_t (gla.h "value gate") ----------------------
def beta_workspace(q, v, log_alpha, chunk=64, subchunk=16, path="auto") -> torch.Tensor:
    n = lib().gla_beta_workspace_size(ctypes.byref(desc(q, v, log_alpha, chunk, subchunk, path)))
    return torch.empty(max(n, 16), dtype=torch.uint8, device=q.device)


def _check_beta(q, v, log_alpha, log_beta):
    _check(log_beta, "log_beta")
    _shape(log_beta, tuple(v.shape), "log_beta")
    if log_beta.dtype != log_alpha.dtype:
        raise RuntimeError("log_beta must have log_alpha's dtype")
    _same_device(q.device, [("log_beta", log_beta)])


def chunk_fwd_beta(q, k, v, log_alpha, log_beta, chunk: int = 64, subchunk: int = 16, initial_state=None,
                   output_final_state: bool = False, path: str = "auto", workspace=None):
    """o [B,H,T,V] and final_state [B,H,K,V] fp32 (or None) with both gates.  gla_chunk_fwd_beta."""
    _check(q, "q")
    _check_problem(q, k, v, log_alpha, initial_state=initial_state)
    _check_beta(q, v, log_alpha, log_beta)
    B, H, T, K = q.shape
    V = v.shape[-1]
    d = desc(q, v, log_alpha, chunk, subchunk, path)
    out = torch.empty((B, H, T, V), dtype=q.dtype, device=q.device)
    fs = torch.empty((B, H, K, V), dtype=torch.float32, device=q.device) if output_final_state else None
    if workspace is None:
        workspace = beta_workspace(q, v, log_alpha, chunk, subchunk, path)
    with torch.cuda.device(q.device):
        _call(lib().gla_chunk_fwd_beta, "gla_chunk_fwd_beta", ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v),
              _ptr(log_alpha), _ptr(log_beta), _ptr(initial_state), _ptr(out), _ptr(fs), _ptr(workspace),
              workspace.numel(), _stream(q.device))
    return out, fs


def chunk_bwd_beta(q, k, v, log_alpha, log_beta, d_out, chunk: int = 64, subchunk: int = 16, initial_state=None,
                   d_final_state=None, need_d_initial_state: bool = False, path: str = "auto", workspace=None):
    """(dq, dk, dv, d_log_alpha fp32, d_log_beta fp32, d_initial_state fp32 or None).  gla_chunk_bwd_beta."""
    _check(q, "q")
    _check_problem(q, k, v, log_alpha, d_out, initial_state, d_final_state)
    _check_beta(q, v, log_alpha, log_beta)
    B, H, T, K = q.shape
    d = desc(q, v, log_alpha, chunk, subchunk, path)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dg = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    dgb = torch.empty(v.shape, dtype=torch.float32, device=q.device)
    dh0 = torch.empty((B, H, K, v.shape[-1]), dtype=torch.float32, device=q.device) if need_d_initial_state else None
    if workspace is None:
        workspace = beta_workspace(q, v, log_alpha, chunk, subchunk, path)
    with torch.cuda.device(q.device):
        _call(lib().gla_chunk_bwd_beta, "gla_chunk_bwd_beta", ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v),
              _ptr(log_alpha), _ptr(log_beta), _ptr(initial_state), _ptr(d_out), _ptr(d_final_state), _ptr(dq),
              _ptr(dk), _ptr(dv), _ptr(dg), _ptr(dgb), _ptr(dh0), _ptr(workspace), workspace.numel(),
              _stream(q.device))
    return dq, dk, dv, dg, dgb, dh0


def recurrent_step_beta(q_t, k_t, v_t, log_alpha_t, log_beta_t, state):
    """One decode step with both gates; ``state`` [B,H,K,V] fp32 updated in place; returns o_t [B,H,V]."""
    for t, n in ((q_t, "q_t"), (k_t, "k_t"), (v_t, "v_t"), (log_alpha_t, "log_alpha_t"), (log_beta_t, "log_beta_t"),
                 (state, "state")):
        _check(t, n)
    B, H, K = q_t.shape
    V = v_t.shape[-1]
    _shape(k_t, (B, H, K), "k_t")
    _shape(log_alpha_t, (B, H, K), "log_alpha_t")
    _shape(v_t, (B, H, V), "v_t")
    _shape(log_beta_t, (B, H, V), "log_beta_t")
    _shape(state, (B, H, K, V), "state")
    if state.dtype != torch.float32:
        raise RuntimeError("state must be fp32")
    out = torch.empty((B, H, V), dtype=q_t.dtype, device=q_t.device)
    _same_device(q_t.device, [("k_t", k_t), ("v_t", v_t), ("log_alpha_t", log_alpha_t), ("log_beta_t", log_beta_t),
                              ("state", state)])
    with torch.cuda.device(q_t.device):
        _call(lib().gla_recurrent_step_beta, "gla_recurrent_step_beta", B, H, K, V, _dt(q_t), _dt(log_alpha_t),
              _ptr(q_t), _ptr(k_t), _ptr(v_t), _ptr(log_alpha_t), _ptr(log_beta_t), _ptr(state), _ptr(out),
              _stream(q_t.device))
    return out
