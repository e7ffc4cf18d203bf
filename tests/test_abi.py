"""C-ABI checks that need no GPU: libgla.so builds/loads, exports every symbol include/gla.h declares,
and validation errors return synchronously (no CUDA call is made on these paths)."""
import ctypes
import os
import re

import pytest
import torch

from paper_2312_06635_b200 import build as gla_build
from paper_2312_06635_b200 import binding as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    gla_build.build()
    return G.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "gla.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\*?\s*(gla_[a-z_]+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported(L):
    names = declared_functions()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(G.EXPORTS)


def test_status_strings(L):
    for s in range(9):
        assert L.gla_status_string(s)
    assert L.gla_version() == 100


def _d(**kw):
    base = dict(B=2, H=2, T=128, K=64, V=64, chunk=64, subchunk=16, qkv_dtype=0, gate_dtype=1, path=0)
    base.update(kw)
    return G._Desc(*[base[n] for n, _ in G._Desc._fields_])


FAKE = ctypes.c_void_p(0x10000)          # aligned, never dereferenced on validation failures
MISAL = ctypes.c_void_p(0x10008)


def fwd(L, d, q=FAKE, out=FAKE, ws=FAKE, wsb=1 << 40):
    return L.gla_chunk_fwd(ctypes.byref(d), q, FAKE, FAKE, FAKE, None, out, None, ws, wsb, None)


@pytest.mark.parametrize("kw,code", [
    (dict(T=100), 2), (dict(subchunk=5), 2), (dict(chunk=256, T=256), 2), (dict(chunk=128, T=256, path=2), 2),
    (dict(chunk=128, T=256, K=256, V=512), 2), (dict(chunk=0), 2),
    (dict(K=0), 1), (dict(V=-1), 1), (dict(K=512), 1), (dict(B=-1), 1),
    (dict(qkv_dtype=7), 3), (dict(gate_dtype=-1), 3), (dict(path=9), 6),
])
def test_fwd_validation(L, kw, code):
    assert fwd(L, _d(**kw)) == code


def test_null_align_workspace(L):
    assert fwd(L, _d(), q=None) == 5
    assert fwd(L, _d(), out=None) == 5
    assert fwd(L, _d(), q=MISAL) == 4
    need = L.gla_fwd_workspace_size(ctypes.byref(_d()))
    if need:
        assert fwd(L, _d(), wsb=need - 1) == 8


def test_bwd_and_helpers_validation(L):
    d = _d(T=96)
    args = [FAKE] * 9
    assert L.gla_chunk_bwd(ctypes.byref(d), *args[:4], None, FAKE, None, *args[:4], None, FAKE, 1 << 40,
                           None) == 2
    d = _d()
    assert L.gla_chunk_bwd(ctypes.byref(d), FAKE, FAKE, FAKE, FAKE, None, None, None, FAKE, FAKE, FAKE, FAKE,
                           None, FAKE, 1 << 40, None) == 5
    assert L.gla_recurrent_step(1, 1, 0, 4, 0, 1, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None) == 1
    assert L.gla_recurrent_step(1, 1, 4, 4, 0, 1, FAKE, FAKE, MISAL, FAKE, FAKE, FAKE, None) == 4
    assert L.gla_state_combine(2, 4, 4, FAKE, None, FAKE, FAKE, None) == 5
    assert L.gla_state_summary(ctypes.byref(_d(T=65)), FAKE, FAKE, FAKE, FAKE, FAKE, None, 0, None) == 2


def test_empty_problems_launch_nothing(L):
    # B*H == 0 returns OK without touching the (fake) pointers or CUDA
    assert fwd(L, _d(B=0)) == 0
    assert fwd(L, _d(H=0)) == 0


def test_path_resolution(L):
    assert L.gla_resolve_path(ctypes.byref(_d(path=1))) == 1
    # fp32 inputs never take the bf16 tensor-core path
    assert L.gla_resolve_path(ctypes.byref(_d(qkv_dtype=1))) == 1


def test_binding_refuses_cpu_tensors(L):
    q = torch.zeros(1, 1, 64, 16)
    with pytest.raises(RuntimeError, match="CUDA"):
        G.chunk_fwd(q, q, torch.zeros(1, 1, 64, 16), q)
