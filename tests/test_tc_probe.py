"""tcgen05 / UMMA-descriptor / TMA conventions (tc_common.cuh) vs torch.matmul, on one CTA."""
import ctypes
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2312_06635_b200",
                   "libgla_probe.so")


@pytest.fixture(scope="module")
def probe():
    L = ctypes.CDLL(LIB)
    L.probe_gemm.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int] * 7
    return L


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (128, 256, 256), (64, 64, 256), (128, 128, 128), (64, 128, 64)])
@pytest.mark.parametrize("a_mn,b_mn,tma", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 1), (1, 0, 1)])
def test_probe_gemm(probe, M, N, K, a_mn, b_mn, tma):
    torch.manual_seed(0)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    At = A.t().contiguous()
    D = torch.full((M, N), float("nan"), device="cuda")
    rc = probe.probe_gemm(A.data_ptr(), At.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, a_mn, b_mn, tma, 0)
    assert rc == 0, rc
    ref = A.float() @ B.float()
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("N,K", [(64, 256), (64, 128), (128, 64), (256, 64)])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_probe_gemm_a_in_tmem(probe, N, K, b_mn):
    """A operand read from TMEM (M = 128 lanes, bf16 pairs per column): the forward's O = SB Q~^T MMA."""
    torch.manual_seed(1)
    A = torch.randn(128, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    D = torch.full((128, N), float("nan"), device="cuda")
    rc = probe.probe_gemm(A.data_ptr(), A.data_ptr(), B.data_ptr(), D.data_ptr(), 128, N, K, 0, b_mn, 0, 1)
    assert rc == 0, rc
    ref = A.float() @ B.float()
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("N,K", [(64, 256), (64, 128), (128, 64)])
def test_probe_tf32_a_in_tmem(N, K):
    """kind::tf32 with the fp32 A operand read from TMEM and a K-major SW128 fp32 B tile (the anchored-frame
    walks' output MMA): equals an fp32 matmul of tf32-truncated operands."""
    L = ctypes.CDLL(LIB)
    L.probe_gemm_tf32.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 2
    torch.manual_seed(2)
    A = torch.randn(128, K, device="cuda")
    B = torch.randn(K, N, device="cuda")
    D = torch.full((128, N), float("nan"), device="cuda")
    assert L.probe_gemm_tf32(A.data_ptr(), B.data_ptr(), D.data_ptr(), N, K) == 0
    ref = A.double() @ B.double()
    err = (D.double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-3, err
