"""tcgen05 GEMM (vc_gemm_bf16) against a torch fp32 reference of the same op
on the same bf16 operands (numerics test for a floating-point kernel)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 176, 100), (1000, 1584, 4752),
                                   (21600 // 8, 14256, 1584), (7, 40, 24), (129, 513, 200)])
def test_gemm_bf16_matches_torch(torch, M, N, K):
    from paper_2501_08453_b200 import _lib
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g)
    out = torch.empty(M, N, device="cuda")
    rc = lib.vc_gemm_bf16(_lib.ptr(a), K, _lib.ptr(b), K, _lib.ptr(bias), _lib.ptr(res),
                          _lib.ptr(out), N, M, N, K, _lib.stream_ptr(torch))
    if K % 8:
        assert rc == _lib.VC_EINVAL
        return
    _lib.check(rc)
    ref = a.float() @ b.float().T + bias + res
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
