"""Projection GEMMs (FP32 FFMA and tcgen05 TF32) vs a plain PyTorch fp32
reference of the same op, in all three orientations the TGN step uses.

Tolerances: FFMA differs from torch only by summation order (rel 1e-5);
TF32 rounds operands to 10-bit mantissas (rel 2e-3 on a K~400 dot product)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def call(impl, which, A, B, Cm, M, N, K, ws):
    from paper_2308_14129_b200._lib import lib
    from paper_2308_14129_b200 import _check
    p = lambda t: C.c_void_p(t.data_ptr())
    _check(lib.spd_debug_gemm(impl, which, p(A), A.stride(0), p(B), B.stride(0), p(Cm),
                              Cm.stride(0), M, N, K, p(ws), ws.numel()))


def padded(rows, cols, gen):
    ld = (cols + 3) // 4 * 4
    t = torch.zeros(rows, ld, device="cuda")
    t[:, :cols] = torch.randn(rows, cols, generator=gen, device="cuda")
    return t


SHAPES = [(60000, 400, 387), (60000, 200, 400), (30001, 416, 388), (6000, 200, 201), (4000, 300, 487), (130, 17, 5), (128, 64, 32),
          (257, 130, 70), (6000, 100, 301)]


@pytest.mark.parametrize("impl,tol", [(0, 1e-5), (1, 3e-3)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_fwd(impl, tol, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A, W = padded(M, K, g), padded(N, K, g)
    Cm = torch.zeros(M, (N + 3) // 4 * 4, device="cuda")
    ws = torch.zeros(1 << 22, device="cuda")
    call(impl, 0, A, W, Cm, M, N, K, ws)
    ref = A[:, :K] @ W[:, :K].T
    err = (Cm[:, :N] - ref).norm() / ref.norm()
    assert err < tol, float(err)


@pytest.mark.parametrize("impl,tol", [(0, 1e-5), (1, 3e-3)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_dgrad(impl, tol, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 5 + K)
    A, W = padded(M, K, g), padded(K, N, g)
    Cm = torch.zeros(M, (N + 3) // 4 * 4, device="cuda")
    ws = torch.zeros(1 << 22, device="cuda")
    call(impl, 1, A, W, Cm, M, N, K, ws)
    ref = A[:, :K] @ W[:, :N]
    err = (Cm[:, :N] - ref).norm() / ref.norm()
    assert err < tol, float(err)


@pytest.mark.parametrize("impl,tol", [(0, 1e-5), (1, 3e-3)])
@pytest.mark.parametrize("M,N,K", [(400, 387, 60000), (256, 300, 20000), (400, 448, 33000), (300, 487, 4000), (200, 201, 6000),
                                   (17, 5, 130), (1, 101, 4000), (100, 301, 6000)])
def test_wgrad_accumulates(impl, tol, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    dY, X = padded(K, M, g), padded(K, N, g)
    C0 = padded(M, N, g)
    Cm = C0.clone()
    ws = torch.zeros(1 << 24, device="cuda")
    call(impl, 2, dY, X, Cm, M, N, K, ws)
    ref = C0[:, :N] + dY[:, :M].T @ X[:, :N]
    err = (Cm[:, :N] - ref).norm() / ref.norm()
    assert err < tol, float(err)
