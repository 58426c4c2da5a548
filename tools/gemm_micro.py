"""Micro-benchmark of the projection GEMMs through the spd_debug_gemm hook."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2308_14129_b200._lib import lib
from paper_2308_14129_b200 import _check

def run(impl, which, M, N, K, lda_pad=0, iters=10):
    ldk = (K + 3) // 4 * 4 + lda_pad
    if which == 0:
        A = torch.randn(M, ldk, device="cuda"); B = torch.randn(N, ldk, device="cuda")
    elif which == 1:
        A = torch.randn(M, ldk, device="cuda"); B = torch.randn(K, (N + 3) // 4 * 4 + lda_pad, device="cuda")
    else:
        A = torch.randn(K, (M + 3) // 4 * 4 + lda_pad, device="cuda"); B = torch.randn(K, (N + 3) // 4 * 4 + lda_pad, device="cuda")
    Cm = torch.zeros(M, (N + 3) // 4 * 4, device="cuda")
    ws = torch.zeros(1 << 24, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    f = lambda: _check(lib.spd_debug_gemm(impl, which, p(A), A.stride(0), p(B), B.stride(0), p(Cm), Cm.stride(0), M, N, K, p(ws), ws.numel()))
    f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3

for args in [(1,0,60000,400,387,0),(1,0,60000,400,387,28),(1,0,60000,400,32,0),(1,0,60000,400,128,0),(1,0,60000,448,384,0),
             (1,0,6000,200,201,0),(1,0,6000,200,32,0),(1,0,128,224,32,0),(1,0,128,224,384,0),
             (0,0,60000,400,387,0),(1,1,60000,200,400,0),(1,1,60000,386,400,0),(1,2,400,387,60000,0)]:
    print(args, f"{run(*args):.1f} us")
