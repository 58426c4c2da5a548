"""Run one projection GEMM shape a few times (for ncu captures)."""
import ctypes as C, sys, torch
sys.path.insert(0, ".")
from paper_2308_14129_b200._lib import lib
from paper_2308_14129_b200 import _check
impl, which, M, N, K = (int(x) for x in sys.argv[1:6])
ld = lambda c: (c + 31) // 32 * 32
if which == 0: A = torch.randn(M, ld(K), device="cuda"); B = torch.randn(N, ld(K), device="cuda")
elif which == 1: A = torch.randn(M, ld(K), device="cuda"); B = torch.randn(K, ld(N), device="cuda")
else: A = torch.randn(K, ld(M), device="cuda"); B = torch.randn(K, ld(N), device="cuda")
Cm = torch.zeros(M, ld(N), device="cuda"); ws = torch.zeros(1 << 24, device="cuda")
p = lambda t: C.c_void_p(t.data_ptr())
for _ in range(3):
    _check(lib.spd_debug_gemm(impl, which, p(A), A.stride(0), p(B), B.stride(0), p(Cm), Cm.stride(0), M, N, K, p(ws), ws.numel()))
