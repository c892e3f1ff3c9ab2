#!/usr/bin/env python3
"""Per-launch device time floor of the tcgen05 GEMM (profiling aid)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import _lib  # noqa: E402

def p(t): return None if t is None else C.c_void_p(t.data_ptr())

def timeit(fn, iters):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000_000)
    e0.record()
    for _ in range(iters): fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters

for (M, N, K) in [(128, 128, 64), (128, 256, 768), (4096, 3072, 768)]:
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(K, N, device="cuda").bfloat16()
    Cm = torch.zeros(M, N, device="cuda").bfloat16()
    for code in [1128, 1256, 2256, 700000 + 1128, 700000 + 2256]:
        args = (M, N, K, 1, p(A), K, 0, p(B), N, 0, 0, 0, p(Cm), N, 1, 0, 0, None, 0, None, None, 0, 0, 2, code)
        f = lambda: _lib.call("hp_debug_gemm", *args)
        print(f"{M}x{N}x{K} code {code}: " + "  ".join(f"it{it}={timeit(f, it):.2f}us" for it in (10, 100)))
x = torch.zeros(1024, device="cuda")
print("torch add_: " + "  ".join(f"it{it}={timeit(lambda: x.add_(1), it):.2f}us" for it in (10, 100)))
