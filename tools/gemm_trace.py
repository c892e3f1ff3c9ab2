#!/usr/bin/env python3
"""CTA-0 clock64 timeline of one tcgen05 GEMM launch (profiling aid).

  python tools/gemm_trace.py M N K code [act]
Prints cycle offsets (from kernel entry) of: prologue done, per k-block
producer-slot / MMA-full / MMA-commit, per tile epilogue start/end."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import _lib  # noqa: E402

def p(t): return None if t is None else C.c_void_p(t.data_ptr())

M, N, K, code = (int(x) for x in sys.argv[1:5])
act = int(sys.argv[5]) if len(sys.argv) > 5 else 0
A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(K, N, device="cuda").bfloat16()
Cm = torch.zeros(M, N, device="cuda").bfloat16()
bias = torch.zeros(N, device="cuda") if act == 1 else None
aux = torch.zeros(M, N, device="cuda").bfloat16() if act else None
args = (M, N, K, 1, p(A), K, 0, p(B), N, 0, 0, 0, p(Cm), N, 1, 0, 0, p(bias), act, p(aux), None, 0, 0, 2, code)
tr = torch.zeros(1024, dtype=torch.int64, device="cuda")
for _ in range(3): _lib.call("hp_debug_gemm", *args)
torch.cuda.synchronize()
_lib.call("hp_debug_gemm_trace", p(tr))
torch.cuda._sleep(50_000_000)
for _ in range(3): _lib.call("hp_debug_gemm", *args)   # the last launch's trace survives
_lib.call("hp_debug_gemm_trace", None)
torch.cuda.synchronize()
t = tr.cpu().tolist()
t0 = t[0]
rel = lambda v: v - t0 if v else None
print(f"prologue done {rel(t[1])}  exit {rel(t[2])}")
its = [i for i in range(256) if t[16 + 256 + i]]
for i in its:
    pp, f, c = rel(t[16 + i]), rel(t[16 + 256 + i]), rel(t[16 + 512 + i])
    print(f"kb {i:3d}  prod_slot {pp}  mma_full {f}  commit {c}")
for ci in range(8):
    if t[900 + 3 * ci]:
        print(f"chunk {ci} ld {rel(t[900+3*ci])}  ld_done {rel(t[901+3*ci])}  epi_done {rel(t[902+3*ci])}")
for j in range(32):
    if t[16 + 768 + 2 * j]:
        print(f"tile {j} epi_start {rel(t[16 + 768 + 2 * j])}  epi_end {rel(t[16 + 768 + 2 * j + 1])}")
