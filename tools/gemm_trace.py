#!/usr/bin/env python3
"""CTA-0 clock64 timeline of one tcgen05 GEMM launch (profiling aid).

  python tools/gemm_trace.py M N K code [act] [a_trans] [c_f32]
(needs a HP_GEMM_PROFILE=1 build of the library)
Prints cycle offsets (from kernel entry) of: prologue done, per k-block
producer-slot / MMA-full / MMA-commit, per tile epilogue start/end."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import _lib  # noqa: E402

def p(t): return None if t is None else C.c_void_p(t.data_ptr())

M, N, K, code = (int(x) for x in sys.argv[1:5])
act = int(sys.argv[5]) if len(sys.argv) > 5 else 0
at = int(sys.argv[6]) if len(sys.argv) > 6 else 0
cf = int(sys.argv[7]) if len(sys.argv) > 7 else 0
A = torch.randn(K, M, device="cuda").bfloat16() if at else torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(K, N, device="cuda").bfloat16()
Cm = torch.zeros(M, N, device="cuda", dtype=torch.float32 if cf else torch.bfloat16)
bias = torch.zeros(N, device="cuda") if act == 1 else None
aux = torch.zeros(M, N, device="cuda").bfloat16() if act else None
args = (M, N, K, 1, p(A), M if at else K, at, p(B), N, 0, 0, 0, p(Cm), N, 0 if cf else 1, 0, 0, p(bias), act,
        p(aux), None, 0, 0, 2, code)
tr = torch.zeros(1024 + 2 * 1024, dtype=torch.int64, device="cuda")
for _ in range(3): _lib.call("hp_debug_gemm", *args)
torch.cuda.synchronize()
_lib.call("hp_debug_gemm_trace", p(tr))
torch.cuda._sleep(50_000_000)
for _ in range(3): _lib.call("hp_debug_gemm", *args)   # the last launch's trace survives
_lib.call("hp_debug_gemm_trace", None)
torch.cuda.synchronize()
t = tr.cpu().tolist()
cta = [(t[1024 + 2 * i], t[1024 + 2 * i + 1]) for i in range(1024) if t[1024 + 2 * i]]
if cta:
    s0 = min(a for a, _ in cta)
    starts = sorted(a - s0 for a, _ in cta)
    ends = sorted(b - s0 for _, b in cta)
    durs = sorted(b - a for a, b in cta)
    pct = lambda v, q: v[min(len(v) - 1, int(q * len(v)))]
    print(f"CTAs {len(cta)}: start ns p0 {starts[0]} p50 {pct(starts, .5)} max {starts[-1]} | "
          f"end p0 {ends[0]} p50 {pct(ends, .5)} max {ends[-1]} | dur p0 {durs[0]} p50 {pct(durs, .5)} max {durs[-1]}")
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
