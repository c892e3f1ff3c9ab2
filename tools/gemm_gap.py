#!/usr/bin/env python3
"""Gap between back-to-back tcgen05 GEMM launches (profiling aid; needs the
HP_GEMM_PROFILE build: HP_LIB_VARIANT=prof).  Launch i writes its per-CTA
[start, end] globaltimer stamps into its own trace buffer; prints, per
launch, the CTA start spread, the longest CTA, and the idle time between the
last CTA end of launch i and the first CTA start of launch i+1.

  python tools/gemm_gap.py M N K [code] [n_launches] [graph]"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import _lib  # noqa: E402

def p(t): return None if t is None else C.c_void_p(t.data_ptr())

M, N, K = (int(x) for x in sys.argv[1:4])
code = int(sys.argv[4]) if len(sys.argv) > 4 else 0
n = int(sys.argv[5]) if len(sys.argv) > 5 else 6
graph = len(sys.argv) > 6 and sys.argv[6] == "graph"
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(K, N, device="cuda").bfloat16()
Cm = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
args = (M, N, K, 1, p(A), K, 0, p(B), N, 0, 0, 0, p(Cm), N, 1, 0, 0, None, 0, None, None, 0, 0, 2, code)
trs = [torch.zeros(1024 + 2 * 1024, dtype=torch.int64, device="cuda") for _ in range(n)]
for _ in range(3): _lib.call("hp_debug_gemm", *args)
torch.cuda.synchronize()

def launch_all():
    for i in range(n):
        _lib.call("hp_debug_gemm_trace", p(trs[i]))
        _lib.call("hp_debug_gemm", *args)
    _lib.call("hp_debug_gemm_trace", None)

if graph:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _lib.call("hp_debug_set_stream", C.c_void_p(torch.cuda.current_stream().cuda_stream))
        launch_all()
        _lib.call("hp_debug_set_stream", None)
    g.replay(); torch.cuda.synchronize()
    for t in trs: t.zero_()
    g.replay()
else:
    torch.cuda._sleep(50_000_000)
    launch_all()
torch.cuda.synchronize()
prev_end = None
for i, t in enumerate(trs):
    v = t.cpu().tolist()
    cta = [(v[1024 + 2 * j], v[1024 + 2 * j + 1]) for j in range(1024) if v[1024 + 2 * j]]
    s0 = min(a for a, _ in cta); s1 = max(a for a, _ in cta); e1 = max(b for _, b in cta)
    gap = (s0 - prev_end) if prev_end else None
    print(f"launch {i}: CTAs {len(cta)} start spread {s1 - s0} ns, span {e1 - s0} ns, gap from previous {gap} ns")
    prev_end = e1
