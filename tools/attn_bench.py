#!/usr/bin/env python3
"""Attention kernels (fwd+bwd through hp_debug_attention) at the C2 shape:
32 sequences x 128 tokens, 12 heads, dk 64; CUDA events, per path."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import _lib  # noqa: E402

def p(t): return None if t is None else C.c_void_p(t.data_ptr())
B, S, H, dk = 32, 128, 12, 64
T = B * S
cu = torch.arange(0, T + 1, S, dtype=torch.int32, device="cuda")
qkv = torch.randn(T, 3 * H * dk, device="cuda").bfloat16()
dO = torch.randn(T, H * dk, device="cuda").bfloat16()
o = torch.zeros(T, H * dk, device="cuda").bfloat16()
lse = torch.zeros(H, T, device="cuda")
dqkv = torch.zeros_like(qkv)
for path, name in ((3, "tcgen05"), (2, "mma.sync")):
    for bwd in (False, True):
        args = (B, p(cu), T, H, dk, 1, p(qkv), p(o), p(lse), p(dO) if bwd else None, p(dqkv), path)
        for _ in range(3): _lib.call("hp_debug_attention", *args)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 20
        e0.record()
        for _ in range(it): _lib.call("hp_debug_attention", *args)
        e1.record(); torch.cuda.synchronize()
        print(f"{name:9s} {'fwd+bwd' if bwd else 'fwd    '} {e0.elapsed_time(e1) * 1e3 / it:8.1f} us (incl. a device sync per call)")

# CTA (0,0) timeline of one forward launch (clock64 cycles from kernel entry)
tr = torch.zeros(1024, dtype=torch.int64, device="cuda")
_lib.call("hp_debug_gemm_trace", p(tr))
args = (B, p(cu), T, H, dk, 1, p(qkv), p(o), p(lse), None, p(dqkv), 3)
_lib.call("hp_debug_attention", *args)
_lib.call("hp_debug_gemm_trace", None)
t = tr[1008:1018].cpu().tolist()
names = ["entry", "cu loaded", "init done", "Q/K/V landed", "S ready (softmax)", "P written",
         "P seen (mma)", "O ready", "epilogue done", "exit"]
print("fwd timeline:", ", ".join(f"{nm} {v - t[0]}" for nm, v in zip(names, t)))
