#!/usr/bin/env python3
"""Microbenchmark of the tcgen05 GEMM on the C2 (BERT-base, 4096-token) step
shapes, with the epilogues the engine uses, against torch.matmul (cuBLAS) on
the same shapes for context.  CUDA events on the launching (default) stream,
warm L2 (weights are re-read every step in the real run too).

  python tools/gemm_bench.py [--iters 20] [--bn 0] [--json out.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import _lib  # noqa: E402

T, D, F, H = 4096, 768, 3072, 12
# name, M, N, K, a_trans, b_trans, c_f32, bias, act, resid, b_group
SHAPES = [
    ("qkv_fwd", T, 3 * D, D, 0, 0, 0, 0, 0, 0, 64),
    ("wo_fwd", T, D, D, 0, 0, 0, 1, 0, 1, 0),
    ("ffn1_fwd_gelu", T, F, D, 0, 0, 0, 1, 1, 0, 0),
    ("ffn2_fwd", T, D, F, 0, 0, 0, 1, 0, 1, 0),
    ("dW2", F, D, T, 1, 0, 1, 0, 0, 0, 0),
    ("dU_dgelu", T, F, D, 0, 1, 0, 0, 2, 0, 0),
    ("dW1", D, F, T, 1, 0, 1, 0, 0, 0, 0),
    ("dX1", T, D, F, 0, 1, 0, 0, 0, 1, 0),
    ("dWo", D, D, T, 1, 0, 1, 0, 0, 0, 0),
    ("dO", T, D, D, 0, 1, 0, 0, 0, 0, 0),
    ("dWqkv", D, 3 * D, T, 1, 0, 1, 0, 0, 0, 0),
    ("dX", T, D, 3 * D, 0, 1, 0, 0, 0, 1, 64),
    ("mlm_logits", 608, 30522, D, 0, 0, 1, 1, 0, 0, 0),
    ("dmlm_w", D, 30522, 608, 1, 0, 1, 0, 0, 0, 0),
    ("dhm", 608, D, 30522, 0, 1, 1, 0, 0, 0, 0),
]
VARIANTS = [
    ("v_plain_bf16", T, F, D, 0, 0, 0, 0, 0, 0, 0),
    ("v_bias_bf16", T, F, D, 0, 0, 0, 1, 0, 0, 0),
    ("v_gelu_aux", T, F, D, 0, 0, 0, 1, 1, 0, 0),
    ("v_plain_f32", T, F, D, 0, 0, 1, 0, 0, 0, 0),
    ("v_kmajor_b", T, F, D, 0, 1, 0, 0, 0, 0, 0),
    ("v_long_k", T, D, F, 0, 0, 0, 0, 0, 0, 0),
]
PER_STEP = {v[0]: 0 for v in VARIANTS}
PER_STEP.update({"qkv_fwd": 12, "wo_fwd": 12, "ffn1_fwd_gelu": 12, "ffn2_fwd": 12, "dW2": 12,
            "dU_dgelu": 12, "dW1": 12, "dX1": 12, "dWo": 12, "dO": 12, "dWqkv": 12, "dX": 12,
            "mlm_logits": 1, "dmlm_w": 1, "dhm": 1})


GRAPH = True


def p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def run(shape, iters, bn):
    name, M, N, K, at, bt, cf32, bias, act, resid, grp = shape
    dev = "cuda"
    bf = torch.bfloat16
    Kp = (K + 7) // 8 * 8
    A = torch.randn(K, M, device=dev).to(bf) if at else torch.randn(M, Kp, device=dev).to(bf)
    lda = M if at else Kp
    Np = (N + 7) // 8 * 8
    if grp and not bt:
        B = torch.randn(N // grp, K, grp, device=dev).to(bf)
        ldb, gs = grp, K * grp
    elif grp and bt:
        B = torch.randn(K // grp, N, grp, device=dev).to(bf)
        ldb, gs = grp, N * grp
    elif bt:
        B = torch.randn(N, ((K + 7) // 8) * 8, device=dev).to(bf)
        ldb, gs = B.shape[1], 0
    else:
        B = torch.randn(K, Np, device=dev).to(bf)
        ldb, gs = Np, 0
    ct = torch.float32 if cf32 else bf
    Cm = torch.zeros(M, N, device=dev, dtype=ct)
    bvec = torch.randn(N, device=dev) if bias else None
    aux = torch.randn(M, N, device=dev).to(ct) if act else None
    R = torch.randn(M, N, device=dev).to(ct) if resid else None
    args = (M, N, K, 1, p(A), lda, at, p(B), ldb, bt, grp, gs, p(Cm), N, 0 if cf32 else 1, 0, 0,
            p(bvec), act, p(aux), p(R), N if resid else 0, 0, 2, bn)
    for _ in range(3):
        _lib.call("hp_debug_gemm", *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # keep the GPU busy while the host enqueues, so the timed launches run
    # back to back (device time, not host launch overhead)
    if GRAPH:
        # the launches as CUDA graph nodes (the engine's mode): stream launches
        # complete on a ~2 us grid on this platform (profiles/r01_launch_granularity.txt)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            _lib.call("hp_debug_set_stream", C.c_void_p(torch.cuda.current_stream().cuda_stream))
            for _ in range(iters):
                _lib.call("hp_debug_gemm", *args)
            _lib.call("hp_debug_set_stream", None)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
    else:
        torch.cuda._sleep(100_000_000)
        e0.record()
        for _ in range(iters):
            _lib.call("hp_debug_gemm", *args)
        e1.record()
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    # cuBLAS on the same math (plain matmul, no epilogue) for context
    a2 = A.t() if at else A
    b2 = (B.reshape(-1, B.shape[-1]) if grp else B)
    x = (a2[:, :K] if not at else a2).contiguous()
    y = torch.randn(K, N, device=dev).to(bf)
    for _ in range(3):
        torch.matmul(x, y)
    torch.cuda.synchronize()
    if GRAPH:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(iters):
                torch.matmul(x, y)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        torch.cuda._sleep(100_000_000)
        e0.record()
        for _ in range(iters):
            torch.matmul(x, y)
        e1.record()
    torch.cuda.synchronize()
    us_cb = e0.elapsed_time(e1) * 1e3 / iters
    fl = 2.0 * M * N * K
    return {"name": name, "M": M, "N": N, "K": K, "us": us, "tflops": fl / us / 1e6,
            "cublas_us": us_cb, "cublas_tflops": fl / us_cb / 1e6, "per_step": PER_STEP[name]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--bn", type=int, default=0)
    ap.add_argument("--json", default=None)
    ap.add_argument("--only", default=None, help="comma-separated shape names")
    ap.add_argument("--stream", action="store_true",
                    help="time stream launches instead of CUDA-graph replays")
    a = ap.parse_args()
    global GRAPH
    GRAPH = not a.stream
    shapes = [s for s in SHAPES + VARIANTS if (not a.only and s in SHAPES) or
              (a.only and (s[0] in a.only.split(",") or (a.only == "variants" and s in VARIANTS)))]
    res = [run(s, a.iters, a.bn) for s in shapes]
    tot = sum(r["us"] * r["per_step"] for r in res)
    tot_cb = sum(r["cublas_us"] * r["per_step"] for r in res)
    fl = sum(2.0 * r["M"] * r["N"] * r["K"] * r["per_step"] for r in res)
    for r in res:
        print(f"{r['name']:>14} {r['M']:5d}x{r['N']:5d}x{r['K']:5d}  {r['us']:8.1f} us {r['tflops']:7.1f} TF/s"
              f"   cuBLAS {r['cublas_us']:8.1f} us {r['cublas_tflops']:7.1f} TF/s")
    if tot > 0:
        print(f"step GEMM total: ours {tot/1e3:.3f} ms ({fl/tot/1e6:.0f} TF/s)  cuBLAS {tot_cb/1e3:.3f} ms ({fl/tot_cb/1e6:.0f} TF/s)")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"shapes": res, "total_ms": tot / 1e3, "cublas_total_ms": tot_cb / 1e3}, f, indent=1)


if __name__ == "__main__":
    main()
