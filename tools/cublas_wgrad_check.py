import torch
T, D, F = 4096, 768, 3072
def t(fn, iters=30):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(iters): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters
bf = torch.bfloat16
X1 = torch.randn(T, D, device="cuda", dtype=bf); dU = torch.randn(T, F, device="cuda", dtype=bf)
G = torch.randn(T, F, device="cuda", dtype=bf); dY = torch.randn(T, D, device="cuda", dtype=bf)
X1t = X1.t().contiguous(); Gt = G.t().contiguous()
for name, fn, fl in [("dW1 = X1^T dU (transA, fp32 out)", lambda: torch.matmul(X1.t(), dU, out_dtype=torch.float32) if False else torch.mm(X1.t(), dU).float(), 2*D*F*T),
                     ("dW1 bf16 out, transA", lambda: torch.mm(X1.t(), dU), 2*D*F*T),
                     ("dW1 bf16 out, pre-transposed A", lambda: torch.mm(X1t, dU), 2*D*F*T),
                     ("dW2 bf16 out, transA", lambda: torch.mm(G.t(), dY), 2*D*F*T),
                     ("dW2 bf16 out, pre-transposed", lambda: torch.mm(Gt, dY), 2*D*F*T)]:
    us = t(fn)
    print(f"{name:36s} {us:7.1f} us {fl/us/1e6:7.1f} TF/s")
