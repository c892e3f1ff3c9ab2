import torch, time
x = torch.zeros(1024, device="cuda")
def timeit(fn, iters=200):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000_000)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters
print("eager add_ per launch us:", timeit(lambda: x.add_(1)))
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    for _ in range(3): x.add_(1)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    for _ in range(100): x.add_(1)
print("graph add_ per node us:", timeit(lambda: g.replay(), 20) / 100)
y = torch.zeros(4096*768, device="cuda")
print("eager 12MB add_ per launch us:", timeit(lambda: y.add_(1)))
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2, stream=s):
    for _ in range(100): y.add_(1)
print("graph 12MB add_ per node us:", timeit(lambda: g2.replay(), 20) / 100)
