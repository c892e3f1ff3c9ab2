#!/usr/bin/env python3
"""C5: gradient-bucket allreduce sweep (BASELINE configs[4]).

fp32 buffers of 1 MB .. 1 GB, cut into the engine's buckets (25 / 50 / 100
MiB caps, contiguous ranges walked from the end), each bucket one in-place
ncclAllReduce(ncclSum) on one stream -- the call the engine issues per bucket
(engine.cpp issue_bucket), replacing the reference's flat all_reduce_sum
(engine.hpp:145).  Device time with CUDA events, max over ranks; rank 0
prints one JSON line per (size, bucket) and a summary line.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node W \\
      --master-addr 127.0.0.1 --master-port 29531 tools/allreduce_sweep.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MB = 1 << 20
SIZES = [1 * MB, 4 * MB, 16 * MB, 64 * MB, 256 * MB, 440 * MB, 1024 * MB]  # 440 MB = C2 grads
BUCKETS = [25.0, 50.0, 100.0]


def main() -> int:
    import torch
    import torch.distributed as dist
    import paper_2009_14783_b200 as hp

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world < 2:
        print(json.dumps({"error": "needs >= 2 ranks (torchrun)"}))
        return 0
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    comm = hp.Communicator(world, rank, local)
    rows = []
    for size in SIZES:
        for bmb in BUCKETS:
            if bmb * MB > 2 * size and bmb != BUCKETS[0]:
                continue  # one bucket either way: same as the 25 MB row
            iters = 20 if size <= 64 * MB else 5
            r = comm.allreduce_bench(size, bmb, iters=iters, warmup=3)
            t = torch.tensor([r["ms"]], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            alg = size / (ms / 1e3) / 1e9
            row = {"bytes": size, "bucket_mb": bmb, "buckets": -(-size // int(bmb * MB)),
                   "ms": ms, "algbw_gbps": alg, "busbw_gbps": alg * 2 * (world - 1) / world}
            rows.append(row)
            if rank == 0:
                print(json.dumps({"world": world, **row}), flush=True)
    if rank == 0:
        best = max(rows, key=lambda r: r["busbw_gbps"])
        print(json.dumps({"summary": "allreduce_sweep", "world": world,
                          "peak_busbw_gbps": best["busbw_gbps"], "at_bytes": best["bytes"],
                          "at_bucket_mb": best["bucket_mb"],
                          "nvlink_per_direction_gbps": 900}), flush=True)
    comm.close()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
