#!/bin/bash
# N = 1, 2, 4 back to back on one 4-GPU box (bench.py defaults), JSON lines to gpurun_out/
python bench.py > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) bench.py --gpus $n > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
done
python - <<'PY'
import json
v = {n: json.load(open(f"gpurun_out/scale_n{n}.json")) for n in (1, 2, 4)}
for n, j in v.items():
    a = j.get("allreduce") or {}
    print(n, round(j["value"], 1), "eff", round(j["value"] / (n * v[1]["value"]), 4), "ms", round(j["ms_per_step"], 3),
          "exposed", a.get("exposed_ms"), "hidden", a.get("hidden_frac"), "busbw", a.get("bus_gbps"))
PY
