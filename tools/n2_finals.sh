#!/bin/bash
# N = 2 A/B: HEAD vs per-final launches (prefin = 405bd79), batched main-stream finals (fin1 = 69e8fe7), + wgrad-stream final (fin2 = 354a774)
run() {
  env $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('$1', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'nocomm', round(a['ms_per_step_without_grad_allreduce'],3))"
}
for rep in 1 2; do
  run HP_X=head
  run HP_LIB_VARIANT=prefin
  run HP_LIB_VARIANT=fin2
done

# N = 1: C2 attention replay, HEAD vs fin2 (before the seq2seq packing code in the attention kernels)
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "N1 [$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["roofline"]["attention"]; print(round(d["value"]), round(d["ms_per_step"],4), "attn replay", round(a["replay_ms_per_step"],4))' 2>&1 | tail -1)"
}
for rep in 1 2; do one HP_X=head; one HP_LIB_VARIANT=fin2; one HP_LIB_VARIANT=prefin; done
