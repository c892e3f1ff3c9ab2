"""World-size-2 host-side logic over torch.distributed (gloo, CPU): every rank
derives the identical epoch plan, rank schedules partition the batches exactly
(dataset.cpp:90-117), lockstep round counts agree, and the NCCL unique id is
shipped rank 0 -> all (the role ProcessGroup::broadcast plays, comm.hpp:25-27)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from helpers import C1_GEN


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2009_14783_b200 as hp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
    out = {}
    for (ms, mt, seed, epoch) in [(8, 0, 21, 0), (5, 200, 3, 2), (3, 0, 9, 1)]:
        plan = hp.build_epoch_batches(rec.token_lengths(), ms, mt, seed, epoch)
        sched = hp.partition_for_rank(plan, world, rank)
        digest = torch.tensor([int(np.concatenate(plan.batches).sum()), len(plan.batches)], dtype=torch.int64)
        alld = [torch.zeros_like(digest) for _ in range(world)]
        dist.all_gather(alld, digest)
        mine = torch.tensor([rb.batch_index if not rb.dummy else -1 for rb in sched], dtype=torch.int64)
        allm = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allm, mine)   # same length on every rank: lockstep rounds
        out[(ms, mt, seed, epoch)] = ([d.tolist() for d in alld], [m.tolist() for m in allm], len(plan.batches))
    # ship a 128-byte id from rank 0 the way Communicator does
    uid = (C.c_uint8 * 128)(*([rank + 1] * 128))
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
    dist.broadcast(t, src=0)
    out["uid"] = t.tolist()
    q.put((rank, out))
    dist.destroy_process_group()


def test_two_rank_schedules_and_id_broadcast():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for key in [k for k in res[0] if k != "uid"]:
        digests, scheds, nb = res[0][key]
        assert digests[0] == digests[1]                      # identical plans everywhere
        real = sorted(b for s in scheds for b in s if b >= 0)
        assert real == list(range(nb))                       # exact partition of the batches
        assert res[1][key][1] == scheds                      # both ranks saw the same gather
    assert res[0]["uid"] == res[1]["uid"] == [1] * 128       # rank 0's id everywhere


def test_tcp_rendezvous_missing_rank_times_out():
    """A rank whose master never appears fails with the reference's comm
    error after the timeout (test_comm.cpp:242-261 role) -- no hang."""
    import time

    import paper_2009_14783_b200 as hp
    import pytest
    t0 = time.time()
    with pytest.raises(hp.CommError, match="tcp rendezvous"):
        hp.Communicator.tcp("127.0.0.1", _free_port(), 2, 1, 0, timeout_ms=500)
    assert time.time() - t0 < 10
