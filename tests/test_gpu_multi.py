"""Multi-GPU parity (real NCCL over NVLink, one process per GPU): the C1 run
at W=2 with the reference's own rank schedule (partition_for_rank) against
the reference W=2 f64 trajectory, identical parameters on both ranks
(params_digest, engine.hpp:170-184), and a dummy-rank round that must be
neutral (test_engine.cpp:296-321)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import C1_GEN, ROOT, golden, rel_norm

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["HP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HP_ROOT"], "tests"))
import torch, torch.distributed as dist
import paper_2009_14783_b200 as hp
from helpers import C1_GEN, C1_SPEC
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(rank)
comm = hp.Communicator(world, rank, rank)
spec = hp.ModelSpec(**C1_SPEC)
eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                    hp.ExecConfig(compute="f32", device=rank, max_tokens=1024, max_batch=16, max_masks=256,
                                  bucket_mb=0.3),
                    comm=comm, seed=21 if rank == 0 else None)
eng.broadcast_params(0)
rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
sched = hp.partition_for_rank(plan, world, rank)
losses = []
for step in range(10):
    rb = sched[step]
    rep = eng.round(rec.batch(plan.batches[rb.batch_index]), rb.dummy, 1e-3)
    losses.append(rep.loss)
rank_seconds = rep.rank_seconds  # gathered on the master only (engine.hpp:158-162)
digest = eng.digest()
p = eng.get_params()
# a round where rank 1 is a dummy: must equal rank 0 training alone (W=1 math)
rb0 = plan.batches[0]
rep = eng.round(rec.batch(rb0), rank == 1, 1e-3)
out = {"losses": losses, "digest": digest, "dummy_loss": rep.loss, "dummy_weight": rep.weight,
       "rank_seconds": rank_seconds}
# the bucketed-allreduce measurement (bench.py / tools/allreduce_sweep.py): 4 MiB in 1 MiB buckets
ar = comm.allreduce_bench(1 << 22, 1.0, iters=2, warmup=1)
out["ar_ok"] = ar["ms"] > 0 and ar["busbw_gbps"] > 0
if rank == 0:
    np.save(os.environ["HP_OUT"] + "/params.npy", p)
with open(os.environ["HP_OUT"] + f"/rank{rank}.json", "w") as f:
    json.dump(out, f)
eng.close(); comm.close()
dist.destroy_process_group()
'''


def test_c1_w2_nccl_matches_reference(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, HP_ROOT=ROOT, HP_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    t = golden("c1_ref_train.npz")
    r0 = json.loads((tmp_path / "rank0.json").read_text())
    r1 = json.loads((tmp_path / "rank1.json").read_text())
    l0 = np.array(r0["losses"])
    assert np.max(np.abs(l0 - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    assert r0["losses"] == r1["losses"]          # identical reports on every rank
    assert r0["digest"] == r1["digest"]          # identical parameters (digest check)
    p = np.load(tmp_path / "params.npy")
    assert rel_norm(p, t["params_f64_as_f32"]) <= 1e-4
    assert r0["dummy_weight"] == 8.0             # only rank 0's 8 sentences count
    assert r0["ar_ok"] and r1["ar_ok"]
    assert len(r0["rank_seconds"]) == 2 and all(t > 0 for t in r0["rank_seconds"])
    assert r1["rank_seconds"] == []


PG_WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["HP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HP_ROOT"], "tests"))
import paper_2009_14783_b200 as hp
from paper_2009_14783_b200 import _lib
from helpers import C1_GEN, C1_SPEC
rank, world = int(os.environ["HP_RANK"]), 2
comm = hp.Communicator.tcp("127.0.0.1", int(os.environ["HP_PORT"]), world, rank, rank)
out = {}
# broadcast: the root's exact bytes, whatever the others pass
out["bcast"] = comm.broadcast(b"root payload \x00\x01\xff" if rank == 1 else b"ignored", root=1).hex()
# all_reduce_sum: the rank-ordered fold (order matters for these values)
vals = [[1e16, 1.0, 0.1], [-1e16, 1.0, 0.2]][rank]
out["ar"] = comm.all_reduce_sum(vals)
out["gather"] = comm.gather_scalars(10.0 + rank)
comm.barrier()
try:
    comm.all_reduce_sum([1.0] * (2 + rank))
    out["mismatch"] = "accepted"
except _lib.CommError as e:
    out["mismatch"] = str(e)
# the engine on the TCP-formed communicator: three C1 rounds at W = 2
eng = hp.StepEngine(hp.ModelSpec(**C1_SPEC), hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                    hp.ExecConfig(compute="f32", device=rank, max_tokens=1024, max_batch=16, max_masks=256),
                    comm=comm, seed=21 if rank == 0 else None)
eng.broadcast_params(0)
rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
sched = hp.partition_for_rank(plan, world, rank)
out["losses"] = [eng.round(rec.batch(plan.batches[sched[s].batch_index]), sched[s].dummy, 1e-3).loss
                 for s in range(3)]
out["digest"] = eng.digest()
with open(os.environ["HP_OUT"] + f"/pg{rank}.json", "w") as f:
    json.dump(out, f)
eng.close(); comm.close()
'''


def test_process_group_over_tcp_rendezvous(tmp_path):
    # NcclProcessGroup (comm.hpp:16-49) on a world formed by the engine's own
    # TCP rendezvous -- no torch.distributed in the processes
    script = tmp_path / "pg.py"
    script.write_text(PG_WORKER)
    procs = []
    for r in range(2):
        env = dict(os.environ, HP_ROOT=ROOT, HP_OUT=str(tmp_path), HP_RANK=str(r), HP_PORT="29533")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    for p in procs:
        out, _ = p.communicate(timeout=600)
        assert p.returncode == 0, out[-3000:]
    r0 = json.loads((tmp_path / "pg0.json").read_text())
    r1 = json.loads((tmp_path / "pg1.json").read_text())
    assert bytes.fromhex(r0["bcast"]) == b"root payload \x00\x01\xff" == bytes.fromhex(r1["bcast"])
    fold = [(1e16 + -1e16), (1.0 + 1.0), (0.1 + 0.2)]
    assert r0["ar"] == fold and r1["ar"] == fold
    assert r0["gather"] == [10.0, 11.0] and r1["gather"] == []
    assert "length mismatch" in r0["mismatch"] and "length mismatch" in r1["mismatch"]
    t = golden("c1_ref_train.npz")
    assert np.max(np.abs(np.array(r0["losses"]) - t["losses_f64"][:3]) / np.abs(t["losses_f64"][:3])) <= 1e-4
    assert r0["losses"] == r1["losses"] and r0["digest"] == r1["digest"]


SPARSE_WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["HP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HP_ROOT"], "tests"))
import torch, torch.distributed as dist
import paper_2009_14783_b200 as hp
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(rank)
comm = hp.Communicator(world, rank, rank)
spec = hp.ModelSpec(arch="bert_encoder", d_model=128, heads=2, vocab=4000, max_seq=64, layers=1,
                    d_ff=256, label_smooth_eps=0.1)
rec = hp.generate_mlm_records(hp.MlmGenConfig(n=64, vocab=4000, min_sentence_words=10,
                                              max_sentence_words=30, seed=3, max_seq_tokens=64))
plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
sched = hp.partition_for_rank(plan, world, rank)
out = {}
for mode in ("1", "0", "1s", "0s"):  # s: split word-embedding update (HP_EMB_SPLIT=1)
    os.environ["HP_SPARSE_EMB"] = mode[0]
    os.environ["HP_EMB_SPLIT"] = "1" if mode.endswith("s") else "0"
    eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                        hp.ExecConfig(compute="f32", device=rank, max_tokens=512, max_batch=8,
                                      max_masks=128, bucket_mb=0.5),
                        comm=comm, seed=21 if rank == 0 else None)
    eng.broadcast_params(0)
    losses = []
    for s in range(4):
        rb = sched[s]
        losses.append(eng.round(rec.batch(plan.batches[rb.batch_index]), rb.dummy, 1e-3).loss)
    # a round where rank 1 is a dummy (empty row set on that rank)
    losses.append(eng.round(rec.batch(plan.batches[0]), rank == 1, 1e-3).loss)
    out[mode] = {"losses": losses, "digest": eng.digest()}
    if rank == 0:
        np.save(os.environ["HP_OUT"] + f"/p{mode}.npy", eng.get_params())
    eng.close()
with open(os.environ["HP_OUT"] + f"/sp{rank}.json", "w") as f:
    json.dump(out, f)
comm.close()
dist.destroy_process_group()
'''


def test_row_sparse_embedding_exchange_matches_dense(tmp_path):
    """N > 1 with the word embedding alone in the last bucket: the row-sparse
    exchange (allgather of (id, row) slots, rank-ordered scatter) trains like
    the dense allreduce (fp32 summation order aside), identical on every rank,
    dummy rounds included."""
    script = tmp_path / "sparse_worker.py"
    script.write_text(SPARSE_WORKER)
    env = dict(os.environ, HP_ROOT=ROOT, HP_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29519", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    r0 = json.loads((tmp_path / "sp0.json").read_text())
    r1 = json.loads((tmp_path / "sp1.json").read_text())
    for mode in ("1", "0", "1s", "0s"):
        assert r0[mode]["losses"] == r1[mode]["losses"]
        assert r0[mode]["digest"] == r1[mode]["digest"]
    # the split update (rows outside every rank's ids during backward, the
    # union's rows after the exchange) is bit-identical to the unsplit one
    for mode in ("1", "0"):
        assert r0[mode + "s"] == r0[mode]
        assert np.array_equal(np.load(tmp_path / f"p{mode}s.npy").view(np.uint32),
                              np.load(tmp_path / f"p{mode}.npy").view(np.uint32))
    a, b = np.array(r0["1"]["losses"]), np.array(r0["0"]["losses"])
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-5
    assert rel_norm(np.load(tmp_path / "p1.npy"), np.load(tmp_path / "p0.npy")) <= 1e-5


DIGEST_WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["HP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HP_ROOT"], "tests"))
import torch, torch.distributed as dist
import paper_2009_14783_b200 as hp
from helpers import C1_GEN, C1_SPEC
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(rank)
comm = hp.Communicator(world, rank, rank)
eng = hp.StepEngine(hp.ModelSpec(**C1_SPEC), hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                    hp.ExecConfig(compute="f32", device=rank, max_tokens=1024, max_batch=16, max_masks=256),
                    comm=comm, seed=21 if rank == 0 else None)
eng.broadcast_params(0)
eng.set_digest_check(1, debug=True)   # every update
rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
sched = hp.partition_for_rank(plan, world, rank)
out = {"clean": []}
for s in range(3):
    out["clean"].append(eng.round(rec.batch(plan.batches[sched[s].batch_index]), sched[s].dummy, 1e-3).loss)
# rank 1 drifts (parameters not broadcast): the next update's check fails on every rank
if rank == 1:
    p = eng.get_params().astype(np.float64)
    p[7] += 1e-3
    eng.set_params(p)
try:
    eng.round(rec.batch(plan.batches[sched[3].batch_index]), sched[3].dummy, 1e-3)
    out["drift"] = "accepted"
except hp.NumericError as e:
    out["drift"] = str(e)
with open(os.environ["HP_OUT"] + f"/dg{rank}.json", "w") as f:
    json.dump(out, f)
eng.close(); comm.close()
dist.destroy_process_group()
'''


def test_digest_cadence_check_detects_divergence(tmp_path):
    """check_digest_on_cadence (engine.hpp:170-184) inside round(): clean
    rounds pass; a rank whose parameters drifted makes every rank raise the
    reference's numeric error."""
    script = tmp_path / "digest_worker.py"
    script.write_text(DIGEST_WORKER)
    env = dict(os.environ, HP_ROOT=ROOT, HP_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29523", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    r0 = json.loads((tmp_path / "dg0.json").read_text())
    r1 = json.loads((tmp_path / "dg1.json").read_text())
    assert r0["clean"] == r1["clean"] and len(r0["clean"]) == 3
    for r in (r0, r1):
        assert "1 ranks diverged from master parameters at step 4" in r["drift"], r["drift"]


TRAIN_WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["HP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HP_ROOT"], "tests"))
import torch, torch.distributed as dist
import paper_2009_14783_b200 as hp
from helpers import C1_GEN, C1_SPEC
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(rank)
comm = hp.Communicator(world, rank, rank)
cfg = hp.EngineConfig(spec=hp.ModelSpec(**C1_SPEC), opt_kind="adam", sched=hp.SchedulerConfig("fixed", 1e-3),
                      seed=21, data_dir=os.environ["HP_SHARDS"], max_sentences=8, update_freq=1,
                      max_steps=10, checkpoint_dir=os.environ["HP_OUT"] + "/ck", debug_checks=True)
rep = hp.train_run(cfg, comm=comm, exec_cfg=hp.ExecConfig(compute="f32", device=rank))
with open(os.environ["HP_OUT"] + f"/tr{rank}.json", "w") as f:
    json.dump({"losses": [s.loss for s in rep.steps], "final_step": rep.final_step,
               "rank_seconds": [len(s.rank_seconds) for s in rep.steps]}, f)
comm.close()
dist.destroy_process_group()
'''


def test_train_run_w2_nccl_matches_reference(tmp_path):
    """The reference's train_run at W = 2 over NCCL (digest checked every
    update): the reference trajectory on both ranks, the final checkpoint
    written by rank 0 holding the reference's parameters."""
    from paper_2009_14783_b200 import api
    shards = tmp_path / "shards"
    api.write_mlm_shards(str(shards), api.generate_mlm_records(api.MlmGenConfig(**C1_GEN)), 4)
    script = tmp_path / "train_worker.py"
    script.write_text(TRAIN_WORKER)
    env = dict(os.environ, HP_ROOT=ROOT, HP_OUT=str(tmp_path), HP_SHARDS=str(shards))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29525", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    t = golden("c1_ref_train.npz")
    r0 = json.loads((tmp_path / "tr0.json").read_text())
    r1 = json.loads((tmp_path / "tr1.json").read_text())
    assert r0["losses"] == r1["losses"] and r0["final_step"] == 10
    assert np.max(np.abs(np.array(r0["losses"]) - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    assert r0["rank_seconds"] == [2] * 10 and r1["rank_seconds"] == [0] * 10
    _, meta, p, _, _ = api.read_checkpoint(str(tmp_path / "ck" / "checkpoint_final.hck"))
    assert meta.step == 10 and meta.world_size == 2
    assert rel_norm(p, t["params_f64_as_f32"]) <= 1e-4


BF16_WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["HP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HP_ROOT"], "tests"))
import torch, torch.distributed as dist
import paper_2009_14783_b200 as hp
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(rank)
comm = hp.Communicator(world, rank, rank)
# the benchmark's execution path at small scale: bf16 tcgen05 GEMMs and
# attention, weight-gradient stream, update stream, row-sparse embedding
# exchange (embedding alone in the last bucket), K = 2 accumulation
spec = hp.ModelSpec(arch="bert_encoder", d_model=128, heads=2, vocab=4000, max_seq=64, layers=2,
                    d_ff=256, label_smooth_eps=0.1)
rec = hp.generate_mlm_records(hp.MlmGenConfig(n=128, vocab=4000, min_sentence_words=10,
                                              max_sentence_words=30, seed=3, max_seq_tokens=64))
plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
sched = hp.partition_for_rank(plan, world, rank)
eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                    hp.ExecConfig(compute="bf16", device=rank, max_tokens=512, max_batch=8,
                                  max_masks=128, bucket_mb=0.5, update_freq=2),
                    comm=comm, seed=21 if rank == 0 else None)
eng.broadcast_params(0)
eng.set_digest_check(1, debug=True)
losses = []
for s in range(4):
    rep = eng.round(rec.batch(plan.batches[sched[s].batch_index]), sched[s].dummy, 1e-3)
    if rep is not None:
        losses.append(rep.loss)
# the pipelined API for the rest: rank_seconds gathered once for the call
reps = eng.rounds((rec.batch(plan.batches[sched[s].batch_index]), sched[s].dummy, 1e-3)
                  for s in range(4, 8))
losses += [r.loss for r in reps if r is not None]
out = {"losses": losses, "digest": eng.digest(),
       "rank_seconds": [len(r.rank_seconds) for r in reps if r is not None]}
with open(os.environ["HP_OUT"] + f"/bf{rank}.json", "w") as f:
    json.dump(out, f)
eng.close(); comm.close()
dist.destroy_process_group()
'''


def test_bf16_benchmark_path_w2_ranks_identical(tmp_path):
    """The benchmark's bf16 path at W = 2 with K = 2 (every stream, bucket and
    exchange of the C2 step at small scale): identical reports and parameters
    on both ranks, the digest checked on every update, a falling loss."""
    script = tmp_path / "bf16_worker.py"
    script.write_text(BF16_WORKER)
    env = dict(os.environ, HP_ROOT=ROOT, HP_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29527", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    r0 = json.loads((tmp_path / "bf0.json").read_text())
    r1 = json.loads((tmp_path / "bf1.json").read_text())
    assert len(r0["losses"]) == 4
    assert r0["losses"] == r1["losses"] and r0["digest"] == r1["digest"]
    assert r0["rank_seconds"] == [2, 2] and r1["rank_seconds"] == [0, 0]
    assert all(np.isfinite(r0["losses"]))
