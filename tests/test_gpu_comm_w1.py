"""The collective path on ONE GPU: a real NCCL communicator of world 1.

Every NCCL call the engine makes at W > 1 is issued here too -- the
pre-backward [loss, weight] allreduce (engine.hpp:133), the bucketed gradient
allreduce (engine.hpp:145; small buckets so there are many), the digest
broadcast + mismatch allreduce of check_digest_on_cadence (engine.hpp:170-184),
the row-sparse word-embedding allgather, the parameter broadcast
(engine.hpp:263) and the NcclProcessGroup control plane (comm.hpp:16-49) --
so a 1-GPU box exercises them.  The W = 2 versions stay in test_gpu_multi.py.
"""
import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from helpers import C1_GEN, C1_SPEC, golden, rel_norm

pytestmark = pytest.mark.gpu


@pytest.fixture
def comm():
    c = hp.Communicator(1, 0, 0)
    yield c
    c.close()


def _c1():
    rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
    plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
    return rec, plan


@pytest.mark.parametrize("K", [1, 2])
def test_c1_trajectory_through_nccl_w1(comm, K):
    """The reference's W = 2 C1 trajectory on one rank that holds both ranks'
    batches (K = 1) or takes them as two accumulated rounds (K = 2), every
    round through NCCL: loss allreduce, 0.3 MB gradient buckets, the
    broadcast of rank 0's parameters and the digest check on every update."""
    rec, plan = _c1()
    t = golden("c1_ref_train.npz")
    eng = hp.StepEngine(hp.ModelSpec(**C1_SPEC), hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                        hp.ExecConfig(compute="f32", max_tokens=1024, max_batch=16, max_masks=256,
                                      bucket_mb=0.3, update_freq=K), comm=comm, seed=21)
    assert len(hp.bucket_plan(hp.ModelSpec(**C1_SPEC), 0.3)) > 3
    eng.broadcast_params(0)
    eng.set_digest_check(1, debug=True)
    losses = []
    for step in range(10):
        r0 = hp.partition_for_rank(plan, 2, 0)[step]
        r1 = hp.partition_for_rank(plan, 2, 1)[step]
        if K == 1:
            ids = np.concatenate([plan.batches[r0.batch_index], plan.batches[r1.batch_index]])
            rep = eng.round(rec.batch(ids), dummy=False, lr=1e-3)
        else:
            assert eng.round(rec.batch(plan.batches[r0.batch_index]), lr=1e-3) is None
            rep = eng.round(rec.batch(plan.batches[r1.batch_index]), lr=1e-3)
        assert rep.step == step + 1 and rep.weight == 16.0
        assert rep.rank_seconds == [rep.seconds]
        losses.append(rep.loss)
    losses = np.array(losses)
    assert np.max(np.abs(losses - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    assert rel_norm(eng.get_params(), t["params_f64_as_f32"]) <= 1e-4
    eng.close()


def test_nccl_w1_equals_no_communicator():
    """With a world-1 communicator the engine computes exactly what it
    computes without one (a one-rank sum is the identity): same losses, same
    parameter bytes, bf16 benchmark path with every stream."""
    spec = hp.ModelSpec(arch="bert_encoder", d_model=128, heads=2, vocab=4000, max_seq=64, layers=2,
                        d_ff=256, label_smooth_eps=0.1)
    rec = hp.generate_mlm_records(hp.MlmGenConfig(n=64, vocab=4000, min_sentence_words=10,
                                                  max_sentence_words=30, seed=3, max_seq_tokens=64))
    plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)

    def run(c):
        eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                            hp.ExecConfig(compute="bf16", max_tokens=512, max_batch=8, max_masks=128,
                                          bucket_mb=0.5), comm=c, seed=21)
        if c:
            eng.set_digest_check(1, debug=True)
        losses = [eng.round(rec.batch(plan.batches[s]), lr=1e-3).loss for s in range(4)]
        d = eng.digest()
        eng.close()
        return losses, d
    c = hp.Communicator(1, 0, 0)
    a = run(c)
    c.close()
    b = run(None)
    assert a == b


def test_sparse_embedding_exchange_w1(monkeypatch):
    """The row-sparse word-embedding exchange (allgather of (id, row) slots +
    rank-ordered scatter, issue_bucket) forced on at world 1 trains like the
    dense bucket allreduce; dummy rounds (an empty row set) included."""
    spec = hp.ModelSpec(arch="bert_encoder", d_model=128, heads=2, vocab=4000, max_seq=64, layers=1,
                        d_ff=256, label_smooth_eps=0.1)
    rec = hp.generate_mlm_records(hp.MlmGenConfig(n=64, vocab=4000, min_sentence_words=10,
                                                  max_sentence_words=30, seed=3, max_seq_tokens=64))
    plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("HP_SPARSE_EMB", mode)
        c = hp.Communicator(1, 0, 0)
        eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9),
                            hp.ExecConfig(compute="f32", max_tokens=512, max_batch=8, max_masks=128,
                                          bucket_mb=0.5), comm=c, seed=21)
        losses = [eng.round(rec.batch(plan.batches[s]), lr=1e-3).loss for s in range(4)]
        # a dummy round next to a real one is impossible at W = 1 (the total
        # weight would be 0): K = 1 dummy must raise, parameters untouched
        p = eng.get_params()
        with pytest.raises(hp.NumericError, match="every rank was dummy"):
            eng.round(rec.batch(plan.batches[0]), dummy=True, lr=1e-3)
        assert np.array_equal(eng.get_params(), p)
        out[mode] = (np.array(losses), p)
        eng.close()
        c.close()
    assert np.max(np.abs(out["1"][0] - out["0"][0]) / np.abs(out["0"][0])) <= 1e-5
    assert rel_norm(out["1"][1], out["0"][1]) <= 1e-5


def test_process_group_contract_w1():
    """NcclProcessGroup (comm.hpp:16-49) on a TCP-formed world of one:
    broadcast returns the root's bytes, all_reduce_sum the input, the master
    gathers its own scalar, barrier returns, and a bad root is an error."""
    c = hp.Communicator.tcp("127.0.0.1", 29541, 1, 0, 0)
    assert c.broadcast(b"payload \x00\xff", root=0) == b"payload \x00\xff"
    assert c.all_reduce_sum([1e16, 1.0, 0.1]) == [1e16, 1.0, 0.1]
    assert c.gather_scalars(7.5) == [7.5]
    c.barrier()
    with pytest.raises(hp.BaseError):
        c.broadcast(b"x", root=1)
    ar = c.allreduce_bench(1 << 22, 1.0, iters=2, warmup=1)
    assert ar["ms"] > 0
    c.close()


def test_train_run_through_nccl_w1(tmp_path):
    """train_run (engine.hpp:197-330) with a world-1 communicator, the digest
    checked every update: the reference's W = 2 trajectory at K = 2."""
    from paper_2009_14783_b200 import api
    d = tmp_path / "shards"
    api.write_mlm_shards(str(d), hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN)), 4)
    cfg = hp.EngineConfig(spec=hp.ModelSpec(**C1_SPEC), opt_kind="adam", beta1=0.9, beta2=0.98,
                          eps=1e-9, sched=hp.SchedulerConfig("fixed", 1e-3), seed=21,
                          data_dir=str(d), max_sentences=8, update_freq=2, max_steps=10,
                          checkpoint_dir=str(tmp_path / "ck"), debug_checks=True)
    c = hp.Communicator(1, 0, 0)
    rep = hp.train_run(cfg, comm=c, exec_cfg=hp.ExecConfig(compute="f32"))
    c.close()
    t = golden("c1_ref_train.npz")
    losses = np.array([s.loss for s in rep.steps])
    assert rep.final_step == 10
    assert np.max(np.abs(losses - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    _, meta, p, _, _ = api.read_checkpoint(str(tmp_path / "ck" / "checkpoint_final.hck"))
    assert meta.step == 10 and rel_norm(p, t["params_f64_as_f32"]) <= 1e-4
