"""Parity of the device step engine (C ABI, libhetpar_b200.so) with the
reference:

* C1 (reference masked_token_model): the 10-step trajectory of the
  reference's W=2 f64 run.  On one GPU the W=2 round is replayed as one rank
  holding both ranks' batches, which the protocol makes equivalent (loss sums,
  weights and gradients are additive; test_engine.cpp:183-235); the real
  2-process NCCL path is in test_gpu_multi.py.  Tolerances (norm-wise, see
  SURVEY §8c): per-step loss rel <= 1e-4, parameters ||dp||/||p|| <= 1e-4.
* per-rank pre-reduce gradients index-for-index vs the reference / oracle.
* the bert_encoder extension vs the numpy oracle (fp32 path) and the bf16
  tcgen05 path within bf16 tolerance.
* protocol edge cases: dummy rounds, all-dummy error, input validation.
"""
import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from helpers import C1_GEN, C1_SPEC, golden, oracle_instances, rel_norm

import model_oracle as mo

pytestmark = pytest.mark.gpu


def c1_engine(**kw):
    spec = hp.ModelSpec(**C1_SPEC)
    ex = hp.ExecConfig(compute="f32", max_tokens=1024, max_batch=16, max_masks=256, **kw)
    return hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9), ex, seed=21)


def c1_batches():
    rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
    plan = hp.build_epoch_batches(rec.token_lengths(), 8, 0, 21, 0)
    return rec, plan


def test_c1_trajectory_matches_reference_w2():
    rec, plan = c1_batches()
    t = golden("c1_ref_train.npz")
    eng = c1_engine()
    losses = []
    for step in range(10):
        r0 = hp.partition_for_rank(plan, 2, 0)[step]
        r1 = hp.partition_for_rank(plan, 2, 1)[step]
        ids = np.concatenate([plan.batches[r0.batch_index], plan.batches[r1.batch_index]])
        rep = eng.round(rec.batch(ids), dummy=False, lr=1e-3)
        assert rep.step == step + 1
        assert rep.weight == 16.0
        losses.append(rep.loss)
    losses = np.array(losses)
    assert np.max(np.abs(losses - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    p = eng.get_params()
    assert rel_norm(p, t["params_f64_as_f32"]) <= 1e-4
    # the reference's own f32 run is within the same tolerance of its f64 run
    assert rel_norm(t["params_f32"], t["params_f64_as_f32"]) <= 1e-5


def test_c1_local_gradients_index_for_index():
    rec, plan = c1_batches()
    g = golden("c1_ref_grads.npz")
    eng = c1_engine()
    eng.set_capture(True)
    for r in range(2):
        eng.set_params(hp.init_parameters(hp.ModelSpec(**C1_SPEC), 21))
        ids = g[f"rank{r}_ids"].astype(np.int64)
        assert np.array_equal(ids, plan.batches[r].astype(np.int64))
        rep = eng.round(rec.batch(ids), lr=0.0)
        local = eng.local_grads()
        assert abs(rep.local_loss_sum - g[f"rank{r}_lw"][0]) <= 1e-5 * g[f"rank{r}_lw"][0]
        assert rep.local_weight == g[f"rank{r}_lw"][1]
        sample = g[f"rank{r}_sample"]
        assert rel_norm(local[::37], sample) <= 1e-4
        assert abs(np.linalg.norm(local) - g[f"rank{r}_norm"][0]) <= 1e-4 * g[f"rank{r}_norm"][0]
        # the full vector against the (reference-pinned) numpy oracle
        s = mo.Spec()
        _, _, og = mo.forward_backward(s, mo.init_parameters(s, 21), oracle_instances(golden("c1_records.npz"), ids))
        assert rel_norm(local, og) <= 1e-4
        # per parameter block too: every bucket region matches
        for sh in hp.param_shapes(hp.ModelSpec(**C1_SPEC)):
            sl = slice(sh.offset, sh.offset + sh.size)
            if np.linalg.norm(og[sl]) > 1e-3:
                assert rel_norm(local[sl], og[sl]) <= 1e-3, sh.name


def test_dummy_round_is_neutral_and_all_dummy_fails():
    rec, plan = c1_batches()
    eng = c1_engine()
    p0 = eng.get_params()
    with pytest.raises(hp.NumericError, match="every rank was dummy"):
        eng.round(rec.batch(plan.batches[0]), dummy=True, lr=1e-3)
    assert np.array_equal(eng.get_params(), p0)
    assert eng.step == 0


def test_input_validation_matches_reference_errors():
    rec, plan = c1_batches()
    eng = c1_engine()
    b = rec.batch(plan.batches[0])
    bad = hp.BatchCSR(**{k: getattr(b, k).copy() for k in ("tok_off", "tokens", "segments", "mask_off", "mask_pos", "mask_orig", "label")})
    bad.tokens[3] = 1000
    with pytest.raises(hp.IndexError_):
        eng.stage(bad)
    bad = hp.BatchCSR(**{k: getattr(b, k).copy() for k in ("tok_off", "tokens", "segments", "mask_off", "mask_pos", "mask_orig", "label")})
    bad.segments[2] = 2
    with pytest.raises(hp.IndexError_):
        eng.stage(bad)
    bad = hp.BatchCSR(**{k: getattr(b, k).copy() for k in ("tok_off", "tokens", "segments", "mask_off", "mask_pos", "mask_orig", "label")})
    bad.mask_pos[0] = 63
    with pytest.raises(hp.IndexError_):
        eng.stage(bad)
    with pytest.raises(hp.ConfigError):
        eng.stage(hp.pack_batch([]))
    long = hp.Instance(np.arange(65) % 900 + 4, np.zeros(65, np.int64), np.array([1]), np.array([5]), 0)
    with pytest.raises(hp.ShapeError):
        eng.stage([long])


def test_digest_matches_fnv_over_params():
    eng = c1_engine()
    p = eng.get_params()
    h = 0xcbf29ce484222325
    for byte in p.tobytes()[:4096]:
        h ^= byte
        h = (h * 0x100000001b3) & (2**64 - 1)
    # full digest computed by the library; compare against a numpy FNV
    from helpers import oracle_lib
    import ctypes as C
    lib = oracle_lib()
    lib.orc_fnv1a64.restype = C.c_uint64
    raw = p.tobytes()
    want = lib.orc_fnv1a64(C.c_char_p(raw), C.c_uint64(len(raw)), C.c_uint64(0xcbf29ce484222325))
    assert eng.digest() == want


def _bert_case(d=64, heads=2, layers=2, dff=128, vocab=97, n=12, seed=3):
    spec = hp.ModelSpec(arch="bert_encoder", d_model=d, heads=heads, vocab=vocab, max_seq=32,
                        layers=layers, d_ff=dff, label_smooth_eps=0.1)
    ospec = mo.Spec(arch="bert_encoder", d_model=d, heads=heads, vocab=vocab, max_seq=32,
                    layers=layers, d_ff=dff, label_smooth_eps=0.1)
    rec = hp.generate_mlm_records(hp.MlmGenConfig(n=n, vocab=vocab, min_sentence_words=5,
                                                  max_sentence_words=12, seed=seed,
                                                  max_seq_tokens=32))
    return spec, ospec, rec


def _oracle_from_records(rec, ids):
    d = {k: getattr(rec, k) for k in ("tok_off", "tokens", "segments", "mask_off", "mask_pos", "mask_orig", "label")}
    return oracle_instances(d, ids)


def test_bert_extension_fp32_matches_oracle():
    spec, ospec, rec = _bert_case()
    eng = hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute="f32", max_tokens=512,
                                                               max_batch=16, max_masks=128), seed=9)
    eng.set_capture(True)
    ids = np.arange(8)
    rep = eng.round(rec.batch(ids), lr=0.0)
    p = mo.init_parameters(ospec, 9)
    l, w, g = mo.forward_backward(ospec, p, _oracle_from_records(rec, ids))
    assert abs(rep.local_loss_sum - l) <= 1e-4 * abs(l)
    assert rep.local_weight == w
    assert rel_norm(eng.local_grads(), g) <= 1e-4


def test_bert_extension_bf16_tcgen05_path():
    # dk = 64 so every GEMM takes the tcgen05 path
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=16)
    eng = hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute="bf16", max_tokens=512,
                                                               max_batch=16, max_masks=128), seed=9)
    eng.set_capture(True)
    ids = np.arange(12)
    rep = eng.round(rec.batch(ids), lr=0.0)
    p = mo.init_parameters(ospec, 9)
    l, w, g = mo.forward_backward(ospec, p, _oracle_from_records(rec, ids))
    assert abs(rep.local_loss_sum - l) <= 2e-2 * abs(l)
    assert rel_norm(eng.local_grads(), g) <= 5e-2
    # and a few steps train (loss decreases on a repeated batch)
    losses = [eng.round(rec.batch(ids), lr=1e-3).loss for _ in range(8)]
    assert losses[-1] < losses[0]


def _long_spec(max_seq=512):
    kw = dict(arch="bert_encoder", d_model=128, heads=2, vocab=203, max_seq=max_seq, layers=1,
              d_ff=256, label_smooth_eps=0.1)
    return hp.ModelSpec(**kw), mo.Spec(**kw)


def _check_long(spec, ospec, batch, oinst):
    eng = hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute="bf16", max_tokens=4096,
                                                               max_batch=16, max_masks=1024), seed=9)
    eng.set_capture(True)
    rep = eng.round(batch, lr=0.0)
    g = eng.local_grads()
    l, w, og = mo.forward_backward(ospec, mo.init_parameters(ospec, 9), oinst)
    assert abs(rep.local_loss_sum - l) <= 2e-2 * abs(l)
    assert rel_norm(g, og) <= 5e-2
    # every attention block on its own: a wrong dQ / dK / dV shows up here even
    # when the embedding / head gradients dominate the flat norm
    for p in hp.param_shapes(spec):
        if p.name.startswith("layer0.w"):
            sl = slice(p.offset, p.offset + p.size)
            assert rel_norm(g[sl], og[sl]) <= 5e-2, p.name
    eng.close()


def test_bert_long_sequences_tcgen05():
    """128 < seq <= 512 (C4's sequence length): the blocked tcgen05 attention
    (forward, dK/dV and dQ kernels) against the f64 oracle, with instances of
    every block count (<= 128, two, three and four 128-row blocks)."""
    spec, ospec = _long_spec()
    rec = hp.generate_mlm_records(hp.MlmGenConfig(n=24, vocab=203, min_sentence_words=20,
                                                  max_sentence_words=255, seed=4,
                                                  max_seq_tokens=512))
    ids = [3, 12, 2, 9, 16, 21, 1, 5]  # lengths 99, 153, 274, 409, 484, 97, 446, 218
    assert sorted(int(rec.token_lengths()[i]) for i in ids) == [97, 99, 153, 218, 274, 409, 446, 484]
    _check_long(spec, ospec, rec.batch(ids), _oracle_from_records(rec, ids))


def test_bert_long_sequences_block_edges():
    """Lengths on the 128-row block edges, up to the 512 cap."""
    spec, ospec = _long_spec()
    rng = np.random.default_rng(11)
    insts, oinst = [], []
    for n in (512, 129, 128, 257, 384, 385, 1 + 2):
        tok = rng.integers(4, 203, n)
        tok[0] = 0
        seg = (np.arange(n) >= n // 2).astype(np.int64)
        mp = np.sort(rng.choice(np.arange(1, n), size=max(1, n // 7), replace=False))
        mo_ = rng.integers(4, 203, len(mp))
        insts.append(hp.Instance(tok, seg, mp, mo_, int(n % 2)))
        oinst.append(mo.Instance(tok, seg, mp, mo_, int(n % 2)))
    _check_long(spec, ospec, hp.pack_batch(insts), oinst)


def test_long_sequences_need_the_bf16_path():
    spec, _ = _long_spec()
    with pytest.raises(hp.ConfigError):
        hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute="f32", max_tokens=1024,
                                                              max_batch=4, max_masks=64), seed=1)


@pytest.mark.parametrize("compute", ["bf16", "f32"])
def test_pipelined_rounds_equal_sequential_rounds(compute):
    """StepEngine.rounds (host staging of batch k+1 behind device round k) is
    the same computation as round() one at a time: identical losses and
    parameter bytes, batches of different shapes included."""
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=24)
    batches = [rec.batch(range(0, 8)), rec.batch(range(8, 14)), rec.batch(range(14, 24)),
               rec.batch(range(0, 8))]
    lrs = [1e-3, 2e-3, 1e-3, 5e-4]

    def make():
        return hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute=compute, max_tokens=1024,
                                                                   max_batch=16, max_masks=256), seed=9)
    a = make()
    la = [a.round(b, lr=lr).loss for b, lr in zip(batches, lrs)]
    da = a.digest()
    a.close()
    b = make()
    lb = [r.loss for r in b.rounds((x, False, lr) for x, lr in zip(batches, lrs))]
    assert la == lb
    assert b.digest() == da
    b.close()


def test_timer_pass_is_the_same_computation():
    """The timer pass (event pairs captured into the round's graph) runs the
    same kernels: identical losses and parameters to an untimed run, and every
    class reports time for the launches it counted."""
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=16)
    b = rec.batch(range(12))

    def run(timed):
        eng = hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute="bf16", max_tokens=512,
                                                                   max_batch=16, max_masks=128), seed=9)
        eng.timers(timed)
        losses = [eng.round(b, lr=1e-3).loss for _ in range(5)]
        t = [eng.timer(i) for i in range(6)]
        d = eng.digest()
        eng.close()
        return losses, d, t
    la, da, _ = run(False)
    lb, db, t = run(True)
    assert la == lb and da == db
    g = t[0]
    assert g["name"] == "gemm" and g["launches"] > 0 and g["ms"] > 0 and g["flops"] > 0


def _graph_run(monkeypatch, graphs, make_engine, batches, lrs):
    monkeypatch.setenv("HP_GRAPHS", "1" if graphs else "0")
    eng = make_engine()
    k0 = eng.kernel_launches()
    losses = [eng.round(b, lr=lr).loss for b, lr in zip(batches, lrs)]
    return np.array(losses), eng.digest(), eng.kernel_launches() - k0


@pytest.mark.parametrize("compute", ["bf16", "f32"])
def test_graph_replay_bit_identical_to_eager(monkeypatch, compute):
    # Two batch shapes alternate, so each shape runs eagerly, is captured on
    # its second sighting and replayed after that; the learning rate changes
    # every step (it reaches the captured Adam through device memory).
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=16)

    def make():
        return hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(
            compute=compute, max_tokens=512, max_batch=16, max_masks=128), seed=9)

    ids = [np.arange(12), np.arange(2, 14)]
    batches = [rec.batch(ids[k % 2]) for k in range(7)]
    lrs = [1e-3 * (1 + 0.5 * k) for k in range(7)]
    lg, dg, ng = _graph_run(monkeypatch, True, make, batches, lrs)
    le, de, ne = _graph_run(monkeypatch, False, make, batches, lrs)
    assert np.array_equal(lg, le)
    assert dg == de
    assert ng == ne  # replays account for the kernels inside the graph


def test_c1_k2_accumulation_matches_reference_w2():
    # W*K equivalence (test_engine.cpp:237-294, acceptance criterion 2): one
    # rank with update_freq = 2 fed rank 0's then rank 1's batch reproduces the
    # reference's W = 2, K = 1 trajectory; the first round of each group
    # returns no report and does not advance the step.
    rec, plan = c1_batches()
    t = golden("c1_ref_train.npz")
    eng = c1_engine(update_freq=2)
    losses = []
    for step in range(10):
        r0 = hp.partition_for_rank(plan, 2, 0)[step]
        r1 = hp.partition_for_rank(plan, 2, 1)[step]
        assert eng.round(rec.batch(plan.batches[r0.batch_index]), lr=1e-3) is None
        rep = eng.round(rec.batch(plan.batches[r1.batch_index]), lr=1e-3)
        assert rep is not None and rep.step == step + 1
        assert rep.weight == 16.0
        losses.append(rep.loss)
    losses = np.array(losses)
    assert np.max(np.abs(losses - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    assert rel_norm(eng.get_params(), t["params_f64_as_f32"]) <= 1e-4


@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_k3_accumulation_equals_combined_batch(compute):
    # K = 3 rounds over batches a, b, c == one K = 1 round over a + b + c
    # (sums stay raw until the flush; the update divides by the total weight)
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=24)
    mk = lambda k: hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(
        compute=compute, max_tokens=1024, max_batch=24, max_masks=256, update_freq=k), seed=9)
    parts = [np.arange(0, 6), np.arange(6, 14), np.arange(14, 20)]
    ek, e1 = mk(3), mk(1)
    for rnd in range(2):
        reps = [ek.round(rec.batch(p), lr=1e-3) for p in parts]
        assert reps[0] is None and reps[1] is None and reps[2].step == rnd + 1
        ref = e1.round(rec.batch(np.concatenate(parts)), lr=1e-3)
        assert abs(reps[2].weight - ref.weight) == 0
        assert abs(reps[2].loss - ref.loss) <= (1e-6 if compute == "f32" else 2e-2) * abs(ref.loss)
    tol = 1e-5 if compute == "f32" else 2e-2
    assert rel_norm(ek.get_params(), e1.get_params()) <= tol


def _hck1_run():
    import json
    import os
    d = os.path.join(os.path.dirname(__file__), "golden", "hck1")
    run = json.load(open(os.path.join(d, "run.json")))
    c = run["config"]
    rec = hp.generate_mlm_records(hp.MlmGenConfig(
        n=c["n"], vocab=c["vocab"], docs=c["docs"], sentences_per_doc=c["spd"],
        min_sentence_words=c["min_words"], max_sentence_words=c["max_words"], seed=c["data_seed"]))
    plan = hp.build_epoch_batches(rec.token_lengths(), c["max_sentences"], 0, c["seed"], 0)
    return d, run, c, rec, plan


def test_resume_from_reference_checkpoint():
    # load the reference's step-2 HCK1 into device state, run updates 3-4 of
    # the same W=2 schedule (both ranks' batches in one round), and land on
    # the reference's final checkpoint; then save and read back.
    import os
    from paper_2009_14783_b200.api import read_checkpoint
    d, run, c, rec, plan = _hck1_run()
    spec, meta, p2, _, _ = read_checkpoint(os.path.join(d, "checkpoint_000002.hck"))
    eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9), hp.ExecConfig(
        compute="f32", max_tokens=2048, max_batch=16, max_masks=512))
    m = eng.load_checkpoint(os.path.join(d, "checkpoint_000002.hck"))
    assert m.step == 2 and m.opt_t == 2 and eng.step_count() == 2
    assert np.array_equal(eng.get_params(), p2)
    e, skip = hp.api.resume_position(rec.token_lengths(), c["max_sentences"], 0, c["seed"], 2, 1, 2)
    assert (e, skip) == (0, 2)
    losses = []
    for rnd in range(skip, skip + 2):
        r0 = hp.partition_for_rank(plan, 2, 0)[rnd]
        r1 = hp.partition_for_rank(plan, 2, 1)[rnd]
        ids = np.concatenate([plan.batches[r0.batch_index], plan.batches[r1.batch_index]])
        losses.append(eng.round(rec.batch(ids), lr=c["lr"]).loss)
    assert np.max(np.abs(np.array(losses) - run["losses"][2:]) / np.abs(run["losses"][2:])) <= 1e-4
    _, mf, pf, _, _ = read_checkpoint(os.path.join(d, "checkpoint_final.hck"))
    assert rel_norm(eng.get_params(), pf) <= 1e-4
    out = os.path.join(os.environ.get("TMPDIR", "/tmp"), "hp_resume_test.hck")
    eng.save_checkpoint(out, hp.api.CheckpointMeta(epoch=0, seed=c["seed"], world_size=2))
    _, ms, ps, mm, vv = read_checkpoint(out)
    assert ms.step == 4 and ms.opt_t == 4 and np.array_equal(ps, eng.get_params())
    em, ev, et = eng.get_adam()
    assert np.array_equal(mm, em) and np.array_equal(vv, ev) and et == 4


@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_save_load_resume_is_bit_exact(compute):
    # acceptance criterion 4 (resume determinism): 4 updates straight ==
    # 2 updates, save, a fresh engine loads, 2 more updates -- same bytes
    import os
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=16)
    mk = lambda: hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(
        compute=compute, max_tokens=512, max_batch=16, max_masks=128), seed=9)
    batches = [rec.batch(np.arange(k, k + 8)) for k in (0, 4, 8, 2)]
    a = mk()
    for b in batches:
        a.round(b, lr=1e-3)
    f = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"hp_resume_{compute}.hck")
    b1 = mk()
    for b in batches[:2]:
        b1.round(b, lr=1e-3)
    b1.save_checkpoint(f, hp.api.CheckpointMeta(seed=9))
    b2 = hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(
        compute=compute, max_tokens=512, max_batch=16, max_masks=128))
    assert b2.load_checkpoint(f).step == 2
    for b in batches[2:]:
        rep = b2.round(b, lr=1e-3)
    assert rep.step == 4
    assert b2.digest() == a.digest()


def test_c1_trained_from_shards_matches_reference(tmp_path):
    # the HSD1 read path end to end: C1 records -> shard files -> one
    # prefetching loader per rank -> pinned staging -> HBM; W = 2 replayed on
    # one GPU as K = 2 (rank 0's batch, then rank 1's), against the
    # reference's W = 2 trajectory
    from paper_2009_14783_b200 import api
    rec = hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN))
    api.write_mlm_shards(str(tmp_path), rec, 4)
    ds = api.ShardDataset(str(tmp_path))
    plan = hp.build_epoch_batches(ds.token_lengths(), 8, 0, 21, 0)
    loaders = [ds.loader(plan, hp.partition_for_rank(plan, 2, r), 2) for r in range(2)]
    t = golden("c1_ref_train.npz")
    eng = c1_engine(update_freq=2)
    losses = []
    for step in range(10):
        assert eng.round(loaders[0].next(), lr=1e-3) is None
        rep = eng.round(loaders[1].next(), lr=1e-3)
        losses.append(rep.loss)
    assert np.max(np.abs(np.array(losses) - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    assert rel_norm(eng.get_params(), t["params_f64_as_f32"]) <= 1e-4


def _c1_run_config(tmp_path, **kw):
    from paper_2009_14783_b200 import api
    d = tmp_path / "shards"
    if not d.exists():
        api.write_mlm_shards(str(d), hp.generate_mlm_records(hp.MlmGenConfig(**C1_GEN)), 4)
    base = dict(spec=hp.ModelSpec(**C1_SPEC), opt_kind="adam", beta1=0.9, beta2=0.98, eps=1e-9,
                sched=hp.SchedulerConfig("fixed", 1e-3), seed=21, data_dir=str(d), max_sentences=8,
                update_freq=2, max_steps=10)
    base.update(kw)
    return hp.EngineConfig(**base)


def test_train_run_matches_reference_trajectory(tmp_path):
    """train_run (engine.hpp:197-330) end to end on one GPU -- shards, epoch
    plans, the rank's loader, scheduled lr, the update protocol -- at W = 1,
    K = 2, which is the reference's W = 2 run (W x K equivalence)."""
    rep = hp.train_run(_c1_run_config(tmp_path), exec_cfg=hp.ExecConfig(compute="f32"))
    t = golden("c1_ref_train.npz")
    losses = np.array([s.loss for s in rep.steps])
    assert rep.steps_run == 10 and rep.final_step == 10 and rep.world == 1
    assert [s.step for s in rep.steps] == list(range(1, 11))
    assert np.max(np.abs(losses - t["losses_f64"]) / np.abs(t["losses_f64"])) <= 1e-4
    assert rep.final_loss == rep.steps[-1].loss


def test_train_run_checkpoint_resume_is_exact(tmp_path):
    """Checkpoints every 4 updates and at the end; resuming from step 4
    (resume fast-forward, engine.hpp:211-245) reaches the same final state
    bit for bit."""
    from paper_2009_14783_b200 import api
    ck_a, ck_b = tmp_path / "a", tmp_path / "b"
    ra = hp.train_run(_c1_run_config(tmp_path, checkpoint_dir=str(ck_a), checkpoint_interval=4),
                      exec_cfg=hp.ExecConfig(compute="f32"))
    assert (ck_a / "checkpoint_000004.hck").exists() and (ck_a / "checkpoint_000008.hck").exists()
    rb = hp.train_run(_c1_run_config(tmp_path, checkpoint_dir=str(ck_b),
                                     resume_path=str(ck_a / "checkpoint_000004.hck")),
                      exec_cfg=hp.ExecConfig(compute="f32"))
    assert [s.step for s in rb.steps] == list(range(5, 11))
    assert [s.loss for s in rb.steps] == [s.loss for s in ra.steps[4:]]
    _, _, pa, ma, va = api.read_checkpoint(str(ck_a / "checkpoint_final.hck"))
    _, _, pb, mb, vb = api.read_checkpoint(str(ck_b / "checkpoint_final.hck"))
    assert np.array_equal(pa, pb) and np.array_equal(ma, mb) and np.array_equal(va, vb)


@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_forward_only_matches_oracle_and_round(compute):
    """StepEngine.forward = model_forward: the batch's summed loss and weight
    without an update (parameters unchanged), equal to the oracle's and to
    the local loss a round reports."""
    spec, ospec, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=16)
    eng = hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(compute=compute, max_tokens=512,
                                                               max_batch=16, max_masks=128), seed=9)
    ids = np.arange(12)
    d0 = eng.digest()
    ls, w = eng.forward(rec.batch(ids))
    assert eng.digest() == d0 and eng.step == 0
    l, ow, _ = mo.forward_backward(ospec, mo.init_parameters(ospec, 9), _oracle_from_records(rec, ids),
                                   need_grad=False)
    tol = 1e-4 if compute == "f32" else 2e-2
    assert abs(ls - l) <= tol * abs(l) and w == ow
    rep = eng.round(rec.batch(ids), lr=1e-3)
    assert rep.local_loss_sum == pytest.approx(ls, rel=1e-6)
    eng.close()


def _split_run(monkeypatch, split, make_engine, batches, lrs):
    monkeypatch.setenv("HP_EMB_SPLIT", "1" if split else "0")
    eng = make_engine()
    k0 = eng.kernel_launches()
    losses = [eng.round(b, lr=lr).loss for b, lr in zip(batches, lrs)]
    launches = eng.kernel_launches() - k0
    m, v, t = eng.get_adam()
    out = (np.array(losses), eng.digest(), eng.get_params(), m.copy(), v.copy(), t, launches)
    eng.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("arch,compute", [("bert_encoder", "bf16"), ("bert_encoder", "f32"),
                                          ("masked_token_model", "f32")])
def test_split_embedding_update_bit_identical(monkeypatch, arch, compute):
    # W = 1, K = 1: the word-embedding rows outside the batch's ids are updated
    # with a zero gradient while backward runs, the batch's rows after it
    # (adam_rows); parameters, Adam state and losses must equal the dense
    # update's bit for bit, eager and graph-replayed rounds alike.
    if arch == "bert_encoder":
        spec, _, rec = _bert_case(d=128, heads=2, dff=256, vocab=203, n=16)
    else:
        spec = hp.ModelSpec(arch="masked_token_model", d_model=128, heads=4, vocab=1000,
                            max_seq=64, label_smooth_eps=0.1)
        rec = hp.generate_mlm_records(hp.MlmGenConfig(n=16, vocab=1000, min_sentence_words=30,
                                                      max_sentence_words=30, seed=7))

    def make():
        return hp.StepEngine(spec, hp.OptimConfig(), hp.ExecConfig(
            compute=compute, max_tokens=1024, max_batch=16, max_masks=256), seed=9)

    ids = [np.arange(12), np.arange(2, 14)]
    batches = [rec.batch(ids[k % 2]) for k in range(6)]
    lrs = [1e-3 * (1 + 0.5 * k) for k in range(6)]
    a = _split_run(monkeypatch, True, make, batches, lrs)
    b = _split_run(monkeypatch, False, make, batches, lrs)
    assert np.array_equal(a[0], b[0])
    assert a[1] == b[1]
    for x, y in zip(a[2:5], b[2:5]):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert a[5] == b[5]
    assert a[6] == b[6] + 2 * len(batches)  # the split ran: two adam_rows launches per round


def test_pipelined_rounds_report_the_first_error_and_roll_back():
    """round_async pipelining (bench.py's value pass) with a failing round in
    the middle: round_sync raises the FIRST error (engine.hpp:134-137), the
    rounds after it do not update, and step / Adam t return to the failing
    round's entry state -- parameters equal one clean round, bit for bit."""
    rec, plan = c1_batches()
    b = rec.batch(plan.batches[0])
    ref = c1_engine()
    ref.round(b, lr=1e-3)
    want = ref.get_params()
    eng = c1_engine()
    eng.stage(b)
    eng.round_async(False, 1e-3)
    eng.round_async(True, 1e-3)    # every rank dummy: total weight 0
    eng.round_async(False, 1e-3)   # must not update after the error
    with pytest.raises(hp.NumericError, match="every rank was dummy"):
        eng.round_sync()
    assert eng.step == 1
    assert eng.get_adam()[2] == 1
    assert np.array_equal(eng.get_params().view(np.uint32), want.view(np.uint32))
    # the engine carries on from there
    rep = eng.round(b, lr=1e-3)
    ref.round(b, lr=1e-3)
    assert rep.step == 2 and np.array_equal(eng.get_params(), ref.get_params())


def test_train_run_partial_accumulation_at_run_end_still_checkpoints(tmp_path, capfd):
    """an epochs-bounded run with update_freq = 2 and an odd number
    of rounds ends inside an update group; like the reference's train_run
    (engine.hpp:310-314) it warns, discards the pending round and still writes
    checkpoint_final with the last update's state."""
    from paper_2009_14783_b200 import api
    cfg = _c1_run_config(tmp_path, max_sentences=7, max_steps=1000, max_epochs=1,
                         checkpoint_dir=str(tmp_path / "ck"))
    rep = hp.train_run(cfg, exec_cfg=hp.ExecConfig(compute="f32"))
    assert rep.final_step == 11  # 23 rounds -> 11 updates + 1 pending
    assert "discarding a partial accumulation of 1 rounds" in capfd.readouterr().err
    _, meta, p, _, _ = api.read_checkpoint(str(tmp_path / "ck" / "checkpoint_final.hck"))
    assert meta.step == 11 and meta.opt_t == 11


def test_resume_takes_the_optimizer_from_the_checkpoint(tmp_path):
    """resuming an Adam checkpoint with a config that says SGD and
    other betas continues with the file's Adam (kind, betas, eps), as the
    reference's load_checkpoint does (checkpoint.cpp:254, 282-289)."""
    ck = tmp_path / "a"
    ra = hp.train_run(_c1_run_config(tmp_path, checkpoint_dir=str(ck), checkpoint_interval=4),
                      exec_cfg=hp.ExecConfig(compute="f32"))
    rb = hp.train_run(_c1_run_config(tmp_path, opt_kind="sgd", beta1=0.5, beta2=0.5, eps=1e-3,
                                     resume_path=str(ck / "checkpoint_000004.hck")),
                      exec_cfg=hp.ExecConfig(compute="f32"))
    assert [s.loss for s in rb.steps] == [s.loss for s in ra.steps[4:]]


def test_adamw_trajectory_and_checkpoint(tmp_path):
    """AdamW (extension; north_star's "fused multi-tensor Adam/AdamW"): the
    engine's 3-update fp32 trajectory equals the oracle's (decoupled decay,
    then the reference's Adam) at the parity tolerance, and the optimizer
    round-trips through an HCK1 checkpoint (kind "adamw", weight_decay)."""
    from paper_2009_14783_b200.api import read_checkpoint
    rec, plan = c1_batches()
    spec = hp.ModelSpec(**C1_SPEC)
    opt = hp.OptimConfig("adamw", 0.9, 0.98, 1e-9, weight_decay=0.05)
    eng = hp.StepEngine(spec, opt, hp.ExecConfig(compute="f32", max_tokens=1024, max_batch=16,
                                                  max_masks=256), seed=21)
    s = mo.Spec()
    p = mo.init_parameters(s, 21).astype(np.float32)
    st = mo.AdamState()
    for k in range(3):
        b = plan.batches[k]
        rep = eng.round(rec.batch(b), lr=1e-3)
        l, w, g = mo.forward_backward(s, p.astype(np.float64), oracle_instances(golden("c1_records.npz"), b))
        p = mo.adam_step(p, g / w, st, 1e-3, np.float32, weight_decay=0.05)
        assert abs(rep.loss - l / w) <= 1e-4 * abs(l / w)
    assert rel_norm(eng.get_params(), p) <= 1e-4
    f = str(tmp_path / "adamw.hck")
    eng.save_checkpoint(f, hp.api.CheckpointMeta(seed=21))
    _, meta, pp, mm, vv = read_checkpoint(f)
    assert meta.optimizer == "adamw" and meta.weight_decay == 0.05 and meta.opt_t == 3
    e2 = hp.StepEngine(spec, hp.OptimConfig("sgd"), hp.ExecConfig(compute="f32", max_tokens=1024,
                                                                  max_batch=16, max_masks=256))
    e2.load_checkpoint(f)
    assert e2.optim.kind == "adamw" and e2.optim.weight_decay == 0.05
    b = plan.batches[3]
    r1, r2 = eng.round(rec.batch(b), lr=1e-3), e2.round(rec.batch(b), lr=1e-3)
    assert r1.loss == r2.loss and eng.digest() == e2.digest()
