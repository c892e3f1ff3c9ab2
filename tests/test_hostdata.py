"""Product host data path (libhetpar_b200.so) vs the reference fixtures and
the oracle: bit-exact shard indexing, record stream, init, bucket layout."""
import os
import re

import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from paper_2009_14783_b200 import _lib
from helpers import C1_GEN, RECORD_KEYS, ROOT, golden, oracle_records

import model_oracle as mo


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hetpar_b200.h")).read()
    declared = set(re.findall(r"^(?:hp_status|const char\*)\s+(hp_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert set(_lib.EXPORTED) >= declared


def test_splitmix_and_shuffle_golden():
    g = golden("rng_golden.npz")
    assert np.array_equal(hp.splitmix64(0, 1000), g["seed_0"])
    assert np.array_equal(hp.splitmix64(1, 1000), g["seed_1"])
    assert np.array_equal(hp.splitmix64(2**64 - 1, 1000), g["seed_max"])
    assert np.array_equal(hp.shuffle_iota(42, 10), g["fisher_yates_n10_seed42"])
    assert len(hp.shuffle_iota(1, 0)) == 0 and list(hp.shuffle_iota(1, 1)) == [0]


@pytest.mark.parametrize("fixture,cfg", [
    ("c1_records.npz", hp.MlmGenConfig(**C1_GEN)),
    ("ragged_records.npz", hp.MlmGenConfig(n=97, vocab=64, min_sentence_words=3,
                                           max_sentence_words=8, seed=11)),
])
def test_record_stream_bit_exact(fixture, cfg):
    want = golden(fixture)
    got = hp.generate_mlm_records(cfg)
    for k in RECORD_KEYS:
        assert np.array_equal(getattr(got, k).astype(np.int64), want[k].astype(np.int64)), k
    assert np.array_equal(got.token_lengths(), want["lens"])


def test_truncation_extension_matches_oracle_and_is_exact_length():
    cfg = hp.MlmGenConfig(n=50, vocab=30522, min_sentence_words=64, max_sentence_words=80,
                          seed=7, max_seq_tokens=128)
    got = hp.generate_mlm_records(cfg)
    assert set(got.token_lengths().tolist()) == {128}
    want = oracle_records(50, 30522, 64, 80, 7, max_seq_tokens=128)
    for k in RECORD_KEYS:
        assert np.array_equal(getattr(got, k).astype(np.int64), want[k].astype(np.int64)), k


def test_plans_bit_exact():
    p = golden("plans.npz")
    recs = {"c1": golden("c1_records.npz"), "c1e3": golden("c1_records.npz"),
            "ragged_tok": golden("ragged_records.npz"), "ragged_w3": golden("ragged_records.npz")}
    for name, rec in recs.items():
        ms, mt, seed, ep, w = [int(x) for x in p[name + "_args"]]
        plan = hp.build_epoch_batches(rec["lens"], ms, mt, seed, ep)
        assert np.array_equal(np.concatenate(plan.batches), p[name + "_order"])
        assert np.array_equal([len(b) for b in plan.batches], p[name + "_sizes"])
        for r in range(w):
            s = hp.partition_for_rank(plan, w, r)
            assert np.array_equal([x.batch_index for x in s], p[f"{name}_rank{r}_batch"])
            assert np.array_equal([x.dummy for x in s], p[f"{name}_rank{r}_dummy"].astype(bool))


def test_batching_errors_and_edges():
    with pytest.raises(hp.ConfigError):
        hp.build_epoch_batches([4, 11, 2], 0, 10, 1, 0)
    assert len(hp.build_epoch_batches([4, 11, 2], 0, 0, 1, 0).batches) == 1
    assert hp.build_epoch_batches([], 4, 0, 1, 0).batches == []
    plan = hp.build_epoch_batches([1] * 5, 2, 0, 42, 0)
    with pytest.raises(hp.ConfigError):
        hp.partition_for_rank(plan, 0, 0)
    with pytest.raises(hp.ConfigError):
        hp.partition_for_rank(plan, 2, 2)
    with pytest.raises(hp.ConfigError):
        hp.partition_for_rank(hp.BatchPlan(0, []), 2, 0)


def test_generator_config_errors():
    with pytest.raises(hp.ConfigError):
        hp.generate_mlm_records(hp.MlmGenConfig(n=3, vocab=5))
    with pytest.raises(hp.ConfigError):
        hp.generate_mlm_records(hp.MlmGenConfig(n=3, min_sentence_words=0))
    with pytest.raises(hp.ConfigError):
        hp.generate_mlm_records(hp.MlmGenConfig(n=3, docs=1))


def test_param_table_matches_reference_order():
    spec = hp.ModelSpec(**{k: v for k, v in dict(arch="masked_token_model", d_model=128, heads=4,
                                                 vocab=1000, max_seq=64).items()})
    shapes = hp.param_shapes(spec)
    ms = mo.param_shapes(mo.Spec())
    assert [(s.name, s.rows, s.cols) for s in shapes] == [(n, r, c) for n, r, c, _, _ in ms]
    assert hp.flat_size(spec) == 323050
    bs = hp.ModelSpec(arch="bert_encoder", d_model=16, heads=2, vocab=30, max_seq=8, layers=2, d_ff=24)
    ob = mo.Spec(arch="bert_encoder", d_model=16, heads=2, vocab=30, max_seq=8, layers=2, d_ff=24)
    assert [(s.name, s.rows, s.cols) for s in hp.param_shapes(bs)] == \
           [(n, r, c) for n, r, c, _, _ in mo.param_shapes(ob)]
    with pytest.raises(hp.ConfigError):
        hp.param_shapes(hp.ModelSpec(d_model=130, heads=4))
    with pytest.raises(hp.ConfigError):
        hp.param_shapes(hp.ModelSpec(label_smooth_eps=1.0))


def test_init_bit_exact():
    spec = hp.ModelSpec()
    p = hp.init_parameters(spec, 21)
    assert np.array_equal(p[::101], golden("c1_ref_train.npz")["init_params_f64"])
    assert np.array_equal(p, mo.init_parameters(mo.Spec(), 21))
    bs = hp.ModelSpec(arch="bert_encoder", d_model=16, heads=2, vocab=30, max_seq=8, layers=2, d_ff=24)
    ob = mo.Spec(arch="bert_encoder", d_model=16, heads=2, vocab=30, max_seq=8, layers=2, d_ff=24)
    assert np.array_equal(hp.init_parameters(bs, 3), mo.init_parameters(ob, 3))


@pytest.mark.parametrize("mb", [0.01, 0.5, 1.0, 25.0])
def test_bucket_layout_contract(mb):
    """buckets are contiguous [lo, hi) ranges of the canonical
    flat order, walked from the end, close-on-overflow; concatenated they
    tile [0, N) exactly and never split a parameter."""
    spec = hp.ModelSpec()
    shapes = hp.param_shapes(spec)
    b = hp.bucket_plan(spec, mb)
    n = hp.flat_size(spec)
    assert b[0][1] == n and b[-1][0] == 0
    for (lo, hi), (lo2, hi2) in zip(b, b[1:]):
        assert hi2 == lo
    starts = {s.offset for s in shapes} | {n}
    cap = mb * 1048576
    # host recomputation of the rule
    i, want = len(shapes), []
    while i > 0:
        hi, size = shapes[i - 1].offset + shapes[i - 1].size, 0
        while True:
            size += 4 * shapes[i - 1].size
            i -= 1
            if i == 0 or size + 4 * shapes[i - 1].size > cap:
                break
        want.append((shapes[i].offset, hi))
    assert b == want
    for lo, hi in b:
        assert lo in starts and hi in starts


def test_seq2seq_param_table_init_and_pairs_match_oracle():
    """transformer_seq2seq (repo extension): the product's parameter table
    and init equal the oracle's (names, shapes, order, draws), and the pair
    generator equals the oracle's restatement bit for bit."""
    kw = dict(arch="transformer_seq2seq", d_model=16, heads=2, vocab=40, max_seq=12, layers=2,
              d_ff=24, label_smooth_eps=0.1)
    spec, ospec = hp.ModelSpec(**kw, with_nsp=False), mo.Spec(**kw, with_nsp=False)
    assert [(s.name, s.rows, s.cols) for s in hp.param_shapes(spec)] == \
           [(n, r, c) for n, r, c, _, _ in mo.param_shapes(ospec)]
    names = [s.name for s in hp.param_shapes(spec)]
    assert names[0] == "embed" and "dec1.cv.1" in names and names[-1] == "dec1.ln3.b"
    assert np.array_equal(hp.init_parameters(spec, 3), mo.init_parameters(ospec, 3))
    r = hp.generate_pair_records(hp.PairGenConfig(n=37, vocab=40, min_len=3, max_len=11, seed=9))
    to, tk, sg = mo.pairs_generate(37, 40, 3, 11, 9)
    assert np.array_equal(r.tok_off, to) and np.array_equal(r.tokens, tk)
    assert np.array_equal(r.segments, sg)
    assert r.tokens.min() >= 4 and r.tokens.max() < 40 and len(r) == 37
    with pytest.raises(hp.ConfigError):
        hp.generate_pair_records(hp.PairGenConfig(n=2, vocab=40, min_len=5, max_len=4))
