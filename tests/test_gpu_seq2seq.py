"""transformer_seq2seq (the paper's encoder-decoder translation Transformer,
BASELINE configs[2] "C3"; repo extension -- parity against the numpy f64
oracle, which is finite-difference pinned, tests/test_oracle.py):

* the fp32 path (SIMT GEMMs / attention) and the bf16 tcgen05 path at small
  shapes: loss, the local gradient (flat and per block), a 3-update
  trajectory;
* the C3 shape itself (6 + 6 layers, d 512, h 8, f 2048, V 32768) on the bf16
  path, 2 pairs of 64 + 64 tokens.
Tolerances: fp32 loss / gradient / parameters <= 1e-4 (norm-wise); bf16 loss
<= 1e-2, gradient <= 5e-2, parameters <= 1e-2.
"""
import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from helpers import oracle_instances, rel_norm

import model_oracle as mo

pytestmark = pytest.mark.gpu


def _case(d, heads, layers, dff, vocab, n, lmin, lmax, seed=3, max_seq=64):
    kw = dict(arch="transformer_seq2seq", d_model=d, heads=heads, vocab=vocab, max_seq=max_seq,
              layers=layers, d_ff=dff, label_smooth_eps=0.1)
    spec, ospec = hp.ModelSpec(**kw, with_nsp=False), mo.Spec(**kw, with_nsp=False)
    rec = hp.generate_pair_records(hp.PairGenConfig(n=n, vocab=vocab, min_len=lmin, max_len=lmax, seed=seed))
    return spec, ospec, rec


def _engine(spec, compute, policy="tokens", max_tokens=1024, max_batch=16, seed=9, **kw):
    return hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9), hp.ExecConfig(
        compute=compute, policy=policy, max_tokens=max_tokens, max_batch=max_batch, max_masks=1, **kw),
        seed=seed)


def _block_worst(spec, got, want):
    tot = np.linalg.norm(want)
    worst = ("", 0.0)
    for sh in hp.param_shapes(spec):
        sl = slice(sh.offset, sh.offset + sh.size)
        if np.linalg.norm(want[sl]) >= 1e-4 * tot:
            e = rel_norm(got[sl], want[sl])
            if e > worst[1]:
                worst = (sh.name, e)
    return worst


@pytest.mark.parametrize("compute,d,heads", [("f32", 64, 2), ("bf16", 128, 2)])
@pytest.mark.parametrize("policy", ["tokens", "sentences"])
def test_seq2seq_gradients_match_oracle(compute, d, heads, policy):
    spec, ospec, rec = _case(d, heads, 2, 2 * d, 211, 12, 5, 40)
    eng = _engine(spec, compute, policy)
    eng.set_capture(True)
    ids = np.arange(8)
    rep = eng.round(rec.batch(ids), lr=0.0)
    l, w, g = mo.forward_backward(ospec, mo.init_parameters(ospec, 9), oracle_instances(rec, ids), policy)
    tol = 1e-4 if compute == "f32" else 2e-2
    assert rep.local_weight == w
    assert abs(rep.local_loss_sum - l) <= tol * abs(l)
    got = eng.local_grads()
    assert rel_norm(got, g) <= (1e-4 if compute == "f32" else 5e-2)
    name, worst = _block_worst(spec, got, g)
    assert worst <= (1e-3 if compute == "f32" else 1.5e-1), (name, worst)
    eng.close()


@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_seq2seq_trajectory_matches_oracle(compute):
    """3 Adam updates (the reference's Optimizer<float>::step on the f64
    gradient / weight, optim.hpp:107-146) on different ragged batches."""
    d, heads = (64, 2) if compute == "f32" else (128, 2)
    spec, ospec, rec = _case(d, heads, 2, 2 * d, 211, 24, 3, 50)
    eng = _engine(spec, compute)
    p = mo.init_parameters(ospec, 9).astype(np.float32)
    st = mo.AdamState()
    for k, ids in enumerate([range(0, 6), range(6, 14), range(14, 24)]):
        rep = eng.round(rec.batch(ids), lr=1e-3)
        l, w, g = mo.forward_backward(ospec, p.astype(np.float64), oracle_instances(rec, ids), "tokens")
        p = mo.adam_step(p, g / w, st, 1e-3, np.float32)
        assert rep.step == k + 1 and rep.weight == w
        assert abs(rep.loss - l / w) <= (1e-4 if compute == "f32" else 1e-2) * abs(l / w)
        assert rel_norm(eng.get_params(), p) <= (1e-4 if compute == "f32" else 1e-2)
    eng.close()


def test_seq2seq_c3_shape_bf16_vs_oracle():
    """The C3 model (6 + 6 layers, d 512, h 8, f 2048, V 32768) on the bf16
    path: step-1 loss and gradient, then 2 more updates, vs the oracle."""
    spec, ospec, rec = _case(512, 8, 6, 2048, 32768, 6, 64, 64, max_seq=64)
    eng = _engine(spec, "bf16", max_tokens=2 * 128, max_batch=2)
    eng.set_capture(True)
    p = mo.init_parameters(ospec, 9).astype(np.float32)
    p0 = p.copy()
    st = mo.AdamState()
    for k, ids in enumerate([[0, 1], [2, 3], [4, 5]]):
        rep = eng.round(rec.batch(ids), lr=1e-4)
        l, w, g = mo.forward_backward(ospec, p.astype(np.float64), oracle_instances(rec, ids), "tokens")
        if k == 0:
            got = eng.local_grads()
            assert rel_norm(got, g) <= 5e-2
            name, worst = _block_worst(spec, got, g)
            assert worst <= 1.5e-1, (name, worst)
        p = mo.adam_step(p, g / w, st, 1e-4, np.float32)
        assert rep.weight == w == 128.0
        assert abs(rep.loss - l / w) <= 1e-2 * abs(l / w)
    assert rel_norm(eng.get_params(), p) <= 1e-2
    assert rel_norm(eng.get_params() - p0, p.astype(np.float64) - p0) <= 0.5  # the updates themselves
    eng.close()


def test_seq2seq_input_validation():
    spec, ospec, rec = _case(64, 2, 1, 128, 211, 4, 5, 10)
    eng = _engine(spec, "f32")
    b = rec.batch([0, 1])
    bad = hp.BatchCSR(**{k: getattr(b, k).copy() for k in ("tok_off", "tokens", "segments", "mask_off",
                                                            "mask_pos", "mask_orig", "label")})
    bad.segments[:] = 0  # no target
    with pytest.raises(hp.ShapeError):
        eng.stage(bad)
    bad.segments[:] = 1  # no source
    with pytest.raises(hp.ShapeError):
        eng.stage(bad)
    bad = hp.BatchCSR(**{k: getattr(b, k).copy() for k in ("tok_off", "tokens", "segments", "mask_off",
                                                            "mask_pos", "mask_orig", "label")})
    bad.tokens[2] = 211
    with pytest.raises(hp.IndexError_):
        eng.stage(bad)
    long = hp.Instance(np.arange(4, 4 + 70) % 200 + 4, np.array([0] * 3 + [1] * 67), np.zeros(0, np.int64),
                       np.zeros(0, np.int64), 0)
    with pytest.raises(hp.ShapeError):
        eng.stage([long])
    eng.close()


def test_seq2seq_packed_attention_matches_unpacked(monkeypatch):
    """bf16 tcgen05 attention with consecutive short pairs packed into one
    128-row tile per CTA (block-diagonal mask; the default) against one pair
    per CTA (HP_ATTN_PACK=0): the same losses and local gradient up to the
    tensor cores' summation order over the zero-masked keys."""
    spec, _, rec = _case(128, 2, 2, 256, 211, 16, 3, 45, seed=5)
    ids = np.arange(12)
    out = {}
    for pack in ("1", "0"):
        monkeypatch.setenv("HP_ATTN_PACK", pack)
        eng = _engine(spec, "bf16")
        eng.set_capture(True)
        rep = eng.round(rec.batch(ids), lr=0.0)
        out[pack] = (rep.local_loss_sum, eng.local_grads())
        eng.close()
    (l1, g1), (l0, g0) = out["1"], out["0"]
    assert abs(l1 - l0) <= 2e-3 * abs(l0)
    assert rel_norm(g1, g0) <= 1e-2
