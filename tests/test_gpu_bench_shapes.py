"""Parity at the BENCHMARKED shapes (BASELINE configs[1] "C2" and configs[3]
"C4"): the exact models bench.py times, run for 3 Adam updates through the
C ABI, against independent restatements of the same math.

* C2 (bert_encoder L=12, d=768, h=12, d_ff=3072, V=30522, seq <= 128) on the
  fp32 path and the bf16 tcgen05 path vs the numpy f64 oracle
  (oracle/model_oracle.py): per-step loss, the step-1 local gradient
  (norm-wise over the flat vector and per parameter block) and the
  parameters after every update (the oracle's update is the reference's
  Optimizer<float>::step, optim.hpp:107-146, on the f64 gradient / weight).
* C4 (L=24, d=1024, h=16, d_ff=4096, seq <= 512; bf16 only -- sequences
  > 128 need the blocked tcgen05 attention) vs the torch fp32 autograd
  restatement (oracle/torch_model.py, itself pinned to the numpy oracle by
  tests/test_oracle.py).

Tolerances (written here, per SURVEY §8c norm-wise rule):
  fp32 path: loss rel <= 1e-4, gradient norm-wise <= 1e-4, parameters
             norm-wise <= 1e-4 after every update.
  bf16 path: loss rel <= 1e-2, gradient norm-wise <= 5e-2, parameters
             norm-wise <= 1e-2 after 3 updates (bf16 operands, fp32
             accumulation and master weights).
Set HP_PARITY_OUT=<file> to write the measured errors as JSON (profiles/).
"""
import json
import os

import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from helpers import oracle_instances, rel_norm

import model_oracle as mo

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

C2 = dict(arch="bert_encoder", d_model=768, heads=12, vocab=30522, max_seq=128, layers=12,
          d_ff=3072, with_nsp=True, label_smooth_eps=0.1)
C4 = dict(arch="bert_encoder", d_model=1024, heads=16, vocab=30522, max_seq=512, layers=24,
          d_ff=4096, with_nsp=True, label_smooth_eps=0.1)
LR = 1e-4
STEPS = 3
PER = 2  # sequences per batch

TOL = {"f32": dict(loss=1e-4, grad=1e-4, params=1e-4),
       "bf16": dict(loss=1e-2, grad=5e-2, params=1e-2)}

_RESULTS = {}


def _record(key, value):
    _RESULTS[key] = value
    out = os.environ.get("HP_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(_RESULTS, f, indent=1, sort_keys=True)


def _records(cfg, n, wmin, wmax):
    return hp.generate_mlm_records(hp.MlmGenConfig(
        n=n, vocab=cfg["vocab"], docs=64, sentences_per_doc=32, min_sentence_words=wmin,
        max_sentence_words=wmax, seed=7, max_seq_tokens=cfg["max_seq"]))


def _engine(cfg, compute, seq):
    spec = hp.ModelSpec(**cfg)
    ex = hp.ExecConfig(compute=compute, max_tokens=PER * seq, max_batch=PER, max_masks=PER * seq // 2)
    eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9), ex, seed=21)
    eng.set_capture(True)
    return eng


def _block_errors(spec, got, want):
    """per-parameter-block norm-wise errors of the blocks carrying >= 1e-4 of
    the gradient norm (the rest are below fp32 resolution of the flat norm)"""
    tot = np.linalg.norm(want)
    out = {}
    for sh in hp.param_shapes(spec):
        sl = slice(sh.offset, sh.offset + sh.size)
        nb = np.linalg.norm(want[sl])
        if nb >= 1e-4 * tot:
            out[sh.name] = rel_norm(got[sl], want[sl])
    return out


# ----------------------------------------------------------------------- C2
@pytest.fixture(scope="module")
def c2_case():
    rec = _records(C2, STEPS * PER, 30, 96)
    batches = [list(range(k * PER, (k + 1) * PER)) for k in range(STEPS)]
    lens = rec.token_lengths()
    assert max(lens) == 128 and min(lens) < 128  # full and ragged sequences
    ospec = mo.Spec(**C2)
    p32 = mo.init_parameters(ospec, 21).astype(np.float32)
    st = mo.AdamState()
    steps = []
    for k, ids in enumerate(batches):
        inst = oracle_instances(rec, ids)
        l, w, g = mo.forward_backward(ospec, p32.astype(np.float64), inst)
        p32 = mo.adam_step(p32, g / w, st, LR, np.float32)
        steps.append(dict(loss=l / w, loss_sum=l, weight=w, params=p32.copy(),
                          grad=g.astype(np.float32) if k == 0 else None))
    return rec, batches, steps


@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_c2_three_adam_steps_vs_numpy_oracle(c2_case, compute):
    rec, batches, steps = c2_case
    spec = hp.ModelSpec(**C2)
    eng = _engine(C2, compute, 128)
    p0 = eng.get_params()
    tol = TOL[compute]
    res = {"loss_rel": [], "params_rel": [], "update_rel": []}
    for k, ids in enumerate(batches):
        rep = eng.round(rec.batch(ids), lr=LR)
        o = steps[k]
        assert rep.step == k + 1 and rep.weight == o["weight"]
        res["loss_rel"].append(abs(rep.loss - o["loss"]) / abs(o["loss"]))
        if k == 0:
            g = eng.local_grads()
            res["grad_rel"] = rel_norm(g, o["grad"])
            blocks = _block_errors(spec, g, o["grad"].astype(np.float64))
            worst = max(blocks, key=blocks.get)
            res["grad_block_worst"] = [worst, blocks[worst]]
            res["grad_blocks_checked"] = len(blocks)
        p = eng.get_params()
        res["params_rel"].append(rel_norm(p, o["params"]))
        res["update_rel"].append(rel_norm(p - p0, o["params"].astype(np.float64) - p0))
    eng.close()
    _record(f"c2_{compute}", res)
    assert max(res["loss_rel"]) <= tol["loss"], res
    assert res["grad_rel"] <= tol["grad"], res
    assert max(res["params_rel"]) <= tol["params"], res
    # every block that carries gradient is right on its own (a broken head /
    # layer cannot hide under the embedding's norm)
    assert res["grad_block_worst"][1] <= (1e-3 if compute == "f32" else 1.5e-1), res


def test_c2_step1_vs_torch_restatement(c2_case):
    """The same C2 step-1 loss and gradient through the second, independent
    restatement (torch fp32 autograd on the GPU)."""
    import torch_model as tm
    rec, batches, steps = c2_case
    ospec = mo.Spec(**C2)
    p32 = mo.init_parameters(ospec, 21).astype(np.float32)
    l, w, g = tm.forward_backward(ospec, p32, oracle_instances(rec, batches[0]))
    g = g.double().cpu().numpy()
    assert w == steps[0]["weight"]
    assert abs(l - steps[0]["loss_sum"]) <= 1e-5 * abs(steps[0]["loss_sum"])
    assert rel_norm(g, steps[0]["grad"]) <= 1e-5
    _record("c2_torch_vs_numpy", {"loss_rel": abs(l - steps[0]["loss_sum"]) / abs(steps[0]["loss_sum"]),
                                  "grad_rel": rel_norm(g, steps[0]["grad"])})


# ----------------------------------------------------------------------- C4
def test_c4_three_adam_steps_vs_torch_fp32():
    import torch_model as tm
    # one full 512-token sequence (bench.py's C4 generator) and one ragged
    # sequence (not a multiple of the 128-row attention block) per batch
    full = _records(C4, STEPS, 256, 384)
    rag = _records(C4, 16, 100, 255)
    rl = rag.token_lengths()
    rag_ids = [i for i in range(len(rl)) if rl[i] % 128 != 0][:STEPS]
    assert all(full.token_lengths() == 512) and len(rag_ids) == STEPS
    insts = [[full.instance(k), rag.instance(rag_ids[k])] for k in range(STEPS)]
    batches = [hp.pack_batch(x) for x in insts]
    oinsts = [[mo.Instance(i.tokens, i.segments, i.mask_positions, i.mask_originals, i.label)
               for i in x] for x in insts]
    ospec = mo.Spec(**C4)
    spec = hp.ModelSpec(**C4)
    eng = _engine(C4, "bf16", 512)
    p = torch.from_numpy(mo.init_parameters(ospec, 21).astype(np.float32)).cuda()
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    p0 = p.clone()
    res = {"loss_rel": [], "params_rel": [], "update_rel": []}
    for k, b in enumerate(batches):
        rep = eng.round(b, lr=LR)
        l, w, g = tm.forward_backward(ospec, p.cpu().numpy(), oinsts[k])
        assert rep.weight == w
        res["loss_rel"].append(abs(rep.loss - l / w) / abs(l / w))
        if k == 0:
            dg = eng.local_grads()
            gn = g.double().cpu().numpy()
            res["grad_rel"] = rel_norm(dg, gn)
            blocks = _block_errors(spec, dg, gn)
            worst = max(blocks, key=blocks.get)
            res["grad_block_worst"] = [worst, blocks[worst]]
            res["grad_blocks_checked"] = len(blocks)
        p, m, v = tm.adam_update_f32(p, m, v, (g.double() / w).float(), k + 1, LR)
        dp = eng.get_params()
        pn = p.cpu().numpy()
        res["params_rel"].append(rel_norm(dp, pn))
        res["update_rel"].append(rel_norm(dp - p0.cpu().numpy(), pn.astype(np.float64) - p0.cpu().numpy()))
    eng.close()
    _record("c4_bf16", res)
    tol = TOL["bf16"]
    assert max(res["loss_rel"]) <= tol["loss"], res
    assert res["grad_rel"] <= tol["grad"], res
    assert max(res["params_rel"]) <= tol["params"], res
    assert res["grad_block_worst"][1] <= 1.5e-1, res
