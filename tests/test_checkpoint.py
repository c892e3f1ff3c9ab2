"""HCK1 checkpoints (src/checkpoint.cpp:165-302) and the resume fast-forward
(include/hetpar/engine.hpp:211-245), host side (no GPU).

Pinned against files written by the REFERENCE itself (tests/golden/hck1/,
tools/make_golden.py: reference train_run<float>, W=2, checkpoint every 2
updates): the repo reads them and re-serialises them byte for byte."""
import json
import os
import shutil

import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from paper_2009_14783_b200 import _lib
from paper_2009_14783_b200.api import read_checkpoint, resume_position, write_checkpoint

HCK1 = os.path.join(os.path.dirname(__file__), "golden", "hck1")
RUN = json.load(open(os.path.join(HCK1, "run.json")))


@pytest.mark.parametrize("name,step", [("checkpoint_000002.hck", 2), ("checkpoint_final.hck", 4)])
def test_reference_checkpoint_reserialises_byte_identical(tmp_path, name, step):
    src = os.path.join(HCK1, name)
    spec, meta, p, m, v = read_checkpoint(src)
    cfg = RUN["config"]
    assert spec.arch == "masked_token_model" and spec.d_model == cfg["d"] and spec.heads == cfg["heads"]
    assert spec.vocab == cfg["vocab"] and spec.max_seq == cfg["max_seq"] and spec.with_nsp
    assert meta.step == step and meta.opt_t == step and meta.seed == cfg["seed"]
    assert meta.world_size == 2 and meta.update_freq == 1 and meta.optimizer == "adam"
    assert (meta.beta1, meta.beta2, meta.eps) == (0.9, 0.98, 1e-9)
    assert meta.scheduler.kind == "fixed" and meta.scheduler.peak_lr == 1e-3
    assert p.size == hp.flat_size(spec) and m.size == p.size and v.size == p.size
    out = tmp_path / "ours.hck"
    write_checkpoint(str(out), spec, meta, p, m, v)
    assert out.read_bytes() == open(src, "rb").read()


def test_roundtrip_bert_extension(tmp_path):
    spec = hp.ModelSpec(arch="bert_encoder", d_model=32, heads=2, vocab=50, max_seq=16, layers=2,
                        d_ff=64, label_smooth_eps=0.1)
    n = hp.flat_size(spec)
    rng = np.random.default_rng(0)
    p, m, v = (rng.standard_normal(n).astype(np.float32) for _ in range(3))
    meta = hp.api.CheckpointMeta(epoch=3, step=17, seed=9, policy="tokens", world_size=4, update_freq=2,
                                 opt_t=17)
    f = str(tmp_path / "b.hck")
    write_checkpoint(f, spec, meta, p, m, v)
    spec2, meta2, p2, m2, v2 = read_checkpoint(f)
    assert spec2 == spec and meta2 == meta
    assert np.array_equal(p, p2) and np.array_equal(m, m2) and np.array_equal(v, v2)


def test_rejects_corrupt_truncated_and_foreign_files(tmp_path):
    src = open(os.path.join(HCK1, "checkpoint_final.hck"), "rb").read()
    bad = bytearray(src)
    bad[200] ^= 1
    (tmp_path / "flip.hck").write_bytes(bytes(bad))
    with pytest.raises(_lib.IoError, match="digest mismatch"):
        read_checkpoint(str(tmp_path / "flip.hck"))
    (tmp_path / "trunc.hck").write_bytes(src[:-100])
    with pytest.raises(_lib.IoError):
        read_checkpoint(str(tmp_path / "trunc.hck"))
    (tmp_path / "x.hck").write_bytes(b"HCK2" + src[4:])
    with pytest.raises(_lib.IoError, match="not a checkpoint"):
        read_checkpoint(str(tmp_path / "x.hck"))
    with pytest.raises(_lib.IoError):
        read_checkpoint(str(tmp_path / "missing.hck"))


def _resume_restated(lens, ms, mt, seed, world, k, step):
    # engine.hpp:225-244
    left = step * k
    e = 0
    while True:
        nb = len(hp.build_epoch_batches(lens, ms, mt, seed, e).batches)
        rounds = (nb + world - 1) // world
        if left < rounds:
            return e, left
        left -= rounds
        e += 1


@pytest.mark.parametrize("world,k", [(1, 1), (2, 1), (3, 2), (8, 1), (2, 4)])
def test_resume_position_matches_restatement(world, k):
    rec = hp.generate_mlm_records(hp.MlmGenConfig(n=97, vocab=64, min_sentence_words=3,
                                                  max_sentence_words=8, seed=11))
    lens = rec.token_lengths()
    for step in (0, 1, 5, 13, 40):
        assert resume_position(lens, 4, 0, 21, world, k, step) == _resume_restated(lens, 4, 0, 21, world, k, step)
