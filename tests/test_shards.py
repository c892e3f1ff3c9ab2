"""HSD1 shard read path (src/shard.cpp:126-218, dataset.cpp:10-50,
datagen.cpp:71-169) and the prefetching loader (loader.cpp:80-139), host side.

Pinned against shards written by the REFERENCE itself (tests/golden/hsd1/,
tools/make_golden.py: generate_mlm_shards for the ragged config)."""
import os

import numpy as np
import pytest

import paper_2009_14783_b200 as hp
from paper_2009_14783_b200 import _lib, api

HSD1 = os.path.join(os.path.dirname(__file__), "golden", "hsd1")
FIELDS = ("tok_off", "tokens", "segments", "mask_off", "mask_pos", "mask_orig", "label")


def ragged_records():
    return hp.generate_mlm_records(hp.MlmGenConfig(n=97, vocab=64, min_sentence_words=3,
                                                   max_sentence_words=8, seed=11))


def same(a, b):
    return all(np.array_equal(getattr(a, f), getattr(b, f)) for f in FIELDS)


def test_reference_shards_index():
    ds = api.ShardDataset(HSD1)
    rec = ragged_records()
    assert ds.total == 97 and ds.nshards == 3
    assert np.array_equal(ds.token_lengths(), rec.token_lengths())


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("depth", [0, 2])
def test_loader_serves_schedule_in_order(world, depth):
    ds = api.ShardDataset(HSD1)
    rec = ragged_records()
    plan = hp.build_epoch_batches(ds.token_lengths(), 4, 0, 21, 1)
    for rank in range(world):
        sched = hp.partition_for_rank(plan, world, rank)
        got = []
        for b in ds.loader(plan, sched, depth):  # arrays valid until the next batch
            assert same(b.to_csr(), rec.batch(plan.batches[b.batch_index]))
            got.append((b.batch_index, b.dummy))
        assert got == [(r.batch_index, r.dummy) for r in sched]


def test_writer_reproduces_reference_shards_bytes(tmp_path):
    api.write_mlm_shards(str(tmp_path), ragged_records(), 3)
    for f in sorted(os.listdir(HSD1)):
        assert (tmp_path / f).read_bytes() == open(os.path.join(HSD1, f), "rb").read(), f


def test_roundtrip_c1_records(tmp_path):
    rec = hp.generate_mlm_records(hp.MlmGenConfig(n=160, vocab=1000, min_sentence_words=30,
                                                  max_sentence_words=30, seed=7))
    api.write_mlm_shards(str(tmp_path), rec, 4)
    ds = api.ShardDataset(str(tmp_path))
    plan = hp.build_epoch_batches(ds.token_lengths(), 8, 0, 21, 0)
    for b in ds.loader(plan, hp.partition_for_rank(plan, 2, 0), 3):
        assert same(b.to_csr(), rec.batch(plan.batches[b.batch_index]))


def test_rejects_bad_shards(tmp_path):
    with pytest.raises(_lib.IoError, match="not a directory"):
        api.ShardDataset(str(tmp_path / "missing"))
    (tmp_path / "empty").mkdir()
    with pytest.raises(_lib.ConfigError, match="no shards"):
        api.ShardDataset(str(tmp_path / "empty"))
    src = open(os.path.join(HSD1, "shard_0000.hsd"), "rb").read()
    for name, data, err in [("magic", b"HSD2" + src[4:], "bad shard magic"),
                            ("trunc", src[:200], "footer|truncated"),
                            ("version", src[:4] + b"\x02\x00" + src[6:], "unsupported shard version")]:
        d = tmp_path / name
        d.mkdir()
        (d / "shard_0000.hsd").write_bytes(data)
        with pytest.raises(_lib.IoError, match=err):
            api.ShardDataset(str(d))


def test_schedule_beyond_plan_is_rejected():
    ds = api.ShardDataset(HSD1)
    plan = hp.build_epoch_batches(ds.token_lengths(), 4, 0, 21, 0)
    with pytest.raises(_lib.ConfigError, match="beyond plan size"):
        ds.loader(plan, [hp.RankBatch(len(plan.batches) + 3, False)], 0)
