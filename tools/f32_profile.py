#!/usr/bin/env python3
"""The C2 model on the fp32 path (bf16x6 GEMMs, the bench's same_config
c2_f32 leg): 3 warm-up rounds then R rounds, for an ncu launch list
(profiling aid).   python tools/f32_profile.py [R]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14783_b200 import api as hp  # noqa: E402
import bench  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
B, S = 32, 128
gen = hp.MlmGenConfig(n=B * 2, vocab=30522, docs=64, sentences_per_doc=32, min_sentence_words=70,
                      max_sentence_words=90, seed=7, max_seq_tokens=S)
rec = hp.generate_mlm_records(gen)
plan = hp.build_epoch_batches(rec.token_lengths(), B, 0, 21, 0)
batch = rec.batch(plan.batches[0])
ex = hp.ExecConfig(compute="f32", policy="sentences", device=0, bucket_mb=200.0, max_tokens=B * S,
                   max_batch=B, max_masks=B * S // 2)
e = hp.StepEngine(hp.ModelSpec(**bench.C2), hp.OptimConfig("adam", 0.9, 0.98, 1e-9), ex, seed=21)
e.stage(batch)
for _ in range(3 + R):
    e.round_async(False, 1e-4)
e.round_sync()
e.close()
print("ok")
