#!/usr/bin/env python3
"""Generate tests/golden/* by running the REFERENCE itself (oracle/_ref/hetpar_ref,
compiled in place from /root/reference by `make -C oracle ref`).

Run in the build container (where /root/reference exists):
    make -C oracle all ref && python tools/make_golden.py
The outputs are small committed fixtures; the GPU box never reads
/root/reference.
"""
from __future__ import annotations

import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "hetpar_ref")
GOLD = os.path.join(ROOT, "tests", "golden")
REF_GOLDEN = "/root/reference/proj/tests/golden"

# C1: masked_token_model d128 h4 V1000, seq 63,
# 8 sentences/rank, W=2, Adam(0.9, 0.98, 1e-9), lr 1e-3, seed 21, 10 steps.
C1 = dict(n=160, vocab=1000, min_words=30, max_words=30, data_seed=7, shards=4,
          d=128, heads=4, max_seq=64, eps_ls=0.1, seed=21, max_sentences=8,
          world=2, steps=10, lr=1e-3, opt="adam")


def run(cmd, **kw):
    args = [REF, cmd] + [f"{k}={v}" for k, v in kw.items()]
    out = subprocess.run(args, check=True, capture_output=True, text=True)
    return out.stdout


def rd(path, dt):
    return np.fromfile(path, dtype=dt)


# HCK1: a small reference run whose checkpoints the repo must read and
# re-serialise byte for byte (tests/test_checkpoint.py) and resume from
# (tests/test_gpu_engine.py); W=2, checkpoint every 2 updates, 4 updates.
HCK1 = dict(n=32, vocab=64, min_words=8, max_words=12, docs=4, spd=4, data_seed=3, shards=2,
            d=16, heads=2, max_seq=40, eps_ls=0.1, seed=5, max_sentences=4,
            world=2, steps=4, lr=1e-3, opt="adam", ckpt_every=2)


def hck1_golden():
    import json
    import shutil
    out = os.path.join(GOLD, "hck1")
    os.makedirs(out, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        t = os.path.join(tmp, "t")
        run("train", out=t, dtype="f32", keep_ckpt=1, **HCK1)
        for f in ("checkpoint_000002.hck", "checkpoint_final.hck"):
            shutil.copy(os.path.join(t, f), os.path.join(out, f))
        losses = rd(os.path.join(t, "losses.f64"), np.float64)
    with open(os.path.join(out, "run.json"), "w") as f:
        json.dump({"config": HCK1, "losses": losses.tolist(),
                   "note": "reference train_run<float>, 2 in-process ranks (oracle/_ref/hetpar_ref)"},
                  f, indent=1)


def hsd1_golden():
    """The reference's own HSD1 files for the ragged generator config: the
    repo's shard reader must decode them record for record and its writer
    must reproduce them byte for byte (tests/test_shards.py)."""
    import shutil
    out = os.path.join(GOLD, "hsd1")
    os.makedirs(out, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        g = os.path.join(tmp, "g")
        run("gen", out=g, n=97, vocab=64, min_words=3, max_words=8, data_seed=11, shards=3, keep_shards=1)
        for f in sorted(os.listdir(os.path.join(g, "kept_shards"))):
            shutil.copy(os.path.join(g, "kept_shards", f), os.path.join(out, f))


def main():
    import sys
    if "--only-hck1" in sys.argv:
        hck1_golden()
        return
    if "--only-hsd1" in sys.argv:
        hsd1_golden()
        return
    hsd1_golden()
    os.makedirs(GOLD, exist_ok=True)
    hck1_golden()
    with tempfile.TemporaryDirectory() as tmp:
        # records of the reference generator, read back through its index
        g = os.path.join(tmp, "gen")
        run("gen", out=g, **{k: C1[k] for k in ("n", "vocab", "min_words", "max_words", "data_seed", "shards")})
        rec = {k: rd(os.path.join(g, f), dt) for k, f, dt in [
            ("tok_off", "tok_off.u64", np.uint64), ("tokens", "tokens.i64", np.int64),
            ("segments", "segments.i64", np.int64), ("mask_off", "mask_off.u64", np.uint64),
            ("mask_pos", "mask_pos.i64", np.int64), ("mask_orig", "mask_orig.i64", np.int64),
            ("label", "label.i64", np.int64), ("lens", "lens.u32", np.uint32)]}
        np.savez_compressed(os.path.join(GOLD, "c1_records.npz"), **rec)

        # a second, ragged generator config (variable sentence lengths)
        g2 = os.path.join(tmp, "gen2")
        run("gen", out=g2, n=97, vocab=64, min_words=3, max_words=8, data_seed=11, shards=3)
        rec2 = {k: rd(os.path.join(g2, f), dt) for k, f, dt in [
            ("tok_off", "tok_off.u64", np.uint64), ("tokens", "tokens.i64", np.int64),
            ("segments", "segments.i64", np.int64), ("mask_off", "mask_off.u64", np.uint64),
            ("mask_pos", "mask_pos.i64", np.int64), ("mask_orig", "mask_orig.i64", np.int64),
            ("label", "label.i64", np.int64), ("lens", "lens.u32", np.uint32)]}
        np.savez_compressed(os.path.join(GOLD, "ragged_records.npz"), **rec2)

        # epoch plans + rank schedules
        plans = {}
        cases = [("c1", rec["lens"], 8, 0, 21, 0, 2), ("c1e3", rec["lens"], 8, 0, 21, 3, 2),
                 ("ragged_tok", rec2["lens"], 6, 40, 5, 1, 4), ("ragged_w3", rec2["lens"], 0, 25, 9, 0, 3)]
        for name, lens, ms, mt, seed, epoch, world in cases:
            lp = os.path.join(tmp, f"{name}.u32")
            lens.astype(np.uint32).tofile(lp)
            po = os.path.join(tmp, f"plan_{name}")
            run("plan", out=po, lens=lp, max_sentences=ms, max_tokens=mt, seed=seed, epoch=epoch, world=world)
            plans[f"{name}_args"] = np.array([ms, mt, seed, epoch, world], dtype=np.uint64)
            plans[f"{name}_order"] = rd(os.path.join(po, "order.u64"), np.uint64)
            plans[f"{name}_sizes"] = rd(os.path.join(po, "sizes.u64"), np.uint64)
            for r in range(world):
                plans[f"{name}_rank{r}_batch"] = rd(os.path.join(po, f"rank{r}_batch.u64"), np.uint64)
                plans[f"{name}_rank{r}_dummy"] = rd(os.path.join(po, f"rank{r}_dummy.u8"), np.uint8)
        np.savez_compressed(os.path.join(GOLD, "plans.npz"), **plans)

        # C1 training trajectory, f64 and f32 reference runs
        kw = {k: C1[k] for k in C1}
        t64 = os.path.join(tmp, "t64")
        run("train", out=t64, dtype="f64", **kw)
        t32 = os.path.join(tmp, "t32")
        run("train", out=t32, dtype="f32", **kw)
        init = os.path.join(tmp, "init")
        run("init", out=init, d=128, heads=4, vocab=1000, max_seq=64, seed=21)
        np.savez_compressed(
            os.path.join(GOLD, "c1_ref_train.npz"),
            losses_f64=rd(os.path.join(t64, "losses.f64"), np.float64),
            weights_f64=rd(os.path.join(t64, "weights.f64"), np.float64),
            params_f64_as_f32=rd(os.path.join(t64, "params.f64"), np.float64).astype(np.float32),
            losses_f32=rd(os.path.join(t32, "losses.f64"), np.float64),
            params_f32=rd(os.path.join(t32, "params.f32"), np.float32),
            init_params_f64=rd(os.path.join(init, "params.f64"), np.float64)[::101].copy(),
        )

        # round-1 per-rank pre-reduce gradients (strided sample + checksums)
        gr = os.path.join(tmp, "grads")
        run("grads", out=gr, **kw)
        gd = {}
        for r in range(C1["world"]):
            gg = rd(os.path.join(gr, f"rank{r}_grads.f64"), np.float64)
            gd[f"rank{r}_sample"] = gg[::37].copy()
            gd[f"rank{r}_norm"] = np.array([np.linalg.norm(gg)])
            gd[f"rank{r}_sum"] = np.array([gg.sum()])
            gd[f"rank{r}_lw"] = rd(os.path.join(gr, f"rank{r}_lw.f64"), np.float64)
            gd[f"rank{r}_ids"] = rd(os.path.join(gr, f"rank{r}_ids.u64"), np.uint64)
        np.savez_compressed(os.path.join(GOLD, "c1_ref_grads.npz"), **gd)

    # the reference's own golden vectors (tests/golden/*.txt) as arrays
    rng = {}
    for name, seed in [("seed_0", 0), ("seed_1", 1), ("seed_max", 2 ** 64 - 1)]:
        with open(os.path.join(REF_GOLDEN, f"splitmix64_{name}.txt")) as f:
            rng[name] = np.array([int(x, 16) for x in f.read().split()], dtype=np.uint64)
    with open(os.path.join(REF_GOLDEN, "fisher_yates_n10_seed42.txt")) as f:
        rng["fisher_yates_n10_seed42"] = np.array([int(x) for x in f.read().split()], dtype=np.uint64)
    np.savez_compressed(os.path.join(GOLD, "rng_golden.npz"), **rng)
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
