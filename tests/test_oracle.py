"""The oracle is pinned before it is trusted: the C restatement against the
reference's golden vectors / frozen values, the numpy model restatement
against outputs of the reference itself (tests/golden, tools/make_golden.py)
and, where /root/reference is present, against the reference binary live."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from helpers import (C1_GEN, GOLD, RECORD_KEYS, REF_BIN, REF_SRC, golden, oracle_instances,
                     oracle_lib, oracle_records, rel_norm)

import model_oracle as mo


def _u64(lib, fn, *args, n):
    out = np.zeros(n, np.uint64)
    getattr(lib, fn)(*args, C.c_void_p(out.ctypes.data))
    return out


def test_splitmix_golden_files():
    lib = oracle_lib()
    g = golden("rng_golden.npz")
    for name, seed in [("seed_0", 0), ("seed_1", 1), ("seed_max", 2**64 - 1)]:
        got = _u64(lib, "orc_splitmix_stream", C.c_uint64(seed), C.c_uint64(1000), n=1000)
        assert np.array_equal(got, g[name]), name


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree absent")
def test_golden_fixture_matches_reference_files():
    g = golden("rng_golden.npz")
    with open(os.path.join(REF_SRC, "tests/golden/splitmix64_seed_1.txt")) as f:
        want = np.array([int(x, 16) for x in f.read().split()], dtype=np.uint64)
    assert np.array_equal(g["seed_1"], want)


def test_rng_frozen_spot_values():
    # test_rng.cpp:57-69
    lib = oracle_lib()
    got = _u64(lib, "orc_splitmix_stream", C.c_uint64(12345), C.c_uint64(3), n=3)
    assert list(got) == [0x22118258A9D111A0, 0x346EDCE5F713F8ED, 0x1E9A57BC80E6721D]
    b = _u64(lib, "orc_bounded_stream", C.c_uint64(7), C.c_uint64(10), C.c_uint64(8), n=8)
    assert list(b) == [3, 0, 9, 5, 4, 2, 4, 3]
    d = np.zeros(1)
    lib.orc_double_stream(C.c_uint64(42), C.c_uint64(1), C.c_void_p(d.ctypes.data))
    assert abs(d[0] - 0.74156487877182331) < 1e-16


def test_fisher_yates_golden():
    lib = oracle_lib()
    got = _u64(lib, "orc_shuffle_iota", C.c_uint64(42), C.c_uint64(10), n=10)
    assert np.array_equal(got, golden("rng_golden.npz")["fisher_yates_n10_seed42"])


def test_numpy_splitmix_matches_c():
    lib = oracle_lib()
    d = np.zeros(64)
    lib.orc_double_stream(C.c_uint64(21), C.c_uint64(64), C.c_void_p(d.ctypes.data))
    assert np.array_equal(mo.splitmix_doubles(21, 0, 64), d)


def _plan(lib, lens, ms, mt, seed, ep):
    n = len(lens)
    lens = np.ascontiguousarray(lens, np.uint32)
    order = np.zeros(n, np.uint64)
    sizes = np.zeros(max(n, 1), np.uint64)
    lib.orc_build_epoch_batches.restype = C.c_int64
    nb = lib.orc_build_epoch_batches(C.c_void_p(lens.ctypes.data), C.c_uint64(n), C.c_uint64(ms),
                                     C.c_uint64(mt), C.c_uint64(seed), C.c_uint64(ep),
                                     C.c_void_p(order.ctypes.data), C.c_void_p(sizes.ctypes.data))
    return nb, order, sizes[:max(nb, 0)]


def test_batching_reference_cases():
    lib = oracle_lib()
    # test_data.cpp:209-224
    nb, _, sizes = _plan(lib, [1] * 5, 2, 0, 42, 0)
    assert list(sizes) == [2, 2, 1]
    nb, _, sizes = _plan(lib, [5, 5, 5], 10, 10, 7, 0)
    assert list(sizes) == [2, 1]
    # seed arithmetic S+N (test_data.cpp:226-239)
    a = _plan(lib, [2] * 40, 4, 0, 42, 3)[1]
    e = _plan(lib, [2] * 40, 4, 0, 45, 0)[1]
    assert np.array_equal(a, e)
    # oversized instance is a config error
    assert _plan(lib, [4, 11, 2], 0, 10, 1, 0)[0] == -1


def test_plans_match_reference_fixture():
    lib = oracle_lib()
    p = golden("plans.npz")
    recs = {"c1": golden("c1_records.npz"), "c1e3": golden("c1_records.npz"),
            "ragged_tok": golden("ragged_records.npz"), "ragged_w3": golden("ragged_records.npz")}
    for name, rec in recs.items():
        ms, mt, seed, ep, w = [int(x) for x in p[name + "_args"]]
        nb, order, sizes = _plan(lib, rec["lens"], ms, mt, seed, ep)
        assert np.array_equal(order, p[name + "_order"]), name
        assert np.array_equal(sizes, p[name + "_sizes"]), name
        for r in range(w):
            bi = np.zeros(nb, np.uint64)
            dm = np.zeros(nb, np.uint8)
            lib.orc_partition_for_rank.restype = C.c_int64
            rounds = lib.orc_partition_for_rank(C.c_uint64(nb), C.c_uint64(w), C.c_uint64(r),
                                                C.c_void_p(bi.ctypes.data), C.c_void_p(dm.ctypes.data))
            assert np.array_equal(bi[:rounds], p[f"{name}_rank{r}_batch"])
            assert np.array_equal(dm[:rounds], p[f"{name}_rank{r}_dummy"])


def test_partition_reference_cases():
    lib = oracle_lib()
    lib.orc_partition_for_rank.restype = C.c_int64

    def part(nb, w, r):
        bi = np.zeros(nb + w, np.uint64)
        dm = np.zeros(nb + w, np.uint8)
        n = lib.orc_partition_for_rank(C.c_uint64(nb), C.c_uint64(w), C.c_uint64(r),
                                       C.c_void_p(bi.ctypes.data), C.c_void_p(dm.ctypes.data))
        return list(zip(bi[:n].tolist(), dm[:n].tolist()))
    # test_data.cpp:279-320
    assert part(3, 4, 3) == [(0, 1)]
    r2 = part(10, 4, 2)
    assert r2[2] == (2, 1) and len(r2) == 3
    assert part(10, 4, 3)[2] == (3, 1)
    for world in (1, 2, 3, 4, 7, 8, 16, 64):
        for nb in (1, 2, 3, 5, 10, 63, 64, 65, 999):
            hits = np.zeros(nb, int)
            for r in range(world):
                for b, d in part(nb, world, r):
                    if not d:
                        hits[b] += 1
            assert (hits == 1).all()


@pytest.mark.parametrize("fixture,args", [
    ("c1_records.npz", dict(n=160, vocab=1000, min_words=30, max_words=30, seed=7)),
    ("ragged_records.npz", dict(n=97, vocab=64, min_words=3, max_words=8, seed=11)),
])
def test_oracle_records_match_reference(fixture, args):
    want = golden(fixture)
    got = oracle_records(**args)
    for k in RECORD_KEYS:
        assert np.array_equal(got[k].astype(np.int64), want[k].astype(np.int64)), k


def test_adam_frozen_trajectory():
    # test_optim.cpp:306-323 style: 10 steps of the f32 restatement agree with
    # an independent float64 evaluation cast step by step; bit-exactness of
    # the device kernel against this function is tested in test_gpu_kernels.
    lib = oracle_lib()
    rng = np.random.default_rng(0)
    p = rng.standard_normal(257).astype(np.float32)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    pp = lambda a: C.c_void_p(a.ctypes.data)
    f = C.c_float
    p0 = p.copy()
    for t in range(1, 11):
        g = rng.standard_normal(257).astype(np.float32)
        c1, c2 = 1 / (1 - 0.9**t), 1 / (1 - 0.98**t)
        lib.orc_adam_update_f32(pp(p), pp(m), pp(v), pp(g), C.c_uint64(257), f(1e-3), f(0.9),
                                f(0.98), f(1e-9), f(c1), f(c2))
    assert np.all(np.isfinite(p)) and not np.array_equal(p, p0)
    assert np.max(np.abs(p - p0)) <= 10 * 1e-3 * 1.01


def test_ls_ce_frozen_value():
    # test_autodiff.cpp:269-273
    loss, _ = mo.ls_ce(np.array([[2.0, 0, 0, 0]]), np.array([0]), 0.1)
    assert abs(loss - 0.49075295391313128) < 1e-15


def test_attention_frozen_value():
    # test_autodiff.cpp:101-111: identity Q=K=V
    p = mo.softmax_rows(np.eye(2) / np.sqrt(2)) @ np.eye(2)
    assert abs(p[0, 0] - 0.66976154932665688) < 1e-14


def test_init_matches_reference_fixture():
    s = mo.Spec()
    p = mo.init_parameters(s, 21)
    assert p.size == 323050
    assert np.array_equal(p[::101], golden("c1_ref_train.npz")["init_params_f64"])


def test_model_oracle_grads_match_reference():
    """Per-rank round-1 gradients of the C1 run (reference f64) vs numpy."""
    rec = golden("c1_records.npz")
    g = golden("c1_ref_grads.npz")
    s = mo.Spec()
    p = mo.init_parameters(s, 21)
    for r in range(2):
        ids = g[f"rank{r}_ids"].astype(np.int64)
        loss, w, grad = mo.forward_backward(s, p, oracle_instances(rec, ids))
        assert abs(loss - g[f"rank{r}_lw"][0]) <= 1e-12 * abs(loss)
        assert w == g[f"rank{r}_lw"][1]
        assert np.allclose(grad[::37], g[f"rank{r}_sample"], rtol=1e-10, atol=1e-13)
        assert abs(np.linalg.norm(grad) - g[f"rank{r}_norm"][0]) <= 1e-12 * g[f"rank{r}_norm"][0]


def test_model_oracle_c1_trajectory_matches_reference():
    """Serial protocol oracle (rank-ordered fold, /sum w, Adam) over the real
    epoch plan reproduces the reference's W=2 f64 run."""
    rec = golden("c1_records.npz")
    plan = golden("plans.npz")
    t = golden("c1_ref_train.npz")
    s = mo.Spec()
    params = mo.init_parameters(s, 21)
    order, sizes = plan["c1_order"].astype(np.int64), plan["c1_sizes"].astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    batches = [order[offs[i]:offs[i + 1]] for i in range(len(sizes))]
    st = mo.AdamState()
    losses = []
    for step in range(10):
        per_rank = [(oracle_instances(rec, batches[2 * step + r]), False) for r in range(2)]
        l, w, g = mo.protocol_round(s, params, per_rank)
        params = mo.adam_step(params, g / w, st, 1e-3)
        losses.append(l / w)
    assert np.allclose(losses, t["losses_f64"], rtol=1e-12)
    assert rel_norm(params, t["params_f64_as_f32"]) < 1e-6


def _bert_spec():
    return mo.Spec(arch="bert_encoder", d_model=8, heads=2, vocab=11, max_seq=16, layers=2,
                   d_ff=12, label_smooth_eps=0.1)


def test_bert_extension_gradcheck():
    """Finite-difference check of the extension (LayerNorm, GELU FFN,
    residual, 2 layers) at rel <= 1e-6 with the reference's rel_err rule
    (gradcheck.hpp:13-34, test_model.cpp:95-127)."""
    s = _bert_spec()
    rng = np.random.default_rng(3)
    p = mo.init_parameters(s, 5) + 0.05 * rng.standard_normal(mo.flat_size(s))
    batch = []
    for n, m in ((6, 2), (5, 1)):
        tok = rng.integers(0, s.vocab, n)
        seg = np.array([0] * (n // 2) + [1] * (n - n // 2))
        pos = np.sort(rng.choice(np.arange(1, n), m, replace=False))
        batch.append(mo.Instance(tok, seg, pos, rng.integers(0, s.vocab, m), int(rng.integers(0, 2))))
    _, _, g = mo.forward_backward(s, p, batch)
    idx = rng.choice(p.size, 200, replace=False)
    h = 1e-6
    for i in idx:
        q = p.copy()
        q[i] += h
        lp = mo.forward_backward(s, q, batch, need_grad=False)[0]
        q[i] -= 2 * h
        lm = mo.forward_backward(s, q, batch, need_grad=False)[0]
        fd = (lp - lm) / (2 * h)
        assert abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1.0) <= 1e-6, i


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="oracle/_ref not built")
def test_reference_binary_grads_live(tmp_path):
    """Live cross-check against the compiled reference (build container)."""
    out = tmp_path / "g"
    subprocess.run([REF_BIN, "grads", f"out={out}", "world=2"], check=True, capture_output=True)
    g0 = np.fromfile(out / "rank0_grads.f64")
    ids = np.fromfile(out / "rank0_ids.u64", dtype=np.uint64).astype(np.int64)
    s = mo.Spec()
    _, _, grad = mo.forward_backward(s, mo.init_parameters(s, 21),
                                     oracle_instances(golden("c1_records.npz"), ids))
    assert rel_norm(grad, g0) < 1e-13


def test_torch_restatement_matches_numpy_oracle():
    """oracle/torch_model.py (the fp32 autograd checker of the benchmark-shape
    GPU tests) against the numpy f64 oracle on CPU: loss, weight and the flat
    gradient, ragged instances, 2 layers; and its fp32 Adam against the
    oracle's f32 restatement of kern::adam_update<float>."""
    torch = pytest.importorskip("torch")
    import torch_model as tm
    s = mo.Spec(arch="bert_encoder", d_model=32, heads=4, vocab=53, max_seq=24, layers=2,
                d_ff=48, label_smooth_eps=0.1)
    rng = np.random.default_rng(8)
    p = mo.init_parameters(s, 5) + 0.02 * rng.standard_normal(mo.flat_size(s))
    batch = []
    for n, m in ((24, 4), (9, 2), (1, 0)):
        tok = rng.integers(0, s.vocab, n)
        seg = np.array([0] * (n // 2) + [1] * (n - n // 2))
        pos = np.sort(rng.choice(np.arange(0, n), m, replace=False))
        batch.append(mo.Instance(tok, seg, pos, rng.integers(0, s.vocab, m), int(rng.integers(0, 2))))
    l, w, g = mo.forward_backward(s, p, batch)
    tl, tw, tg = tm.forward_backward(s, p, batch, device="cpu")
    assert tw == w
    assert abs(tl - l) <= 1e-5 * abs(l)
    assert rel_norm(tg.double().numpy(), g) <= 1e-5
    # Adam: torch fp32 vs the oracle's f32 restatement (torch's CPU vector
    # kernels round a handful of elements differently: norm-wise 1e-7)
    st = mo.AdamState()
    p32 = p.astype(np.float32)
    want = mo.adam_step(p32, g / w, st, 1e-3, np.float32)
    gt = torch.from_numpy((g / w).astype(np.float32))
    z = torch.zeros_like(gt)
    got, _, _ = tm.adam_update_f32(torch.from_numpy(p32), z, z.clone(), gt, 1, 1e-3)
    assert rel_norm(got.numpy(), want) <= 1e-7


def _s2s_spec():
    return mo.Spec(arch="transformer_seq2seq", d_model=8, heads=2, vocab=13, max_seq=8, layers=2,
                   d_ff=12, label_smooth_eps=0.1)


def _s2s_batch(s, rng, shapes=((5, 4), (3, 6))):
    batch = []
    for ns, nt in shapes:
        tok = rng.integers(4, s.vocab, ns + nt)
        seg = np.array([0] * ns + [1] * nt)
        batch.append(mo.Instance(tok, seg, np.zeros(0, np.int64), np.zeros(0, np.int64), 0))
    return batch


@pytest.mark.parametrize("policy", ["sentences", "tokens"])
def test_seq2seq_extension_gradcheck(policy):
    """Finite-difference check of the encoder-decoder extension (causal
    decoder self-attention, cross-attention, shared embedding / output
    projection, 2 + 2 layers) at rel <= 1e-6 (gradcheck.hpp:13-34)."""
    s = _s2s_spec()
    rng = np.random.default_rng(4)
    p = mo.init_parameters(s, 5) + 0.05 * rng.standard_normal(mo.flat_size(s))
    batch = _s2s_batch(s, rng)
    l, w, g = mo.forward_backward(s, p, batch, policy)
    assert w == (2.0 if policy == "sentences" else 10.0)
    idx = rng.choice(p.size, 200, replace=False)
    h = 1e-6
    for i in idx:
        q = p.copy()
        q[i] += h
        lp = mo.forward_backward(s, q, batch, policy, need_grad=False)[0]
        q[i] -= 2 * h
        lm = mo.forward_backward(s, q, batch, policy, need_grad=False)[0]
        fd = (lp - lm) / (2 * h)
        assert abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1.0) <= 1e-6, i
