"""Kernel-level numerics on the B200: the tcgen05/TMA GEMM (every operand
major-ness, grouped per-head operands, tails, fused epilogues) and the SIMT
fp32 GEMM against a torch fp32 reference; Adam bit-exact against the C
oracle's restatement of kern::scalar::adam_update<float>."""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import oracle_lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _lib():
    from paper_2009_14783_b200 import _lib
    return _lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def run_gemm(M, N, K, dtype, a_trans, b_trans, path, bn=0, group=0, bias=False, act=0, resid=False,
             accumulate=False, c_dtype=None, c_group=0, seed=0, b_pad=0):
    L = _lib()
    g = torch.Generator(device="cpu").manual_seed(seed)
    dev = "cuda"
    c_dtype = c_dtype or dtype
    A = torch.randn(M, K, generator=g).to(dev, dtype)       # logical A
    if group:
        nb = N // group if not b_trans else K // group
    Bl = torch.randn(K, N, generator=g).to(dev, dtype)      # logical B
    # storage
    A_st = A.t().contiguous() if a_trans else A.contiguous()
    lda = M if a_trans else K
    if group and not b_trans:      # grouped along N: [N/g][K][g]
        B_st = Bl.reshape(K, N // group, group).permute(1, 0, 2).contiguous()
        ldb, gstride = group, K * group
    elif group and b_trans:        # grouped along K: [K/g][N][g]
        B_st = Bl.reshape(K // group, group, N).permute(0, 2, 1).contiguous()
        ldb, gstride = group, N * group
    elif b_trans:
        B_st = Bl.t().contiguous()
        ldb, gstride = K, 0
    else:
        B_st = torch.zeros(K, N + b_pad, device=dev, dtype=dtype)
        B_st[:, :N] = Bl
        ldb, gstride = N + b_pad, 0
    ref = A.float() @ Bl.float()
    bvec = torch.randn(N, generator=g).to(dev) if bias else None
    if bvec is not None:
        ref = ref + bvec
    aux = None
    if act == 1:
        aux = torch.zeros(M, N, device=dev, dtype=c_dtype)
        pre = ref.clone()
        ref = torch.nn.functional.gelu(ref)
    elif act == 2:
        aux = torch.randn(M, N, generator=g).to(dev, c_dtype)
        x = aux.float()
        dg = 0.5 * (1 + torch.erf(x / 2**0.5)) + x * torch.exp(-0.5 * x * x) / (2 * np.pi) ** 0.5
        ref = ref * dg
    R = torch.randn(M, N, generator=g).to(dev, c_dtype) if resid else None
    if R is not None:
        ref = ref + R.float()
    C0 = torch.randn(M, N, generator=g).to(dev, c_dtype) if accumulate else torch.zeros(M, N, device=dev, dtype=c_dtype)
    if accumulate:
        ref = ref + C0.float()
    if c_group:
        Cst = C0.reshape(M, N // c_group, c_group).permute(1, 0, 2).contiguous()
        ldc, cgs = c_group, M * c_group
    else:
        Cst = C0.clone()
        ldc, cgs = N, 0
    L.call("hp_debug_gemm", M, N, K, int(dtype == torch.bfloat16), _ptr(A_st), lda, int(a_trans),
           _ptr(B_st), ldb, int(b_trans), group, gstride, _ptr(Cst), ldc,
           int(c_dtype == torch.bfloat16), c_group, cgs, _ptr(bvec), act, _ptr(aux), _ptr(R),
           N if resid else 0, int(accumulate), path, bn)
    L.call("hp_debug_sync")
    out = Cst.permute(1, 0, 2).reshape(M, N) if c_group else Cst
    res = {"out": out.float(), "ref": ref}
    if act == 1:
        res["aux"] = aux.float()
        res["pre"] = pre
    return res


@pytest.fixture(params=[0, 1], ids=["specialised", "generic"])
def epi_kind(request):
    """Run a test with the per-kind specialised epilogue kernels (default
    selection) and again with every launch forced onto the generic one."""
    L = _lib()
    L.call("hp_debug_gemm_generic", request.param)
    yield request.param
    L.call("hp_debug_gemm_generic", 0)


def _tol(dtype, K):
    return (2e-2 if dtype == torch.bfloat16 else 1e-4) * max(1.0, (K / 64) ** 0.5)


def _check(res, dtype, K):
    err = (res["out"] - res["ref"]).abs().max().item()
    scale = res["ref"].abs().max().item() + 1e-6
    assert err / scale < _tol(dtype, K), (err, scale)


@pytest.mark.parametrize("a_trans", [0, 1])
@pytest.mark.parametrize("b_trans", [0, 1])
@pytest.mark.parametrize("bn", [1128, 1192, 1256, 2128, 2256])
def test_tc_gemm_layouts(a_trans, b_trans, bn):
    res = run_gemm(384, 512, 320, torch.bfloat16, a_trans, b_trans, path=2, bn=bn, c_dtype=torch.float32)
    _check(res, torch.bfloat16, 320)


@pytest.mark.parametrize("shape", [(200, 136, 72), (136, 264, 104), (8, 64, 16), (4096, 768, 64)])
def test_tc_gemm_tails(shape):
    M, N, K = shape
    for a_trans, b_trans in ((0, 0), (0, 1), (1, 0)):
        res = run_gemm(M, N, K, torch.bfloat16, a_trans, b_trans, path=2, c_dtype=torch.float32)
        _check(res, torch.bfloat16, K)


@pytest.mark.parametrize("b_trans", [0, 1])
def test_tc_gemm_grouped_heads(b_trans):
    # QKV fwd (grouped N) and dgrad (grouped K), dk = 64
    res = run_gemm(256, 384, 384, torch.bfloat16, 0, b_trans, path=2, group=64)
    _check(res, torch.bfloat16, 384)


def test_tc_gemm_grouped_output(epi_kind):
    # QKV wgrad: C scattered into [N/64][M][64] blocks (fp32 flat gradient)
    res = run_gemm(256, 384, 512, torch.bfloat16, 1, 0, path=2, c_dtype=torch.float32, c_group=64)
    _check(res, torch.bfloat16, 512)


def test_tc_gemm_epilogues(epi_kind):
    res = run_gemm(256, 512, 256, torch.bfloat16, 0, 0, path=2, bias=True, act=1)
    _check(res, torch.bfloat16, 256)
    assert (res["aux"] - res["pre"]).abs().max().item() < 0.05 * res["pre"].abs().max().item()
    res = run_gemm(256, 512, 256, torch.bfloat16, 0, 1, path=2, act=2)
    _check(res, torch.bfloat16, 256)
    res = run_gemm(256, 384, 256, torch.bfloat16, 0, 0, path=2, bias=True, resid=True)
    _check(res, torch.bfloat16, 256)
    res = run_gemm(256, 384, 256, torch.bfloat16, 1, 0, path=2, accumulate=True, c_dtype=torch.float32)
    _check(res, torch.bfloat16, 256)


def test_tc_gemm_unaligned_output_rows():
    # MLM head wgrad: fp32 C with ldc = V = 30522 (rows not 16B aligned)
    res = run_gemm(128, 1002, 96, torch.bfloat16, 1, 0, path=2, c_dtype=torch.float32, b_pad=6)
    _check(res, torch.bfloat16, 96)


@pytest.mark.parametrize("a_trans,b_trans", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_simt_gemm_fp32(a_trans, b_trans):
    res = run_gemm(100, 70, 45, torch.float32, a_trans, b_trans, path=1, bias=True)
    _check(res, torch.float32, 45)
    res = run_gemm(64, 96, 64, torch.float32, a_trans, b_trans, path=1, group=32 if not a_trans else 0)
    _check(res, torch.float32, 64)


def test_adam_bit_exact_vs_reference_scalar():
    L = _lib()
    orc = oracle_lib()
    rng = np.random.default_rng(1)
    n = 100003
    p = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    dp, dm, dv = (torch.from_numpy(x.copy()).cuda() for x in (p, m, v))
    f = C.c_float
    pp = lambda a: C.c_void_p(a.ctypes.data)
    for t in range(1, 6):
        g = (rng.standard_normal(n) * 10.0 ** rng.integers(-8, 2, n)).astype(np.float32)
        c1, c2 = 1 / (1 - 0.9**t), 1 / (1 - 0.98**t)
        args = (f(1e-3), f(0.9), f(0.98), f(1e-9), f(c1), f(c2))
        orc.orc_adam_update_f32(pp(p), pp(m), pp(v), pp(g), C.c_uint64(n), *args)
        dg = torch.from_numpy(g).cuda()
        L.call("hp_debug_adam", _ptr(dp), _ptr(dm), _ptr(dv), _ptr(dg), n, *[a.value for a in args], 0, 0.0)
    assert np.array_equal(dp.cpu().numpy().view(np.uint32), p.view(np.uint32))
    assert np.array_equal(dm.cpu().numpy().view(np.uint32), m.view(np.uint32))
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), v.view(np.uint32))
    # SGD
    g = rng.standard_normal(n).astype(np.float32)
    orc.orc_sgd_update_f32(pp(p), pp(g), C.c_uint64(n), f(0.1))
    L.call("hp_debug_adam", _ptr(dp), _ptr(dm), _ptr(dv), _ptr(torch.from_numpy(g).cuda()), n,
           0.1, 0.9, 0.98, 1e-9, 1.0, 1.0, 1, 0.0)
    assert np.array_equal(dp.cpu().numpy().view(np.uint32), p.view(np.uint32))


def test_adam_non_finite_gradient_reported_with_lowest_index():
    """optim.hpp:131-133: a non-finite gradient is a numeric error; the device
    update reports the lowest offending flat index, leaves those elements
    untouched and updates the others exactly as the scalar kernel does."""
    L = _lib()
    orc = oracle_lib()
    rng = np.random.default_rng(2)
    n = 70001
    p = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    g[[40000, 12345, 69999]] = [np.inf, np.nan, -np.inf]
    dp, dm, dv, dg = (torch.from_numpy(x.copy()).cuda() for x in (p, m, v, g))
    with pytest.raises(L.NumericError, match="flat index 12345"):
        L.call("hp_debug_adam", _ptr(dp), _ptr(dm), _ptr(dv), _ptr(dg), n, 1e-3, 0.9, 0.98, 1e-9,
               10.0, 50.0, 0, 0.0)
    ok = np.isfinite(g)
    f = C.c_float
    pp = lambda a: C.c_void_p(a.ctypes.data)
    g2 = np.where(ok, g, 0).astype(np.float32)
    p2, m2, v2 = p.copy(), m.copy(), v.copy()
    orc.orc_adam_update_f32(pp(p2), pp(m2), pp(v2), pp(g2), C.c_uint64(n), f(1e-3), f(0.9), f(0.98),
                            f(1e-9), f(10.0), f(50.0))
    got = dp.cpu().numpy()
    assert np.array_equal(got[ok].view(np.uint32), p2[ok].view(np.uint32))
    assert np.array_equal(got[~ok].view(np.uint32), p[~ok].view(np.uint32))


def test_adamw_bit_exact_vs_f32_restatement():
    """AdamW (extension): the device update equals the oracle's fp32
    restatement -- p -= (lr wd) p, then kern::adam_update<float> -- bit for
    bit over 5 steps."""
    import model_oracle as mo
    L = _lib()
    rng = np.random.default_rng(3)
    n = 50021
    p = rng.standard_normal(n).astype(np.float32)
    dp, dm, dv = (torch.from_numpy(x.copy()).cuda() for x in (p, np.zeros(n, np.float32), np.zeros(n, np.float32)))
    st = mo.AdamState()
    for t in range(1, 6):
        g = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 1, n)).astype(np.float32)
        c1, c2 = 1 / (1 - 0.9**t), 1 / (1 - 0.98**t)
        L.call("hp_debug_adam", _ptr(dp), _ptr(dm), _ptr(dv), _ptr(torch.from_numpy(g).cuda()), n,
               1e-3, 0.9, 0.98, 1e-9, c1, c2, 0, 0.01)
        p = mo.adam_step(p, g.astype(np.float64), st, 1e-3, np.float32, weight_decay=0.01)
    assert np.array_equal(dp.cpu().numpy().view(np.uint32), p.view(np.uint32))


def _attn_ref(qkv, cu, H, dk):
    """torch fp32 reference of the varlen attention forward/backward."""
    T = qkv.shape[0]
    d = H * dk
    q = qkv[:, :d].float().reshape(T, H, dk).requires_grad_(True)
    k = qkv[:, d:2 * d].float().reshape(T, H, dk).requires_grad_(True)
    v = qkv[:, 2 * d:].float().reshape(T, H, dk).requires_grad_(True)
    outs = []
    for i in range(len(cu) - 1):
        a, b = cu[i], cu[i + 1]
        s = torch.einsum("qhd,khd->hqk", q[a:b], k[a:b]) / dk ** 0.5
        p = torch.softmax(s, dim=-1)
        outs.append(torch.einsum("hqk,khd->qhd", p, v[a:b]))
    o = torch.cat(outs).reshape(T, d)
    return o, (q, k, v)


@pytest.mark.parametrize("path,dtype,dk", [(3, torch.bfloat16, 64), (2, torch.bfloat16, 64),
                                           (1, torch.bfloat16, 64),
                                           (1, torch.float32, 32), (1, torch.float32, 64),
                                           (1, torch.bfloat16, 32)])
def test_attention_varlen_fwd_bwd(path, dtype, dk):
    L = _lib()
    H = 3
    lens = [128, 1, 17, 63, 64, 100, 5]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    g = torch.Generator(device="cpu").manual_seed(1)
    qkv = (torch.randn(T, 3 * H * dk, generator=g) * 1.5).to("cuda", dtype)
    dO = torch.randn(T, H * dk, generator=g).to("cuda", dtype)
    o = torch.zeros(T, H * dk, device="cuda", dtype=dtype)
    lse = torch.zeros(H, T, device="cuda")
    dqkv = torch.zeros_like(qkv)
    dcu = torch.from_numpy(cu).cuda()
    L.call("hp_debug_attention", len(lens), _ptr(dcu), T, H, dk, int(dtype == torch.bfloat16),
           _ptr(qkv), _ptr(o), _ptr(lse), _ptr(dO), _ptr(dqkv), path)
    ref, (q, k, v) = _attn_ref(qkv, cu.tolist(), H, dk)
    ref.backward(dO.float())
    dref = torch.cat([q.grad.reshape(T, -1), k.grad.reshape(T, -1), v.grad.reshape(T, -1)], 1)
    tol = 3e-2 if dtype == torch.bfloat16 else 1e-4
    eo = (o.float() - ref).abs().max().item() / ref.abs().max().item()
    eg = (dqkv.float() - dref).abs().max().item() / dref.abs().max().item()
    assert eo < tol and eg < tol, (eo, eg)


@pytest.mark.parametrize("splits", [2, 3, 8])
def test_tc_gemm_split_k(splits, epi_kind):
    # weight-gradient shape: few output tiles, long K -> split-K reductions
    res = run_gemm(256, 384, 2048, torch.bfloat16, 1, 0, path=2, bn=128 + 1000 + 10000 * splits,
                   c_dtype=torch.float32)
    _check(res, torch.bfloat16, 2048)
    res = run_gemm(128, 192, 1024, torch.bfloat16, 1, 0, path=2, bn=192 + 1000 + 10000 * splits,
                   c_dtype=torch.float32, c_group=64)
    _check(res, torch.bfloat16, 1024)
    # CTA-pair split-K
    res = run_gemm(512, 512, 2048, torch.bfloat16, 1, 0, path=2, bn=256 + 2000 + 10000 * splits,
                   c_dtype=torch.float32)
    _check(res, torch.bfloat16, 2048)


def test_tc_gemm_auto_heuristic_shapes(epi_kind):
    # the engine's shapes at small scale: auto BN / split choice
    for (M, N, K, at, bt, ct) in [(512, 768, 768, 0, 0, torch.bfloat16), (768, 768, 512, 1, 0, torch.float32),
                                  (512, 2304, 768, 0, 0, torch.bfloat16), (512, 768, 2304, 0, 1, torch.bfloat16)]:
        res = run_gemm(M, N, K, torch.bfloat16, at, bt, path=2, c_dtype=ct)
        _check(res, torch.bfloat16, K)


@pytest.mark.parametrize("cg", [1, 2])
def test_tc_gemm_pair_and_single_edge_cases(cg, epi_kind):
    tile = 256
    code = cg * 1000 + tile
    for (M, N, K, at, bt) in [(600, 1000, 200, 0, 0), (130, 264, 104, 0, 1), (512, 384, 64, 1, 0)]:
        res = run_gemm(M, N, K, torch.bfloat16, at, bt, path=2, bn=code, c_dtype=torch.float32)
        _check(res, torch.bfloat16, K)
    res = run_gemm(512, 384, 384, torch.bfloat16, 0, 0, path=2, bn=code, group=64)
    _check(res, torch.bfloat16, 384)
    res = run_gemm(512, 384, 384, torch.bfloat16, 0, 1, path=2, bn=code, group=64)
    _check(res, torch.bfloat16, 384)
    res = run_gemm(512, 512, 256, torch.bfloat16, 0, 0, path=2, bn=code, bias=True, act=1)
    _check(res, torch.bfloat16, 256)
    res = run_gemm(512, 512, 256, torch.bfloat16, 0, 1, path=2, bn=code, act=2, resid=True)
    _check(res, torch.bfloat16, 256)
    res = run_gemm(256, 384, 512, torch.bfloat16, 1, 0, path=2, bn=code, c_dtype=torch.float32, c_group=64)
    _check(res, torch.bfloat16, 512)


def test_tc_gemm_pair_192_kmajor_b(epi_kind):
    """CTA pair with a 256 x 192 tile (96 B rows per CTA): the data-gradient
    GEMMs with N = 768 and a K-major weight operand (dO, dX1, grouped dX)."""
    for (M, N, K, resid) in [(4096, 768, 768, 0), (1000, 768, 3072, 1), (600, 384, 200, 0),
                             (130, 192, 104, 1)]:
        res = run_gemm(M, N, K, torch.bfloat16, 0, 1, path=2, bn=2192, resid=bool(resid))
        _check(res, torch.bfloat16, K)
    res = run_gemm(512, 768, 2304, torch.bfloat16, 0, 1, path=2, bn=2192, group=64, resid=True)
    _check(res, torch.bfloat16, 2304)
    res = run_gemm(512, 768, 768, torch.bfloat16, 0, 1, path=2, bn=2192, c_dtype=torch.float32)
    _check(res, torch.bfloat16, 768)


def test_tc_gemm_weight_gradient_shapes():
    """Split-K fp32 GEMMs (the weight gradients: A^T dY over the tokens) at
    the C2 shapes, with grouped (per-head) output, tails and an odd number of
    K blocks, MN- and K-major operands, against torch."""
    for (M, N, K, at, bt, cgrp) in [(768, 3072, 4096, 1, 0, 0), (3072, 768, 4096, 1, 0, 0),
                                    (768, 768, 4096, 1, 0, 0), (768, 2304, 4096, 1, 0, 64),
                                    (200, 160, 1000, 1, 0, 0), (200, 136, 1000, 1, 0, 0),
                                    (384, 512, 192, 1, 0, 0), (512, 1024, 512, 0, 1, 0),
                                    (300, 700, 1000, 1, 0, 0)]:
        res = run_gemm(M, N, K, torch.bfloat16, at, bt, path=0, c_dtype=torch.float32, c_group=cgrp, seed=7)
        _check(res, torch.bfloat16, K)


def _kern_ref(name, dt, a, b, y, s, extra=None):
    """numpy restatement of hetpar::kern::scalar (kernels_scalar.cpp:12-83):
    IEEE-rounded elementwise ops, the L-lane reduction order."""
    T = dt.type
    L = 8 if dt == np.float32 else 4
    n = len(a)
    n0 = n - n % L
    if name in ("dot", "sum", "maxv"):
        acc = np.full(L, -np.inf if name == "maxv" else 0, dt)
        for i in range(0, n0, L):
            if name == "dot":
                acc = acc + a[i:i + L] * b[i:i + L]
            elif name == "sum":
                acc = acc + a[i:i + L]
            else:
                acc = np.where(a[i:i + L] > acc, a[i:i + L], acc)
        r = acc[0]
        for k in range(1, L):
            r = (acc[k] if acc[k] > r else r) if name == "maxv" else T(r + acc[k])
        for i in range(n0, n):
            if name == "dot":
                r = T(r + T(a[i] * b[i]))
            elif name == "sum":
                r = T(r + a[i])
            else:
                r = a[i] if a[i] > r else r
        return np.array([r], dt)
    if name == "add":
        return a + b
    if name == "scale":
        return a * T(s)
    if name == "axpy":
        return y + T(s) * a
    if name == "relu":
        return np.where(a > 0, a, T(0))
    if name == "relu_bwd":
        return y + np.where(a > 0, b, T(0))
    if name == "sgd_update":
        return y - T(s) * a
    raise ValueError(name)


@pytest.mark.parametrize("sfx", ["f32", "f64"])
def test_operator_table_bit_exact_vs_reference_kernels(sfx):
    """hp_kern_* (the reference's operator table on device pointers) equal
    the reference's scalar kernels bit for bit, tails included."""
    L = _lib()
    dt = np.dtype(np.float32 if sfx == "f32" else np.float64)
    tdt = torch.float32 if sfx == "f32" else torch.float64
    rng = np.random.default_rng(3)
    n = 1003
    a = rng.standard_normal(n).astype(dt)
    b = rng.standard_normal(n).astype(dt)
    y = rng.standard_normal(n).astype(dt)
    cs = C.c_float if sfx == "f32" else C.c_double
    keep = []  # device copies stay alive until the kernels that read them have run

    def dev(x):
        t = torch.from_numpy(x.copy()).to("cuda")
        keep.append(t)
        return t
    for name in ("dot", "sum", "maxv"):
        out = torch.zeros(1, dtype=tdt, device="cuda")
        args = (_ptr(dev(a)), _ptr(dev(b))) if name == "dot" else (_ptr(dev(a)),)
        L.call(f"hp_kern_{name}_{sfx}", *args, n, _ptr(out), None)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == _kern_ref(name, dt, a, b, y, 0).tobytes(), name
    s = dt.type(0.37)
    cases = {"add": lambda o: (_ptr(dev(a)), _ptr(dev(b)), _ptr(o), n),
             "scale": lambda o: (_ptr(dev(a)), cs(s), _ptr(o), n),
             "relu": lambda o: (_ptr(dev(a)), _ptr(o), n)}
    for name, argf in cases.items():
        o = torch.zeros(n, dtype=tdt, device="cuda")
        L.call(f"hp_kern_{name}_{sfx}", *argf(o), None)
        torch.cuda.synchronize()
        assert o.cpu().numpy().tobytes() == _kern_ref(name, dt, a, b, y, s).tobytes(), name
    yy = dev(y)
    L.call(f"hp_kern_axpy_{sfx}", cs(s), _ptr(dev(a)), _ptr(yy), n, None)
    torch.cuda.synchronize()
    assert yy.cpu().numpy().tobytes() == _kern_ref("axpy", dt, a, b, y, s).tobytes()
    yy = dev(y)
    L.call(f"hp_kern_relu_bwd_{sfx}", _ptr(dev(a)), _ptr(dev(b)), _ptr(yy), n, None)
    torch.cuda.synchronize()
    assert yy.cpu().numpy().tobytes() == _kern_ref("relu_bwd", dt, a, b, y, 0).tobytes()
    yy = dev(y)
    L.call(f"hp_kern_sgd_update_{sfx}", _ptr(yy), _ptr(dev(a)), n, cs(s), None)
    torch.cuda.synchronize()
    assert yy.cpu().numpy().tobytes() == _kern_ref("sgd_update", dt, a, b, y, s).tobytes()
    # adam_update (kernels_scalar.cpp:74-83)
    T = dt.type
    p, m, v, g = (rng.standard_normal(n).astype(dt) for _ in range(4))
    v = np.abs(v)
    lr, b1, b2, eps, c1, c2 = (T(x) for x in (1e-3, 0.9, 0.98, 1e-9, 1 / (1 - 0.9 ** 3), 1 / (1 - 0.98 ** 3)))
    dp, dm, dv = dev(p), dev(m), dev(v)
    L.call(f"hp_kern_adam_update_{sfx}", _ptr(dp), _ptr(dm), _ptr(dv), _ptr(dev(g)), n,
           *(cs(x) for x in (lr, b1, b2, eps, c1, c2)), None)
    torch.cuda.synchronize()
    m2 = b1 * m + (T(1) - b1) * g
    v2 = b2 * v + (T(1) - b2) * (g * g)
    p2 = p - lr * ((m2 * c1) / (np.sqrt(v2 * c2) + eps))
    assert dm.cpu().numpy().tobytes() == m2.tobytes()
    assert dv.cpu().numpy().tobytes() == v2.tobytes()
    assert dp.cpu().numpy().tobytes() == p2.tobytes()


@pytest.mark.parametrize("d", [64, 256, 512, 768, 1024])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("T", [1, 37, 4096])
def test_layernorm_fwd_bwd_vs_torch(d, dtype, T):
    """The engine's LayerNorm forward / backward (bf16 with d % 256 == 0 runs
    the bulk-copy kernels ln_fwd_bulk / ln_bwd_bulk + ln_part_final the C2 and
    C4 steps use) against torch fp32 autograd: y, dx, dgamma, dbeta and the
    fused bias gradient colsum(dx); deferred (engine) and direct finals."""
    L = _lib()
    g = torch.Generator(device="cpu").manual_seed(d + T)
    x = (torch.randn(T, d, generator=g) * 2 + 0.5).to("cuda", dtype)
    gam = (1 + 0.1 * torch.randn(d, generator=g)).cuda()
    bet = (0.1 * torch.randn(d, generator=g)).cuda()
    dy = torch.randn(T, d, generator=g).to("cuda", dtype)
    xr = x.float().requires_grad_(True)
    gr = gam.clone().requires_grad_(True)
    br = bet.clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xr, (d,), gr, br, eps=1e-12)
    ref.backward(dy.float())
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    for deferred in (1, 0):
        y = torch.zeros_like(x)
        dx = torch.zeros_like(x)
        mean = torch.zeros(T, device="cuda")
        rstd = torch.zeros(T, device="cuda")
        dg, db, dbias = (torch.zeros(d, device="cuda") for _ in range(3))
        L.call("hp_debug_layernorm", T, d, int(dtype == torch.bfloat16), _ptr(x), _ptr(gam), _ptr(bet),
               _ptr(y), _ptr(mean), _ptr(rstd), _ptr(dy), _ptr(dx), _ptr(dg), _ptr(db), _ptr(dbias),
               deferred)
        rel = lambda a, b: ((a.float() - b).norm() / b.norm().clamp_min(1e-30)).item()
        assert rel(y, ref.detach()) < tol
        assert rel(mean, xr.detach().mean(1)) < 1e-4
        assert rel(dx, xr.grad) < tol
        assert rel(dg, gr.grad) < tol
        assert rel(db, br.grad) < tol
        # colsum of the dx the kernel wrote (what the next kernel reads)
        assert rel(dbias, dx.float().sum(0)) < 1e-4 + (1e-3 if T > 1 else 0)


def _attn2_ref(q, k, v, cu_q, cu_kv, H, dk, causal, dO):
    """torch fp32 autograd reference: per instance and head softmax(q k^T /
    sqrt(dk)) v over the instance's keys, causal mask j <= i."""
    q = q.float().detach().requires_grad_(True)
    k = k.float().detach().requires_grad_(True)
    v = v.float().detach().requires_grad_(True)
    outs = []
    for b in range(len(cu_q) - 1):
        a, e = cu_q[b], cu_q[b + 1]
        c, f = cu_kv[b], cu_kv[b + 1]
        qq = q[a:e].reshape(e - a, H, dk)
        kk = k[c:f].reshape(f - c, H, dk)
        vv = v[c:f].reshape(f - c, H, dk)
        s = torch.einsum("qhd,khd->hqk", qq, kk) / dk ** 0.5
        if causal:
            s = s.masked_fill(torch.ones(e - a, f - c, device=s.device).triu(1).bool(), float("-inf"))
        outs.append(torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), vv).reshape(e - a, H * dk))
    o = torch.cat(outs)
    o.backward(dO.float())
    return o.detach(), q.grad, k.grad, v.grad


@pytest.mark.parametrize("path,dtype", [(3, torch.bfloat16), (1, torch.float32), (1, torch.bfloat16)])
@pytest.mark.parametrize("mode", ["cross", "causal"])
def test_attention_cross_and_causal(path, dtype, mode):
    """Generalised attention (AttnArgs): cross-attention with queries from one
    tensor and keys / values from another, different lengths per side (the
    seq2seq decoder's encoder-decoder attention), and causal self-attention
    over packed QKV (the decoder's self-attention), against torch fp32."""
    L = _lib()
    H, dk = 3, 64
    g = torch.Generator(device="cpu").manual_seed(7)
    if mode == "cross":
        lq, lk = [64, 1, 17, 128, 40], [64, 90, 3, 128, 7]
    else:
        lq = lk = [64, 1, 17, 128, 100]
    cq = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
    ck = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
    Tq, Tk, d = int(cq[-1]), int(ck[-1]), H * dk
    if mode == "cross":
        qb = (torch.randn(Tq, d, generator=g) * 1.5).to("cuda", dtype)
        kvb = (torch.randn(Tk, 2 * d, generator=g) * 1.5).to("cuda", dtype)
        q, ldq, qcol = qb, d, 0
        k, ldk, kcol = kvb, 2 * d, 0
        v, ldv, vcol = kvb, 2 * d, d
        q_l, k_l, v_l = qb, kvb[:, :d], kvb[:, d:]
        dq = torch.zeros_like(qb)
        dkv = torch.zeros_like(kvb)
        outs = (dq, d, 0, dkv, 2 * d, 0, dkv, 2 * d, d)
    else:
        qkv = (torch.randn(Tq, 3 * d, generator=g) * 1.5).to("cuda", dtype)
        q = k = v = qkv
        ldq = ldk = ldv = 3 * d
        qcol, kcol, vcol = 0, d, 2 * d
        q_l, k_l, v_l = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
        dqkv = torch.zeros_like(qkv)
        outs = (dqkv, 3 * d, 0, dqkv, 3 * d, d, dqkv, 3 * d, 2 * d)
    dO = torch.randn(Tq, d, generator=g).to("cuda", dtype)
    o = torch.zeros(Tq, d, device="cuda", dtype=dtype)
    lse = torch.zeros(H, Tq, device="cuda")
    dcq, dck = torch.from_numpy(cq).cuda(), torch.from_numpy(ck).cuda()
    L.call("hp_debug_attention2", len(lq), _ptr(dcq), _ptr(dck), Tq, Tk, max(lq), max(lk), H, dk,
           int(dtype == torch.bfloat16), _ptr(q), ldq, qcol, _ptr(k), ldk, kcol, _ptr(v), ldv, vcol,
           _ptr(o), _ptr(lse), _ptr(dO), _ptr(outs[0]), outs[1], outs[2], _ptr(outs[3]), outs[4],
           outs[5], _ptr(outs[6]), outs[7], outs[8], int(mode == "causal"), path)
    ref, gq, gk, gv = _attn2_ref(q_l, k_l, v_l, cq.tolist(), ck.tolist(), H, dk, mode == "causal", dO)
    if mode == "cross":
        got_q, got_k, got_v = dq, dkv[:, :d], dkv[:, d:]
    else:
        got_q, got_k, got_v = dqkv[:, :d], dqkv[:, d:2 * d], dqkv[:, 2 * d:]
    tol = 3e-2 if dtype == torch.bfloat16 else 1e-4
    for got, want in ((o, ref), (got_q, gq), (got_k, gk), (got_v, gv)):
        err = (got.float() - want).abs().max().item() / want.abs().max().item()
        assert err < tol, (mode, err)


@pytest.mark.parametrize("a_trans,b_trans", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_x6_fp32_gemm_on_tensor_cores(a_trans, b_trans):
    """fp32 operands on the tcgen05 kernel through the bf16x6 split (path 4):
    fp32-level accuracy -- within 3x of the fp32 SIMT kernel's error against
    the same torch fp32 reference, or 5e-6 of the output scale -- for every
    operand major-ness, grouped per-head B (dk 32 and 64), GELU / dGELU /
    residual / accumulate epilogues and grouped C."""
    cases = [dict(M=300, N=200, K=1000), dict(M=128, N=96, K=64, group=32),
             dict(M=256, N=192, K=128, group=64), dict(M=512, N=256, K=384, bias=True, act=1),
             dict(M=256, N=256, K=256, act=2, resid=True), dict(M=200, N=128, K=512, accumulate=True),
             dict(M=256, N=256, K=200, c_group=64)]
    for c in cases:
        if c.get("group") and (c["group"] and ((not b_trans and c["N"] % c["group"]) or (b_trans and c["K"] % c["group"]))):
            continue
        kw = {k: v for k, v in c.items() if k not in ("M", "N", "K")}
        x6 = run_gemm(c["M"], c["N"], c["K"], torch.float32, a_trans, b_trans, path=4, seed=3, **kw)
        simt = run_gemm(c["M"], c["N"], c["K"], torch.float32, a_trans, b_trans, path=1, seed=3, **kw)
        scale = x6["ref"].abs().max().item()
        e6 = (x6["out"] - x6["ref"]).abs().max().item()
        es = (simt["out"] - simt["ref"]).abs().max().item()
        assert e6 <= max(3 * es, 5e-6 * scale), (c, e6, es, scale)
