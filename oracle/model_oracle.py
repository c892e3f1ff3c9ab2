"""TEST INFRASTRUCTURE, NOT PRODUCT CODE -- numpy f64 restatement of the
reference model math (arxiv/paper_2009_14783 "hetpar"), used only as the
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.

Pinned parity: for ``masked_token_model`` (model.hpp:334-393) every function
here is checked against the reference compiled from /root/reference
(oracle/_ref, fixtures in tests/golden/, made by tools/make_golden.py): the
per-rank pre-reduce gradients and the 10-step C1 trajectory.

The ``bert_encoder`` extension (LayerNorm, GELU FFN, residual, L layers) has
NO reference counterpart: it follows the Tape conventions (tape.hpp:21-324)
and the parameter naming/order convention (model.hpp:91-142) and is pinned
only by finite differences (tests/test_model_oracle.py) -- "parity unpinned"
against the reference itself, as DESIGN.md states.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
LN_EPS = 1e-12  # extension only; BERT's LayerNorm epsilon


# --------------------------------------------------------------------------
# spec / parameter table (model.hpp:28-142)
@dataclass
class Spec:
    arch: str = "masked_token_model"  # or "bert_encoder" (repo extension)
    d_model: int = 128
    heads: int = 4
    vocab: int = 1000
    max_seq: int = 512
    layers: int = 1  # bert_encoder only
    d_ff: int = 512  # bert_encoder only
    with_nsp: bool = True
    label_smooth_eps: float = 0.1

    @property
    def dk(self) -> int:
        return self.d_model // self.heads


def param_shapes(s: Spec):
    """Canonical (name, rows, cols, row_table, bias) list, model.hpp:91-142.
    bert_encoder extends the pattern with ``layer{l}.`` prefixes."""
    out = []
    w = lambda n, r, c: out.append((n, r, c, False, False))
    tbl = lambda n, r, c: out.append((n, r, c, True, False))
    b = lambda n, c: out.append((n, 1, c, False, True))
    d, dk = s.d_model, s.dk

    def attn(prefix):
        for kind in ("wq", "wk", "wv"):
            for i in range(s.heads):
                w(f"{prefix}{kind}.{i}", d, dk)
        w(f"{prefix}wo", d, d)

    if s.arch == "masked_token_model":
        tbl("embed", s.vocab, d)
        tbl("seg0", 1, d)
        tbl("seg1", 1, d)
        attn("")
    elif s.arch == "bert_encoder":
        tbl("embed", s.vocab, d)
        tbl("seg0", 1, d)
        tbl("seg1", 1, d)
        out.append(("emb_ln.g", 1, d, False, False))
        b("emb_ln.b", d)
        for l in range(s.layers):
            p = f"layer{l}."
            attn(p)
            b(p + "bo", d)
            out.append((p + "ln1.g", 1, d, False, False))
            b(p + "ln1.b", d)
            w(p + "ffn.w1", d, s.d_ff)
            b(p + "ffn.b1", s.d_ff)
            w(p + "ffn.w2", s.d_ff, d)
            b(p + "ffn.b2", d)
            out.append((p + "ln2.g", 1, d, False, False))
            b(p + "ln2.b", d)
    else:
        raise ValueError(s.arch)
    w("mlm.w", d, s.vocab)
    b("mlm.b", s.vocab)
    if s.with_nsp:
        w("nsp.w", d, 2)
        b("nsp.b", 2)
    return out


def flat_size(s: Spec) -> int:
    return sum(r * c for _, r, c, _, _ in param_shapes(s))


def offsets(s: Spec):
    off, o = {}, 0
    for n, r, c, _, _ in param_shapes(s):
        off[n] = (o, r, c)
        o += r * c
    return off


def splitmix_doubles(seed: int, start: int, n: int) -> np.ndarray:
    """Draws start..start+n-1 of next_double() (rng.hpp:15-27). splitmix64 is
    counter based: draw k mixes seed + (k+1)*gamma."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def init_parameters(s: Spec, seed: int) -> np.ndarray:
    """model.hpp:171-184 with derived_rng(seed, 0): U(-a,a), a=1/sqrt(fan_in).
    LayerNorm gains (extension) initialise to 1 and draw nothing."""
    out = np.zeros(flat_size(s))
    o, k = 0, 0
    for name, r, c, row_table, bias in param_shapes(s):
        n = r * c
        if name.endswith(".g"):
            out[o:o + n] = 1.0
        elif not bias:
            a = 1.0 / math.sqrt(c if row_table else r)
            u = splitmix_doubles(seed, k, n)
            out[o:o + n] = -a + 2.0 * a * u
            k += n
        o += n
    return out


def sinusoidal_positions(n: int, d: int) -> np.ndarray:
    """attention.hpp:53-67, computed in double."""
    pos = np.arange(n, dtype=np.float64)[:, None]
    i = np.arange(d // 2, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, (2.0 * i) / d)
    pe = np.zeros((n, d))
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang)
    return pe


# --------------------------------------------------------------------------
# primitives (tape.hpp) with their backward rules
def softmax_rows(z):  # tape.hpp:123-140
    e = np.exp(z - z.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def ls_ce(z, targets, eps):
    """tape.hpp:180-209 (value) and 302-321 (gradient wrt z for go = 1)."""
    V = z.shape[1]
    mx = z.max(axis=1, keepdims=True)
    e = np.exp(z - mx)
    se = e.sum(axis=1, keepdims=True)
    lse = (mx + np.log(se))[:, 0]
    rows = np.arange(z.shape[0])
    loss = float(np.sum(lse - (1 - eps) * z[rows, targets] - (eps / V) * z.sum(axis=1)))
    dz = e / se - eps / V
    dz[rows, targets] -= 1 - eps
    return loss, dz


def layer_norm(x, g, b):
    mu = x.mean(axis=1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xh = xc * rstd
    return xh * g + b, (xh, rstd)


def layer_norm_bwd(dy, g, cache):
    xh, rstd = cache
    dg = (dy * xh).sum(axis=0)
    db = dy.sum(axis=0)
    dxh = dy * g
    d = xh.shape[1]
    dx = rstd / d * (d * dxh - dxh.sum(axis=1, keepdims=True)
                     - xh * (dxh * xh).sum(axis=1, keepdims=True))
    return dx, dg, db


def gelu(u):  # exact erf GELU (BERT)
    from scipy.special import erf
    return 0.5 * u * (1.0 + erf(u / math.sqrt(2.0)))


def gelu_grad(u):
    from scipy.special import erf
    cdf = 0.5 * (1.0 + erf(u / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * u * u) / math.sqrt(2.0 * math.pi)
    return cdf + u * pdf


# --------------------------------------------------------------------------
@dataclass
class Instance:
    tokens: np.ndarray
    segments: np.ndarray
    mask_positions: np.ndarray
    mask_originals: np.ndarray
    label: int = 0
    token_length: int = 0


def _mha_fwd(x, P, prefix, s):
    d, h, dk = s.d_model, s.heads, s.dk
    scale = 1.0 / math.sqrt(dk)  # attention.hpp:22-23
    heads = []
    cache = []
    for i in range(h):
        q = x @ P[f"{prefix}wq.{i}"]
        k = x @ P[f"{prefix}wk.{i}"]
        v = x @ P[f"{prefix}wv.{i}"]
        p = softmax_rows((q @ k.T) * scale)
        heads.append(p @ v)
        cache.append((q, k, v, p))
    cat = np.concatenate(heads, axis=1)  # concat_cols order
    return cat @ P[f"{prefix}wo"], (cat, cache)


def _mha_bwd(dout, x, P, G, prefix, s, mcache):
    cat, cache = mcache
    dk = s.dk
    scale = 1.0 / math.sqrt(dk)
    G[f"{prefix}wo"] += cat.T @ dout
    dcat = dout @ P[f"{prefix}wo"].T
    dx = np.zeros_like(x)
    for i, (q, k, v, p) in enumerate(cache):
        dh = dcat[:, i * dk:(i + 1) * dk]
        dp = dh @ v.T
        dv = p.T @ dh
        ds = p * (dp - (dp * p).sum(axis=1, keepdims=True)) * scale
        dq = ds @ k
        dkk = ds.T @ q
        for kind, dd in (("wq", dq), ("wk", dkk), ("wv", dv)):
            G[f"{prefix}{kind}.{i}"] += x.T @ dd
            dx += dd @ P[f"{prefix}{kind}.{i}"].T
    return dx


def forward_backward(s: Spec, flat: np.ndarray, batch, policy="sentences",
                     need_grad=True):
    """model_forward (model.hpp:260-403) + backward_gradients (405-417) for
    one batch: returns (loss_sum, weight, flat f64 gradient)."""
    offs = offsets(s)
    P = {n: flat[o:o + r * c].reshape(r, c) for n, (o, r, c) in offs.items()}
    grad = np.zeros_like(flat)
    G = {n: grad[o:o + r * c].reshape(r, c) for n, (o, r, c) in offs.items()}
    eps = s.label_smooth_eps
    loss_total, weight = 0.0, 0.0
    for inst in batch:
        tok = np.asarray(inst.tokens, dtype=np.int64)
        seg = np.asarray(inst.segments, dtype=np.int64)
        n = tok.size
        if n == 0 or n > s.max_seq:
            raise ValueError("sequence length")
        x = P["embed"][tok] + np.where(seg[:, None] == 0, P["seg0"], P["seg1"]) \
            + sinusoidal_positions(n, s.d_model)
        caches = []
        if s.arch == "bert_encoder":
            x, emb_ln = layer_norm(x, P["emb_ln.g"], P["emb_ln.b"])
            for l in range(s.layers):
                p = f"layer{l}."
                a, mc = _mha_fwd(x, P, p, s)
                x1, ln1 = layer_norm(x + a + P[p + "bo"], P[p + "ln1.g"], P[p + "ln1.b"])
                u = x1 @ P[p + "ffn.w1"] + P[p + "ffn.b1"]
                gu = gelu(u)
                f = gu @ P[p + "ffn.w2"] + P[p + "ffn.b2"]
                x2, ln2 = layer_norm(x1 + f, P[p + "ln2.g"], P[p + "ln2.b"])
                caches.append((x, mc, x1, ln1, u, gu, ln2))
                x = x2
            hfin = x
        else:
            hfin, mc = _mha_fwd(x, P, "", s)
            caches.append((x, mc))
        dh = np.zeros_like(hfin)
        inst_w = 0.0
        mpos = np.asarray(inst.mask_positions, dtype=np.int64)
        if mpos.size:
            hm = hfin[mpos]
            z = hm @ P["mlm.w"] + P["mlm.b"]
            l, dz = ls_ce(z, np.asarray(inst.mask_originals, dtype=np.int64), eps)
            loss_total += l
            inst_w += mpos.size
            if need_grad:
                G["mlm.w"] += hm.T @ dz
                G["mlm.b"] += dz.sum(axis=0, keepdims=True)
                np.add.at(dh, mpos, dz @ P["mlm.w"].T)
        if s.with_nsp:
            h0 = hfin[0:1]
            z = h0 @ P["nsp.w"] + P["nsp.b"]
            l, dz = ls_ce(z, np.array([inst.label]), 0.0)
            loss_total += l
            inst_w += 1.0
            if need_grad:
                G["nsp.w"] += h0.T @ dz
                G["nsp.b"] += dz
                dh[0:1] += dz @ P["nsp.w"].T
        weight += 1.0 if policy == "sentences" else inst_w
        if not need_grad:
            continue
        if s.arch == "bert_encoder":
            dx = dh
            for l in reversed(range(s.layers)):
                p = f"layer{l}."
                xin, mc, x1, ln1, u, gu, ln2 = caches[l]
                dy2, dg2, db2 = layer_norm_bwd(dx, P[p + "ln2.g"], ln2)
                G[p + "ln2.g"] += dg2
                G[p + "ln2.b"] += db2
                G[p + "ffn.b2"] += dy2.sum(axis=0)
                G[p + "ffn.w2"] += gu.T @ dy2
                du = (dy2 @ P[p + "ffn.w2"].T) * gelu_grad(u)
                G[p + "ffn.b1"] += du.sum(axis=0)
                G[p + "ffn.w1"] += x1.T @ du
                dx1 = dy2 + du @ P[p + "ffn.w1"].T
                dy1, dg1, db1 = layer_norm_bwd(dx1, P[p + "ln1.g"], ln1)
                G[p + "ln1.g"] += dg1
                G[p + "ln1.b"] += db1
                G[p + "bo"] += dy1.sum(axis=0)
                dx = dy1 + _mha_bwd(dy1, xin, P, G, p, s, mc)
            dx, dge, dbe = layer_norm_bwd(dx, P["emb_ln.g"], emb_ln)
            G["emb_ln.g"] += dge
            G["emb_ln.b"] += dbe
        else:
            xin, mc = caches[0]
            dx = _mha_bwd(dh, xin, P, G, "", s, mc)
        np.add.at(G["embed"], tok, dx)
        G["seg0"] += dx[seg == 0].sum(axis=0)
        G["seg1"] += dx[seg == 1].sum(axis=0)
    return loss_total, weight, grad


# --------------------------------------------------------------------------
# protocol (engine.hpp:125-165) as the SerialOracle restates it
# (test_engine.cpp:87-127): rank-ordered fold, divide by total weight, one
# identical optimizer update.
@dataclass
class AdamState:
    beta1: float = 0.9
    beta2: float = 0.98
    eps: float = 1e-9
    t: int = 0
    m: np.ndarray | None = None
    v: np.ndarray | None = None


def adam_step(params, grad, st: AdamState, lr, dtype=np.float64):
    """optim.hpp:107-146 -> kern::adam_update (kernels_scalar.cpp:74-83):
    c1, c2 in double, then everything cast to the parameter dtype."""
    st.t += 1
    c1 = 1.0 / (1.0 - st.beta1 ** st.t)
    c2 = 1.0 / (1.0 - st.beta2 ** st.t)
    T = dtype
    if st.m is None:
        st.m = np.zeros(params.size, dtype=T)
        st.v = np.zeros(params.size, dtype=T)
    g = grad.astype(T)
    b1, b2, e, lr_, c1_, c2_ = (T(st.beta1), T(st.beta2), T(st.eps), T(lr), T(c1), T(c2))
    st.m = b1 * st.m + (T(1) - b1) * g
    st.v = b2 * st.v + (T(1) - b2) * (g * g)
    mh = st.m * c1_
    vh = st.v * c2_
    return params - lr_ * (mh / (np.sqrt(vh) + e))


def protocol_round(s, params, per_rank, policy="sentences"):
    """One lockstep round: per_rank = [(batch, dummy)]; returns the folded
    (loss_sum, weight, grad_sum)."""
    ls, ws, gs = [], [], []
    for batch, dummy in per_rank:
        if dummy:
            ls.append(0.0)
            ws.append(0.0)
            gs.append(np.zeros_like(params))
            continue
        l, w, g = forward_backward(s, params, batch, policy)
        ls.append(l)
        ws.append(w)
        gs.append(g)
    tot_l, tot_w, tot_g = ls[0], ws[0], gs[0].copy()
    for r in range(1, len(ls)):
        tot_l += ls[r]
        tot_w += ws[r]
        tot_g += gs[r]
    return tot_l, tot_w, tot_g
