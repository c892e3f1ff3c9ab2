"""TEST INFRASTRUCTURE, NOT PRODUCT CODE -- numpy f64 restatement of the
reference model math (arxiv/paper_2009_14783 "hetpar"), used only as the
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.

Pinned parity: for ``masked_token_model`` (model.hpp:334-393) every function
here is checked against the reference compiled from /root/reference
(oracle/_ref, fixtures in tests/golden/, made by tools/make_golden.py): the
per-rank pre-reduce gradients and the 10-step C1 trajectory.

The ``bert_encoder`` extension (LayerNorm, GELU FFN, residual, L layers) and
the ``transformer_seq2seq`` extension (the encoder-decoder Transformer of the
paper's translation workload: post-LN encoder and decoder
blocks, causal decoder self-attention, encoder-decoder cross-attention, one
embedding table shared by both inputs and the output projection) have NO
reference counterpart: they follow the Tape conventions (tape.hpp:21-324) and
the parameter naming/order convention (model.hpp:91-142) and are pinned only
by finite differences (tests/test_oracle.py) -- "parity unpinned" against the
reference itself, as DESIGN.md states.
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
    arch: str = "masked_token_model"  # or "bert_encoder" / "transformer_seq2seq" (extensions)
    d_model: int = 128
    heads: int = 4
    vocab: int = 1000
    max_seq: int = 512
    layers: int = 1  # bert_encoder; transformer_seq2seq: encoder = decoder layers
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
    elif s.arch == "transformer_seq2seq":
        tbl("embed", s.vocab, d)  # shared: encoder / decoder inputs, output projection
        for l in range(s.layers):
            p = f"enc{l}."
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
        for l in range(s.layers):
            p = f"dec{l}."
            attn(p)
            b(p + "bo", d)
            out.append((p + "ln1.g", 1, d, False, False))
            b(p + "ln1.b", d)
            for kind in ("cq", "ck", "cv"):
                for i in range(s.heads):
                    w(f"{p}{kind}.{i}", d, dk)
            w(p + "co", d, d)
            b(p + "cbo", d)
            out.append((p + "ln2.g", 1, d, False, False))
            b(p + "ln2.b", d)
            w(p + "ffn.w1", d, s.d_ff)
            b(p + "ffn.b1", s.d_ff)
            w(p + "ffn.w2", s.d_ff, d)
            b(p + "ffn.b2", d)
            out.append((p + "ln3.g", 1, d, False, False))
            b(p + "ln3.b", d)
        return out
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


BOS = 2  # decoder start token (fairseq's prev_output_tokens start with EOS = 2)


def _attn(q, k, v, causal, scale):
    z = (q @ k.T) * scale
    if causal:
        z = np.where(np.tril(np.ones(z.shape, bool)), z, -np.inf)
    p = softmax_rows(z)
    return p @ v, p


def _attn_bwd(dout, q, k, v, p, scale):
    dp = dout @ v.T
    dv = p.T @ dout
    ds = p * (dp - (dp * p).sum(axis=1, keepdims=True)) * scale
    return ds @ k, ds.T @ q, dv


def _heads(P, prefix, kinds, h):
    return [np.concatenate([P[f"{prefix}{kd}.{i}"] for i in range(h)], axis=1) for kd in kinds]


def _mha2_fwd(xq, xkv, P, prefix, kinds, out_w, s, causal):
    """multi-head attention with the per-head [d x dk] blocks of `kinds`
    (q, k, v), queries from xq, keys / values from xkv"""
    h, dk = s.heads, s.dk
    scale = 1.0 / math.sqrt(dk)
    wq, wk, wv = _heads(P, prefix, kinds, h)
    Q, K, Vv = xq @ wq, xkv @ wk, xkv @ wv
    outs, ps = [], []
    for i in range(h):
        sl = slice(i * dk, (i + 1) * dk)
        o, pr = _attn(Q[:, sl], K[:, sl], Vv[:, sl], causal, scale)
        outs.append(o)
        ps.append(pr)
    cat = np.concatenate(outs, axis=1)
    return cat @ P[prefix + out_w], (Q, K, Vv, ps, cat)


def _mha2_bwd(dout, xq, xkv, P, G, prefix, kinds, out_w, s, cache):
    h, dk = s.heads, s.dk
    scale = 1.0 / math.sqrt(dk)
    Q, K, Vv, ps, cat = cache
    G[prefix + out_w] += cat.T @ dout
    dcat = dout @ P[prefix + out_w].T
    dQ, dK, dV = np.zeros_like(Q), np.zeros_like(K), np.zeros_like(Vv)
    for i in range(h):
        sl = slice(i * dk, (i + 1) * dk)
        dq, dkk, dv = _attn_bwd(dcat[:, sl], Q[:, sl], K[:, sl], Vv[:, sl], ps[i], scale)
        dQ[:, sl], dK[:, sl], dV[:, sl] = dq, dkk, dv
    wq, wk, wv = _heads(P, prefix, kinds, h)
    for kd, dd, xx in ((kinds[0], dQ, xq), (kinds[1], dK, xkv), (kinds[2], dV, xkv)):
        gw = xx.T @ dd
        for i in range(h):
            G[f"{prefix}{kd}.{i}"] += gw[:, i * dk:(i + 1) * dk]
    return dQ @ wq.T, dK @ wk.T + dV @ wv.T


def _ffn_block_fwd(x, P, p, lnname):
    u = x @ P[p + "ffn.w1"] + P[p + "ffn.b1"]
    gu = gelu(u)
    f = gu @ P[p + "ffn.w2"] + P[p + "ffn.b2"]
    y, ln = layer_norm(x + f, P[p + lnname + ".g"], P[p + lnname + ".b"])
    return y, (x, u, gu, ln)


def _ffn_block_bwd(dy, P, G, p, lnname, cache):
    x, u, gu, ln = cache
    dy2, dg, db = layer_norm_bwd(dy, P[p + lnname + ".g"], ln)
    G[p + lnname + ".g"] += dg
    G[p + lnname + ".b"] += db
    G[p + "ffn.b2"] += dy2.sum(axis=0)
    G[p + "ffn.w2"] += gu.T @ dy2
    du = (dy2 @ P[p + "ffn.w2"].T) * gelu_grad(u)
    G[p + "ffn.b1"] += du.sum(axis=0)
    G[p + "ffn.w1"] += x.T @ du
    return dy2 + du @ P[p + "ffn.w1"].T


def seq2seq_split(inst):
    """Instance -> (source ids, decoder input ids, target ids): tokens holds
    the source (segment 0) then the target (segment 1); the decoder reads
    [BOS] + target[:-1] and predicts target."""
    tok = np.asarray(inst.tokens, dtype=np.int64)
    seg = np.asarray(inst.segments, dtype=np.int64)
    src, tgt = tok[seg == 0], tok[seg == 1]
    return src, np.concatenate([[BOS], tgt[:-1]]).astype(np.int64), tgt


def _seq2seq_forward_backward(s, P, G, batch, policy, need_grad):
    eps = s.label_smooth_eps
    d = s.d_model
    es = math.sqrt(d)  # embedding scale (fairseq embed_scale)
    loss_total, weight = 0.0, 0.0
    for inst in batch:
        src, din, tgt = seq2seq_split(inst)
        ns, nt = src.size, tgt.size
        if ns == 0 or nt == 0 or ns > s.max_seq or nt > s.max_seq:
            raise ValueError("sequence length")
        x = es * P["embed"][src] + sinusoidal_positions(ns, d)
        enc_c = []
        for l in range(s.layers):
            p = f"enc{l}."
            a, mc = _mha2_fwd(x, x, P, p, ("wq", "wk", "wv"), "wo", s, False)
            x1, ln1 = layer_norm(x + a + P[p + "bo"], P[p + "ln1.g"], P[p + "ln1.b"])
            x2, fc = _ffn_block_fwd(x1, P, p, "ln2")
            enc_c.append((x, mc, ln1, fc))
            x = x2
        mem = x
        y = es * P["embed"][din] + sinusoidal_positions(nt, d)
        dec_c = []
        for l in range(s.layers):
            p = f"dec{l}."
            a, mc = _mha2_fwd(y, y, P, p, ("wq", "wk", "wv"), "wo", s, True)
            y1, ln1 = layer_norm(y + a + P[p + "bo"], P[p + "ln1.g"], P[p + "ln1.b"])
            c, cc = _mha2_fwd(y1, mem, P, p, ("cq", "ck", "cv"), "co", s, False)
            y2, ln2 = layer_norm(y1 + c + P[p + "cbo"], P[p + "ln2.g"], P[p + "ln2.b"])
            y3, fc = _ffn_block_fwd(y2, P, p, "ln3")
            dec_c.append((y, mc, ln1, y1, cc, ln2, fc))
            y = y3
        z = y @ P["embed"].T  # tied output projection, no bias
        l_, dz = ls_ce(z, tgt, eps)
        loss_total += l_
        weight += 1.0 if policy == "sentences" else float(nt)
        if not need_grad:
            continue
        G["embed"] += dz.T @ y
        dy = dz @ P["embed"]
        dmem = np.zeros_like(mem)
        for l in reversed(range(s.layers)):
            p = f"dec{l}."
            yin, mc, ln1, y1, cc, ln2, fc = dec_c[l]
            dy2 = _ffn_block_bwd(dy, P, G, p, "ln3", fc)
            dc, dg2, db2 = layer_norm_bwd(dy2, P[p + "ln2.g"], ln2)
            G[p + "ln2.g"] += dg2
            G[p + "ln2.b"] += db2
            G[p + "cbo"] += dc.sum(axis=0)
            dq_in, dkv_in = _mha2_bwd(dc, y1, mem, P, G, p, ("cq", "ck", "cv"), "co", s, cc)
            dmem += dkv_in
            dy1 = dc + dq_in
            da, dg1, db1 = layer_norm_bwd(dy1, P[p + "ln1.g"], ln1)
            G[p + "ln1.g"] += dg1
            G[p + "ln1.b"] += db1
            G[p + "bo"] += da.sum(axis=0)
            dq_s, dkv_s = _mha2_bwd(da, yin, yin, P, G, p, ("wq", "wk", "wv"), "wo", s, mc)
            dy = da + dq_s + dkv_s
        np.add.at(G["embed"], din, es * dy)
        dx = dmem
        for l in reversed(range(s.layers)):
            p = f"enc{l}."
            xin, mc, ln1, fc = enc_c[l]
            dx1 = _ffn_block_bwd(dx, P, G, p, "ln2", fc)
            da, dg1, db1 = layer_norm_bwd(dx1, P[p + "ln1.g"], ln1)
            G[p + "ln1.g"] += dg1
            G[p + "ln1.b"] += db1
            G[p + "bo"] += da.sum(axis=0)
            dq_s, dkv_s = _mha2_bwd(da, xin, xin, P, G, p, ("wq", "wk", "wv"), "wo", s, mc)
            dx = da + dq_s + dkv_s
        np.add.at(G["embed"], src, es * dx)
    return loss_total, weight


def forward_backward(s: Spec, flat: np.ndarray, batch, policy="sentences",
                     need_grad=True):
    """model_forward (model.hpp:260-403) + backward_gradients (405-417) for
    one batch: returns (loss_sum, weight, flat f64 gradient)."""
    offs = offsets(s)
    if s.arch == "transformer_seq2seq":
        P = {n: flat[o:o + r * c].reshape(r, c) for n, (o, r, c) in offs.items()}
        grad = np.zeros_like(flat)
        G = {n: grad[o:o + r * c].reshape(r, c) for n, (o, r, c) in offs.items()}
        l, w = _seq2seq_forward_backward(s, P, G, batch, policy, need_grad)
        return l, w, grad
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


def adam_step(params, grad, st: AdamState, lr, dtype=np.float64, weight_decay=0.0):
    """optim.hpp:107-146 -> kern::adam_update (kernels_scalar.cpp:74-83):
    c1, c2 in double, then everything cast to the parameter dtype.
    weight_decay != 0: the AdamW extension, p -= (lr wd) p (in dtype) first."""
    st.t += 1
    c1 = 1.0 / (1.0 - st.beta1 ** st.t)
    c2 = 1.0 / (1.0 - st.beta2 ** st.t)
    T = dtype
    if st.m is None:
        st.m = np.zeros(params.size, dtype=T)
        st.v = np.zeros(params.size, dtype=T)
    g = grad.astype(T)
    b1, b2, e, lr_, c1_, c2_ = (T(st.beta1), T(st.beta2), T(st.eps), T(lr), T(c1), T(c2))
    if weight_decay:
        params = params - (lr_ * T(weight_decay)) * params
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


def pairs_generate(n, vocab, min_len, max_len, seed):
    """The seq2seq extension's synthetic pair stream (hp_pairs_generate,
    include/hetpar_b200.h): per pair the source and target lengths, then the
    source and target word ids, all from one SeededRng(seed) stream
    (bounded(n) = hi64(u * n), rng.hpp:15-55).  Returns CSR (tok_off, tokens,
    segments)."""
    state = seed & (2**64 - 1)
    M = 2**64

    def nxt():
        nonlocal state
        state = (state + 0x9E3779B97F4A7C15) % M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % M
        return z ^ (z >> 31)

    def bounded(k):
        return (nxt() * k) >> 64

    tok_off, tokens, segments = [0], [], []
    for _ in range(n):
        ls = min_len + bounded(max_len - min_len + 1)
        lt = min_len + bounded(max_len - min_len + 1)
        for i in range(ls + lt):
            tokens.append(4 + bounded(vocab - 4))
            segments.append(0 if i < ls else 1)
        tok_off.append(len(tokens))
    return (np.array(tok_off, np.uint64), np.array(tokens, np.int64), np.array(segments, np.int64))
