"""TEST INFRASTRUCTURE, NOT PRODUCT CODE -- a torch fp32 autograd restatement
of the ``bert_encoder`` model math of model_oracle.py, used only as a checker
by tests/ (the C2 / C4 benchmark-shape parity tests, where the numpy f64
oracle would be too slow at BERT-large size).

It restates the same functions as model_oracle.forward_backward:
  embedding E[tok] + seg_s + sinusoidal PE (attention.hpp:53-67, PE in double
  then cast), embedding LayerNorm, per layer post-LN blocks
  LN1(x + MHA(x) Wo + bo), LN2(x1 + GELU(x1 W1 + b1) W2 + b2) with the
  per-head [d x dk] projection blocks wq.i / wk.i / wv.i and the concat_cols
  head order (attention.hpp:31-50), the MLM head with label-smoothed CE
  summed over the masked rows (tape.hpp:180-209) and the NSP head with plain
  CE (model.hpp:381-388); the gradient of the summed loss w.r.t. the flat
  canonical parameter vector (backward_gradients, model.hpp:405-417).

Pinned against model_oracle at small shapes by tests/test_oracle.py (CPU).
TF32 is switched off: every contraction is IEEE fp32.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

import model_oracle as mo


def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False


def forward_backward(s: mo.Spec, flat, batch, device="cuda", need_grad=True, policy="sentences"):
    """(loss_sum, weight, flat fp32 gradient as a torch tensor on `device`)."""
    if s.arch != "bert_encoder":
        raise ValueError("torch restatement covers bert_encoder only")
    _no_tf32()
    offs = mo.offsets(s)
    leaf = torch.as_tensor(np.asarray(flat, np.float32), device=device).clone()
    leaf.requires_grad_(need_grad)
    P = {n: leaf[o:o + r * c].view(r, c) for n, (o, r, c) in offs.items()}
    d, H, dk = s.d_model, s.heads, s.dk
    eps = s.label_smooth_eps
    layers = []
    for l in range(s.layers):
        p = f"layer{l}."
        wq = torch.cat([P[f"{p}wq.{i}"] for i in range(H)], 1)
        wk = torch.cat([P[f"{p}wk.{i}"] for i in range(H)], 1)
        wv = torch.cat([P[f"{p}wv.{i}"] for i in range(H)], 1)
        layers.append((p, wq, wk, wv))
    pe_all = torch.as_tensor(mo.sinusoidal_positions(s.max_seq, d).astype(np.float32), device=device)
    total = torch.zeros((), device=device)
    weight = 0.0
    for inst in batch:
        tok = torch.as_tensor(np.asarray(inst.tokens, np.int64), device=device)
        seg = torch.as_tensor(np.asarray(inst.segments, np.int64), device=device)
        n = tok.numel()
        x = P["embed"][tok] + torch.where(seg[:, None] == 0, P["seg0"], P["seg1"]) + pe_all[:n]
        x = F.layer_norm(x, (d,), P["emb_ln.g"][0], P["emb_ln.b"][0], eps=mo.LN_EPS)
        for p, wq, wk, wv in layers:
            q = (x @ wq).view(n, H, dk).transpose(0, 1)
            k = (x @ wk).view(n, H, dk).transpose(0, 1)
            v = (x @ wv).view(n, H, dk).transpose(0, 1)
            a = torch.softmax((q @ k.transpose(1, 2)) * (1.0 / dk ** 0.5), dim=-1) @ v
            cat = a.transpose(0, 1).reshape(n, d)
            x1 = F.layer_norm(x + cat @ P[p + "wo"] + P[p + "bo"][0], (d,), P[p + "ln1.g"][0],
                              P[p + "ln1.b"][0], eps=mo.LN_EPS)
            f = F.gelu(x1 @ P[p + "ffn.w1"] + P[p + "ffn.b1"][0]) @ P[p + "ffn.w2"] + P[p + "ffn.b2"][0]
            x = F.layer_norm(x1 + f, (d,), P[p + "ln2.g"][0], P[p + "ln2.b"][0], eps=mo.LN_EPS)
        inst_w = 0.0
        mpos = np.asarray(inst.mask_positions, np.int64)
        if mpos.size:
            hm = x[torch.as_tensor(mpos, device=device)]
            z = hm @ P["mlm.w"] + P["mlm.b"][0]
            tgt = torch.as_tensor(np.asarray(inst.mask_originals, np.int64), device=device)
            total = total + F.cross_entropy(z, tgt, label_smoothing=eps, reduction="sum")
            inst_w += mpos.size
        if s.with_nsp:
            z = x[0:1] @ P["nsp.w"] + P["nsp.b"][0]
            total = total + F.cross_entropy(z, torch.tensor([int(inst.label)], device=device),
                                            reduction="sum")
            inst_w += 1.0
        weight += 1.0 if policy == "sentences" else inst_w
    grad = None
    if need_grad:
        total.backward()
        grad = leaf.grad.detach()
    return float(total.detach()), weight, grad


def adam_update_f32(p, m, v, g, t, lr, beta1=0.9, beta2=0.98, eps=1e-9):
    """Optimizer<float>::step -> kern::adam_update<float> (optim.hpp:107-146,
    kernels_scalar.cpp:74-83) on torch fp32 tensors: c1, c2 in double then cast,
    g = (float) g, no fused multiply-adds (separate elementwise kernels).
    Returns the new (p, m, v)."""
    c1 = torch.tensor(1.0 / (1.0 - beta1 ** t), dtype=torch.float32)
    c2 = torch.tensor(1.0 / (1.0 - beta2 ** t), dtype=torch.float32)
    b1 = torch.tensor(beta1, dtype=torch.float32)
    b2 = torch.tensor(beta2, dtype=torch.float32)
    one = torch.tensor(1.0, dtype=torch.float32)
    e = torch.tensor(eps, dtype=torch.float32)
    lr_ = torch.tensor(lr, dtype=torch.float32)
    dev = p.device
    b1, b2, one, e, lr_, c1, c2 = (x.to(dev) for x in (b1, b2, one, e, lr_, c1, c2))
    m = b1 * m + (one - b1) * g
    v = b2 * v + (one - b2) * (g * g)
    p = p - lr_ * ((m * c1) / (torch.sqrt(v * c2) + e))
    return p, m, v
