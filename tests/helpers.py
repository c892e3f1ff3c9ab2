"""Shared test helpers: golden fixtures, the C oracle (ctypes), oracle batches."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libhetpar_oracle.so")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "hetpar_ref")
REF_SRC = "/root/reference/proj"

RECORD_KEYS = ("tok_off", "tokens", "segments", "mask_off", "mask_pos", "mask_orig", "label")

# C1: reference masked_token_model d128 h4 V1000, seq 63, 8/rank, W=2
C1_SPEC = dict(arch="masked_token_model", d_model=128, heads=4, vocab=1000, max_seq=64,
               with_nsp=True, label_smooth_eps=0.1)
C1_GEN = dict(n=160, vocab=1000, min_sentence_words=30, max_sentence_words=30, seed=7)


def golden(name: str):
    return np.load(os.path.join(GOLD, name))


def oracle_lib():
    """The C restatement (test infrastructure); built on demand with gcc."""
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True,
                       capture_output=True)
    lib = C.CDLL(ORACLE_SO)
    f, u, p = C.c_float, C.c_uint64, C.c_void_p
    lib.orc_adam_update_f32.argtypes = [p, p, p, p, u, f, f, f, f, f, f]
    lib.orc_adam_update_f32.restype = None
    lib.orc_sgd_update_f32.argtypes = [p, p, u, f]
    lib.orc_sgd_update_f32.restype = None
    return lib


class OracleMlmCfg(C.Structure):
    _fields_ = [("n", C.c_uint64), ("vocab", C.c_int64), ("docs", C.c_uint64),
                ("sentences_per_doc", C.c_uint64), ("min_words", C.c_uint64),
                ("max_words", C.c_uint64), ("p_select", C.c_double), ("p_mask", C.c_double),
                ("p_random", C.c_double), ("seed", C.c_uint64), ("max_seq_tokens", C.c_uint64)]


def oracle_records(n, vocab, min_words, max_words, seed, docs=8, spd=12, max_seq_tokens=0):
    lib = oracle_lib()
    cfg = OracleMlmCfg(n, vocab, docs, spd, min_words, max_words, 0.15, 0.8, 0.1, seed,
                       max_seq_tokens)
    cap = n * (2 * max_words + 3)
    out = dict(tok_off=np.zeros(n + 1, np.uint64), tokens=np.zeros(cap, np.int64),
               segments=np.zeros(cap, np.int64), mask_off=np.zeros(n + 1, np.uint64),
               mask_pos=np.zeros(cap, np.int64), mask_orig=np.zeros(cap, np.int64),
               label=np.zeros(n, np.int64))
    p = lambda a: C.c_void_p(a.ctypes.data)
    rc = lib.orc_mlm_generate(C.byref(cfg), C.c_uint64(cap), C.c_uint64(cap), p(out["tok_off"]),
                              p(out["tokens"]), p(out["segments"]), p(out["mask_off"]),
                              p(out["mask_pos"]), p(out["mask_orig"]), p(out["label"]))
    assert rc == 0, rc
    nt, nm = int(out["tok_off"][-1]), int(out["mask_off"][-1])
    for k in ("tokens", "segments"):
        out[k] = out[k][:nt]
    for k in ("mask_pos", "mask_orig"):
        out[k] = out[k][:nm]
    return out


def oracle_instances(rec, ids):
    """Records (dict of CSR arrays or api.Records) -> model_oracle Instances."""
    import model_oracle as mo
    g = (lambda k: rec[k]) if isinstance(rec, dict) or hasattr(rec, "files") else (lambda k: getattr(rec, k))
    to, mo_ = g("tok_off").astype(np.int64), g("mask_off").astype(np.int64)
    out = []
    for i in ids:
        i = int(i)
        a, b = to[i], to[i + 1]
        c, d = mo_[i], mo_[i + 1]
        out.append(mo.Instance(g("tokens")[a:b], g("segments")[a:b], g("mask_pos")[c:d],
                               g("mask_orig")[c:d], int(g("label")[i]), int(b - a)))
    return out


def rel_norm(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
