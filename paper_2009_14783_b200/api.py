"""Host-side mirror of the reference's DP-step API (arxiv/paper_2009_14783
"hetpar", C++), over the C ABI in include/hetpar_b200.h.

Names, argument meaning and error behaviour follow the reference:
  ModelSpec / param_shapes / init_parameters      include/hetpar/model.hpp:28-184
  Instance / Batch                                model.hpp:72-83
  build_epoch_batches / partition_for_rank        src/dataset.cpp:52-117
  generate_mlm_records (generate_mlm_shards' stream) src/datagen.cpp:71-127
  StepEngine.round(batch, dummy) -> StepReport    include/hetpar/engine.hpp:114-165
  scheduled_lr                                    include/hetpar/optim.hpp:19-70
Errors are raised as the reference's taxonomy (ShapeError, ConfigError, ...).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (BaseError, CommError, ConfigError, CudaError, IndexError_, IoError,
                   NumericError, ShapeError, call)

__all__ = [
    "ModelSpec", "ParamShape", "param_shapes", "flat_size", "init_parameters", "bucket_plan",
    "Instance", "BatchCSR", "pack_batch", "BatchPlan", "RankBatch", "build_epoch_batches",
    "partition_for_rank", "MlmGenConfig", "Records", "generate_mlm_records", "splitmix64",
    "PairGenConfig", "generate_pair_records",
    "shuffle_iota", "OptimConfig", "ExecConfig", "StepReport", "Communicator", "StepEngine",
    "SchedulerConfig", "scheduled_lr", "inverse_sqrt_lr", "linear_warmup_decay_lr",
    "BaseError", "ShapeError", "ConfigError", "IndexError_", "IoError", "CommError",
    "NumericError", "CudaError",
]


def _p(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------- rng
def splitmix64(seed: int, n: int) -> np.ndarray:
    """SeededRng(seed).next_u64() x n (rng.hpp:15-22)."""
    out = np.empty(n, dtype=np.uint64)
    call("hp_splitmix64", seed & (2**64 - 1), n, _p(out))
    return out


def shuffle_iota(seed: int, n: int) -> np.ndarray:
    """shuffle(iota(n), SeededRng(seed)) (rng.hpp:74-82)."""
    out = np.empty(n, dtype=np.uint64)
    call("hp_shuffle_iota", seed & (2**64 - 1), n, _p(out))
    return out


# --------------------------------------------------------------------- model
_ARCH = {"masked_token_model": _lib.HP_ARCH_MASKED_TOKEN_MODEL,
         "bert_encoder": _lib.HP_ARCH_BERT_ENCODER,
         "transformer_seq2seq": _lib.HP_ARCH_SEQ2SEQ}
_POLICY = {"sentences": _lib.HP_POLICY_SENTENCES, "tokens": _lib.HP_POLICY_TOKENS}


@dataclass
class ModelSpec:
    """ModelSpec (model.hpp:28-67).  ``masked_token_model`` is exactly the
    reference architecture (one attention block); the repo extensions are
    ``bert_encoder`` (L post-LN blocks with a GELU FFN) and
    ``transformer_seq2seq`` (L encoder + L decoder blocks of the paper's
    translation Transformer, one embedding shared by the inputs and the output
    projection; a pair is an Instance whose tokens are the source (segment 0)
    then the target (segment 1), see generate_pair_records)."""
    arch: str = "masked_token_model"
    d_model: int = 128
    heads: int = 4
    vocab: int = 1000
    max_seq: int = 64
    layers: int = 1
    d_ff: int = 0
    with_nsp: bool = True
    label_smooth_eps: float = 0.1

    def desc(self) -> _lib.ModelDesc:
        if self.arch not in _ARCH:
            raise ConfigError(f"config: unsupported architecture {self.arch}")
        return _lib.ModelDesc(_ARCH[self.arch], self.d_model, self.heads, self.vocab, self.max_seq,
                              self.layers, self.d_ff, int(self.with_nsp), self.label_smooth_eps)


@dataclass
class ParamShape:
    name: str
    rows: int
    cols: int
    offset: int
    kind: int  # 0 weight, 1 row table, 2 bias, 3 LayerNorm gain

    @property
    def size(self) -> int:
        return self.rows * self.cols


def param_shapes(spec: ModelSpec) -> list[ParamShape]:
    """Canonical parameter list and flat offsets (model.hpp:91-142)."""
    d = spec.desc()
    n, e = C.c_uint64(), C.c_uint64()
    call("hp_param_count", C.byref(d), C.byref(n), C.byref(e))
    out = []
    name = C.create_string_buffer(128)
    for i in range(n.value):
        r, c, o, k = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        call("hp_param_info", C.byref(d), i, name, 128, C.byref(r), C.byref(c), C.byref(o),
             C.byref(k))
        out.append(ParamShape(name.value.decode(), r.value, c.value, o.value, k.value))
    return out


def flat_size(spec: ModelSpec) -> int:
    d = spec.desc()
    n, e = C.c_uint64(), C.c_uint64()
    call("hp_param_count", C.byref(d), C.byref(n), C.byref(e))
    return e.value


def init_parameters(spec: ModelSpec, seed: int) -> np.ndarray:
    """init_parameters<double>(spec, derived_rng(seed, 0)) as a flat f64
    vector in canonical order (model.hpp:171-184)."""
    out = np.empty(flat_size(spec), dtype=np.float64)
    d = spec.desc()
    call("hp_init_parameters", C.byref(d), seed & (2**64 - 1), _p(out))
    return out


def bucket_plan(spec: ModelSpec, bucket_mb: float) -> list[tuple[int, int]]:
    """Gradient buckets as [lo, hi) flat ranges, bucket 0 ending at N."""
    n = len(param_shapes(spec))
    lo = np.empty(n, dtype=np.uint64)
    hi = np.empty(n, dtype=np.uint64)
    nb = C.c_uint64()
    d = spec.desc()
    call("hp_bucket_plan", C.byref(d), float(bucket_mb), _p(lo), _p(hi), C.byref(nb))
    return [(int(lo[i]), int(hi[i])) for i in range(nb.value)]


# --------------------------------------------------------------------- data
@dataclass
class Instance:
    """One training instance (model.hpp:72-80)."""
    tokens: np.ndarray
    segments: np.ndarray
    mask_positions: np.ndarray
    mask_originals: np.ndarray
    label: int = 0

    @property
    def token_length(self) -> int:
        return int(len(self.tokens))


@dataclass
class BatchCSR:
    """A Batch (vector<Instance>) flattened to CSR int64 arrays."""
    tok_off: np.ndarray
    tokens: np.ndarray
    segments: np.ndarray
    mask_off: np.ndarray
    mask_pos: np.ndarray
    mask_orig: np.ndarray
    label: np.ndarray

    @property
    def n_inst(self) -> int:
        return int(len(self.label))

    @property
    def n_tokens(self) -> int:
        return int(self.tok_off[-1])

    @property
    def n_masks(self) -> int:
        return int(self.mask_off[-1])

    def desc(self) -> _lib.BatchDesc:
        return _lib.BatchDesc(self.n_inst, self.tok_off.ctypes.data, self.tokens.ctypes.data,
                              self.segments.ctypes.data, self.mask_off.ctypes.data,
                              self.mask_pos.ctypes.data, self.mask_orig.ctypes.data,
                              self.label.ctypes.data)

    def host_bytes(self) -> int:
        return sum(a.nbytes for a in (self.tok_off, self.tokens, self.segments, self.mask_off,
                                      self.mask_pos, self.mask_orig, self.label))


def pack_batch(batch: Sequence[Instance]) -> BatchCSR:
    tl = np.array([0] + [len(i.tokens) for i in batch], dtype=np.uint64).cumsum().astype(np.uint64)
    ml = np.array([0] + [len(i.mask_positions) for i in batch], dtype=np.uint64).cumsum().astype(np.uint64)
    cat = lambda xs: (np.concatenate([np.asarray(x, dtype=np.int64) for x in xs])
                      if len(xs) else np.zeros(0, dtype=np.int64))
    return BatchCSR(tl, cat([i.tokens for i in batch]), cat([i.segments for i in batch]), ml,
                    cat([i.mask_positions for i in batch]), cat([i.mask_originals for i in batch]),
                    np.array([i.label for i in batch], dtype=np.int64))


@dataclass
class BatchPlan:
    epoch: int
    batches: list  # list of np.ndarray[uint64] of global ids


def build_epoch_batches(token_lengths, max_sentences: int, max_tokens: int, base_seed: int,
                        epoch: int) -> BatchPlan:
    """dataset.cpp:52-88: shuffle with derived_rng(S, N), greedy close-on-overflow packing."""
    lens = np.ascontiguousarray(token_lengths, dtype=np.uint32)
    n = len(lens)
    order = np.empty(n, dtype=np.uint64)
    sizes = np.empty(max(n, 1), dtype=np.uint64)
    nb = C.c_uint64()
    call("hp_build_epoch_batches", _p(lens) if n else None, n, max_sentences, max_tokens,
         base_seed & (2**64 - 1), epoch, _p(order) if n else None, _p(sizes) if n else None,
         C.byref(nb))
    out, o = [], 0
    for s in sizes[:nb.value]:
        out.append(order[o:o + int(s)])
        o += int(s)
    return BatchPlan(epoch, out)


@dataclass
class RankBatch:
    batch_index: int
    dummy: bool


def partition_for_rank(plan: BatchPlan, world_size: int, rank: int) -> list[RankBatch]:
    """dataset.cpp:90-117."""
    nb = len(plan.batches)
    rounds = (nb + world_size - 1) // world_size if world_size else 0
    bi = np.empty(max(rounds, 1), dtype=np.uint64)
    dm = np.empty(max(rounds, 1), dtype=np.uint8)
    r = C.c_uint64()
    call("hp_partition_for_rank", nb, world_size, rank, _p(bi), _p(dm), C.byref(r))
    return [RankBatch(int(bi[t]), bool(dm[t])) for t in range(r.value)]


@dataclass
class MlmGenConfig:
    """MlmGenConfig (datagen.hpp:25-37) + max_seq_tokens (repo extension)."""
    n: int = 1000
    vocab: int = 64
    docs: int = 8
    sentences_per_doc: int = 12
    min_sentence_words: int = 3
    max_sentence_words: int = 8
    p_select: float = 0.15
    p_mask: float = 0.8
    p_random: float = 0.1
    seed: int = 7
    max_seq_tokens: int = 0

    def desc(self) -> _lib.MlmGenDesc:
        return _lib.MlmGenDesc(self.n, self.vocab, self.docs, self.sentences_per_doc,
                               self.min_sentence_words, self.max_sentence_words, self.p_select,
                               self.p_mask, self.p_random, self.seed, self.max_seq_tokens)


@dataclass
class Records:
    """The generated record stream in CSR form (global record order)."""
    tok_off: np.ndarray
    tokens: np.ndarray
    segments: np.ndarray
    mask_off: np.ndarray
    mask_pos: np.ndarray
    mask_orig: np.ndarray
    label: np.ndarray

    def __len__(self) -> int:
        return len(self.label)

    def token_lengths(self) -> np.ndarray:
        return np.diff(self.tok_off).astype(np.uint32)

    def instance(self, g: int) -> Instance:
        a, b = int(self.tok_off[g]), int(self.tok_off[g + 1])
        c, d = int(self.mask_off[g]), int(self.mask_off[g + 1])
        return Instance(self.tokens[a:b], self.segments[a:b], self.mask_pos[c:d],
                        self.mask_orig[c:d], int(self.label[g]))

    def batch(self, ids: Iterable[int]) -> BatchCSR:
        """Gather records into one packed rank batch (the loader's assemble,
        loader.cpp:80-96)."""
        ids = np.asarray(list(ids), dtype=np.int64)
        ta, tb = self.tok_off[ids].astype(np.int64), self.tok_off[ids + 1].astype(np.int64)
        ma, mb = self.mask_off[ids].astype(np.int64), self.mask_off[ids + 1].astype(np.int64)
        tidx = np.concatenate([np.arange(a, b) for a, b in zip(ta, tb)]) if len(ids) else np.zeros(0, np.int64)
        midx = np.concatenate([np.arange(a, b) for a, b in zip(ma, mb)]) if len(ids) else np.zeros(0, np.int64)
        tl = np.concatenate([[0], np.cumsum(tb - ta)]).astype(np.uint64)
        ml = np.concatenate([[0], np.cumsum(mb - ma)]).astype(np.uint64)
        return BatchCSR(tl, self.tokens[tidx].copy(), self.segments[tidx].copy(), ml,
                        self.mask_pos[midx].copy(), self.mask_orig[midx].copy(),
                        self.label[ids].copy())


@dataclass
class PairGenConfig:
    """Synthetic translation pairs (repo generator for transformer_seq2seq,
    include/hetpar_b200.h hp_pairs_generate)."""
    n: int = 64
    vocab: int = 32768
    min_len: int = 64
    max_len: int = 64
    seed: int = 7

    def desc(self) -> _lib.PairGenDesc:
        return _lib.PairGenDesc(self.n, self.vocab, self.min_len, self.max_len, self.seed)


def generate_pair_records(cfg: PairGenConfig) -> Records:
    """Translation pairs as Records: tokens = source ++ target per record,
    segments 0 / 1, no masks."""
    d = cfg.desc()
    nt = C.c_uint64()
    call("hp_pairs_generate_size", C.byref(d), C.byref(nt))
    r = Records(np.empty(cfg.n + 1, np.uint64), np.empty(nt.value, np.int64),
                np.empty(nt.value, np.int64), np.zeros(cfg.n + 1, np.uint64),
                np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(cfg.n, np.int64))
    call("hp_pairs_generate", C.byref(d), _p(r.tok_off), _p(r.tokens), _p(r.segments))
    return r


def generate_mlm_records(cfg: MlmGenConfig) -> Records:
    d = cfg.desc()
    nt, nm = C.c_uint64(), C.c_uint64()
    call("hp_mlm_generate_size", C.byref(d), C.byref(nt), C.byref(nm))
    r = Records(np.empty(cfg.n + 1, np.uint64), np.empty(nt.value, np.int64),
                np.empty(nt.value, np.int64), np.empty(cfg.n + 1, np.uint64),
                np.empty(max(nm.value, 1), np.int64), np.empty(max(nm.value, 1), np.int64),
                np.empty(cfg.n, np.int64))
    call("hp_mlm_generate", C.byref(d), _p(r.tok_off), _p(r.tokens), _p(r.segments),
         _p(r.mask_off), _p(r.mask_pos), _p(r.mask_orig), _p(r.label))
    r.mask_pos = r.mask_pos[:nm.value]
    r.mask_orig = r.mask_orig[:nm.value]
    return r


# --------------------------------------------------------------------- schedules
@dataclass
class SchedulerConfig:
    """SchedulerConfig (optim.hpp:51-57)."""
    kind: str = "fixed"  # fixed | inverse_sqrt | linear
    peak_lr: float = 1e-3
    d_model: int = 512
    warmup_steps: int = 4000
    total_steps: int = 1000000


def inverse_sqrt_lr(step: int, d_model: int, warmup_steps: int) -> float:
    """optim.hpp:19-29."""
    if step == 0:
        raise ConfigError("config: inverse_sqrt_lr: step must be >= 1")
    if d_model == 0:
        raise ConfigError("config: inverse_sqrt_lr: d_model must be >= 1")
    if warmup_steps == 0:
        raise ConfigError("config: inverse_sqrt_lr: warmup_steps must be >= 1")
    s, w = float(step), float(warmup_steps)
    return min(1.0 / math.sqrt(s), s * w ** -1.5) / math.sqrt(float(d_model))


def linear_warmup_decay_lr(step: int, peak: float, warmup: int, total: int) -> float:
    """optim.hpp:31-47."""
    if warmup >= total:
        raise ConfigError("config: linear_warmup_decay_lr: warmup must be < total")
    if step > total or step == 0:
        return 0.0
    if step <= warmup:
        return peak * (float(step) / float(warmup))
    return peak * (float(total - step) / float(total - warmup))


def scheduled_lr(c: SchedulerConfig, step: int) -> float:
    """optim.hpp:59-70; `step` counts updates, 1 for the first."""
    if c.kind == "fixed":
        return c.peak_lr
    if c.kind == "inverse_sqrt":
        return inverse_sqrt_lr(step, c.d_model, c.warmup_steps)
    if c.kind == "linear":
        return linear_warmup_decay_lr(step, c.peak_lr, c.warmup_steps, c.total_steps)
    raise ConfigError("config: scheduled_lr: unknown scheduler kind")


# --------------------------------------------------------------------- engine
@dataclass
class OptimConfig:
    kind: str = "adam"  # adam | sgd (OptKind, optim.hpp:77) | adamw (extension)
    beta1: float = 0.9
    beta2: float = 0.98
    eps: float = 1e-9
    weight_decay: float = 0.0  # adamw: p -= lr * wd * p before the Adam step

    def desc(self) -> _lib.OptimDesc:
        k = {"adam": _lib.HP_OPT_ADAM, "sgd": _lib.HP_OPT_SGD, "adamw": _lib.HP_OPT_ADAMW}.get(self.kind)
        if k is None:
            raise ConfigError(f"config: unknown optimizer {self.kind}")
        return _lib.OptimDesc(k, self.beta1, self.beta2, self.eps, self.weight_decay)


@dataclass
class ExecConfig:
    compute: str = "f32"  # f32 (parity path) | bf16 (tcgen05 path)
    policy: str = "sentences"
    device: int = 0
    bucket_mb: float = 25.0
    max_tokens: int = 4096
    max_batch: int = 64
    max_masks: int = 1024
    update_freq: int = 1

    def desc(self) -> _lib.ExecDesc:
        comp = {"f32": _lib.HP_COMPUTE_F32, "bf16": _lib.HP_COMPUTE_BF16}[self.compute]
        pol = {"sentences": _lib.HP_POLICY_SENTENCES, "tokens": _lib.HP_POLICY_TOKENS}[self.policy]
        return _lib.ExecDesc(comp, pol, self.device, self.bucket_mb, self.max_tokens,
                             self.max_batch, self.max_masks, self.update_freq)


@dataclass
class StepReport:
    """StepReport (engine.hpp:26-32)."""
    step: int = 0
    loss: float = 0.0
    weight: float = 0.0
    seconds: float = 0.0
    rank_seconds: list = field(default_factory=list)
    local_loss_sum: float = 0.0
    local_weight: float = 0.0
    updated: bool = True


# ---------------------------------------------------------------- HSD1 shards
def write_mlm_shards(directory: str, records: "Records", shards: int) -> None:
    """generate_mlm_shards' files (datagen.cpp:71-127) for these records:
    ``shards`` contiguous chunks (earlier ones one longer), shard_%04d.hsd,
    byte-identical to the reference writer for the same records."""
    r = records
    call("hp_mlm_write_shards", directory.encode(), len(r.label), shards, _p(r.tok_off), _p(r.tokens),
         _p(r.segments), _p(r.mask_off), _p(r.mask_pos), _p(r.mask_orig), _p(r.label))


class LoadedBatch:
    """One scheduled batch from a ShardLoader (LoadedBatch, loader.hpp): its
    arrays live in the loader until the next ``next()``; ``stage()`` it
    right away, or ``to_csr()`` to keep a copy."""

    def __init__(self, d: _lib.LoadedDesc):
        self._d = d
        self.batch_index = d.batch_index
        self.dummy = bool(d.dummy)

    def desc(self) -> _lib.BatchDesc:
        return self._d.batch

    @property
    def n_inst(self) -> int:
        return int(self._d.batch.n_inst)

    def to_csr(self) -> BatchCSR:
        b = self._d.batch
        n = b.n_inst

        def arr(ptr, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                         shape=(count,)).copy()
        tok_off = arr(b.tok_off, n + 1, np.uint64)
        mask_off = arr(b.mask_off, n + 1, np.uint64)
        t, m = int(tok_off[-1]), int(mask_off[-1])
        return BatchCSR(tok_off, arr(b.tokens, t, np.int64), arr(b.segments, t, np.int64), mask_off,
                        arr(b.mask_pos, m, np.int64), arr(b.mask_orig, m, np.int64),
                        arr(b.label, n, np.int64))

    def host_bytes(self) -> int:
        return self.to_csr().host_bytes()


class ShardLoader:
    """BatchLoader (loader.cpp:80-139): serves one rank's schedule in order;
    a producer thread keeps ``prefetch_depth`` batches decoded ahead (0:
    decode on demand).  Iterating yields LoadedBatch."""

    def __init__(self, data: "ShardDataset", plan: BatchPlan, schedule, prefetch_depth: int = 2):
        order = np.ascontiguousarray(np.concatenate(plan.batches) if plan.batches else np.zeros(0),
                                     np.uint64)
        sizes = np.ascontiguousarray([len(b) for b in plan.batches], np.uint64)
        sb = np.ascontiguousarray([rb.batch_index for rb in schedule], np.uint64)
        sd = np.ascontiguousarray([1 if rb.dummy else 0 for rb in schedule], np.uint8)
        self._data = data  # keeps the mapping alive
        self._h = C.c_void_p()
        call("hp_loader_create", data._h, _p(order), _p(sizes), len(sizes), _p(sb), _p(sd), len(sb),
             prefetch_depth, C.byref(self._h))

    def next(self) -> Optional[LoadedBatch]:
        d, has = _lib.LoadedDesc(), C.c_int()
        call("hp_loader_next", self._h, C.byref(d), C.byref(has))
        return LoadedBatch(d) if has.value else None

    def __iter__(self):
        while True:
            b = self.next()
            if b is None:
                return
            yield b

    def close(self):
        if self._h:
            call("hp_loader_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardDataset:
    """list_shards + build_index (dataset.cpp:10-50): every *.hsd file of a
    directory, sorted, memory-mapped as one global record space."""

    def __init__(self, directory: str):
        self._h = C.c_void_p()
        call("hp_shards_open", directory.encode(), C.byref(self._h))
        t, k = C.c_uint64(), C.c_uint64()
        call("hp_shards_info", self._h, C.byref(t), C.byref(k))
        self.total, self.nshards = t.value, k.value

    def token_lengths(self) -> np.ndarray:
        out = np.empty(self.total, np.uint32)
        call("hp_shards_token_lengths", self._h, _p(out), self.total)
        return out

    def loader(self, plan: BatchPlan, schedule, prefetch_depth: int = 2) -> ShardLoader:
        return ShardLoader(self, plan, schedule, prefetch_depth)

    def close(self):
        if self._h:
            call("hp_shards_close", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_OPT = {"sgd": _lib.HP_OPT_SGD, "adam": _lib.HP_OPT_ADAM, "adamw": _lib.HP_OPT_ADAMW}
_OPT_NAME = {v: k for k, v in _OPT.items()}


@dataclass
class CheckpointMeta:
    """TrainState fields an HCK1 file carries besides the tensors
    (checkpoint.hpp:15-37, checkpoint.cpp:54-79).  ``step`` and the optimizer
    fields are filled from the engine on save and from the file on load."""
    epoch: int = 0
    step: int = 0
    seed: int = 0
    policy: str = "sentences"
    world_size: int = 1
    update_freq: int = 1
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    optimizer: str = "adam"
    beta1: float = 0.9
    beta2: float = 0.98
    eps: float = 1e-9
    opt_t: int = 0
    weight_decay: float = 0.0

    def desc(self) -> _lib.CkptDesc:
        sk = {"fixed": 0, "inverse_sqrt": 1, "linear": 2}[self.scheduler.kind]
        return _lib.CkptDesc(self.epoch, self.step, self.seed, _POLICY[self.policy],
                             self.world_size, self.update_freq, sk, self.scheduler.peak_lr,
                             self.scheduler.d_model, self.scheduler.warmup_steps,
                             self.scheduler.total_steps, _OPT[self.optimizer],
                             self.beta1, self.beta2, self.eps, self.opt_t, self.weight_decay)

    @staticmethod
    def from_desc(d: _lib.CkptDesc) -> "CheckpointMeta":
        sched = SchedulerConfig(kind=("fixed", "inverse_sqrt", "linear")[d.sched_kind],
                                peak_lr=d.peak_lr, d_model=d.sched_d_model,
                                warmup_steps=d.warmup_steps, total_steps=d.total_steps)
        return CheckpointMeta(d.epoch, d.step, d.seed, "tokens" if d.policy == 2 else "sentences",
                              d.world_size, d.update_freq, sched,
                              _OPT_NAME[d.opt_kind], d.beta1, d.beta2, d.eps, d.opt_t, d.weight_decay)


_ARCH_NAME = {v: k for k, v in _ARCH.items()}


def write_checkpoint(path: str, spec: ModelSpec, meta: CheckpointMeta, params: np.ndarray,
                     adam_m: Optional[np.ndarray] = None, adam_v: Optional[np.ndarray] = None) -> None:
    """save_checkpoint<float> (checkpoint.cpp:165-212): one HCK1 file, written
    atomically; byte-identical to the reference writer for the same state."""
    p = np.ascontiguousarray(params, np.float32)
    m = None if adam_m is None else np.ascontiguousarray(adam_m, np.float32)
    v = None if adam_v is None else np.ascontiguousarray(adam_v, np.float32)
    md, cd = spec.desc(), meta.desc()
    call("hp_checkpoint_write", path.encode(), C.byref(md), C.byref(cd), _p(p),
         None if m is None else _p(m), None if v is None else _p(v))


def read_checkpoint(path: str):
    """load_checkpoint<float> (checkpoint.cpp:214-287) -> (spec, meta, params,
    adam_m, adam_v); digest, version, dtype, names and shapes validated."""
    md, cd = _lib.ModelDesc(), _lib.CkptDesc()
    call("hp_checkpoint_read", path.encode(), C.byref(md), C.byref(cd), None, None, None, 0)
    spec = ModelSpec(_ARCH_NAME[md.arch], md.d_model, md.heads, md.vocab, md.max_seq,
                     md.layers if md.arch != _ARCH["masked_token_model"] else 1, md.d_ff,
                     bool(md.with_nsp), md.label_smooth_eps)
    n = flat_size(spec)
    p, m, v = (np.empty(n, np.float32) for _ in range(3))
    call("hp_checkpoint_read", path.encode(), None, None, _p(p), _p(m), _p(v), n)
    meta = CheckpointMeta.from_desc(cd)
    if meta.optimizer == "sgd":
        m = v = None
    return spec, meta, p, m, v


def resume_position(token_lengths, max_sentences: int, max_tokens: int, seed: int, world: int,
                    update_freq: int, step: int) -> tuple[int, int]:
    """Epoch and rounds to skip when resuming after ``step`` updates
    (engine.hpp:225-244: P updates consumed exactly P*K lockstep rounds)."""
    lens = np.ascontiguousarray(token_lengths, np.uint32)
    e, k = C.c_uint64(), C.c_uint64()
    call("hp_resume_position", _p(lens), len(lens), max_sentences, max_tokens, seed, world,
         update_freq, step, C.byref(e), C.byref(k))
    return e.value, k.value


class Communicator:
    """NCCL communicator over NVLink/NVSwitch, one process per GPU.  The
    ncclUniqueId is created on rank 0 and shipped with a torch.distributed
    broadcast (the role ProcessGroup::broadcast plays in the reference)."""

    def __init__(self, world: int, rank: int, device: int, pg=None):
        uid = (C.c_uint8 * 128)()
        if world > 1:
            import torch
            import torch.distributed as dist
            if rank == 0:
                call("hp_comm_unique_id", uid)
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            dist.broadcast(t, src=0, group=pg)
            uid = (C.c_uint8 * 128)(*t.tolist())
        else:
            call("hp_comm_unique_id", uid)
        self._h = C.c_void_p()
        call("hp_comm_create", world, rank, device, uid, C.byref(self._h))
        self.world, self.rank, self.device = world, rank, device

    @classmethod
    def tcp(cls, host: str, port: int, world: int, rank: int, device: int,
            timeout_ms: int = 30000) -> "Communicator":
        """Form the world with the engine's own TCP rendezvous (rank 0 serves
        the ncclUniqueId on host:port) -- no torch.distributed involved."""
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        call("hp_comm_create_tcp", host.encode(), port, world, rank, device, timeout_ms,
             C.byref(self._h))
        self.world, self.rank, self.device = world, rank, device
        return self

    @property
    def handle(self):
        return self._h

    # ---- ProcessGroup (comm.hpp:16-49): the NcclProcessGroup control plane
    def broadcast(self, payload: bytes, root: int = 0, max_len: int = 1 << 20) -> bytes:
        """Every rank returns the root's exact bytes (non-root inputs ignored)."""
        buf = (C.c_uint8 * max(max_len, 1))()
        n = C.c_uint64()
        src = (C.c_uint8 * max(len(payload), 1)).from_buffer_copy(payload or b"\0")
        call("hp_pg_broadcast", self._h, src, len(payload), root, buf, max_len, C.byref(n))
        return bytes(buf[:n.value])

    def all_reduce_sum(self, values) -> list:
        """Rank-ordered left fold (0 -> world-1), identical bytes on every rank."""
        v = np.ascontiguousarray(values, np.float64)
        out = np.empty_like(v)
        call("hp_pg_all_reduce_sum", self._h, _p(v), len(v), _p(out))
        return out.tolist()

    def gather_scalars(self, value: float) -> list:
        """Master receives [v_0 .. v_{w-1}] in rank order; other ranks get []."""
        out = np.empty(self.world, np.float64)
        call("hp_pg_gather_scalars", self._h, float(value), _p(out))
        return out.tolist() if self.rank == 0 else []

    def barrier(self) -> None:
        call("hp_pg_barrier", self._h)

    def allreduce_bench(self, nbytes: int, bucket_mb: float = 25.0, iters: int = 10,
                        warmup: int = 3) -> dict:
        """Time the engine's bucketed gradient allreduce (fp32, ncclSum, buckets
        of <= bucket_mb MiB) over nbytes; collective.  busbw = S/t * 2(W-1)/W."""
        ms = C.c_double()
        call("hp_comm_allreduce_bench", self._h, int(nbytes), float(bucket_mb), int(iters),
             int(warmup), C.byref(ms))
        t = ms.value / 1e3
        w = self.world
        algbw = nbytes / t / 1e9
        return {"bytes": int(nbytes), "bucket_mb": float(bucket_mb), "ms": ms.value,
                "algbw_gbps": algbw, "busbw_gbps": algbw * 2 * (w - 1) / w}

    def close(self):
        if self._h:
            call("hp_comm_destroy", self._h)
            self._h = C.c_void_p()


class StepEngine:
    """StepEngine<T> (engine.hpp:114-192) on the device.

    round(batch, dummy, lr) runs: forward -> [loss, weight] allreduce ->
    backward with bucketed gradient allreduce -> /sum(weight) -> update, and
    returns the StepReport of the update."""

    def __init__(self, spec: ModelSpec, optim: OptimConfig = None, exec_cfg: ExecConfig = None,
                 comm: Optional[Communicator] = None, params: Optional[np.ndarray] = None,
                 seed: Optional[int] = None):
        self.spec = spec
        self.optim = optim or OptimConfig()
        self.exec = exec_cfg or ExecConfig()
        self.comm = comm
        self.n = flat_size(spec)
        self._h = C.c_void_p()
        md, od, xd = spec.desc(), self.optim.desc(), self.exec.desc()
        call("hp_engine_create", C.byref(md), C.byref(od), C.byref(xd),
             comm.handle if comm else None, C.byref(self._h))
        if params is None and seed is not None:
            params = init_parameters(spec, seed)
        if params is not None:
            self.set_params(params)
        self.last_h2d_bytes = 0
        self._group_t0 = None  # start of the pending update group (K > 1)

    def close(self):
        if self._h:
            call("hp_engine_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state
    def set_params(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat)
        dt = 1 if flat.dtype == np.float64 else 0
        if dt == 0:
            flat = flat.astype(np.float32, copy=False)
        call("hp_engine_set_params", self._h, _p(flat), flat.size, dt)

    def get_params(self, dtype=np.float32) -> np.ndarray:
        out = np.empty(self.n, dtype=dtype)
        call("hp_engine_get_params", self._h, _p(out), self.n, 1 if dtype == np.float64 else 0)
        return out

    def broadcast_params(self, root: int = 0):
        call("hp_engine_broadcast_params", self._h, root)

    def get_adam(self):
        m = np.empty(self.n, np.float32)
        v = np.empty(self.n, np.float32)
        t = C.c_uint64()
        call("hp_engine_get_adam", self._h, _p(m), _p(v), C.byref(t))
        return m, v, t.value

    def save_checkpoint(self, path: str, meta: CheckpointMeta) -> None:
        """HCK1 from device state (master rank; checkpoint.cpp:165-212).  The
        engine supplies step, optimizer kind / hyper-parameters and moments."""
        cd = meta.desc()
        call("hp_engine_save_checkpoint", self._h, path.encode(), C.byref(cd))

    def load_checkpoint(self, path: str) -> CheckpointMeta:
        """HCK1 into device state: parameters, Adam m / v / t, step, and the
        file's optimizer and weight policy (checkpoint.cpp:254, 282-289)."""
        cd = _lib.CkptDesc()
        call("hp_engine_load_checkpoint", self._h, path.encode(), C.byref(cd))
        meta = CheckpointMeta.from_desc(cd)
        self.optim = OptimConfig(meta.optimizer, meta.beta1, meta.beta2, meta.eps, meta.weight_decay)
        self.exec.policy = meta.policy
        return meta

    def step_count(self) -> int:
        s = C.c_uint64()
        call("hp_engine_step_count", self._h, C.byref(s))
        return s.value

    def set_capture(self, on: bool):
        call("hp_engine_set_capture", self._h, int(on))

    def forward(self, batch) -> tuple:
        """model_forward (model.hpp:260-390) alone: (loss_sum, weight) of the
        batch under the current parameters; no backward, collective or update."""
        self.stage(batch)
        ls, w = C.c_double(), C.c_double()
        call("hp_engine_forward", self._h, C.byref(ls), C.byref(w))
        return ls.value, w.value

    def set_digest_check(self, every: int = 100, debug: bool = False):
        """check_digest_on_cadence (engine.hpp:170-184): after every `every`-th
        update (each update with debug) the ranks compare parameter digests
        with rank 0's; a divergence raises NumericError on every rank."""
        call("hp_engine_set_digest_check", self._h, int(every), int(debug))

    def set_grad_comm(self, on: bool):
        """Measurement only: off skips the gradient-bucket allreduces (ranks
        diverge); bench.py uses it for the exposed-communication figure."""
        call("hp_engine_set_grad_comm", self._h, int(on))

    def local_grads(self) -> np.ndarray:
        out = np.empty(self.n, np.float32)
        call("hp_engine_get_local_grads", self._h, _p(out), self.n)
        return out

    def digest(self) -> int:
        d = C.c_uint64()
        call("hp_engine_params_digest", self._h, C.byref(d))
        return d.value

    def pending_rounds(self) -> int:
        """StepEngine::pending_rounds (engine.hpp:165): rounds accumulated
        since the last update."""
        n = C.c_uint64()
        call("hp_engine_pending_rounds", self._h, C.byref(n))
        return n.value

    @property
    def step(self) -> int:
        s = C.c_uint64()
        call("hp_engine_step_count", self._h, C.byref(s))
        return s.value

    # -- rounds
    def stage(self, batch) -> None:
        """Validate the rank batch and queue its H2D copy (from the engine's
        pinned staging block).  Accepts a BatchCSR, a LoadedBatch straight
        from a ShardLoader, or a list of instances."""
        if isinstance(batch, LoadedBatch):
            d = batch.desc()
            call("hp_engine_stage_batch", self._h, C.byref(d))
            self.last_h2d_bytes = 0
            return
        csr = batch if isinstance(batch, BatchCSR) else pack_batch(batch)
        self._staged = csr
        d = csr.desc()
        call("hp_engine_stage_batch", self._h, C.byref(d))
        self.last_h2d_bytes = csr.host_bytes()

    def round_async(self, dummy: bool = False, lr: float = 1e-3) -> None:
        call("hp_engine_round_async", self._h, int(dummy), float(lr))

    def round_sync(self) -> StepReport:
        o = _lib.RoundOut()
        call("hp_engine_round_sync", self._h, C.byref(o))
        return StepReport(o.step, o.loss, o.weight, 0.0, [], o.local_loss_sum, o.local_weight,
                          bool(o.updated))

    def round(self, batch, dummy: bool = False, lr: float = 1e-3) -> Optional[StepReport]:
        """StepEngine::round (engine.hpp:125-165): None on the first K-1 rounds
        of an update group (update_freq = K), the report on the K-th; seconds
        run from the group's first round, as the reference's group_start_."""
        t0 = time.perf_counter()
        if self._group_t0 is None:
            self._group_t0 = t0
        self.stage(batch)
        self.round_async(dummy, lr)
        rep = self.round_sync()
        if not rep.updated:
            return None
        rep.seconds = time.perf_counter() - self._group_t0
        self._group_t0 = None
        self._gather_seconds(rep)
        return rep

    def _gather_seconds(self, rep: StepReport) -> None:
        # rank_seconds: every rank's seconds on the master (group_.gather_scalars,
        # engine.hpp:158-162); a collective on the communicator
        if self.comm is not None and self.comm.world > 1:
            rep.rank_seconds = self.comm.gather_scalars(rep.seconds)
        else:
            rep.rank_seconds = [rep.seconds]

    def rounds(self, work) -> list:
        """round() over a sequence of (batch, dummy, lr), pipelined: while the
        device runs round k, the host validates and stages batch k+1 (its H2D
        copy is queued on the compute stream behind round k, so the device
        buffer is only overwritten once round k is done).  Every round still
        copies its batch host->device and reads [loss, weight] back.  Returns
        what round() returns for each (None on the first K-1 rounds of an
        update group)."""
        it = iter(work)
        out = []
        cur = next(it, None)
        if cur is None:
            return out
        self.stage(cur[0])
        while cur is not None:
            if self._group_t0 is None:
                self._group_t0 = time.perf_counter()
            self.round_async(cur[1], cur[2])
            nxt = next(it, None)
            if nxt is not None:
                self.stage(nxt[0])
            rep = self.round_sync()
            if rep.updated:
                rep.seconds = time.perf_counter() - self._group_t0
                self._group_t0 = None
                out.append(rep)
            else:
                out.append(None)
            cur = nxt
        # rank_seconds for every update of the call in ONE collective after the
        # last round (a per-update host-staged gather would stall the pipeline):
        # each rank's seconds at its own offset, summed with zeros elsewhere
        reps = [r for r in out if r is not None]
        if self.comm is not None and self.comm.world > 1:
            w, k = self.comm.world, len(reps)
            v = np.zeros(w * k)
            v[self.comm.rank * k:(self.comm.rank + 1) * k] = [r.seconds for r in reps]
            allv = self.comm.all_reduce_sum(v) if k else []
            for i, r in enumerate(reps):
                r.rank_seconds = [allv[q * k + i] for q in range(w)] if self.comm.rank == 0 else []
        else:
            for r in reps:
                r.rank_seconds = [r.seconds]
        return out

    # -- instrumentation
    def mark(self, slot: int):
        """Record a CUDA event on the engine's compute stream."""
        call("hp_engine_mark", self._h, slot)

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        call("hp_engine_elapsed", self._h, a, b, C.byref(ms))
        return ms.value

    def synchronize(self):
        call("hp_engine_synchronize", self._h)

    def io_bytes(self) -> tuple[int, int]:
        """(host->device bytes per staged batch, device->host bytes per round)."""
        a, b = C.c_uint64(), C.c_uint64()
        call("hp_engine_io_bytes", self._h, C.byref(a), C.byref(b))
        return a.value, b.value

    def timers(self, on: bool):
        call("hp_engine_timers", self._h, int(on))

    def timer(self, which: int) -> dict:
        name = C.create_string_buffer(64)
        ms, fl, by = C.c_double(), C.c_double(), C.c_double()
        n = C.c_uint64()
        call("hp_engine_timer_read", self._h, which, name, 64, C.byref(ms), C.byref(n),
             C.byref(by), C.byref(fl))
        return {"name": name.value.decode(), "ms": ms.value, "launches": n.value,
                "bytes": by.value, "flops": fl.value}

    def class_replay(self, which: int, iters: int = 10) -> dict:
        """Measurement: one round's kernels of class `which` (0 GEMM, 1
        attention) replayed back to back from a CUDA graph -- the class's
        serialised time per round, its FLOPs and launches (runs one eager
        round first; overwrites the class's outputs)."""
        ms, fl = C.c_double(), C.c_double()
        n = C.c_uint64()
        call("hp_engine_class_replay", self._h, which, iters, C.byref(ms), C.byref(fl), C.byref(n))
        return {"ms": ms.value, "flops": fl.value, "launches": n.value}

    @staticmethod
    def kernel_launches() -> int:
        n = C.c_uint64()
        call("hp_engine_kernel_launches", None, C.byref(n))
        return n.value
