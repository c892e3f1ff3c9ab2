"""train_run: the reference's full per-rank training loop (engine.hpp:197-330)
over the device engine.

EngineConfig / RunReport mirror the reference's (engine.hpp:40-75,
engine.hpp:34-42); `exec_cfg` adds what the device engine needs (compute
path, device, bucket size; capacities are derived from the data).  The loop
is the reference's: HSD1 shards -> token lengths -> resume position (P
updates consumed P*K lockstep rounds) -> rank 0's parameters broadcast ->
per epoch: build_epoch_batches, partition_for_rank, a prefetching loader
that skips the resumed rounds, StepEngine rounds with scheduled_lr(P + 1),
checkpoints every `checkpoint_interval` updates and at the end (rank 0,
after a barrier), stop at max_steps / max_epochs.
"""
from __future__ import annotations

import math
import os
import sys
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import api
from ._lib import ConfigError


@dataclass
class EngineConfig:
    """EngineConfig (engine.hpp:44-75)."""
    spec: api.ModelSpec
    policy: str = "sentences"
    opt_kind: str = "sgd"
    beta1: float = 0.9
    beta2: float = 0.98
    eps: float = 1e-9
    weight_decay: float = 0.0  # adamw (extension)
    sched: api.SchedulerConfig = field(default_factory=api.SchedulerConfig)
    seed: int = 1
    data_dir: str = ""
    max_sentences: int = 0
    max_tokens: int = 0
    update_freq: int = 1
    max_steps: int = 0
    max_epochs: int = 0
    checkpoint_dir: str = ""
    checkpoint_interval: int = 0
    resume_path: str = ""
    check_interval: int = 100
    debug_checks: bool = False


@dataclass
class RunReport:
    """RunReport (engine.hpp:34-42)."""
    world: int = 1
    steps_run: int = 0
    final_step: int = 0
    epochs_completed: int = 0
    total_seconds: float = 0.0
    avg_step_seconds: float = 0.0
    final_loss: float = math.nan
    steps: List[api.StepReport] = field(default_factory=list)


def checkpoint_step_path(directory: str, step: int) -> str:
    """engine.cpp:8-12."""
    return os.path.join(directory, f"checkpoint_{step:06d}.hck")


def checkpoint_final_path(directory: str) -> str:
    """engine.cpp:14-16."""
    return os.path.join(directory, "checkpoint_final.hck")


def _capacities(lengths: np.ndarray, cfg: EngineConfig, K_world: int):
    # a rank batch never exceeds the caps (build_epoch_batches closes a batch
    # before it would): tokens <= max_tokens, instances <= max_sentences
    longest = int(lengths.max())
    if cfg.max_tokens:
        tok = int(cfg.max_tokens)
    else:
        tok = int(cfg.max_sentences) * longest
    inst = int(cfg.max_sentences) if cfg.max_sentences else max(1, tok // int(lengths.min()))
    return max(tok, longest), inst, max(tok, 1)


def train_run(cfg: EngineConfig, comm: Optional[api.Communicator] = None,
              exec_cfg: Optional[api.ExecConfig] = None) -> RunReport:
    """engine.hpp:197-330 with the device StepEngine; one call per rank
    (one process per GPU), every rank with the same config."""
    world = comm.world if comm else 1
    rank = comm.rank if comm else 0
    if cfg.update_freq == 0:
        raise ConfigError("config: update_freq must be >= 1")
    ds = api.ShardDataset(cfg.data_dir)
    lengths = ds.token_lengths()
    if len(lengths) == 0:
        raise ConfigError(f"config: no shards found under {cfg.data_dir}")

    spec = cfg.spec
    skip_rounds, epoch, state = 0, 0, None
    if cfg.resume_path:
        ck_spec, meta, _, _, _ = api.read_checkpoint(cfg.resume_path)
        if meta.world_size * meta.update_freq != world * cfg.update_freq:
            raise ConfigError(
                f"config: resume must preserve world_size x update_freq: checkpoint has "
                f"{meta.world_size} x {meta.update_freq}, run has {world} x {cfg.update_freq}")
        if api.param_shapes(ck_spec) != api.param_shapes(spec) or ck_spec.arch != spec.arch:
            raise ConfigError("config: resume model spec does not match the checkpoint")
        epoch, skip_rounds = api.resume_position(lengths, cfg.max_sentences, cfg.max_tokens,
                                                 meta.seed, world, cfg.update_freq, meta.step)
        state = meta

    ex = exec_cfg or api.ExecConfig()
    tok, inst, masks = _capacities(lengths, cfg, world * cfg.update_freq)
    ex = api.ExecConfig(**{**ex.__dict__, "max_tokens": tok, "max_batch": inst,
                           "max_masks": masks, "policy": cfg.policy,
                           "update_freq": cfg.update_freq})
    # a resumed run takes the optimizer, its hyper-parameters, the weight
    # policy, the scheduler and the seed from the checkpoint (TrainState,
    # checkpoint.cpp:254, 282-289), not from cfg
    if state:
        opt = api.OptimConfig(state.optimizer, state.beta1, state.beta2, state.eps, state.weight_decay)
        policy = state.policy
        ex.policy = policy
    else:
        opt = api.OptimConfig(cfg.opt_kind, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay)
        policy = cfg.policy
    seed = state.seed if state else cfg.seed
    eng = api.StepEngine(spec, opt, ex, comm=comm, seed=seed)
    try:
        if cfg.resume_path:
            eng.load_checkpoint(cfg.resume_path)
        # the master's parameters are authoritative from the first round
        if comm is not None and world > 1:
            eng.broadcast_params(0)
        eng.set_digest_check(cfg.check_interval, cfg.debug_checks)

        saving = bool(cfg.checkpoint_dir)
        if saving and rank == 0:
            os.makedirs(cfg.checkpoint_dir, exist_ok=True)
        sched = state.scheduler if state else cfg.sched

        def save_now(path: str) -> None:
            if comm is not None and world > 1:
                comm.barrier()
            if rank == 0:
                eng.save_checkpoint(path, api.CheckpointMeta(
                    epoch=epoch, seed=seed, policy=policy, world_size=world,
                    update_freq=cfg.update_freq, scheduler=sched))

        report = RunReport(world=world)
        start_epoch = epoch
        t0 = time.perf_counter()
        stopped = eng.step >= cfg.max_steps
        while not stopped and not (cfg.max_epochs != 0 and epoch >= cfg.max_epochs):
            plan = api.build_epoch_batches(lengths, cfg.max_sentences, cfg.max_tokens, seed, epoch)
            schedule = api.partition_for_rank(plan, world, rank)
            loader = ds.loader(plan, schedule)
            try:
                for _ in range(skip_rounds if epoch == start_epoch else 0):
                    loader.next()
                while True:
                    lb = loader.next()
                    if lb is None:
                        break
                    rep = eng.round(lb, lb.dummy, api.scheduled_lr(sched, eng.step + 1))
                    if rep is None:
                        continue
                    report.steps.append(rep)
                    if saving and cfg.checkpoint_interval and eng.step % cfg.checkpoint_interval == 0:
                        save_now(checkpoint_step_path(cfg.checkpoint_dir, eng.step))
                    if eng.step >= cfg.max_steps:
                        stopped = True
                        break
            finally:
                loader.close()
            if not stopped:
                epoch += 1
        if eng.pending_rounds() != 0:
            print(f"hetpar_b200: warning: discarding a partial accumulation of "
                  f"{eng.pending_rounds()} rounds at run end", file=sys.stderr)
        if saving:
            save_now(checkpoint_final_path(cfg.checkpoint_dir))
        if comm is not None and world > 1:
            comm.barrier()
        report.steps_run = len(report.steps)
        report.final_step = eng.step
        report.epochs_completed = epoch
        report.total_seconds = time.perf_counter() - t0
        report.avg_step_seconds = report.total_seconds / report.steps_run if report.steps_run else 0.0
        if report.steps:
            report.final_loss = report.steps[-1].loss
        return report
    finally:
        eng.close()
        ds.close()
