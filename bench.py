#!/usr/bin/env python3
"""Benchmark of the data-parallel training step (BASELINE.json metric:
train samples/sec at 1/2/4/8 B200).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json configs[1], "C2"): BERT-base-shaped encoder MLM step:
bert_encoder L=12, d=768, h=12, d_ff=3072, V=30522, seq 128 (every synthetic
record exactly 128 tokens), per-GPU batch 32, NSP head, Adam, bf16 tcgen05
GEMMs with fp32 master weights.  One "step" = one StepEngine round on every
rank (forward, [loss, weight] allreduce, backward with bucketed gradient
allreduce, Adam).

value:  whole-job samples/s, batch resident in HBM, CUDA events on the
        engine's compute stream, max over ranks.
e2e:    same metric through the public API with host batches: every step
        stages its rank batch host->device and reads the loss back.
--impl reference: the reference's own CPU implementation (oracle/_ref,
        compiled from the unmodified reference sources) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train samples/sec at 1/2/4/8 B200 + scaling eff.; allreduce bus GB/s"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "hetpar_ref")

C2 = dict(arch="bert_encoder", d_model=768, heads=12, vocab=30522, max_seq=128, layers=12,
          d_ff=3072, with_nsp=True, label_smooth_eps=0.1)
BATCH = 32
SEQ = 128
# BASELINE configs[3] ("C4"), selectable with --workload c4 (not the headline
# line): BERT-large-shaped, seq 512, per-GPU batch 16
C4 = dict(arch="bert_encoder", d_model=1024, heads=16, vocab=30522, max_seq=512, layers=24,
          d_ff=4096, with_nsp=True, label_smooth_eps=0.1)
# BASELINE configs[2] ("C3"), --workload c3: the paper's Transformer-base
# translation model (fairseq transformer_wmt_en_de shape: 6 + 6 layers, d 512,
# h 8, f 2048, shared 32768-word embedding), 64 synthetic pairs of 64 source +
# 64 target tokens per GPU (4096 target tokens), label smoothing 0.1, the
# "tokens" weight policy; samples = sentence pairs
C3 = dict(arch="transformer_seq2seq", d_model=512, heads=8, vocab=32768, max_seq=64, layers=6,
          d_ff=2048, with_nsp=False, label_smooth_eps=0.1)
WORKLOADS = {
    "c2": (C2, 32, 128, 64, 96, "C2: BERT-base-shaped encoder MLM+NSP step (bert_encoder L12 d768 "
           "h12 ff3072 V30522), seq 128, Adam", "bert_encoder-L12-d768"),
    "c4": (C4, 16, 512, 256, 384, "C4: BERT-large-shaped encoder MLM+NSP step (bert_encoder L24 "
           "d1024 h16 ff4096 V30522), seq 512, Adam", "bert_encoder-L24-d1024"),
    "c3": (C3, 64, 64, 64, 64, "C3: Transformer-base translation step (transformer_seq2seq 6+6 "
           "layers d512 h8 ff2048, shared V32768), 64 pairs x (64 source + 64 target tokens), Adam, "
           "tokens weight policy", "transformer_seq2seq-6+6-d512"),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- reference arm
def run_ref_bench(threads: int, batch: int, rounds: int, warmup: int) -> dict:
    cmd = [REF_BIN, "bench", "arch=masked_token_model", f"d={C2['d_model']}",
           f"heads={C2['heads']}", f"vocab={C2['vocab']}", f"max_seq={SEQ}", f"world={threads}",
           f"batch={batch}", f"seq={SEQ}", f"rounds={rounds}", f"warmup={int(warmup > 0)}",
           "eps_ls=0.1"]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def port_bench() -> dict:
    """Oracle port (numpy) timing, used only when oracle/_ref is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import model_oracle as mo
    s = mo.Spec(**{k: v for k, v in dict(arch="bert_encoder", d_model=768, heads=12, vocab=30522,
                                           max_seq=128, layers=12, d_ff=3072).items()})
    p = mo.init_parameters(s, 21)
    rng = np.random.default_rng(0)
    inst = mo.Instance(rng.integers(4, 30522, SEQ), np.array([0] * 64 + [1] * 64),
                       np.arange(1, SEQ, 7), rng.integers(4, 30522, len(range(1, SEQ, 7))), 0)
    t0 = time.perf_counter()
    mo.forward_backward(s, p, [inst])
    dt = time.perf_counter() - t0
    return {"seconds": dt, "samples": 1, "samples_per_s": 1 / dt, "world": 1, "batch": 1}


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    if os.path.exists(REF_BIN):
        threads = ref_threads()
        r = run_ref_bench(threads, 1, max(1, args.steps), args.warmup)
        kind = "reference"
        sample = (f"reference StepEngine<float>::round (engine.hpp:125-165) on {threads} in-process "
                  f"rank threads x 1 sequence of {SEQ} tokens per round, {max(1, args.steps)} timed "
                  f"rounds; 1-block proxy: the reference's masked_token_model at d=768 h=12 "
                  f"V=30522 (it cannot express 12 layers / LayerNorm / FFN)")
    else:
        threads = 1
        r = port_bench()
        kind = "port"
        sample = "numpy oracle port, one 128-token sequence of the full 12-layer model"
    line = {"impl": "reference", "metric": METRIC, "value": r["samples_per_s"], "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * r["seconds"] / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "C2 BERT-base-shaped MLM step (reference 1-block proxy)",
                       "global_batch": r.get("world", 1) * r.get("batch", 1), "seq_len": SEQ,
                       "parallelism": f"inproc threads x{threads}"},
            "cpu_baseline": {"value": r["samples_per_s"], "unit": "samples/s", "cores": threads,
                             "kind": kind, "sample": sample},
            "e2e": {"value": r["samples_per_s"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# The JSON line is the only thing on stdout: native libraries print to fd 1
# (NCCL's "NCCL version ..." banner at communicator init on rank 0), so fd 1
# is pointed at stderr for the whole run and the line goes to a saved copy.
_JSON_FD = None


def _stdout_to_stderr():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def ref_threads() -> int:
    """Rank threads of the reference arm (all host cores, at most 32)."""
    return max(1, min(os.cpu_count() or 1, 32))


def check_first_loss(eng, wspec, batch, policy="sentences") -> dict:
    """Round 1's local loss (the engine's forward on batch 0 under the initial
    parameters) against the numpy f64 oracle's forward of the same batch from
    its own init of seed 21.  Tolerance 1e-2 relative (bf16 GEMM operands)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import model_oracle as mo  # the checker
    t0 = time.perf_counter()
    ls, w = eng.forward(batch)
    ospec = mo.Spec(**wspec)
    p = mo.init_parameters(ospec, 21).astype(np.float32).astype(np.float64)
    n = batch.n_inst
    insts = []
    for i in range(n):
        a, b = int(batch.tok_off[i]), int(batch.tok_off[i + 1])
        c, d = int(batch.mask_off[i]), int(batch.mask_off[i + 1])
        insts.append(mo.Instance(batch.tokens[a:b], batch.segments[a:b], batch.mask_pos[c:d],
                                 batch.mask_orig[c:d], int(batch.label[i])))
    ol, ow, _ = mo.forward_backward(ospec, p, insts, policy, need_grad=False)
    rel = abs(ls - ol) / abs(ol)
    out = {"engine_loss": ls / w, "oracle_loss": ol / ow, "rel": rel, "tol": 1e-2,
           "ok": bool(rel <= 1e-2 and w == ow), "seconds": time.perf_counter() - t0,
           "oracle": "oracle/model_oracle.py forward (numpy f64), batch 0, init seed 21"}
    if not out["ok"]:
        raise RuntimeError(f"bench loss check failed: {out}")
    return out


def same_config_runs(hp, batch, args) -> dict:
    """The reference arm's own workload on the GPU: masked_token_model (the
    reference architecture, model.hpp:334-393) at d=768 h=12 V=30522 seq 128,
    per-step batch of BATCH sequences, on the fp32 path and on the bf16
    tcgen05 path; resident batch, CUDA events on the engine stream."""
    spec = hp.ModelSpec(arch="masked_token_model", d_model=768, heads=12, vocab=30522, max_seq=SEQ,
                        label_smooth_eps=0.1)
    out = {"workload": f"masked_token_model d=768 h=12 V=30522 seq {SEQ} (the reference arm's "
                       f"1-block proxy), {BATCH} sequences per step, Adam", "sequences_per_step": BATCH}
    for comp in ("f32", "bf16"):
        ex = hp.ExecConfig(compute=comp, policy="sentences", device=0, bucket_mb=200.0,
                           max_tokens=BATCH * SEQ, max_batch=BATCH, max_masks=BATCH * SEQ // 2)
        e = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9), ex, seed=21)
        e.stage(batch)
        for _ in range(max(3, args.warmup)):
            e.round_async(False, 1e-4)
        e.round_sync()
        steps = max(5, min(args.steps, 20))
        e.mark(0)
        for _ in range(steps):
            e.round_async(False, 1e-4)
        e.mark(1)
        ms = e.elapsed_ms(0, 1)
        e.round_sync()
        out[comp] = {"value": BATCH * steps / (ms / 1e3), "unit": "samples/s", "steps": steps,
                     "ms_per_step": ms / steps}
        e.close()
    # the headline C2 model itself on the fp32 path (the reference's precision:
    # fp32 operands, fp32-accurate GEMMs on the tensor cores via the bf16x6
    # split), beside the bf16 headline
    ex = hp.ExecConfig(compute="f32", policy="sentences", device=0, bucket_mb=200.0,
                       max_tokens=BATCH * SEQ, max_batch=BATCH, max_masks=BATCH * SEQ // 2)
    e = hp.StepEngine(hp.ModelSpec(**C2), hp.OptimConfig("adam", 0.9, 0.98, 1e-9), ex, seed=21)
    e.stage(batch)
    for _ in range(3):
        e.round_async(False, 1e-4)
    e.round_sync()
    steps = 5
    e.mark(0)
    for _ in range(steps):
        e.round_async(False, 1e-4)
    e.mark(1)
    ms = e.elapsed_ms(0, 1)
    e.round_sync()
    e.close()
    out["c2_f32"] = {"workload": "the C2 model (bert_encoder L12 d768) on the fp32 path", "value":
                     BATCH * steps / (ms / 1e3), "unit": "samples/s", "steps": steps,
                     "ms_per_step": ms / steps}
    return out


# ---------------------------------------------------------------- our arm
def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # gradient bucket cap: 50 MB when buckets are allreduced (N > 1, measured
    # against 25 / 100 MB); at N = 1 buckets only set the update granularity
    # and 200 MB measured best (profiles/r01_ab_bucket_n1.txt)
    ap.add_argument("--bucket-mb", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-loss-check", action="store_true")
    ap.add_argument("--no-same-config", action="store_true")
    args = ap.parse_args(argv)
    _stdout_to_stderr()
    global BATCH, SEQ
    wspec, BATCH, SEQ, wmin, wmax, wdesc, wmodel = WORKLOADS[args.workload]
    if args.workload != "c2":
        args.no_cpu_baseline = True  # the CPU baseline is quoted on the headline config
        args.no_same_config = True
    if args.workload == "c4":
        args.no_loss_check = True  # the numpy oracle's 24-layer seq-512 forward takes minutes
    args.warmup = max(args.warmup, 3)

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.bucket_mb is None:
        args.bucket_mb = 50.0 if world > 1 else 200.0
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import numpy as np
    import torch
    import paper_2009_14783_b200 as hp

    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    comm = hp.Communicator(world, rank, local) if world > 1 else None
    spec = hp.ModelSpec(**wspec)
    s2s = wspec["arch"] == "transformer_seq2seq"
    tok_cap = BATCH * SEQ * (2 if s2s else 1)  # seq2seq: source + target tokens
    ex = hp.ExecConfig(compute="bf16", policy="tokens" if s2s else "sentences", device=local,
                       bucket_mb=args.bucket_mb, max_tokens=tok_cap, max_batch=BATCH,
                       max_masks=1 if s2s else BATCH * SEQ // 2)
    eng = hp.StepEngine(spec, hp.OptimConfig("adam", 0.9, 0.98, 1e-9), ex, comm=comm,
                        seed=21 if rank == 0 else None)
    if comm:
        eng.broadcast_params(0)  # rank 0's parameters win (engine.hpp:263-264)

    # synthetic records (reference generator + exact-length truncation), the
    # epoch plan and this rank's schedule -- identical on every rank
    rounds_needed = args.warmup + args.steps
    if s2s:
        rec = hp.generate_pair_records(hp.PairGenConfig(n=BATCH * world * min(rounds_needed, 8),
                                                        vocab=wspec["vocab"], min_len=wmin,
                                                        max_len=wmax, seed=7))
    else:
        gen = hp.MlmGenConfig(n=BATCH * world * min(rounds_needed, 8), vocab=wspec["vocab"], docs=64,
                              sentences_per_doc=32, min_sentence_words=wmin, max_sentence_words=wmax,
                              seed=7, max_seq_tokens=SEQ)
        rec = hp.generate_mlm_records(gen)
    plan = hp.build_epoch_batches(rec.token_lengths(), BATCH, 0, 21, 0)
    sched = hp.partition_for_rank(plan, world, rank)
    batches = [rec.batch(plan.batches[rb.batch_index]) for rb in sched]
    dummies = [rb.dummy for rb in sched]
    lr = 1e-4

    # ---- first step's loss against the oracle (outside every timed region):
    # the engine's forward on batch 0 under the initial parameters is round
    # 1's local loss; the numpy f64 oracle (oracle/model_oracle.py, the
    # checker) recomputes it from its own init of the same seed
    loss_check = None
    if rank == 0 and not args.no_loss_check:
        loss_check = check_first_loss(eng, wspec, batches[0], "tokens" if s2s else "sentences")

    # ---- value: batch resident in HBM ----
    eng.stage(batches[0])
    for _ in range(args.warmup):
        eng.round_async(dummies[0], lr)
    eng.round_sync()
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before the timed region
    launches0 = hp.StepEngine.kernel_launches()
    eng.mark(0)
    for _ in range(args.steps):
        eng.round_async(dummies[0], lr)
    eng.mark(1)
    launches = hp.StepEngine.kernel_launches() - launches0
    ms = eng.elapsed_ms(0, 1)
    rep = eng.round_sync()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms_max = max_over_ranks(ms)
    value = BATCH * world * args.steps / (ms_max / 1e3)

    # ---- the same K steps again with per-kernel-class CUDA events (roofline
    # and breakdown); kept out of the value pass so the events cost nothing there
    # (timed rounds are graph replays too: the first sighting of the timed
    # shape runs eagerly and the second is captured, so warm both, then reset)
    eng.timers(True)
    for _ in range(2):
        eng.round_async(dummies[0], lr)
        eng.round_sync()
    eng.timers(True)
    eng.mark(2)
    for _ in range(args.steps):
        eng.round_async(dummies[0], lr)
    eng.mark(3)
    ms_timed = eng.elapsed_ms(2, 3)
    eng.round_sync()
    timers = [eng.timer(i) for i in range(6)]
    eng.timers(False)

    # ---- e2e: public API, host batches, H2D + D2H inside the timed region ----
    e2e = None
    if not args.no_e2e:
        h2d, d2h = eng.io_bytes()
        # untimed warm-up through the same API: every distinct batch shape
        # twice, so each CUDA graph is captured before the timed region
        for k in range(max(args.warmup, 2 * len(batches))):
            i = k % len(batches)
            eng.round(batches[i], dummies[i], lr)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        # StepEngine.rounds: batch k+1 is validated / staged on the host while
        # the device runs round k (each round's H2D + D2H stay in the region)
        eng.rounds((batches[k % len(batches)], dummies[k % len(batches)], lr)
                   for k in range(args.steps))
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": BATCH * world * args.steps / e2e_s, "unit": "samples/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": 1e3 * e2e_s / args.steps}
    # ---- gradient allreduce (N > 1): bus GB/s of the engine's bucketed
    # allreduce alone, and how much of it backward hides: exposed = step time
    # with the bucket allreduces - step time without them (last: ranks diverge)
    allreduce = None
    if comm:
        nbytes = 4 * hp.flat_size(spec)
        ar = comm.allreduce_bench(nbytes, args.bucket_mb, iters=5, warmup=2)
        eng.set_grad_comm(False)
        for _ in range(3):
            eng.round_async(dummies[0], lr)
        eng.round_sync()
        torch.cuda.synchronize()
        barrier()
        eng.mark(4)
        for _ in range(args.steps):
            eng.round_async(dummies[0], lr)
        eng.mark(5)
        eng.round_sync()
        ms_nocomm = max_over_ranks(eng.elapsed_ms(4, 5)) / args.steps
        eng.set_grad_comm(True)
        exposed = max(0.0, ms_max / args.steps - ms_nocomm)
        allreduce = {"bus_gbps": ar["busbw_gbps"], "alg_gbps": ar["algbw_gbps"],
                     "bytes_per_step": nbytes, "bucket_mb": args.bucket_mb,
                     "ms_alone": ar["ms"], "ms_per_step_without_grad_allreduce": ms_nocomm,
                     "exposed_ms": exposed,
                     "hidden_frac": max(0.0, 1.0 - exposed / ar["ms"]) if ar["ms"] > 0 else None,
                     "note": "busbw = S/t*2(W-1)/W, S = fp32 gradient bytes, buckets alone on "
                             "one stream; exposed = t_step - t_step(no gradient allreduce)"}
    # ---- the reference's own proxy workload on the GPU (like-for-like anchor) ----
    same = None
    if rank == 0 and world == 1 and not args.no_same_config:
        same = same_config_runs(hp, batches[0], args)

    # ---- roofline of the dominant kernel class (tcgen05 GEMMs).  In-step
    # time = the class's share of the serialised per-kernel time (the timer
    # pass: an event pair around every launch, side streams serialised -- the
    # quantity the committed ncu launch list sums) x the measured step time;
    # achieved = the round's GEMM FLOPs / that time.  Beside it, the GEMMs
    # replayed back to back from a CUDA graph (their isolated serial time).
    # The attention class likewise. ----
    gr = eng.class_replay(0, iters=10)
    ar_ = eng.class_replay(1, iters=10)
    clocks.stop()
    peaks, peak_src = load_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    step_ms = ms_max / args.steps
    t_total = sum(t["ms"] for t in timers)
    t_by = {t["name"]: t["ms"] for t in timers}

    def in_step(cls, flops):
        share = t_by.get(cls, 0.0) / t_total if t_total > 0 else None
        ms_in = share * step_ms if share else None
        tf = flops / (ms_in / 1e3) / 1e12 if ms_in else None
        return share, ms_in, tf

    def tf_of(fl, ms):
        return fl / (ms / 1e3) / 1e12 if ms > 0 else None

    g_share, g_ms, g_tf = in_step("gemm", gr["flops"])
    a_share, a_ms, a_tf = in_step("attention", ar_["flops"])
    roofline = {"bound": "tensor", "kernel": "gemm_tc_kernel (all GEMMs of the step)",
                "achieved": g_tf, "peak": peak, "unit": "TFLOP/s",
                "frac": g_tf / peak if peak and g_tf else None, "traffic": traffic,
                "peak_source": f"bf16_tflops_sustained of {peak_src}",
                "method": "in-step: the GEMMs' share of the serialised per-kernel time (timer "
                          "pass, as the ncu launch list sums it) x ms_per_step; achieved = the "
                          "round's GEMM FLOPs / that time",
                "gemm_flops_per_step": gr["flops"],
                "gemm_ms_per_step": g_ms,
                "gemm_share_of_step": g_share,
                "gemm_launches_per_step": gr["launches"],
                "replay": {"ms_per_step": gr["ms"], "tflops": tf_of(gr["flops"], gr["ms"]),
                           "frac": tf_of(gr["flops"], gr["ms"]) / peak if peak and gr["ms"] > 0 else None,
                           "method": "one round's GEMMs replayed back to back from a CUDA graph "
                                     "on one stream"},
                "attention": {"ms_per_step": a_ms, "flops_per_step": ar_["flops"],
                              "tflops": a_tf, "frac": a_tf / peak if peak and a_tf else None,
                              "share_of_step": a_share,
                              "launches_per_step": ar_["launches"],
                              "replay_ms_per_step": ar_["ms"],
                              "replay_frac": tf_of(ar_["flops"], ar_["ms"]) / peak
                              if peak and ar_["ms"] > 0 else None}}
    breakdown = {t["name"]: round(t["ms"] / args.steps, 4) for t in timers}
    # the memory-bound classes against the measured HBM copy bandwidth
    # (algorithmic bytes / their serialised event time)
    hbm_peak = peaks.get("hbm_gbs")
    hbm_kernels = {}
    for t in timers:
        if t["name"] in ("adam", "layernorm", "embedding", "heads") and t["ms"] > 0 and t["bytes"]:
            gbps = t["bytes"] / (t["ms"] / 1e3) / 1e9
            hbm_kernels[t["name"]] = {"achieved_gbps": round(gbps, 1),
                                      "frac": round(gbps / hbm_peak, 3) if hbm_peak else None,
                                      "launches_per_step": t["launches"] / args.steps}

    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            if os.path.exists(REF_BIN):
                threads = ref_threads()
                r = run_ref_bench(threads, 1, 2, 1)
                cpu = {"value": r["samples_per_s"], "unit": "samples/s", "cores": threads,
                       "kind": "reference",
                       "sample": f"{threads} in-process rank threads x 1 sequence of 128 tokens, "
                                 "1 warm-up + 2 timed StepEngine<float>::round of the reference "
                                 "compiled from source (oracle/_ref) -- the reference arm's own "
                                 "configuration; 1-block proxy of C2 (masked_token_model d=768 "
                                 "h=12 V=30522)"}
            else:
                r = port_bench()
                cpu = {"value": r["samples_per_s"], "unit": "samples/s", "cores": 1,
                       "kind": "port", "sample": "numpy oracle, 1 sequence, full 12-layer model"}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic",
                "config": {"workload": wdesc,
                           "model": wmodel, "global_batch": BATCH * world,
                           "seq_len": SEQ, "parallelism": f"dp{world}",
                           "l2": "no flush: per-step working set (GBs of weights, grads, "
                                 "Adam state, activations) exceeds the 126 MB L2",
                           "bucket_mb": args.bucket_mb},
                "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": launches,
                "roofline": roofline, "hbm_kernels": hbm_kernels, "allreduce": allreduce,
                "cpu_baseline": cpu, "breakdown_ms_per_step": breakdown,
                "breakdown_note": "per-class CUDA events of a timer pass with the side streams "
                                  "serialised (sums above the overlapped step)",
                "loss_check": loss_check, "final_loss": rep.loss}
        if same is not None:
            ref_v = cpu["value"] if cpu and cpu.get("value") else None
            for k in ("f32", "bf16"):
                if k in same and ref_v:
                    same[k]["ratio_vs_reference_cpu"] = same[k]["value"] / ref_v
            same["reference_cpu"] = {"value": ref_v, "cores": cpu.get("cores") if cpu else None}
            line["same_config"] = same
        emit(line)
    eng.close()
    if comm:
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
