/*
 * hetpar_b200.h -- C ABI of the B200-native data-parallel training step.
 *
 * Drop-in boundary for the reference's per-rank DP step (arxiv/paper_2009_14783,
 * "hetpar"): the C++ wrapper include/hetpar_b200/step_engine.hpp and the Python
 * binding paper_2009_14783_b200/_lib.py sit on top of exactly these entry points.
 * Every reference interface an entry point replaces is cited beside it
 * (paths relative to the reference's proj/ directory).
 *
 * Conventions: plain pointers and sizes, no torch types; every call returns an
 * hp_status; on failure hp_last_error() (thread-local) holds the message.  The
 * status codes map 1:1 onto the reference's error taxonomy
 * (include/hetpar/common.hpp:14-34) so a C++ caller can re-throw the matching
 * hetpar::*_error.
 */
#ifndef HETPAR_B200_H
#define HETPAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HP_OK = 0,
  HP_ESHAPE = 1,   /* shape_error   common.hpp:17 */
  HP_ECONFIG = 2,  /* config_error  common.hpp:20 */
  HP_EINDEX = 3,   /* index_error   common.hpp:23 */
  HP_EIO = 4,      /* io_error      common.hpp:26 */
  HP_ECOMM = 5,    /* comm_error    common.hpp:29 */
  HP_ENUMERIC = 6, /* numeric_error common.hpp:32 */
  HP_ECUDA = 7     /* device failure (no reference counterpart) */
} hp_status;

const char* hp_last_error(void);
const char* hp_version(void);

/* ------------------------------------------------------------------------
 * Host data path (bit-exact with the reference).
 * ---------------------------------------------------------------------- */

/* SeededRng::next_u64 stream (include/hetpar/rng.hpp:15-22). */
hp_status hp_splitmix64(uint64_t seed, uint64_t n, uint64_t* out);
/* shuffle(iota(n), SeededRng(seed)) (rng.hpp:74-82). */
hp_status hp_shuffle_iota(uint64_t seed, uint64_t n, uint64_t* out);

/* build_epoch_batches (src/dataset.cpp:52-88). order[n] receives the shuffled
 * global ids, sizes[*nbatches] the batch lengths (batch b is the next
 * sizes[b] ids of order). HP_ECONFIG when an instance exceeds max_tokens. */
hp_status hp_build_epoch_batches(const uint32_t* token_lengths, uint64_t n,
                                 uint64_t max_sentences, uint64_t max_tokens,
                                 uint64_t base_seed, uint64_t epoch,
                                 uint64_t* order, uint64_t* sizes,
                                 uint64_t* nbatches);

/* partition_for_rank (src/dataset.cpp:90-117): rounds = ceil(nbatches/world)
 * entries; batch_index/dummy have capacity for them. */
hp_status hp_partition_for_rank(uint64_t nbatches, uint64_t world,
                                uint64_t rank, uint64_t* batch_index,
                                uint8_t* dummy, uint64_t* rounds);

/* Synthetic MLM record stream: generate_mlm_shards' record sequence
 * (src/datagen.cpp:71-127; make_nsp_pair / assemble_pair / mask_tokens,
 * src/textgen.cpp:24-95), in memory instead of HSD1 shards.  max_seq_tokens>0
 * is a repo extension: BERT-style truncation of the pair (no extra draws). */
typedef struct {
  uint64_t n;
  int64_t vocab;
  uint64_t docs;
  uint64_t sentences_per_doc;
  uint64_t min_words;
  uint64_t max_words;
  double p_select;
  double p_mask;
  double p_random;
  uint64_t seed;
  uint64_t max_seq_tokens;
} hp_mlm_gen_desc;

hp_status hp_mlm_generate_size(const hp_mlm_gen_desc* d, uint64_t* tokens_total,
                               uint64_t* masks_total);
/* CSR output: tok_off[n+1], tokens/segments[tokens_total];
 * mask_off[n+1], mask_pos/mask_orig[masks_total]; label[n]. */
hp_status hp_mlm_generate(const hp_mlm_gen_desc* d, uint64_t* tok_off,
                          int64_t* tokens, int64_t* segments,
                          uint64_t* mask_off, int64_t* mask_pos,
                          int64_t* mask_orig, int64_t* label);

/* Synthetic translation pairs for the seq2seq extension (repo generator, no
 * reference counterpart): pair k draws, from SeededRng(seed) in this order,
 * its source length and target length (min_len + bounded(max_len - min_len
 * + 1) each), then the source and the target word ids (4 + bounded(vocab - 4)
 * each).  Record k = tokens [source..., target...] with segments 0 / 1; no
 * masks, label 0 -- the hp_batch encoding of a pair (see hp_engine_round). */
typedef struct {
  uint64_t n;
  int64_t vocab;
  uint64_t min_len, max_len;
  uint64_t seed;
} hp_pair_gen_desc;
hp_status hp_pairs_generate_size(const hp_pair_gen_desc* d, uint64_t* tokens_total);
hp_status hp_pairs_generate(const hp_pair_gen_desc* d, uint64_t* tok_off, int64_t* tokens,
                            int64_t* segments);

/* ------------------------------------------------------------------------
 * Model description and canonical parameter table.
 * ---------------------------------------------------------------------- */
enum {
  HP_ARCH_MASKED_TOKEN_MODEL = 3, /* Arch::masked_token_model, model.hpp:16 */
  HP_ARCH_BERT_ENCODER = 16,      /* repo extension: L post-LN BERT blocks   */
  HP_ARCH_SEQ2SEQ = 17            /* repo extension: L + L encoder-decoder
                                     Transformer, shared
                                     embedding / output projection */
};

/* ModelSpec (include/hetpar/model.hpp:28-67) + the extension's fields. */
typedef struct {
  int arch;
  uint64_t d_model;
  uint64_t heads;
  uint64_t vocab;
  uint64_t max_seq;
  uint64_t layers; /* bert_encoder; seq2seq: encoder layers = decoder layers */
  uint64_t d_ff;   /* bert_encoder, seq2seq */
  int with_nsp;    /* ignored by seq2seq (no NSP head) */
  double label_smooth_eps;
} hp_model_desc;

enum { HP_PARAM_WEIGHT = 0, HP_PARAM_TABLE = 1, HP_PARAM_BIAS = 2, HP_PARAM_GAIN = 3 };

/* param_shapes (model.hpp:91-142): count and flat element total. */
hp_status hp_param_count(const hp_model_desc* m, uint64_t* nparams,
                         uint64_t* nelems);
hp_status hp_param_info(const hp_model_desc* m, uint64_t i, char* name,
                        uint64_t name_cap, uint64_t* rows, uint64_t* cols,
                        uint64_t* offset, int* kind);
/* init_parameters<double> with derived_rng(seed, 0) (model.hpp:171-184). */
hp_status hp_init_parameters(const hp_model_desc* m, uint64_t seed, double* out);

/* Gradient buckets: whole parameters walked in reverse canonical
 * order, closed when the next would exceed bucket_bytes (fp32). bucket i is
 * the flat range [lo[i], hi[i]).  Capacity nparams. */
hp_status hp_bucket_plan(const hp_model_desc* m, double bucket_mb,
                         uint64_t* lo, uint64_t* hi, uint64_t* nbuckets);

/* ------------------------------------------------------------------------
 * Communicator: one process per GPU, NCCL over NVLink/NVSwitch.  The 128-byte
 * id is created on rank 0 and shipped with ProcessGroup::broadcast
 * (comm.hpp:25-27) or torch.distributed.
 * ---------------------------------------------------------------------- */
typedef struct hp_comm hp_comm;
hp_status hp_comm_unique_id(uint8_t id[128]);
hp_status hp_comm_create(int world, int rank, int device, const uint8_t id[128],
                         hp_comm** out);
hp_status hp_comm_destroy(hp_comm* c);
/* Form the world without a Python control plane: rank 0 listens on
 * host:port and serves its ncclUniqueId to the other ranks (the rendezvous
 * role of comm_tcp.cpp:154-237); retries / waits up to timeout_ms. */
hp_status hp_comm_create_tcp(const char* host, uint16_t port, int world, int rank, int device,
                             int timeout_ms, hp_comm** out);
/* ProcessGroup (comm.hpp:16-49) over the communicator -- the NcclProcessGroup
 * control plane; host-staged, blocking:
 *   broadcast: every rank gets the root's bytes (*out_len = their length;
 *     HP_ECONFIG when cap is smaller);
 *   all_reduce_sum: the rank-ordered left fold 0..world-1, identical bytes on
 *     every rank; differing lengths are HP_ECOMM;
 *   gather_scalars: the master (rank 0) receives [v_0..v_{w-1}] in out;
 *   barrier: returns once every rank entered. */
hp_status hp_pg_broadcast(hp_comm* c, const void* payload, uint64_t len, uint64_t root, void* out,
                          uint64_t cap, uint64_t* out_len);
hp_status hp_pg_all_reduce_sum(hp_comm* c, const double* v, uint64_t n, double* out);
hp_status hp_pg_gather_scalars(hp_comm* c, double v, double* out);
hp_status hp_pg_barrier(hp_comm* c);
/* Gradient-allreduce measurement (BASELINE metric "allreduce bus GB/s", the
 * C5 sweep): `bytes` of fp32 on this rank's device, cut into contiguous
 * buckets of at most bucket_mb MiB (the engine's layout), each bucket one
 * in-place ncclAllReduce(ncclSum) on one stream -- the engine's call
 * (engine.cpp issue_bucket; the reference's all_reduce_sum,
 * engine.hpp:145).  warmup untimed iterations, then iters timed with CUDA
 * events on that stream; *ms = mean milliseconds per iteration (every
 * bucket of the buffer).  Collective: every rank calls it with the same
 * arguments. */
hp_status hp_comm_allreduce_bench(hp_comm* c, uint64_t bytes, double bucket_mb, int iters,
                                  int warmup, double* ms);

/* ------------------------------------------------------------------------
 * Step engine: StepEngine<T>::round (include/hetpar/engine.hpp:125-165).
 * ---------------------------------------------------------------------- */
typedef struct hp_engine hp_engine;

enum { HP_OPT_SGD = 0, HP_OPT_ADAM = 1,            /* OptKind, optim.hpp:77 */
       HP_OPT_ADAMW = 2 };  /* extension: Adam + decoupled weight decay (p -= lr wd p, then Adam) */
enum { HP_POLICY_SENTENCES = 1, HP_POLICY_TOKENS = 2 }; /* WeightPolicy */
enum { HP_COMPUTE_F32 = 0, HP_COMPUTE_BF16 = 1 };

typedef struct {
  int kind;
  double beta1, beta2, eps;
  double weight_decay; /* HP_OPT_ADAMW only */
} hp_optim_desc;

typedef struct {
  int compute;          /* HP_COMPUTE_F32: fp32 parity path; BF16: tcgen05 */
  int policy;           /* weight policy */
  int device;           /* CUDA ordinal */
  double bucket_mb;     /* gradient bucket cap */
  uint64_t max_tokens;  /* capacity: tokens per rank batch */
  uint64_t max_batch;   /* capacity: instances per rank batch */
  uint64_t max_masks;   /* capacity: masked positions per rank batch */
  uint64_t update_freq; /* K micro rounds per update (Accumulator) */
} hp_exec_desc;

/* Batch = vector<Instance> (model.hpp:72-83), flattened to CSR. */
typedef struct {
  uint64_t n_inst;
  const uint64_t* tok_off;   /* [n_inst+1] */
  const int64_t* tokens;     /* [tok_off[n]] */
  const int64_t* segments;   /* [tok_off[n]] */
  const uint64_t* mask_off;  /* [n_inst+1] */
  const int64_t* mask_pos;   /* within-instance positions */
  const int64_t* mask_orig;
  const int64_t* label;      /* [n_inst] NSP label */
} hp_batch;

/* StepReport (engine.hpp:26-32) minus the host timing fields. */
typedef struct {
  int updated;       /* 1 when this round completed an update (K-th round) */
  uint64_t step;     /* P after this update */
  double loss;       /* global loss_sum / weight of the update */
  double weight;     /* global weight of the update */
  double local_loss_sum;
  double local_weight;
} hp_round_out;

hp_status hp_engine_create(const hp_model_desc* m, const hp_optim_desc* o,
                           const hp_exec_desc* x, hp_comm* comm /* NULL: world 1 */,
                           hp_engine** out);
hp_status hp_engine_destroy(hp_engine* e);
/* canonical flat parameters (params_to_bytes order, model.hpp:190-195);
 * dtype 0 = f32, 1 = f64. */
hp_status hp_engine_set_params(hp_engine* e, const void* flat, uint64_t n, int dtype);
hp_status hp_engine_get_params(hp_engine* e, void* flat, uint64_t n, int dtype);
/* rank root's parameters win (engine.hpp:263-264). */
hp_status hp_engine_broadcast_params(hp_engine* e, int root);
/* Adam state (for HCK1): m, v in canonical order, t. */
hp_status hp_engine_get_adam(hp_engine* e, float* m, float* v, uint64_t* t);
hp_status hp_engine_set_adam(hp_engine* e, const float* m, const float* v, uint64_t t);

/* ------------------------------------------------------------------------
 * HSD1 shard read path (src/shard.cpp:126-218, dataset.cpp:10-50,
 * loader.cpp:80-139): shards of a directory memory-mapped as one global
 * record space; a loader assembles one rank's schedule into hp_batch CSR
 * arrays on a prefetch thread (prefetch_depth batches ahead; 0 = on demand).
 * ---------------------------------------------------------------------- */
typedef struct hp_shards hp_shards;
typedef struct hp_loader hp_loader;
hp_status hp_shards_open(const char* dir, hp_shards** out);
hp_status hp_shards_info(hp_shards* s, uint64_t* total, uint64_t* nshards);
hp_status hp_shards_token_lengths(hp_shards* s, uint32_t* out, uint64_t n);
hp_status hp_shards_close(hp_shards* s);
/* generate_mlm_shards' files (datagen.cpp:71-127) for n records in CSR form */
hp_status hp_mlm_write_shards(const char* dir, uint64_t n, uint64_t shards, const uint64_t* tok_off,
                              const int64_t* tokens, const int64_t* segments,
                              const uint64_t* mask_off, const int64_t* mask_pos,
                              const int64_t* mask_orig, const int64_t* label);
/* The epoch plan (batch_order = concatenated global ids, batch_sizes) and one
 * rank's schedule (partition_for_rank) to serve, in order. */
hp_status hp_loader_create(hp_shards* s, const uint64_t* batch_order, const uint64_t* batch_sizes,
                           uint64_t nbatches, const uint64_t* sched_batch,
                           const uint8_t* sched_dummy, uint64_t nsched, uint64_t prefetch_depth,
                           hp_loader** out);
typedef struct {
  uint64_t batch_index;
  int dummy;
  hp_batch batch; /* arrays owned by the loader, valid until the next call */
} hp_loaded_batch;
/* *has = 0 (and out untouched) once the schedule is exhausted */
hp_status hp_loader_next(hp_loader* l, hp_loaded_batch* out, int* has);
hp_status hp_loader_destroy(hp_loader* l);

/* ------------------------------------------------------------------------
 * HCK1 checkpoints (src/checkpoint.cpp:165-302) and resume fast-forward
 * (include/hetpar/engine.hpp:211-245).  Files are byte-compatible with the
 * reference's save_checkpoint<float> / load_checkpoint<float>.
 * ---------------------------------------------------------------------- */
typedef struct {
  uint64_t epoch, step, seed;  /* TrainState (checkpoint.hpp:15-37) */
  int policy;                  /* HP_POLICY_* */
  uint64_t world_size, update_freq;
  int sched_kind;              /* SchedulerKind: 0 fixed, 1 inverse_sqrt, 2 linear */
  double peak_lr;
  uint64_t sched_d_model, warmup_steps, total_steps;
  int opt_kind;                /* HP_OPT_* */
  double beta1, beta2, eps;
  uint64_t opt_t;              /* Adam step counter */
  double weight_decay;         /* HP_OPT_ADAMW (spec key "weight_decay") */
} hp_ckpt_desc;
/* Host-side writer / reader of one f32 checkpoint; params, m, v are flat
 * canonical vectors (m, v read/written only for Adam).  hp_checkpoint_read
 * validates magic, digest, version, policy, dtype, names and shapes; the
 * output pointers may be null for a metadata-only read (n = their capacity). */
hp_status hp_checkpoint_write(const char* path, const hp_model_desc* m, const hp_ckpt_desc* c,
                              const float* params, const float* adam_m, const float* adam_v);
hp_status hp_checkpoint_read(const char* path, hp_model_desc* m, hp_ckpt_desc* c, float* params,
                             float* adam_m, float* adam_v, uint64_t n);
/* save_checkpoint from device state (master rank): c supplies epoch, seed,
 * policy, world, update_freq and the scheduler; step, the optimizer and its
 * moments come from the engine.  Inside a partially accumulated update group
 * (K > 1) the file holds the last update's state and the pending rounds stay
 * pending (the format has no accumulator block, as the reference's). */
hp_status hp_engine_save_checkpoint(hp_engine* e, const char* path, const hp_ckpt_desc* c);
/* load_checkpoint into device state: parameters, Adam moments and t, step,
 * and the file's optimizer (kind, betas, eps) and weight policy, as the
 * reference's TrainState (checkpoint.cpp:254, 282-289); the file's model must
 * equal the engine's; a pending accumulation is dropped.  c (may be null)
 * receives the file's metadata. */
hp_status hp_engine_load_checkpoint(hp_engine* e, const char* path, hp_ckpt_desc* c);
/* Epoch and rounds to skip after `step` updates of world x update_freq
 * lockstep rounds (engine.hpp:225-244). */
hp_status hp_resume_position(const uint32_t* lens, uint64_t n, uint64_t max_sentences,
                             uint64_t max_tokens, uint64_t seed, uint64_t world,
                             uint64_t update_freq, uint64_t step, uint64_t* epoch,
                             uint64_t* skip_rounds);
/* local (pre-reduce) gradient of the last round, canonical order; valid after
 * hp_engine_round_sync when debug capture is on. */
hp_status hp_engine_set_capture(hp_engine* e, int on);
hp_status hp_engine_get_local_grads(hp_engine* e, float* flat, uint64_t n);

/* Stage a rank batch: host CSR -> pinned -> one H2D copy on the engine's
 * stream.  Returns as soon as the copy is enqueued. */
hp_status hp_engine_stage_batch(hp_engine* e, const hp_batch* b);
/* One lockstep round on the staged batch: forward -> [loss, weight] allreduce
 * -> backward with bucketed gradient allreduce on a side stream -> (K-th round)
 * /sum(weight) and the optimizer update.  lr = scheduled_lr(P+1).  _async
 * enqueues only; _sync waits and fills out (and raises numeric errors the way
 * engine.hpp:134-138 does). hp_engine_round = async + sync. */
/* model_forward (model.hpp:260-390) on the staged batch alone: its summed
 * loss (ForwardResult::loss_sum) and weight; no backward, no collective, no
 * update (evaluation). */
hp_status hp_engine_forward(hp_engine* e, double* loss_sum, double* weight);
hp_status hp_engine_round_async(hp_engine* e, int dummy, double lr);
hp_status hp_engine_round_sync(hp_engine* e, hp_round_out* out);
hp_status hp_engine_round(hp_engine* e, int dummy, double lr, hp_round_out* out);
/* params_digest (model.hpp:211-217): FNV-1a over the f32 parameter bytes. */
hp_status hp_engine_params_digest(hp_engine* e, uint64_t* digest);
/* check_digest_on_cadence (engine.hpp:170-184), run by hp_engine_round_sync
 * after an update whose step is a multiple of `every` (every update when
 * debug != 0; every = 0 disables; default 100, the reference's
 * EngineConfig::check_interval): rank 0's parameter digest is broadcast,
 * mismatches are summed over the ranks, and any mismatch is HP_ENUMERIC
 * ("k ranks diverged from master parameters at step P") on every rank.
 * Collective whenever the engine has a communicator (world 1 included). */
hp_status hp_engine_set_digest_check(hp_engine* e, uint64_t every, int debug);
/* Number of this library's kernels launched since creation (for bench). */
hp_status hp_engine_kernel_launches(hp_engine* e, uint64_t* n);
/* CUDA-event time (ms) of the dominant kernel class over the last sync
 * window; name receives its label. */
hp_status hp_engine_timers(hp_engine* e, int enable);
hp_status hp_engine_timer_read(hp_engine* e, int which, char* name, uint64_t cap,
                               double* ms, uint64_t* launches, double* bytes,
                               double* flops);
/* Measurement: the kernels of one class (0 GEMM, 1 attention; the
 * hp_engine_timer_read classes) of one round, recorded during one eager round
 * (a real update on the staged batch, lr 0) and replayed back to back on one
 * stream from a CUDA graph `iters` times: *ms = the class's serialised time
 * per round (what a per-kernel profile sums), *flops its algorithmic FLOPs,
 * *launches its kernels per round.  Overwrites the class's outputs. */
hp_status hp_engine_class_replay(hp_engine* e, int which, int iters, double* ms, double* flops,
                                 uint64_t* launches);
hp_status hp_engine_step_count(hp_engine* e, uint64_t* step);
/* TrainState::step (checkpoint.hpp:27) of a state handed to the engine by a
 * caller that owns it (the C++ drop-in for StepEngine<T>, reference_dropin.hpp):
 * P, the completed updates; refused inside a partial update group. */
hp_status hp_engine_set_step(hp_engine* e, uint64_t step);
/* StepEngine::pending_rounds (engine.hpp:165): rounds accumulated since the
 * last update (0 .. update_freq - 1). */
hp_status hp_engine_pending_rounds(hp_engine* e, uint64_t* n);
/* CUDA events on the engine's compute stream (the stream every kernel of the
 * step is launched on): mark(slot) records, elapsed(a, b) waits for b and
 * returns milliseconds between the two marks. slots 0..7. */
hp_status hp_engine_mark(hp_engine* e, int slot);
hp_status hp_engine_elapsed(hp_engine* e, int a, int b, double* ms);
hp_status hp_engine_synchronize(hp_engine* e);
/* bytes one hp_engine_stage_batch copies host->device, and one round copies
 * device->host (the [loss, weight] readback + status flags). */
hp_status hp_engine_io_bytes(hp_engine* e, uint64_t* h2d, uint64_t* d2h);
/* Measurement only (bench.py's overlap figure): on = 0 skips the gradient
 * bucket allreduces of later rounds (the [loss, weight] allreduce stays), so
 * t_step(on) - t_step(off) is the gradient communication left exposed behind
 * backward.  Ranks then diverge; default on. */
hp_status hp_engine_set_grad_comm(hp_engine* e, int on);


/* ------------------------------------------------------------------------
 * Operator table: hetpar::kern (include/hetpar/kernels.hpp:44-68,
 * src/kernels_scalar.cpp) on DEVICE pointers, ordered on `stream` (NULL: the
 * legacy default stream); a reduction writes its scalar to device memory.
 * Bit-identical to the reference's kernels: explicitly rounded operations
 * (no FMA), IEEE sqrt / divide, and the reference's lane contract for
 * reductions (L = 8 lanes for f32, 4 for f64 over the leading multiple-of-L
 * prefix, lanes folded left to right, then the tail in order) -- sequential
 * per lane by definition, so reductions run L threads wide.
 * ---------------------------------------------------------------------- */
hp_status hp_kern_dot_f32(const float* a, const float* b, uint64_t n, float* out, void* stream);
hp_status hp_kern_sum_f32(const float* a, uint64_t n, float* out, void* stream);
hp_status hp_kern_maxv_f32(const float* a, uint64_t n, float* out, void* stream);
hp_status hp_kern_add_f32(const float* a, const float* b, float* out, uint64_t n, void* stream);
hp_status hp_kern_scale_f32(const float* a, float s, float* out, uint64_t n, void* stream);
hp_status hp_kern_axpy_f32(float alpha, const float* x, float* y, uint64_t n, void* stream);
hp_status hp_kern_relu_f32(const float* a, float* out, uint64_t n, void* stream);
hp_status hp_kern_relu_bwd_f32(const float* a, const float* g, float* da, uint64_t n, void* stream);
hp_status hp_kern_sgd_update_f32(float* p, const float* g, uint64_t n, float lr, void* stream);
hp_status hp_kern_adam_update_f32(float* p, float* m, float* v, const float* g, uint64_t n, float lr, float b1,
                                  float b2, float eps, float c1, float c2, void* stream);
hp_status hp_kern_dot_f64(const double* a, const double* b, uint64_t n, double* out, void* stream);
hp_status hp_kern_sum_f64(const double* a, uint64_t n, double* out, void* stream);
hp_status hp_kern_maxv_f64(const double* a, uint64_t n, double* out, void* stream);
hp_status hp_kern_add_f64(const double* a, const double* b, double* out, uint64_t n, void* stream);
hp_status hp_kern_scale_f64(const double* a, double s, double* out, uint64_t n, void* stream);
hp_status hp_kern_axpy_f64(double alpha, const double* x, double* y, uint64_t n, void* stream);
hp_status hp_kern_relu_f64(const double* a, double* out, uint64_t n, void* stream);
hp_status hp_kern_relu_bwd_f64(const double* a, const double* g, double* da, uint64_t n, void* stream);
hp_status hp_kern_sgd_update_f64(double* p, const double* g, uint64_t n, double lr, void* stream);
hp_status hp_kern_adam_update_f64(double* p, double* m, double* v, const double* g, uint64_t n, double lr, double b1,
                                  double b2, double eps, double c1, double c2, void* stream);

/* ------------------------------------------------------------------------
 * Test hooks (used by tests/ only): run one GEMM of the engine's dispatch on
 * caller-owned device buffers.  path: 0 auto, 1 SIMT fp32, 2 tcgen05, 4 fp32
 * operands on tcgen05 through the bf16x6 split (kernels.cu).
 * act: 0 none, 1 GELU (pre-activation to aux), 2 dGELU (multiply by
 * GELU'(aux)).  bn = 10000 * s + 1000 * cg + tile: tile width (0 = heuristic,
 * 128, 192 or 256), cg CTA group (0 heuristic, 1 single CTA, 2 CTA pair), s a
 * forced s-way split-K (fp32 C without epilogue ops).
 * ---------------------------------------------------------------------- */
hp_status hp_debug_gemm(int M, int N, int K, int ab_bf16, const void* A, int64_t lda,
                        int a_trans, const void* B, int64_t ldb, int b_trans,
                        int64_t b_group, int64_t b_gstride, void* C, int64_t ldc,
                        int c_bf16, int64_t c_group, int64_t c_gstride,
                        const float* bias, int act, void* aux, const void* resid,
                        int64_t ld_resid, int accumulate, int path, int bn);
hp_status hp_debug_sync(void);
/* stream for hp_debug_gemm (NULL: the legacy default stream) -- lets a
 * microbenchmark capture its launches into a CUDA graph */
hp_status hp_debug_set_stream(void* stream);
/* Profiling hook: when buf (device, >= 1024 u64) is non-null, CTA 0 of every
 * following tcgen05 GEMM writes a clock64 timeline into it; null disables. */
hp_status hp_debug_gemm_trace(unsigned long long* buf);
/* Test hook: 1 forces every tcgen05 GEMM onto the generic epilogue kernel
 * (all epilogue flags at run time) instead of the per-kind specialisation. */
hp_status hp_debug_gemm_generic(int on);
/* Varlen self-attention on caller-owned device buffers: cu[B+1] (int32,
 * device), qkv [T x 3*H*dk], o [T x H*dk], lse [H x T], dO, dqkv.  bf16 = 1
 * selects bf16 I/O; path: 0 auto, 1 SIMT, 2 tensor-core (mma.sync), 3 tcgen05. */
hp_status hp_debug_attention(int B, const int* cu, int T, int H, int dk, int bf16,
                             const void* qkv, void* o, float* lse, const void* dO,
                             void* dqkv, int path);
/* LayerNorm of the engine (x [T x d] -> y, mean/rstd [T]) and, when dy is
 * non-null, its backward: dx, dg = colsum(dy * xhat), db = colsum(dy) and
 * (dbias non-null) colsum(dx).  bf16 = 1: bf16 x / y / dy / dx (d % 256 == 0,
 * d <= 1024 takes the bulk-copy kernels the BERT step runs); deferred = 1
 * runs the column-sum final as a separate launch, as the engine does. */
hp_status hp_debug_layernorm(int T, int d, int bf16, const void* x, const float* g, const float* b,
                             void* y, float* mean, float* rstd, const void* dy, void* dx, float* dg,
                             float* db, float* dbias, int deferred);
/* Generalised attention (self or cross, causal or not; kernels.h AttnArgs)
 * on caller-owned device buffers: queries of instance b are rows
 * [cu_q[b], cu_q[b+1]) of q (pitch ldq, head h at column qcol + h dk), keys /
 * values rows [cu_kv[b], cu_kv[b+1]) of k / v; o [T_q x H dk], lse [H x T_q];
 * when dO is non-null the backward writes dq / dk / dv with their pitches
 * and column offsets.  path: 0 auto, 1 SIMT, 3 tcgen05. */
hp_status hp_debug_attention2(int B, const int* cu_q, const int* cu_kv, int T_q, int T_kv,
                              int max_q, int max_kv, int H, int dk, int bf16, const void* q,
                              int64_t ldq, int qcol, const void* k, int64_t ldk, int kcol,
                              const void* v, int64_t ldv, int vcol, void* o, float* lse,
                              const void* dO, void* dq, int64_t lddq, int dqcol, void* dkk,
                              int64_t lddk, int dkcol, void* dv, int64_t lddv, int dvcol,
                              int causal, int path);
/* One Adam (sgd=0) or SGD (sgd=1) update of the device kernel on caller-owned
 * device fp32 buffers, no scaling: compare with kern::adam_update<float>;
 * wd != 0: AdamW (p -= (lr wd) p before the Adam step, fp32, RN). */
hp_status hp_debug_adam(float* p, float* m, float* v, const float* g, uint64_t n,
                        float lr, float b1, float b2, float eps, float c1, float c2,
                        int sgd, float wd);

#ifdef __cplusplus
}
#endif
#endif /* HETPAR_B200_H */
