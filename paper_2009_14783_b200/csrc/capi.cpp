// extern "C" boundary (include/hetpar_b200.h).  Every entry point converts
// exceptions into hp_status + a thread-local message.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include <memory>

#include "checkpoint.h"
#include "shards.h"
#include "engine.h"
#include "hetpar_b200.h"
#include "hostdata.h"
#include "hp_common.h"

namespace hp {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace hp

using hp::fail;

struct hp_engine {
  hp::Engine* e = nullptr;
};
struct hp_shards {
  std::shared_ptr<const hp::ShardSet> set;
};
struct hp_loader {
  std::unique_ptr<hp::ShardLoader> loader;
  hp::ShardLoader::Loaded cur;
};

static void need(const void* p, const char* what) {
  if (!p) fail(HP_ECONFIG, std::string("null pointer: ") + what);
}

extern "C" {

const char* hp_last_error(void) { return hp::g_last_error.c_str(); }
const char* hp_version(void) { return "hetpar_b200 0.1 (sm_100a)"; }

hp_status hp_splitmix64(uint64_t seed, uint64_t n, uint64_t* out) {
  HP_API_BEGIN
  need(out, "out");
  hp::SplitMix r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.next();
  HP_API_END
}

hp_status hp_shuffle_iota(uint64_t seed, uint64_t n, uint64_t* out) {
  HP_API_BEGIN
  need(out, "out");
  std::vector<uint64_t> a(n);
  for (uint64_t i = 0; i < n; ++i) a[i] = i;
  hp::SplitMix r(seed);
  hp::shuffle_u64(a, r);
  std::memcpy(out, a.data(), n * 8);
  HP_API_END
}

hp_status hp_build_epoch_batches(const uint32_t* lens, uint64_t n, uint64_t max_sentences,
                                 uint64_t max_tokens, uint64_t base_seed, uint64_t epoch,
                                 uint64_t* order, uint64_t* sizes, uint64_t* nbatches) {
  HP_API_BEGIN
  need(nbatches, "nbatches");
  if (n) {
    need(lens, "token_lengths");
    need(order, "order");
    need(sizes, "sizes");
  }
  auto p = hp::build_epoch_batches(lens, n, max_sentences, max_tokens, base_seed, epoch);
  if (n) std::memcpy(order, p.order.data(), n * 8);
  if (!p.sizes.empty()) std::memcpy(sizes, p.sizes.data(), p.sizes.size() * 8);
  *nbatches = p.sizes.size();
  HP_API_END
}

hp_status hp_partition_for_rank(uint64_t nbatches, uint64_t world, uint64_t rank,
                                uint64_t* batch_index, uint8_t* dummy, uint64_t* rounds) {
  HP_API_BEGIN
  need(rounds, "rounds");
  auto s = hp::partition_for_rank(nbatches, world, rank);
  need(batch_index, "batch_index");
  need(dummy, "dummy");
  for (size_t t = 0; t < s.size(); ++t) {
    batch_index[t] = s[t].batch_index;
    dummy[t] = s[t].dummy ? 1 : 0;
  }
  *rounds = s.size();
  HP_API_END
}

hp_status hp_mlm_generate_size(const hp_mlm_gen_desc* d, uint64_t* tokens_total,
                               uint64_t* masks_total) {
  HP_API_BEGIN
  need(d, "desc");
  auto r = hp::mlm_generate(*d);
  *tokens_total = r.tokens.size();
  *masks_total = r.mask_pos.size();
  HP_API_END
}

hp_status hp_mlm_generate(const hp_mlm_gen_desc* d, uint64_t* tok_off, int64_t* tokens,
                          int64_t* segments, uint64_t* mask_off, int64_t* mask_pos,
                          int64_t* mask_orig, int64_t* label) {
  HP_API_BEGIN
  need(d, "desc");
  auto r = hp::mlm_generate(*d);
  std::memcpy(tok_off, r.tok_off.data(), r.tok_off.size() * 8);
  std::memcpy(tokens, r.tokens.data(), r.tokens.size() * 8);
  std::memcpy(segments, r.segments.data(), r.segments.size() * 8);
  std::memcpy(mask_off, r.mask_off.data(), r.mask_off.size() * 8);
  if (!r.mask_pos.empty()) {
    std::memcpy(mask_pos, r.mask_pos.data(), r.mask_pos.size() * 8);
    std::memcpy(mask_orig, r.mask_orig.data(), r.mask_orig.size() * 8);
  }
  std::memcpy(label, r.label.data(), r.label.size() * 8);
  HP_API_END
}

hp_status hp_pairs_generate_size(const hp_pair_gen_desc* d, uint64_t* tokens_total) {
  HP_API_BEGIN
  need(d, "desc");
  need(tokens_total, "tokens_total");
  *tokens_total = hp::pairs_generate(*d).tokens.size();
  HP_API_END
}

hp_status hp_pairs_generate(const hp_pair_gen_desc* d, uint64_t* tok_off, int64_t* tokens,
                            int64_t* segments) {
  HP_API_BEGIN
  need(d, "desc");
  auto r = hp::pairs_generate(*d);
  std::memcpy(tok_off, r.tok_off.data(), r.tok_off.size() * 8);
  std::memcpy(tokens, r.tokens.data(), r.tokens.size() * 8);
  std::memcpy(segments, r.segments.data(), r.segments.size() * 8);
  HP_API_END
}

hp_status hp_param_count(const hp_model_desc* m, uint64_t* nparams, uint64_t* nelems) {
  HP_API_BEGIN
  need(m, "model");
  auto t = hp::param_table(*m);
  *nparams = t.size();
  *nelems = t.back().offset + t.back().size();
  HP_API_END
}

hp_status hp_param_info(const hp_model_desc* m, uint64_t i, char* name, uint64_t name_cap,
                        uint64_t* rows, uint64_t* cols, uint64_t* offset, int* kind) {
  HP_API_BEGIN
  need(m, "model");
  auto t = hp::param_table(*m);
  if (i >= t.size()) fail(HP_EINDEX, "parameter index out of range");
  const auto& e = t[i];
  if (name && name_cap) {
    std::strncpy(name, e.name.c_str(), name_cap - 1);
    name[name_cap - 1] = 0;
  }
  if (rows) *rows = e.rows;
  if (cols) *cols = e.cols;
  if (offset) *offset = e.offset;
  if (kind) *kind = e.kind;
  HP_API_END
}

hp_status hp_init_parameters(const hp_model_desc* m, uint64_t seed, double* out) {
  HP_API_BEGIN
  need(m, "model");
  need(out, "out");
  auto v = hp::init_parameters(*m, seed);
  std::memcpy(out, v.data(), v.size() * 8);
  HP_API_END
}

hp_status hp_bucket_plan(const hp_model_desc* m, double bucket_mb, uint64_t* lo, uint64_t* hi,
                         uint64_t* nbuckets) {
  HP_API_BEGIN
  need(m, "model");
  auto b = hp::bucket_plan(hp::param_table(*m), bucket_mb);
  for (size_t i = 0; i < b.size(); ++i) {
    lo[i] = b[i].lo;
    hi[i] = b[i].hi;
  }
  *nbuckets = b.size();
  HP_API_END
}

hp_status hp_comm_unique_id(uint8_t id[128]) {
  HP_API_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  HP_NCCL(ncclGetUniqueId(&u));
  std::memcpy(id, &u, 128);
  HP_API_END
}

hp_status hp_comm_create(int world, int rank, int device, const uint8_t id[128], hp_comm** out) {
  HP_API_BEGIN
  need(out, "out");
  if (world < 1 || rank < 0 || rank >= world)
    fail(HP_ECOMM, "rank " + std::to_string(rank) + " out of range for world_size " +
                       std::to_string(world));
  HP_CUDA(cudaSetDevice(device));
  auto* c = new hp_comm;
  c->world = world;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    fail(HP_ECOMM, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  HP_API_END
}

hp_status hp_comm_destroy(hp_comm* c) {
  HP_API_BEGIN
  if (c) {
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->pg_buf) cudaFree(c->pg_buf);
    if (c->pg_stream) cudaStreamDestroy(c->pg_stream);
    delete c;
  }
  HP_API_END
}

hp_status hp_engine_create(const hp_model_desc* m, const hp_optim_desc* o, const hp_exec_desc* x,
                           hp_comm* comm, hp_engine** out) {
  HP_API_BEGIN
  need(m, "model");
  need(o, "optim");
  need(x, "exec");
  need(out, "out");
  auto* h = new hp_engine;
  try {
    h->e = new hp::Engine(*m, *o, *x, comm);
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  HP_API_END
}

hp_status hp_engine_destroy(hp_engine* e) {
  HP_API_BEGIN
  if (e) {
    delete e->e;
    delete e;
  }
  HP_API_END
}

#define ENG(e)           \
  need(e, "engine");     \
  hp::Engine& E = *(e)->e

hp_status hp_engine_set_params(hp_engine* e, const void* flat, uint64_t n, int dtype) {
  HP_API_BEGIN
  ENG(e);
  need(flat, "flat");
  E.set_params(flat, n, dtype);
  HP_API_END
}
hp_status hp_engine_get_params(hp_engine* e, void* flat, uint64_t n, int dtype) {
  HP_API_BEGIN
  ENG(e);
  need(flat, "flat");
  E.get_params(flat, n, dtype);
  HP_API_END
}
hp_status hp_engine_broadcast_params(hp_engine* e, int root) {
  HP_API_BEGIN
  ENG(e);
  E.broadcast_params(root);
  HP_API_END
}
hp_status hp_engine_get_adam(hp_engine* e, float* m, float* v, uint64_t* t) {
  HP_API_BEGIN
  ENG(e);
  E.get_adam(m, v, t);
  HP_API_END
}
hp_status hp_engine_set_adam(hp_engine* e, const float* m, const float* v, uint64_t t) {
  HP_API_BEGIN
  ENG(e);
  E.set_adam(m, v, t);
  HP_API_END
}
hp_status hp_engine_set_capture(hp_engine* e, int on) {
  HP_API_BEGIN
  ENG(e);
  E.set_capture(on != 0);
  HP_API_END
}
hp_status hp_engine_forward(hp_engine* e, double* loss_sum, double* weight) {
  HP_API_BEGIN
  ENG(e);
  if (!loss_sum || !weight) hp::fail(HP_ECONFIG, "hp_engine_forward: null output");
  E.forward_only(loss_sum, weight);
  HP_API_END
}
hp_status hp_engine_set_digest_check(hp_engine* e, uint64_t every, int debug) {
  HP_API_BEGIN
  ENG(e);
  E.set_digest_check(every, debug != 0);
  HP_API_END
}
hp_status hp_engine_set_grad_comm(hp_engine* e, int on) {
  HP_API_BEGIN
  ENG(e);
  E.set_grad_comm(on != 0);
  HP_API_END
}
hp_status hp_engine_get_local_grads(hp_engine* e, float* flat, uint64_t n) {
  HP_API_BEGIN
  ENG(e);
  E.get_local_grads(flat, n);
  HP_API_END
}
hp_status hp_engine_stage_batch(hp_engine* e, const hp_batch* b) {
  HP_API_BEGIN
  ENG(e);
  need(b, "batch");
  E.stage_batch(*b);
  HP_API_END
}
hp_status hp_engine_round_async(hp_engine* e, int dummy, double lr) {
  HP_API_BEGIN
  ENG(e);
  E.round_async(dummy, lr);
  HP_API_END
}
hp_status hp_engine_round_sync(hp_engine* e, hp_round_out* out) {
  HP_API_BEGIN
  ENG(e);
  E.round_sync(out);
  HP_API_END
}
hp_status hp_engine_round(hp_engine* e, int dummy, double lr, hp_round_out* out) {
  HP_API_BEGIN
  ENG(e);
  E.round_async(dummy, lr);
  E.round_sync(out);
  HP_API_END
}
hp_status hp_engine_params_digest(hp_engine* e, uint64_t* digest) {
  HP_API_BEGIN
  ENG(e);
  *digest = E.digest();
  HP_API_END
}
hp_status hp_engine_kernel_launches(hp_engine* e, uint64_t* n) {
  HP_API_BEGIN
  (void)e;
  *n = hp::kernel_launch_count();
  HP_API_END
}
hp_status hp_engine_timers(hp_engine* e, int enable) {
  HP_API_BEGIN
  ENG(e);
  E.timers(enable != 0);
  HP_API_END
}
hp_status hp_engine_timer_read(hp_engine* e, int which, char* name, uint64_t cap, double* ms,
                               uint64_t* launches, double* bytes, double* flops) {
  HP_API_BEGIN
  ENG(e);
  std::string nm;
  E.timer_read(which, &nm, ms, launches, bytes, flops);
  if (name && cap) {
    std::strncpy(name, nm.c_str(), cap - 1);
    name[cap - 1] = 0;
  }
  HP_API_END
}
hp_status hp_engine_class_replay(hp_engine* e, int which, int iters, double* ms, double* flops,
                                 uint64_t* launches) {
  HP_API_BEGIN
  ENG(e);
  need(ms, "ms");
  need(flops, "flops");
  need(launches, "launches");
  if (which < 0 || which >= hp::TM_COUNT) fail(HP_EINDEX, "timer class out of range");
  E.class_replay(which, iters, ms, flops, launches);
  HP_API_END
}
hp_status hp_engine_step_count(hp_engine* e, uint64_t* step) {
  HP_API_BEGIN
  ENG(e);
  *step = E.step();
  HP_API_END
}

hp_status hp_engine_set_step(hp_engine* e, uint64_t step) {
  HP_API_BEGIN
  ENG(e);
  E.set_step(step);
  HP_API_END
}

hp_status hp_engine_pending_rounds(hp_engine* e, uint64_t* n) {
  HP_API_BEGIN
  ENG(e);
  need(n, "n");
  *n = E.pending_rounds();
  HP_API_END
}

hp_status hp_engine_mark(hp_engine* e, int slot) {
  HP_API_BEGIN
  ENG(e);
  E.mark(slot);
  HP_API_END
}
hp_status hp_engine_elapsed(hp_engine* e, int a, int b, double* ms) {
  HP_API_BEGIN
  ENG(e);
  need(ms, "ms");
  *ms = E.elapsed(a, b);
  HP_API_END
}
hp_status hp_engine_synchronize(hp_engine* e) {
  HP_API_BEGIN
  ENG(e);
  E.synchronize();
  HP_API_END
}

hp_status hp_engine_io_bytes(hp_engine* e, uint64_t* h2d, uint64_t* d2h) {
  HP_API_BEGIN
  ENG(e);
  if (h2d) *h2d = E.stage_bytes();
  if (d2h) *d2h = E.readback_bytes();
  HP_API_END
}

namespace {
cudaStream_t g_debug_stream = nullptr;  // hp_debug_gemm's stream (0: legacy default)
}
hp_status hp_debug_set_stream(void* stream) {
  HP_API_BEGIN
  g_debug_stream = static_cast<cudaStream_t>(stream);
  HP_API_END
}

hp_status hp_debug_gemm(int M, int N, int K, int ab_bf16, const void* A, int64_t lda, int a_trans,
                        const void* B, int64_t ldb, int b_trans, int64_t b_group, int64_t b_gstride,
                        void* C, int64_t ldc, int c_bf16, int64_t c_group, int64_t c_gstride,
                        const float* bias, int act, void* aux, const void* resid, int64_t ld_resid,
                        int accumulate, int path, int bn) {
  HP_API_BEGIN
  hp::GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.ab = ab_bf16 ? hp::DType::bf16 : hp::DType::f32;
  g.a = hp::Operand{A, lda, a_trans, 0, 0};
  g.b = hp::Operand{B, ldb, b_trans, b_group, b_gstride};
  g.c = C; g.ldc = ldc; g.c_group = c_group; g.c_gstride = c_gstride;
  g.ct = c_bf16 ? hp::DType::bf16 : hp::DType::f32;
  g.bias = bias; g.act = act; g.aux = aux; g.resid = resid; g.ld_resid = ld_resid;
  g.accumulate = accumulate;
  if (path == 1) {
    hp::gemm_simt(g, g_debug_stream);
  } else if (path == 2) {
    hp::gemm_tc_set_bn(bn % 1000);
    hp::gemm_tc_set_cg((bn / 1000) % 10);
    hp::gemm_tc_set_splits((bn / 10000) % 10);
    hp::gemm_tc_set_debug(bn / 100000);
    hp::gemm_tc(g, g_debug_stream);
    hp::gemm_tc_set_debug(0);
    hp::gemm_tc_set_bn(0);
    hp::gemm_tc_set_cg(0);
    hp::gemm_tc_set_splits(0);
  } else if (path == 4) {  // fp32 operands through the bf16x6 tensor-core split
    if (!hp::gemm_x6(g, g_debug_stream)) fail(HP_ECONFIG, "bf16x6: unsupported operand layout");
  } else {
    hp::gemm(g, g_debug_stream);
  }
  HP_API_END
}

hp_status hp_debug_adam(float* p, float* m, float* v, const float* g, uint64_t n, float lr,
                        float b1, float b2, float eps, float c1, float c2, int sgd, float wd) {
  HP_API_BEGIN
  unsigned long long* err = nullptr;
  HP_CUDA(cudaMalloc(&err, hp::kErrWords * 8));
  const unsigned long long e0[hp::kErrWords] = {0ull, ~0ull, ~0ull, ~0ull};
  HP_CUDA(cudaMemcpy(err, e0, sizeof(e0), cudaMemcpyHostToDevice));
  hp::AdamArgs a{};
  a.p = p; a.m = m; a.v = v; a.g = g; a.n = n;
  a.lr = lr; a.b1 = b1; a.b2 = b2; a.eps = eps; a.c1 = c1; a.c2 = c2;
  a.err = err; a.sgd = sgd; a.wd = wd;
  std::vector<uint64_t> items;
  for (uint64_t o = 0; o < n; o += 65536)
    items.insert(items.end(), {o, std::min<uint64_t>(65536, n - o), o, 1, 1});
  uint64_t* d_items = nullptr;
  HP_CUDA(cudaMalloc(&d_items, items.size() * 8 + 8));
  HP_CUDA(cudaMemcpy(d_items, items.data(), items.size() * 8, cudaMemcpyHostToDevice));
  a.items = d_items;
  a.nitems = static_cast<int>(items.size() / 5);
  hp::adam_update(a, 0);
  HP_CUDA(cudaDeviceSynchronize());
  unsigned long long h[hp::kErrWords];
  HP_CUDA(cudaMemcpy(h, err, sizeof(h), cudaMemcpyDeviceToHost));
  HP_CUDA(cudaFree(err));
  HP_CUDA(cudaFree(d_items));
  // the other elements are updated; the lowest offending index is reported
  if (h[2] != ~0ull) hp::fail(HP_ENUMERIC, "non-finite gradient at flat index " + std::to_string(h[2]));
  HP_API_END
}

hp_status hp_debug_layernorm(int T, int d, int bf16, const void* x, const float* g, const float* b,
                             void* y, float* mean, float* rstd, const void* dy, void* dx, float* dg,
                             float* db, float* dbias, int deferred) {
  HP_API_BEGIN
  const hp::DType t = bf16 ? hp::DType::bf16 : hp::DType::f32;
  hp::layernorm_fwd(T, d, x, t, g, b, y, t, mean, rstd, 0);
  if (dy) {
    const size_t fl = std::max(hp::colsum_scratch_floats(T, d), hp::colsum_part_floats(T, d));
    float* scratch = nullptr;
    HP_CUDA(cudaMalloc(&scratch, fl * 4));
    hp::DeferredFinal f;
    f.part = scratch;
    // deferred: the engine's form (partials now, the final launched separately)
    hp::layernorm_bwd(T, d, dy, t, x, t, mean, rstd, g, dx, t, dg, db, dbias, scratch, 0,
                      deferred ? &f : nullptr);
    if (deferred) hp::launch_final(f, 0);
    HP_CUDA(cudaDeviceSynchronize());
    HP_CUDA(cudaFree(scratch));
  }
  HP_CUDA(cudaDeviceSynchronize());
  HP_API_END
}

hp_status hp_debug_attention2(int B, const int* cu_q, const int* cu_kv, int T_q, int T_kv,
                              int max_q, int max_kv, int H, int dk, int bf16, const void* q,
                              int64_t ldq, int qcol, const void* k, int64_t ldk, int kcol,
                              const void* v, int64_t ldv, int vcol, void* o, float* lse,
                              const void* dO, void* dq, int64_t lddq, int dqcol, void* dkk,
                              int64_t lddk, int dkcol, void* dv, int64_t lddv, int dvcol,
                              int causal, int path) {
  HP_API_BEGIN
  hp::AttnArgs a;
  a.B = B; a.H = H; a.dk = dk;
  a.cu_q = cu_q; a.cu_kv = cu_kv; a.T_q = T_q; a.T_kv = T_kv; a.max_q = max_q; a.max_kv = max_kv;
  a.q = q; a.ldq = ldq; a.qcol = qcol;
  a.k = k; a.ldk = ldk; a.kcol = kcol;
  a.v = v; a.ldv = ldv; a.vcol = vcol;
  a.o = o; a.lse = lse; a.causal = causal;
  a.dO = dO;
  a.dq = dq; a.lddq = lddq; a.dqcol = dqcol;
  a.dk_ = dkk; a.lddk = lddk; a.dkcol = dkcol;
  a.dv = dv; a.lddv = lddv; a.dvcol = dvcol;
  const hp::DType t = bf16 ? hp::DType::bf16 : hp::DType::f32;
  if (path == 3 && !hp::attention2_tc_ok(a, t)) fail(HP_ECONFIG, "tcgen05 attention: unsupported shape");
  if (path == 3 || (path == 0 && hp::attention2_tc_ok(a, t))) {
    hp::attention_tc_fwd(a, 0);
    if (dO) hp::attention_tc_bwd(a, 0);
  } else {
    hp::attention_simt_fwd(a, t, 0);
    if (dO) hp::attention_simt_bwd(a, t, 0);
  }
  HP_CUDA(cudaDeviceSynchronize());
  HP_API_END
}

hp_status hp_debug_attention(int B, const int* cu, int T, int H, int dk, int bf16,
                             const void* qkv, void* o, float* lse, const void* dO, void* dqkv,
                             int path) {
  HP_API_BEGIN
  hp::DevBatch b;
  b.B = B;
  b.T = T;
  b.cu = cu;
  const bool tcp = path == 3 || (path == 0 && bf16 && hp::attention_tc_supported(dk, 128));
  const bool mma = !tcp && (path == 2 || (path == 0 && bf16 && hp::attention_mma_supported(dk, 128)));
  if (tcp) {
    hp::attention_fwd_tc(b, H, qkv, o, lse, 0);
    if (dO) hp::attention_bwd_tc(b, H, qkv, o, dO, lse, dqkv, 0);
  } else if (mma) {
    hp::attention_fwd_mma(b, H, qkv, o, lse, 0);
    if (dO) hp::attention_bwd_mma(b, H, qkv, o, dO, lse, dqkv, 0);
  } else {
    const hp::DType t = bf16 ? hp::DType::bf16 : hp::DType::f32;
    hp::attention_fwd(b, H, dk, qkv, o, lse, t, 0);
    if (dO) hp::attention_bwd(b, H, dk, qkv, o, dO, lse, dqkv, t, 0);
  }
  HP_CUDA(cudaDeviceSynchronize());
  HP_API_END
}

hp_status hp_shards_open(const char* dir, hp_shards** out) {
  HP_API_BEGIN
  need(dir, "dir");
  need(out, "out");
  auto h = std::make_unique<hp_shards>();
  h->set = std::make_shared<const hp::ShardSet>(dir);
  *out = h.release();
  HP_API_END
}

hp_status hp_shards_info(hp_shards* s, uint64_t* total, uint64_t* nshards) {
  HP_API_BEGIN
  need(s, "shards");
  if (total) *total = s->set->total();
  if (nshards) *nshards = s->set->nshards();
  HP_API_END
}

hp_status hp_shards_token_lengths(hp_shards* s, uint32_t* out, uint64_t n) {
  HP_API_BEGIN
  need(s, "shards");
  need(out, "out");
  const auto& l = s->set->token_lengths();
  if (n != l.size()) fail(HP_ESHAPE, "token length table has " + std::to_string(l.size()) + " entries");
  std::memcpy(out, l.data(), 4 * n);
  HP_API_END
}

hp_status hp_shards_close(hp_shards* s) {
  HP_API_BEGIN
  delete s;
  HP_API_END
}

hp_status hp_mlm_write_shards(const char* dir, uint64_t n, uint64_t shards, const uint64_t* tok_off,
                              const int64_t* tokens, const int64_t* segments,
                              const uint64_t* mask_off, const int64_t* mask_pos,
                              const int64_t* mask_orig, const int64_t* label) {
  HP_API_BEGIN
  need(dir, "dir");
  need(tok_off, "tok_off");
  need(mask_off, "mask_off");
  hp::write_mlm_shards(dir, n, shards, tok_off, tokens, segments, mask_off, mask_pos, mask_orig, label);
  HP_API_END
}

hp_status hp_loader_create(hp_shards* s, const uint64_t* batch_order, const uint64_t* batch_sizes,
                           uint64_t nbatches, const uint64_t* sched_batch,
                           const uint8_t* sched_dummy, uint64_t nsched, uint64_t prefetch_depth,
                           hp_loader** out) {
  HP_API_BEGIN
  need(s, "shards");
  need(out, "out");
  std::vector<std::vector<uint64_t>> plan(nbatches);
  uint64_t at = 0;
  for (uint64_t b = 0; b < nbatches; ++b) {
    plan[b].assign(batch_order + at, batch_order + at + batch_sizes[b]);
    at += batch_sizes[b];
  }
  auto h = std::make_unique<hp_loader>();
  h->loader = std::make_unique<hp::ShardLoader>(
      s->set, std::move(plan), std::vector<uint64_t>(sched_batch, sched_batch + nsched),
      std::vector<uint8_t>(sched_dummy, sched_dummy + nsched), prefetch_depth);
  *out = h.release();
  HP_API_END
}

hp_status hp_loader_next(hp_loader* l, hp_loaded_batch* out, int* has) {
  HP_API_BEGIN
  need(l, "loader");
  need(out, "out");
  need(has, "has");
  *has = l->loader->next(l->cur) ? 1 : 0;
  if (*has) {
    const auto& c = l->cur.csr;
    out->batch_index = l->cur.batch_index;
    out->dummy = l->cur.dummy ? 1 : 0;
    out->batch = hp_batch{c.label.size(), c.tok_off.data(), c.tokens.data(), c.segments.data(),
                          c.mask_off.data(), c.mask_pos.data(), c.mask_orig.data(), c.label.data()};
  }
  HP_API_END
}

hp_status hp_loader_destroy(hp_loader* l) {
  HP_API_BEGIN
  delete l;
  HP_API_END
}

hp_status hp_checkpoint_write(const char* path, const hp_model_desc* m, const hp_ckpt_desc* c,
                              const float* params, const float* adam_m, const float* adam_v) {
  HP_API_BEGIN
  if (!path || !m || !c || !params) hp::fail(HP_ECONFIG, "hp_checkpoint_write: null argument");
  hp::write_file_atomic(path, hp::hck1_serialize(*m, *c, params, adam_m, adam_v));
  HP_API_END
}

hp_status hp_checkpoint_read(const char* path, hp_model_desc* m, hp_ckpt_desc* c, float* params,
                             float* adam_m, float* adam_v, uint64_t n) {
  HP_API_BEGIN
  if (!path) hp::fail(HP_ECONFIG, "hp_checkpoint_read: null path");
  hp::hck1_parse(hp::read_file(path), m, c, params, adam_m, adam_v, n);
  HP_API_END
}

hp_status hp_engine_save_checkpoint(hp_engine* e, const char* path, const hp_ckpt_desc* c) {
  HP_API_BEGIN
  if (!e || !path || !c) hp::fail(HP_ECONFIG, "hp_engine_save_checkpoint: null argument");
  e->e->save_checkpoint(path, *c);
  HP_API_END
}

hp_status hp_engine_load_checkpoint(hp_engine* e, const char* path, hp_ckpt_desc* c) {
  HP_API_BEGIN
  if (!e || !path) hp::fail(HP_ECONFIG, "hp_engine_load_checkpoint: null argument");
  e->e->load_checkpoint(path, c);
  HP_API_END
}

hp_status hp_resume_position(const uint32_t* lens, uint64_t n, uint64_t max_sentences,
                             uint64_t max_tokens, uint64_t seed, uint64_t world,
                             uint64_t update_freq, uint64_t step, uint64_t* epoch,
                             uint64_t* skip_rounds) {
  HP_API_BEGIN
  if (!lens || !epoch || !skip_rounds) hp::fail(HP_ECONFIG, "hp_resume_position: null argument");
  hp::resume_position(std::vector<uint32_t>(lens, lens + n), max_sentences, max_tokens, seed, world,
                      update_freq, step, epoch, skip_rounds);
  HP_API_END
}

hp_status hp_debug_sync(void) {
  HP_API_BEGIN
  HP_CUDA(cudaDeviceSynchronize());
  HP_API_END
}

hp_status hp_debug_gemm_trace(unsigned long long* buf) {
  HP_API_BEGIN
  hp::gemm_tc_set_trace(buf);
  hp::attention_tc_set_trace(buf ? buf + 1008 : nullptr);  // slots 1008.. (attention)
  HP_API_END
}

hp_status hp_debug_gemm_generic(int on) {
  HP_API_BEGIN
  hp::gemm_tc_set_generic(on);
  HP_API_END
}

}  // extern "C"
