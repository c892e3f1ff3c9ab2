// Launch wrappers for the sm_100a kernels of the DP step.  All take an
// explicit stream; none synchronizes.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace hp {

enum class DType : int { f32 = 0, bf16 = 1 };

// Strided operand of a GEMM (row-major everywhere).
//   A(m,k): trans=0 -> p[m*ld + k];  trans=1 -> p[k*ld + m]
//   B(k,n): trans=0 -> p[(n/g)*gs + k*ld + n%g];  trans=1 -> p[(k/g)*gs + n*ld + k%g]
//   C(m,n): p[(n/g)*gs + m*ld + n%g]
// g == 0 disables grouping.  Grouping describes the per-head projection
// matrices wq.0..wq.{h-1}, wk.*, wv.* which the canonical layout keeps as
// separate [d x dk] blocks (model.hpp:103-112).
struct Operand {
  const void* p = nullptr;
  int64_t ld = 0;
  int trans = 0;
  int64_t group = 0;
  int64_t gstride = 0;
};

// ACT_GELU: store pre-activation to aux, apply GELU.
// ACT_DGELU: multiply by GELU'(aux) (aux = saved pre-activation, read only).
enum Act { ACT_NONE = 0, ACT_GELU = 1, ACT_DGELU = 2 };

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  DType ab = DType::f32;  // A and B element type
  Operand a, b;
  void* c = nullptr;
  int64_t ldc = 0;
  int64_t c_group = 0, c_gstride = 0;
  DType ct = DType::f32;
  float alpha = 1.f;
  int accumulate = 0;          // C += result (f32 C only)
  const float* bias = nullptr; // [N], added before the activation
  int act = ACT_NONE;
  void* aux = nullptr;         // pre-activation (ct type), ld = ldc
  const void* resid = nullptr; // C = epi(...) + R(m,n), R of type ct
  int64_t ld_resid = 0;
  int max_splits = 0;          // split-K cap for the tcgen05 path (0: heuristic)
  // K-chunk partials (tcgen05 path, fp32 C, no epilogue): chunk s covers
  // K [s * part_kc, (s + 1) * part_kc) and is stored at c + s * part_stride;
  // one launch for all chunks (the bf16x6 split's RN partial sums)
  int part_chunks = 0, part_kc = 0;
  int64_t part_stride = 0;
  // > 0 (tcgen05 path, fp32 C): K in stints of rs_kc, each its own
  // accumulation chain, summed in order in fp32 on chip (128-wide tiles)
  int rs_kc = 0;
};

// Dispatch: tcgen05 for bf16 operands whose layout TMA can describe; fp32
// operands on the same tcgen05 kernel through the bf16x6 split (HP_F32_GEMM=simt:
// the fp32 SIMT kernel); SIMT otherwise.
int gemm(const GemmArgs& g, cudaStream_t s);  // 0 SIMT, 1 tcgen05 bf16, 2 tcgen05 bf16x6 (fp32)
// fp32 operands on the bf16 tensor cores, fp32-accurate (bf16x6 split, see
// kernels.cu); false when the split operands' layout is unsupported
bool gemm_x6(const GemmArgs& g, cudaStream_t s);
void gemm_simt(const GemmArgs& g, cudaStream_t s);
bool gemm_tc_supported(const GemmArgs& g);
void gemm_tc(const GemmArgs& g, cudaStream_t s);
void gemm_tc_force(int mode);  // test hook: 0 auto, 1 never tcgen05
void gemm_tc_set_bn(int bn);   // test hook: 0 heuristic, 128, 192 or 256
// SMs the persistent GEMM grids may use (0: all): at N > 1 the engine leaves
// some to the NCCL kernels of the concurrent gradient allreduce
void gemm_tc_set_sm_budget(int n);
void gemm_tc_set_splits(int s);  // test hook: 0 heuristic, else forced split-K
void gemm_tc_set_cg(int cg);     // test hook: 0 heuristic, 1 single CTA, 2 CTA pair
void gemm_tc_set_debug(int mode);  // profiling hook: bits 1 no loads, 2 no MMA, 4 no epilogue
void gemm_tc_set_trace(unsigned long long* buf);  // profiling hook: CTA 0 clock64 timeline
void gemm_tc_set_generic(int on);  // test hook: 1 forces the generic (all-flags) epilogue

// Device batch (one rank batch, SoA int32), see engine.cpp.
struct DevBatch {
  int T = 0, B = 0, M = 0;
  const int* tok = nullptr;     // [T]
  const int* seg = nullptr;     // [T]
  const int* pos = nullptr;     // [T] position within its instance
  const int* cu = nullptr;      // [B+1] instance token offsets
  const int* mrow = nullptr;    // [M] global token row of each masked position
  const int* morig = nullptr;   // [M] original token id (MLM target)
  const int* label = nullptr;   // [B] NSP label
  // distinct token ids for the embedding gradient: uid[u], its tokens
  // perm[useg[u] .. useg[u+1]) in position order; ulist = the u's with few
  // tokens (ucount[0] of them), then the hot ones (ucount[1])
  const int* perm = nullptr;    // [T]
  const int* uid = nullptr;     // [T]
  const int* useg = nullptr;    // [T+1]
  const int* ulist = nullptr;   // [T]
  const int* ucount = nullptr;  // [2]
};

// x[t] = E[tok] + seg_{s}[.] + PE[pos] ; optional LN afterwards is separate.
void embed_fwd(const DevBatch& b, int d, const void* E, const void* seg0,
               const void* seg1, DType wt, const float* pe, void* x, DType xt,
               cudaStream_t s);
// Row-sparse form of the word-embedding gradient for the N > 1 exchange:
// slot u of `rows` (stride d + 4 floats) = [distinct token id u as int bits,
// 3 pad, its d gradient values]; slots [U, cap) carry id -1.  Segment
// gradients as embed_bwd (skipped when dseg0 is null).
void embed_bwd_rows(const DevBatch& b, int d, const void* dx, DType xt, float* rows, int cap,
                    float* dseg0, float* dseg1, float* scratch, cudaStream_t s);
// dE[id] += scale * row for every slot of one rank's gathered row set (ids
// are distinct within a set; call once per rank, in rank order)
void embed_rows_scatter(const float* rows, int cap, int d, float* dE, cudaStream_t s,
                        float scale = 1.f);
// seq2seq: x[t] = scale * E[tok[t]] + PE[pos[t]]
void embed_scaled_fwd(int T, int d, const int* tok, const int* pos, const void* E, DType wt,
                      float scale, const float* pe, void* x, DType xt, cudaStream_t s);
// dE[id] = sum of dx over the tokens with that id (dE zeroed by the caller;
// deterministic, position order), dseg{0,1} = column sums over the segment's tokens.
void embed_bwd(const DevBatch& b, int d, const void* dx, DType xt, float* dE,
               float* dseg0, float* dseg1, float* scratch, cudaStream_t s);

// Deferred final of a column reduction (LayerNorm-backward dgamma/dbeta/dbias,
// bias column sums): when the caller passes one, the bf16 partial kernel writes
// its [chunks x N] partial rows into `part` (caller-owned, colsum_part_floats
// floats) and leaves the last, tiny reduction to launch_final() -- which the
// engine issues on its side stream, off the backward's critical path (the
// results are only read by the bucket's allreduce / update on that stream).
struct DeferredFinal {
  float* part = nullptr;  // in
  bool queued = false;    // out: launch_final() must run
  int kind = 0, chunks = 0, d = 0, stride = 0, n = 0;
  float *o0 = nullptr, *o1 = nullptr, *o2 = nullptr;
};
void launch_final(const DeferredFinal& f, cudaStream_t s);
size_t colsum_part_floats(int R, int N);

void layernorm_fwd(int T, int d, const void* x, DType xt, const float* g,
                   const float* bta, void* y, DType yt, float* mean, float* rstd,
                   cudaStream_t s);
// dx = LN'(dy); dg/db column sums written (not accumulated) to dg, db; when
// dbias is given it receives colsum(dx) (the bias gradient of the linear whose
// output, through the residual, fed this LayerNorm).
void layernorm_bwd(int T, int d, const void* dy, DType dyt, const void* x,
                   DType xt, const float* mean, const float* rstd, const float* g,
                   void* dx, DType dxt, float* dg, float* db, float* dbias, float* scratch,
                   cudaStream_t s, DeferredFinal* df = nullptr);
// scratch floats the column-sum kernels need for an R x N reduction
size_t colsum_scratch_floats(int R, int N);

// Varlen multi-head attention, self or cross, optionally causal (the
// seq2seq decoder): instance b's queries are rows [cu_q[b], cu_q[b+1]) of Q,
// its keys / values rows [cu_kv[b], cu_kv[b+1]) of K / V; head h reads the dk
// columns starting at col + h * dk of each operand (row pitch ld).  O is
// [T_q x H dk] (row pitch H dk, head h at columns h dk), lse [H x T_q].  The
// backward writes dQ / dK / dV with their own pitches and column offsets.
// causal: query i sees keys j <= i (positions within the instance).
struct AttnArgs {
  int B = 0, H = 0, dk = 0;
  const int* cu_q = nullptr;
  const int* cu_kv = nullptr;
  int T_q = 0, T_kv = 0;
  int max_q = 0, max_kv = 0;  // longest instance on each side
  const void* q = nullptr; int64_t ldq = 0; int qcol = 0;
  const void* k = nullptr; int64_t ldk = 0; int kcol = 0;
  const void* v = nullptr; int64_t ldv = 0; int vcol = 0;
  void* o = nullptr;
  float* lse = nullptr;
  int causal = 0;
  const void* dO = nullptr;  // backward
  void* dq = nullptr; int64_t lddq = 0; int dqcol = 0;
  void* dk_ = nullptr; int64_t lddk = 0; int dkcol = 0;
  void* dv = nullptr; int64_t lddv = 0; int dvcol = 0;
  // packing (tcgen05 kernels only): CTA b takes instances [grp[b], grp[b+1])
  // -- consecutive instances whose queries and keys each fit one 128-row
  // tile, block-diagonal mask -- for b < *ngrp; the grid stays B wide
  const int* grp = nullptr;
  const int* ngrp = nullptr;
};
// self-attention over packed QKV [T x 3d] (q heads | k heads | v heads)
AttnArgs self_attn_args(const DevBatch& b, int H, int dk, int max_seq, const void* qkv, void* o,
                        float* lse, const void* dO = nullptr, void* dqkv = nullptr, int causal = 0);
// dispatch: tcgen05 kernels for bf16, dk = 64, both sides <= 128 tokens;
// the SIMT kernels otherwise (fp32 parity path)
void attention2_fwd(const AttnArgs& a, DType t, cudaStream_t s);
void attention2_bwd(const AttnArgs& a, DType t, cudaStream_t s);
bool attention2_tc_ok(const AttnArgs& a, DType t);
void attention_simt_fwd(const AttnArgs& a, DType t, cudaStream_t s);
void attention_simt_bwd(const AttnArgs& a, DType t, cudaStream_t s);
void attention_tc_fwd(const AttnArgs& a, cudaStream_t s);
void attention_tc_bwd(const AttnArgs& a, cudaStream_t s);

// Varlen multi-head self-attention over packed QKV [T x 3d] (columns:
// q heads | k heads | v heads, dk each).  O [T x d], lse [H x T].
void attention_fwd(const DevBatch& b, int H, int dk, const void* qkv, void* o,
                   float* lse, DType t, cudaStream_t s);
void attention_bwd(const DevBatch& b, int H, int dk, const void* qkv,
                   const void* o, const void* dO, const float* lse, void* dqkv,
                   DType t, cudaStream_t s);

// Tensor-core (mma.sync bf16) attention for dk == 64, sequences <= 128.
bool attention_mma_supported(int dk, int max_seq);
void attention_fwd_mma(const DevBatch& b, int H, const void* qkv, void* o, float* lse,
                       cudaStream_t s);
void attention_bwd_mma(const DevBatch& b, int H, const void* qkv, const void* o, const void* dO,
                       const float* lse, void* dqkv, cudaStream_t s);

// tcgen05 attention (attn_tc.cu): dk == 64, sequences <= 128, bf16.
bool attention_tc_supported(int dk, int max_seq);
void attention_tc_set_trace(unsigned long long* buf);  // profiling: CTA (0,0) timeline
void attention_fwd_tc(const DevBatch& b, int H, const void* qkv, void* o, float* lse,
                      cudaStream_t s);
void attention_bwd_tc(const DevBatch& b, int H, const void* qkv, const void* o, const void* dO,
                      const float* lse, void* dqkv, cudaStream_t s);
// tcgen05 attention for 128 < seq <= 512 (attn_tc.cu, C4): 128-row query /
// key blocks; forward, then backward as a dK/dV kernel and a dQ kernel
bool attention_long_supported(int dk, int max_seq);
void attention_fwd_long(const DevBatch& b, int H, int max_seq, const void* qkv, void* o, float* lse,
                        cudaStream_t s);
void attention_bwd_long(const DevBatch& b, int H, int max_seq, const void* qkv, const void* o,
                        const void* dO, const float* lse, void* dqkv, cudaStream_t s);

// rows of src selected by idx -> dst (dst[r] = src[idx[r]]); idx < 0 marks a
// padding row (zeros here, skipped by the scatters, no loss in ls_ce).
void gather_rows(int R, int d, const int* idx, const void* src, void* dst, DType t,
                 cudaStream_t s);
// dst[idx[r]] = src[r] (rows unique), other rows untouched.
void scatter_rows(int R, int d, const int* idx, const void* src, void* dst,
                  DType t, cudaStream_t s);
// same with an fp32 source converted to the destination type
void scatter_rows_f32(int R, int d, const int* idx, const float* src, void* dst, DType t,
                      cudaStream_t s);

// Label-smoothed CE over logits [R x V] (ld), tape.hpp:180-209/302-321.
// Per-row losses -> row_loss[R]; dz = p - q - eps/V written to dz (ld_dz).
void ls_ce(int R, int V, const float* z, int64_t ldz, const int* target,
           float eps, float* row_loss, void* dz, DType dzt, int64_t ld_dz,
           cudaStream_t s);

// NSP head (model.hpp:381-388): h0 = H[cu[b]], z = h0 W + b, CE(eps=0);
// writes row losses, dW [d x 2], db [2] (overwrite), and dH[cu[b]] += dz W^T.
void nsp_head(const DevBatch& b, int d, const void* H, DType ht, const float* W,
              const float* bias, float* row_loss, float* dW, float* db, void* dH,
              int compute_grad, cudaStream_t s);

// Column sums of a [R x N] matrix into out[N] (overwrite).
void col_sum(int R, int N, const void* x, int64_t ld, DType t, float* out,
             float* scratch, cudaStream_t s, DeferredFinal* df = nullptr);

// out[0] += sum(a[0..na)) + sum(b[0..nb)) in double, deterministic order.
void loss_reduce(const float* a, int na, const float* b, int nb, double* out,
                 cudaStream_t s);

// Numeric-error state of the rounds issued since the last sync (sticky, so a
// pipelined round_async sequence reports its FIRST error):
//   err[0]  loss/weight flags (|= 1 non-finite aggregated loss, |= 2 weight <= 0)
//   err[1]  sequence number of the round that first set err[0]
//   err[2]  lowest flat index of a non-finite gradient
//   err[3]  lowest sequence number of a round with a non-finite gradient
// Reset to {0, ~0, ~0, ~0} by the engine before the first round after a sync.
// A round's sequence number travels in hyper[3] (uint32 bits).
constexpr int kErrWords = 4;
// lw = [loss, weight]: finalize after the allreduce; inv_w = 1/weight (f32)
// and the loss/weight checks of engine.hpp:134-137 into err.
void finalize_weight(const double* lw, float* inv_w, double* inv_w64, unsigned long long* err,
                     const float* hyper, cudaStream_t s);

// Adam (kernels_scalar.cpp:74-83) bit-exact in f32 on identical inputs:
//   g = grad * scale (scale from *inv_w64 when non-null, else 1)
// shadow: optional bf16 working copy written with the param table's padded
// layout (see engine.cpp), segs describe [offset, cols, shadow_off, pcols].
struct AdamArgs {
  float* p; float* m; float* v; const float* g; uint64_t n;
  float lr, b1, b2, eps, c1, c2;
  const float* hyper;     // device [lr, c1, c2]; overrides the scalars when non-null
  float* g2;              // K > 1: earlier rounds' gradient sums, added then zeroed (or null)
  const double* inv_w64;  // may be null
  // error state (see kErrWords; may be null): the update is skipped when this
  // or an earlier unsynced round failed a check; a non-finite f64 gradient
  // (optim.hpp:131-133) skips that element and records its flat index
  unsigned long long* err;
  int sgd;
  float wd;               // AdamW decoupled weight decay (0: Adam)
  void* shadow;
  // work items [nitems][5] = {flat_lo, count, shadow_lo, cols, pcols}; one
  // CTA per item (see Engine: contiguous runs merged, <= 64K elements each)
  const uint64_t* items; int nitems;
};
void adam_update(const AdamArgs& a, cudaStream_t s);
// word-embedding rows [V x d] at flat offset lo (shadow slo, row pitch pcols),
// split around nl sorted distinct-id lists (uids + l * stride, length
// ucnts[2 l] + ucnts[2 l + 1]): mode 0 = the rows in no list, zero gradient;
// mode 1 = the union's rows, each once
void adam_rows(const AdamArgs& a, int mode, const int* uids, const int* ucnts, int nl, int stride,
               int V, int d, uint64_t lo, uint64_t slo, uint64_t pcols, cudaStream_t s);
// K > 1 gradient accumulation (Accumulator, optim.hpp:154-202)
void accumulate_weight(const double* lw, double* acc, double* out, double* inv_w64, int final_round,
                       cudaStream_t s);
void accumulate_grad(float* acc, const float* g, uint64_t n, cudaStream_t s);

// bf16 shadow refresh from fp32 params (after set_params / broadcast).
void refresh_shadow(const float* p, void* shadow, const uint64_t* seg_table,
                    int nseg, uint64_t n, cudaStream_t s);
void fill_f32(float* p, uint64_t n, float v, cudaStream_t s);
// FNV-1a over bytes (params_digest) -- single-thread kernel, off the hot path.
void fnv1a(const uint8_t* p, uint64_t n, uint64_t* out, cudaStream_t s);
// parallel digest for the cross-rank cadence check: FNV-1a over the FNV-1a
// values of 64 KB blocks (scratch: fnv1a_chunked_scratch(n) u64); *bad =
// (d[0] != d[1]) as a double
void fnv1a_chunked(const void* p, uint64_t n, uint64_t* scratch, uint64_t* out, cudaStream_t s);
size_t fnv1a_chunked_scratch(uint64_t n);
void digest_mismatch(const uint64_t* d, double* bad, cudaStream_t s);

uint64_t kernel_launch_count();
void count_launch(int n = 1);

}  // namespace hp
