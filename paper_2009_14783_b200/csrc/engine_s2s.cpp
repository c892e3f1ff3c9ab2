// transformer_seq2seq on the device engine: the encoder-decoder Transformer
// of the paper's translation workload (timed at PAPER.md:434;
// BASELINE configs[2] "C3": 6 + 6 layers, d = 512, h = 8, f = 2048, one
// 32768-word table shared by both inputs and the output projection).  A repo
// extension -- the reference model zoo has no decoder (model.hpp:16) -- built
// from the same pieces as bert_encoder and checked against the numpy oracle
// (oracle/model_oracle.py, finite-difference pinned).
//
// A pair is one Instance: tokens = source (segment 0) then target (segment
// 1).  The encoder reads the source; the decoder reads [BOS] + target[:-1]
// (BOS = 2) and predicts target; the loss is the label-smoothed CE summed over
// every target token (tape.hpp:180-209), weight = target tokens ("tokens"
// policy) or pairs ("sentences").  Embeddings are scaled by sqrt(d) and get
// sinusoidal positions (attention.hpp:53-67); blocks are post-LN:
//   encoder  x1 = LN1(x + MHA(x) Wo + bo),  out = LN2(x1 + FFN(x1))
//   decoder  y1 = LN1(y + causal MHA(y) Wo + bo)
//            y2 = LN2(y1 + MHA(q = y1, kv = memory) Wco + cbo)
//            out = LN3(y2 + FFN(y2))
//   logits   Z = out E^T (tied, no bias)
// Device layout: source tokens [T_s x d] and decoder tokens [T_t x d] packed
// token-major like the encoder path; the cross-attention reads the decoder's
// queries and the memory's K | V columns of one grouped [T_s x 2d] GEMM
// output (ck.* then cv.*, canonical order); d(memory) accumulates over the
// decoder layers in place; the embedding gradient is dE = dZ^T out (the
// output projection) plus sqrt(d) times the input rows of both sides, summed
// per distinct id in a fixed order (embed_bwd_rows + embed_rows_scatter).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "engine.h"
#include "hp_common.h"

namespace hp {

namespace {
constexpr int kBos = 2;
}

void Engine::s2s_alloc() {
  const size_t T = x_.max_tokens, Bm = x_.max_batch;
  auto act = [&](size_t cols) { return dalloc(T * cols * asz_); };
  auto f32 = [&](size_t n) { return static_cast<float*>(dalloc(n * 4)); };
  layers_.resize(L_);
  dec_layers_.resize(L_);
  for (int side = 0; side < 2; ++side)
    for (int l = 0; l < L_; ++l) {
      Layer& y = side ? dec_layers_[l] : layers_[l];
      y.x = act(d_);
      y.qkv = act(3 * d_);
      y.o = act(d_);
      y.lse = f32(T * H_);
      y.p1 = act(d_);
      y.x1 = act(d_);
      y.u = act(F_);
      y.g = act(F_);
      y.p2 = act(d_);
      y.mean1 = f32(T);
      y.rstd1 = f32(T);
      y.mean2 = f32(T);
      y.rstd2 = f32(T);
      if (side) {
        y.qc = act(d_);
        y.kvc = act(2 * d_);
        y.oc = act(d_);
        y.lsec = f32(T * H_);
        y.x2 = act(d_);
        y.p3 = act(d_);
        y.mean3 = f32(T);
        y.rstd3 = f32(T);
      }
    }
  mem_ = act(d_);
  x_final_ = act(d_);
  z_ = f32(T * Vp_);
  dz_ = dalloc(T * Vp_ * asz_);
  HP_CUDA(cudaMemset(dz_, 0, T * Vp_ * asz_));
  row_loss_ = f32(T + Bm);
  dA_ = act(d_);
  dB_ = act(d_);
  dC_ = act(std::max(d_, F_));
  dU_ = act(F_);
  dqkv_ = act(3 * d_);
  dqc_ = act(d_);
  dkvc_ = act(2 * d_);
  dmem_ = act(d_);
  demb_ = act(d_);  // rows [0, T_s) source, [T_s, T_s + T_t) decoder inputs
  emb_cap_ = static_cast<int>(T);
  emb_rows_ = f32(T * (d_ + 4));
}

// The pair batch -> the staged block (layout: constructor, enc_ / dec_ /
// embp_ / tgt_), validation in the order of the encoder path's stage_batch.
void Engine::stage_s2s(const hp_batch& b, int* h, double* weight) {
  const uint64_t B = b.n_inst, Tm = x_.max_tokens, Bm = x_.max_batch;
  int *etok = h, *epos = h + Tm, *ecu = h + 2 * Tm;
  int *dtok = ecu + Bm + 1, *dpos = dtok + Tm, *dcu = dpos + Tm, *tgt = dcu + Bm + 1;
  int *perm = tgt + Tm, *uid = perm + Tm, *useg = uid + Tm, *ulist = useg + Tm + 1,
      *ucount = ulist + Tm, *grp = ucount + 2, *ngrp = grp + Bm + 1;
  uint64_t Ts = 0, Tt = 0;
  double w = 0.0;
  for (uint64_t i = 0; i < B; ++i) {
    const uint64_t t0 = b.tok_off[i], t1 = b.tok_off[i + 1];
    if (t1 == t0) fail(HP_ESHAPE, "seq2seq: empty pair");
    if (b.mask_off[i + 1] != b.mask_off[i])
      fail(HP_ECONFIG, "seq2seq: a translation pair carries no masked positions");
    uint64_t ns = 0;
    while (t0 + ns < t1 && b.segments[t0 + ns] == 0) ++ns;
    const uint64_t nt = t1 - t0 - ns;
    for (uint64_t t = t0 + ns; t < t1; ++t)
      if (b.segments[t] != 1) fail(HP_EINDEX, "seq2seq: segments must be 0 (source) then 1 (target)");
    if (ns == 0 || nt == 0) fail(HP_ESHAPE, "seq2seq: a pair needs a source and a target");
    if (ns > m_.max_seq || nt > m_.max_seq) fail(HP_ESHAPE, "seq2seq: sequence length exceeds max_seq");
    for (uint64_t t = t0; t < t1; ++t)
      if (b.tokens[t] < 0 || static_cast<uint64_t>(b.tokens[t]) >= m_.vocab)
        fail(HP_EINDEX, "gather_rows: row " + std::to_string(b.tokens[t]) + " outside [0," +
                            std::to_string(m_.vocab) + ")");
    ecu[i] = static_cast<int>(Ts);
    dcu[i] = static_cast<int>(Tt);
    for (uint64_t j = 0; j < ns; ++j) {
      etok[Ts + j] = static_cast<int>(b.tokens[t0 + j]);
      epos[Ts + j] = static_cast<int>(j);
    }
    for (uint64_t j = 0; j < nt; ++j) {
      dtok[Tt + j] = j == 0 ? kBos : static_cast<int>(b.tokens[t0 + ns + j - 1]);
      dpos[Tt + j] = static_cast<int>(j);
      tgt[Tt + j] = static_cast<int>(b.tokens[t0 + ns + j]);
    }
    Ts += ns;
    Tt += nt;
    w += x_.policy == HP_POLICY_SENTENCES ? 1.0 : static_cast<double>(nt);
  }
  ecu[B] = static_cast<int>(Ts);
  dcu[B] = static_cast<int>(Tt);
  // embedding-gradient plan over the input rows of both sides (demb_ rows:
  // source at [0, T_s), decoder inputs at [T_s, T_s + T_t)), grouped by id
  const uint64_t R = Ts + Tt;
  auto& order = sort_buf_;
  order.resize(R);
  for (uint64_t r = 0; r < Ts; ++r) order[r] = (static_cast<uint64_t>(etok[r]) << 32) | r;
  for (uint64_t r = 0; r < Tt; ++r) order[Ts + r] = (static_cast<uint64_t>(dtok[r]) << 32) | (Ts + r);
  std::sort(order.begin(), order.end());
  int U = 0;
  for (uint64_t k = 0; k < R; ++k) {
    const int id = static_cast<int>(order[k] >> 32);
    perm[k] = static_cast<int>(order[k] & 0xffffffffu);
    if (k == 0 || id != uid[U - 1]) {
      uid[U] = id;
      useg[U] = static_cast<int>(k);
      ++U;
    }
  }
  useg[U] = static_cast<int>(R);
  int ns = 0, nh = 0;
  for (int u = 0; u < U; ++u)
    if (useg[u + 1] - useg[u] <= kEmbHotTokens) ulist[ns++] = u;
  for (int u = 0; u < U; ++u)
    if (useg[u + 1] - useg[u] > kEmbHotTokens) ulist[ns + nh++] = u;
  ucount[0] = ns;
  ucount[1] = nh;
  // attention packing: greedy runs of consecutive pairs whose sources and
  // whose targets each total <= 128 tokens (one tile for all three kinds:
  // encoder self, decoder self, cross)
  int G = 0;
  for (uint64_t i = 0; i < B;) {
    grp[G++] = static_cast<int>(i);
    int src = ecu[i + 1] - ecu[i], dst = dcu[i + 1] - dcu[i];
    ++i;
    while (i < B && src + (ecu[i + 1] - ecu[i]) <= 128 && dst + (dcu[i + 1] - dcu[i]) <= 128) {
      src += ecu[i + 1] - ecu[i];
      dst += dcu[i + 1] - dcu[i];
      ++i;
    }
  }
  grp[G] = static_cast<int>(B);
  *ngrp = G;
  enc_.T = static_cast<int>(Ts);
  enc_.B = static_cast<int>(B);
  dec_.T = static_cast<int>(Tt);
  dec_.B = static_cast<int>(B);
  embp_.T = static_cast<int>(R);
  embp_.B = static_cast<int>(B);
  // graph key (T, B, M) and the loss rows (M)
  batch_.T = static_cast<int>(Ts);
  batch_.B = static_cast<int>(B);
  batch_.M = static_cast<int>(Tt);
  *weight = w;
}

// GEMM whose B operand is the grouped per-head [d x dk] blocks starting at
// parameter `first` (wq.*..wv.*, cq.*, ck.* cv.*): N = blocks x dk (b_trans 0)
// or the transposed use in the data gradient (K = blocks x dk, b_trans 1)
GemmArgs Engine::grouped_b(int first, int N, int K, const void* a, int64_t lda, int a_trans,
                           int b_trans) const {
  const int64_t gs = bf16_ ? static_cast<int64_t>(shadow_off_[first + 1] - shadow_off_[first])
                           : static_cast<int64_t>(table_[first + 1].offset - table_[first].offset);
  GemmArgs g;
  g.N = N;
  g.K = K;
  g.ab = at_;
  g.a = Operand{a, lda, a_trans, 0, 0};
  g.b = Operand{w(first), wld(first), b_trans, dk_, gs};
  return g;
}

void Engine::ln_fwd(int T, const void* x, int ig, void* y, float* mean, float* rstd) {
  tstart(TM_NORM);
  layernorm_fwd(T, d_, x, at_, pp(ig), pp(ig + 1), y, at_, mean, rstd, s_main_);
  tstop(TM_NORM, 0, (double)T * d_ * asz_ * 2);
}

void Engine::ln_bwd(int T, const void* dy, const void* x, const float* mean, const float* rstd, int ig,
                    void* dx, float* dbias) {
  tstart(TM_NORM);
  DeferredFinal f = final_slot(colsum_part_floats((int)x_.max_tokens, d_));
  layernorm_bwd(T, d_, dy, at_, x, at_, mean, rstd, pp(ig), dx, at_, gp(ig), gp(ig + 1), dbias,
                scratch_, s_main_, &f);
  issue_final(f);
  tstop(TM_NORM, 0, (double)T * d_ * asz_ * 3);
}

void Engine::attn_op_fwd(const AttnArgs& a0) {
  const DType t = at_;
  AttnArgs a = a0;
  if (attn_pack_) {
    a.grp = s2s_grp_;
    a.ngrp = s2s_ngrp_;
  }
  auto op = [a, t](cudaStream_t st) { attention2_fwd(a, t, st); };
  const double fl = 4.0 * a.H * a.dk * (double)a.T_q * (double)std::max(a.max_kv, 1);
  tstart(TM_ATTN);
  op(s_main_);
  tstop(TM_ATTN, fl, 0);
  record(TM_ATTN, fl, op);
}

void Engine::attn_op_bwd(const AttnArgs& a0) {
  const DType t = at_;
  AttnArgs a = a0;
  if (attn_pack_) {
    a.grp = s2s_grp_;
    a.ngrp = s2s_ngrp_;
  }
  auto op = [a, t](cudaStream_t st) { attention2_bwd(a, t, st); };
  const double fl = 8.0 * a.H * a.dk * (double)a.T_q * (double)std::max(a.max_kv, 1);
  tstart(TM_ATTN);
  op(s_main_);
  tstop(TM_ATTN, fl, 0);
  record(TM_ATTN, fl, op);
}

namespace {
GemmArgs plain(int M, int N, int K, DType ab, Operand a, Operand b, void* c, int64_t ldc, DType ct) {
  GemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.ab = ab;
  g.a = a;
  g.b = b;
  g.c = c;
  g.ldc = ldc;
  g.ct = ct;
  return g;
}
}  // namespace

void Engine::forward_s2s() {
  const int Ts = enc_.T, Tt = dec_.T, d = d_, F = F_, ms = static_cast<int>(m_.max_seq);
  const int per_enc = 3 * H_ + 10, per_dec = 6 * H_ + 14;
  tstart(TM_EMBED);
  embed_scaled_fwd(Ts, d, enc_.tok, enc_.pos, w(0), at_, emb_scale_, pe_, layers_[0].x, at_, s_main_);
  embed_scaled_fwd(Tt, d, dec_.tok, dec_.pos, w(0), at_, emb_scale_, pe_, dec_layers_[0].x, at_, s_main_);
  tstop(TM_EMBED, 0, (double)(Ts + Tt) * d * 2 * asz_);

  // shared block pieces: QKV projection + self-attention, output projection
  // + bias + residual -> LN, FFN -> LN
  auto self_block = [&](Layer& y, int iq, int T, const DevBatch& bt, int causal) {
    GemmArgs q = grouped_b(iq, 3 * d, d, y.x, d, 0, 0);
    q.M = T;
    q.c = y.qkv;
    q.ldc = 3 * d;
    q.ct = at_;
    gemm_t(q);
    attn_op_fwd(self_attn_args(bt, H_, dk_, ms, y.qkv, y.o, y.lse, nullptr, nullptr, causal));
    const int iwo = iq + 3 * H_;
    GemmArgs o = plain(T, d, d, at_, Operand{y.o, d, 0, 0, 0}, Operand{w(iwo), wld(iwo), 0, 0, 0},
                       y.p1, d, at_);
    o.bias = pp(iwo + 1);
    o.resid = y.x;
    o.ld_resid = d;
    gemm_t(o);
    ln_fwd(T, y.p1, iwo + 2, y.x1, y.mean1, y.rstd1);
  };
  auto ffn_block = [&](Layer& y, const void* x, int iw1, int T, void* p, int ig, void* out, float* mean,
                       float* rstd) {
    GemmArgs f1 = plain(T, F, d, at_, Operand{x, d, 0, 0, 0}, Operand{w(iw1), wld(iw1), 0, 0, 0}, y.g,
                        F, at_);
    f1.bias = pp(iw1 + 1);
    f1.act = ACT_GELU;
    f1.aux = y.u;
    gemm_t(f1);
    GemmArgs f2 = plain(T, d, F, at_, Operand{y.g, F, 0, 0, 0}, Operand{w(iw1 + 2), wld(iw1 + 2), 0, 0, 0},
                        p, d, at_);
    f2.bias = pp(iw1 + 3);
    f2.resid = x;
    f2.ld_resid = d;
    gemm_t(f2);
    ln_fwd(T, p, ig, out, mean, rstd);
  };

  for (int l = 0; l < L_; ++l) {  // encoder
    Layer& y = layers_[l];
    const int iq = 1 + l * per_enc, iwo = iq + 3 * H_;
    void* out = l + 1 < L_ ? layers_[l + 1].x : mem_;
    self_block(y, iq, Ts, enc_, 0);
    ffn_block(y, y.x1, iwo + 4, Ts, y.p2, iwo + 8, out, y.mean2, y.rstd2);
  }
  for (int l = 0; l < L_; ++l) {  // decoder
    Layer& y = dec_layers_[l];
    const int iq = 1 + L_ * per_enc + l * per_dec, iwo = iq + 3 * H_, icq = iwo + 4, ico = icq + 3 * H_;
    void* out = l + 1 < L_ ? dec_layers_[l + 1].x : x_final_;
    self_block(y, iq, Tt, dec_, 1);
    // cross-attention: Qc = Y1 Wcq, [Kc | Vc] = memory [Wck | Wcv]
    GemmArgs qc = grouped_b(icq, d, d, y.x1, d, 0, 0);
    qc.M = Tt;
    qc.c = y.qc;
    qc.ldc = d;
    qc.ct = at_;
    gemm_t(qc);
    GemmArgs kv = grouped_b(icq + H_, 2 * d, d, mem_, d, 0, 0);
    kv.M = Ts;
    kv.c = y.kvc;
    kv.ldc = 2 * d;
    kv.ct = at_;
    gemm_t(kv);
    AttnArgs a;
    a.B = dec_.B; a.H = H_; a.dk = dk_;
    a.cu_q = dec_.cu; a.cu_kv = enc_.cu; a.T_q = Tt; a.T_kv = Ts; a.max_q = ms; a.max_kv = ms;
    a.q = y.qc; a.ldq = d; a.qcol = 0;
    a.k = y.kvc; a.ldk = 2 * d; a.kcol = 0;
    a.v = y.kvc; a.ldv = 2 * d; a.vcol = d;
    a.o = y.oc; a.lse = y.lsec;
    attn_op_fwd(a);
    GemmArgs co = plain(Tt, d, d, at_, Operand{y.oc, d, 0, 0, 0}, Operand{w(ico), wld(ico), 0, 0, 0}, y.p2,
                        d, at_);
    co.bias = pp(ico + 1);
    co.resid = y.x1;
    co.ld_resid = d;
    gemm_t(co);
    ln_fwd(Tt, y.p2, ico + 2, y.x2, y.mean2, y.rstd2);
    ffn_block(y, y.x2, ico + 4, Tt, y.p3, ico + 8, out, y.mean3, y.rstd3);
  }
  // tied output projection Z = out E^T (fp32 logits), label-smoothed CE
  GemmArgs z = plain(Tt, V_, d, at_, Operand{x_final_, d, 0, 0, 0}, Operand{w(0), wld(0), 1, 0, 0}, z_,
                     Vp_, DType::f32);
  if (Tt > 0) gemm_t(z);
  tstart(TM_HEAD);
  ls_ce(Tt, V_, z_, Vp_, tgt_, static_cast<float>(m_.label_smooth_eps), row_loss_, dz_, at_, Vp_, s_main_);
  tstop(TM_HEAD, 0, (double)Tt * V_ * 8);
}

void Engine::backward_s2s() {
  const int Ts = enc_.T, Tt = dec_.T, d = d_, F = F_, ms = static_cast<int>(m_.max_seq);
  const int per_enc = 3 * H_ + 10, per_dec = 6 * H_ + 14;
  const DType f32 = DType::f32;
  auto wg = [&](int M, int N, int K, const void* a, int64_t lda, const void* b, int64_t ldb, int idx) {
    gemm_t(plain(M, N, K, at_, Operand{a, lda, 1, 0, 0}, Operand{b, ldb, 0, 0, 0}, gp(idx),
                 static_cast<int64_t>(table_[idx].cols), f32));
  };
  // grouped weight gradient into the per-head blocks starting at `first`
  auto wg_grouped = [&](int M, int N, int K, const void* a, const void* b, int64_t ldb, int first) {
    GemmArgs g = plain(M, N, K, at_, Operand{a, d, 1, 0, 0}, Operand{b, ldb, 0, 0, 0}, gp(first), dk_, f32);
    g.c_group = dk_;
    g.c_gstride = static_cast<int64_t>(table_[first + 1].offset - table_[first].offset);
    gemm_t(g);
  };
  // FFN block backward: dY (out of LN) -> d(input of the block) into dxo
  auto ffn_bwd = [&](Layer& y, int T, const void* dY, const void* p, const float* mean, const float* rstd,
                     int ig, const void* xin, int iw1, void* dxo) {
    ln_bwd(T, dY, p, mean, rstd, ig, dB_, gp(iw1 + 3));  // dP (+ d(ffn.b2))
    wg(F, d, T, y.g, F, dB_, d, iw1 + 2);
    GemmArgs du = plain(T, F, d, at_, Operand{dB_, d, 0, 0, 0}, Operand{w(iw1 + 2), wld(iw1 + 2), 1, 0, 0},
                        dU_, F, at_);
    du.act = ACT_DGELU;
    du.aux = y.u;
    gemm_t(du);
    wg(d, F, T, xin, d, dU_, F, iw1);
    tstart(TM_NORM);
    {
      DeferredFinal f = final_slot(colsum_part_floats((int)x_.max_tokens, F));
      col_sum(T, F, dU_, F, at_, gp(iw1 + 1), scratch_, s_main_, &f);
      issue_final(f);
    }
    tstop(TM_NORM, 0, 0);
    GemmArgs dx = plain(T, d, F, at_, Operand{dU_, F, 0, 0, 0}, Operand{w(iw1), wld(iw1), 1, 0, 0}, dxo, d,
                        at_);
    dx.resid = dB_;
    dx.ld_resid = d;
    gemm_t(dx);
  };
  // self-attention block backward: dY (out of LN1) -> d(block input) into dxo
  auto self_bwd = [&](Layer& y, int iq, int T, const DevBatch& bt, int causal, const void* dY, void* dxo) {
    const int iwo = iq + 3 * H_;
    ln_bwd(T, dY, y.p1, y.mean1, y.rstd1, iwo + 2, dB_, gp(iwo + 1));  // dP1 (+ d(bo))
    wg(d, d, T, y.o, d, dB_, d, iwo);
    gemm_t(plain(T, d, d, at_, Operand{dB_, d, 0, 0, 0}, Operand{w(iwo), wld(iwo), 1, 0, 0}, dC_, d, at_));
    attn_op_bwd(self_attn_args(bt, H_, dk_, ms, y.qkv, y.o, y.lse, dC_, dqkv_, causal));
    wg_grouped(d, 3 * d, T, y.x, dqkv_, 3 * d, iq);
    GemmArgs dx = grouped_b(iq, d, 3 * d, dqkv_, 3 * d, 0, 1);
    dx.M = T;
    dx.c = dxo;
    dx.ldc = d;
    dx.ct = at_;
    dx.resid = dB_;
    dx.ld_resid = d;
    gemm_t(dx);
  };

  // output projection: dE = dZ^T out (first writer of the embedding
  // gradient), d(out) = dZ E
  if (Tt > 0) {
    gemm_t(plain(V_, d, Tt, at_, Operand{dz_, Vp_, 1, 0, 0}, Operand{x_final_, d, 0, 0, 0}, gp(0), d, f32));
    gemm_t(plain(Tt, d, V_, at_, Operand{dz_, Vp_, 0, 0, 0}, Operand{w(0), wld(0), 0, 0, 0}, dA_, d, at_));
  } else {
    HP_CUDA(cudaMemsetAsync(gp(0), 0, sizeof(float) * table_[0].size(), s_main_));
  }
  char* const demb = static_cast<char*>(demb_);
  for (int l = L_ - 1; l >= 0; --l) {  // decoder
    Layer& y = dec_layers_[l];
    const int iq = 1 + L_ * per_enc + l * per_dec, iwo = iq + 3 * H_, icq = iwo + 4, ico = icq + 3 * H_;
    ffn_bwd(y, Tt, dA_, y.p3, y.mean3, y.rstd3, ico + 8, y.x2, ico + 4, dC_);  // dC_ = d(y2)
    // cross block
    ln_bwd(Tt, dC_, y.p2, y.mean2, y.rstd2, ico + 2, dB_, gp(ico + 1));  // dP2 (+ d(cbo))
    wg(d, d, Tt, y.oc, d, dB_, d, ico);
    gemm_t(plain(Tt, d, d, at_, Operand{dB_, d, 0, 0, 0}, Operand{w(ico), wld(ico), 1, 0, 0}, dC_, d, at_));
    AttnArgs a;
    a.B = dec_.B; a.H = H_; a.dk = dk_;
    a.cu_q = dec_.cu; a.cu_kv = enc_.cu; a.T_q = Tt; a.T_kv = Ts; a.max_q = ms; a.max_kv = ms;
    a.q = y.qc; a.ldq = d; a.qcol = 0;
    a.k = y.kvc; a.ldk = 2 * d; a.kcol = 0;
    a.v = y.kvc; a.ldv = 2 * d; a.vcol = d;
    a.o = y.oc; a.lse = y.lsec; a.dO = dC_;
    a.dq = dqc_; a.lddq = d; a.dqcol = 0;
    a.dk_ = dkvc_; a.lddk = 2 * d; a.dkcol = 0;
    a.dv = dkvc_; a.lddv = 2 * d; a.dvcol = d;
    attn_op_bwd(a);
    wg_grouped(d, d, Tt, y.x1, dqc_, d, icq);
    GemmArgs dx1 = grouped_b(icq, d, d, dqc_, d, 0, 1);  // d(y1) = dQc Wcq^T + dP2
    dx1.M = Tt;
    dx1.c = dA_;
    dx1.ldc = d;
    dx1.ct = at_;
    dx1.resid = dB_;
    dx1.ld_resid = d;
    gemm_t(dx1);
    wg_grouped(d, 2 * d, Ts, mem_, dkvc_, 2 * d, icq + H_);
    GemmArgs dm = grouped_b(icq + H_, d, 2 * d, dkvc_, 2 * d, 0, 1);  // d(memory) += dKVc Wckv^T
    dm.M = Ts;
    dm.c = dmem_;
    dm.ldc = d;
    dm.ct = at_;
    if (l + 1 < L_) {
      dm.resid = dmem_;  // in place: every element read then written by one thread
      dm.ld_resid = d;
    }
    gemm_t(dm);
    // self block (causal); layer 0's input gradient lands in the decoder rows of demb_
    self_bwd(y, iq, Tt, dec_, 1, dA_, l == 0 ? demb + (size_t)Ts * d * asz_ : dA_);
    grads_ready(iq);
  }
  const void* dY = dmem_;
  for (int l = L_ - 1; l >= 0; --l) {  // encoder
    Layer& y = layers_[l];
    const int iq = 1 + l * per_enc, iwo = iq + 3 * H_;
    ffn_bwd(y, Ts, dY, y.p2, y.mean2, y.rstd2, iwo + 8, y.x1, iwo + 4, dC_);  // dC_ = d(x1)
    self_bwd(y, iq, Ts, enc_, 0, dC_, l == 0 ? demb_ : dA_);
    dY = dA_;
    grads_ready(iq);
  }
  // input embeddings of both sides: per distinct id, rows summed in a fixed
  // order, then dE[id] += sqrt(d) * row
  tstart(TM_EMBED);
  embed_bwd_rows(embp_, d, demb_, at_, emb_rows_, emb_cap_, nullptr, nullptr, scratch_, s_main_);
  embed_rows_scatter(emb_rows_, emb_cap_, d, gp(0), s_main_, emb_scale_);
  tstop(TM_EMBED, 0, (double)(Ts + Tt) * d * (asz_ + 8));
  grads_ready(0);
}

}  // namespace hp
