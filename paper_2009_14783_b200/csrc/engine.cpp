// DeviceStepEngine: one rank's share of the data-parallel step on a B200.
//
// Reference protocol (include/hetpar/engine.hpp:125-165), per round:
//   forward -> allreduce [loss_sum, weight] BEFORE backward (engine.hpp:133)
//   -> backward -> allreduce of the flat gradient (engine.hpp:145)
//   -> divide by the total weight (engine.hpp:151) -> identical update.
// B200 mapping:
//   * forward/backward are sm_100a kernels on the main stream; activations and
//     the canonical flat parameter / gradient buffers live in HBM;
//   * the 16-byte [loss, weight] allreduce runs on the comm stream as soon as
//     the loss kernel retires -- it does not block backward (gradients are
//     unnormalized sums);
//   * gradient buckets (contiguous ranges of the canonical flat order, walked
//     from the end) are allreduced (plain ncclSum) on the comm
//     stream as soon as backward finishes their parameters;
//   * the update divides each reduced bucket by sum(weight) in f64 -- the
//     reference's order, all_reduce_sum then g /= weight (engine.hpp:145-151)
//     -- and runs Adam (bit-exact f32 kern::adam_update) on the fp32 master
//     copy, refreshing the bf16 working copy the tcgen05 GEMMs read.
#include <nvtx3/nvToolsExt.h>  // header-only NVTX ranges (nsys / ncu range filters)
#include "engine.h"

#include <cstdlib>

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>

#include "checkpoint.h"
#include "hp_common.h"

namespace hp {
namespace {
// host-side NVTX range for the phases of a round (eager and captured rounds
// show the phases; a replayed round shows as one "hp.round" range)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace


namespace {
uint64_t pad8(uint64_t v) { return (v + 7) & ~uint64_t(7); }
constexpr int kAttnMaxSeq = 128;
}  // namespace

void* Engine::dalloc(size_t bytes) {
  void* p = nullptr;
  HP_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
  allocs_.push_back(p);
  return p;
}

int Engine::pidx(const std::string& name) const {
  for (size_t i = 0; i < table_.size(); ++i)
    if (table_[i].name == name) return static_cast<int>(i);
  fail(HP_EINDEX, "no parameter named " + name);
}

std::string Engine::param_at(uint64_t flat_index) const {
  for (const ParamEntry& p : table_)
    if (flat_index >= p.offset && flat_index < p.offset + p.size()) return p.name;
  return "#" + std::to_string(flat_index);
}

const void* Engine::w(int idx) const {
  if (bf16_) return static_cast<const __nv_bfloat16*>(shadow_) + shadow_off_[idx];
  return params_ + table_[idx].offset;
}
int64_t Engine::wld(int idx) const {
  return bf16_ ? static_cast<int64_t>(shadow_ld_[idx]) : static_cast<int64_t>(table_[idx].cols);
}

Engine::Engine(const hp_model_desc& m, const hp_optim_desc& o, const hp_exec_desc& x,
               hp_comm* comm)
    : m_(m), o_(o), x_(x), comm_(comm) {
  table_ = param_table(m_);
  if (x_.update_freq == 0) fail(HP_ECONFIG, "update_freq must be >= 1");
  if (x_.max_tokens == 0 || x_.max_batch == 0)
    fail(HP_ECONFIG, "exec capacities max_tokens/max_batch must be > 0");
  if (m_.max_seq > static_cast<uint64_t>(kAttnMaxSeq) &&
      !(x_.compute == HP_COMPUTE_BF16 && m_.heads > 0 && m_.d_model / m_.heads == 64 &&
        m_.max_seq <= 512 && m_.arch != HP_ARCH_SEQ2SEQ))
    fail(HP_ECONFIG, "max_seq > 128 needs the bf16 path with d_model / heads == 64 (max 512)");
  if (o_.kind != HP_OPT_ADAM && o_.kind != HP_OPT_SGD && o_.kind != HP_OPT_ADAMW)
    fail(HP_ECONFIG, "unknown optimizer kind");
  if (o_.kind == HP_OPT_ADAMW && !(o_.weight_decay >= 0.0))
    fail(HP_ECONFIG, "AdamW weight_decay must be >= 0");
  if (x_.policy != HP_POLICY_SENTENCES && x_.policy != HP_POLICY_TOKENS)
    fail(HP_ECONFIG, "unknown weight policy");
  if (comm_ && comm_->device != x_.device)
    fail(HP_ECONFIG, "communicator device differs from the engine device");
  HP_CUDA(cudaSetDevice(x_.device));

  bf16_ = x_.compute == HP_COMPUTE_BF16;
  at_ = bf16_ ? DType::bf16 : DType::f32;
  asz_ = bf16_ ? 2 : 4;
  bert_ = m_.arch == HP_ARCH_BERT_ENCODER;
  s2s_ = m_.arch == HP_ARCH_SEQ2SEQ;
  if (s2s_) m_.with_nsp = 0;  // no NSP head
  emb_scale_ = s2s_ ? static_cast<float>(std::sqrt(static_cast<double>(m_.d_model))) : 1.f;
  d_ = static_cast<int>(m_.d_model);
  H_ = static_cast<int>(m_.heads);
  dk_ = d_ / H_;
  V_ = static_cast<int>(m_.vocab);
  Vp_ = static_cast<int>(pad8(m_.vocab));
  L_ = (bert_ || s2s_) ? static_cast<int>(m_.layers) : 1;
  F_ = (bert_ || s2s_) ? static_cast<int>(m_.d_ff) : 0;
  n_ = table_.back().offset + table_.back().size();
  buckets_ = bucket_plan(table_, x_.bucket_mb > 0 ? x_.bucket_mb : 25.0);

  // bf16 working-copy layout: every parameter 16-byte aligned, rows padded to
  // a multiple of 8 elements (TMA strides must be 16-byte multiples).
  shadow_off_.resize(table_.size());
  shadow_ld_.resize(table_.size());
  std::vector<uint64_t> seg;
  for (size_t i = 0; i < table_.size(); ++i) {
    shadow_off_[i] = pad8(n_shadow_);
    shadow_ld_[i] = pad8(table_[i].cols);
    n_shadow_ = shadow_off_[i] + table_[i].rows * shadow_ld_[i];
    seg.insert(seg.end(), {table_[i].offset, table_[i].cols, shadow_off_[i], shadow_ld_[i]});
  }
  nseg_ = static_cast<int>(table_.size());

  // compute stream at the highest priority: the side stream's collectives and
  // per-bucket updates fill in behind the backward GEMMs
  int prio_lo = 0, prio_hi = 0;
  HP_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  HP_CUDA(cudaStreamCreateWithPriority(&s_main_, cudaStreamNonBlocking, prio_hi));
  // (the NCCL buckets' stream at the compute stream's priority measured
  // neutral at N = 2 and 4, profiles/r01_ab_comm_prio.txt)
  HP_CUDA(cudaStreamCreateWithPriority(&s_comm_, cudaStreamNonBlocking, prio_lo));
  if (comm_) {
    // per-bucket updates on their own stream, so bucket k+1's allreduce
    // starts as soon as bucket k's finishes instead of behind k's update
    HP_CUDA(cudaStreamCreateWithPriority(&s_upd_, cudaStreamNonBlocking, prio_lo));
    HP_CUDA(cudaEventCreateWithFlags(&ev_upd_done_, cudaEventDisableTiming));
  }
  HP_CUDA(cudaEventCreateWithFlags(&ev_fwd_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&ev_comm_done_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming));
  ev_bucket_.resize(buckets_.size());
  for (auto& e : ev_bucket_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  {
    // row-sparse word-embedding exchange: worth it when every rank's rows
    // (max_tokens x (d + 4) floats, allgathered) are fewer bytes than the
    // dense ring allreduce moves (2 (W-1)/W V d)
    const char* e = std::getenv("HP_SPARSE_EMB");
    const Bucket& last = buckets_.back();
    const uint64_t W = comm_ ? static_cast<uint64_t>(comm_->world) : 1;
    // (HP_SPARSE_EMB=1 forces it whenever the engine has a communicator --
    // world 1 included, so one GPU runs the exchange's collectives)
    const bool forced = comm_ && e && std::string(e) == "1";
    // (seq2seq: the output projection makes the embedding gradient dense)
    sparse_emb_ = (forced || (W > 1 && !(e && std::string(e) == "0") &&
                              x_.max_tokens * (d_ + 4) * W < 2 * (W - 1) * m_.vocab * d_)) &&
                  last.first_param == 0 && last.last_param == 0 && d_ % 8 == 0 && !s2s_;
    if (sparse_emb_) {
      emb_cap_ = static_cast<int>(x_.max_tokens);
      emb_rows_ = static_cast<float*>(dalloc((size_t)emb_cap_ * (d_ + 4) * 4));
      emb_gath_ = static_cast<float*>(dalloc((size_t)W * emb_cap_ * (d_ + 4) * 4));
    }
  }
  {
    // At N > 1 the persistent GEMMs (one CTA per SM, ~200 KB of smem, 168
    // registers a thread) leave no SM to the NCCL kernels of the bucket
    // allreduces running beside backward: their grids stop at 140 SMs
    // (C2, N = 2: 13908 / 13879 vs 13632 / 13628 samples/s, exposed allreduce
    // 0.43 vs 0.46 ms; at N = 1 a cap only costs, 7305 vs 7579;
    // profiles/r02_ab_gemm_sm_budget.txt).  HP_GEMM_SMS overrides (0: all).
    // Forward has no bucket allreduce beside it (the previous round's last
    // update has joined the compute stream): its GEMMs take every SM
    // (HP_GEMM_SMS_FWD overrides).
    const char* e = std::getenv("HP_GEMM_SMS");
    sms_bwd_ = e ? std::atoi(e) : (comm_ && comm_->world > 1 ? 140 : 0);
    const char* f = std::getenv("HP_GEMM_SMS_FWD");
    sms_fwd_ = f ? std::atoi(f) : (e ? sms_bwd_ : 0);
    gemm_tc_set_sm_budget(sms_bwd_);
  }
  ev_reduced_.resize(buckets_.size());
  for (auto& e : ev_reduced_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  {
    const char* e = std::getenv("HP_WGRAD_STREAM");
    wg_on_ = bert_ && !(e && std::string(e) == "0");
  }
  if (bert_) {  // events exist whenever the call sites index them (stream or not)
    if (wg_on_) HP_CUDA(cudaStreamCreateWithPriority(&s_wg_, cudaStreamNonBlocking, prio_lo));
    auto mk = [](std::vector<cudaEvent_t>& v, size_t n) {
      v.resize(n);
      for (auto& e : v) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    };
    mk(ev_fork_, 4 * static_cast<size_t>(L_) + 1);
    mk(ev_w2_, L_);
    mk(ev_w1_, L_);
    mk(ev_wo_, L_);
    mk(ev_wq_, L_);
    mk(ev_wgb_, buckets_.size());
    HP_CUDA(cudaEventCreateWithFlags(&ev_wg_join_, cudaEventDisableTiming));
    HP_CUDA(cudaEventCreateWithFlags(&ev_emb_zero_, cudaEventDisableTiming));
    HP_CUDA(cudaEventCreateWithFlags(&ev_head_fork_, cudaEventDisableTiming));
  }

  params_ = static_cast<float*>(dalloc(n_ * 4));
  // (an ncclMemAlloc'd, communicator-registered gradient buffer measured no
  // gain, profiles/r01_ab_nccl_register.txt)
  grads_ = static_cast<float*>(dalloc(n_ * 4));
  adam_m_ = static_cast<float*>(dalloc(n_ * 4));
  adam_v_ = static_cast<float*>(dalloc(n_ * 4));
  HP_CUDA(cudaMemset(params_, 0, n_ * 4));
  HP_CUDA(cudaMemset(grads_, 0, n_ * 4));
  HP_CUDA(cudaMemset(adam_m_, 0, n_ * 4));
  HP_CUDA(cudaMemset(adam_v_, 0, n_ * 4));
  if (bf16_) {
    shadow_ = dalloc(n_shadow_ * 2);
    HP_CUDA(cudaMemset(shadow_, 0, n_shadow_ * 2));
  }
  seg_table_ = static_cast<uint64_t*>(dalloc(seg.size() * 8));
  HP_CUDA(cudaMemcpy(seg_table_, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice));
  {
    // Adam work items, per gradient bucket (each bucket is updated as soon as
    // its reduced gradient is final): runs of parameters whose working copy
    // is laid out contiguously are merged; every item is cut to <= 8K elements
    // so even one 25 MB bucket spreads over ~800 CTAs.
    constexpr uint64_t kChunk = 8192;
    std::vector<uint64_t> items;
    bucket_items_.clear();
    auto build_items = [&](size_t first_param, size_t last_param) {
      std::vector<std::array<uint64_t, 5>> runs;
      for (size_t i = first_param; i <= last_param; ++i) {
        const uint64_t lo = table_[i].offset, n = table_[i].size();
        const uint64_t slo = bf16_ ? shadow_off_[i] : lo;
        const uint64_t cols = table_[i].cols, pc = bf16_ ? shadow_ld_[i] : cols;
        if (cols == pc && !runs.empty() && runs.back()[3] == runs.back()[4] &&
            runs.back()[0] + runs.back()[1] == lo && runs.back()[2] + runs.back()[1] == slo) {
          runs.back()[1] += n;
        } else {
          runs.push_back({lo, n, slo, cols == pc ? 1 : cols, cols == pc ? 1 : pc});
        }
      }
      const int first = static_cast<int>(items.size() / 5);
      for (const auto& r : runs) {
        const bool contig = r[3] == r[4];
        const uint64_t step = contig ? kChunk : std::max<uint64_t>(1, kChunk / r[3]) * r[3];
        for (uint64_t o = 0; o < r[1]; o += step) {
          const uint64_t cnt = std::min(step, r[1] - o);
          const uint64_t srow = contig ? o : (o / r[3]) * r[4];
          items.insert(items.end(), {r[0] + o, cnt, r[2] + srow, r[3], r[4]});
        }
      }
      return std::make_pair(first, static_cast<int>(items.size() / 5) - first);
    };
    for (const Bucket& bk : buckets_) bucket_items_.push_back(build_items(bk.first_param, bk.last_param));
    // the last bucket without the word embedding (its rows go through
    // adam_rows around the round's ids when the update is split, see round_body)
    const Bucket& lb = buckets_.back();
    // opt-in (HP_EMB_SPLIT=1): bit-identical, measured neutral on C2 at N = 1
    // (profiles/r01_ab_emb_split.txt) -- the dense tail is not what bounds the step
    const char* es = std::getenv("HP_EMB_SPLIT");
    split_emb_ = es && std::string(es) == "1" && lb.first_param == 0 && !s2s_ &&
                 table_[0].rows == static_cast<uint64_t>(V_) && table_[0].cols == static_cast<uint64_t>(d_) &&
                 d_ % 4 == 0 && table_[0].offset % 4 == 0;
    if (split_emb_) {
      emb_rest_items_ = lb.last_param >= 1 ? build_items(1, lb.last_param) : std::make_pair(0, 0);
      // every rank's distinct-id list (W > 1: allgathered before backward) and
      // the zero count a dummy round contributes
      const int W = comm_ ? comm_->world : 1;
      uid_all_ = static_cast<int*>(dalloc(sizeof(int) * x_.max_tokens * W));
      ucnt_all_ = static_cast<int*>(dalloc(sizeof(int) * 2 * W));
      ucount_zero_ = static_cast<int*>(dalloc(sizeof(int) * 2));
      HP_CUDA(cudaMemset(ucount_zero_, 0, sizeof(int) * 2));
    }
    nitems_ = static_cast<int>(items.size() / 5);
    adam_items_ = static_cast<uint64_t*>(dalloc(items.size() * 8));
    HP_CUDA(cudaMemcpy(adam_items_, items.data(), items.size() * 8, cudaMemcpyHostToDevice));
  }

  // sinusoidal positions computed in double then cast (attention.hpp:53-67)
  {
    std::vector<float> pe(m_.max_seq * d_);
    for (uint64_t p = 0; p < m_.max_seq; ++p)
      for (int i = 0; 2 * i < d_; ++i) {
        const double ang = static_cast<double>(p) /
                           std::pow(10000.0, (2.0 * i) / static_cast<double>(d_));
        pe[p * d_ + 2 * i] = static_cast<float>(std::sin(ang));
        pe[p * d_ + 2 * i + 1] = static_cast<float>(std::cos(ang));
      }
    pe_ = static_cast<float*>(dalloc(pe.size() * 4));
    HP_CUDA(cudaMemcpy(pe_, pe.data(), pe.size() * 4, cudaMemcpyHostToDevice));
  }

  // masked positions are padded to a multiple of mpad_ (index -1 rows: no
  // loss, no gradient) so CUDA graphs keyed by the padded count get reused
  mpad_ = bf16_ ? 64 : 1;
  {
    const char* e = std::getenv("HP_GRAPHS");
    graphs_on_ = !(e && std::string(e) == "0");
    // attention: tcgen05 kernels when the shape allows (HP_ATTN=mma selects
    // the mma.sync kernels, for A/B comparisons)
    const char* a = std::getenv("HP_ATTN");
    attn_tc_ = bf16_ && attention_tc_supported(dk_, (int)m_.max_seq) && !(a && std::string(a) == "mma");
    attn_long_ = bf16_ && !attention_tc_supported(dk_, (int)m_.max_seq) &&
                 attention_long_supported(dk_, (int)m_.max_seq);
  }
  // staged batch block (fixed layout at capacity)
  const uint64_t Tm = x_.max_tokens, Bm = x_.max_batch,
                 Mm = (std::max<uint64_t>(x_.max_masks, 1) + mpad_ - 1) / mpad_ * mpad_;
  // (seq2seq layout: see stage_s2s)
  const size_t ints = std::max<size_t>(3 * Tm + (Bm + 1) + 2 * Mm + Bm + (4 * Tm + 3),
                                       9 * Tm + 3 * (Bm + 1) + 4);
  stage_bytes_ = ((ints * 4 + 7) & ~size_t(7)) + 8;
  for (int i = 0; i < kStageBufs; ++i) {
    HP_CUDA(cudaMallocHost(&h_stage_[i], stage_bytes_));
    std::memset(h_stage_[i], 0, stage_bytes_);
    HP_CUDA(cudaEventCreateWithFlags(&ev_stage_[i], cudaEventDisableTiming));
  }
  d_stage_ = dalloc(stage_bytes_);
  {
    int* base = static_cast<int*>(d_stage_);
    batch_.tok = base;
    batch_.seg = base + Tm;
    batch_.pos = base + 2 * Tm;
    batch_.cu = base + 3 * Tm;
    batch_.mrow = base + 3 * Tm + Bm + 1;
    batch_.morig = batch_.mrow + Mm;
    batch_.label = batch_.morig + Mm;
    batch_.perm = batch_.label + Bm;
    batch_.uid = batch_.perm + Tm;
    batch_.useg = batch_.uid + Tm;
    batch_.ulist = batch_.useg + Tm + 1;
    batch_.ucount = batch_.ulist + Tm;
    d_weight_ = reinterpret_cast<double*>(static_cast<char*>(d_stage_) + stage_bytes_ - 8);
    if (s2s_) {  // [enc tok, pos | cu | dec tok, pos | cu | targets | embedding plan]
      enc_.tok = base;
      enc_.pos = base + Tm;
      enc_.cu = base + 2 * Tm;
      dec_.tok = enc_.cu + Bm + 1;
      dec_.pos = dec_.tok + Tm;
      dec_.cu = dec_.pos + Tm;
      tgt_ = dec_.cu + Bm + 1;
      embp_.perm = tgt_ + Tm;
      embp_.uid = embp_.perm + Tm;
      embp_.useg = embp_.uid + Tm;
      embp_.ulist = embp_.useg + Tm + 1;
      embp_.ucount = embp_.ulist + Tm;
      s2s_grp_ = embp_.ucount + 2;
      s2s_ngrp_ = s2s_grp_ + Bm + 1;
      const char* e = std::getenv("HP_ATTN_PACK");  // A/B: 0 = one pair per CTA
      attn_pack_ = !(e && std::string(e) == "0");
    }
  }

  // activations
  const size_t T = Tm;
  if (s2s_) {
    s2s_alloc();
  } else {
  layers_.resize(L_);
  for (int l = 0; l < L_; ++l) {
    Layer& y = layers_[l];
    y.x = dalloc(T * d_ * asz_);
    y.qkv = dalloc(T * 3 * d_ * asz_);
    y.o = dalloc(T * d_ * asz_);
    y.lse = static_cast<float*>(dalloc(T * H_ * 4));
    if (bert_) {
      y.p1 = dalloc(T * d_ * asz_);
      y.x1 = dalloc(T * d_ * asz_);
      y.u = dalloc(T * F_ * asz_);
      y.g = dalloc(T * F_ * asz_);
      y.p2 = dalloc(T * d_ * asz_);
      y.mean1 = static_cast<float*>(dalloc(T * 4));
      y.rstd1 = static_cast<float*>(dalloc(T * 4));
      y.mean2 = static_cast<float*>(dalloc(T * 4));
      y.rstd2 = static_cast<float*>(dalloc(T * 4));
    }
  }
  x_final_ = dalloc(T * d_ * asz_);
  if (bert_) {
    p0_ = dalloc(T * d_ * asz_);
    mean0_ = static_cast<float*>(dalloc(T * 4));
    rstd0_ = static_cast<float*>(dalloc(T * 4));
  }
  hm_ = dalloc(Mm * d_ * asz_);
  dhm_ = dalloc(Mm * d_ * 4);  // fp32: the vocab-long dgrad runs split-K
  z_ = static_cast<float*>(dalloc(Mm * Vp_ * 4));
  dz_ = dalloc(Mm * Vp_ * asz_);
  HP_CUDA(cudaMemset(dz_, 0, Mm * Vp_ * asz_));
  row_loss_ = static_cast<float*>(dalloc((Mm + Bm) * 4));
  dA_ = dalloc(T * d_ * asz_);
  dB_ = dalloc(T * d_ * asz_);
  dC_ = dalloc(T * std::max<size_t>(d_, F_) * asz_);
  dU_ = bert_ ? dalloc(T * F_ * asz_) : nullptr;
  dqkv_ = dalloc(T * 3 * d_ * asz_);
  if (bert_) {
    // per-layer-parity gradient buffers (layer l uses slot l & 1): a buffer a
    // weight-gradient GEMM reads is rewritten two layers later, so the
    // data-gradient chain does not wait on the weight-gradient stream
    rd_ = 2;
    pbuf_[0] = dB_;
    for (int i = 1; i < 4; ++i) pbuf_[i] = dalloc(T * d_ * asz_);
    ubuf_[0] = dU_;
    ubuf_[1] = dalloc(T * F_ * asz_);
    qbuf_[0] = dqkv_;
    qbuf_[1] = dalloc(T * 3 * d_ * asz_);
  }
  }  // !s2s_
  const size_t wmax = std::max<size_t>(d_, F_);
  const size_t scratch = std::max({colsum_scratch_floats((int)T, (int)wmax),
                                   colsum_scratch_floats((int)(s2s_ ? T : Mm), Vp_),
                                   colsum_scratch_floats((int)T, d_)});
  scratch_ = static_cast<float*>(dalloc(scratch * 4));
  if (wg_on_) scratch_wg_ = static_cast<float*>(dalloc(colsum_scratch_floats((int)T, F_) * 4));
  // [round loss, round weight, local loss, local weight, K-total loss, K-total weight]
  d_lw_ = static_cast<double*>(dalloc(8 * 8));  // [0,6): round scalars, [6]: forward_only
  HP_CUDA(cudaMemset(d_lw_, 0, 6 * 8));
  if (x_.update_freq > 1) {
    acc_grads_ = static_cast<float*>(dalloc(n_ * 4));
    HP_CUDA(cudaMemset(acc_grads_, 0, n_ * 4));
    d_acc_lw_ = static_cast<double*>(dalloc(2 * 8));
    HP_CUDA(cudaMemset(d_acc_lw_, 0, 2 * 8));
  }
  inv_w_ = static_cast<float*>(dalloc(4));
  inv_w64_ = static_cast<double*>(dalloc(8));
  err_ = static_cast<unsigned long long*>(dalloc(kErrWords * 8));
  d_hyper_ = static_cast<float*>(dalloc(4 * 4));
  HP_CUDA(cudaMallocHost(&h_lw_, 6 * 8));
  HP_CUDA(cudaMallocHost(&h_err_, kErrWords * 8));

  if (comm_) {
    // gradient buckets reduce with plain ncclSum (NVLS-eligible: the NVSwitch
    // does the reduction and NCCL needs few SMs); the 1/total-weight scale is
    // applied in f64 inside the update, the reference's own order
    // (all_reduce_sum, then g /= weight; engine.hpp:145-151)
  }
  HP_CUDA(cudaDeviceSynchronize());
}

Engine::~Engine() {
  if (s_main_) cudaStreamSynchronize(s_main_);
  if (s_comm_) cudaStreamSynchronize(s_comm_);
  if (s_upd_) cudaStreamSynchronize(s_upd_);
  for (auto& kv : graphs_) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto& gt : kv.second.timers)
      for (auto& pr : gt.ev) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
  }
  for (auto& t : tm_)
    for (auto& pr : t.ev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  for (void* p : allocs_) cudaFree(p);
  for (int i = 0; i < kStageBufs; ++i) {
    if (h_stage_[i]) cudaFreeHost(h_stage_[i]);
    if (ev_stage_[i]) cudaEventDestroy(ev_stage_[i]);
  }
  if (h_lw_) cudaFreeHost(h_lw_);
  if (h_err_) cudaFreeHost(h_err_);
  if (h_params_) cudaFreeHost(h_params_);
  for (auto& e : ev_bucket_) cudaEventDestroy(e);
  if (ev_ser_) cudaEventDestroy(ev_ser_);
  for (auto& e : final_evs_) cudaEventDestroy(e);
  for (auto* v : {&ev_fork_, &ev_w2_, &ev_w1_, &ev_wo_, &ev_wq_, &ev_wgb_})
    for (auto& e : *v) cudaEventDestroy(e);
  if (ev_wg_join_) cudaEventDestroy(ev_wg_join_);
  if (ev_emb_zero_) cudaEventDestroy(ev_emb_zero_);
  if (ev_head_fork_) cudaEventDestroy(ev_head_fork_);
  if (s_wg_) cudaStreamDestroy(s_wg_);
  for (auto& e : marks_)
    if (e) cudaEventDestroy(e);
  if (ev_fwd_) cudaEventDestroy(ev_fwd_);
  if (ev_comm_done_) cudaEventDestroy(ev_comm_done_);
  if (ev_done_) cudaEventDestroy(ev_done_);
  if (s_main_) cudaStreamDestroy(s_main_);
  if (s_comm_) cudaStreamDestroy(s_comm_);
  if (s_upd_) cudaStreamDestroy(s_upd_);
  if (ev_upd_done_) cudaEventDestroy(ev_upd_done_);
  for (auto& e : ev_reduced_) cudaEventDestroy(e);
}

// ------------------------------------------------------------------ state I/O
void Engine::set_params(const void* flat, uint64_t n, int dtype) {
  if (n != n_)
    fail(HP_EIO, "state dict payload has " + std::to_string(n) + " values, expected " +
                     std::to_string(n_));
  std::vector<float> tmp(n_);
  if (dtype == 1) {
    const double* s = static_cast<const double*>(flat);
    for (uint64_t i = 0; i < n_; ++i) tmp[i] = static_cast<float>(s[i]);
  } else {
    std::memcpy(tmp.data(), flat, n_ * 4);
  }
  HP_CUDA(cudaMemcpyAsync(params_, tmp.data(), n_ * 4, cudaMemcpyHostToDevice, s_main_));
  if (bf16_) refresh_shadow(params_, shadow_, seg_table_, nseg_, n_, s_main_);
  HP_CUDA(cudaStreamSynchronize(s_main_));
}

void Engine::get_params(void* flat, uint64_t n, int dtype) {
  if (n != n_) fail(HP_ESHAPE, "get_params: wrong element count");
  std::vector<float> tmp(n_);
  HP_CUDA(cudaMemcpyAsync(tmp.data(), params_, n_ * 4, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaStreamSynchronize(s_main_));
  if (dtype == 1) {
    double* d = static_cast<double*>(flat);
    for (uint64_t i = 0; i < n_; ++i) d[i] = tmp[i];
  } else {
    std::memcpy(flat, tmp.data(), n_ * 4);
  }
}

void Engine::broadcast_params(int root) {
  if (comm_) {
    HP_NCCL(ncclBroadcast(params_, params_, n_, ncclFloat, root, comm_->nccl, s_main_));
    if (bf16_) refresh_shadow(params_, shadow_, seg_table_, nseg_, n_, s_main_);
  }
  HP_CUDA(cudaStreamSynchronize(s_main_));
}

void Engine::set_step(uint64_t s) {
  if (in_flight_ || acc_count_ != 0) fail(HP_ECONFIG, "set_step inside a round or an update group");
  step_ = s;
}

void Engine::get_adam(float* m, float* v, uint64_t* t) {
  HP_CUDA(cudaMemcpyAsync(m, adam_m_, n_ * 4, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaMemcpyAsync(v, adam_v_, n_ * 4, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaStreamSynchronize(s_main_));
  *t = adam_t_;
}

void Engine::set_adam(const float* m, const float* v, uint64_t t) {
  HP_CUDA(cudaMemcpyAsync(adam_m_, m, n_ * 4, cudaMemcpyHostToDevice, s_main_));
  HP_CUDA(cudaMemcpyAsync(adam_v_, v, n_ * 4, cudaMemcpyHostToDevice, s_main_));
  HP_CUDA(cudaStreamSynchronize(s_main_));
  adam_t_ = t;
}

// ------------------------------------------------------------------ HCK1
// save_checkpoint / load_checkpoint (checkpoint.cpp:165-302) from / into the
// device state; the byte format lives in checkpoint.cpp.
void Engine::save_checkpoint(const std::string& path, const hp_ckpt_desc& c) {
  if (in_flight_) fail(HP_ECONFIG, "save_checkpoint while a round is in flight");
  // inside a partially accumulated update group (K > 1) the file holds the
  // state of the last update, as the reference's does (TrainState has no
  // accumulator, checkpoint.cpp:165-212); the pending rounds stay pending
  std::vector<float> p(n_), m(n_), v(n_);
  synchronize();
  HP_CUDA(cudaMemcpy(p.data(), params_, n_ * 4, cudaMemcpyDeviceToHost));
  HP_CUDA(cudaMemcpy(m.data(), adam_m_, n_ * 4, cudaMemcpyDeviceToHost));
  HP_CUDA(cudaMemcpy(v.data(), adam_v_, n_ * 4, cudaMemcpyDeviceToHost));
  hp_ckpt_desc d = c;
  d.step = step_;
  d.opt_kind = o_.kind;
  d.beta1 = o_.beta1;
  d.beta2 = o_.beta2;
  d.eps = o_.eps;
  d.weight_decay = o_.kind == HP_OPT_ADAMW ? o_.weight_decay : 0.0;
  d.opt_t = adam_t_;
  write_file_atomic(path, hck1_serialize(m_, d, p.data(), m.data(), v.data()));
}

void Engine::load_checkpoint(const std::string& path, hp_ckpt_desc* out) {
  if (in_flight_) fail(HP_ECONFIG, "load_checkpoint while a round is in flight");
  hp_model_desc md{};
  hp_ckpt_desc d{};
  std::vector<float> p(n_), m(n_), v(n_);
  hck1_parse(read_file(path), &md, &d, nullptr, nullptr, nullptr, 0);  // metadata first
  const auto ft = param_table(md);
  if (md.arch != m_.arch || ft.size() != table_.size() ||
      md.label_smooth_eps != m_.label_smooth_eps || md.with_nsp != m_.with_nsp)
    fail(HP_ECONFIG, "resume model spec does not match the checkpoint");
  for (size_t i = 0; i < ft.size(); ++i)
    if (ft[i].name != table_[i].name || ft[i].rows != table_[i].rows || ft[i].cols != table_[i].cols)
      fail(HP_ECONFIG, "resume model spec does not match the checkpoint");
  // the optimizer and the weight policy come from the file, as
  // load_checkpoint's TrainState does (checkpoint.cpp:254, 282-289)
  if (d.opt_kind != HP_OPT_ADAM && d.opt_kind != HP_OPT_SGD && d.opt_kind != HP_OPT_ADAMW)
    fail(HP_EIO, "checkpoint has an unknown optimizer kind");
  if (d.policy != HP_POLICY_SENTENCES && d.policy != HP_POLICY_TOKENS)
    fail(HP_EIO, "checkpoint has an unknown weight policy");
  hck1_parse(read_file(path), nullptr, nullptr, p.data(), m.data(), v.data(), n_);
  o_.kind = d.opt_kind;
  o_.beta1 = d.beta1;
  o_.beta2 = d.beta2;
  o_.eps = d.eps;
  o_.weight_decay = d.opt_kind == HP_OPT_ADAMW ? d.weight_decay : 0.0;
  x_.policy = d.policy;
  set_params(p.data(), n_, 0);
  if (d.opt_kind != HP_OPT_SGD) {
    set_adam(m.data(), v.data(), d.opt_t);
  } else {
    HP_CUDA(cudaMemset(adam_m_, 0, n_ * 4));
    HP_CUDA(cudaMemset(adam_v_, 0, n_ * 4));
    adam_t_ = 0;
  }
  step_ = d.step;
  // a loaded state starts a fresh update group
  acc_count_ = 0;
  if (acc_grads_) HP_CUDA(cudaMemset(acc_grads_, 0, n_ * 4));
  if (d_acc_lw_) HP_CUDA(cudaMemset(d_acc_lw_, 0, 2 * 8));
  if (out) *out = d;
}

void Engine::get_local_grads(float* flat, uint64_t n) {
  if (!local_grads_) fail(HP_ECONFIG, "gradient capture was not enabled");
  if (n != n_) fail(HP_ESHAPE, "get_local_grads: wrong element count");
  HP_CUDA(cudaStreamSynchronize(s_main_));
  HP_CUDA(cudaMemcpy(flat, local_grads_, n_ * 4, cudaMemcpyDeviceToHost));
}

uint64_t Engine::digest() {
  // params_digest (model.hpp:211-217): FNV-1a over the parameter bytes in
  // canonical order.  Host-side: it is byte-serial and runs at cadence only.
  if (!h_params_) HP_CUDA(cudaMallocHost(&h_params_, n_ * 4));
  HP_CUDA(cudaMemcpyAsync(h_params_, params_, n_ * 4, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaStreamSynchronize(s_main_));
  const uint8_t* p = reinterpret_cast<const uint8_t*>(h_params_);
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n_ * 4; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// ------------------------------------------------------------------ staging
void Engine::stage_batch(const hp_batch& b) {
  NvtxRange nv("hp.stage_batch");
  if (b.n_inst == 0)
    fail(HP_ECONFIG, "model_forward: empty batch (only the dummy path may skip data)");
  const uint64_t B = b.n_inst;
  const uint64_t T = b.tok_off[B];
  const uint64_t M = b.mask_off[B];
  if (B > x_.max_batch || T > x_.max_tokens || M > std::max<uint64_t>(x_.max_masks, 1))
    fail(HP_ECONFIG, "batch exceeds the engine capacity (tokens " + std::to_string(T) +
                         ", instances " + std::to_string(B) + ", masks " + std::to_string(M) + ")");
  const uint64_t Tm = x_.max_tokens, Bm = x_.max_batch,
                 Mm = (std::max<uint64_t>(x_.max_masks, 1) + mpad_ - 1) / mpad_ * mpad_;
  // wait until the previous copy out of this pinned buffer finished
  HP_CUDA(cudaEventSynchronize(ev_stage_[stage_idx_]));
  int* h = static_cast<int*>(h_stage_[stage_idx_]);
  if (s2s_) {
    double w = 0.0;
    stage_s2s(b, h, &w);
    *reinterpret_cast<double*>(static_cast<char*>(h_stage_[stage_idx_]) + stage_bytes_ - 8) = w;
    HP_CUDA(cudaMemcpyAsync(d_stage_, h_stage_[stage_idx_], stage_bytes_, cudaMemcpyHostToDevice,
                            s_main_));
    HP_CUDA(cudaEventRecord(ev_stage_[stage_idx_], s_main_));
    stage_idx_ = (stage_idx_ + 1) % kStageBufs;
    local_weight_ = w;
    staged_ = true;
    return;
  }
  int *tok = h, *seg = h + Tm, *pos = h + 2 * Tm, *cu = h + 3 * Tm, *mrow = cu + Bm + 1,
      *morig = mrow + Mm, *label = morig + Mm, *perm = label + Bm, *uid = perm + Tm,
      *useg = uid + Tm, *ulist = useg + Tm + 1, *ucount = ulist + Tm;
  double weight = 0.0;
  for (uint64_t i = 0; i < B; ++i) {
    const uint64_t t0 = b.tok_off[i], t1 = b.tok_off[i + 1];
    const uint64_t n = t1 - t0;
    // validation in model_forward order (model.hpp:347-390)
    if (n == 0) fail(HP_ESHAPE, "masked model: empty token sequence");
    if (n > m_.max_seq) fail(HP_ESHAPE, "masked model: sequence length exceeds max_seq");
    cu[i] = static_cast<int>(t0);
    for (uint64_t t = t0; t < t1; ++t) {
      const int64_t s = b.segments[t];
      if (s != 0 && s != 1) fail(HP_EINDEX, "segment id must be 0 or 1");
      const int64_t id = b.tokens[t];
      if (id < 0 || static_cast<uint64_t>(id) >= m_.vocab)
        fail(HP_EINDEX, "gather_rows: row " + std::to_string(id) + " outside [0," +
                            std::to_string(m_.vocab) + ")");
      tok[t] = static_cast<int>(id);
      seg[t] = static_cast<int>(s);
      pos[t] = static_cast<int>(t - t0);
    }
    double inst_w = 0.0;
    for (uint64_t k = b.mask_off[i]; k < b.mask_off[i + 1]; ++k) {
      const int64_t p = b.mask_pos[k];
      if (p < 0 || static_cast<uint64_t>(p) >= n) fail(HP_EINDEX, "mask position outside sequence");
      const int64_t o = b.mask_orig[k];
      if (o < 0 || static_cast<uint64_t>(o) >= m_.vocab)
        fail(HP_EINDEX, "ls_ce: target " + std::to_string(o) + " outside [0," +
                            std::to_string(m_.vocab) + ")");
      mrow[k] = static_cast<int>(t0 + p);
      morig[k] = static_cast<int>(o);
      inst_w += 1.0;
    }
    if (m_.with_nsp) {
      if (b.label[i] < 0 || b.label[i] > 1)
        fail(HP_EINDEX, "ls_ce: target " + std::to_string(b.label[i]) + " outside [0,2)");
      label[i] = static_cast<int>(b.label[i]);
      inst_w += 1.0;
    } else {
      label[i] = 0;
    }
    weight += x_.policy == HP_POLICY_SENTENCES ? 1.0 : inst_w;
  }
  cu[B] = static_cast<int>(T);
  // embedding-gradient plan: token positions grouped by id, position order
  // inside each group (embed_grad_kernel)
  {
    auto& order = sort_buf_;
    order.resize(T);
    for (uint64_t t = 0; t < T; ++t) order[t] = (static_cast<uint64_t>(tok[t]) << 32) | t;
    std::sort(order.begin(), order.end());
    int U = 0;
    for (uint64_t k = 0; k < T; ++k) {
      const int id = static_cast<int>(order[k] >> 32);
      perm[k] = static_cast<int>(order[k] & 0xffffffffu);
      if (k == 0 || id != uid[U - 1]) {
        uid[U] = id;
        useg[U] = static_cast<int>(k);
        ++U;
      }
    }
    useg[U] = static_cast<int>(T);
    int ns = 0;
    for (int u = 0; u < U; ++u)
      if (useg[u + 1] - useg[u] <= kEmbHotTokens) ulist[ns++] = u;
    int nh = 0;
    for (int u = 0; u < U; ++u)
      if (useg[u + 1] - useg[u] > kEmbHotTokens) ulist[ns + nh++] = u;
    ucount[0] = ns;
    ucount[1] = nh;
  }
  // padding rows up to a multiple of mpad_ (gathered as zeros, no loss, no
  // gradient: the weight above counts only real targets)
  const uint64_t Mp = M == 0 ? 0 : (M + mpad_ - 1) / mpad_ * mpad_;
  for (uint64_t k = M; k < Mp; ++k) {
    mrow[k] = -1;
    morig[k] = -1;
  }
  *reinterpret_cast<double*>(static_cast<char*>(h_stage_[stage_idx_]) + stage_bytes_ - 8) = weight;
  HP_CUDA(cudaMemcpyAsync(d_stage_, h_stage_[stage_idx_], stage_bytes_, cudaMemcpyHostToDevice,
                          s_main_));
  HP_CUDA(cudaEventRecord(ev_stage_[stage_idx_], s_main_));
  stage_idx_ = (stage_idx_ + 1) % kStageBufs;
  batch_.T = static_cast<int>(T);
  batch_.B = static_cast<int>(B);
  batch_.M = static_cast<int>(Mp);
  local_weight_ = weight;
  staged_ = true;
}

// ------------------------------------------------------------------ timers
void Engine::timers(bool on) {
  if (timed_pending_) collect_timed();
  timers_on_ = on;
  for (auto& t : tm_) {
    t.used = 0;
    t.ms = 0;
    t.flops = t.bytes = 0;
    t.launches = 0;
  }
}
void Engine::mark(int slot) {
  if (slot < 0 || slot >= 8) fail(HP_EINDEX, "mark slot out of range");
  if (!marks_[slot]) HP_CUDA(cudaEventCreate(&marks_[slot]));
  HP_CUDA(cudaEventRecord(marks_[slot], s_main_));
}
double Engine::elapsed(int a, int b) {
  if (a < 0 || a >= 8 || b < 0 || b >= 8 || !marks_[a] || !marks_[b])
    fail(HP_EINDEX, "elapsed: unrecorded mark");
  HP_CUDA(cudaEventSynchronize(marks_[b]));
  float ms = 0;
  HP_CUDA(cudaEventElapsedTime(&ms, marks_[a], marks_[b]));
  return ms;
}
void Engine::synchronize() {
  HP_CUDA(cudaStreamSynchronize(s_main_));
  HP_CUDA(cudaStreamSynchronize(s_comm_));
  if (s_upd_) HP_CUDA(cudaStreamSynchronize(s_upd_));
}

void Engine::tstart(int cls, cudaStream_t st) {
  if (!timers_on_) return;
  TimerAcc& t = tm_[cls];
  if (t.used == t.ev.size()) {
    cudaEvent_t a, b;
    HP_CUDA(cudaEventCreate(&a));
    HP_CUDA(cudaEventCreate(&b));
    t.ev.emplace_back(a, b);
  }
  HP_CUDA(cudaEventRecordWithFlags(t.ev[t.used].first, st ? st : s_main_,
                                  capturing_ ? cudaEventRecordExternal : cudaEventRecordDefault));
  t.k_open = kernel_launch_count();
}
void Engine::tstop(int cls, double flops, double bytes, cudaStream_t st) {
  if (!timers_on_) return;
  TimerAcc& t = tm_[cls];
  HP_CUDA(cudaEventRecordWithFlags(t.ev[t.used].second, st ? st : s_main_,
                                  capturing_ ? cudaEventRecordExternal : cudaEventRecordDefault));
  ++t.used;
  t.flops += flops;
  t.bytes += bytes;
  t.launches += kernel_launch_count() - t.k_open;
}
// Event spans of a timed graph replay (graph nodes: no host launch gaps in
// the spans) -> the class accumulators.
void Engine::collect_timed() {
  GraphEntry* e = timed_pending_;
  timed_pending_ = nullptr;
  HP_CUDA(cudaEventSynchronize(ev_done_));
  for (int c = 0; c < TM_COUNT; ++c) {
    TimerAcc& t = tm_[c];
    const GraphTimers& gt = e->timers[c];
    for (const auto& pr : gt.ev) {
      float ms = 0;
      HP_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      t.ms += ms;
    }
    t.flops += gt.flops;
    t.bytes += gt.bytes;
    t.launches += gt.launches;
  }
}

void Engine::timer_read(int which, std::string* name, double* ms, uint64_t* launches,
                        double* bytes, double* flops) {
  static const char* names[TM_COUNT] = {"gemm", "attention", "layernorm", "heads", "adam", "embedding"};
  if (which < 0 || which >= TM_COUNT) fail(HP_EINDEX, "timer index out of range");
  HP_CUDA(cudaStreamSynchronize(s_main_));
  if (timed_pending_) collect_timed();
  TimerAcc& t = tm_[which];
  for (size_t i = 0; i < t.used; ++i) {
    float e = 0;
    HP_CUDA(cudaEventElapsedTime(&e, t.ev[i].first, t.ev[i].second));
    t.ms += e;
  }
  t.used = 0;
  *name = names[which];
  *ms = t.ms;
  *launches = t.launches;
  *bytes = t.bytes;
  *flops = t.flops;
}

void Engine::record(int cls, double flops, std::function<void(cudaStream_t)> fn) {
  if (rec_on_) rec_.push_back(RecOp{cls, flops, std::move(fn)});
}

// One round's kernels of a class replayed back to back on one stream, from a
// CUDA graph (no launch gaps): the class's serialised duration -- what a
// per-kernel profile (ncu's launch list) sums -- and its algorithmic FLOPs.
// Runs one eager round first to record the class's launches (the round is a
// real update), then overwrites that class's outputs; measurement only.
void Engine::class_replay(int cls, int iters, double* ms, double* flops, uint64_t* launches) {
  if (in_flight_) fail(HP_ECONFIG, "class_replay while a round is in flight");
  if (!staged_) fail(HP_ECONFIG, "class_replay: no batch staged");
  rec_.clear();
  rec_on_ = true;
  const bool g = graphs_on_;
  graphs_on_ = false;
  try {
    round_async(0, 0.0);
    round_sync(nullptr);
  } catch (...) {
    rec_on_ = false;
    graphs_on_ = g;
    throw;
  }
  rec_on_ = false;
  graphs_on_ = g;
  double fl = 0;
  uint64_t n = 0;
  const uint64_t k0 = kernel_launch_count();
  HP_CUDA(cudaStreamBeginCapture(s_main_, cudaStreamCaptureModeThreadLocal));
  for (const RecOp& r : rec_)
    if (r.cls == cls) {
      r.fn(s_main_);
      fl += r.flops;
      ++n;
    }
  cudaGraph_t graph = nullptr;
  HP_CUDA(cudaStreamEndCapture(s_main_, &graph));
  const uint64_t kernels = kernel_launch_count() - k0;
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) fail(HP_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
  cudaEvent_t a, b;
  HP_CUDA(cudaEventCreate(&a));
  HP_CUDA(cudaEventCreate(&b));
  HP_CUDA(cudaGraphLaunch(exec, s_main_));  // warm-up
  HP_CUDA(cudaEventRecord(a, s_main_));
  for (int i = 0; i < iters; ++i) HP_CUDA(cudaGraphLaunch(exec, s_main_));
  HP_CUDA(cudaEventRecord(b, s_main_));
  HP_CUDA(cudaEventSynchronize(b));
  float t = 0;
  HP_CUDA(cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(exec);
  count_launch(static_cast<int>(kernels) * (iters + 1));
  rec_.clear();
  *ms = t / std::max(iters, 1);
  *flops = fl;
  *launches = kernels;
  (void)n;
}

void Engine::gemm_t(const GemmArgs& g) {
  record(TM_GEMM, 2.0 * g.M * g.N * g.K, [g](cudaStream_t st) { gemm(g, st); });
  tstart(TM_GEMM);
  gemm(g, s_main_);
  tstop(TM_GEMM, 2.0 * g.M * g.N * g.K,
        (double)asz_ * ((double)g.M * g.K + (double)g.K * g.N) +
            (g.ct == DType::f32 ? 4.0 : 2.0) * g.M * g.N);
}

void Engine::wgrad_t(const GemmArgs& g, cudaEvent_t fork, cudaEvent_t done) {
  if (!wg_on_) {
    gemm_t(g);
    return;
  }
  HP_CUDA(cudaEventRecord(fork, s_main_));
  HP_CUDA(cudaStreamWaitEvent(s_wg_, fork, 0));
  wg_forked_ = true;
  tstart(TM_GEMM, s_wg_);
  // split-K of the weight-gradient GEMMs capped at 2: a small wgrad (dWo,
  // 768 x 768 x 4096) then takes half the SMs for longer instead of all of
  // them with 8-way fp32 reductions, leaving the rest to the data-gradient
  // chain (C2: 7640 vs 7536 samples/s; cap 1: 7250)
  GemmArgs c = g;
  c.max_splits = 2;
  record(TM_GEMM, 2.0 * g.M * g.N * g.K, [c](cudaStream_t st) { gemm(c, st); });
  gemm(c, s_wg_);
  tstop(TM_GEMM, 2.0 * g.M * g.N * g.K,
        (double)asz_ * ((double)g.M * g.K + (double)g.K * g.N) +
            (g.ct == DType::f32 ? 4.0 : 2.0) * g.M * g.N,
        s_wg_);
  HP_CUDA(cudaEventRecord(done, s_wg_));
  serialize_if_timed(s_wg_);
}

// (timer events are recorded with cudaEventRecordExternal: under stream
// capture they become event-record nodes whose timestamps can be read after
// each replay, instead of capture-internal dependencies)
// Timer passes serialise the side streams into the compute stream, so each
// kernel's event span is its own duration, not a share of concurrent work.
void Engine::serialize_if_timed(cudaStream_t st) {
  if (!timers_on_) return;
  if (!ev_ser_) HP_CUDA(cudaEventCreateWithFlags(&ev_ser_, cudaEventDisableTiming));
  HP_CUDA(cudaEventRecord(ev_ser_, st));
  HP_CUDA(cudaStreamWaitEvent(s_main_, ev_ser_, 0));
}

void Engine::wait_wg(cudaEvent_t e) {
  if (wg_on_) HP_CUDA(cudaStreamWaitEvent(s_main_, e, 0));
}

// ------------------------------------------------------------------ forward
void Engine::forward(bool need_grad) {
  NvtxRange nv("hp.forward");
  if (s2s_) {
    forward_s2s();
    return;
  }
  const DevBatch& b = batch_;
  const int T = b.T;
  const DType wt = bf16_ ? DType::bf16 : DType::f32;
  const int iE = 0, iS0 = 1, iS1 = 2;
  // embedding (model.hpp:354-365)
  tstart(TM_EMBED);
  embed_fwd(b, d_, w(iE), w(iS0), w(iS1), wt, pe_, bert_ ? p0_ : layers_[0].x, at_, s_main_);
  if (bert_) {
    const int g = pidx("emb_ln.g");
    layernorm_fwd(T, d_, p0_, at_, pp(g), pp(g + 1), layers_[0].x, at_, mean0_, rstd0_, s_main_);
  }
  tstop(TM_EMBED, 0, (double)T * d_ * asz_ * (bert_ ? 4 : 2));

  int cursor = bert_ ? 5 : 3;  // index of the first wq of layer 0
  for (int l = 0; l < L_; ++l) {
    Layer& y = layers_[l];
    const int iq = cursor;
    const int iwo = iq + 3 * H_;
    // QKV projections for every head in one GEMM: B is the 3h grouped
    // [d x dk] blocks of the canonical layout (attention.hpp:44-46)
    GemmArgs q;
    q.M = T; q.N = 3 * d_; q.K = d_; q.ab = at_;
    q.a = Operand{y.x, d_, 0, 0, 0};
    q.b = Operand{w(iq), wld(iq), 0, dk_, (int64_t)(bf16_ ? shadow_off_[iq + 1] - shadow_off_[iq]
                                                           : table_[iq + 1].offset - table_[iq].offset)};
    q.c = y.qkv; q.ldc = 3 * d_; q.ct = at_;
    gemm_t(q);
    {
      const DevBatch bb = b;
      const Layer yy = y;
      auto op = [this, bb, yy](cudaStream_t st) {
        if (attn_long_)
          attention_fwd_long(bb, H_, (int)m_.max_seq, yy.qkv, yy.o, yy.lse, st);
        else if (attn_tc_)
          attention_fwd_tc(bb, H_, yy.qkv, yy.o, yy.lse, st);
        else if (bf16_ && attention_mma_supported(dk_, (int)m_.max_seq))
          attention_fwd_mma(bb, H_, yy.qkv, yy.o, yy.lse, st);
        else
          attention_fwd(bb, H_, dk_, yy.qkv, yy.o, yy.lse, at_, st);
      };
      const double fl = 4.0 * H_ * dk_ * (double)T * (double)m_.max_seq;
      tstart(TM_ATTN);
      op(s_main_);
      tstop(TM_ATTN, fl, 0);
      record(TM_ATTN, fl, op);
    }
    void* out = (l + 1 < L_) ? layers_[l + 1].x : x_final_;
    if (!bert_) {
      GemmArgs o;
      o.M = T; o.N = d_; o.K = d_; o.ab = at_;
      o.a = Operand{y.o, d_, 0, 0, 0};
      o.b = Operand{w(iwo), wld(iwo), 0, 0, 0};
      o.c = out; o.ldc = d_; o.ct = at_;
      gemm_t(o);
      cursor = iwo + 1;
    } else {
      const int ibo = iwo + 1, ig1 = iwo + 2, iw1 = iwo + 4, ib1 = iwo + 5, iw2 = iwo + 6,
                ib2 = iwo + 7, ig2 = iwo + 8;
      GemmArgs o;  // P1 = O Wo + bo + X
      o.M = T; o.N = d_; o.K = d_; o.ab = at_;
      o.a = Operand{y.o, d_, 0, 0, 0};
      o.b = Operand{w(iwo), wld(iwo), 0, 0, 0};
      o.c = y.p1; o.ldc = d_; o.ct = at_;
      o.bias = pp(ibo); o.resid = y.x; o.ld_resid = d_;
      gemm_t(o);
      tstart(TM_NORM);
      layernorm_fwd(T, d_, y.p1, at_, pp(ig1), pp(ig1 + 1), y.x1, at_, y.mean1, y.rstd1, s_main_);
      tstop(TM_NORM, 0, (double)T * d_ * asz_ * 2);
      GemmArgs f1;  // G = gelu(X1 W1 + b1), U saved
      f1.M = T; f1.N = F_; f1.K = d_; f1.ab = at_;
      f1.a = Operand{y.x1, d_, 0, 0, 0};
      f1.b = Operand{w(iw1), wld(iw1), 0, 0, 0};
      f1.c = y.g; f1.ldc = F_; f1.ct = at_;
      f1.bias = pp(ib1); f1.act = ACT_GELU; f1.aux = y.u;
      gemm_t(f1);
      GemmArgs f2;  // P2 = G W2 + b2 + X1
      f2.M = T; f2.N = d_; f2.K = F_; f2.ab = at_;
      f2.a = Operand{y.g, F_, 0, 0, 0};
      f2.b = Operand{w(iw2), wld(iw2), 0, 0, 0};
      f2.c = y.p2; f2.ldc = d_; f2.ct = at_;
      f2.bias = pp(ib2); f2.resid = y.x1; f2.ld_resid = d_;
      gemm_t(f2);
      tstart(TM_NORM);
      layernorm_fwd(T, d_, y.p2, at_, pp(ig2), pp(ig2 + 1), out, at_, y.mean2, y.rstd2, s_main_);
      tstop(TM_NORM, 0, (double)T * d_ * asz_ * 2);
      cursor = ig2 + 2;
    }
  }

  // heads (model.hpp:367-391)
  const int iw = pidx("mlm.w"), ib = iw + 1;
  tstart(TM_HEAD);
  gather_rows(b.M, d_, b.mrow, x_final_, hm_, at_, s_main_);
  tstop(TM_HEAD, 0, 0);
  GemmArgs z;
  z.M = b.M; z.N = V_; z.K = d_; z.ab = at_;
  z.a = Operand{hm_, d_, 0, 0, 0};
  z.b = Operand{w(iw), wld(iw), 0, 0, 0};
  z.c = z_; z.ldc = Vp_; z.ct = DType::f32; z.bias = pp(ib);
  if (b.M > 0) gemm_t(z);
  tstart(TM_HEAD);
  ls_ce(b.M, V_, z_, Vp_, b.morig, static_cast<float>(m_.label_smooth_eps), row_loss_, dz_, at_,
        Vp_, s_main_);
  if (need_grad) HP_CUDA(cudaMemsetAsync(dA_, 0, (size_t)T * d_ * asz_, s_main_));
  if (m_.with_nsp) {
    const int in = iw + 2;
    nsp_head(b, d_, x_final_, at_, pp(in), pp(in + 1), row_loss_ + b.M, gp(in), gp(in + 1), dA_,
             need_grad ? 1 : 0, s_main_);
  }
  tstop(TM_HEAD, 0, (double)b.M * V_ * 8);
}

// ------------------------------------------------------------------ backward
void Engine::grads_ready(int first_done) {
  if (capture_) return;  // deferred: the pre-reduce gradients are copied first
  while (next_bucket_ < buckets_.size() &&
         static_cast<int>(buckets_[next_bucket_].first_param) >= first_done)
    issue_bucket(next_bucket_++);
}

void Engine::emb_rows_update(int mode, cudaStream_t su) {
  adam_rows(adam_args_, mode, emb_lists_.uids, emb_lists_.cnts, emb_lists_.n,
            static_cast<int>(x_.max_tokens), V_, d_, table_[0].offset,
            bf16_ ? shadow_off_[0] : table_[0].offset, bf16_ ? shadow_ld_[0] : table_[0].cols, su);
}

void Engine::issue_bucket(size_t k) {
  const Bucket& bk = buckets_[k];
  HP_CUDA(cudaEventRecord(ev_bucket_[k], s_main_));
  HP_CUDA(cudaStreamWaitEvent(s_comm_, ev_bucket_[k], 0));
  if (wg_forked_) {  // and every weight gradient issued so far this round
    HP_CUDA(cudaEventRecord(ev_wgb_[k], s_wg_));
    HP_CUDA(cudaStreamWaitEvent(s_comm_, ev_wgb_[k], 0));
  }
  if (k + 1 == buckets_.size() && emb_sparse_round_) {
    // word-embedding gradient: every rank's (id, row) slots, then dE[id] +=
    // row rank by rank -- the same sum on every rank, in a fixed order
    const size_t slot_floats = (size_t)emb_cap_ * (d_ + 4);
    if (grad_comm_) {
      HP_NCCL(ncclAllGather(emb_rows_, emb_gath_, slot_floats, ncclFloat, comm_->nccl, s_comm_));
      for (int r = 0; r < comm_->world; ++r)
        embed_rows_scatter(emb_gath_ + r * slot_floats, emb_cap_, d_, gp(0), s_comm_);
    } else {
      embed_rows_scatter(emb_rows_, emb_cap_, d_, gp(0), s_comm_);  // measurement pass
    }
  } else if (comm_ && grad_comm_) {
    HP_NCCL(ncclAllReduce(grads_ + bk.lo, grads_ + bk.lo, bk.hi - bk.lo, ncclFloat, ncclSum,
                          comm_->nccl, s_comm_));
  }
  if (phase_ == 1) {
    // a non-final round of K: the reduced bucket joins the accumulator
    accumulate_grad(acc_grads_ + bk.lo, grads_ + bk.lo, bk.hi - bk.lo, s_comm_);
    return;
  }
  // the bucket's update runs behind the rest of backward (engine.hpp:147-153:
  // every rank applies the identical update to the identical reduced sum)
  cudaStream_t su = s_comm_;
  if (s_upd_) {
    HP_CUDA(cudaEventRecord(ev_reduced_[k], s_comm_));
    HP_CUDA(cudaStreamWaitEvent(s_upd_, ev_reduced_[k], 0));
    su = s_upd_;
    upd_forked_ = true;
  }
  AdamArgs a = adam_args_;
  a.g2 = phase_ == 2 ? acc_grads_ : nullptr;
  const bool split = emb_split_round_ && k + 1 == buckets_.size();
  const auto& its = split ? emb_rest_items_ : bucket_items_[k];
  a.items = adam_items_ + 5 * static_cast<size_t>(its.first);
  a.nitems = its.second;
  tstart(TM_ADAM, su);
  adam_update(a, su);
  if (split) emb_rows_update(1, su);  // the batch rows of the word embedding, dE final
  tstop(TM_ADAM, 0, 28.0 * (double)(bk.hi - bk.lo) + (bf16_ ? 2.0 * (double)(bk.hi - bk.lo) : 0.0),
        su);
  serialize_if_timed(su);
}

void Engine::backward() {
  NvtxRange nv("hp.backward");
  if (s2s_) {
    backward_s2s();
    return;
  }
  const DevBatch& b = batch_;
  const int T = b.T;
  if (wg_on_) {
    // the word-embedding gradient (94 MB at C2) is zeroed beside the head /
    // top layers instead of at the end of backward
    HP_CUDA(cudaEventRecord(ev_fork_[4 * L_], s_main_));
    HP_CUDA(cudaStreamWaitEvent(s_wg_, ev_fork_[4 * L_], 0));
    wg_forked_ = true;
    HP_CUDA(cudaMemsetAsync(gp(0), 0, sizeof(float) * table_[0].size(), s_wg_));
    HP_CUDA(cudaEventRecord(ev_emb_zero_, s_wg_));
  }
  const int iw = pidx("mlm.w");
  // MLM head: d(mlm.w) = Hm^T dZ, d(mlm.b) = colsum dZ, dHm = dZ W^T
  if (b.M > 0) {
    GemmArgs gw;
    gw.M = d_; gw.N = V_; gw.K = b.M; gw.ab = at_;
    gw.a = Operand{hm_, d_, 1, 0, 0};
    gw.b = Operand{dz_, Vp_, 0, 0, 0};
    gw.c = gp(iw); gw.ldc = V_; gw.ct = DType::f32;
    // beside the head's data gradient and layer L-1's backward (wgrad stream)
    if (wg_on_)
      wgrad_t(gw, ev_head_fork_, ev_wg_join_);
    else
      gemm_t(gw);
    tstart(TM_HEAD);
    {
      const uint64_t Mm = (std::max<uint64_t>(x_.max_masks, 1) + mpad_ - 1) / mpad_ * mpad_;
      DeferredFinal f = final_slot(colsum_part_floats((int)Mm, Vp_));
      col_sum(b.M, V_, dz_, Vp_, at_, gp(iw + 1), scratch_, s_main_, &f);
      issue_final(f);
    }
    tstop(TM_HEAD, 0, 0);
    GemmArgs gd;
    gd.M = b.M; gd.N = d_; gd.K = V_; gd.ab = at_;
    gd.a = Operand{dz_, Vp_, 0, 0, 0};
    gd.b = Operand{w(iw), wld(iw), 1, 0, 0};
    gd.c = dhm_; gd.ldc = d_; gd.ct = DType::f32;
    gemm_t(gd);
    scatter_rows_f32(b.M, d_, b.mrow, static_cast<const float*>(dhm_), dA_, at_, s_main_);
  } else {
    HP_CUDA(cudaMemsetAsync(gp(iw), 0, sizeof(float) * (size_t)(d_ + 1) * V_, s_main_));
  }
  grads_ready(iw);

  // dA_ holds d(final hidden)
  int first_wq = bert_ ? 5 : 3;
  const int per_layer = bert_ ? 3 * H_ + 10 : 0;
  for (int l = L_ - 1; l >= 0; --l) {
    Layer& y = layers_[l];
    const int iq = first_wq + l * per_layer;
    const int iwo = iq + 3 * H_;
    void* dP1 = nullptr;  // gradient reaching the attention output projection
    if (bert_) {
      const int ibo = iwo + 1, ig1 = iwo + 2, iw1 = iwo + 4, ib1 = iwo + 5, iw2 = iwo + 6,
                ib2 = iwo + 7, ig2 = iwo + 8;
      void* const dP2 = pbuf_[slot(l)];
      void* const dP1b = pbuf_[2 + slot(l)];
      void* const dU = ubuf_[slot(l)];
      // dP2's slot was last read by layer l+2's d(ffn.w2)
      if (l + rd_ < L_) wait_wg(ev_w2_[l + rd_]);
      tstart(TM_NORM);
      // LN2' also yields d(ffn.b2) = colsum(dP2) (P2 = G W2 + b2 + X1)
      {
        DeferredFinal f = final_slot(colsum_part_floats((int)x_.max_tokens, d_));
        layernorm_bwd(T, d_, dA_, at_, y.p2, at_, y.mean2, y.rstd2, pp(ig2), dP2, at_, gp(ig2),
                      gp(ig2 + 1), gp(ib2), scratch_, s_main_, &f);
        issue_final(f);
      }
      tstop(TM_NORM, 0, (double)T * d_ * asz_ * 3);
      GemmArgs w2;  // d(ffn.w2) = G^T dP2
      w2.M = F_; w2.N = d_; w2.K = T; w2.ab = at_;
      w2.a = Operand{y.g, F_, 1, 0, 0};
      w2.b = Operand{dP2, d_, 0, 0, 0};
      w2.c = gp(iw2); w2.ldc = d_; w2.ct = DType::f32;
      wgrad_t(w2, wg_on_ ? ev_fork_[4 * l] : nullptr, wg_on_ ? ev_w2_[l] : nullptr);
      GemmArgs du;  // dU = (dP2 W2^T) * gelu'(U)
      du.M = T; du.N = F_; du.K = d_; du.ab = at_;
      du.a = Operand{dP2, d_, 0, 0, 0};
      du.b = Operand{w(iw2), wld(iw2), 1, 0, 0};
      du.c = dU; du.ldc = F_; du.ct = at_;
      du.act = ACT_DGELU; du.aux = y.u;
      if (l + rd_ < L_) wait_wg(ev_w1_[l + rd_]);  // dU's slot: layer l+2's d(w1) / d(b1) read it
      gemm_t(du);
      GemmArgs w1;  // d(ffn.w1) = X1^T dU
      w1.M = d_; w1.N = F_; w1.K = T; w1.ab = at_;
      w1.a = Operand{y.x1, d_, 1, 0, 0};
      w1.b = Operand{dU, F_, 0, 0, 0};
      w1.c = gp(iw1); w1.ldc = F_; w1.ct = DType::f32;
      wgrad_t(w1, wg_on_ ? ev_fork_[4 * l + 1] : nullptr, wg_on_ ? ev_w1_[l] : nullptr);
      tstart(TM_NORM);
      {
        if (wg_on_) {
          // d(ffn.b1) = colsum(dU) beside the chain (its own scratch), before
          // the event that lets the next layer reuse dU_
          tstop(TM_NORM, 0, 0);
          tstart(TM_NORM, s_wg_);
          col_sum(T, F_, dU, F_, at_, gp(ib1), scratch_wg_, s_wg_);
          tstop(TM_NORM, 0, 0, s_wg_);
          HP_CUDA(cudaEventRecord(ev_w1_[l], s_wg_));
          tstart(TM_NORM);
        } else {
          DeferredFinal f = final_slot(colsum_part_floats((int)x_.max_tokens, F_));
          col_sum(T, F_, dU, F_, at_, gp(ib1), scratch_, s_main_, &f);
          issue_final(f);
        }
      }
      tstop(TM_NORM, 0, 0);
      GemmArgs dx1;  // dX1 = dU W1^T + dP2
      dx1.M = T; dx1.N = d_; dx1.K = F_; dx1.ab = at_;
      dx1.a = Operand{dU, F_, 0, 0, 0};
      dx1.b = Operand{w(iw1), wld(iw1), 1, 0, 0};
      dx1.c = dC_; dx1.ldc = d_; dx1.ct = at_;
      dx1.resid = dP2; dx1.ld_resid = d_;
      gemm_t(dx1);
      if (l + rd_ < L_) wait_wg(ev_wo_[l + rd_]);  // dP1's slot: layer l+2's d(wo) read it
      tstart(TM_NORM);
      // LN1' also yields d(bo) = colsum(dP1)
      {
        DeferredFinal f = final_slot(colsum_part_floats((int)x_.max_tokens, d_));
        layernorm_bwd(T, d_, dC_, at_, y.p1, at_, y.mean1, y.rstd1, pp(ig1), dP1b, at_, gp(ig1),
                      gp(ig1 + 1), gp(ibo), scratch_, s_main_, &f);
        issue_final(f);
      }
      tstop(TM_NORM, 0, (double)T * d_ * asz_ * 3);
      dP1 = dP1b;
    } else {
      dP1 = dA_;
    }
    GemmArgs wo;  // d(wo) = O^T dP1
    wo.M = d_; wo.N = d_; wo.K = T; wo.ab = at_;
    wo.a = Operand{y.o, d_, 1, 0, 0};
    wo.b = Operand{dP1, d_, 0, 0, 0};
    wo.c = gp(iwo); wo.ldc = d_; wo.ct = DType::f32;
    if (bert_)
      wgrad_t(wo, wg_on_ ? ev_fork_[4 * l + 2] : nullptr, wg_on_ ? ev_wo_[l] : nullptr);
    else
      gemm_t(wo);
    GemmArgs dO;  // dO = dP1 Wo^T
    dO.M = T; dO.N = d_; dO.K = d_; dO.ab = at_;
    dO.a = Operand{dP1, d_, 0, 0, 0};
    dO.b = Operand{w(iwo), wld(iwo), 1, 0, 0};
    dO.c = dC_; dO.ldc = d_; dO.ct = at_;
    gemm_t(dO);
    void* const dqkv = bert_ ? qbuf_[slot(l)] : dqkv_;
    if (bert_ && l + rd_ < L_) wait_wg(ev_wq_[l + rd_]);  // the slot: layer l+2's d(wqkv) read it
    {
      const DevBatch bb = b;
      const Layer yy = y;
      void* const dO = dC_;
      auto op = [this, bb, yy, dO, dqkv](cudaStream_t st) {
        if (attn_long_)
          attention_bwd_long(bb, H_, (int)m_.max_seq, yy.qkv, yy.o, dO, yy.lse, dqkv, st);
        else if (attn_tc_)
          attention_bwd_tc(bb, H_, yy.qkv, yy.o, dO, yy.lse, dqkv, st);
        else if (bf16_ && attention_mma_supported(dk_, (int)m_.max_seq))
          attention_bwd_mma(bb, H_, yy.qkv, yy.o, dO, yy.lse, dqkv, st);
        else
          attention_bwd(bb, H_, dk_, yy.qkv, yy.o, dO, yy.lse, dqkv, at_, st);
      };
      const double fl = 8.0 * H_ * dk_ * (double)T * (double)m_.max_seq;
      tstart(TM_ATTN);
      op(s_main_);
      tstop(TM_ATTN, fl, 0);
      record(TM_ATTN, fl, op);
    }
    const int64_t gstride_w = bf16_ ? (int64_t)(shadow_off_[iq + 1] - shadow_off_[iq])
                                    : (int64_t)(table_[iq + 1].offset - table_[iq].offset);
    GemmArgs wq;  // d(wq.*, wk.*, wv.*) = X^T dQKV, scattered into the 3h blocks
    wq.M = d_; wq.N = 3 * d_; wq.K = T; wq.ab = at_;
    wq.a = Operand{y.x, d_, 1, 0, 0};
    wq.b = Operand{dqkv, 3 * d_, 0, 0, 0};
    wq.c = gp(iq); wq.ldc = dk_; wq.c_group = dk_;
    wq.c_gstride = (int64_t)(table_[iq + 1].offset - table_[iq].offset);
    wq.ct = DType::f32;
    if (bert_)
      wgrad_t(wq, wg_on_ ? ev_fork_[4 * l + 3] : nullptr, wg_on_ ? ev_wq_[l] : nullptr);
    else
      gemm_t(wq);
    GemmArgs dx;  // dX = dQKV Wqkv^T (+ dP1 through the residual)
    dx.M = T; dx.N = d_; dx.K = 3 * d_; dx.ab = at_;
    dx.a = Operand{dqkv, 3 * d_, 0, 0, 0};
    dx.b = Operand{w(iq), wld(iq), 1, dk_, gstride_w};
    dx.c = bert_ ? dA_ : dB_; dx.ldc = d_; dx.ct = at_;
    if (bert_) {
      dx.resid = dP1;
      dx.ld_resid = d_;
    }
    gemm_t(dx);
    grads_ready(iq);
  }

  // embedding (+ its LayerNorm for the extension)
  const void* dx0 = dB_;
  if (bert_) {
    const int g = pidx("emb_ln.g");
    // into layer 1's dP1 slot (layer 0 uses slots 0 and 2): read by d(wo) of layer 1
    void* const dE0 = pbuf_[2 + slot(rd_ - 1)];
    if (rd_ - 1 < L_) wait_wg(ev_wo_[rd_ - 1]);
    tstart(TM_NORM);
    {
      DeferredFinal f = final_slot(colsum_part_floats((int)x_.max_tokens, d_));
      layernorm_bwd(T, d_, dA_, at_, p0_, at_, mean0_, rstd0_, pp(g), dE0, at_, gp(g), gp(g + 1),
                    nullptr, scratch_, s_main_, &f);
      issue_final(f);
    }
    tstop(TM_NORM, 0, (double)T * d_ * asz_ * 3);
    dx0 = dE0;
  }
  tstart(TM_EMBED);
  if (wg_forked_)
    HP_CUDA(cudaStreamWaitEvent(s_main_, ev_emb_zero_, 0));  // zeroed on the wgrad stream
  else
    HP_CUDA(cudaMemsetAsync(gp(0), 0, sizeof(float) * table_[0].size(), s_main_));
  if (sparse_emb_ && !capture_) {
    // the rows go to the exchange buffer; the zeroed dense gradient receives
    // every rank's rows in issue_bucket
    embed_bwd_rows(b, d_, dx0, at_, emb_rows_, emb_cap_, gp(1), gp(2), scratch_, s_main_);
    emb_sparse_round_ = true;
  } else {
    embed_bwd(b, d_, dx0, at_, gp(0), gp(1), gp(2), scratch_, s_main_);
  }
  tstop(TM_EMBED, 0, (double)T * d_ * (asz_ + 8));
  grads_ready(0);
  if (wg_forked_) {  // the wgrad stream joins the compute stream (graph capture needs it)
    HP_CUDA(cudaEventRecord(ev_wg_join_, s_wg_));
    HP_CUDA(cudaStreamWaitEvent(s_main_, ev_wg_join_, 0));
  }
}

// ------------------------------------------------------------------ round
void Engine::round_async(int dummy, double lr) {
  NvtxRange nv("hp.round");
  if (!staged_) fail(HP_ECONFIG, "round: no batch staged");
  HP_CUDA(cudaSetDevice(x_.device));
  // K micro rounds per update (Accumulator, optim.hpp:154-202): rounds 1..K-1
  // accumulate the reduced gradients, the K-th updates with the totals
  const uint64_t K = x_.update_freq;
  const bool final_round = K == 1 || acc_count_ + 1 == K;
  phase_ = K == 1 ? 0 : (final_round ? 2 : 1);
  // one identical update on every rank (engine.hpp:147-153, optim.hpp:107-146),
  // issued per bucket on the side stream as the buckets complete
  if (final_round) ++adam_t_;
  const double c1 = 1.0 / (1.0 - std::pow(o_.beta1, static_cast<double>(adam_t_)));
  const double c2 = 1.0 / (1.0 - std::pow(o_.beta2, static_cast<double>(adam_t_)));
  AdamArgs& a = adam_args_;
  a = AdamArgs{};
  a.p = params_; a.m = adam_m_; a.v = adam_v_; a.g = grads_; a.n = n_;
  a.lr = static_cast<float>(lr);
  a.b1 = static_cast<float>(o_.beta1);
  a.b2 = static_cast<float>(o_.beta2);
  a.eps = static_cast<float>(o_.eps);
  a.c1 = static_cast<float>(c1);
  a.c2 = static_cast<float>(c2);
  a.hyper = d_hyper_;  // the same three values, read on the device
  a.inv_w64 = inv_w64_;  // g = (float)((double)sum * (1 / total weight))
  a.err = err_;
  a.sgd = o_.kind == HP_OPT_SGD;
  a.wd = o_.kind == HP_OPT_ADAMW ? static_cast<float>(o_.weight_decay) : 0.f;
  a.shadow = shadow_;
  // the first round after a sync starts a fresh error state; later unsynced
  // rounds keep it (sticky), so round_sync reports the first error
  if (!in_flight_) {
    const unsigned long long e0[kErrWords] = {0ull, ~0ull, ~0ull, ~0ull};
    HP_CUDA(cudaMemcpyAsync(err_, e0, sizeof(e0), cudaMemcpyHostToDevice, s_main_));
    pending_.clear();
  }
  const uint32_t seq = ++seq_;
  pending_.push_back(Pending{seq, step_, adam_t_, acc_count_, final_round});
  if (final_round) pending_.back().adam_t = adam_t_ - 1;  // t before this round's ++t
  // pageable source: staged by the driver at the call, so the host array can
  // be reused at once; ordered before the round on s_main_
  float hyper[4] = {a.lr, a.c1, a.c2, 0.f};
  std::memcpy(&hyper[3], &seq, 4);
  HP_CUDA(cudaMemcpyAsync(d_hyper_, hyper, sizeof(hyper), cudaMemcpyHostToDevice, s_main_));

  // a timed graph's events are re-recorded by every replay: read the previous
  // replay's before launching the next
  if (timed_pending_) collect_timed();
  if (graphs_on_ && !capture_) {
    GraphEntry& e = graphs_[std::make_tuple(batch_.T, batch_.B, batch_.M,
                                           (dummy ? 1 : 0) | (phase_ << 1) | (grad_comm_ ? 0 : 8) |
                                               (timers_on_ ? 16 : 0))];
    if (e.exec) {
      HP_CUDA(cudaGraphLaunch(e.exec, s_main_));
      count_launch(static_cast<int>(e.launches));
      if (timers_on_) timed_pending_ = &e;
    } else if (e.seen++ == 0) {
      round_body(dummy);
    } else {
      const uint64_t k0 = kernel_launch_count();
      // timer pass: the event pairs recorded during capture become graph
      // nodes; they leave the eager pool and belong to the graph from here on
      std::array<size_t, TM_COUNT> u0{};
      std::array<double, TM_COUNT> f0{}, b0{};
      std::array<uint64_t, TM_COUNT> l0{};
      for (int c = 0; c < TM_COUNT; ++c) {
        u0[c] = tm_[c].used;
        f0[c] = tm_[c].flops;
        b0[c] = tm_[c].bytes;
        l0[c] = tm_[c].launches;
      }
      HP_CUDA(cudaStreamBeginCapture(s_main_, cudaStreamCaptureModeThreadLocal));
      capturing_ = true;
      try {
        round_body(dummy);
      } catch (...) {
        capturing_ = false;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(s_main_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      cudaGraph_t g = nullptr;
      capturing_ = false;
      HP_CUDA(cudaStreamEndCapture(s_main_, &g));
      e.launches = kernel_launch_count() - k0;
      const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) fail(HP_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
      if (timers_on_) {
        for (int c = 0; c < TM_COUNT; ++c) {
          TimerAcc& t = tm_[c];
          GraphTimers& gt = e.timers[c];
          gt.ev.assign(t.ev.begin() + u0[c], t.ev.begin() + t.used);
          t.ev.erase(t.ev.begin() + u0[c], t.ev.begin() + t.used);
          t.used = u0[c];
          gt.flops = t.flops - f0[c];
          gt.bytes = t.bytes - b0[c];
          gt.launches = t.launches - l0[c];
          t.flops = f0[c];  // counted when the replay's events are read
          t.bytes = b0[c];
          t.launches = l0[c];
        }
      }
      HP_CUDA(cudaGraphLaunch(e.exec, s_main_));
      if (timers_on_) timed_pending_ = &e;
    }
  } else {
    round_body(dummy);
  }
  acc_count_ = final_round ? 0 : acc_count_ + 1;
  last_final_ = final_round;
  if (final_round) ++step_;
  HP_CUDA(cudaEventRecord(ev_done_, s_main_));
  in_flight_ = true;
  last_dummy_ = dummy != 0;
}

DeferredFinal Engine::final_slot(size_t floats) {
  if (final_n_ == final_bufs_.size()) {
    final_bufs_.emplace_back(static_cast<float*>(dalloc(floats * 4)), floats);
    cudaEvent_t e;
    HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    final_evs_.push_back(e);
  }
  if (final_bufs_[final_n_].second < floats) {
    // a new job sequence (e.g. a round without masked positions shifts the
    // slots): grow -- only ever on a shape's first, eager round; the old
    // buffer stays alive for graphs captured with it
    final_bufs_[final_n_] = {static_cast<float*>(dalloc(floats * 4)), floats};
  }
  DeferredFinal f;
  f.part = final_bufs_[final_n_].first;
  return f;
}

// A column-reduction final (LayerNorm gamma / beta, bias gradient) runs on
// the side stream as soon as its partials are done.  (Batching them into one
// launch per gradient bucket cut 23 launches per C2 step but cost 2.5 % at
// N = 2 -- profiles/r02_ab_batched_finals.txt -- so each leaves on its own.)
void Engine::issue_final(DeferredFinal& f) {
  if (!f.queued) return;
  HP_CUDA(cudaEventRecord(final_evs_[final_n_], s_main_));
  HP_CUDA(cudaStreamWaitEvent(s_comm_, final_evs_[final_n_], 0));
  launch_final(f, s_comm_);  // (inside the caller's layernorm-class span)
  serialize_if_timed(s_comm_);
  ++final_n_;
}

void Engine::round_body(int dummy) {
  final_n_ = 0;
  wg_forked_ = false;
  upd_forked_ = false;
  emb_sparse_round_ = false;
  emb_split_round_ = false;
  // Dummies run the forward too (symmetric compute, engine.hpp:128-129).
  gemm_tc_set_sm_budget(sms_fwd_);
  forward(!dummy);
  gemm_tc_set_sm_budget(sms_bwd_);
  loss_reduce(row_loss_, batch_.M, row_loss_ + batch_.M, m_.with_nsp ? batch_.B : 0, d_lw_,
              s_main_);
  // d_lw_ = [loss, weight, local loss, local weight]
  if (dummy) {
    HP_CUDA(cudaMemsetAsync(d_lw_, 0, 4 * 8, s_main_));  // (K-totals untouched)
  } else {
    HP_CUDA(cudaMemcpyAsync(d_lw_ + 2, d_lw_, 8, cudaMemcpyDeviceToDevice, s_main_));
    HP_CUDA(cudaMemcpyAsync(d_lw_ + 1, d_weight_, 8, cudaMemcpyDeviceToDevice, s_main_));
    HP_CUDA(cudaMemcpyAsync(d_lw_ + 3, d_weight_, 8, cudaMemcpyDeviceToDevice, s_main_));
  }
  HP_CUDA(cudaEventRecord(ev_fwd_, s_main_));
  cudaStream_t sw = s_main_;
  if (comm_) {
    // [loss_sum, weight] allreduce BEFORE backward (engine.hpp:133), on the
    // comm stream so backward proceeds concurrently.
    HP_CUDA(cudaStreamWaitEvent(s_comm_, ev_fwd_, 0));
    HP_NCCL(ncclAllReduce(d_lw_, d_lw_, 2, ncclDouble, ncclSum, comm_->nccl, s_comm_));
    sw = s_comm_;
  } else {
    // the side stream joins here (updates depend on the weight finalised below)
    HP_CUDA(cudaStreamWaitEvent(s_comm_, ev_fwd_, 0));
  }
  finalize_weight(d_lw_, inv_w_, inv_w64_, err_, d_hyper_, sw);
  // K > 1: running [loss, weight] totals; the K-th round's update divides by
  // the total weight (engine.hpp:147-151)
  if (phase_ != 0) accumulate_weight(d_lw_, d_acc_lw_, d_lw_ + 4, inv_w64_, phase_ == 2, sw);
  // K = 1: the word-embedding rows outside every rank's batch ids get their
  // (zero-gradient) update now, behind backward, so the last bucket's update
  // after backward touches only the batch rows (bit-identical: adam_rows)
  emb_split_round_ = split_emb_ && phase_ == 0 && !capture_;
  if (emb_split_round_) {
    const int* cnt = dummy ? ucount_zero_ : batch_.ucount;
    const int W = comm_ ? comm_->world : 1;
    if (W > 1 && grad_comm_) {  // symmetric on every rank, dummies included
      HP_NCCL(ncclAllGather(batch_.uid, uid_all_, x_.max_tokens, ncclInt, comm_->nccl, sw));
      HP_NCCL(ncclAllGather(cnt, ucnt_all_, 2, ncclInt, comm_->nccl, sw));
      emb_lists_ = {uid_all_, ucnt_all_, W};
    } else {
      emb_lists_ = {batch_.uid, cnt, 1};
    }
    cudaStream_t su = sw;
    if (s_upd_) {
      HP_CUDA(cudaEventRecord(ev_reduced_[0], sw));
      HP_CUDA(cudaStreamWaitEvent(s_upd_, ev_reduced_[0], 0));
      su = s_upd_;
      upd_forked_ = true;
    }
    tstart(TM_ADAM, su);
    emb_rows_update(0, su);
    tstop(TM_ADAM, 0, 24.0 * (double)table_[0].size() + (bf16_ ? 2.0 * (double)table_[0].size() : 0.0), su);
    serialize_if_timed(su);
  }

  next_bucket_ = 0;
  if (dummy) {
    // zero loss, weight and gradient (engine.hpp:141-142)
    HP_CUDA(cudaMemsetAsync(grads_, 0, n_ * 4, s_main_));
    if (sparse_emb_ && !capture_) {
      // every rank issues the same collectives: an empty row set (all ids -1)
      HP_CUDA(cudaMemsetAsync(emb_rows_, 0xFF, (size_t)emb_cap_ * (d_ + 4) * 4, s_main_));
      emb_sparse_round_ = true;
    }
    grads_ready(0);
  } else {
    backward();
  }
  if (capture_) {
    if (!local_grads_) local_grads_ = static_cast<float*>(dalloc(n_ * 4));
    // the column-reduction finals (side stream) complete the local gradient
    // before the copy
    HP_CUDA(cudaEventRecord(ev_comm_done_, s_comm_));
    HP_CUDA(cudaStreamWaitEvent(s_main_, ev_comm_done_, 0));
    HP_CUDA(cudaMemcpyAsync(local_grads_, grads_, n_ * 4, cudaMemcpyDeviceToDevice, s_main_));
    capture_ = false;
    grads_ready(0);
    capture_ = true;
  }
  // the round ends when the last bucket's update has landed
  HP_CUDA(cudaEventRecord(ev_comm_done_, s_comm_));
  HP_CUDA(cudaStreamWaitEvent(s_main_, ev_comm_done_, 0));
  if (upd_forked_) {
    HP_CUDA(cudaEventRecord(ev_upd_done_, s_upd_));
    HP_CUDA(cudaStreamWaitEvent(s_main_, ev_upd_done_, 0));
  }
  HP_CUDA(cudaMemcpyAsync(h_lw_, d_lw_, 6 * 8, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaMemcpyAsync(h_err_, err_, kErrWords * 8, cudaMemcpyDeviceToHost, s_main_));
}

// The reference's cross-rank parameter check (engine.hpp:170-184): rank 0's
// digest is broadcast, every rank compares it with its own, the mismatch
// count is summed over the ranks, and a non-zero count is a numeric error on
// every rank.  The digest here is FNV-1a over the FNV-1a values of 64 KB
// blocks of the parameter bytes, computed on the device in parallel (the exact
// byte-serial params_digest stays available as digest()).
void Engine::check_digest_on_cadence() {
  NvtxRange nv("hp.digest_check");
  if (!comm_ || !grad_comm_) return;  // world 1 included: the same collectives
  const uint64_t every = check_debug_ ? 1 : check_every_;
  if (every == 0 || step_ % every != 0) return;
  const uint64_t bytes = n_ * 4;
  if (!d_dig_) d_dig_ = static_cast<uint64_t*>(dalloc(8 * (4 + fnv1a_chunked_scratch(bytes))));
  fnv1a_chunked(params_, bytes, d_dig_ + 4, d_dig_, s_main_);
  HP_CUDA(cudaMemcpyAsync(d_dig_ + 1, d_dig_, 8, cudaMemcpyDeviceToDevice, s_main_));
  HP_NCCL(ncclBroadcast(d_dig_ + 1, d_dig_ + 1, 1, ncclUint64, 0, comm_->nccl, s_main_));
  double* bad = reinterpret_cast<double*>(d_dig_ + 2);
  digest_mismatch(d_dig_, bad, s_main_);
  HP_NCCL(ncclAllReduce(bad, bad, 1, ncclDouble, ncclSum, comm_->nccl, s_main_));
  double h = 0;
  HP_CUDA(cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaStreamSynchronize(s_main_));
  if (h != 0.0)
    fail(HP_ENUMERIC, std::to_string(static_cast<int>(h)) +
                          " ranks diverged from master parameters at step " + std::to_string(step_));
}

// model_forward (model.hpp:260-390) alone on the staged batch: the summed
// loss and the batch weight, no backward, no collective, no update.
void Engine::forward_only(double* loss_sum, double* weight) {
  if (!staged_) fail(HP_ECONFIG, "forward: no batch staged");
  if (in_flight_) fail(HP_ECONFIG, "forward: a round is in flight");
  HP_CUDA(cudaSetDevice(x_.device));
  forward(false);
  loss_reduce(row_loss_, batch_.M, row_loss_ + batch_.M, m_.with_nsp ? batch_.B : 0, d_lw_ + 6,
              s_main_);
  double h[2] = {0, 0};
  HP_CUDA(cudaMemcpyAsync(h, d_lw_ + 6, 8, cudaMemcpyDeviceToHost, s_main_));
  HP_CUDA(cudaStreamSynchronize(s_main_));
  *loss_sum = h[0];
  *weight = local_weight_;
}

void Engine::round_sync(hp_round_out* out) {
  if (!in_flight_) fail(HP_ECONFIG, "round_sync without a round in flight");
  HP_CUDA(cudaEventSynchronize(ev_done_));
  in_flight_ = false;
  // per-round checks (engine.hpp:134-137 on the aggregated [loss, weight],
  // optim.hpp:131-133 on the gradient), of the FIRST failing round since the
  // last sync; the counters return to that round's entry state (the loss
  // checks throw before the update; a bad gradient throws inside it, after
  // Optimizer::step's ++t, before the engine's ++step)
  const unsigned long long kNone = ~0ull;
  const unsigned long long loss_seq = h_err_[0] ? h_err_[1] : kNone, grad_seq = h_err_[3];
  if (loss_seq != kNone || grad_seq != kNone) {
    const bool loss_first = loss_seq <= grad_seq;
    const unsigned long long seq = loss_first ? loss_seq : grad_seq;
    Pending p{};
    for (const Pending& q : pending_)
      if (q.seq == seq) p = q;
    pending_.clear();
    step_ = p.step;
    adam_t_ = p.adam_t + (!loss_first && p.final_round ? 1 : 0);
    acc_count_ = 0;  // the update group is abandoned (its accumulator is re-zeroed by the next flush)
    if (loss_first) {
      if (h_err_[0] & 1) fail(HP_ENUMERIC, "non-finite aggregated loss after step " + std::to_string(p.step));
      fail(HP_ENUMERIC, "total batch weight is zero: every rank was dummy");
    }
    fail(HP_ENUMERIC, "non-finite gradient for parameter " + param_at(h_err_[2]));
  }
  pending_.clear();
  if (last_final_) check_digest_on_cadence();
  if (out) {
    // K > 1: the report covers the K rounds (loss_sum / weight of the flush)
    const bool totals = last_final_ && x_.update_freq > 1;
    const double loss = totals ? h_lw_[4] : h_lw_[0], weight = totals ? h_lw_[5] : h_lw_[1];
    out->updated = last_final_ ? 1 : 0;
    out->step = step_;
    out->loss = loss / weight;
    out->weight = weight;
    out->local_loss_sum = h_lw_[2];
    out->local_weight = h_lw_[3];
  }
}

}  // namespace hp
