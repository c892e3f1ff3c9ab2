// DeviceStepEngine: the B200 implementation of StepEngine<T>::round
// (include/hetpar/engine.hpp:125-165) for one rank (one process per GPU).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "hetpar_b200.h"
#include "hostdata.h"
#include "kernels.h"

struct hp_comm {
  ncclComm_t nccl = nullptr;
  int world = 1, rank = 0, device = 0;
  // control-plane collectives (pgroup.cpp): their stream and device scratch
  cudaStream_t pg_stream = nullptr;
  void* pg_buf = nullptr;
  size_t pg_cap = 0;
};

namespace hp {

constexpr int kEmbHotTokens = 32;  // = kEmbHot in kernels.cu (embedding-gradient plan)

// Timer classes for the roofline accounting (CUDA events on the launching
// stream around every launch of the class).
enum TimerClass { TM_GEMM = 0, TM_ATTN, TM_NORM, TM_HEAD, TM_ADAM, TM_EMBED, TM_COUNT };

class Engine {
 public:
  Engine(const hp_model_desc& m, const hp_optim_desc& o, const hp_exec_desc& x, hp_comm* comm);
  ~Engine();

  uint64_t nparams() const { return n_; }
  void set_params(const void* flat, uint64_t n, int dtype);
  void get_params(void* flat, uint64_t n, int dtype);
  void broadcast_params(int root);
  void get_adam(float* m, float* v, uint64_t* t);
  void set_adam(const float* m, const float* v, uint64_t t);
  void save_checkpoint(const std::string& path, const hp_ckpt_desc& c);
  void load_checkpoint(const std::string& path, hp_ckpt_desc* out);
  void set_capture(bool on) { capture_ = on; }
  void set_grad_comm(bool on) { grad_comm_ = on; }
  void set_digest_check(uint64_t every, bool debug) {
    check_every_ = every;
    check_debug_ = debug;
  }
  void get_local_grads(float* flat, uint64_t n);
  void stage_batch(const hp_batch& b);
  void round_async(int dummy, double lr);
  void round_sync(hp_round_out* out);
  void forward_only(double* loss_sum, double* weight);
  uint64_t digest();
  uint64_t step() const { return step_; }
  void set_step(uint64_t s);
  uint64_t pending_rounds() const { return acc_count_; }
  void timers(bool on);
  void mark(int slot);
  double elapsed(int a, int b);
  void synchronize();
  uint64_t stage_bytes() const { return stage_bytes_; }
  uint64_t readback_bytes() const { return 6 * 8 + kErrWords * 8; }
  void timer_read(int which, std::string* name, double* ms, uint64_t* launches, double* bytes,
                  double* flops);
  void class_replay(int cls, int iters, double* ms, double* flops, uint64_t* launches);

 private:
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  void* dalloc(size_t bytes);
  const void* w(int idx) const;   // GEMM view of a weight (shadow or fp32)
  int64_t wld(int idx) const;     // its row stride
  float* gp(int idx) const { return grads_ + table_[idx].offset; }
  float* pp(int idx) const { return params_ + table_[idx].offset; }
  int pidx(const std::string& name) const;
  void gemm_t(const GemmArgs& g);
  // launches of a class recorded during one eager round (class_replay)
  struct RecOp {
    int cls;
    double flops;
    std::function<void(cudaStream_t)> fn;
  };
  std::vector<RecOp> rec_;
  bool rec_on_ = false;
  void record(int cls, double flops, std::function<void(cudaStream_t)> fn);
  // a weight-gradient GEMM on the wgrad stream (see backward): forks from the
  // compute stream, records `done` when finished
  void wgrad_t(const GemmArgs& g, cudaEvent_t fork, cudaEvent_t done);
  void wait_wg(cudaEvent_t e);
  void serialize_if_timed(cudaStream_t st);  // compute stream waits for a pending wgrad
  void tstart(int cls, cudaStream_t st = nullptr);
  void tstop(int cls, double flops, double bytes, cudaStream_t st = nullptr);
  void forward(bool need_grad_state);
  void backward();
  // transformer_seq2seq extension (engine_s2s.cpp)
  void stage_s2s(const hp_batch& b, int* h, double* weight);
  void forward_s2s();
  void backward_s2s();
  void s2s_alloc();
  GemmArgs grouped_b(int first_block, int N, int K, const void* a, int64_t lda, int a_trans,
                     int b_trans) const;
  void ln_fwd(int T, const void* x, int ig, void* y, float* mean, float* rstd);
  void ln_bwd(int T, const void* dy, const void* x, const float* mean, const float* rstd, int ig,
              void* dx, float* dbias);
  void attn_op_fwd(const AttnArgs& a);
  void attn_op_bwd(const AttnArgs& a);
  void grads_ready(int first_done_param);
  void issue_bucket(size_t b);
  void round_body(int dummy);  // the device work of one round (eager or captured)
  DeferredFinal final_slot(size_t floats);  // partial buffer for the next deferred final
  void issue_final(DeferredFinal& f);        // its final on the side stream

  hp_model_desc m_;
  hp_optim_desc o_;
  hp_exec_desc x_;
  hp_comm* comm_;
  bool bf16_;
  DType at_;
  size_t asz_;
  int d_, H_, dk_, V_, Vp_, L_, F_;
  bool bert_;
  bool s2s_ = false;  // HP_ARCH_SEQ2SEQ
  float emb_scale_ = 1.f;
  std::vector<ParamEntry> table_;
  std::vector<Bucket> buckets_;
  std::vector<uint64_t> shadow_off_, shadow_ld_;
  uint64_t n_ = 0, n_shadow_ = 0;

  std::vector<void*> allocs_;
  float *params_ = nullptr, *grads_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr;
  void* shadow_ = nullptr;
  uint64_t* seg_table_ = nullptr;
  uint64_t* adam_items_ = nullptr;
  int nitems_ = 0;
  int nseg_ = 0;
  float* pe_ = nullptr;

  // staged batch
  static constexpr int kStageBufs = 2;
  void* h_stage_[kStageBufs] = {nullptr, nullptr};
  cudaEvent_t ev_stage_[kStageBufs] = {};
  int stage_idx_ = 0;
  size_t stage_bytes_ = 0;
  void* d_stage_ = nullptr;
  DevBatch batch_;
  double* d_weight_ = nullptr;  // inside the staged block
  double local_weight_ = 0;
  bool staged_ = false;
  std::vector<uint64_t> sort_buf_;

  // activations
  struct Layer {
    void *x = nullptr, *qkv = nullptr, *o = nullptr, *p1 = nullptr, *x1 = nullptr, *u = nullptr,
         *g = nullptr, *p2 = nullptr;
    float *lse = nullptr, *mean1 = nullptr, *rstd1 = nullptr, *mean2 = nullptr, *rstd2 = nullptr;
    // seq2seq decoder: cross-attention (qc, kvc, oc, lsec), x2 = LN2 output,
    // p3 / LN3 around the FFN
    void *qc = nullptr, *kvc = nullptr, *oc = nullptr, *x2 = nullptr, *p3 = nullptr;
    float *lsec = nullptr, *mean3 = nullptr, *rstd3 = nullptr;
  };
  std::vector<Layer> layers_;
  // seq2seq: decoder layers (layers_ holds the encoder), the encoder output
  // (memory), per-side batches, decoder targets, the embedding-gradient plan
  // over [source tokens, decoder-input tokens], its input-gradient rows
  std::vector<Layer> dec_layers_;
  void* mem_ = nullptr;
  DevBatch enc_, dec_, embp_;
  const int* tgt_ = nullptr;
  // seq2seq attention packing: consecutive pairs whose sources and targets
  // each fit one 128-row tile share a CTA (s2s_grp_[0..*s2s_ngrp_], staged)
  const int* s2s_grp_ = nullptr;
  const int* s2s_ngrp_ = nullptr;
  bool attn_pack_ = true;
  int sms_fwd_ = 0, sms_bwd_ = 0;  // GEMM grid SM budget in forward / the rest (0: all)
  void *dqc_ = nullptr, *dkvc_ = nullptr, *dmem_ = nullptr, *demb_ = nullptr;
  void *x_final_ = nullptr, *p0_ = nullptr;
  float *mean0_ = nullptr, *rstd0_ = nullptr;
  void *hm_ = nullptr, *dz_ = nullptr, *dhm_ = nullptr;
  float *z_ = nullptr, *row_loss_ = nullptr;
  void *dA_ = nullptr, *dB_ = nullptr, *dC_ = nullptr, *dqkv_ = nullptr, *dU_ = nullptr;
  // bert: layer-parity slots -- pbuf_ {dP2 even, dP2 odd, dP1 even, dP1 odd}
  // (pbuf_[0] = dB_), ubuf_ dU (ubuf_[0] = dU_), qbuf_ dQKV (qbuf_[0] = dqkv_)
  void* pbuf_[4] = {};
  int rd_ = 2;  // slots per buffer = reuse distance in layers
  int slot(int l) const { return rd_ == 2 ? (l & 1) : 0; }
  void* ubuf_[2] = {};
  void* qbuf_[2] = {};
  float* scratch_ = nullptr;
  double* d_lw_ = nullptr;  // [loss, weight] (global after the allreduce)
  float* inv_w_ = nullptr;
  double* inv_w64_ = nullptr;
  unsigned long long* err_ = nullptr;    // numeric-error state (kernels.h kErrWords)
  double* h_lw_ = nullptr;
  unsigned long long* h_err_ = nullptr;
  // rounds issued since the last sync: a pipelined error rolls the counters
  // back to the failing round (its sequence number travels in hyper[3])
  struct Pending {
    uint32_t seq;
    uint64_t step, adam_t, acc_count;
    bool final_round;
  };
  std::vector<Pending> pending_;
  uint32_t seq_ = 0;
  std::string param_at(uint64_t flat_index) const;
  float* h_params_ = nullptr;

  cudaStream_t s_main_ = nullptr, s_comm_ = nullptr;
  cudaStream_t s_upd_ = nullptr;   // N > 1: per-bucket updates beside the allreduces
  cudaEvent_t ev_upd_done_ = nullptr;
  std::vector<cudaEvent_t> ev_reduced_;
  bool upd_forked_ = false;
  // weight-gradient GEMMs run beside the data-gradient chain (bert_encoder):
  // they fill the SMs the N = d GEMMs leave idle and the GEMM tails
  cudaStream_t s_wg_ = nullptr;
  bool wg_on_ = false;
  bool wg_forked_ = false;  // the wgrad stream took work this round (capture-safe waits)
  std::vector<cudaEvent_t> ev_fork_;                      // [4 L + 1] fork points
  std::vector<cudaEvent_t> ev_w2_, ev_w1_, ev_wo_, ev_wq_;  // [L] wgrad done
  std::vector<cudaEvent_t> ev_wgb_;                        // [buckets] wgrads so far
  cudaEvent_t ev_wg_join_ = nullptr;
  cudaEvent_t ev_emb_zero_ = nullptr, ev_head_fork_ = nullptr;
  float* scratch_wg_ = nullptr;  // column-sum scratch of the wgrad stream
  cudaEvent_t ev_fwd_ = nullptr, ev_comm_done_ = nullptr, ev_done_ = nullptr;
  std::vector<cudaEvent_t> ev_bucket_;
  size_t next_bucket_ = 0;

  bool capture_ = false;
  // N > 1, word embedding alone in the last bucket: its gradient leaves the
  // rank row-sparse (distinct ids of the batch) -- allgather + rank-ordered
  // scatter instead of a dense allreduce (see backward / issue_bucket)
  bool sparse_emb_ = false, emb_sparse_round_ = false;
  // K = 1 split of the word-embedding update (round_body, issue_bucket)
  bool split_emb_ = false, emb_split_round_ = false;
  std::pair<int, int> emb_rest_items_{0, 0};  // last bucket's items without param 0
  int* uid_all_ = nullptr;     // [W][max_tokens] every rank's sorted distinct ids
  int* ucnt_all_ = nullptr;    // [W][2] their counts
  int* ucount_zero_ = nullptr; // [2] a dummy round's (empty) count
  struct { const int* uids; const int* cnts; int n; } emb_lists_{nullptr, nullptr, 0};
  void emb_rows_update(int mode, cudaStream_t su);
  int emb_cap_ = 0;
  float* emb_rows_ = nullptr;  // [cap][d + 4]
  float* emb_gath_ = nullptr;  // [world][cap][d + 4]
  bool attn_long_ = false;  // 128 < max_seq <= 512: attention_*_long
  bool grad_comm_ = true;  // measurement toggle (hp_engine_set_grad_comm)
  // check_digest_on_cadence (engine.hpp:170-184): every check_every_ updates
  // (every update when check_debug_), N > 1
  uint64_t check_every_ = 100;
  bool check_debug_ = false;
  uint64_t* d_dig_ = nullptr;  // [4 + chunks]: mine, master, bad (double)
  void check_digest_on_cadence();
  float* local_grads_ = nullptr;
  uint64_t step_ = 0, adam_t_ = 0;
  bool in_flight_ = false;
  bool last_dummy_ = false;
  // K > 1 accumulation state (Accumulator, optim.hpp:154-202)
  float* acc_grads_ = nullptr;   // reduced gradient sums of the pending rounds
  double* d_acc_lw_ = nullptr;   // their [loss, weight] totals
  uint64_t acc_count_ = 0;       // rounds accumulated since the last update
  int phase_ = 0;                // current round: 0 K=1, 1 accumulate, 2 final of K
  bool last_final_ = true;

  bool timers_on_ = false;
  cudaEvent_t ev_ser_ = nullptr;
  struct TimerAcc {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t used = 0;
    double flops = 0, bytes = 0;
    double ms = 0;
    uint64_t launches = 0;      // kernels launched inside the class's spans
    uint64_t k_open = 0;        // kernel_launch_count() at the open span's start
    cudaEvent_t cur = nullptr;
  };
  std::array<TimerAcc, TM_COUNT> tm_;

  // CUDA graphs of round_body, keyed by batch shape (T, B, padded M, dummy):
  // first sighting runs eagerly, the second is captured, later ones replay
  // (one graph launch instead of ~300 kernel launches per round).
  // timer event pairs baked into a captured (timed) graph, per class, and the
  // work they stand for; accumulated after every replay
  struct GraphTimers {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    double flops = 0, bytes = 0;
    uint64_t launches = 0;
  };
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;  // kernels inside, for kernel_launch_count()
    int seen = 0;
    std::array<GraphTimers, TM_COUNT> timers;  // timed graphs only
  };
  GraphEntry* timed_pending_ = nullptr;
  bool capturing_ = false;  // inside cudaStreamBeginCapture .. EndCapture  // a timed replay whose events are unread
  void collect_timed();
  std::map<std::tuple<int, int, int, int>, GraphEntry> graphs_;
  bool graphs_on_ = true;
  bool attn_tc_ = false;      // tcgen05 attention kernels (attn_tc.cu)
  float* d_hyper_ = nullptr;  // [lr, c1, c2, 0] of the current round (device)
  // deferred column-reduction finals: one partial buffer + event per job of a
  // round (the job sequence is fixed by the model), allocated on first use
  std::vector<std::pair<float*, size_t>> final_bufs_;
  std::vector<cudaEvent_t> final_evs_;
  size_t final_n_ = 0;
  int mpad_ = 1;              // masked positions padded to a multiple (bf16: 64)
  std::array<cudaEvent_t, 8> marks_{};
  AdamArgs adam_args_{};
  std::vector<std::pair<int, int>> bucket_items_;  // [first item, count] per bucket
};

}  // namespace hp
