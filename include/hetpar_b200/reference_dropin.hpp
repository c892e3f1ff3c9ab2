// hetpar_b200/reference_dropin.hpp -- the literal drop-in for the reference's
// own C++ types.  Include it where the reference's headers are on the include
// path (-I <reference>/proj/include): it builds on hetpar::TrainState,
// hetpar::ProcessGroup, hetpar::Batch and hetpar::StepReport themselves, so
// the reference's round loop (train_run, engine.hpp:274-310; the tests'
// StepEngine drivers, test_engine.cpp:203-256) switches engines by changing
// one type name:
//
//   hetpar::StepEngine<float> engine(st, group, check_interval, debug);  // CPU
//   hetpar::b200::StepEngine<float> engine(st, group, check_interval, debug);  // B200
//
//   reference                                     this header
//   StepEngine<T>(TrainState<T>&, ProcessGroup&,  StepEngine<float>(same), device state
//     check_interval, debug)  engine.hpp:117-123    mirrored back into the TrainState
//   round(const Batch&, bool dummy)               round(): lr = scheduled_lr(st.sched,
//     -> optional<StepReport>  engine.hpp:125-165   st.step + 1) inside, as the reference
//   pending_rounds()          engine.hpp:165       pending_rounds()
//   ProcessGroup (comm.hpp:16-49)                 NcclProcessGroup : hetpar::ProcessGroup
//   make_tcp_group (comm.hpp:70-84)               NcclProcessGroup(host, port, world, rank, device)
//
// Errors are the reference's own exception types (common.hpp:14-34).
// State: the device keeps the fp32 master parameters and Adam moments; after
// every update they are copied back into st.params / st.opt (and st.step is
// set) so anything that reads the TrainState between rounds -- the digest,
// save_checkpoint(st, path), the caller's own code -- sees the reference's
// state.  Callers that do not read it between rounds pass
// sync_every_update = false and call sync_state() when they do.
#pragma once

#include <chrono>
#include <cstring>
#include <optional>
#include <string>
#include <type_traits>
#include <vector>

#include "hetpar/checkpoint.hpp"
#include "hetpar/comm.hpp"
#include "hetpar/engine.hpp"
#include "hetpar/model.hpp"
#include "hetpar/optim.hpp"
#include "hetpar_b200.h"

namespace hetpar::b200 {

// hp_status -> the reference's exception (the C ABI's message carries the
// reference's "kind: " prefix, which the reference's constructors add back)
[[noreturn]] inline void throw_reference(hp_status s) {
  std::string m = hp_last_error();
  auto strip = [&m](const char* p) {
    const size_t n = std::strlen(p);
    if (m.compare(0, n, p) == 0) m = m.substr(n);
  };
  switch (s) {
    case HP_ESHAPE: strip("shape: "); throw hetpar::shape_error(m);
    case HP_ECONFIG: strip("config: "); throw hetpar::config_error(m);
    case HP_EINDEX: strip("index: "); throw hetpar::index_error(m);
    case HP_EIO: strip("io: "); throw hetpar::io_error(m);
    case HP_ECOMM: strip("comm: "); throw hetpar::comm_error(m);
    case HP_ENUMERIC: strip("numeric: "); throw hetpar::numeric_error(m);
    default: throw hetpar::base_error(m);  // device failure: no reference counterpart
  }
}
inline void ok(hp_status s) {
  if (s != HP_OK) throw_reference(s);
}

// ProcessGroup over the NCCL communicator (one process per GPU): the
// control-plane collectives of the reference's contract -- root's exact bytes,
// the rank-ordered f64 fold, master-only gather, barrier -- host-staged; the
// step engine runs its own collectives on the same communicator.
class NcclProcessGroup final : public hetpar::ProcessGroup {
 public:
  // the world formed by the engine's TCP rendezvous (rank 0 serves the
  // ncclUniqueId; the rendezvous role of comm_tcp.cpp:154-237)
  NcclProcessGroup(const std::string& host, uint16_t port, size_t world, size_t rank, int device,
                   int timeout_ms = 30000)
      : ProcessGroup(world, rank), device_(device) {
    ok(hp_comm_create_tcp(host.c_str(), port, static_cast<int>(world), static_cast<int>(rank), device,
                          timeout_ms, &c_));
  }
  // the world formed over an existing group: rank 0's ncclUniqueId travels
  // with that group's broadcast (comm.hpp:25-27)
  NcclProcessGroup(hetpar::ProcessGroup& bootstrap, int device)
      : ProcessGroup(bootstrap.world_size(), bootstrap.rank()), device_(device) {
    std::vector<uint8_t> id(128, 0);
    if (bootstrap.rank() == 0) ok(hp_comm_unique_id(id.data()));
    id = bootstrap.broadcast(id, 0);
    ok(hp_comm_create(static_cast<int>(world_), static_cast<int>(rank_), device, id.data(), &c_));
  }
  ~NcclProcessGroup() override {
    if (c_) hp_comm_destroy(c_);
  }
  NcclProcessGroup(const NcclProcessGroup&) = delete;
  NcclProcessGroup& operator=(const NcclProcessGroup&) = delete;

  std::vector<uint8_t> broadcast(const std::vector<uint8_t>& payload, size_t root) override {
    // the root's length first, so every rank sizes its buffer
    const double mine = rank_ == root ? static_cast<double>(payload.size()) : 0.0;
    const std::vector<double> len = all_reduce_sum({mine});
    std::vector<uint8_t> out(static_cast<size_t>(len[0]));
    uint64_t got = 0;
    ok(hp_pg_broadcast(c_, payload.data(), payload.size(), root, out.data(), out.size(), &got));
    out.resize(got);
    return out;
  }
  std::vector<double> all_reduce_sum(const std::vector<double>& v) override {
    std::vector<double> out(v.size());
    ok(hp_pg_all_reduce_sum(c_, v.data(), v.size(), out.data()));
    return out;
  }
  std::vector<double> gather_scalars(double v) override {
    std::vector<double> out(world_);
    ok(hp_pg_gather_scalars(c_, v, out.data()));
    if (rank_ != 0) out.clear();
    return out;
  }
  void barrier() override { ok(hp_pg_barrier(c_)); }

  hp_comm* handle() const { return c_; }
  int device() const { return device_; }

 private:
  hp_comm* c_ = nullptr;
  int device_ = 0;
};

// StepEngine<T> (engine.hpp:114-192) on the B200.  T = float: the device keeps
// fp32 master weights (the fp32 parity path, compute = f32 by default; pass
// HP_COMPUTE_BF16 for the tcgen05 path).  The group is an NcclProcessGroup for
// world > 1; at world 1 any ProcessGroup works (no device collective needed).
template <class T>
class StepEngine {
  static_assert(std::is_same_v<T, float>, "the device engine keeps fp32 master weights");

 public:
  StepEngine(TrainState<T>& st, ProcessGroup& group, uint64_t check_interval, bool debug_checks,
             int compute = HP_COMPUTE_F32, bool sync_every_update = true)
      : st_(st), group_(group), check_interval_(check_interval), debug_(debug_checks),
        compute_(compute), sync_(sync_every_update) {
    if (st.spec.arch != Arch::masked_token_model)
      throw config_error("the device engine implements the masked_token_model architecture");
    st.spec.validate();
    if (auto* n = dynamic_cast<NcclProcessGroup*>(&group)) {
      comm_ = n->handle();
      device_ = n->device();
    } else if (group.world_size() > 1) {
      throw config_error("the device engine needs an NcclProcessGroup for world_size > 1");
    }
    // capacities for a batch of 64 full-length instances; a larger batch
    // re-creates the engine from the TrainState (grow())
    cap_batch_ = 64;
    cap_tokens_ = cap_batch_ * st.spec.max_seq;
    create();
  }
  ~StepEngine() {
    if (h_) hp_engine_destroy(h_);
  }
  StepEngine(const StepEngine&) = delete;
  StepEngine& operator=(const StepEngine&) = delete;

  std::optional<StepReport> round(const Batch& batch, bool dummy) {
    if (pending_rounds() == 0) group_start_ = std::chrono::steady_clock::now();
    // the batch as CSR arrays (hp_batch); validation happens in the engine,
    // in model_forward's order and with its messages
    uint64_t tokens = 0, masks = 0;
    for (const auto& in : batch) {
      tokens += in.tokens.size();
      masks += in.mask_positions.size();
    }
    if (batch.size() > cap_batch_ || tokens > cap_tokens_ || masks > cap_tokens_)
      grow(batch.size(), tokens, masks);
    std::vector<uint64_t> tok_off{0}, mask_off{0};
    std::vector<int64_t> tok, seg, mpos, morig, label;
    for (const auto& in : batch) {
      if (in.segments.size() != in.tokens.size())
        throw shape_error("masked model: segment ids length != tokens");
      if (in.mask_originals.size() != in.mask_positions.size())
        throw shape_error("masked model: originals/positions length mismatch");
      tok.insert(tok.end(), in.tokens.begin(), in.tokens.end());
      seg.insert(seg.end(), in.segments.begin(), in.segments.end());
      mpos.insert(mpos.end(), in.mask_positions.begin(), in.mask_positions.end());
      morig.insert(morig.end(), in.mask_originals.begin(), in.mask_originals.end());
      label.push_back(in.label);
      tok_off.push_back(tok.size());
      mask_off.push_back(mpos.size());
    }
    const hp_batch b{batch.size(), tok_off.data(), tok.data(), seg.data(), mask_off.data(),
                     mpos.data(), morig.data(), label.data()};
    ok(hp_engine_stage_batch(h_, &b));
    // the learning rate of update P + 1, inside the round (engine.hpp:152)
    const double lr = scheduled_lr(st_.sched, st_.step + 1);
    hp_round_out o{};
    try {
      ok(hp_engine_round(h_, dummy ? 1 : 0, lr, &o));
    } catch (const numeric_error&) {
      uint64_t s = 0;
      hp_engine_step_count(h_, &s);
      st_.step = s;  // the engine left P unchanged (engine.hpp:153-154)
      throw;
    }
    if (!o.updated) return std::nullopt;
    st_.step = o.step;
    if (sync_) sync_state();
    StepReport r;
    r.step = o.step;
    r.loss = o.loss;
    r.weight = o.weight;
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - group_start_).count();
    r.rank_seconds = group_.gather_scalars(r.seconds);  // engine.hpp:158-162
    return r;
  }

  uint64_t pending_rounds() const {
    uint64_t n = 0;
    ok(hp_engine_pending_rounds(h_, &n));
    return n;
  }

  // device parameters / Adam state -> the TrainState (canonical order)
  void sync_state() {
    std::vector<float> p(n_);
    ok(hp_engine_get_params(h_, p.data(), n_, 0));
    size_t o = 0;
    for (auto& e : st_.params.v) {
      std::memcpy(e.m.d.data(), p.data() + o, e.m.size() * sizeof(float));
      o += e.m.size();
    }
    if (st_.opt.kind == OptKind::adam) {
      std::vector<float> m(n_), v(n_);
      uint64_t t = 0;
      ok(hp_engine_get_adam(h_, m.data(), v.data(), &t));
      o = 0;
      for (size_t i = 0; i < st_.params.v.size(); ++i) {
        const size_t k = st_.params.v[i].m.size();
        std::memcpy(st_.opt.m[i].data(), m.data() + o, k * sizeof(float));
        std::memcpy(st_.opt.v[i].data(), v.data() + o, k * sizeof(float));
        o += k;
      }
      st_.opt.t = t;
    }
  }

 private:
  hp_model_desc model_desc() const {
    const ModelSpec& s = st_.spec;
    return hp_model_desc{HP_ARCH_MASKED_TOKEN_MODEL, s.d_model, s.heads, s.vocab, s.max_seq, 1, 0,
                         s.with_nsp ? 1 : 0, s.label_smooth_eps};
  }
  // the TrainState -> a fresh device engine
  void create() {
    const hp_model_desc md = model_desc();
    const hp_optim_desc od{st_.opt.kind == OptKind::adam ? HP_OPT_ADAM : HP_OPT_SGD, st_.opt.beta1,
                           st_.opt.beta2, st_.opt.eps, 0.0};
    const hp_exec_desc xd{compute_,
                          st_.policy == WeightPolicy::tokens ? HP_POLICY_TOKENS : HP_POLICY_SENTENCES,
                          device_, 25.0, cap_tokens_, cap_batch_, cap_tokens_, st_.update_freq};
    ok(hp_engine_create(&md, &od, &xd, comm_, &h_));
    ok(hp_engine_set_digest_check(h_, check_interval_, debug_ ? 1 : 0));
    std::vector<float> p;
    for (const auto& e : st_.params.v) p.insert(p.end(), e.m.d.begin(), e.m.d.end());
    n_ = p.size();
    ok(hp_engine_set_params(h_, p.data(), n_, 0));
    if (st_.opt.kind == OptKind::adam && !st_.opt.m.empty()) {
      std::vector<float> m, v;
      for (size_t i = 0; i < st_.params.v.size(); ++i) {
        m.insert(m.end(), st_.opt.m[i].begin(), st_.opt.m[i].end());
        v.insert(v.end(), st_.opt.v[i].begin(), st_.opt.v[i].end());
      }
      ok(hp_engine_set_adam(h_, m.data(), v.data(), st_.opt.t));
    }
    ok(hp_engine_set_step(h_, st_.step));
  }
  void grow(uint64_t inst, uint64_t tokens, uint64_t masks) {
    if (pending_rounds() != 0)
      throw config_error("batch larger than the device capacity inside an update group");
    sync_state();
    hp_engine_destroy(h_);
    h_ = nullptr;
    while (cap_batch_ < inst) cap_batch_ *= 2;
    while (cap_tokens_ < tokens || cap_tokens_ < masks) cap_tokens_ *= 2;
    create();
  }

  TrainState<T>& st_;
  ProcessGroup& group_;
  uint64_t check_interval_;
  bool debug_;
  int compute_;
  bool sync_;
  hp_comm* comm_ = nullptr;
  int device_ = 0;
  hp_engine* h_ = nullptr;
  uint64_t n_ = 0, cap_batch_ = 0, cap_tokens_ = 0;
  std::chrono::steady_clock::time_point group_start_{};
};

}  // namespace hetpar::b200
