// hetpar_b200/step_engine.hpp -- header-only C++ host layer over the C ABI
// (include/hetpar_b200.h), mirroring the reference's C++ model/trainer API for
// the data-parallel step so reference callers switch by changing the type:
//
//   reference (arxiv/paper_2009_14783, proj/include/hetpar/)   this header
//   ModelSpec            model.hpp:28-67                       hetpar::b200::ModelSpec
//   Instance / Batch     model.hpp:72-83                       hetpar::b200::Instance / Batch
//   StepReport           engine.hpp:26-32                      hetpar::b200::StepReport
//   StepEngine<T>::round engine.hpp:125-165                    hetpar::b200::DeviceStepEngine::round
//   build_epoch_batches  dataset.cpp:52-88                     hetpar::b200::build_epoch_batches
//   partition_for_rank   dataset.cpp:90-117                    hetpar::b200::partition_for_rank
//   init_parameters      model.hpp:171-184                     hetpar::b200::init_parameters
//   scheduled_lr         optim.hpp:59-70                       (caller, unchanged)
//
// Errors are thrown as the reference taxonomy (common.hpp:14-34) re-declared
// here under hetpar::b200 with the same names and message prefixes.
#pragma once

#include <chrono>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "hetpar_b200.h"

namespace hetpar::b200 {

struct base_error : std::runtime_error {
  explicit base_error(const std::string& m) : std::runtime_error(m) {}
};
struct shape_error : base_error { using base_error::base_error; };
struct config_error : base_error { using base_error::base_error; };
struct index_error : base_error { using base_error::base_error; };
struct io_error : base_error { using base_error::base_error; };
struct comm_error : base_error { using base_error::base_error; };
struct numeric_error : base_error { using base_error::base_error; };
struct device_error : base_error { using base_error::base_error; };

inline void check(hp_status s) {
  if (s == HP_OK) return;
  const std::string m = hp_last_error();
  switch (s) {
    case HP_ESHAPE: throw shape_error(m);
    case HP_ECONFIG: throw config_error(m);
    case HP_EINDEX: throw index_error(m);
    case HP_EIO: throw io_error(m);
    case HP_ECOMM: throw comm_error(m);
    case HP_ENUMERIC: throw numeric_error(m);
    default: throw device_error(m);
  }
}

enum class Arch : int { masked_token_model = HP_ARCH_MASKED_TOKEN_MODEL, bert_encoder = HP_ARCH_BERT_ENCODER };
enum class WeightPolicy : int { sentences = HP_POLICY_SENTENCES, tokens = HP_POLICY_TOKENS };

struct ModelSpec {
  Arch arch = Arch::masked_token_model;
  size_t d_model = 0, heads = 1, vocab = 0, max_seq = 0;
  size_t layers = 1, d_ff = 0;  // bert_encoder extension
  bool with_nsp = true;
  double label_smooth_eps = 0.0;
  hp_model_desc desc() const {
    return hp_model_desc{static_cast<int>(arch), d_model, heads, vocab, max_seq, layers, d_ff,
                         with_nsp ? 1 : 0, label_smooth_eps};
  }
};

struct Instance {
  std::vector<int64_t> tokens, segments, mask_positions, mask_originals;
  int64_t label = 0;
};
using Batch = std::vector<Instance>;

struct StepReport {
  uint64_t step = 0;
  double loss = 0.0, weight = 0.0, seconds = 0.0;
  std::vector<double> rank_seconds;  // master only (gather_scalars), engine.hpp:158-162
};

inline uint64_t flat_size(const ModelSpec& s) {
  const hp_model_desc d = s.desc();
  uint64_t n = 0, e = 0;
  check(hp_param_count(&d, &n, &e));
  return e;
}

inline std::vector<double> init_parameters(const ModelSpec& s, uint64_t seed) {
  const hp_model_desc d = s.desc();
  std::vector<double> out(flat_size(s));
  check(hp_init_parameters(&d, seed, out.data()));
  return out;
}

struct BatchPlan {
  uint64_t epoch = 0;
  std::vector<std::vector<uint64_t>> batches;
};

inline BatchPlan build_epoch_batches(const std::vector<uint32_t>& lens, size_t max_sentences,
                                     uint64_t max_tokens, uint64_t base_seed, uint64_t epoch) {
  std::vector<uint64_t> order(lens.size()), sizes(lens.size() + 1);
  uint64_t nb = 0;
  check(hp_build_epoch_batches(lens.data(), lens.size(), max_sentences, max_tokens, base_seed,
                               epoch, order.data(), sizes.data(), &nb));
  BatchPlan p;
  p.epoch = epoch;
  size_t o = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    p.batches.emplace_back(order.begin() + o, order.begin() + o + sizes[b]);
    o += sizes[b];
  }
  return p;
}

struct RankBatch {
  uint64_t batch_index = 0;
  bool dummy = false;
};

inline std::vector<RankBatch> partition_for_rank(const BatchPlan& plan, size_t world, size_t rank) {
  const uint64_t nb = plan.batches.size();
  const uint64_t cap = world ? (nb + world - 1) / world + 1 : 1;
  std::vector<uint64_t> bi(cap);
  std::vector<uint8_t> dm(cap);
  uint64_t rounds = 0;
  check(hp_partition_for_rank(nb, world, rank, bi.data(), dm.data(), &rounds));
  std::vector<RankBatch> out(rounds);
  for (uint64_t t = 0; t < rounds; ++t) out[t] = {bi[t], dm[t] != 0};
  return out;
}

// RAII communicator (one process per GPU). The 128-byte id travels over the
// caller's existing control plane (ProcessGroup::broadcast in the reference).
class Communicator {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(128);
    check(hp_comm_unique_id(id.data()));
    return id;
  }
  Communicator(int world, int rank, int device, const std::vector<uint8_t>& id)
      : world_(world), rank_(rank) {
    check(hp_comm_create(world, rank, device, id.data(), &h_));
  }
  int world() const { return world_; }
  int rank() const { return rank_; }
  ~Communicator() { if (h_) hp_comm_destroy(h_); }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  hp_comm* handle() const { return h_; }

 private:
  hp_comm* h_ = nullptr;
  int world_ = 1, rank_ = 0;
};

// StepEngine<T> on the device: round(batch, dummy) = forward -> [loss, weight]
// allreduce -> backward with bucketed gradient allreduce -> / sum(weight) ->
// identical optimizer update; returns the update's StepReport.
class DeviceStepEngine {
 public:
  // check_interval / debug: the reference StepEngine's digest cadence
  // (engine.hpp:117-123, 170-184)
  DeviceStepEngine(const ModelSpec& spec, const hp_optim_desc& opt, const hp_exec_desc& exec,
                   Communicator* comm = nullptr, uint64_t check_interval = 100, bool debug = false)
      : n_(flat_size(spec)), comm_(comm) {
    const hp_model_desc d = spec.desc();
    check(hp_engine_create(&d, &opt, &exec, comm ? comm->handle() : nullptr, &h_));
    check(hp_engine_set_digest_check(h_, check_interval, debug ? 1 : 0));
  }
  ~DeviceStepEngine() { if (h_) hp_engine_destroy(h_); }
  DeviceStepEngine(const DeviceStepEngine&) = delete;
  DeviceStepEngine& operator=(const DeviceStepEngine&) = delete;

  void set_params(const std::vector<double>& flat) { check(hp_engine_set_params(h_, flat.data(), flat.size(), 1)); }
  std::vector<float> params() const {
    std::vector<float> p(n_);
    check(hp_engine_get_params(h_, p.data(), n_, 0));
    return p;
  }
  void broadcast_params(int root) { check(hp_engine_broadcast_params(h_, root)); }
  uint64_t digest() const {
    uint64_t d = 0;
    check(hp_engine_params_digest(h_, &d));
    return d;
  }

  std::optional<StepReport> round(const Batch& batch, bool dummy, double lr) {
    // seconds run from the update group's first round (engine.hpp:126)
    if (!in_group_) group_start_ = std::chrono::steady_clock::now();
    in_group_ = true;
    std::vector<uint64_t> tok_off{0}, mask_off{0};
    std::vector<int64_t> tokens, segments, mpos, morig, label;
    for (const auto& in : batch) {
      if (in.segments.size() != in.tokens.size())
        throw shape_error("shape: masked model: segment ids length != tokens");
      if (in.mask_originals.size() != in.mask_positions.size())
        throw shape_error("shape: masked model: originals/positions length mismatch");
      tokens.insert(tokens.end(), in.tokens.begin(), in.tokens.end());
      segments.insert(segments.end(), in.segments.begin(), in.segments.end());
      mpos.insert(mpos.end(), in.mask_positions.begin(), in.mask_positions.end());
      morig.insert(morig.end(), in.mask_originals.begin(), in.mask_originals.end());
      label.push_back(in.label);
      tok_off.push_back(tokens.size());
      mask_off.push_back(mpos.size());
    }
    const hp_batch b{batch.size(), tok_off.data(), tokens.data(), segments.data(), mask_off.data(),
                     mpos.data(), morig.data(), label.data()};
    check(hp_engine_stage_batch(h_, &b));
    hp_round_out o{};
    check(hp_engine_round(h_, dummy ? 1 : 0, lr, &o));
    if (!o.updated) return std::nullopt;
    in_group_ = false;
    StepReport r;
    r.step = o.step;
    r.loss = o.loss;
    r.weight = o.weight;
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - group_start_).count();
    if (comm_) {  // the per-rank seconds reach the master (group_.gather_scalars)
      std::vector<double> all(static_cast<size_t>(comm_->world()));
      check(hp_pg_gather_scalars(comm_->handle(), r.seconds, all.data()));
      if (comm_->rank() == 0) r.rank_seconds = std::move(all);
    } else {
      r.rank_seconds = {r.seconds};
    }
    return r;
  }

 private:
  hp_engine* h_ = nullptr;
  uint64_t n_;
  Communicator* comm_ = nullptr;
  bool in_group_ = false;
  std::chrono::steady_clock::time_point group_start_{};
};

}  // namespace hetpar::b200
