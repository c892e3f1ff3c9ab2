// dropin_demo.cpp -- TEST INFRASTRUCTURE (built by oracle/Makefile `dropin`
// against the reference's own headers and objects under /root/reference/proj,
// linked with libhetpar_b200.so).
//
// The reference's own round loop -- train_run's (engine.hpp:274-310): epoch
// plan, rank schedule, BatchLoader, instance_from_record, engine.round(batch,
// lb.dummy) until max_steps -- run twice over the same shards and the same
// TrainState, once with the reference's hetpar::StepEngine<float> (CPU, an
// in-process ProcessGroup of world 1) and once with the drop-in
// hetpar::b200::StepEngine<float> (B200, an NcclProcessGroup formed over that
// same in-process group).  Prints one JSON line: both loss trajectories, the
// final TrainState parameter difference, steps, Adam t and a checkpoint
// round trip of the device-backed TrainState through the reference's own
// save_checkpoint / load_checkpoint.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <string>
#include <vector>

#include "hetpar/checkpoint.hpp"
#include "hetpar/comm.hpp"
#include "hetpar/datagen.hpp"
#include "hetpar/dataset.hpp"
#include "hetpar/engine.hpp"
#include "hetpar/loader.hpp"
#include "hetpar/model.hpp"
#include "hetpar_b200/reference_dropin.hpp"

using namespace hetpar;
namespace fs = std::filesystem;

namespace {

TrainState<float> make_state(const ModelSpec& spec) {
  TrainState<float> st;
  st.spec = spec;
  st.policy = WeightPolicy::sentences;
  st.sched.kind = SchedulerKind::fixed;
  st.sched.peak_lr = 1e-3;
  st.seed = 21;
  st.world = 1;
  st.update_freq = 2;  // W x K: one rank at K = 2 is the reference's W = 2 run
  auto rng = derived_rng(st.seed, 0);
  st.params = init_parameters<float>(spec, rng);
  st.opt = Optimizer<float>::make_adam(st.params, 0.9, 0.98, 1e-9);
  return st;
}

// train_run's epoch / round loop (engine.hpp:280-310), generic in the engine
template <class Engine>
std::vector<double> run_rounds(Engine& engine, TrainState<float>& st, const DatasetIndex& index,
                               const std::vector<uint32_t>& lens, uint64_t max_steps) {
  const auto& schema = index.shards.at(0)->schema();
  std::vector<double> losses;
  while (st.step < max_steps) {
    auto plan = build_epoch_batches(lens, 8, 0, st.seed, st.epoch);
    auto schedule = partition_for_rank(plan, 1, 0);
    BatchLoader loader(index, plan, schedule, LoaderOptions{});
    LoadedBatch lb;
    while (loader.next(lb)) {
      const auto& global_ids = plan.batches.at(lb.batch_index);
      Batch batch;
      for (size_t i = 0; i < lb.records.size(); ++i)
        batch.push_back(instance_from_record(schema, lb.records[i], lens[global_ids[i]]));
      auto rep = engine.round(batch, lb.dummy);
      if (!rep) continue;
      losses.push_back(rep->loss);
      if (st.step >= max_steps) break;
    }
    if (st.step < max_steps) ++st.epoch;
  }
  return losses;
}

double rel_norm(const TrainState<float>& a, const TrainState<float>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.params.v.size(); ++i)
    for (size_t j = 0; j < a.params.v[i].m.d.size(); ++j) {
      const double x = a.params.v[i].m.d[j], y = b.params.v[i].m.d[j];
      num += (x - y) * (x - y);
      den += y * y;
    }
  return std::sqrt(num / den);
}

void print_list(const char* key, const std::vector<double>& v) {
  std::printf("\"%s\": [", key);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]");
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "dropin_out";
  fs::remove_all(dir);
  fs::create_directories(dir);
  MlmGenConfig g;  // the C1 data: 160 records, 30-word sentences
  g.n = 160;
  g.vocab = 1000;
  g.min_sentence_words = 30;
  g.max_sentence_words = 30;
  g.seed = 7;
  g.shards = 4;
  generate_mlm_shards(dir + "/shards", g);
  auto index = build_index(list_shards(dir + "/shards"));
  auto lens = global_token_lengths(index);
  ModelSpec spec;
  spec.arch = Arch::masked_token_model;
  spec.d_model = 128;
  spec.heads = 4;
  spec.vocab = 1000;
  spec.max_seq = 64;
  spec.with_nsp = true;
  spec.label_smooth_eps = 0.1;

  auto hub = make_inproc_hub(1, 30000);
  auto group = make_inproc_group(hub, 0);

  TrainState<float> st_ref = make_state(spec);
  std::vector<double> ref_losses;
  {
    hetpar::StepEngine<float> engine(st_ref, *group, 100, false);
    ref_losses = run_rounds(engine, st_ref, index, lens, 10);
  }
  TrainState<float> st_dev = make_state(spec);
  std::vector<double> dev_losses;
  uint64_t pending = 0;
  {
    hetpar::b200::NcclProcessGroup nccl(*group, 0);
    hetpar::b200::StepEngine<float> engine(st_dev, nccl, 100, /*debug=*/true);
    dev_losses = run_rounds(engine, st_dev, index, lens, 10);
    pending = engine.pending_rounds();
  }
  // the device-backed TrainState through the reference's own checkpoint code
  save_checkpoint(st_dev, dir + "/dev.hck");
  TrainState<float> back = load_checkpoint<float>(dir + "/dev.hck");
  std::printf("{");
  print_list("ref_losses", ref_losses);
  std::printf(", ");
  print_list("dev_losses", dev_losses);
  std::printf(", \"params_rel\": %.6g, \"ref_step\": %llu, \"dev_step\": %llu, \"ref_t\": %llu, "
              "\"dev_t\": %llu, \"pending\": %llu, \"ckpt_rel\": %.6g, \"ckpt_step\": %llu}\n",
              rel_norm(st_dev, st_ref), (unsigned long long)st_ref.step, (unsigned long long)st_dev.step,
              (unsigned long long)st_ref.opt.t, (unsigned long long)st_dev.opt.t,
              (unsigned long long)pending, rel_norm(back, st_dev), (unsigned long long)back.step);
  fs::remove_all(dir + "/shards");
  return 0;
}
