// ref_driver.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A thin repo-side driver that links the UNMODIFIED reference sources under
// /root/reference/proj (compiled in place by oracle/Makefile into
// oracle/_ref/) and dumps what the parity tests and the CPU baseline need:
//
//   gen    : generate_mlm_shards (datagen.cpp:71-127) -> read back through
//            build_index/read_global (dataset.cpp:10-50) -> CSR dump
//   plan   : build_epoch_batches + partition_for_rank (dataset.cpp:52-117)
//   train  : train_run<T> (engine.hpp:197-330) over W in-process rank threads
//            (the CLI's run_inproc, hetpar_main.cpp:95-129), final HCK1
//            checkpoint read back -> losses + final params (+ Adam m, v)
//   grads  : the first lockstep round of the same run, per rank:
//            model_forward/backward_gradients (model.hpp:260-417) -> pre-reduce
//            flat f64 gradients, loss_sum, weight (the SerialOracle pattern,
//            test_engine.cpp:87-127)
//   init   : init_parameters<double> (model.hpp:171-184) in canonical order
//   bench  : StepEngine<float>::round on W rank threads for a timed sample
//            (the CPU baseline of bench.py --impl reference)
//
// Output files are raw little-endian arrays plus a key=value manifest.
#include <atomic>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "hetpar/checkpoint.hpp"
#include "hetpar/comm.hpp"
#include "hetpar/datagen.hpp"
#include "hetpar/dataset.hpp"
#include "hetpar/engine.hpp"
#include "hetpar/loader.hpp"
#include "hetpar/model.hpp"

using namespace hetpar;
namespace fs = std::filesystem;

namespace {

using Args = std::map<std::string, std::string>;

std::string arg(const Args& a, const std::string& k, const std::string& def) {
  auto it = a.find(k);
  return it == a.end() ? def : it->second;
}
uint64_t argu(const Args& a, const std::string& k, uint64_t def) {
  auto it = a.find(k);
  return it == a.end() ? def : std::stoull(it->second);
}
double argd(const Args& a, const std::string& k, double def) {
  auto it = a.find(k);
  return it == a.end() ? def : std::stod(it->second);
}

template <class T>
void dump(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
}

MlmGenConfig gen_cfg(const Args& a) {
  MlmGenConfig g;
  g.n = argu(a, "n", 160);
  g.vocab = static_cast<int64_t>(argu(a, "vocab", 1000));
  g.docs = argu(a, "docs", 8);
  g.sentences_per_doc = argu(a, "spd", 12);
  g.min_sentence_words = argu(a, "min_words", 30);
  g.max_sentence_words = argu(a, "max_words", 30);
  g.seed = argu(a, "data_seed", 7);
  g.shards = argu(a, "shards", 4);
  return g;
}

ModelSpec model_spec(const Args& a) {
  ModelSpec s;
  std::string arch = arg(a, "arch", "masked_token_model");
  if (arch == "masked_token_model") {
    s.arch = Arch::masked_token_model;
  } else if (arch == "attention_classifier") {
    s.arch = Arch::attention_classifier;
  } else {
    throw config_error("ref_driver: unsupported arch " + arch);
  }
  s.d_model = argu(a, "d", 128);
  s.heads = argu(a, "heads", 4);
  s.vocab = argu(a, "vocab", 1000);
  s.max_seq = argu(a, "max_seq", 512);
  s.classes = argu(a, "classes", 2);
  s.with_nsp = argu(a, "nsp", 1) != 0;
  s.label_smooth_eps = argd(a, "eps_ls", 0.1);
  return s;
}

EngineConfig engine_cfg(const Args& a, const std::string& data_dir) {
  EngineConfig c;
  c.spec = model_spec(a);
  c.policy = arg(a, "policy", "sentences") == "tokens" ? WeightPolicy::tokens
                                                        : WeightPolicy::sentences;
  c.opt_kind = arg(a, "opt", "adam") == "adam" ? OptKind::adam : OptKind::sgd;
  c.beta1 = argd(a, "beta1", 0.9);
  c.beta2 = argd(a, "beta2", 0.98);
  c.eps = argd(a, "eps", 1e-9);
  c.sched.kind = SchedulerKind::fixed;
  c.sched.peak_lr = argd(a, "lr", 1e-3);
  c.seed = argu(a, "seed", 21);
  c.data_dir = data_dir;
  c.max_sentences = argu(a, "max_sentences", 8);
  c.max_tokens = argu(a, "max_tokens", 0);
  c.update_freq = argu(a, "update_freq", 1);
  c.max_steps = argu(a, "steps", 10);
  c.max_epochs = 0;
  c.check_interval = 100;
  return c;
}

int cmd_gen(const Args& a) {
  std::string out = arg(a, "out", "gen_out");
  fs::create_directories(out);
  std::string data = out + "/shards";
  fs::remove_all(data);
  generate_mlm_shards(data, gen_cfg(a));
  auto idx = build_index(list_shards(data));
  auto lens = global_token_lengths(idx);
  std::vector<uint64_t> tok_off{0}, mask_off{0};
  std::vector<int64_t> tokens, segs, mpos, morig, label;
  for (uint64_t g = 0; g < idx.total; ++g) {
    Instance in = instance_from_record(idx.shards[0]->schema(), read_global(idx, g),
                                       lens[g]);
    tokens.insert(tokens.end(), in.tokens.begin(), in.tokens.end());
    segs.insert(segs.end(), in.segments.begin(), in.segments.end());
    mpos.insert(mpos.end(), in.mask_positions.begin(), in.mask_positions.end());
    morig.insert(morig.end(), in.mask_originals.begin(), in.mask_originals.end());
    label.push_back(in.label);
    tok_off.push_back(tokens.size());
    mask_off.push_back(mpos.size());
  }
  dump(out + "/tok_off.u64", tok_off);
  dump(out + "/tokens.i64", tokens);
  dump(out + "/segments.i64", segs);
  dump(out + "/mask_off.u64", mask_off);
  dump(out + "/mask_pos.i64", mpos);
  dump(out + "/mask_orig.i64", morig);
  dump(out + "/label.i64", label);
  dump(out + "/lens.u32", lens);
  if (argu(a, "keep_shards", 0)) {
    // keep the reference-written HSD1 files (golden fixtures, tools/make_golden.py)
    fs::create_directories(out + "/kept_shards");
    for (const auto& f : fs::directory_iterator(data))
      fs::copy_file(f.path(), out + "/kept_shards/" + f.path().filename().string(),
                    fs::copy_options::overwrite_existing);
  }
  fs::remove_all(data);
  std::printf("records=%" PRIu64 "\n", idx.total);
  return 0;
}

int cmd_plan(const Args& a) {
  std::string out = arg(a, "out", "plan_out");
  fs::create_directories(out);
  std::vector<uint32_t> lens;
  {
    std::ifstream f(arg(a, "lens", ""), std::ios::binary);
    uint32_t x;
    while (f.read(reinterpret_cast<char*>(&x), 4)) lens.push_back(x);
  }
  auto plan = build_epoch_batches(lens, argu(a, "max_sentences", 0),
                                  argu(a, "max_tokens", 0), argu(a, "seed", 0),
                                  argu(a, "epoch", 0));
  std::vector<uint64_t> order, sizes;
  for (const auto& b : plan.batches) {
    sizes.push_back(b.size());
    order.insert(order.end(), b.begin(), b.end());
  }
  dump(out + "/order.u64", order);
  dump(out + "/sizes.u64", sizes);
  uint64_t world = argu(a, "world", 1);
  for (uint64_t r = 0; r < world; ++r) {
    auto sched = partition_for_rank(plan, world, r);
    std::vector<uint64_t> bi;
    std::vector<uint8_t> dm;
    for (const auto& rb : sched) {
      bi.push_back(rb.batch_index);
      dm.push_back(rb.dummy ? 1 : 0);
    }
    dump(out + "/rank" + std::to_string(r) + "_batch.u64", bi);
    dump(out + "/rank" + std::to_string(r) + "_dummy.u8", dm);
  }
  std::printf("batches=%zu\n", plan.batches.size());
  return 0;
}

template <class T>
int cmd_train_t(const Args& a) {
  std::string out = arg(a, "out", "train_out");
  fs::create_directories(out);
  std::string data = out + "/shards";
  fs::remove_all(data);
  generate_mlm_shards(data, gen_cfg(a));
  EngineConfig cfg = engine_cfg(a, data);
  cfg.checkpoint_dir = out + "/ckpt";
  cfg.checkpoint_interval = argu(a, "ckpt_every", 0);
  const size_t world = argu(a, "world", 2);
  auto hub = make_inproc_hub(world, 600000);
  std::vector<RunReport> reports(world);
  std::vector<std::string> errs(world);
  std::vector<std::thread> th;
  for (size_t r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        auto g = make_inproc_group(hub, r);
        reports[r] = train_run<T>(cfg, *g);
      } catch (const std::exception& e) {
        errs[r] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (size_t r = 0; r < world; ++r)
    if (!errs[r].empty()) {
      std::fprintf(stderr, "rank %zu: %s\n", r, errs[r].c_str());
      return 1;
    }
  std::vector<double> losses, weights;
  for (const auto& s : reports[0].steps) {
    losses.push_back(s.loss);
    weights.push_back(s.weight);
  }
  dump(out + "/losses.f64", losses);
  dump(out + "/weights.f64", weights);
  auto st = load_checkpoint<T>(checkpoint_final_path(cfg.checkpoint_dir));
  std::vector<T> flat, m, v;
  for (size_t i = 0; i < st.params.v.size(); ++i) {
    const auto& e = st.params.v[i];
    flat.insert(flat.end(), e.m.d.begin(), e.m.d.end());
    if (st.opt.kind == OptKind::adam) {
      m.insert(m.end(), st.opt.m[i].begin(), st.opt.m[i].end());
      v.insert(v.end(), st.opt.v[i].begin(), st.opt.v[i].end());
    }
  }
  std::string suf = sizeof(T) == 8 ? ".f64" : ".f32";
  dump(out + "/params" + suf, flat);
  dump(out + "/adam_m" + suf, m);
  dump(out + "/adam_v" + suf, v);
  fs::remove_all(data);
  if (argu(a, "keep_ckpt", 0)) {
    // keep the reference-written HCK1 files (golden fixtures, tools/make_golden.py)
    for (const auto& f : fs::directory_iterator(cfg.checkpoint_dir))
      fs::copy_file(f.path(), out + "/" + f.path().filename().string(),
                    fs::copy_options::overwrite_existing);
  }
  fs::remove_all(cfg.checkpoint_dir);
  std::printf("steps=%zu final_loss=%.17g params=%zu\n", losses.size(),
              losses.empty() ? 0.0 : losses.back(), flat.size());
  return 0;
}

int cmd_grads(const Args& a) {
  // First lockstep round of the run `train` performs, per rank, in f64.
  std::string out = arg(a, "out", "grads_out");
  fs::create_directories(out);
  std::string data = out + "/shards";
  fs::remove_all(data);
  generate_mlm_shards(data, gen_cfg(a));
  EngineConfig cfg = engine_cfg(a, data);
  const size_t world = argu(a, "world", 2);
  auto idx = build_index(list_shards(data));
  auto lens = global_token_lengths(idx);
  const auto& schema = idx.shards.at(0)->schema();
  auto plan = build_epoch_batches(lens, cfg.max_sentences, cfg.max_tokens,
                                  cfg.seed, 0);
  auto rng = derived_rng(cfg.seed, 0);
  auto params = init_parameters<double>(cfg.spec, rng);
  for (size_t r = 0; r < world; ++r) {
    auto sched = partition_for_rank(plan, world, r);
    const auto& ids = plan.batches.at(sched.at(0).batch_index);
    Batch b;
    for (uint64_t g : ids)
      b.push_back(instance_from_record(schema, read_global(idx, g), lens[g]));
    auto fr = model_forward(cfg.spec, params, b, cfg.policy);
    double lw[2] = {fr.loss_sum, fr.weight};
    auto g = backward_gradients(fr, params);
    dump(out + "/rank" + std::to_string(r) + "_grads.f64", g);
    dump(out + "/rank" + std::to_string(r) + "_lw.f64",
         std::vector<double>(lw, lw + 2));
    dump(out + "/rank" + std::to_string(r) + "_ids.u64", ids);
  }
  fs::remove_all(data);
  return 0;
}

int cmd_init(const Args& a) {
  std::string out = arg(a, "out", "init_out");
  fs::create_directories(out);
  ModelSpec spec = model_spec(a);
  auto rng = derived_rng(argu(a, "seed", 21), 0);
  auto p = init_parameters<double>(spec, rng);
  std::vector<double> flat;
  std::ofstream names(out + "/shapes.txt");
  for (const auto& sh : param_shapes(spec))
    names << sh.name << " " << sh.rows << " " << sh.cols << " " << sh.row_table
          << " " << sh.bias << "\n";
  for (const auto& e : p.v) flat.insert(flat.end(), e.m.d.begin(), e.m.d.end());
  dump(out + "/params.f64", flat);
  std::printf("params=%zu digest=%016" PRIx64 "\n", flat.size(),
              params_digest(p));
  return 0;
}

// CPU baseline: `rounds` lockstep rounds of StepEngine<float>::round on
// `world` rank threads, each rank training on its own batch of `batch`
// synthetic sequences of `seq` tokens.  Prints samples/s over the timed
// rounds (after one untimed warm-up round).
int cmd_bench(const Args& a) {
  ModelSpec spec = model_spec(a);
  const size_t world = argu(a, "world", 1);
  const size_t bsz = argu(a, "batch", 4);
  const size_t seq = argu(a, "seq", 128);
  const size_t rounds = argu(a, "rounds", 1);
  SeededRng drng(argu(a, "data_seed", 7));
  std::vector<Batch> batches(world);
  for (size_t r = 0; r < world; ++r)
    for (size_t i = 0; i < bsz; ++i) {
      Instance in;
      for (size_t t = 0; t < seq; ++t) {
        in.tokens.push_back(t == 0 ? 0 : 4 + static_cast<int64_t>(drng.bounded(spec.vocab - 4)));
        in.segments.push_back(t < seq / 2 ? 0 : 1);
      }
      for (size_t t = 1; t < seq; t += 7) {
        in.mask_positions.push_back(static_cast<int64_t>(t));
        in.mask_originals.push_back(4 + static_cast<int64_t>(drng.bounded(spec.vocab - 4)));
      }
      in.label = static_cast<int64_t>(drng.bounded(2));
      in.token_length = static_cast<int64_t>(seq);
      batches[r].push_back(std::move(in));
    }
  auto hub = make_inproc_hub(world, 3600000);
  std::vector<double> secs(world, 0.0);
  std::vector<std::string> errs(world);
  std::vector<std::thread> th;
  for (size_t r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        auto g = make_inproc_group(hub, r);
        TrainState<float> st;
        st.spec = spec;
        auto rng = derived_rng(21, 0);
        st.params = init_parameters<float>(spec, rng);
        st.opt = Optimizer<float>::make_adam(st.params, 0.9, 0.98, 1e-9);
        st.sched.kind = SchedulerKind::fixed;
        st.sched.peak_lr = 1e-4;
        st.world = world;
        st.rank = r;
        st.update_freq = 1;
        StepEngine<float> eng(st, *g, 1000000, false);
        if (argu(a, "warmup", 1)) eng.round(batches[r], false);
        g->barrier();
        auto t0 = std::chrono::steady_clock::now();
        for (size_t k = 0; k < rounds; ++k) eng.round(batches[r], false);
        g->barrier();
        secs[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      } catch (const std::exception& e) {
        errs[r] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (size_t r = 0; r < world; ++r)
    if (!errs[r].empty()) {
      std::fprintf(stderr, "rank %zu: %s\n", r, errs[r].c_str());
      return 1;
    }
  double s = 0;
  for (double x : secs) s = std::max(s, x);
  double samples = static_cast<double>(world * bsz * rounds);
  std::printf("{\"seconds\": %.6f, \"samples\": %.0f, \"samples_per_s\": %.6f, "
              "\"world\": %zu, \"batch\": %zu, \"seq\": %zu, \"rounds\": %zu}\n",
              s, samples, samples / s, world, bsz, seq, rounds);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: hetpar_ref {gen|plan|train|grads|init|bench} key=value...\n");
    return 2;
  }
  Args a;
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    auto eq = s.find('=');
    if (eq == std::string::npos) {
      std::fprintf(stderr, "bad arg %s\n", s.c_str());
      return 2;
    }
    a[s.substr(0, eq)] = s.substr(eq + 1);
  }
  std::string cmd = argv[1];
  try {
    if (cmd == "gen") return cmd_gen(a);
    if (cmd == "plan") return cmd_plan(a);
    if (cmd == "train")
      return arg(a, "dtype", "f64") == "f32" ? cmd_train_t<float>(a)
                                             : cmd_train_t<double>(a);
    if (cmd == "grads") return cmd_grads(a);
    if (cmd == "init") return cmd_init(a);
    if (cmd == "bench") return cmd_bench(a);
  } catch (const config_error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
