// A reference-style C++ caller of the drop-in layer (include/hetpar_b200/
// step_engine.hpp): the host data path always, and with argument "gpu" ten C1
// rounds through DeviceStepEngine::round (W=1, both ranks' batches merged,
// which the protocol makes equivalent to the reference's W=2 rounds).
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <vector>

#include "hetpar_b200/step_engine.hpp"

using namespace hetpar::b200;

int main(int argc, char** argv) {
  // host data path: reference golden values (rng.hpp, dataset.cpp)
  uint64_t first = 0;
  check(hp_splitmix64(0, 1, &first));
  std::vector<uint64_t> fy(10);
  check(hp_shuffle_iota(42, 10, fy.data()));
  auto plan = build_epoch_batches(std::vector<uint32_t>(5, 1), 2, 0, 42, 0);
  auto r3 = partition_for_rank(BatchPlan{0, {{0}, {1}, {2}}}, 4, 3);
  ModelSpec spec;
  spec.d_model = 128; spec.heads = 4; spec.vocab = 1000; spec.max_seq = 64; spec.label_smooth_eps = 0.1;
  auto init = init_parameters(spec, 21);
  bool config_threw = false;
  try {
    build_epoch_batches({4, 11, 2}, 0, 10, 1, 0);
  } catch (const config_error&) {
    config_threw = true;
  }
  std::printf("{\"splitmix0\": \"%016" PRIx64 "\", \"fy\": [", first);
  for (int i = 0; i < 10; ++i) std::printf("%s%" PRIu64, i ? ", " : "", fy[i]);
  std::printf("], \"sizes\": [%zu, %zu, %zu], \"r3_dummy\": %d, \"r3_index\": %" PRIu64
              ", \"nparams\": %zu, \"init0\": %.17g, \"config_threw\": %d",
              plan.batches[0].size(), plan.batches[1].size(), plan.batches[2].size(),
              (int)r3[0].dummy, r3[0].batch_index, init.size(), init[0], (int)config_threw);
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    hp_mlm_gen_desc g{160, 1000, 8, 12, 30, 30, 0.15, 0.8, 0.1, 7, 0};
    uint64_t nt = 0, nm = 0;
    check(hp_mlm_generate_size(&g, &nt, &nm));
    std::vector<uint64_t> to(161), mo(161);
    std::vector<int64_t> tok(nt), seg(nt), mp(nm), mor(nm), lab(160);
    check(hp_mlm_generate(&g, to.data(), tok.data(), seg.data(), mo.data(), mp.data(), mor.data(), lab.data()));
    std::vector<uint32_t> lens(160);
    for (int i = 0; i < 160; ++i) lens[i] = static_cast<uint32_t>(to[i + 1] - to[i]);
    auto ep = build_epoch_batches(lens, 8, 0, 21, 0);
    hp_optim_desc opt{HP_OPT_ADAM, 0.9, 0.98, 1e-9};
    hp_exec_desc ex{HP_COMPUTE_F32, HP_POLICY_SENTENCES, 0, 25.0, 1024, 16, 256, 1};
    DeviceStepEngine eng(spec, opt, ex);
    eng.set_params(init);
    std::printf(", \"losses\": [");
    for (int step = 0; step < 10; ++step) {
      Batch b;
      for (int r = 0; r < 2; ++r)
        for (uint64_t id : ep.batches[2 * step + r]) {
          Instance in;
          in.tokens.assign(tok.begin() + to[id], tok.begin() + to[id + 1]);
          in.segments.assign(seg.begin() + to[id], seg.begin() + to[id + 1]);
          in.mask_positions.assign(mp.begin() + mo[id], mp.begin() + mo[id + 1]);
          in.mask_originals.assign(mor.begin() + mo[id], mor.begin() + mo[id + 1]);
          in.label = lab[id];
          b.push_back(std::move(in));
        }
      auto rep = eng.round(b, false, 1e-3);
      std::printf("%s%.17g", step ? ", " : "", rep->loss);
    }
    std::printf("], \"digest\": \"%016" PRIx64 "\"", eng.digest());
  }
  std::printf("}\n");
  return 0;
}
