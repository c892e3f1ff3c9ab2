// Host data path: deterministic indexing, synthetic records, parameter table.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hetpar_b200.h"

namespace hp {

// SeededRng (include/hetpar/rng.hpp:11-70).
struct SplitMix {
  uint64_t state;
  explicit SplitMix(uint64_t s) : state(s) {}
  uint64_t next() {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t bounded(uint64_t n) {
    unsigned __int128 w = static_cast<unsigned __int128>(next()) * n;
    return static_cast<uint64_t>(w >> 64);
  }
};

void shuffle_u64(std::vector<uint64_t>& a, SplitMix& r);

struct Plan {
  std::vector<uint64_t> order;
  std::vector<uint64_t> sizes;
};
Plan build_epoch_batches(const uint32_t* lens, uint64_t n, uint64_t max_sentences,
                         uint64_t max_tokens, uint64_t base_seed, uint64_t epoch);

struct RankRound {
  uint64_t batch_index;
  bool dummy;
};
std::vector<RankRound> partition_for_rank(uint64_t nbatches, uint64_t world,
                                          uint64_t rank);

struct MlmRecords {
  std::vector<uint64_t> tok_off{0}, mask_off{0};
  std::vector<int64_t> tokens, segments, mask_pos, mask_orig, label;
};
MlmRecords mlm_generate(const hp_mlm_gen_desc& d);
MlmRecords pairs_generate(const hp_pair_gen_desc& d);  // seq2seq extension

// Parameter table (model.hpp:91-142 + the bert_encoder extension).
struct ParamEntry {
  std::string name;
  uint64_t rows, cols, offset;
  int kind;  // HP_PARAM_*
  uint64_t size() const { return rows * cols; }
};
void validate_model(const hp_model_desc& m);
std::vector<ParamEntry> param_table(const hp_model_desc& m);
std::vector<double> init_parameters(const hp_model_desc& m, uint64_t seed);

struct Bucket {
  uint64_t lo, hi;          // flat range
  uint64_t first_param;     // param index range [first_param, last_param]
  uint64_t last_param;
};
std::vector<Bucket> bucket_plan(const std::vector<ParamEntry>& t, double bucket_mb);

}  // namespace hp
