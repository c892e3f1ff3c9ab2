// HCK1 checkpoints (reference src/checkpoint.cpp:165-302) on the host, byte
// compatible with the reference writer, plus the resume fast-forward of
// train_run (include/hetpar/engine.hpp:211-245).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hetpar_b200.h"

namespace hp {

// Serialise one f32 checkpoint.  params / m / v are the flat canonical
// vectors (param_table order); m and v are written only for Adam.
std::vector<uint8_t> hck1_serialize(const hp_model_desc& m, const hp_ckpt_desc& c,
                                    const float* params, const float* adam_m,
                                    const float* adam_v);
// Parse + validate (magic, digest, version, policy, f32 dtype, parameter
// names and shapes against the model the spec block describes).  Payload
// pointers may be null (metadata only); n = their capacity in elements.
void hck1_parse(const std::vector<uint8_t>& bytes, hp_model_desc* m, hp_ckpt_desc* c,
                float* params, float* adam_m, float* adam_v, uint64_t n);

std::vector<uint8_t> read_file(const std::string& path);
void write_file_atomic(const std::string& path, const std::vector<uint8_t>& bytes);

// Epoch and rounds to skip for a run resumed after `step` updates
// (P updates consumed exactly P*K lockstep rounds; engine.hpp:225-244).
void resume_position(const std::vector<uint32_t>& lens, uint64_t max_sentences, uint64_t max_tokens,
                     uint64_t seed, uint64_t world, uint64_t update_freq, uint64_t step,
                     uint64_t* epoch, uint64_t* skip_rounds);

}  // namespace hp
