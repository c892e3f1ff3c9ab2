// Host data path of the DP step, bit-exact with the reference:
//   * epoch plan + rank schedule   (src/dataset.cpp:52-117)
//   * synthetic MLM record stream   (src/datagen.cpp:71-127, src/textgen.cpp:24-95)
//   * canonical parameter table / init / bucket plan (model.hpp:91-184,
//     SURVEY §8e bucket contract)
// These run once per epoch / run on the host; the per-round output (one rank
// batch) is staged to HBM by the engine.
#include "hostdata.h"

#include <cmath>
#include <numeric>

#include "hp_common.h"

namespace hp {

void shuffle_u64(std::vector<uint64_t>& a, SplitMix& r) {
  // Fisher-Yates, descending i, j = bounded(i + 1)   (rng.hpp:74-82)
  for (size_t i = a.size(); i-- > 1;) {
    uint64_t j = r.bounded(i + 1);
    std::swap(a[i], a[j]);
  }
}

Plan build_epoch_batches(const uint32_t* lens, uint64_t n, uint64_t max_sentences,
                         uint64_t max_tokens, uint64_t base_seed, uint64_t epoch) {
  if (max_tokens > 0)
    for (uint64_t i = 0; i < n; ++i)
      if (lens[i] > max_tokens)
        fail(HP_ECONFIG, "instance " + std::to_string(i) + " has " +
                             std::to_string(lens[i]) +
                             " tokens, exceeding max_tokens " +
                             std::to_string(max_tokens));
  Plan p;
  p.order.resize(n);
  std::iota(p.order.begin(), p.order.end(), uint64_t{0});
  SplitMix r(base_seed + epoch);  // derived_rng(S, N): wrapping add
  shuffle_u64(p.order, r);
  // Greedy close-on-overflow packing in shuffled order.
  uint64_t in_batch = 0, tok = 0;
  for (uint64_t g : p.order) {
    const uint64_t len = lens[g];
    const bool full = (max_sentences && in_batch + 1 > max_sentences) ||
                      (max_tokens && tok + len > max_tokens);
    if (in_batch && full) {
      p.sizes.push_back(in_batch);
      in_batch = tok = 0;
    }
    ++in_batch;
    tok += len;
  }
  if (in_batch) p.sizes.push_back(in_batch);
  return p;
}

std::vector<RankRound> partition_for_rank(uint64_t nbatches, uint64_t world,
                                          uint64_t rank) {
  if (world == 0) fail(HP_ECONFIG, "world_size must be >= 1");
  if (rank >= world)
    fail(HP_ECONFIG, "rank " + std::to_string(rank) +
                         " out of range for world_size " + std::to_string(world));
  if (nbatches == 0) fail(HP_ECONFIG, "epoch has no batches to partition");
  const uint64_t rounds = (nbatches + world - 1) / world;
  const uint64_t fallback = rank < nbatches ? rank : 0;
  std::vector<RankRound> s(rounds);
  for (uint64_t t = 0; t < rounds; ++t) {
    const uint64_t i = t * world + rank;
    s[t] = i < nbatches ? RankRound{i, false} : RankRound{fallback, true};
  }
  return s;
}

MlmRecords mlm_generate(const hp_mlm_gen_desc& d) {
  constexpr int64_t kCls = 0, kSep = 1, kMask = 2, kFirstWord = 4;
  if (d.vocab < kFirstWord + 2) fail(HP_ECONFIG, "datagen: mlm vocab needs >= 2 word ids");
  if (d.docs < 2 || d.sentences_per_doc < 2)
    fail(HP_ECONFIG, "datagen: corpus needs >= 2 documents of >= 2 sentences");
  if (d.min_words == 0 || d.min_words > d.max_words)
    fail(HP_ECONFIG, "datagen: bad sentence length range");
  if (d.p_mask + d.p_random > 1.0)
    fail(HP_ECONFIG, "mask_tokens: branch probabilities exceed 1");
  if (d.max_seq_tokens != 0 && d.max_seq_tokens < 5)
    fail(HP_ECONFIG, "datagen: max_seq_tokens must be 0 or >= 5");

  SplitMix r(d.seed);
  const uint64_t n_words = static_cast<uint64_t>(d.vocab - kFirstWord);
  // Corpus as one flat word array + sentence offsets (docs x spd sentences).
  const uint64_t nsent = d.docs * d.sentences_per_doc;
  std::vector<uint64_t> soff(nsent + 1, 0);
  std::vector<int64_t> words;
  for (uint64_t s = 0; s < nsent; ++s) {
    const uint64_t len = d.min_words + r.bounded(d.max_words - d.min_words + 1);
    for (uint64_t w = 0; w < len; ++w)
      words.push_back(kFirstWord + static_cast<int64_t>(r.bounded(n_words)));
    soff[s + 1] = words.size();
  }

  MlmRecords out;
  std::vector<int64_t> seq;
  for (uint64_t k = 0; k < d.n; ++k) {
    // make_nsp_pair: label 1 = true successor, 0 = random other document.
    const uint64_t doc = r.bounded(d.docs);
    const uint64_t i = r.bounded(d.sentences_per_doc - 1);
    const uint64_t a = doc * d.sentences_per_doc + i;
    uint64_t b;
    int64_t label;
    if (r.next_double() < 0.5) {
      label = 1;
      b = a + 1;
    } else {
      label = 0;
      uint64_t o = r.bounded(d.docs - 1);
      o += (o >= doc);
      b = o * d.sentences_per_doc + r.bounded(d.sentences_per_doc);
    }
    uint64_t la = soff[a + 1] - soff[a], lb = soff[b + 1] - soff[b];
    if (d.max_seq_tokens) {  // extension: truncate_seq_pair, back pops
      while (la + lb + 3 > d.max_seq_tokens) (la > lb ? la : lb) -= 1;
    }
    // assemble_pair: [CLS] A [SEP] B [SEP]; segment 0 through the first SEP.
    seq.clear();
    seq.push_back(kCls);
    seq.insert(seq.end(), words.begin() + soff[a], words.begin() + soff[a] + la);
    seq.push_back(kSep);
    const size_t seg1_start = seq.size();
    seq.insert(seq.end(), words.begin() + soff[b], words.begin() + soff[b] + lb);
    seq.push_back(kSep);
    // mask_tokens: per eligible position one selection draw, then the branch
    // draw and (random branch) the replacement draw.
    for (size_t q = 0; q < seq.size(); ++q) {
      const int64_t orig = seq[q];
      int64_t t = orig;
      if (orig >= kFirstWord && r.next_double() < d.p_select) {
        out.mask_pos.push_back(static_cast<int64_t>(q));
        out.mask_orig.push_back(orig);
        const double br = r.next_double();
        if (br < d.p_mask) {
          t = kMask;
        } else if (br < d.p_mask + d.p_random) {
          if (n_words < 2) fail(HP_ECONFIG, "mask_tokens: random branch needs >= 2 words");
          int64_t rr = static_cast<int64_t>(r.bounded(n_words - 1));
          rr += (rr >= orig - kFirstWord);
          t = kFirstWord + rr;
        }
      }
      out.tokens.push_back(t);
      out.segments.push_back(q < seg1_start ? 0 : 1);
    }
    out.label.push_back(label);
    out.tok_off.push_back(out.tokens.size());
    out.mask_off.push_back(out.mask_pos.size());
  }
  return out;
}

MlmRecords pairs_generate(const hp_pair_gen_desc& d) {
  constexpr int64_t kFirstWord = 4;
  if (d.vocab < kFirstWord + 2) fail(HP_ECONFIG, "datagen: pair vocab needs >= 2 word ids");
  if (d.min_len == 0 || d.min_len > d.max_len) fail(HP_ECONFIG, "datagen: bad pair length range");
  SplitMix r(d.seed);
  const uint64_t n_words = static_cast<uint64_t>(d.vocab - kFirstWord);
  MlmRecords out;
  for (uint64_t k = 0; k < d.n; ++k) {
    const uint64_t ls = d.min_len + r.bounded(d.max_len - d.min_len + 1);
    const uint64_t lt = d.min_len + r.bounded(d.max_len - d.min_len + 1);
    for (uint64_t i = 0; i < ls + lt; ++i) {
      out.tokens.push_back(kFirstWord + static_cast<int64_t>(r.bounded(n_words)));
      out.segments.push_back(i < ls ? 0 : 1);
    }
    out.label.push_back(0);
    out.tok_off.push_back(out.tokens.size());
    out.mask_off.push_back(0);
  }
  return out;
}

void validate_model(const hp_model_desc& m) {
  if (!(m.label_smooth_eps >= 0.0 && m.label_smooth_eps < 1.0))
    fail(HP_ECONFIG, "label_smooth_eps outside [0,1)");
  if (m.arch != HP_ARCH_MASKED_TOKEN_MODEL && m.arch != HP_ARCH_BERT_ENCODER &&
      m.arch != HP_ARCH_SEQ2SEQ)
    fail(HP_ECONFIG, "unsupported architecture id " + std::to_string(m.arch));
  if (m.d_model == 0 || m.vocab == 0 || m.max_seq == 0)
    fail(HP_ECONFIG, "masked model needs d_model/vocab/max_seq");
  if (m.heads == 0 || m.d_model % m.heads != 0)
    fail(HP_ECONFIG, "d_model not divisible by heads");
  if (m.d_model % 2 != 0) fail(HP_ECONFIG, "d_model must be even");
  if (m.arch == HP_ARCH_BERT_ENCODER && (m.layers == 0 || m.d_ff == 0))
    fail(HP_ECONFIG, "bert_encoder needs layers >= 1 and d_ff >= 1");
  if (m.arch == HP_ARCH_SEQ2SEQ && (m.layers == 0 || m.d_ff == 0))
    fail(HP_ECONFIG, "transformer_seq2seq needs layers >= 1 and d_ff >= 1");
}

std::vector<ParamEntry> param_table(const hp_model_desc& m) {
  validate_model(m);
  std::vector<ParamEntry> t;
  uint64_t off = 0;
  auto add = [&](std::string n, uint64_t r, uint64_t c, int kind) {
    t.push_back({std::move(n), r, c, off, kind});
    off += r * c;
  };
  const uint64_t d = m.d_model, dk = m.d_model / m.heads;
  auto attention = [&](const std::string& p) {
    for (const char* k : {"wq.", "wk.", "wv."})
      for (uint64_t i = 0; i < m.heads; ++i)
        add(p + k + std::to_string(i), d, dk, HP_PARAM_WEIGHT);
    add(p + "wo", d, d, HP_PARAM_WEIGHT);
  };
  auto ffn = [&](const std::string& p, const char* ln) {
    add(p + "ffn.w1", d, m.d_ff, HP_PARAM_WEIGHT);
    add(p + "ffn.b1", 1, m.d_ff, HP_PARAM_BIAS);
    add(p + "ffn.w2", m.d_ff, d, HP_PARAM_WEIGHT);
    add(p + "ffn.b2", 1, d, HP_PARAM_BIAS);
    add(p + ln + ".g", 1, d, HP_PARAM_GAIN);
    add(p + ln + ".b", 1, d, HP_PARAM_BIAS);
  };
  if (m.arch == HP_ARCH_SEQ2SEQ) {
    // one table for the encoder / decoder inputs and the output projection;
    // encoder blocks as the bert_encoder layer, decoder blocks add the
    // cross-attention projections cq / ck / cv / co (+ cbo, ln2) between the
    // self-attention and the FFN (whose LayerNorm becomes ln3)
    add("embed", m.vocab, d, HP_PARAM_TABLE);
    for (uint64_t l = 0; l < m.layers; ++l) {
      const std::string p = "enc" + std::to_string(l) + ".";
      attention(p);
      add(p + "bo", 1, d, HP_PARAM_BIAS);
      add(p + "ln1.g", 1, d, HP_PARAM_GAIN);
      add(p + "ln1.b", 1, d, HP_PARAM_BIAS);
      ffn(p, "ln2");
    }
    for (uint64_t l = 0; l < m.layers; ++l) {
      const std::string p = "dec" + std::to_string(l) + ".";
      attention(p);
      add(p + "bo", 1, d, HP_PARAM_BIAS);
      add(p + "ln1.g", 1, d, HP_PARAM_GAIN);
      add(p + "ln1.b", 1, d, HP_PARAM_BIAS);
      for (const char* k : {"cq.", "ck.", "cv."})
        for (uint64_t i = 0; i < m.heads; ++i)
          add(p + k + std::to_string(i), d, dk, HP_PARAM_WEIGHT);
      add(p + "co", d, d, HP_PARAM_WEIGHT);
      add(p + "cbo", 1, d, HP_PARAM_BIAS);
      add(p + "ln2.g", 1, d, HP_PARAM_GAIN);
      add(p + "ln2.b", 1, d, HP_PARAM_BIAS);
      ffn(p, "ln3");
    }
    return t;
  }
  add("embed", m.vocab, d, HP_PARAM_TABLE);
  add("seg0", 1, d, HP_PARAM_TABLE);
  add("seg1", 1, d, HP_PARAM_TABLE);
  if (m.arch == HP_ARCH_MASKED_TOKEN_MODEL) {
    attention("");
  } else {
    add("emb_ln.g", 1, d, HP_PARAM_GAIN);
    add("emb_ln.b", 1, d, HP_PARAM_BIAS);
    for (uint64_t l = 0; l < m.layers; ++l) {
      const std::string p = "layer" + std::to_string(l) + ".";
      attention(p);
      add(p + "bo", 1, d, HP_PARAM_BIAS);
      add(p + "ln1.g", 1, d, HP_PARAM_GAIN);
      add(p + "ln1.b", 1, d, HP_PARAM_BIAS);
      add(p + "ffn.w1", d, m.d_ff, HP_PARAM_WEIGHT);
      add(p + "ffn.b1", 1, m.d_ff, HP_PARAM_BIAS);
      add(p + "ffn.w2", m.d_ff, d, HP_PARAM_WEIGHT);
      add(p + "ffn.b2", 1, d, HP_PARAM_BIAS);
      add(p + "ln2.g", 1, d, HP_PARAM_GAIN);
      add(p + "ln2.b", 1, d, HP_PARAM_BIAS);
    }
  }
  add("mlm.w", d, m.vocab, HP_PARAM_WEIGHT);
  add("mlm.b", 1, m.vocab, HP_PARAM_BIAS);
  if (m.with_nsp) {
    add("nsp.w", d, 2, HP_PARAM_WEIGHT);
    add("nsp.b", 1, 2, HP_PARAM_BIAS);
  }
  return t;
}

std::vector<double> init_parameters(const hp_model_desc& m, uint64_t seed) {
  auto t = param_table(m);
  std::vector<double> out(t.empty() ? 0 : t.back().offset + t.back().size(), 0.0);
  SplitMix r(seed);  // derived_rng(seed, 0)
  for (const auto& e : t) {
    double* p = out.data() + e.offset;
    if (e.kind == HP_PARAM_BIAS) continue;  // zeros, no draws
    if (e.kind == HP_PARAM_GAIN) {          // extension: LayerNorm gain = 1
      for (uint64_t i = 0; i < e.size(); ++i) p[i] = 1.0;
      continue;
    }
    const double fan_in = static_cast<double>(e.kind == HP_PARAM_TABLE ? e.cols : e.rows);
    const double a = 1.0 / std::sqrt(fan_in);
    for (uint64_t i = 0; i < e.size(); ++i) p[i] = -a + 2.0 * a * r.next_double();
  }
  return out;
}

std::vector<Bucket> bucket_plan(const std::vector<ParamEntry>& t, double bucket_mb) {
  if (!(bucket_mb > 0)) fail(HP_ECONFIG, "bucket_mb must be > 0");
  const double cap = bucket_mb * 1048576.0;
  std::vector<Bucket> out;
  // Reverse canonical order: the head's gradients are ready first.
  // A bucket always takes at least one parameter, then closes when the next
  // one would overflow the cap (the close-on-overflow rule of
  // build_epoch_batches, dataset.cpp:76-82).
  auto bytes_of = [&](size_t k) { return 4.0 * static_cast<double>(t[k].size()); };
  size_t i = t.size();
  while (i > 0) {
    Bucket b{0, t[i - 1].offset + t[i - 1].size(), 0, i - 1};
    double bytes = 0;
    do {
      bytes += bytes_of(--i);
    } while (i > 0 && bytes + bytes_of(i - 1) <= cap);
    b.first_param = i;
    b.lo = t[i].offset;
    out.push_back(b);
  }
  return out;
}

}  // namespace hp
