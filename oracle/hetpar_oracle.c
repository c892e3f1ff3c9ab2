/*
 * hetpar_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the integer / byte-exact parts of the reference
 * data-parallel step (arxiv/paper_2009_14783, "hetpar"), used only as the
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * Nothing in paper_2009_14783_b200/ links or calls this file.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * the reference's golden files (splitmix64 seeds 0/1/max, Fisher-Yates n=10
 * seed 42), its frozen spot values (test_rng.cpp:57-69), its batch / partition
 * cases (test_data.cpp:209-340), and against fixtures produced by the
 * reference itself compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile and tools/make_golden.py).
 *
 * Compile with -ffp-contract=off (as the reference does, CMakeLists.txt:10-12)
 * so the Adam restatement is bit-exact to kern::scalar::adam_update.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- splitmix64 (rng.hpp:15-22) --------------------------------------- */
typedef struct {
  uint64_t state;
  double spare;
  int have_spare;
} orc_rng;

static void rng_init(orc_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->have_spare = 0;
}

static uint64_t rng_next(orc_rng* r) {
  r->state += 0x9E3779B97F4A7C15ull;
  uint64_t z = r->state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* rng.hpp:25-27: top 53 bits scaled by 2^-53 */
static double rng_double(orc_rng* r) {
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:30-32 */
static double rng_double_open(orc_rng* r) {
  return (double)((rng_next(r) >> 11) + 1) * 0x1.0p-53;
}

/* rng.hpp:37-41: high 64 bits of u * n */
static uint64_t rng_bounded(orc_rng* r, uint64_t n) {
  unsigned __int128 w = (unsigned __int128)rng_next(r) * (unsigned __int128)n;
  return (uint64_t)(w >> 64);
}

/* rng.hpp:44-55: Box-Muller, one value cached */
static double rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_double_open(r);
  double u2 = rng_double(r);
  double rad = sqrt(-2.0 * log(u1));
  double a = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

void orc_splitmix_stream(uint64_t seed, uint64_t n, uint64_t* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_next(&r);
}

void orc_bounded_stream(uint64_t seed, uint64_t bound, uint64_t n,
                        uint64_t* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_bounded(&r, bound);
}

void orc_double_stream(uint64_t seed, uint64_t n, double* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_double(&r);
}

void orc_gaussian_stream(uint64_t seed, uint64_t n, double* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_gaussian(&r);
}

/* rng.hpp:74-82: Fisher-Yates over descending i with bounded(i+1) */
static void shuffle_u64(uint64_t* a, uint64_t n, orc_rng* r) {
  if (n < 2) return;
  for (uint64_t i = n - 1; i >= 1; --i) {
    uint64_t j = rng_bounded(r, i + 1);
    uint64_t t = a[i];
    a[i] = a[j];
    a[j] = t;
  }
}

void orc_shuffle_iota(uint64_t seed, uint64_t n, uint64_t* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = i;
  shuffle_u64(out, n, &r);
}

/* ---- batching (dataset.cpp:52-88) -------------------------------------
 * Returns the number of batches (>=0), or -1 when an instance exceeds
 * max_tokens (the reference throws config_error).  order[] receives the
 * shuffled global ids; sizes[b] the batch lengths, so batch b is
 * order[sum(sizes[:b]) : +sizes[b]].                                       */
int64_t orc_build_epoch_batches(const uint32_t* lens, uint64_t n,
                                uint64_t max_sentences, uint64_t max_tokens,
                                uint64_t base_seed, uint64_t epoch,
                                uint64_t* order, uint64_t* sizes) {
  if (max_tokens > 0)
    for (uint64_t i = 0; i < n; ++i)
      if (lens[i] > max_tokens) return -1;
  orc_rng r;
  rng_init(&r, base_seed + epoch); /* derived_rng: wrapping S + N */
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  shuffle_u64(order, n, &r);
  int64_t nb = 0;
  uint64_t cur = 0, cur_tokens = 0;
  for (uint64_t k = 0; k < n; ++k) {
    uint64_t len = lens[order[k]];
    int over_s = max_sentences > 0 && cur + 1 > max_sentences;
    int over_t = max_tokens > 0 && cur_tokens + len > max_tokens;
    if (cur > 0 && (over_s || over_t)) {
      sizes[nb++] = cur;
      cur = 0;
      cur_tokens = 0;
    }
    cur += 1;
    cur_tokens += len;
  }
  if (cur > 0) sizes[nb++] = cur;
  return nb;
}

/* ---- partition (dataset.cpp:90-117) ----------------------------------- */
int64_t orc_partition_for_rank(uint64_t nbatches, uint64_t world,
                               uint64_t rank, uint64_t* batch_index,
                               uint8_t* dummy) {
  if (world == 0 || rank >= world || nbatches == 0) return -1;
  uint64_t first_real = rank < nbatches ? rank : 0;
  uint64_t rounds = (nbatches + world - 1) / world;
  for (uint64_t t = 0; t < rounds; ++t) {
    uint64_t i = t * world + rank;
    if (i < nbatches) {
      batch_index[t] = i;
      dummy[t] = 0;
    } else {
      batch_index[t] = first_real;
      dummy[t] = 1;
    }
  }
  return (int64_t)rounds;
}

/* ---- synthetic MLM records (datagen.cpp:71-127, textgen.cpp:24-95) -----
 * Extension (repo, documented in DESIGN.md): max_seq_tokens > 0 truncates
 * the assembled pair BERT-style (pop from the back of the longer sentence,
 * ties pop B) BEFORE masking.  It draws no random numbers, so with
 * max_seq_tokens == 0 the stream is the reference's exactly.             */
typedef struct {
  uint64_t n;
  int64_t vocab;
  uint64_t docs, sentences_per_doc, min_words, max_words;
  double p_select, p_mask, p_random;
  uint64_t seed;
  uint64_t max_seq_tokens;
} orc_mlm_cfg;

/* Outputs: CSR over records.  tok_off[n+1], tokens/segments[tok_off[n]];
 * mask_off[n+1], mask_pos/mask_orig[mask_off[n]]; label[n].  Capacities are
 * caller-provided; returns 0, or -1 on a config error, -2 on capacity.   */
int orc_mlm_generate(const orc_mlm_cfg* c, uint64_t tok_cap, uint64_t mask_cap,
                     uint64_t* tok_off, int64_t* tokens, int64_t* segments,
                     uint64_t* mask_off, int64_t* mask_pos, int64_t* mask_orig,
                     int64_t* label) {
  if (c->vocab < 4 + 2) return -1;
  if (c->docs < 2 || c->sentences_per_doc < 2) return -1;
  if (c->min_words == 0 || c->min_words > c->max_words) return -1;
  if (c->p_mask + c->p_random > 1.0) return -1;
  orc_rng r;
  rng_init(&r, c->seed);
  const uint64_t n_words = (uint64_t)(c->vocab - 4);
  const uint64_t nsent = c->docs * c->sentences_per_doc;
  uint64_t* slen = (uint64_t*)malloc(nsent * sizeof(uint64_t));
  int64_t** sent = (int64_t**)malloc(nsent * sizeof(int64_t*));
  for (uint64_t s = 0; s < nsent; ++s) {
    uint64_t len = c->min_words + rng_bounded(&r, c->max_words - c->min_words + 1);
    slen[s] = len;
    sent[s] = (int64_t*)malloc(len * sizeof(int64_t));
    for (uint64_t w = 0; w < len; ++w)
      sent[s][w] = 4 + (int64_t)rng_bounded(&r, n_words);
  }
  int rc = 0;
  uint64_t to = 0, mo = 0;
  int64_t* buf = NULL;
  uint64_t bufcap = 0;
  tok_off[0] = 0;
  mask_off[0] = 0;
  for (uint64_t k = 0; k < c->n; ++k) {
    /* make_nsp_pair (textgen.cpp:59-81) */
    uint64_t d = rng_bounded(&r, c->docs);
    uint64_t i = rng_bounded(&r, c->sentences_per_doc - 1);
    uint64_t sa = d * c->sentences_per_doc + i, sb;
    int64_t lab;
    if (rng_double(&r) < 0.5) {
      lab = 1;
      sb = sa + 1;
    } else {
      lab = 0;
      uint64_t o = rng_bounded(&r, c->docs - 1);
      if (o >= d) ++o;
      sb = o * c->sentences_per_doc + rng_bounded(&r, c->sentences_per_doc);
    }
    uint64_t la = slen[sa], lb = slen[sb];
    if (c->max_seq_tokens > 0) {
      if (c->max_seq_tokens < 5) { rc = -1; break; }
      uint64_t budget = c->max_seq_tokens - 3;
      while (la + lb > budget) {
        if (la > lb) --la; else --lb;
      }
    }
    /* assemble_pair (textgen.cpp:83-95) */
    uint64_t n = la + lb + 3;
    if (to + n > tok_cap) { rc = -2; break; }
    if (n > bufcap) {
      bufcap = n;
      buf = (int64_t*)realloc(buf, bufcap * sizeof(int64_t));
    }
    uint64_t p = 0;
    buf[p++] = 0;
    for (uint64_t w = 0; w < la; ++w) buf[p++] = sent[sa][w];
    buf[p++] = 1;
    uint64_t first_seg = p;
    for (uint64_t w = 0; w < lb; ++w) buf[p++] = sent[sb][w];
    buf[p++] = 1;
    /* mask_tokens (textgen.cpp:24-57) */
    for (uint64_t q = 0; q < n; ++q) {
      int64_t t = buf[q];
      tokens[to + q] = t;
      segments[to + q] = q < first_seg ? 0 : 1;
      if (t < 4) continue;
      if (rng_double(&r) >= c->p_select) continue;
      if (mo + 1 > mask_cap) { rc = -2; break; }
      mask_pos[mo] = (int64_t)q;
      mask_orig[mo] = t;
      ++mo;
      double br = rng_double(&r);
      if (br < c->p_mask) {
        tokens[to + q] = 2;
      } else if (br < c->p_mask + c->p_random) {
        int64_t rr = (int64_t)rng_bounded(&r, n_words - 1);
        if (rr >= t - 4) ++rr;
        tokens[to + q] = 4 + rr;
      }
    }
    if (rc) break;
    to += n;
    tok_off[k + 1] = to;
    mask_off[k + 1] = mo;
    label[k] = lab;
  }
  free(buf);
  for (uint64_t s = 0; s < nsent; ++s) free(sent[s]);
  free(sent);
  free(slen);
  return rc;
}

/* ---- parameter init (model.hpp:171-184) -------------------------------
 * One call per parameter in canonical order, sharing one stream: U(-a, a)
 * with a = 1/sqrt(fan_in), drawn row-major; biases draw nothing.         */
typedef struct {
  orc_rng r;
} orc_init_state;

void orc_init_begin(orc_init_state* st, uint64_t seed) {
  rng_init(&st->r, seed);
}

void orc_init_param(orc_init_state* st, uint64_t count, double fan_in,
                    int is_bias, double* out) {
  if (is_bias) {
    memset(out, 0, count * sizeof(double));
    return;
  }
  double a = 1.0 / sqrt(fan_in);
  for (uint64_t i = 0; i < count; ++i) out[i] = -a + 2.0 * a * rng_double(&st->r);
}

uint64_t orc_init_state_size(void) { return sizeof(orc_init_state); }

/* ---- optimizer (kernels_scalar.cpp:71-83, optim.hpp:107-146) ---------- */
void orc_adam_update_f32(float* p, float* m, float* v, const float* g,
                         uint64_t n, float lr, float b1, float b2, float eps,
                         float c1, float c2) {
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0f - b1) * g[i];
    v[i] = b2 * v[i] + (1.0f - b2) * (g[i] * g[i]);
    float mh = m[i] * c1;
    float vh = v[i] * c2;
    p[i] = p[i] - lr * (mh / (sqrtf(vh) + eps));
  }
}

void orc_adam_update_f64(double* p, double* m, double* v, const double* g,
                         uint64_t n, double lr, double b1, double b2,
                         double eps, double c1, double c2) {
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * (g[i] * g[i]);
    double mh = m[i] * c1;
    double vh = v[i] * c2;
    p[i] = p[i] - lr * (mh / (sqrt(vh) + eps));
  }
}

void orc_sgd_update_f32(float* p, const float* g, uint64_t n, float lr) {
  for (uint64_t i = 0; i < n; ++i) p[i] = p[i] - lr * g[i];
}

/* c1, c2 as optim.hpp:120-122 computes them: in double, before the cast. */
void orc_adam_coeffs(double b1, double b2, uint64_t t, double* c1, double* c2) {
  *c1 = 1.0 / (1.0 - pow(b1, (double)t));
  *c2 = 1.0 / (1.0 - pow(b2, (double)t));
}

/* ---- FNV-1a (common.hpp:37-47) ---------------------------------------- */
uint64_t orc_fnv1a64(const uint8_t* p, uint64_t n, uint64_t h) {
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
