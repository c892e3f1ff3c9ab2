// HCK1 checkpoint format (reference src/checkpoint.cpp:165-302), written and
// read on the host.  Layout, little-endian:
//   "HCK1" | u16 version=1 | u64 epoch | u64 step | u64 seed | u8 policy |
//   u32 len + spec JSON | u32 count | per parameter: u16 len + name, u8 dtype
//   (1 = f32), u8 rank = 2, u32 rows, u32 cols, payload | u8 optimizer kind |
//   (Adam) u64 t, all m payloads, all v payloads | u64 FNV-1a of everything
//   before it.
// The spec block is what nlohmann::json::dump() produces for the reference's
// build_spec_json (checkpoint.cpp:54-79): object keys sorted, no whitespace,
// numbers in Grisu2 shortest round-trip form; this writer reproduces it byte
// for byte (tests/test_checkpoint.py: a reference-written file re-serialises
// identically).
#include "checkpoint.h"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>

#include "hostdata.h"
#include "hp_common.h"

namespace hp {

namespace {

constexpr char kMagic[4] = {'H', 'C', 'K', '1'};
constexpr uint16_t kVersion = 1;
constexpr uint8_t kDtypeF32 = 1;

uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

template <class T>
void put(std::vector<uint8_t>& b, T v) {
  uint8_t t[sizeof(T)];
  std::memcpy(t, &v, sizeof(T));
  b.insert(b.end(), t, t + sizeof(T));
}
void put_bytes(std::vector<uint8_t>& b, const void* p, size_t n) {
  const uint8_t* q = static_cast<const uint8_t*>(p);
  b.insert(b.end(), q, q + n);
}

// ---- JSON output in nlohmann::json::dump() form
// Shortest round-trip digits; fixed notation while the decimal point falls in
// (-4, 15] digits of the first digit (1.0 -> "1.0", 0.001 -> "0.001"), else
// "d[.ddd]e+XX" with a signed, at least two-digit exponent (1e-09).
std::string json_number(double x) {
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
  std::string sci(buf, r.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci.erase(0, 1);
  }
  const size_t e = sci.find('e');
  std::string digits;
  for (size_t i = 0; i < e; ++i)
    if (sci[i] != '.') digits += sci[i];
  const int e10 = std::stoi(sci.substr(e + 1));
  const int k = static_cast<int>(digits.size());
  const int n = e10 + 1;  // position of the decimal point after the first digit
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int ex = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  return sign + out;
}

const char* arch_name(int arch) {
  return arch == HP_ARCH_BERT_ENCODER ? "bert_encoder"
         : arch == HP_ARCH_SEQ2SEQ    ? "transformer_seq2seq"
                                      : "masked_token_model";
}
const char* sched_name(int k) { return k == 1 ? "inverse_sqrt" : k == 2 ? "linear" : "fixed"; }

// build_spec_json (checkpoint.cpp:54-79); the bert_encoder extension adds
// d_ff and encoder_layers (keys stay sorted).
std::string spec_json(const hp_model_desc& m, const hp_ckpt_desc& c) {
  const bool bert = m.arch == HP_ARCH_BERT_ENCODER || m.arch == HP_ARCH_SEQ2SEQ;
  std::string j = "{";
  j += "\"arch\":\"" + std::string(arch_name(m.arch)) + "\"";
  j += ",\"classes\":2";
  if (bert) j += ",\"d_ff\":" + std::to_string(m.d_ff);
  j += ",\"d_model\":" + std::to_string(m.d_model);
  j += ",\"dtype\":\"f32\"";
  if (bert) j += ",\"encoder_layers\":" + std::to_string(m.layers);
  j += ",\"heads\":" + std::to_string(m.heads);
  j += ",\"label_smooth_eps\":" + json_number(m.label_smooth_eps);
  j += ",\"layers\":[]";
  j += ",\"max_seq\":" + std::to_string(m.max_seq);
  j += ",\"optimizer\":{\"beta1\":" + json_number(c.beta1) + ",\"beta2\":" + json_number(c.beta2) +
       ",\"eps\":" + json_number(c.eps) + ",\"kind\":\"" +
       (c.opt_kind == HP_OPT_ADAM ? "adam" : c.opt_kind == HP_OPT_ADAMW ? "adamw" : "sgd") + "\"" +
       (c.opt_kind == HP_OPT_ADAMW ? ",\"weight_decay\":" + json_number(c.weight_decay) : std::string()) +
       "}";
  j += ",\"scheduler\":{\"d_model\":" + std::to_string(c.sched_d_model) + ",\"kind\":\"" +
       sched_name(c.sched_kind) + "\",\"peak_lr\":" + json_number(c.peak_lr) +
       ",\"total_steps\":" + std::to_string(c.total_steps) +
       ",\"warmup_steps\":" + std::to_string(c.warmup_steps) + "}";
  j += ",\"update_freq\":" + std::to_string(c.update_freq);
  j += ",\"vocab\":" + std::to_string(m.vocab);
  j += ",\"with_nsp\":" + std::string(m.with_nsp ? "true" : "false");
  j += ",\"world_size\":" + std::to_string(c.world_size);
  j += "}";
  return j;
}

// ---- minimal JSON reader (objects, arrays, strings, numbers, booleans)
struct JVal {
  enum Kind { NUM, STR, BOOL, ARR, OBJ, NUL } kind = NUL;
  double num = 0;
  std::string str;
  bool b = false;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};
struct JParser {
  const std::string& s;
  size_t i = 0;
  [[noreturn]] void bad() { fail(HP_EIO, "checkpoint spec block is not valid json"); }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
  }
  JVal value() {
    ws();
    if (i >= s.size()) bad();
    JVal v;
    const char c = s[i];
    if (c == '{') {
      v.kind = JVal::OBJ;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') { ++i; return v; }
      for (;;) {
        ws();
        JVal k = value();
        if (k.kind != JVal::STR) bad();
        ws();
        if (i >= s.size() || s[i] != ':') bad();
        ++i;
        v.obj[k.str] = value();
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == '}') { ++i; return v; }
        bad();
      }
    }
    if (c == '[') {
      v.kind = JVal::ARR;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') { ++i; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == ']') { ++i; return v; }
        bad();
      }
    }
    if (c == '"') {
      v.kind = JVal::STR;
      ++i;
      while (i < s.size() && s[i] != '"') {
        if (s[i] == '\\') ++i;
        if (i < s.size()) v.str += s[i++];
      }
      if (i >= s.size()) bad();
      ++i;
      return v;
    }
    if (s.compare(i, 4, "true") == 0) { v.kind = JVal::BOOL; v.b = true; i += 4; return v; }
    if (s.compare(i, 5, "false") == 0) { v.kind = JVal::BOOL; v.b = false; i += 5; return v; }
    if (s.compare(i, 4, "null") == 0) { i += 4; return v; }
    size_t j = i;
    while (j < s.size() && std::strchr("+-0123456789.eE", s[j])) ++j;
    if (j == i) bad();
    v.kind = JVal::NUM;
    v.num = std::strtod(s.substr(i, j - i).c_str(), nullptr);
    i = j;
    return v;
  }
};
const JVal& field(const JVal& o, const char* k) {
  auto it = o.obj.find(k);
  if (o.kind != JVal::OBJ || it == o.obj.end())
    fail(HP_EIO, std::string("checkpoint spec block is missing fields: ") + k);
  return it->second;
}
uint64_t fu(const JVal& o, const char* k) { return static_cast<uint64_t>(field(o, k).num); }
double fd(const JVal& o, const char* k) { return field(o, k).num; }
std::string fs(const JVal& o, const char* k) { return field(o, k).str; }

struct Reader {
  const uint8_t* p;
  size_t n, at = 0;
  const uint8_t* raw(size_t k) {
    if (at + k > n) fail(HP_EIO, "checkpoint truncated");
    const uint8_t* q = p + at;
    at += k;
    return q;
  }
  template <class T>
  T get() {
    T v;
    std::memcpy(&v, raw(sizeof(T)), sizeof(T));
    return v;
  }
};

}  // namespace

std::vector<uint8_t> read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(HP_EIO, "cannot open " + path);
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

void write_file_atomic(const std::string& path, const std::vector<uint8_t>& bytes) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) fail(HP_EIO, "cannot write " + tmp);
    f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!f) fail(HP_EIO, "short write to " + tmp);
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) fail(HP_EIO, "cannot rename " + tmp + " to " + path);
}

std::vector<uint8_t> hck1_serialize(const hp_model_desc& m, const hp_ckpt_desc& c,
                                    const float* params, const float* adam_m,
                                    const float* adam_v) {
  validate_model(m);
  if (c.policy != HP_POLICY_SENTENCES && c.policy != HP_POLICY_TOKENS)
    fail(HP_ECONFIG, "checkpoint: invalid weight policy");
  if (c.opt_kind != HP_OPT_ADAM && c.opt_kind != HP_OPT_SGD && c.opt_kind != HP_OPT_ADAMW)
    fail(HP_ECONFIG, "checkpoint: invalid optimizer kind");
  if (c.opt_kind != HP_OPT_SGD && (!adam_m || !adam_v))
    fail(HP_ECONFIG, "checkpoint: Adam moments missing");
  const auto table = param_table(m);
  std::vector<uint8_t> b;
  put_bytes(b, kMagic, 4);
  put<uint16_t>(b, kVersion);
  put<uint64_t>(b, c.epoch);
  put<uint64_t>(b, c.step);
  put<uint64_t>(b, c.seed);
  put<uint8_t>(b, static_cast<uint8_t>(c.policy));
  const std::string js = spec_json(m, c);
  put<uint32_t>(b, static_cast<uint32_t>(js.size()));
  put_bytes(b, js.data(), js.size());
  put<uint32_t>(b, static_cast<uint32_t>(table.size()));
  for (const auto& e : table) {
    put<uint16_t>(b, static_cast<uint16_t>(e.name.size()));
    put_bytes(b, e.name.data(), e.name.size());
    put<uint8_t>(b, kDtypeF32);
    put<uint8_t>(b, 2);
    put<uint32_t>(b, static_cast<uint32_t>(e.rows));
    put<uint32_t>(b, static_cast<uint32_t>(e.cols));
    put_bytes(b, params + e.offset, e.size() * 4);
  }
  put<uint8_t>(b, static_cast<uint8_t>(c.opt_kind));
  if (c.opt_kind != HP_OPT_SGD) {
    put<uint64_t>(b, c.opt_t);
    for (const auto& e : table) put_bytes(b, adam_m + e.offset, e.size() * 4);
    for (const auto& e : table) put_bytes(b, adam_v + e.offset, e.size() * 4);
  }
  put<uint64_t>(b, fnv1a(b.data(), b.size()));
  return b;
}

void hck1_parse(const std::vector<uint8_t>& bytes, hp_model_desc* m, hp_ckpt_desc* c,
                float* params, float* adam_m, float* adam_v, uint64_t n) {
  if (bytes.size() < 4 + 2 + 8) fail(HP_EIO, "checkpoint too small to be valid");
  if (std::memcmp(bytes.data(), kMagic, 4) != 0) fail(HP_EIO, "not a checkpoint file");
  uint64_t stored;
  std::memcpy(&stored, bytes.data() + bytes.size() - 8, 8);
  if (fnv1a(bytes.data(), bytes.size() - 8) != stored)
    fail(HP_EIO, "checkpoint digest mismatch (truncated or corrupt file)");
  Reader r{bytes.data(), bytes.size() - 8};
  r.raw(4);
  if (r.get<uint16_t>() != kVersion) fail(HP_EIO, "unsupported checkpoint version");
  hp_ckpt_desc cd{};
  cd.epoch = r.get<uint64_t>();
  cd.step = r.get<uint64_t>();
  cd.seed = r.get<uint64_t>();
  cd.policy = r.get<uint8_t>();
  if (cd.policy != HP_POLICY_SENTENCES && cd.policy != HP_POLICY_TOKENS)
    fail(HP_EIO, "checkpoint carries invalid weight policy");
  const uint32_t jl = r.get<uint32_t>();
  const std::string js(reinterpret_cast<const char*>(r.raw(jl)), jl);
  JParser jp{js};
  const JVal j = jp.value();
  if (fs(j, "dtype") != "f32")
    fail(HP_ECONFIG, "checkpoint dtype is " + fs(j, "dtype") + ", the device engine keeps f32 master weights");
  hp_model_desc md{};
  const std::string arch = fs(j, "arch");
  if (arch == "masked_token_model") {
    md.arch = HP_ARCH_MASKED_TOKEN_MODEL;
  } else if (arch == "bert_encoder" || arch == "transformer_seq2seq") {
    md.arch = arch == "bert_encoder" ? HP_ARCH_BERT_ENCODER : HP_ARCH_SEQ2SEQ;
    md.layers = fu(j, "encoder_layers");
    md.d_ff = fu(j, "d_ff");
  } else {
    fail(HP_EIO, "checkpoint names unsupported architecture '" + arch + "'");
  }
  md.d_model = fu(j, "d_model");
  md.heads = fu(j, "heads");
  md.vocab = fu(j, "vocab");
  md.max_seq = fu(j, "max_seq");
  md.with_nsp = field(j, "with_nsp").b ? 1 : 0;
  md.label_smooth_eps = fd(j, "label_smooth_eps");
  cd.world_size = fu(j, "world_size");
  cd.update_freq = fu(j, "update_freq");
  const JVal& oj = field(j, "optimizer");
  cd.beta1 = fd(oj, "beta1");
  cd.beta2 = fd(oj, "beta2");
  cd.eps = fd(oj, "eps");
  const JVal& sj = field(j, "scheduler");
  const std::string sk = fs(sj, "kind");
  if (sk == "fixed") cd.sched_kind = 0;
  else if (sk == "inverse_sqrt") cd.sched_kind = 1;
  else if (sk == "linear") cd.sched_kind = 2;
  else fail(HP_EIO, "checkpoint names unknown scheduler '" + sk + "'");
  cd.peak_lr = fd(sj, "peak_lr");
  cd.sched_d_model = fu(sj, "d_model");
  cd.warmup_steps = fu(sj, "warmup_steps");
  cd.total_steps = fu(sj, "total_steps");

  const auto table = param_table(md);
  const uint32_t count = r.get<uint32_t>();
  if (count != table.size())
    fail(HP_EIO, "checkpoint has " + std::to_string(count) + " parameters, spec defines " +
                     std::to_string(table.size()));
  const uint64_t total = table.back().offset + table.back().size();
  if ((params || adam_m || adam_v) && n < total) fail(HP_ECONFIG, "checkpoint: output buffers too small");
  for (const auto& e : table) {
    const uint16_t nl = r.get<uint16_t>();
    const std::string name(reinterpret_cast<const char*>(r.raw(nl)), nl);
    const uint8_t dt = r.get<uint8_t>(), rank = r.get<uint8_t>();
    const uint32_t rows = r.get<uint32_t>(), cols = r.get<uint32_t>();
    if (dt != kDtypeF32) fail(HP_EIO, "checkpoint parameter '" + name + "' has invalid dtype");
    if (rank != 2) fail(HP_EIO, "checkpoint parameter '" + name + "' has rank " + std::to_string(rank));
    if (name != e.name || rows != e.rows || cols != e.cols)
      fail(HP_EIO, "checkpoint parameter '" + name + "' " + std::to_string(rows) + "x" +
                       std::to_string(cols) + ", spec defines '" + e.name + "' " +
                       std::to_string(e.rows) + "x" + std::to_string(e.cols));
    const uint8_t* p = r.raw(e.size() * 4);
    if (params) std::memcpy(params + e.offset, p, e.size() * 4);
  }
  cd.opt_kind = r.get<uint8_t>();
  if (cd.opt_kind != HP_OPT_SGD && cd.opt_kind != HP_OPT_ADAM && cd.opt_kind != HP_OPT_ADAMW)
    fail(HP_EIO, "checkpoint carries invalid optimizer kind");
  const std::string kname = fs(oj, "kind");
  if (kname != (cd.opt_kind == HP_OPT_ADAM ? "adam" : cd.opt_kind == HP_OPT_ADAMW ? "adamw" : "sgd"))
    fail(HP_EIO, "optimizer kind disagrees between spec block and blocks");
  if (cd.opt_kind == HP_OPT_ADAMW) cd.weight_decay = fd(oj, "weight_decay");
  if (cd.opt_kind != HP_OPT_SGD) {
    cd.opt_t = r.get<uint64_t>();
    for (const auto& e : table) {
      const uint8_t* p = r.raw(e.size() * 4);
      if (adam_m) std::memcpy(adam_m + e.offset, p, e.size() * 4);
    }
    for (const auto& e : table) {
      const uint8_t* p = r.raw(e.size() * 4);
      if (adam_v) std::memcpy(adam_v + e.offset, p, e.size() * 4);
    }
  }
  if (r.at != r.n) fail(HP_EIO, "checkpoint has trailing bytes");
  if (m) *m = md;
  if (c) *c = cd;
}

void resume_position(const std::vector<uint32_t>& lens, uint64_t max_sentences, uint64_t max_tokens,
                     uint64_t seed, uint64_t world, uint64_t update_freq, uint64_t step,
                     uint64_t* epoch, uint64_t* skip_rounds) {
  if (world == 0 || update_freq == 0) fail(HP_ECONFIG, "resume: world and update_freq must be >= 1");
  uint64_t left = step * update_freq;
  for (uint64_t e = 0;; ++e) {
    const Plan plan = build_epoch_batches(lens.data(), lens.size(), max_sentences, max_tokens, seed, e);
    if (plan.sizes.empty()) fail(HP_ECONFIG, "dataset produces no batches");
    const uint64_t rounds = (plan.sizes.size() + world - 1) / world;
    if (left < rounds) {
      *epoch = e;
      *skip_rounds = left;
      return;
    }
    left -= rounds;
  }
}

}  // namespace hp
