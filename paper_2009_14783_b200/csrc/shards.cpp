// HSD1 shards (see shards.h).  File layout (shard.hpp:11-17), little-endian:
//   "HSD1" | u16 version=1 | u16 F | per field: u8 len + name, u8 dtype,
//   u8 rank | u64 R | u64 token-table offset | per record, per field:
//   u32 dims[rank] + payload | u64 record offsets [R] | u32 token lengths [R]
#include "shards.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <filesystem>

#include "checkpoint.h"  // write_file_atomic
#include "hp_common.h"

namespace hp {

namespace {

constexpr char kMagic[4] = {'H', 'S', 'D', '1'};
constexpr uint16_t kVersion = 1;

size_t dtype_size(uint8_t d) {
  if (d == 1) return 4;
  if (d == 2 || d == 3) return 8;
  fail(HP_EIO, "unknown dtype code");
}

struct Cursor {
  const uint8_t* p;
  size_t n, at;
  const std::string* path;
  const uint8_t* raw(size_t k) {
    if (at + k > n) fail(HP_EIO, "truncated shard " + *path);
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

template <class T>
void put(std::vector<uint8_t>& b, T v) {
  uint8_t t[sizeof(T)];
  std::memcpy(t, &v, sizeof(T));
  b.insert(b.end(), t, t + sizeof(T));
}

}  // namespace

void ShardSet::Csr::clear() {
  tok_off.assign(1, 0);
  mask_off.assign(1, 0);
  tokens.clear();
  segments.clear();
  mask_pos.clear();
  mask_orig.clear();
  label.clear();
}

ShardSet::ShardSet(const std::string& dir) {
  try {
    open_all(dir);
  } catch (...) {
    for (auto& sm : shards_)
      if (sm.base) ::munmap(const_cast<uint8_t*>(sm.base), sm.size);
    shards_.clear();
    throw;
  }
}

void ShardSet::open_all(const std::string& dir) {
  namespace fs = std::filesystem;
  if (!fs::is_directory(dir)) fail(HP_EIO, "not a directory: " + dir);
  std::vector<std::string> paths;
  for (const auto& e : fs::directory_iterator(dir))
    if (e.is_regular_file() && e.path().extension() == ".hsd") paths.push_back(e.path().string());
  std::sort(paths.begin(), paths.end());
  if (paths.empty()) fail(HP_ECONFIG, "no shards found under " + dir);
  for (const auto& path : paths) {
    ShardMap s;
    s.path = path;
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(HP_EIO, "cannot open shard " + path);
    struct stat st;
    if (::fstat(fd, &st) != 0) {
      ::close(fd);
      fail(HP_EIO, "cannot stat shard " + path);
    }
    s.size = static_cast<size_t>(st.st_size);
    if (s.size > 0) {
      void* m = ::mmap(nullptr, s.size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m == MAP_FAILED) {
        ::close(fd);
        fail(HP_EIO, "cannot map shard " + path);
      }
      s.base = static_cast<const uint8_t*>(m);
    }
    ::close(fd);
    shards_.push_back(std::move(s));  // unmapped by the destructor from here on
    ShardMap& sm = shards_.back();
    Cursor c{sm.base, sm.size, 0, &sm.path};
    if (std::memcmp(c.raw(4), kMagic, 4) != 0) fail(HP_EIO, "bad shard magic in " + path);
    const uint16_t version = c.get<uint16_t>();
    if (version != kVersion)
      fail(HP_EIO, "unsupported shard version " + std::to_string(version) + " in " + path);
    const uint16_t nf = c.get<uint16_t>();
    for (uint16_t i = 0; i < nf; ++i) {
      ShardField f;
      const uint8_t nl = c.get<uint8_t>();
      f.name.assign(reinterpret_cast<const char*>(c.raw(nl)), nl);
      f.dtype = c.get<uint8_t>();
      if (f.dtype < 1 || f.dtype > 3) fail(HP_EIO, "bad dtype code in " + path);
      f.rank = c.get<uint8_t>();
      sm.schema.push_back(std::move(f));
    }
    const uint64_t count = c.get<uint64_t>(), table = c.get<uint64_t>();
    if (table < 8 * count || table + 4 * count > sm.size) fail(HP_EIO, "bad footer offsets in " + path);
    sm.records_end = table - 8 * count;
    sm.offsets.resize(count);
    sm.token_lengths.resize(count);
    if (count) {
      std::memcpy(sm.offsets.data(), sm.base + sm.records_end, 8 * count);
      std::memcpy(sm.token_lengths.data(), sm.base + table, 4 * count);
    }
    for (uint64_t i = 0; i < count; ++i) {
      const uint64_t end = i + 1 < count ? sm.offsets[i + 1] : sm.records_end;
      if (sm.offsets[i] > end || end > sm.size) fail(HP_EIO, "bad record offsets in " + path);
    }
    const auto& s0 = shards_.front().schema;
    const bool same = s0.size() == sm.schema.size() &&
                      std::equal(s0.begin(), s0.end(), sm.schema.begin(), [](const ShardField& a, const ShardField& b) {
                        return a.name == b.name && a.dtype == b.dtype && a.rank == b.rank;
                      });
    if (!same) fail(HP_ECONFIG, "shard " + path + " schema does not match " + shards_.front().path);
    total_ += count;
    cumulative_.push_back(total_);
    lens_.insert(lens_.end(), sm.token_lengths.begin(), sm.token_lengths.end());
  }
  // MLM fields (instance_from_record, datagen.cpp:141-169): i64, rank 1
  const auto& sc = shards_.front().schema;
  for (size_t i = 0; i < sc.size(); ++i) {
    const std::string& n = sc[i].name;
    int* slot = n == "tokens" ? &fi_tokens_ : n == "segments" ? &fi_segments_
              : n == "mask_positions" ? &fi_mpos_ : n == "mask_originals" ? &fi_morig_
              : n == "label" ? &fi_label_ : nullptr;
    if (!slot) fail(HP_ECONFIG, "unknown field name in shard: " + n);
    if (sc[i].dtype != 3 || sc[i].rank != 1) fail(HP_ESHAPE, "field " + n + " must be an i64 vector");
    *slot = static_cast<int>(i);
  }
  if (fi_tokens_ < 0 || fi_segments_ < 0 || fi_mpos_ < 0 || fi_morig_ < 0 || fi_label_ < 0)
    fail(HP_ECONFIG, "shards do not carry the masked-token-model fields");
}

ShardSet::~ShardSet() {
  for (auto& s : shards_)
    if (s.base) ::munmap(const_cast<uint8_t*>(s.base), s.size);
}

void ShardSet::append_mlm(uint64_t g, Csr& out) const {
  if (g >= total_)
    fail(HP_EINDEX, "global record " + std::to_string(g) + " out of range (total " + std::to_string(total_) + ")");
  const size_t k = static_cast<size_t>(std::upper_bound(cumulative_.begin(), cumulative_.end(), g) -
                                       cumulative_.begin());
  const ShardMap& s = shards_[k];
  const uint64_t local = g - (k ? cumulative_[k - 1] : 0);
  const uint64_t end = local + 1 < s.offsets.size() ? s.offsets[local + 1] : s.records_end;
  Cursor c{s.base, end, s.offsets[local], &s.path};
  const int64_t* field_ptr[5] = {};
  uint32_t field_n[5] = {};
  for (size_t f = 0; f < s.schema.size(); ++f) {
    const uint32_t n = c.get<uint32_t>();  // rank 1: one dim
    const uint8_t* payload = c.raw(static_cast<size_t>(n) * dtype_size(s.schema[f].dtype));
    const int slot = static_cast<int>(f) == fi_tokens_ ? 0 : static_cast<int>(f) == fi_segments_ ? 1
                   : static_cast<int>(f) == fi_mpos_ ? 2 : static_cast<int>(f) == fi_morig_ ? 3 : 4;
    field_ptr[slot] = reinterpret_cast<const int64_t*>(payload);  // possibly unaligned: memcpy below
    field_n[slot] = n;
  }
  if (field_n[1] != field_n[0]) fail(HP_ESHAPE, "segments length differs from tokens");
  if (field_n[3] != field_n[2]) fail(HP_ESHAPE, "mask_originals length differs from mask_positions");
  if (field_n[4] != 1) fail(HP_ESHAPE, "label field must hold one value");
  auto app = [](std::vector<int64_t>& v, const int64_t* p, uint32_t n) {
    const size_t at = v.size();
    v.resize(at + n);
    if (n) std::memcpy(v.data() + at, p, 8ull * n);
  };
  app(out.tokens, field_ptr[0], field_n[0]);
  app(out.segments, field_ptr[1], field_n[1]);
  app(out.mask_pos, field_ptr[2], field_n[2]);
  app(out.mask_orig, field_ptr[3], field_n[3]);
  app(out.label, field_ptr[4], 1);
  out.tok_off.push_back(out.tokens.size());
  out.mask_off.push_back(out.mask_pos.size());
}

// ------------------------------------------------------------------ loader
ShardLoader::ShardLoader(std::shared_ptr<const ShardSet> set, std::vector<std::vector<uint64_t>> plan,
                         std::vector<uint64_t> sched_batch, std::vector<uint8_t> sched_dummy,
                         size_t prefetch_depth)
    : set_(std::move(set)),
      plan_(std::move(plan)),
      sched_batch_(std::move(sched_batch)),
      sched_dummy_(std::move(sched_dummy)),
      depth_(prefetch_depth) {
  if (sched_batch_.size() != sched_dummy_.size()) fail(HP_ECONFIG, "loader: schedule arrays differ in length");
  for (uint64_t b : sched_batch_)
    if (b >= plan_.size())
      fail(HP_ECONFIG, "schedule references batch " + std::to_string(b) + " beyond plan size " +
                           std::to_string(plan_.size()));
  if (depth_ > 0) thread_ = std::thread([this] { producer(); });
}

ShardLoader::~ShardLoader() {
  if (thread_.joinable()) {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    thread_.join();
  }
}

ShardLoader::Loaded ShardLoader::assemble(size_t cursor) const {
  Loaded out;
  out.batch_index = sched_batch_[cursor];
  out.dummy = sched_dummy_[cursor] != 0;
  for (uint64_t g : plan_[out.batch_index]) set_->append_mlm(g, out.csr);
  return out;
}

void ShardLoader::producer() {
  try {
    for (size_t cursor = 0; cursor < sched_batch_.size(); ++cursor) {
      Loaded b = assemble(cursor);
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [this] { return stop_ || queue_.size() < depth_; });
      if (stop_) return;
      queue_.push_back(std::move(b));
      lk.unlock();
      cv_.notify_all();
    }
    std::lock_guard<std::mutex> g(mu_);
    done_ = true;
    cv_.notify_all();
  } catch (...) {
    std::lock_guard<std::mutex> g(mu_);
    error_ = std::current_exception();
    done_ = true;
    cv_.notify_all();
  }
}

bool ShardLoader::next(Loaded& out) {
  if (depth_ == 0) {
    if (sync_cursor_ >= sched_batch_.size()) return false;
    out = assemble(sync_cursor_++);
    return true;
  }
  std::unique_lock<std::mutex> lk(mu_);
  cv_.wait(lk, [this] { return !queue_.empty() || done_; });
  if (!queue_.empty()) {
    out = std::move(queue_.front());
    queue_.pop_front();
    lk.unlock();
    cv_.notify_all();
    return true;
  }
  if (error_) std::rethrow_exception(error_);
  return false;
}

// ------------------------------------------------------------------ writer
void write_mlm_shards(const std::string& dir, uint64_t n, uint64_t shards, const uint64_t* tok_off,
                      const int64_t* tokens, const int64_t* segments, const uint64_t* mask_off,
                      const int64_t* mask_pos, const int64_t* mask_orig, const int64_t* label) {
  if (shards == 0) fail(HP_ECONFIG, "datagen: shards must be >= 1");
  std::filesystem::create_directories(dir);
  static const char* kNames[5] = {"tokens", "segments", "mask_positions", "mask_originals", "label"};
  uint64_t rec = 0;
  for (uint64_t k = 0; k < shards; ++k) {
    const uint64_t cnt = n / shards + (k < n % shards ? 1 : 0);  // chunk_sizes, datagen.cpp:21-26
    std::vector<uint8_t> b;
    b.insert(b.end(), kMagic, kMagic + 4);
    put<uint16_t>(b, kVersion);
    put<uint16_t>(b, 5);
    for (const char* nm : kNames) {
      put<uint8_t>(b, static_cast<uint8_t>(std::strlen(nm)));
      b.insert(b.end(), nm, nm + std::strlen(nm));
      put<uint8_t>(b, 3);  // i64
      put<uint8_t>(b, 1);  // rank 1
    }
    put<uint64_t>(b, cnt);
    const size_t table_field = b.size();
    put<uint64_t>(b, 0);
    std::vector<uint64_t> offsets;
    std::vector<uint32_t> lens;
    for (uint64_t r = 0; r < cnt; ++r, ++rec) {
      offsets.push_back(b.size());
      auto field = [&](const int64_t* p, uint64_t lo, uint64_t hi) {
        put<uint32_t>(b, static_cast<uint32_t>(hi - lo));
        const uint8_t* q = reinterpret_cast<const uint8_t*>(p + lo);
        b.insert(b.end(), q, q + 8 * (hi - lo));
      };
      field(tokens, tok_off[rec], tok_off[rec + 1]);
      field(segments, tok_off[rec], tok_off[rec + 1]);
      field(mask_pos, mask_off[rec], mask_off[rec + 1]);
      field(mask_orig, mask_off[rec], mask_off[rec + 1]);
      field(label, rec, rec + 1);
      lens.push_back(static_cast<uint32_t>(tok_off[rec + 1] - tok_off[rec]));
    }
    for (uint64_t o : offsets) put<uint64_t>(b, o);
    const uint64_t table = b.size();
    for (uint32_t t : lens) put<uint32_t>(b, t);
    std::memcpy(b.data() + table_field, &table, 8);
    char name[32];
    std::snprintf(name, sizeof(name), "shard_%04llu.hsd", static_cast<unsigned long long>(k));
    write_file_atomic((std::filesystem::path(dir) / name).string(), b);
  }
}

}  // namespace hp
