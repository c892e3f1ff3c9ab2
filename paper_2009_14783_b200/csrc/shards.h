// HSD1 shard read path (reference src/shard.cpp:126-218, dataset.cpp:10-50,
// datagen.cpp:71-169, loader.cpp:80-139): shard files memory-mapped once,
// MLM records decoded straight into the engine's CSR batch layout by a
// prefetch thread, in the rank schedule's order.  Plus the MLM shard writer
// (generate_mlm_shards' file layout) for the repo's synthetic data.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hetpar_b200.h"

namespace hp {

struct ShardField {
  std::string name;
  uint8_t dtype = 0;  // 1 f32, 2 f64, 3 i64
  uint8_t rank = 0;
};

// One mapped shard: header (schema), footer (record offsets, token lengths).
struct ShardMap {
  std::string path;
  const uint8_t* base = nullptr;
  size_t size = 0;
  std::vector<ShardField> schema;
  std::vector<uint64_t> offsets;
  std::vector<uint32_t> token_lengths;
  uint64_t records_end = 0;
};

// list_shards + build_index: every *.hsd file of `dir`, sorted by path, one
// schema; the global id space is their concatenation.
class ShardSet {
 public:
  explicit ShardSet(const std::string& dir);
  ~ShardSet();
  ShardSet(const ShardSet&) = delete;
  ShardSet& operator=(const ShardSet&) = delete;

  uint64_t total() const { return total_; }
  const std::vector<uint32_t>& token_lengths() const { return lens_; }
  size_t nshards() const { return shards_.size(); }
  const std::vector<ShardField>& schema() const { return shards_.at(0).schema; }

  // instance_from_record (datagen.cpp:141-169) of global record g, appended
  // to the CSR arrays (positions stay within-instance)
  struct Csr {
    std::vector<uint64_t> tok_off{0}, mask_off{0};
    std::vector<int64_t> tokens, segments, mask_pos, mask_orig, label;
    void clear();
  };
  void append_mlm(uint64_t g, Csr& out) const;

 private:
  void open_all(const std::string& dir);
  std::vector<ShardMap> shards_;
  std::vector<uint64_t> cumulative_;
  std::vector<uint32_t> lens_;
  uint64_t total_ = 0;
  int fi_tokens_ = -1, fi_segments_ = -1, fi_mpos_ = -1, fi_morig_ = -1, fi_label_ = -1;
};

// BatchLoader (loader.cpp): serves one rank's schedule in order; with
// prefetch_depth > 0 a producer thread keeps that many batches assembled.
class ShardLoader {
 public:
  ShardLoader(std::shared_ptr<const ShardSet> set, std::vector<std::vector<uint64_t>> plan,
              std::vector<uint64_t> sched_batch, std::vector<uint8_t> sched_dummy,
              size_t prefetch_depth);
  ~ShardLoader();
  struct Loaded {
    uint64_t batch_index = 0;
    bool dummy = false;
    ShardSet::Csr csr;
  };
  bool next(Loaded& out);  // false once the schedule is exhausted

 private:
  Loaded assemble(size_t cursor) const;
  void producer();
  std::shared_ptr<const ShardSet> set_;
  std::vector<std::vector<uint64_t>> plan_;
  std::vector<uint64_t> sched_batch_;
  std::vector<uint8_t> sched_dummy_;
  size_t depth_;
  size_t sync_cursor_ = 0;
  std::thread thread_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Loaded> queue_;
  bool done_ = false, stop_ = false;
  std::exception_ptr error_;
};

// generate_mlm_shards' files (datagen.cpp:71-127) for the given records:
// `shards` contiguous chunks, earlier chunks one longer, shard_%04zu.hsd.
void write_mlm_shards(const std::string& dir, uint64_t n, uint64_t shards, const uint64_t* tok_off,
                      const int64_t* tokens, const int64_t* segments, const uint64_t* mask_off,
                      const int64_t* mask_pos, const int64_t* mask_orig, const int64_t* label);

}  // namespace hp
