// tg_host.cpp -- host-side helpers exported by libtg_loss.so (no device access).
//
//  tg_scored_states  the toy-table policy's "model forward" (which logits row
//                    each mask-true token is scored in): FNV-1a 64 over
//                    little-endian (context_key u64, position i64, prev i64)
//                    mod num_buckets, prev reset to -1 after mask-false tokens.
//                    Restates encoding.py:19-35 and policy.py:152-161, 181-191.
//  tg_group_by_task  ExperienceBuffer.sample_batch(group_by_task=True) group
//                    indexing (buffer.py:240-264): per task, ordered READY
//                    experiences are cut into consecutive chunks of exactly
//                    group_size (incomplete leftovers dropped), chunks sorted by
//                    their lead element with the flat path's comparator.
#include <stdint.h>

#include <algorithm>
#include <map>
#include <numeric>
#include <vector>

#include "tg_loss.h"

namespace {

constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001B3ull;

inline uint64_t fnv_bytes(uint64_t h, uint64_t v) {  // 8 little-endian bytes
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xffu;
    h *= kFnvPrime;
  }
  return h;
}

}  // namespace

extern "C" {

int64_t tg_scored_states(const int64_t* tokens, const uint8_t* mask, const int64_t* tok_off,
                         const int64_t* prompt_len, int64_t n_exp, int64_t num_buckets,
                         int64_t* states_out, int32_t* target_out, int64_t capacity) {
  if (!tokens || !mask || !tok_off || !prompt_len || num_buckets < 1 || n_exp < 0) return -1;
  int64_t n = 0;
  for (int64_t e = 0; e < n_exp; ++e) {
    const int64_t a = tok_off[e], b = tok_off[e + 1];
    const int64_t pl = prompt_len[e];
    if (b < a || pl < 0 || pl > b - a) return -1;
    uint64_t key = kFnvOffset;  // sequence_key(prompt): FNV-1a over int64 LE words
    for (int64_t i = a; i < a + pl; ++i) key = fnv_bytes(key, uint64_t(tokens[i]));
    int64_t prev = -1;  // CONTEXT_SENTINEL, policy.py:29
    for (int64_t i = a; i < b; ++i) {
      const int64_t pos = i - a;
      if (mask[i]) {
        uint64_t h = kFnvOffset;
        h = fnv_bytes(h, key);
        h = fnv_bytes(h, uint64_t(pos));
        h = fnv_bytes(h, uint64_t(prev));
        if (n >= capacity) return -1;
        if (states_out) states_out[n] = int64_t(h % uint64_t(num_buckets));
        if (target_out) target_out[n] = int32_t(tokens[i]);
        ++n;
        prev = tokens[i];
      } else {
        prev = -1;
      }
    }
  }
  return n;
}

int64_t tg_group_by_task(const int64_t* task_key, const double* priority, const int64_t* id_rank,
                         const uint8_t* ready, int64_t n, int64_t group_size, int64_t n_take,
                         int32_t policy, int64_t* groups_out) {
  if (!task_key || !ready || n < 0 || group_size < 1 || n_take < 1) return -1;
  if (policy == 1 && (!priority || !id_rank)) return -1;
  std::vector<int64_t> ids;
  for (int64_t i = 0; i < n; ++i)
    if (ready[i]) ids.push_back(i);
  // _order_ids (buffer.py:201-205): FIFO = insertion order; PRIORITY = (-priority, sample_id)
  if (policy == 1) {
    std::stable_sort(ids.begin(), ids.end(), [&](int64_t x, int64_t y) {
      if (priority[x] != priority[y]) return priority[x] > priority[y];
      return id_rank[x] < id_rank[y];
    });
  }
  // per task, in first-seen order of the ordered ids (dict insertion order)
  std::vector<int64_t> task_order;
  std::map<int64_t, std::vector<int64_t>> per_task;
  for (int64_t i : ids) {
    auto it = per_task.find(task_key[i]);
    if (it == per_task.end()) {
      task_order.push_back(task_key[i]);
      per_task[task_key[i]] = {i};
    } else {
      it->second.push_back(i);
    }
  }
  std::vector<std::vector<int64_t>> chunks;
  for (int64_t t : task_order) {
    const auto& v = per_task[t];
    for (size_t s = 0; s + size_t(group_size) <= v.size(); s += size_t(group_size))
      chunks.emplace_back(v.begin() + s, v.begin() + s + group_size);
  }
  // chunks.sort(key=lead element) -- Python's sort is stable
  std::stable_sort(chunks.begin(), chunks.end(),
                   [&](const std::vector<int64_t>& x, const std::vector<int64_t>& y) {
                     const int64_t a = x[0], b = y[0];
                     if (policy == 1) {
                       if (priority[a] != priority[b]) return priority[a] > priority[b];
                       return id_rank[a] < id_rank[b];
                     }
                     return a < b;  // FIFO: insertion sequence
                   });
  const int64_t take = std::min<int64_t>(n_take, int64_t(chunks.size()));
  for (int64_t g = 0; g < take; ++g)
    for (int64_t j = 0; j < group_size; ++j) groups_out[g * group_size + j] = chunks[g][j];
  return take;
}

}  // extern "C"
