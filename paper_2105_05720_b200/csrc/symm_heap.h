// Host-only symmetric-heap allocator (no CUDA): included by internal.h and
// compiled stand-alone by tests/test_symm_heap_host.py.
#pragma once

#include <cstddef>
#include <iterator>
#include <map>

// Symmetric-heap allocator: deterministic first-fit over a free list ordered
// by offset, 256-byte granules, neighbours coalesced on free. Every rank runs
// the same alloc/free sequence (calls are collective), so every rank gets the
// same offsets - the symmetric-heap invariant kernels rely on.
struct SymmHeap {
  std::map<size_t, size_t> free_;  // offset -> bytes
  std::map<size_t, size_t> used_;  // offset -> bytes
  size_t begin = 0, end = 0, high = 0;

  void init(size_t b, size_t e) {
    begin = b;
    end = e;
    high = b;
    free_.clear();
    used_.clear();
    if (e > b) free_[b] = e - b;
  }
  // returns false when no free block is large enough
  bool alloc(size_t bytes, size_t* off) {
    const size_t sz = (bytes + 255) & ~size_t(255);
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second >= sz) {
        *off = it->first;
        const size_t rest = it->second - sz;
        free_.erase(it);
        if (rest) free_[*off + sz] = rest;
        used_[*off] = sz;
        if (*off + sz > high) high = *off + sz;
        return true;
      }
    return false;
  }
  bool release(size_t off) {
    auto u = used_.find(off);
    if (u == used_.end()) return false;
    size_t start = off, size = u->second;
    used_.erase(u);
    auto next = free_.lower_bound(start);
    if (next != free_.end() && start + size == next->first) {  // merge with the following block
      size += next->second;
      next = free_.erase(next);
    }
    if (next != free_.begin()) {  // merge with the preceding block
      auto prev = std::prev(next);
      if (prev->first + prev->second == start) {
        start = prev->first;
        size += prev->second;
        free_.erase(prev);
      }
    }
    free_[start] = size;
    return true;
  }
  size_t largest_free() const {
    size_t m = 0;
    for (auto& [o, s] : free_) m = s > m ? s : m;
    return m;
  }
};

