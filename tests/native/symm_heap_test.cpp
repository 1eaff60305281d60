// Randomised check of the symmetric-heap allocator (csrc/symm_heap.h), run by
// tests/test_symm_heap_host.py: live blocks never overlap and stay 256-byte
// aligned inside [begin, end); freeing everything coalesces back to one block;
// the same operation sequence gives the same offsets (the symmetric invariant);
// double free and foreign offsets are rejected.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "symm_heap.h"

static int fail(const char* what) {
  std::printf("FAIL %s\n", what);
  return 1;
}

static std::vector<size_t> run(unsigned seed, SymmHeap& h, size_t begin, size_t end) {
  std::mt19937_64 rng(seed);
  h.init(begin, end);
  std::map<size_t, size_t> live;
  std::vector<size_t> trace;
  for (int step = 0; step < 20000; ++step) {
    if (live.empty() || rng() % 3) {
      size_t bytes = 1 + rng() % (1 << 16);
      size_t off = 0;
      if (h.alloc(bytes, &off)) {
        trace.push_back(off);
        live[off] = (bytes + 255) & ~size_t(255);
      } else {
        trace.push_back(size_t(-1));
      }
    } else {
      auto it = live.begin();
      std::advance(it, rng() % live.size());
      if (!h.release(it->first)) std::exit(fail("release of a live block"));
      trace.push_back(it->first | (size_t(1) << 62));
      live.erase(it);
    }
    size_t prev_end = begin;
    for (auto& [o, s] : live) {
      if (o % 256) std::exit(fail("alignment"));
      if (o < prev_end) std::exit(fail("overlap"));
      prev_end = o + s;
    }
    if (prev_end > end) std::exit(fail("out of range"));
  }
  for (auto& [o, s] : live) h.release(o);
  return trace;
}

int main() {
  const size_t begin = 8 << 20, end = begin + (64 << 20);
  SymmHeap a, b;
  auto ta = run(7, a, begin, end);
  auto tb = run(7, b, begin, end);
  if (ta != tb) return fail("determinism");
  if (a.free_.size() != 1 || a.free_.begin()->first != begin || a.free_.begin()->second != end - begin)
    return fail("coalescing back to one block");
  size_t off = 0;
  if (!a.alloc(100, &off) || off != begin) return fail("first fit after full free");
  if (!a.release(off) || a.release(off)) return fail("double free must be rejected");
  if (a.release(begin + 12345)) return fail("foreign offset must be rejected");
  if (a.alloc(end - begin + 1, &off)) return fail("oversize allocation must fail");
  std::printf("OK %zu ops\n", ta.size());
  return 0;
}
