// Device bucket tables for tensor-list collectives (paper §5.4 "scattered
// tensors"; reference BucketTable / build_bucket_table, runtime.hpp:575-614,
// and scattered_collective, runtime.hpp:624-675).
//
// The reference flattens every tensor into one buffer in bucket order, runs
// one AllReduce, and scatters the result back (two full copies). Here the
// bucket order is only an INDEX SPACE: kernels walk "segments" (a bucket, or
// the part of it inside one rank's flat chunk) and read/write the caller's
// tensors in place, so there is no flatten copy.
//
// Segment tables built once on the host (plan_tlist, no device needed):
//   TWO_SHOT : per rank r, the segments of flat chunk [total*r/W,
//              total*(r+1)/W) (runtime.hpp:63-66); `sidx` indexes the rank's
//              padded shard storage for sliced state (m, v).
//   ONE_SHOT : every bucket, split at chunk boundaries so each segment has a
//              single ring owner; `sidx` indexes the padded full state.
// Shard/state indices are padded so that sidx == toff (mod 4): a 4-element
// quad of a tensor maps to one aligned 16-byte quad of state.
#include <algorithm>
#include <cstring>

#include "fused_opt.h"

using namespace coconet;

namespace {

struct HostSeg {
  int64_t toff;
  int32_t tensor, len, owner;
  int64_t flat;
};

int plan_tlist(coconet_tlist* tl, int W, int n_tensors, const int64_t* counts, int64_t bucket_cap) {
  if (!counts) return set_error(COCONET_ERR_INVALID_INPUT, "null counts");
  if (n_tensors < 1) return set_error(COCONET_ERR_INVALID_INPUT, "empty tensor list");
  if (W < 1 || W > kMaxRanks) return set_error(COCONET_ERR_NO_SUCH_RANK, "bad group size");
  if (bucket_cap < 4 || bucket_cap > (1 << 20) || (bucket_cap & 3))
    return set_error(COCONET_ERR_INVALID_INPUT, "bucket capacity must be a multiple of 4 in [4, 2^20]");
  tl->world = W;
  tl->n_tensors = n_tensors;
  tl->bucket_cap = bucket_cap;
  tl->counts.assign(counts, counts + n_tensors);
  tl->total = 0;
  for (int i = 0; i < n_tensors; ++i) {
    // build_bucket_table: "tensor has no elements" (runtime.hpp:596)
    if (counts[i] <= 0)
      return set_error(COCONET_ERR_INVALID_INPUT, "tensor " + std::to_string(i) + " has no elements");
    tl->total += counts[i];
  }
  // scattered_collective: "fewer bucketed elements than ranks" (runtime.hpp:630)
  if (tl->total < W) return set_error(COCONET_ERR_DIVISIBILITY, "fewer bucketed elements than ranks");
  // round-robin bucket order (runtime.hpp:604-613)
  std::vector<int64_t> cursor(static_cast<size_t>(n_tensors), 0);
  std::vector<HostSeg> buckets;
  int64_t remaining = 0;
  for (int i = 0; i < n_tensors; ++i) remaining += (counts[i] + bucket_cap - 1) / bucket_cap;
  buckets.reserve(size_t(remaining));
  int64_t flat = 0;
  while (remaining > 0) {
    for (int i = 0; i < n_tensors; ++i) {
      if (cursor[size_t(i)] >= counts[i]) continue;
      HostSeg b{};
      b.tensor = i;
      b.toff = cursor[size_t(i)];
      b.len = int32_t(std::min(bucket_cap, counts[i] - b.toff));
      b.flat = flat;
      flat += b.len;
      cursor[size_t(i)] += b.len;
      buckets.push_back(b);
      --remaining;
    }
  }
  tl->n_buckets = int64_t(buckets.size());
  for (int r = 0; r <= W; ++r) tl->chunk_lo[r] = tl->total * r / W;
  // split buckets at chunk boundaries
  std::vector<HostSeg> pieces;
  pieces.reserve(buckets.size() + size_t(W));
  for (auto& b : buckets) {
    int64_t s = b.flat, e = b.flat + b.len;
    while (s < e) {
      int owner = int(std::upper_bound(tl->chunk_lo, tl->chunk_lo + W + 1, s) - tl->chunk_lo) - 1;
      int64_t cut = std::min(e, tl->chunk_lo[owner + 1]);
      HostSeg p = b;
      p.toff = b.toff + (s - b.flat);
      p.len = int32_t(cut - s);
      p.flat = s;
      p.owner = owner;
      pieces.push_back(p);
      s = cut;
    }
  }
  // TWO_SHOT tables: pieces grouped by owner (already ordered by flat position)
  std::vector<Seg>& table = tl->table;
  table.clear();
  table.reserve(pieces.size() * 2);
  tl->host_flat.clear();
  tl->host_sidx.clear();
  int64_t shard_max = 0;
  tl->seg_begin[0] = 0;
  size_t pi = 0;
  for (int r = 0; r < W; ++r) {
    int64_t cur = 0;
    while (pi < pieces.size() && pieces[pi].owner == r) {
      HostSeg& p = pieces[pi++];
      cur += ((p.toff & 3) - (cur & 3) + 4) & 3;
      table.push_back(Seg{p.toff, cur, pack_meta(p.tensor, p.len, r)});
      tl->host_flat.push_back(p.flat);
      tl->host_sidx.push_back(cur);
      cur += p.len;
    }
    tl->seg_begin[r + 1] = int64_t(table.size());
    shard_max = std::max(shard_max, cur);
  }
  tl->shard_elems = (shard_max + 3) & ~int64_t(3);
  // ONE_SHOT table: every piece, padded full state
  tl->os_begin = int64_t(table.size());
  int64_t cur = 0;
  for (auto& p : pieces) {
    cur += ((p.toff & 3) - (cur & 3) + 4) & 3;
    table.push_back(Seg{p.toff, cur, pack_meta(p.tensor, p.len, p.owner)});
    cur += p.len;
  }
  tl->os_end = int64_t(table.size());
  tl->full_state_elems = (cur + 3) & ~int64_t(3);
  // per-tensor segment lists of each rank (TWO_SHOT), for deterministic
  // per-tensor reductions (LAMB): CSR over [seg_begin[r], seg_begin[r+1])
  tl->csr_ptr.clear();
  tl->csr_idx.clear();
  for (int r = 0; r < W; ++r) {
    std::vector<std::vector<int64_t>> per(static_cast<size_t>(n_tensors));
    for (int64_t s = tl->seg_begin[r]; s < tl->seg_begin[r + 1]; ++s)
      per[size_t(meta_tensor(table[size_t(s)].meta))].push_back(s);
    tl->csr_begin[r] = int64_t(tl->csr_ptr.size());
    int64_t acc = int64_t(tl->csr_idx.size());
    for (int t = 0; t < n_tensors; ++t) {
      tl->csr_ptr.push_back(acc);
      for (auto s : per[size_t(t)]) tl->csr_idx.push_back(s);
      acc = int64_t(tl->csr_idx.size());
    }
    tl->csr_ptr.push_back(acc);
  }
  tl->n_segs = int64_t(table.size());
  tl->metadata_bytes = int64_t(table.size() * sizeof(Seg));
  return COCONET_OK;
}

int upload_tlist(coconet_tlist* tl) {
  const auto& table = tl->table;
  size_t bytes_segs = table.size() * sizeof(Seg);
  size_t bytes_ptr = tl->csr_ptr.size() * sizeof(int64_t);
  size_t bytes_idx = std::max<size_t>(1, tl->csr_idx.size()) * sizeof(int64_t);
  size_t bytes_offs = size_t(tl->n_tensors) * 2 * sizeof(int64_t);
  size_t bytes_part = size_t(table.size()) * 2 * sizeof(double);
  size_t total = bytes_segs + bytes_ptr + bytes_idx + bytes_offs + bytes_part + 5 * 256;
  CN_CUDA(cudaMalloc(&tl->dev_mem, total));
  char* p = static_cast<char*>(tl->dev_mem);
  auto carve = [&](size_t n) {
    char* q = p;
    p += (n + 255) & ~size_t(255);
    return q;
  };
  tl->d_segs = reinterpret_cast<Seg*>(carve(bytes_segs));
  tl->d_csr_ptr = reinterpret_cast<int64_t*>(carve(bytes_ptr));
  tl->d_csr_idx = reinterpret_cast<int64_t*>(carve(bytes_idx));
  tl->d_offs = reinterpret_cast<int64_t*>(carve(bytes_offs));
  tl->d_seg_part = reinterpret_cast<double*>(carve(bytes_part));
  CN_CUDA(cudaMemcpy(tl->d_segs, table.data(), bytes_segs, cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_csr_ptr, tl->csr_ptr.data(), bytes_ptr, cudaMemcpyHostToDevice));
  if (!tl->csr_idx.empty())
    CN_CUDA(cudaMemcpy(tl->d_csr_idx, tl->csr_idx.data(), tl->csr_idx.size() * sizeof(int64_t),
                       cudaMemcpyHostToDevice));
  tl->last_offs.assign(size_t(tl->n_tensors) * 2, -1);
  return COCONET_OK;
}

}  // namespace

extern "C" {

int coconet_tlist_create(coconet_ctx_t c, int group, int n_tensors, const int64_t* counts,
                         int64_t bucket_cap, coconet_tlist_t* out) {
  if (!c || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  *out = nullptr;
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  auto* tl = new coconet_tlist();
  tl->ctx = c;
  tl->group = group;
  int rc = plan_tlist(tl, c->groups[size_t(group)].size, n_tensors, counts, bucket_cap);
  if (!rc) rc = upload_tlist(tl);
  if (rc) {
    coconet_tlist_destroy(tl);
    return rc;
  }
  *out = tl;
  return COCONET_OK;
}

int coconet_tlist_plan(int world, int n_tensors, const int64_t* counts, int64_t bucket_cap,
                       coconet_tlist_t* out) {
  if (!out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  *out = nullptr;
  auto* tl = new coconet_tlist();
  int rc = plan_tlist(tl, world, n_tensors, counts, bucket_cap);
  if (rc) {
    delete tl;
    return rc;
  }
  *out = tl;
  return COCONET_OK;
}

int coconet_tlist_destroy(coconet_tlist_t tl) {
  if (!tl) return COCONET_OK;
  if (tl->dev_mem || tl->stream_mem || tl->win_mem || tl->oc_mem) cudaDeviceSynchronize();
  if (tl->dev_mem) cudaFree(tl->dev_mem);
  if (tl->stream_mem) cudaFree(tl->stream_mem);
  if (tl->win_mem) cudaFree(tl->win_mem);
  if (tl->oc_mem) cudaFree(tl->oc_mem);
  delete tl;
  return COCONET_OK;
}

int64_t coconet_tlist_shard_elems(coconet_tlist_t tl) { return tl ? tl->shard_elems : -1; }
int64_t coconet_tlist_onchip_spilled(coconet_tlist_t tl) { return tl && tl->oc_mem ? tl->oc_spilled : -1; }
int64_t coconet_tlist_total(coconet_tlist_t tl) { return tl ? tl->total : -1; }
int64_t coconet_tlist_state_elems(coconet_tlist_t tl) { return tl ? tl->full_state_elems : -1; }
int64_t coconet_tlist_buckets(coconet_tlist_t tl) { return tl ? tl->n_buckets : -1; }
int64_t coconet_tlist_metadata_bytes(coconet_tlist_t tl) { return tl ? tl->metadata_bytes : -1; }

int coconet_tlist_chunk(coconet_tlist_t tl, int r, int64_t* lo, int64_t* hi) {
  if (!tl) return set_error(COCONET_ERR_INVALID_INPUT, "null tlist");
  if (r < 0 || r >= tl->world) return set_error(COCONET_ERR_NO_SUCH_RANK, "rank out of range");
  if (lo) *lo = tl->chunk_lo[r];
  if (hi) *hi = tl->chunk_lo[r + 1];
  return COCONET_OK;
}

int64_t coconet_tlist_shard_index(coconet_tlist_t tl, int64_t pos) {
  if (!tl || pos < 0 || pos >= tl->total) return -1;
  // TWO_SHOT segments are ordered by flat position across ranks
  auto it = std::upper_bound(tl->host_flat.begin(), tl->host_flat.end(), pos);
  size_t s = size_t(it - tl->host_flat.begin()) - 1;
  return tl->host_sidx[s] + (pos - tl->host_flat[s]);
}

int64_t coconet_tlist_segments(coconet_tlist_t tl, int r, int64_t* tensor, int64_t* toff,
                               int64_t* len, int64_t* sidx, int64_t cap) {
  if (!tl) return set_error(COCONET_ERR_INVALID_INPUT, "null tlist");
  if (r < -1 || r >= tl->world) return set_error(COCONET_ERR_NO_SUCH_RANK, "rank out of range");
  int64_t b = r < 0 ? tl->os_begin : tl->seg_begin[r];
  int64_t e = r < 0 ? tl->os_end : tl->seg_begin[r + 1];
  if (e - b > cap) return -(e - b);
  for (int64_t i = 0; i < e - b; ++i) {
    const Seg& s = tl->table[size_t(b + i)];
    tensor[i] = meta_tensor(s.meta);
    toff[i] = s.toff;
    len[i] = meta_len(s.meta);
    sidx[i] = s.sidx;
  }
  return e - b;
}

int64_t coconet_tlist_stream_items(coconet_tlist_t tl, int64_t lag, int r, int64_t* tensor,
                                   int64_t* toff, int64_t* len, int64_t* pass, int64_t cap) {
  if (!tl) return set_error(COCONET_ERR_INVALID_INPUT, "null tlist");
  if (r < 0 || r >= tl->world) return set_error(COCONET_ERR_NO_SUCH_RANK, "rank out of range");
  int rc = tlist_stream_plan(tl, lag);
  if (rc) return -(int64_t(1) << 62);  // message in coconet_last_error
  const int64_t b = tl->item_begin[r], e = tl->item_begin[r + 1];
  if (e - b > cap) return -(e - b);
  for (int64_t i = 0; i < e - b; ++i) {
    const Item& it = tl->items[size_t(b + i)];
    tensor[i] = meta_tensor(it.meta);
    toff[i] = it.toff;
    len[i] = meta_len(it.meta);
    pass[i] = meta_pass(it.meta);
  }
  return e - b;
}

}  // extern "C"

namespace coconet {

// STREAMED-LAMB work lists. One GLOBAL sequence of groups (pass, tensor) is
// built from the tensors' largest per-rank share (so it is identical on every
// rank): pass-1 groups in tensor order, and the pass-2 group of tensor t is
// emitted as soon as the pass-1 stream has advanced `lag` elements past the
// end of t's pass 1 (all remaining pass-2 groups at the end). Every rank lists
// its own segments group by group, each group in CSR (toff) order.
//  - L2 reuse: t's m, v, p are re-read about `lag` (+ t) elements of pass-1
//    traffic after they were touched, so a lag that covers the grid's
//    in-flight window (gridDim.x items) but fits L2 keeps pass 2 out of HBM.
//  - No deadlock: every rank's list is a subsequence of the global sequence,
//    and P2(t) follows P1(t) in it. CTAs walk their items in list order, so the
//    unfinished item first in (group, rank, index) order always has its
//    dependencies (P1(t) items of every rank, in earlier groups) done.
//  - The pass-1 items of a tensor are contiguous, so its norm partials reduce
//    without an index list.
int tlist_stream_plan(coconet_tlist* tl, int64_t lag) {
  if (lag <= 0) return set_error(COCONET_ERR_INVALID_INPUT, "lag must be positive");
  if (tl->stream_wave == lag) return COCONET_OK;
  const int W = tl->world, n = tl->n_tensors;
  std::vector<int64_t> size(size_t(n), 0);
  tl->holders.assign(size_t(n), 0);
  {
    std::vector<int64_t> elems(size_t(W) * size_t(n), 0);
    for (int r = 0; r < W; ++r)
      for (int64_t s = tl->seg_begin[r]; s < tl->seg_begin[r + 1]; ++s) {
        const Seg& g = tl->table[size_t(s)];
        elems[size_t(r) * size_t(n) + size_t(meta_tensor(g.meta))] += meta_len(g.meta);
      }
    for (int t = 0; t < n; ++t)
      for (int r = 0; r < W; ++r) {
        const int64_t e = elems[size_t(r) * size_t(n) + size_t(t)];
        size[size_t(t)] = std::max(size[size_t(t)], e);
        if (e > 0) tl->holders[size_t(t)] |= 1u << r;
      }
  }
  // the global group sequence: (pass, tensor)
  std::vector<std::pair<int, int>> groups;
  groups.reserve(size_t(2 * n));
  std::vector<std::pair<int, int64_t>> pending;  // (tensor, pass-1 end position)
  size_t head = 0;
  int64_t pos = 0;
  for (int t = 0; t < n; ++t) {
    groups.emplace_back(0, t);
    pos += size[size_t(t)];
    pending.emplace_back(t, pos);
    while (head < pending.size() && pending[head].second + lag <= pos) groups.emplace_back(1, pending[head++].first);
  }
  while (head < pending.size()) groups.emplace_back(1, pending[head++].first);
  tl->items.clear();
  tl->p1_first.assign(size_t(W) * size_t(n), 0);
  for (int r = 0; r < W; ++r) {
    tl->item_begin[r] = int64_t(tl->items.size());
    const int64_t* ptr = tl->csr_ptr.data() + tl->csr_begin[r];
    for (auto [pass, t] : groups) {
      if (pass == 0) tl->p1_first[size_t(r) * size_t(n) + size_t(t)] = int64_t(tl->items.size());
      for (int64_t i = ptr[t]; i < ptr[t + 1]; ++i) {
        const Seg& g = tl->table[size_t(tl->csr_idx[size_t(i)])];
        tl->items.push_back(Item{g.toff, g.sidx, g.meta | (pass ? kPass2Bit : 0)});
      }
    }
  }
  tl->item_begin[W] = int64_t(tl->items.size());
  tl->stream_wave = lag;
  if (!tl->dev_mem) return COCONET_OK;  // plan-only list
  // device copies: items, p1_first, holders, counters [kMaxRanks][n], partials
  if (tl->stream_mem) {
    CN_CUDA(cudaDeviceSynchronize());
    CN_CUDA(cudaFree(tl->stream_mem));
    tl->stream_mem = nullptr;
  }
  const size_t b_items = tl->items.size() * sizeof(Item);
  const size_t b_first = tl->p1_first.size() * sizeof(int64_t);
  const size_t b_hold = size_t(n) * sizeof(uint32_t);
  const size_t b_cnt = size_t(kMaxRanks) * size_t(n) * sizeof(uint32_t);
  const size_t b_part = std::max<size_t>(1, tl->items.size()) * 2 * sizeof(double);
  const size_t total = b_items + b_first + b_hold + b_cnt + b_part + 5 * 256;
  CN_CUDA(cudaMalloc(&tl->stream_mem, total));
  char* p = static_cast<char*>(tl->stream_mem);
  auto carve = [&](size_t nb) {
    char* q = p;
    p += (nb + 255) & ~size_t(255);
    return q;
  };
  tl->d_items = reinterpret_cast<Item*>(carve(b_items));
  tl->d_p1_first = reinterpret_cast<int64_t*>(carve(b_first));
  tl->d_holders = reinterpret_cast<uint32_t*>(carve(b_hold));
  tl->d_cnt = reinterpret_cast<uint32_t*>(carve(b_cnt));
  tl->d_item_part = reinterpret_cast<double*>(carve(b_part));
  CN_CUDA(cudaMemcpy(tl->d_items, tl->items.data(), b_items, cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_p1_first, tl->p1_first.data(), b_first, cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_holders, tl->holders.data(), b_hold, cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemset(tl->d_cnt, 0, b_cnt));
  tl->stream_calls = 0;
  return COCONET_OK;
}

// Uploads per-tensor heap offsets of the g/x and p/out tensors when they
// changed since the last call (pageable source: the copy is staged before
// cudaMemcpyAsync returns, and it is stream-ordered after earlier kernels).
// Windows of consecutive tensors (rank 0's CSR order) holding about
// win_elems elements each (a tensor larger than that is a window alone), and
// their chunk items: every segment of the window's tensors, tensor by tensor,
// cut into chunks of chunk_q quads (segment | chunk << 40), so the persistent
// grid splits a window evenly by chunks.
int tlist_window_plan(coconet_tlist* tl, int64_t win_elems, int chunk_q) {
  if (tl->win_elems == win_elems && tl->win_chunk_q == chunk_q && tl->win_mem) return COCONET_OK;
  const int64_t* ptr = tl->csr_ptr.data() + tl->csr_begin[0];
  std::vector<int64_t> items, win_item{0}, titem{0};
  std::vector<int> win_t{0};
  int64_t acc = 0;
  for (int t = 0; t < tl->n_tensors; ++t) {
    for (int64_t i = ptr[t]; i < ptr[t + 1]; ++i) {
      const int64_t s = tl->csr_idx[size_t(i)];
      const Seg& sg = tl->table[size_t(s)];
      const int64_t q0 = sg.toff >> 2, q1 = (sg.toff + meta_len(sg.meta) + 3) >> 2;
      for (int64_t k = 0; q0 + k * chunk_q < q1; ++k) items.push_back(s | (k << 40));
    }
    titem.push_back(int64_t(items.size()));
    acc += tl->counts[size_t(t)];
    if (acc >= win_elems || t == tl->n_tensors - 1) {
      win_item.push_back(int64_t(items.size()));
      win_t.push_back(t + 1);
      acc = 0;
    }
  }
  const int K = int(win_item.size()) - 1;
  if (tl->win_mem) {
    cudaDeviceSynchronize();
    cudaFree(tl->win_mem);
    tl->win_mem = nullptr;
  }
  const size_t b_items = std::max<size_t>(1, items.size()) * sizeof(int64_t);
  const size_t b_wi = size_t(K + 1) * sizeof(int64_t), b_ti = size_t(tl->n_tensors + 1) * sizeof(int64_t);
  const size_t b_wt = size_t(K + 1) * sizeof(int), b_part = std::max<size_t>(1, items.size()) * sizeof(float2);
  const size_t b_ratio = size_t(tl->n_tensors) * sizeof(float);
  const size_t b_tick = size_t(K) * 2 * sizeof(unsigned long long), b_cnt = size_t(K) * sizeof(uint32_t);
  const size_t b_state = (b_tick + 15) / 16 * 16 + 2 * ((b_cnt + 15) / 16 * 16);
  const size_t total = b_items + b_wi + b_ti + b_wt + b_part + b_ratio + b_state + 8 * 16;
  CN_CUDA(cudaMalloc(&tl->win_mem, total));
  CN_CUDA(cudaMemset(tl->win_mem, 0, total));
  char* p = static_cast<char*>(tl->win_mem);
  auto carve = [&](size_t n) {
    char* q = p;
    p += (n + 15) / 16 * 16;
    return q;
  };
  tl->d_win_items = reinterpret_cast<int64_t*>(carve(b_items));
  tl->d_win_item = reinterpret_cast<int64_t*>(carve(b_wi));
  tl->d_titem = reinterpret_cast<int64_t*>(carve(b_ti));
  tl->d_win_t = reinterpret_cast<int*>(carve(b_wt));
  tl->d_ipart = reinterpret_cast<float2*>(carve(b_part));
  tl->d_ratio = reinterpret_cast<float*>(carve(b_ratio));
  tl->win_state = p;
  tl->win_state_bytes = b_state;
  tl->d_win_tick = reinterpret_cast<unsigned long long*>(carve(b_tick));
  tl->d_win_cnt = reinterpret_cast<uint32_t*>(carve(b_cnt));
  tl->d_win_ready = reinterpret_cast<uint32_t*>(carve(b_cnt));
  if (!items.empty())
    CN_CUDA(cudaMemcpy(tl->d_win_items, items.data(), items.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_win_item, win_item.data(), b_wi, cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_titem, titem.data(), b_ti, cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_win_t, win_t.data(), b_wt, cudaMemcpyHostToDevice));
  tl->win_elems = win_elems;
  tl->win_chunk_q = chunk_q;
  tl->n_windows = K;
  tl->n_items = int64_t(items.size());
  tl->win_calls = 0;
  tl->win_blocks = 0;
  return COCONET_OK;
}

// ONCHIP plan. Items are the segments of rank 0's CSR lists (tensor order)
// cut into chunks of chunk_q quads; item i belongs to CTA i mod blocks, so a
// window of at most blocks * hold items gives every CTA at most `hold` of
// them to keep on chip. Windows hold whole tensors: a tensor of more items
// is a window alone and its CTAs spill the items beyond `hold`.
int tlist_onchip_plan(coconet_tlist* tl, int blocks, int hold, int chunk_q, int head, int head2) {
  if (tl->oc_mem && tl->oc_blocks == blocks && tl->oc_hold == hold && tl->oc_chunk_q == chunk_q &&
      tl->oc_head == head && tl->oc_head2 == head2)
    return COCONET_OK;
  const int64_t* ptr = tl->csr_ptr.data() + tl->csr_begin[0];
  std::vector<OcItem> items;
  std::vector<int64_t> wi{0}, titem{0};
  std::vector<int> tfirst{0};
  const int64_t cap = int64_t(blocks) * hold;
  int max_t = 0;
  for (int t = 0; t < tl->n_tensors; ++t) {
    const int64_t before = int64_t(items.size());
    for (int64_t i = ptr[t]; i < ptr[t + 1]; ++i) {
      const Seg& sg = tl->table[size_t(tl->csr_idx[size_t(i)])];
      const int len = meta_len(sg.meta);
      const int64_t q0 = sg.toff >> 2, q1 = (sg.toff + len + 3) >> 2;
      for (int64_t qa = q0; qa < q1; qa += chunk_q) items.push_back(OcItem{sg.toff, sg.sidx, qa, len, t});
    }
    titem.push_back(int64_t(items.size()));
    // close the open window before t when t does not fit in it
    const int64_t wb = wi.back();
    const int nt = t - tfirst.back();
    if (nt > 0 && (int64_t(items.size()) - wb > cap || nt >= kOcMaxTensors)) {
      wi.push_back(before);
      tfirst.push_back(t);
      max_t = std::max(max_t, nt);
    }
  }
  if (tl->n_tensors > tfirst.back()) {
    wi.push_back(int64_t(items.size()));
    max_t = std::max(max_t, tl->n_tensors - tfirst.back());
    tfirst.push_back(tl->n_tensors);
  }
  const int K = int(wi.size()) - 1;
  // elements of the items a CTA does not hold (its j-th of n items of a
  // window: j >= hold, or one of the head2 cover items after the head; the
  // kernel's oc_held)
  int64_t spilled = 0;
  for (int w = 0; w < K; ++w)
    for (int64_t i = wi[size_t(w)]; i < wi[size_t(w) + 1]; ++i) {
      const int64_t c = i % blocks;
      int64_t f = wi[size_t(w)] + ((c - wi[size_t(w)]) % blocks + blocks) % blocks;
      const int64_t j = (i - f) / blocks, n = (wi[size_t(w) + 1] - 1 - f) / blocks + 1;
      const int64_t h = std::min<int64_t>(head, n), h2 = std::min<int64_t>(head2, n - h);
      if (j < hold && !(j >= h && j < h + h2)) continue;
      const OcItem& it = items[size_t(i)];
      const int64_t e0 = std::max(it.toff, it.qa * 4), e1 = std::min(it.toff + it.len, (it.qa + chunk_q) * 4);
      spilled += e1 - e0;
    }
  if (tl->oc_mem) {
    cudaDeviceSynchronize();
    cudaFree(tl->oc_mem);
    tl->oc_mem = nullptr;
  }
  auto al = [](size_t n) { return (std::max<size_t>(n, 1) + 255) / 256 * 256; };
  const size_t b_items = al(items.size() * sizeof(OcItem)), b_wi = al(wi.size() * sizeof(int64_t));
  const size_t b_tf = al(tfirst.size() * sizeof(int)), b_ti = al(titem.size() * sizeof(int64_t));
  const size_t b_part = al(size_t(tl->n_tensors) * blocks * sizeof(double2)), b_cnt = al(size_t(K + 1 + tl->n_tensors) * sizeof(uint32_t));
  CN_CUDA(cudaMalloc(&tl->oc_mem, b_items + b_wi + b_tf + b_ti + b_part + b_cnt));
  char* p = static_cast<char*>(tl->oc_mem);
  tl->d_oc_items = reinterpret_cast<OcItem*>(p);
  tl->d_oc_wi = reinterpret_cast<int64_t*>(p += b_items);
  tl->d_oc_tfirst = reinterpret_cast<int*>(p += b_wi);
  tl->d_oc_titem = reinterpret_cast<int64_t*>(p += b_tf);
  tl->d_oc_part = reinterpret_cast<double2*>(p += b_ti);
  tl->d_oc_cnt = reinterpret_cast<uint32_t*>(p += b_part);
  if (!items.empty())
    CN_CUDA(cudaMemcpy(tl->d_oc_items, items.data(), items.size() * sizeof(OcItem), cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_oc_wi, wi.data(), wi.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_oc_tfirst, tfirst.data(), tfirst.size() * sizeof(int), cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemcpy(tl->d_oc_titem, titem.data(), titem.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  CN_CUDA(cudaMemset(tl->d_oc_cnt, 0, b_cnt));
  tl->oc_blocks = blocks;
  tl->oc_hold = hold;
  tl->oc_head = head;
  tl->oc_head2 = head2;
  tl->oc_chunk_q = chunk_q;
  tl->oc_K = K;
  tl->oc_n_items = int64_t(items.size());
  tl->oc_max_t = max_t;
  tl->oc_spilled = spilled;
  return COCONET_OK;
}

int tlist_bind(coconet_tlist* tl, const void* const* a, const void* const* b, int a_elem_bytes,
               int b_elem_bytes, cudaStream_t stream) {
  const coconet_ctx* c = tl->ctx;
  if (!c || !tl->dev_mem) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list has no device table (plan-only)");
  std::vector<int64_t> offs(size_t(tl->n_tensors) * 2);
  for (int i = 0; i < tl->n_tensors; ++i) {
    int64_t oa = 0, ob = 0;
    int rc = heap_offset(c, a[i], &oa);
    if (rc) return rc;
    rc = heap_offset(c, b[i], &ob);
    if (rc) return rc;
    if ((oa % (4 * a_elem_bytes)) || (ob % (4 * b_elem_bytes)))
      return set_error(COCONET_ERR_INVALID_INPUT,
                       "tensor " + std::to_string(i) + " is not aligned to 4 elements");
    if (oa + tl->counts[size_t(i)] * a_elem_bytes > int64_t(c->heap_bytes) ||
        ob + tl->counts[size_t(i)] * b_elem_bytes > int64_t(c->heap_bytes))
      return set_error(COCONET_ERR_INVALID_INPUT, "tensor " + std::to_string(i) + " overruns the heap");
    offs[size_t(i)] = oa;
    offs[size_t(tl->n_tensors + i)] = ob;
  }
  if (offs != tl->last_offs) {
    CN_CUDA(cudaMemcpyAsync(tl->d_offs, offs.data(), offs.size() * sizeof(int64_t),
                            cudaMemcpyHostToDevice, stream));
    tl->last_offs = offs;
  }
  return COCONET_OK;
}

}  // namespace coconet
