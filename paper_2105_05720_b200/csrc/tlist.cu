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
// Segment tables built once on the host:
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
  int64_t toff, sidx;
  int32_t tensor, len, owner;
  int64_t flat;
};

}  // namespace

extern "C" {

int coconet_tlist_create(coconet_ctx_t c, int group, int n_tensors, const int64_t* counts,
                         int64_t bucket_cap, coconet_tlist_t* out) {
  if (!c || !out || !counts) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  *out = nullptr;
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  if (n_tensors < 1) return set_error(COCONET_ERR_INVALID_INPUT, "empty tensor list");
  if (bucket_cap < 4 || bucket_cap > (1 << 20) || (bucket_cap & 3))
    return set_error(COCONET_ERR_INVALID_INPUT, "bucket capacity must be a multiple of 4 in [4, 2^20]");
  const int W = c->groups[size_t(group)].size;
  auto* tl = new coconet_tlist();
  tl->ctx = c;
  tl->group = group;
  tl->n_tensors = n_tensors;
  tl->bucket_cap = bucket_cap;
  tl->counts.assign(counts, counts + n_tensors);
  for (int i = 0; i < n_tensors; ++i) {
    if (counts[i] <= 0) {
      delete tl;
      // build_bucket_table: "tensor has no elements" (runtime.hpp:596)
      return set_error(COCONET_ERR_INVALID_INPUT, "tensor " + std::to_string(i) + " has no elements");
    }
    tl->total += counts[i];
  }
  if (tl->total < W) {
    delete tl;
    return set_error(COCONET_ERR_DIVISIBILITY, "fewer bucketed elements than ranks");
  }
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
  std::vector<Seg> table;
  table.reserve(pieces.size() * 2);
  int64_t shard_max = 0;
  tl->seg_begin[0] = 0;
  size_t pi = 0;
  for (int r = 0; r < W; ++r) {
    int64_t cur = 0;
    while (pi < pieces.size() && pieces[pi].owner == r) {
      HostSeg& p = pieces[pi++];
      cur += ((p.toff & 3) - (cur & 3) + 4) & 3;
      Seg s;
      s.toff = p.toff;
      s.sidx = cur;
      s.meta = pack_meta(p.tensor, p.len, r);
      table.push_back(s);
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
    Seg s;
    s.toff = p.toff;
    s.sidx = cur;
    s.meta = pack_meta(p.tensor, p.len, p.owner);
    table.push_back(s);
    cur += p.len;
  }
  tl->os_end = int64_t(table.size());
  tl->full_state_elems = (cur + 3) & ~int64_t(3);
  // per-tensor segment lists of each rank (TWO_SHOT), for deterministic
  // per-tensor reductions (LAMB): CSR over [seg_begin[r], seg_begin[r+1])
  std::vector<int64_t> csr_ptr, csr_idx;
  for (int r = 0; r < W; ++r) {
    std::vector<std::vector<int64_t>> per(static_cast<size_t>(n_tensors));
    for (int64_t s = tl->seg_begin[r]; s < tl->seg_begin[r + 1]; ++s)
      per[size_t(meta_tensor(table[size_t(s)].meta))].push_back(s);
    tl->csr_begin[r] = int64_t(csr_ptr.size());
    int64_t acc = int64_t(csr_idx.size());
    for (int t = 0; t < n_tensors; ++t) {
      csr_ptr.push_back(acc);
      for (auto s : per[size_t(t)]) csr_idx.push_back(s);
      acc = int64_t(csr_idx.size());
    }
    csr_ptr.push_back(acc);
  }
  tl->n_segs = int64_t(table.size());
  size_t bytes_segs = table.size() * sizeof(Seg);
  size_t bytes_ptr = csr_ptr.size() * sizeof(int64_t);
  size_t bytes_idx = std::max<size_t>(1, csr_idx.size()) * sizeof(int64_t);
  size_t bytes_offs = size_t(n_tensors) * 2 * sizeof(int64_t);
  size_t bytes_part = size_t(table.size()) * 2 * sizeof(double);
  size_t total = bytes_segs + bytes_ptr + bytes_idx + bytes_offs + bytes_part + 5 * 256;
  cudaError_t e = cudaMalloc(&tl->dev_mem, total);
  if (e != cudaSuccess) {
    delete tl;
    return cuda_fail(e, "tlist cudaMalloc");
  }
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
  tl->metadata_bytes = int64_t(bytes_segs);
  e = cudaMemcpy(tl->d_segs, table.data(), bytes_segs, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(tl->d_csr_ptr, csr_ptr.data(), bytes_ptr, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !csr_idx.empty())
    e = cudaMemcpy(tl->d_csr_idx, csr_idx.data(), csr_idx.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    coconet_tlist_destroy(tl);
    return cuda_fail(e, "tlist upload");
  }
  tl->last_offs.assign(size_t(n_tensors) * 2, -1);
  *out = tl;
  return COCONET_OK;
}

int coconet_tlist_destroy(coconet_tlist_t tl) {
  if (!tl) return COCONET_OK;
  if (tl->dev_mem) {
    cudaDeviceSynchronize();
    cudaFree(tl->dev_mem);
  }
  delete tl;
  return COCONET_OK;
}

int64_t coconet_tlist_shard_elems(coconet_tlist_t tl) { return tl ? tl->shard_elems : -1; }
int64_t coconet_tlist_total(coconet_tlist_t tl) { return tl ? tl->total : -1; }
int64_t coconet_tlist_state_elems(coconet_tlist_t tl) { return tl ? tl->full_state_elems : -1; }
int64_t coconet_tlist_buckets(coconet_tlist_t tl) { return tl ? tl->n_buckets : -1; }
int64_t coconet_tlist_metadata_bytes(coconet_tlist_t tl) { return tl ? tl->metadata_bytes : -1; }

int coconet_tlist_chunk(coconet_tlist_t tl, int r, int64_t* lo, int64_t* hi) {
  if (!tl) return set_error(COCONET_ERR_INVALID_INPUT, "null tlist");
  int W = tl->ctx->groups[size_t(tl->group)].size;
  if (r < 0 || r >= W) return set_error(COCONET_ERR_NO_SUCH_RANK, "rank out of range");
  if (lo) *lo = tl->chunk_lo[r];
  if (hi) *hi = tl->chunk_lo[r + 1];
  return COCONET_OK;
}

int64_t coconet_tlist_shard_index(coconet_tlist_t tl, int64_t pos) {
  if (!tl || pos < 0 || pos >= tl->total) return -1;
  // segments are ordered by flat position across ranks
  auto it = std::upper_bound(tl->host_flat.begin(), tl->host_flat.end(), pos);
  size_t s = size_t(it - tl->host_flat.begin()) - 1;
  return tl->host_sidx[s] + (pos - tl->host_flat[s]);
}

}  // extern "C"

namespace coconet {

// Uploads per-tensor heap offsets of the g/x and p/out tensors when they
// changed since the last call (pageable source: the copy is staged before
// cudaMemcpyAsync returns, and it is stream-ordered after earlier kernels).
int tlist_bind(coconet_tlist* tl, const void* const* a, const void* const* b, int a_elem_bytes,
               int b_elem_bytes, cudaStream_t stream) {
  const coconet_ctx* c = tl->ctx;
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

extern "C" int64_t coconet_tlist_segments(coconet_tlist_t tl, int r, int64_t* tensor, int64_t* toff,
                                          int64_t* len, int64_t* sidx, int64_t cap) {
  if (!tl) return set_error(COCONET_ERR_INVALID_INPUT, "null tlist");
  int W = tl->ctx->groups[size_t(tl->group)].size;
  if (r < -1 || r >= W) return set_error(COCONET_ERR_NO_SUCH_RANK, "rank out of range");
  int64_t b = r < 0 ? tl->os_begin : tl->seg_begin[r];
  int64_t e = r < 0 ? tl->os_end : tl->seg_begin[r + 1];
  if (e - b > cap) return -(e - b);
  std::vector<Seg> h(size_t(e - b));
  if (e > b) {
    cudaError_t err = cudaMemcpy(h.data(), tl->d_segs + b, size_t(e - b) * sizeof(Seg), cudaMemcpyDeviceToHost);
    if (err != cudaSuccess) return cuda_fail(err, "segments D2H");
  }
  for (size_t i = 0; i < h.size(); ++i) {
    tensor[i] = meta_tensor(h[i].meta);
    toff[i] = h[i].toff;
    len[i] = meta_len(h[i].meta);
    sidx[i] = h[i].sidx;
  }
  return e - b;
}
