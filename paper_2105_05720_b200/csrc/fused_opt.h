// Tensor-list structures shared by the fused optimizer and AllReduce kernels.
#pragma once

#include <vector>

#include "internal.h"

namespace coconet {

// One unit of work: a bucket (or the part of a bucket inside one flat chunk)
// of one tensor. 24 bytes; read once per segment by a whole warp (broadcast).
struct Seg {
  int64_t toff;  // element offset inside the tensor
  int64_t sidx;  // index of the first element in shard/state storage (== toff mod 4)
  int64_t meta;  // tensor (32 bits) | len (24 bits) | owner rank (8 bits)
};

// One STREAMED-LAMB work item: a segment whose meta carries its pass in bit 7
// of the owner byte (0: RS + m/v update + norm partials, 1: trust ratio +
// p update + AG); the owner of a TWO_SHOT segment is the rank itself.
using Item = Seg;
constexpr int64_t kPass2Bit = 0x80;

// One ONCHIP-LAMB chunk item: quads [qa, min(qa + chunk, end of segment)) of
// the segment (toff, len, sidx) of `tensor`. 32 bytes, read by the producer.
struct OcItem {
  int64_t toff, sidx, qa;
  int len, tensor;
};
constexpr int kOcMaxTensors = 96;  // tensors per ONCHIP window (shared-memory ratio table)

__host__ __device__ __forceinline__ int64_t pack_meta(int tensor, int len, int owner) {
  return (int64_t(tensor) << 32) | (int64_t(len & 0xffffff) << 8) | int64_t(owner & 0xff);
}
__host__ __device__ __forceinline__ int meta_tensor(int64_t m) { return int(m >> 32); }
__host__ __device__ __forceinline__ int meta_len(int64_t m) { return int((m >> 8) & 0xffffff); }
__host__ __device__ __forceinline__ int meta_owner(int64_t m) { return int(m & 0x7f); }
__host__ __device__ __forceinline__ int meta_pass(int64_t m) { return (m & kPass2Bit) ? 1 : 0; }

}  // namespace coconet

struct coconet_tlist {
  coconet_ctx* ctx = nullptr;  // null for a plan-only list (coconet_tlist_plan)
  int group = 0;
  int world = 1;
  int n_tensors = 0;
  int64_t bucket_cap = 1024;
  std::vector<int64_t> counts;
  int64_t total = 0;
  int64_t n_buckets = 0;
  int64_t n_segs = 0;
  int64_t chunk_lo[coconet::kMaxRanks + 1] = {};
  int64_t seg_begin[coconet::kMaxRanks + 1] = {};  // TWO_SHOT table of rank r
  int64_t csr_begin[coconet::kMaxRanks] = {};      // per-rank per-tensor segment lists
  int64_t os_begin = 0, os_end = 0;                // ONE_SHOT table
  int64_t shard_elems = 0;
  int64_t full_state_elems = 0;
  int64_t metadata_bytes = 0;
  std::vector<coconet::Seg> table;             // TWO_SHOT tables, then the ONE_SHOT table
  std::vector<int64_t> csr_ptr, csr_idx;
  std::vector<int64_t> host_flat, host_sidx;  // TWO_SHOT segments, flat order
  std::vector<int64_t> last_offs;
  void* dev_mem = nullptr;
  coconet::Seg* d_segs = nullptr;
  int64_t* d_csr_ptr = nullptr;
  int64_t* d_csr_idx = nullptr;
  int64_t* d_offs = nullptr;       // [2][n_tensors] heap offsets bound per call
  double* d_seg_part = nullptr;    // per-segment partial sums (LAMB)
  // STREAMED LAMB schedule (built on first use for a lag, tlist_stream_plan)
  int64_t stream_wave = -1;              // the lag the lists were built for
  int64_t item_begin[coconet::kMaxRanks + 1] = {};
  std::vector<coconet::Item> items;      // per rank, execution order (tlist_stream_plan)
  std::vector<int64_t> p1_first;         // [rank][tensor]: item index of the tensor's first pass-1 item
  std::vector<uint32_t> holders;         // [tensor]: bitmask of ranks holding segments of it
  void* stream_mem = nullptr;
  coconet::Item* d_items = nullptr;
  int64_t* d_p1_first = nullptr;
  uint32_t* d_holders = nullptr;
  uint32_t* d_cnt = nullptr;             // [rank][tensor] pass-1 completion counters
  double* d_item_part = nullptr;         // per pass-1 item: sum p^2, sum u^2
  uint32_t stream_calls = 0;
  // WINDOWED LAMB schedule (W = 1): consecutive-tensor windows of about
  // win_elems elements, cut into chunk items (built on first use,
  // tlist_window_plan)
  int64_t win_elems = -1;
  int win_chunk_q = 0;
  int n_windows = 0;
  int64_t n_items = 0;
  void* win_mem = nullptr;
  int64_t* d_win_items = nullptr;  // [n_items] segment | chunk << 40, window by window, tensor-major
  int64_t* d_win_item = nullptr;   // [K+1] item range of each window
  int64_t* d_titem = nullptr;      // [n_tensors+1] item range of each tensor
  int* d_win_t = nullptr;          // [K+1] first tensor of each window
  float2* d_ipart = nullptr;       // [n_items] per-item norm partials
  float* d_ratio = nullptr;        // [n_tensors] trust ratios
  void* win_state = nullptr;       // the cumulative counters below, zeroed together
  size_t win_state_bytes = 0;
  unsigned long long* d_win_tick = nullptr;  // [K][2] tickets
  uint32_t* d_win_cnt = nullptr;   // [K] pass-1 arrivals
  uint32_t* d_win_ready = nullptr; // [K] call number once a window's ratios are published
  uint32_t win_calls = 0;
  int win_blocks = 0;              // grid size the counters were advanced with
  // ONCHIP LAMB schedule (group size 1): windows of whole tensors sized so that
  // every CTA holds its share of a window's u on chip (TMEM + shared memory),
  // built on first use for a grid size / hold depth (tlist_onchip_plan)
  int oc_blocks = 0, oc_hold = 0, oc_chunk_q = 0, oc_K = 0, oc_head = 0, oc_head2 = 0;
  int64_t oc_n_items = 0;
  void* oc_mem = nullptr;
  coconet::OcItem* d_oc_items = nullptr;  // [n_items] chunk items, tensor-major
  int64_t* d_oc_wi = nullptr;             // [K+1] item range of each window
  int* d_oc_tfirst = nullptr;             // [K+1] tensor range of each window
  int64_t* d_oc_titem = nullptr;          // [n_tensors+1] first item of each tensor
  double2* d_oc_part = nullptr;           // [n_tensors][blocks] per-CTA (sum p^2, sum u^2)
  uint32_t* d_oc_cnt = nullptr;           // [K] pass-1 arrivals, [K] CTAs out (zeroed by the last CTA)
  int oc_max_t = 0;                       // most tensors in one window
  int64_t oc_spilled = 0;                 // elements of items beyond a CTA's hold (pass 2 re-reads m', v')
};

namespace coconet {
// Builds (or keeps) the STREAMED-LAMB work lists for a pass-1 -> pass-2 lag
// of `lag` elements; uploads them when the list has a device table.
int tlist_stream_plan(coconet_tlist* tl, int64_t lag);
// Builds (or keeps) the WINDOWED-LAMB windows for a target window size and
// chunk items of chunk_q quads.
int tlist_window_plan(coconet_tlist* tl, int64_t win_elems, int chunk_q);
// Builds (or keeps) the ONCHIP-LAMB plan: chunk items of chunk_q quads in
// tensor order, cut into windows of whole tensors of at most blocks * hold
// items (a longer tensor is a window alone) and kOcMaxTensors tensors.
// head / head2: the kernel's cover items (oc_held), so the spilled count
// includes the head2 cover items that take the m', v' re-read path
int tlist_onchip_plan(coconet_tlist* tl, int blocks, int hold, int chunk_q, int head = 1, int head2 = 0);
int tlist_bind(coconet_tlist* tl, const void* const* a, const void* const* b, int a_elem_bytes,
               int b_elem_bytes, cudaStream_t stream);
}
