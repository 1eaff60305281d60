// Synthetic inputs on the device, bit-exact with gen_decl_values
// (state.hpp:55-74): value(gi) = float(0.1 + 0.8 * counter_uniform(seed, key,
// gi)), key = fnv1a(name) ^ (rank+1)*phi for Local decls (rank-independent
// otherwise); a Sliced(d) decl stores only the rank's slice, element li of
// the slice being global index DistView::to_global(rank, li) (view.hpp:62-70).
// Generating on the device avoids a bulk H2D copy of the workload.
#include "internal.h"

using namespace coconet;

namespace {

struct GenArgs {
  uint64_t seed, key;
  int64_t n_local;
  // sliced map: gi = (before*G_d + rank*per + lc)*stride_d + after
  int sliced;
  int64_t stride_d, per, global_d;
  int rank;
};

__device__ __forceinline__ int64_t to_global(const GenArgs& a, int64_t li) {
  if (!a.sliced) return li;
  int64_t before = li / (a.stride_d * a.per);
  int64_t lc = (li / a.stride_d) % a.per;
  int64_t after = li % a.stride_d;
  return (before * a.global_d + int64_t(a.rank) * a.per + lc) * a.stride_d + after;
}

template <typename T>
__global__ void __launch_bounds__(256) gen_kernel(T* __restrict__ dst, GenArgs a) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n_local; i += stride) {
    const double u = counter_uniform(a.seed, a.key, uint64_t(to_global(a, i)));
    dst[i] = from_f32<T>(float(0.1 + 0.8 * u));
  }
}

}  // namespace

extern "C" int coconet_gen_values(coconet_ctx_t c, void* dst, int out_elem, uint64_t seed,
                                  uint64_t name_key, int is_local, int rank, int ndim,
                                  const int64_t* shape, int sliced_dim, int group_size,
                                  void* stream) {
  if (!c || !dst) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (ndim < 0 || ndim > 8 || (ndim > 0 && !shape)) return set_error(COCONET_ERR_INVALID_INPUT, "bad shape");
  if (group_size < 1 || rank < 0 || rank >= group_size) return set_error(COCONET_ERR_NO_SUCH_RANK, "bad rank");
  GenArgs a{};
  a.seed = seed;
  a.key = is_local ? name_key ^ (uint64_t(rank + 1) * 0x9e3779b97f4a7c15ull) : name_key;
  int64_t total = 1;
  for (int i = 0; i < ndim; ++i) total *= shape[i];
  a.rank = rank;
  a.sliced = sliced_dim >= 0;
  if (a.sliced) {
    if (sliced_dim >= ndim) return set_error(COCONET_ERR_INVALID_INPUT, "sliced dim out of range");
    if (shape[sliced_dim] % group_size)
      return set_error(COCONET_ERR_DIVISIBILITY, "extent " + std::to_string(shape[sliced_dim]) +
                                                     " over " + std::to_string(group_size) + " ranks");
    a.global_d = shape[sliced_dim];
    a.per = shape[sliced_dim] / group_size;
    a.stride_d = 1;
    for (int i = sliced_dim + 1; i < ndim; ++i) a.stride_d *= shape[i];
    a.n_local = total / group_size;
  } else {
    a.n_local = total;
  }
  if (a.n_local == 0) return COCONET_OK;
  int64_t blocks = (a.n_local + 255) / 256;
  if (blocks > int64_t(c->sm_count) * 16) blocks = int64_t(c->sm_count) * 16;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (out_elem) {
    case COCONET_F32: gen_kernel<float><<<unsigned(blocks), 256, 0, s>>>(static_cast<float*>(dst), a); break;
    case COCONET_F16: gen_kernel<__half><<<unsigned(blocks), 256, 0, s>>>(static_cast<__half*>(dst), a); break;
    case COCONET_BF16:
      gen_kernel<__nv_bfloat16><<<unsigned(blocks), 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), a);
      break;
    default: return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  }
  CN_CUDA(cudaGetLastError());
  c->launches++;
  return COCONET_OK;
}
