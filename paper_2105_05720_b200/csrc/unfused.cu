// The unfused GPU baseline the north star measures the fused kernels against
// ("NCCL plus separate kernels"; the paper's LAMB comparison point is PyTorch
// DDP's AllReduce followed by apex FusedLAMB). This is that
// optimizer half: the same LAMB step as apex FusedLAMB's separate multi-tensor
// kernels, over a group-size-1 tensor list (every rank updates every element
// after the all-reduce, replicated state):
//   1. stage 1      g, m, v, p -> m', v' and the update direction u (scratch)
//   2. l2norm       per-segment partial sums of p^2 and u^2
//   3. combine      per-tensor norms (segment CSR, fixed order)
//   4. stage 2      p -= lr * ||p|| / ||u|| * u
// HBM bytes per element at fp16 g: 26 + 8 + 12 = 46, against the fused
// kernel's 38 (it keeps u in registers and folds the norms into its passes).
// Same element math as the fused FAST kernel (fp32, fp64 norms).
#include <algorithm>
#include <cmath>

#include "fused_opt.h"

using namespace coconet;

namespace {

constexpr int kThreads = 256;

struct UnArgs {
  const Seg* segs;      // the size-1 group's segment table
  const int64_t* offs;  // [0,n): g heap offsets, [n,2n): p heap offsets
  int n_tensors;
  int64_t seg0, n_segs;  // the group's segments [seg0, seg0 + n_segs) of the table
  char* heap;
  int64_t m_off, v_off, u_off;
  const int64_t* csr_ptr;
  const int64_t* csr_idx;
  double* seg_part;  // [seg][2]
  double* tnorm;     // [tensor][2]
};

struct UnK {
  double lr;
  float fb1, fb2, fcm, fcv, frbc1, frbc2, feps, fwd;
  int guard;
};

template <typename G>
__device__ __forceinline__ void load_g4(const G* p, float o[4]) {
  if constexpr (sizeof(G) == 4) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
  } else {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    const G* h = reinterpret_cast<const G*>(&x);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = to_f32(h[i]);
  }
}

__device__ __forceinline__ void ld4f(const float* p, float o[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
}

// masked quad store (partial quads at segment edges lane by lane)
__device__ __forceinline__ void st4f(float* p, const float v[4], int lo, int hi) {
  if (lo == 0 && hi == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i >= lo && i < hi) p[i] = v[i];
  }
}

struct SegView {
  int64_t toff, sidx, aoff, boff, q0, q1;
  int len, tensor;
};

__device__ __forceinline__ SegView seg_view(const UnArgs& a, int64_t s) {
  const Seg sg = a.segs[s];
  SegView d;
  d.toff = sg.toff;
  d.sidx = sg.sidx;
  d.len = meta_len(sg.meta);
  d.tensor = meta_tensor(sg.meta);
  d.aoff = a.offs[d.tensor];
  d.boff = a.offs[a.n_tensors + d.tensor];
  d.q0 = d.toff >> 2;
  d.q1 = (d.toff + d.len + 3) >> 2;
  return d;
}

// 1. stage 1: m' = b1*m + (1-b1)*g ; v' = b2*v + (1-b2)*g^2 ; u = m'/bc1/(sqrt(v'/bc2)+eps) + wd*p
template <typename G>
__global__ void __launch_bounds__(kThreads) unfused_stage1(UnArgs a, UnK k) {
  float* m = reinterpret_cast<float*>(a.heap + a.m_off);
  float* v = reinterpret_cast<float*>(a.heap + a.v_off);
  float* u = reinterpret_cast<float*>(a.heap + a.u_off);
  for (int64_t s = a.seg0 + blockIdx.x; s < a.seg0 + a.n_segs; s += gridDim.x) {
    const SegView d = seg_view(a, s);
    for (int64_t q = d.q0 + threadIdx.x; q < d.q1; q += kThreads) {
      const int64_t e0 = q << 2, si = d.sidx + (e0 - d.toff);
      const int lo = int(max(int64_t(0), d.toff - e0)), hi = int(min(int64_t(4), d.toff + d.len - e0));
      float g[4], mm[4], vv[4], pp[4], uu[4];
      load_g4(reinterpret_cast<const G*>(a.heap + d.aoff) + e0, g);
      ld4f(m + si, mm);
      ld4f(v + si, vv);
      ld4f(reinterpret_cast<const float*>(a.heap + d.boff) + e0, pp);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mm[i] = fmaf(k.fcm, g[i], mm[i] * k.fb1);
        vv[i] = fmaf(k.fcv * g[i], g[i], vv[i] * k.fb2);
        uu[i] = __fdividef(mm[i] * k.frbc1, sqrtf(vv[i] * k.frbc2) + k.feps) + k.fwd * pp[i];
      }
      st4f(m + si, mm, lo, hi);
      st4f(v + si, vv, lo, hi);
      st4f(u + si, uu, lo, hi);
    }
  }
}

__device__ __forceinline__ double block_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) t += red[i];
  return t;
}

// 2. l2norm partials: sum p^2 and u^2 per segment (fixed order)
__global__ void __launch_bounds__(kThreads) unfused_norms(UnArgs a) {
  __shared__ double red[kThreads / 32];
  const float* u = reinterpret_cast<const float*>(a.heap + a.u_off);
  for (int64_t s = a.seg0 + blockIdx.x; s < a.seg0 + a.n_segs; s += gridDim.x) {
    const SegView d = seg_view(a, s);
    float sp = 0.f, su = 0.f;
    for (int64_t q = d.q0 + threadIdx.x; q < d.q1; q += kThreads) {
      const int64_t e0 = q << 2, si = d.sidx + (e0 - d.toff);
      const int lo = int(max(int64_t(0), d.toff - e0)), hi = int(min(int64_t(4), d.toff + d.len - e0));
      float pp[4], uu[4];
      ld4f(reinterpret_cast<const float*>(a.heap + d.boff) + e0, pp);
      ld4f(u + si, uu);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i >= lo && i < hi) {
          sp = fmaf(pp[i], pp[i], sp);
          su = fmaf(uu[i], uu[i], su);
        }
    }
    const double tp = block_sum(double(sp), red);
    const double tu = block_sum(double(su), red);
    if (threadIdx.x == 0) {
      a.seg_part[2 * s] = tp;
      a.seg_part[2 * s + 1] = tu;
    }
  }
}

// 3. per-tensor norms from the segment partials (CSR order)
__global__ void __launch_bounds__(kThreads) unfused_combine(UnArgs a) {
  const int64_t t = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  if (t >= a.n_tensors) return;
  double P = 0.0, U = 0.0;
  for (int64_t i = a.csr_ptr[t]; i < a.csr_ptr[t + 1]; ++i) {
    P += a.seg_part[2 * a.csr_idx[i]];
    U += a.seg_part[2 * a.csr_idx[i] + 1];
  }
  a.tnorm[2 * t] = P;
  a.tnorm[2 * t + 1] = U;
}

// 4. stage 2: p -= ratio * u
__global__ void __launch_bounds__(kThreads) unfused_stage2(UnArgs a, UnK k) {
  const float* u = reinterpret_cast<const float*>(a.heap + a.u_off);
  for (int64_t s = a.seg0 + blockIdx.x; s < a.seg0 + a.n_segs; s += gridDim.x) {
    const SegView d = seg_view(a, s);
    const double P = a.tnorm[2 * d.tensor], U = a.tnorm[2 * d.tensor + 1];
    const float ratio = (k.guard && (P == 0.0 || U == 0.0)) ? float(k.lr) : float((k.lr * sqrt(P)) / sqrt(U));
    float* p = reinterpret_cast<float*>(a.heap + d.boff);
    for (int64_t q = d.q0 + threadIdx.x; q < d.q1; q += kThreads) {
      const int64_t e0 = q << 2, si = d.sidx + (e0 - d.toff);
      const int lo = int(max(int64_t(0), d.toff - e0)), hi = int(min(int64_t(4), d.toff + d.len - e0));
      float pp[4], uu[4];
      ld4f(p + e0, pp);
      ld4f(u + si, uu);
#pragma unroll
      for (int i = 0; i < 4; ++i) pp[i] -= ratio * uu[i];
      st4f(p + e0, pp, lo, hi);
    }
  }
}

}  // namespace

extern "C" {

int coconet_unfused_lamb(coconet_ctx_t c, coconet_tlist_t tl, const void* const* g, int g_elem, float* const* p,
                         float* m, float* v, float* u_scratch, double* norms_scratch,
                         const coconet_lamb_params* hp, void* stream_) {
  if (!c || !tl || !g || !p || !m || !v || !u_scratch || !norms_scratch || !hp)
    return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (tl->ctx != c) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list belongs to another context");
  if (c->groups[size_t(tl->group)].size != 1)
    return set_error(COCONET_ERR_UNSUPPORTED, "the unfused baseline updates a size-1 group's list (replicated state)");
  if (g_elem < COCONET_F32 || g_elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  int rc = tlist_bind(tl, g, reinterpret_cast<const void* const*>(p), g_elem == COCONET_F32 ? 4 : 2, 4, s);
  if (rc) return rc;
  UnArgs a{};
  a.segs = tl->d_segs;
  a.seg0 = tl->seg_begin[0];
  a.offs = tl->d_offs;
  a.n_tensors = tl->n_tensors;
  a.n_segs = tl->seg_begin[1] - tl->seg_begin[0];
  a.heap = c->heap[c->mode == COCONET_MODE_VIRTUAL ? c->groups[size_t(tl->group)].first : c->rank];
  rc = heap_offset(c, m, &a.m_off);
  if (!rc) rc = heap_offset(c, v, &a.v_off);
  if (!rc) rc = heap_offset(c, u_scratch, &a.u_off);
  if (rc) return rc;
  if ((a.m_off | a.v_off | a.u_off) % 16) return set_error(COCONET_ERR_INVALID_INPUT, "state buffers must be 16-byte aligned");
  a.csr_ptr = tl->d_csr_ptr + tl->csr_begin[0];
  a.csr_idx = tl->d_csr_idx;
  a.seg_part = tl->d_seg_part;
  a.tnorm = norms_scratch;
  UnK k{};
  k.lr = double(hp->lr);
  k.fb1 = hp->beta1;
  k.fb2 = hp->beta2;
  k.fcm = float(1.0 - double(hp->beta1));
  k.fcv = float(1.0 - double(hp->beta2));
  k.frbc1 = float(1.0 / (1.0 - std::pow(double(hp->beta1), double(hp->t))));
  k.frbc2 = float(1.0 / (1.0 - std::pow(double(hp->beta2), double(hp->t))));
  k.feps = hp->eps;
  k.fwd = hp->wd;
  k.guard = hp->trust_guard;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(a.n_segs, int64_t(c->sm_count) * 8)));
  if (g_elem == COCONET_F32) unfused_stage1<float><<<grid, kThreads, 0, s>>>(a, k);
  else if (g_elem == COCONET_F16) unfused_stage1<__half><<<grid, kThreads, 0, s>>>(a, k);
  else unfused_stage1<__nv_bfloat16><<<grid, kThreads, 0, s>>>(a, k);
  unfused_norms<<<grid, kThreads, 0, s>>>(a);
  unfused_combine<<<unsigned((tl->n_tensors + kThreads - 1) / kThreads), kThreads, 0, s>>>(a);
  unfused_stage2<<<grid, kThreads, 0, s>>>(a, k);
  CN_CUDA(cudaGetLastError());
  c->launches += 4;
  return COCONET_OK;
}

}  // extern "C"
