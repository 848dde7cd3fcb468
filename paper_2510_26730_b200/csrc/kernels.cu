// kernels.cu — sm_100a kernels of the ExpertFlow MoE decode path and their
// C-ABI launchers (include/expertflow.h).
//
//   (a) ef_router_logits + ef_route_permute : router GEMV, top-k keyed on fp32
//       logits (+ cache-aware bias), routing weights, stable permutation
//   (b) ef_router_logits with R > 1          : future-layer pre-gate rows
//   (c) ef_route_permute / ef_combine        : permute, unpermute + combine
//   (d) ef_expert_ffn_decode                 : slot-indirected weight-streaming
//       GEMV (gate+up+SiLU fused, then down), 16-byte L1-bypassing loads,
//       warp-shuffle reductions
//   engine pipeline (pipeline.h): router_route_kernel / router_route_row_kernel
//       (router + route + previous combine + device-side slot resolution in one
//       launch), ffn_gemv_kernel with the gate folded into grid column 0
// Decode GEMVs are HBM-bound (arithmetic intensity ~ n_rows FLOP/B); they keep
// many independent 16 B loads in flight per lane instead of using tensor cores.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstddef>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/expertflow.h"
#include "kernels.cuh"
#include "pipeline.h"

// Programmatic dependent launch (PDL): the decode kernels start with
// griddepcontrol.wait (a no-op without a PDL primary), so a kernel launched
// with programmatic stream serialisation may be scheduled while its
// predecessor drains and only its launch latency overlaps — results are the
// same as with plain stream order.
namespace ef {
bool g_use_pdl = false;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... K, typename... A>
static cudaError_t launch_k(void (*kern)(K...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t c{};
  c.gridDim = grid;
  c.blockDim = block;
  c.dynamicSmemBytes = smem;
  c.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = at;
  c.numAttrs = ef::g_use_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&c, kern, std::forward<A>(args)...);
}

namespace ef {
extern thread_local std::string g_last_error;
}

using namespace efk;

#define EF_CUDA_RET(expr)                                                         \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ef::g_last_error = std::string(#expr) + ": " + cudaGetErrorString(_e);     \
      return EF_ECUDA;                                                            \
    }                                                                             \
  } while (0)

#define EF_CHECK_ARG(cond, msg)     \
  do {                                \
    if (!(cond)) {                    \
      ef::g_last_error = msg;         \
      return EF_EINVAL;               \
    }                                 \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ============================================================ synthetic weights
template <typename T>
__global__ void fill_uniform_kernel(T* dst, int64_t n, uint64_t key, float scale, int64_t offset) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t h = mix64(key + (uint64_t)(offset + i + 1) * kGolden);
    int32_t u = (int32_t)(h >> 40) - 8388608;
    float v = __fmul_rn((float)u, scale);
    WTraits<T>::store(dst + i, v);
  }
}

extern "C" uint64_t ef_stream_key(uint64_t seed, int32_t layer, int32_t expert, int32_t mat) {
  uint64_t tag = ((uint64_t)(uint32_t)layer << 32) | ((uint64_t)(uint32_t)expert << 8) |
                 (uint64_t)(uint32_t)mat;
  return mix64(seed ^ mix64(tag + kGolden));
}

extern "C" int ef_fill_uniform(void* stream, void* dst, int dtype, int64_t n, uint64_t key,
                               float scale, int64_t offset) {
  EF_CHECK_ARG(dst && n >= 0, "bad fill arguments");
  if (n == 0) return EF_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dtype == EF_BF16)
    fill_uniform_kernel<__nv_bfloat16><<<blocks, 256, 0, S(stream)>>>(
        (__nv_bfloat16*)dst, n, key, scale, offset);
  else
    fill_uniform_kernel<float><<<blocks, 256, 0, S(stream)>>>((float*)dst, n, key, scale, offset);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// ============================================================ rmsnorm
__device__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  float t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  float r = red[0];
  __syncthreads();
  return r;
}

__global__ void rmsnorm_kernel(const float* __restrict__ h, float* __restrict__ x, int d,
                               float eps) {
  __shared__ float red[32];
  const float* hr = h + (int64_t)blockIdx.x * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += hr[i] * hr[i];
  ss = block_sum(ss, red);
  float inv = 1.0f / sqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) x[(int64_t)blockIdx.x * d + i] = hr[i] * inv;
}

// v = h[t] + (sum_r wts[t,r] * y[inv[t,r]] in rank order + g_t * ys[t]) into
// vout (may alias h[t]); returns the block-wide sum of v^2.  float4 lanes with
// P passes in flight so the L2 round trips overlap (d % 4 == 0).  Any block
// size; all threads of the block must call it.
template <int P = 4>
__device__ float combine_row(int t, const float* h, float* vout, const float* __restrict__ y,
                             const int32_t* __restrict__ inv, const float* __restrict__ wts,
                             const float* __restrict__ ys, const float* __restrict__ gate_logit,
                             int d, int k, float* red) {
  const float g = gate_logit ? 1.0f / (1.0f + expf(-gate_logit[t])) : 1.f;
  const float* hr = h + (int64_t)t * d;
  const int step = blockDim.x * 4;
  float ss = 0.f;
  // routing weights and y rows of every rank in one round trip (k <= 16)
  float wr_s[16];
  int ir_s[16];
#pragma unroll
  for (int r = 0; r < 16; ++r)
    if (r < k) {
      wr_s[r] = __ldcg(wts + t * k + r);
      ir_s[r] = inv ? __ldcg(inv + t * k + r) : t * k + r;  // inv null: y in slot order
    }
  for (int base = threadIdx.x * 4; base < d; base += step * P) {
    float4 hv[P], sv[P], acc[P];
    // the first two ranks' y rows are issued with h, so at top-2 every load
    // of the row lands in one round trip
    float4 y0[P], y1[P];
    const float* yr0 = y + (int64_t)ir_s[0] * d;
    const float* yr1 = y + (int64_t)ir_s[k > 1 ? 1 : 0] * d;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int i = base + p * step;
      acc[p] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < d) {
        hv[p] = __ldcg(reinterpret_cast<const float4*>(hr + i));
        if (ys) sv[p] = __ldcg(reinterpret_cast<const float4*>(ys + (int64_t)t * d + i));
        y0[p] = __ldcg(reinterpret_cast<const float4*>(yr0 + i));
        if (k > 1) y1[p] = __ldcg(reinterpret_cast<const float4*>(yr1 + i));
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      acc[p].x = fmaf(wr_s[0], y0[p].x, acc[p].x);
      acc[p].y = fmaf(wr_s[0], y0[p].y, acc[p].y);
      acc[p].z = fmaf(wr_s[0], y0[p].z, acc[p].z);
      acc[p].w = fmaf(wr_s[0], y0[p].w, acc[p].w);
      if (k > 1) {
        acc[p].x = fmaf(wr_s[1], y1[p].x, acc[p].x);
        acc[p].y = fmaf(wr_s[1], y1[p].y, acc[p].y);
        acc[p].z = fmaf(wr_s[1], y1[p].z, acc[p].z);
        acc[p].w = fmaf(wr_s[1], y1[p].w, acc[p].w);
      }
    }
#pragma unroll
    for (int r = 2; r < 16; ++r) {
      if (r >= k) break;
      const float w = wr_s[r];
      const float* yr = y + (int64_t)ir_s[r] * d;
      float4 yv[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int i = base + p * step;
        if (i < d) yv[p] = __ldcg(reinterpret_cast<const float4*>(yr + i));
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        acc[p].x = fmaf(w, yv[p].x, acc[p].x);
        acc[p].y = fmaf(w, yv[p].y, acc[p].y);
        acc[p].z = fmaf(w, yv[p].z, acc[p].z);
        acc[p].w = fmaf(w, yv[p].w, acc[p].w);
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int i = base + p * step;
      if (i < d) {
        if (ys) {
          acc[p].x = fmaf(g, sv[p].x, acc[p].x);
          acc[p].y = fmaf(g, sv[p].y, acc[p].y);
          acc[p].z = fmaf(g, sv[p].z, acc[p].z);
          acc[p].w = fmaf(g, sv[p].w, acc[p].w);
        }
        float4 v;
        v.x = hv[p].x + acc[p].x;
        v.y = hv[p].y + acc[p].y;
        v.z = hv[p].z + acc[p].z;
        v.w = hv[p].w + acc[p].w;
        *reinterpret_cast<float4*>(vout + i) = v;
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
    }
  }
  return block_sum(ss, red);
}

// h[t] += sum_r wts[t,r] * y[inv[t,r]] (rank order) + g_t * ys[t]; x[t] = rmsnorm(h[t])
// (x null: h only).
__device__ void combine_token(int t, float* __restrict__ h, float* __restrict__ x,
                              const float* __restrict__ y, const int32_t* __restrict__ inv,
                              const float* __restrict__ wts, const float* __restrict__ ys,
                              const float* __restrict__ gate_logit, int d, int k, float eps,
                              float* red) {
  float* hr = h + (int64_t)t * d;
  const float ss = combine_row(t, h, hr, y, inv, wts, ys, gate_logit, d, k, red);
  if (!x) return;  // after the last layer: no next rmsnorm
  const float invn = 1.0f / sqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(hr + i);
    v.x *= invn;
    v.y *= invn;
    v.z *= invn;
    v.w *= invn;
    *reinterpret_cast<float4*>(x + (int64_t)t * d + i) = v;
  }
}

extern "C" int ef_rmsnorm(void* stream, const float* h, float* x, int B, int d, float eps) {
  EF_CHECK_ARG(B >= 0 && d > 0, "bad rmsnorm shape");
  if (B == 0) return EF_OK;
  rmsnorm_kernel<<<B, 1024, 0, S(stream)>>>(h, x, d, eps);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// ============================================================ (a)(b) router GEMV
// One warp per router row (r, m); all B tokens accumulate in registers while
// the row streams through once.  x is tiny and stays in L1/L2.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <typename WT, int MAXB>
__global__ void router_kernel(const float* __restrict__ x, const WT* __restrict__ w, int rows,
                              int B, int d, int M, float* __restrict__ logits,
                              unsigned long long* stamp) {
  constexpr int V = WTraits<WT>::kPer16;
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *stamp = gtimer();
  const int t0 = blockIdx.y * MAXB;  // token chunk of this CTA row
  const int nb = min(MAXB, B - t0);
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const WT* wr = w + (int64_t)warp * d;
  float acc[MAXB];
#pragma unroll
  for (int t = 0; t < MAXB; ++t) acc[t] = 0.f;
  for (int c = lane * V; c < d; c += 32 * V) {
    float f[V];
    WTraits<WT>::unpack(ld_stream16(wr + c), f);
#pragma unroll
    for (int t = 0; t < MAXB; ++t) {
      if (t < nb) {
        const float4* xp = reinterpret_cast<const float4*>(x + (int64_t)(t0 + t) * d + c);
#pragma unroll
        for (int q = 0; q < V / 4; ++q) {
          float4 xv = __ldg(xp + q);
          acc[t] = fmaf(f[4 * q + 0], xv.x, acc[t]);
          acc[t] = fmaf(f[4 * q + 1], xv.y, acc[t]);
          acc[t] = fmaf(f[4 * q + 2], xv.z, acc[t]);
          acc[t] = fmaf(f[4 * q + 3], xv.w, acc[t]);
        }
      }
    }
  }
  int r = warp / M, m = warp % M;
#pragma unroll
  for (int t = 0; t < MAXB; ++t) {
    if (t < nb) {
      float s = warp_sum(acc[t]);
      if (lane == 0) logits[((int64_t)r * B + t0 + t) * M + m] = s;
    }
  }
}

template <typename WT>
static void launch_router(cudaStream_t st, const float* x, const void* w, int R, int B, int d,
                          int M, float* logits, unsigned long long* stamp = nullptr) {
  const int rows = R * M, threads = 256;
  const int blocks = (rows * 32 + threads - 1) / threads;
  // one launch; grid.y walks token chunks of 8 (bounds the accumulators)
  if (B == 1)
    router_kernel<WT, 1><<<dim3(blocks, 1), threads, 0, st>>>(x, (const WT*)w, rows, B, d, M, logits,
                                                              stamp);
  else
    router_kernel<WT, 8><<<dim3(blocks, (B + 7) / 8), threads, 0, st>>>(x, (const WT*)w, rows, B, d,
                                                                          M, logits, stamp);
}

namespace ef {
int router_logits_stamped(cudaStream_t st, const float* x, const void* w, int dtype, int R, int B,
                          int d, int M, float* logits, unsigned long long* stamp) {
  if (B == 0) return EF_OK;
  if (dtype == EF_BF16)
    launch_router<__nv_bfloat16>(st, x, w, R, B, d, M, logits, stamp);
  else
    launch_router<float>(st, x, w, R, B, d, M, logits, stamp);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}
}  // namespace ef

extern "C" int ef_router_logits(void* stream, const float* x, const void* w, int dtype, int R,
                                int B, int d, int M, float* logits) {
  EF_CHECK_ARG(R >= 1 && B >= 0 && M >= 1, "bad router shape");
  EF_CHECK_ARG(d % (dtype == EF_BF16 ? 8 : 4) == 0, "router d must be a multiple of 8 (bf16) / 4");
  if (B == 0) return EF_OK;
  if (dtype == EF_BF16)
    launch_router<__nv_bfloat16>(S(stream), x, w, R, B, d, M, logits);
  else
    launch_router<float>(S(stream), x, w, R, B, d, M, logits);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// ============================================================ (a)+(c) route + permute
// One CTA of 1024 threads.  Top-k per token (value desc, index asc), routing
// weights, then a stable counting sort of the B*k (token, rank) slots by
// expert using warp match/ballot ranks — deterministic, O(B*k).
constexpr int kRouteThreads = 1024;
constexpr int kMaxExperts = 256;

struct RouteSmem {
  int32_t warp_cnt[32][kMaxExperts];
  int32_t base[kMaxExperts];
  int32_t total[kMaxExperts];
};

// Top-k of one token's logits by one warp (M <= 128), keyed on
// logit + bias for resident experts (value desc, index asc — SURVEY H6), and
// the routing weights from the raw logits.  sel/wts written by lane 0;
// sel_sh (optional) gets a shared-memory copy.
__device__ void topk_token(const float* __restrict__ lg, int M, int k, int mode, float bias,
                           uint64_t mlo, uint64_t mhi, int32_t* sel, float* wts, int32_t* sel_sh) {
  const int lane = threadIdx.x & 31;
  float v[4], key[4];
  bool taken[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < M ? __ldcg(lg + e) : -INFINITY;
    const bool res = e < 64 ? ((mlo >> e) & 1ull) : ((mhi >> (e - 64)) & 1ull);
    key[i] = (e < M && res && bias != 0.f) ? __fadd_rn(v[i], bias) : v[i];
    taken[i] = e >= M;
  }
  float mx_all = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx_all = fmaxf(mx_all, __shfl_xor_sync(0xffffffffu, mx_all, o));
  float chosen_v[16];
  int chosen_e[16];
  // fully unrolled over the 16 possible ranks so the arrays stay in registers
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    if (r >= k) break;
    float bk = 0.f;
    int be = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = lane + 32 * i;
      if (!taken[i] && (be == 0x7fffffff || key[i] > bk)) {
        bk = key[i];
        be = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      const bool other_better =
          oe != 0x7fffffff && (be == 0x7fffffff || ok > bk || (ok == bk && oe < be));
      if (other_better) {
        bk = ok;
        be = oe;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i == be) taken[i] = true;
    chosen_e[r] = be;
    // raw logit of the winner (weights ignore the bias), from its owning lane
    const int bi = be >> 5;
    const float mine = bi == 0 ? v[0] : bi == 1 ? v[1] : bi == 2 ? v[2] : v[3];
    chosen_v[r] = __shfl_sync(0xffffffffu, mine, be & 31);
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r >= k) break;
      sel[r] = chosen_e[r];
      if (sel_sh) sel_sh[r] = chosen_e[r];
    }
  }
  if (mode == EF_ROUTE_MIXTRAL) {
    if (lane == 0) {
      float mx = -INFINITY;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < k) mx = fmaxf(mx, chosen_v[r]);
      float ev[16], sum = 0.f;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r < k) {
          ev[r] = expf(chosen_v[r] - mx);
          sum += ev[r];
        }
      }
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < k) wts[r] = ev[r] / sum;
    }
  } else {
    float part = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < M) part += expf(v[i] - mx_all);
    const float sum = warp_sum(part);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < k) wts[r] = expf(chosen_v[r] - mx_all) / sum;
    }
  }
}

// Cache-aware routing mask top-up (oracle/numerics.py routing_mask; the rule
// is ours, the reference only reorders groups, engine.py:192-209).  When the
// host asks for U > 0 experts, the residents in (mlo, mhi) are joined by the
// best U - n non-resident experts by router votes: the number of tokens whose
// UNBIASED top-k (raw fp32 logits, value desc / index asc) contains the
// expert, then its largest logit over the batch, then the lower index — the
// set that changes the fewest tokens' selections.  Whole CTA; every thread
// gets the final mask.  All comparisons are exact (no arithmetic), so the
// oracle reproduces it bit for bit.
struct TopupSmem {
  int votes[kMaxExperts];
  int maxl[kMaxExperts];
  uint64_t m[2];
};
__device__ __forceinline__ int float_order(float f) {
  const int i = __float_as_int(__fadd_rn(f, 0.0f));  // -0 -> +0
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ bool mask_has(uint64_t lo, uint64_t hi, int e) {
  return e < 64 ? ((lo >> e) & 1ull) : ((hi >> (e - 64)) & 1ull);
}
struct CtaBar {
  __device__ void operator()() const { __syncthreads(); }
};
// tid / nthr: this thread's index in the participating group (the whole CTA,
// or one 4-warp worker of the persistent decode kernel) and its size
template <typename Bar = CtaBar>
__device__ void topup_mask(TopupSmem& ts, const float* __restrict__ logits, int B, int M, int k,
                           int U, uint64_t& mlo, uint64_t& mhi, int tid = -1, int nthr = 0,
                           Bar bar = Bar{}) {
  if (tid < 0) {
    tid = threadIdx.x;
    nthr = blockDim.x;
  }
  const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
  for (int e = tid; e < kMaxExperts; e += nthr) {
    ts.votes[e] = 0;
    ts.maxl[e] = INT_MIN;
  }
  bar();
  for (int t = wid; t < B; t += nw) {
    const float* lg = logits + (int64_t)t * M;
    float v[4];
    bool taken[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = lane + 32 * i;
      v[i] = e < M ? __ldcg(lg + e) : -INFINITY;
      taken[i] = e >= M;
      if (e < M) atomicMax(&ts.maxl[e], float_order(v[i]));
    }
    for (int r = 0; r < k; ++r) {
      float bk = 0.f;
      int be = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!taken[i] && (be == 0x7fffffff || v[i] > bk)) {
          bk = v[i];
          be = lane + 32 * i;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ok = __shfl_xor_sync(0xffffffffu, bk, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (oe != 0x7fffffff && (be == 0x7fffffff || ok > bk || (ok == bk && oe < be))) {
          bk = ok;
          be = oe;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (lane + 32 * i == be) taken[i] = true;
      if (lane == 0 && be != 0x7fffffff) atomicAdd(&ts.votes[be], 1);
    }
  }
  bar();
  if (wid == 0) {
    uint64_t lo = mlo, hi = mhi;
    int n = __popcll(lo) + __popcll(hi);
    for (; n < U; ++n) {
      int bv = -1, bm = INT_MIN, be = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = lane + 32 * i;
        if (e < M && !mask_has(lo, hi, e)) {
          const int cv = ts.votes[e], cm = ts.maxl[e];
          if (be == 0x7fffffff || cv > bv || (cv == bv && cm > bm)) {
            bv = cv;
            bm = cm;
            be = e;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int om = __shfl_xor_sync(0xffffffffu, bm, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (oe != 0x7fffffff &&
            (be == 0x7fffffff || ov > bv || (ov == bv && (om > bm || (om == bm && oe < be))))) {
          bv = ov;
          bm = om;
          be = oe;
        }
      }
      if (be == 0x7fffffff) break;
      if (be < 64)
        lo |= 1ull << be;
      else
        hi |= 1ull << (be - 64);
    }
    if (lane == 0) {
      ts.m[0] = lo;
      ts.m[1] = hi;
    }
  }
  bar();
  mlo = ts.m[0];
  mhi = ts.m[1];
}

// Route body, usable by any block size (the standalone kernel runs it with
// 1024 threads, the fused router kernel with the last router CTA).
__device__ void route_body(RouteSmem& sm, const float* __restrict__ logits, int B, int M, int k,
                           int mode, float bias, uint64_t mlo, uint64_t mhi, int topup_U,
                           uint64_t* mask_out, int32_t* __restrict__ sel, float* __restrict__ wts,
                           int32_t* __restrict__ counts, int32_t* __restrict__ offsets,
                           int32_t* __restrict__ perm, int32_t* __restrict__ inv,
                           uint64_t* host_mask, int32_t* host_sel, float* host_logits,
                           volatile uint32_t* host_done, unsigned long long* stamp, int n_pub) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (stamp && tid == 0) *stamp = gtimer();
  if (topup_U > 0) {
    __shared__ TopupSmem ts;
    topup_mask(ts, logits, B, M, k, topup_U, mlo, mhi);
  }
  if (mask_out && tid == 0) {
    mask_out[0] = mlo;
    mask_out[1] = mhi;
  }

  // ---- top-k and weights: one warp per token, logits in registers (M <= 128),
  // k rounds of a warp arg-max keyed (value desc, index asc) — SURVEY H6
  for (int t = wid; t < B; t += blockDim.x / 32)
    topk_token(logits + (int64_t)t * M, M, k, mode, bias, mlo, mhi, sel + t * k, wts + t * k,
               nullptr);
  __syncthreads();

  // ---- stable counting sort by expert over flat slots f = t*k + r
  const int N = B * k;
  for (int e = tid; e < M; e += blockDim.x) {
    sm.base[e] = 0;
    sm.total[e] = 0;
  }
  __syncthreads();
  for (int c0 = 0; c0 < N; c0 += blockDim.x) {
    for (int i = tid; i < 32 * M; i += blockDim.x) sm.warp_cnt[i / M][i % M] = 0;
    __syncthreads();
    int f = c0 + tid;
    int e = (f < N) ? sel[f] : -1;
    unsigned same = __match_any_sync(0xffffffffu, e);
    int rank_in_warp = __popc(same & ((1u << lane) - 1u));
    if (e >= 0 && rank_in_warp == 0) sm.warp_cnt[wid][e] = __popc(same);
    __syncthreads();
    // exclusive prefix over warps, per expert
    for (int x = tid; x < M; x += blockDim.x) {
      int run = sm.base[x];
      for (int w = 0; w < 32; ++w) {
        int c = sm.warp_cnt[w][x];
        sm.warp_cnt[w][x] = run;
        run += c;
      }
      sm.base[x] = run;
    }
    __syncthreads();
    if (e >= 0) perm[f] = sm.warp_cnt[wid][e] + rank_in_warp;  // rank within expert (temp)
    __syncthreads();
  }
  // counts and offsets
  if (tid == 0) {
    int run = 0;
    for (int x = 0; x < M; ++x) {
      counts[x] = sm.base[x];
      offsets[x] = run;
      sm.total[x] = run;
      run += sm.base[x];
    }
    offsets[M] = run;
  }
  __syncthreads();
  for (int f = tid; f < N; f += blockDim.x) {
    int pos = sm.total[sel[f]] + perm[f];
    inv[f] = pos;
  }
  __syncthreads();
  for (int f = tid; f < N; f += blockDim.x) perm[inv[f]] = f;
  if (host_done && wid == 0) {
    // publish the selection and the logits rows (row 0 = this layer, rows
    // 1.. = pre-gate scores of later layers) to mapped host memory from one
    // warp: a system-scope fence costs microseconds per warp that issues it
    for (int f = lane; f < N; f += 32) host_sel[f] = sel[f];
    for (int i = lane; i < n_pub; i += 32) host_logits[i] = __ldcg(logits + i);
    if (host_mask && lane == 0) {
      host_mask[0] = mlo;
      host_mask[1] = mhi;
    }
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
      *host_done = 1u;
      if (stamp) stamp[3] = gtimer();  // slot 9: selection published
    }
  }
}

__global__ void __launch_bounds__(kRouteThreads) route_permute_kernel(
    const float* __restrict__ logits, int B, int M, int k, int mode, float bias, uint64_t mlo,
    uint64_t mhi, int topup_U, int32_t* __restrict__ sel, float* __restrict__ wts,
    int32_t* __restrict__ counts, int32_t* __restrict__ offsets, int32_t* __restrict__ perm,
    int32_t* __restrict__ inv, uint64_t* host_mask, int32_t* host_sel, float* host_logits,
    volatile uint32_t* host_done, unsigned long long* stamp, int n_pub) {
  __shared__ RouteSmem sm;
  route_body(sm, logits, B, M, k, mode, bias, mlo, mhi, topup_U, nullptr, sel, wts, counts,
             offsets, perm, inv, host_mask, host_sel, host_logits, host_done, stamp, n_pub);
}

// Engine decode path: router GEMV rows, then the last CTA to finish runs
// the route body (top-k, weights, permutation, host publish) — one kernel
// boundary instead of two on the per-layer critical path.
struct RouteArgs {
  int B, M, k, mode;
  float bias;
  uint64_t mlo, mhi;
  int topup_U;          // > 0: top the mask up to U experts by router votes
  uint64_t* mask_out;   // device copy of the final mask (the fused gate publishes it)
  uint64_t* host_mask;  // mapped host copy (configurations where the route publishes)
  int32_t *sel, *counts, *offsets, *perm, *inv, *host_sel;
  float *wts, *host_logits;
  uint32_t* host_done;  // null: the fused gate warp publishes instead
  unsigned long long* stamp_route;
  int* counter;
  ef::RouteFast rf;  // device-side slot resolution (rf.dc null: off)
  // Qwen's sigmoid-gated shared expert: its gate logit x.w_sg rides as one
  // extra router row (row index rows_main) written to sgl_out[t]
  const void* sgate_w;
  float* sgl_out;
  int rows_main;
};

__device__ __forceinline__ int2 ld_volatile_v2(const void* p) {
  int2 v;
  asm volatile("ld.volatile.global.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// Device-side slot resolution (one warp): if every routed expert of this
// layer is in the device copy of the slot table, write the FFN's decision
// block {slot, row offset, rows, fill seq} straight into DevCtrl and mark the
// layer fast — the routed FFN then starts without the host round trip (the
// host still decides the layer; its slots are pinned until FFN(l) is done).
__device__ void resolve_fast(const ef::RouteFast& rf, const int32_t* counts,
                             const int32_t* offsets, int M, unsigned long long* stamp_fast) {
  const int lane = threadIdx.x & 31;
  int base = 0;
  bool ok = true;
  for (int e0 = 0; e0 < M; e0 += 32) {
    const int e = e0 + lane;
    const int c = e < M ? __ldcg(counts + e) : 0;
    int2 t = make_int2(-1, 0);
    if (c > 0) t = rf.tab[e];
    ok = ok && !__any_sync(0xffffffffu, c > 0 && t.x < 0);
    const unsigned m = __ballot_sync(0xffffffffu, c > 0);
    const int pos = base + __popc(m & ((1u << lane) - 1u));
    if (c > 0 && pos < ef::kMaxActive) rf.dc->ent[pos] = make_int4(t.x, __ldcg(offsets + e), c, t.y);
    base += __popc(m);
  }
  ok = ok && base <= ef::kMaxActive;
  if (lane == 0) {
    if (ok) rf.dc->n_active = base;
    __threadfence();
    *rf.fast_word = ok ? rf.seq : 0u;
    if (stamp_fast) *stamp_fast = ok ? 1ull : 0ull;
  }
}

// Small-batch route (B*k <= 32, one warp per token): top-k into shared
// memory, then warp 0 does the stable sort of the <= 32 (token, rank) slots
// with shuffles only, writes sel/wts/counts/offsets/perm/inv, and — with the
// slot-table row preloaded in registers — resolves the layer's decision
// block on the device.  No dependent global-memory round trips.
__device__ void route_small(const float* __restrict__ logits, const RouteArgs& ra,
                            const int2 (&tabv)[4], unsigned long long* stamp) {
  __shared__ int32_t sel_sh[32];
  const int B = ra.B, M = ra.M, k = ra.k, N = B * k;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (stamp && threadIdx.x == 0) *stamp = gtimer();
  uint64_t mlo = ra.mlo, mhi = ra.mhi;
  if (ra.topup_U > 0) {
    __shared__ TopupSmem ts;
    topup_mask(ts, logits, B, M, k, ra.topup_U, mlo, mhi);
  }
  if (ra.mask_out && threadIdx.x == 0) {
    ra.mask_out[0] = mlo;
    ra.mask_out[1] = mhi;
  }
  if (wid < B)
    topk_token(logits + (int64_t)wid * M, M, k, ra.mode, ra.bias, mlo, mhi, ra.sel + wid * k,
               ra.wts + wid * k, sel_sh + wid * k);
  __syncthreads();
  if (wid != 0) return;
  const int e = lane < N ? sel_sh[lane] : 0x7fffffff;
  // rank within the expert (stable in f) and number of slots with a smaller expert
  const unsigned same = __match_any_sync(0xffffffffu, e);
  const int rank = __popc(same & ((1u << lane) - 1u));
  int below = 0;
  for (int j = 0; j < N; ++j) below += __shfl_sync(0xffffffffu, e, j) < e;
  if (lane < N) {
    const int pos = below + rank;
    ra.inv[lane] = pos;
    ra.perm[pos] = lane;
  }
  // per-expert counts / offsets (lane owns experts lane + 32 i)
  int cnt[4], off[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) cnt[i] = off[i] = 0;
  for (int j = 0; j < N; ++j) {
    const int ej = __shfl_sync(0xffffffffu, e, j);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      cnt[i] += ej == lane + 32 * i;
      off[i] += ej < lane + 32 * i;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int x = lane + 32 * i;
    if (x < M) {
      ra.counts[x] = cnt[i];
      ra.offsets[x] = off[i];
    }
  }
  if (lane == 0) ra.offsets[M] = N;
  if (ra.rf.dc) {  // device-side slot resolution, experts in ascending order
    int base = 0;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = lane + 32 * i;
      const bool act = x < M && cnt[i] > 0;
      ok = ok && !__any_sync(0xffffffffu, act && tabv[i].x < 0);
      const unsigned m = __ballot_sync(0xffffffffu, act);
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      if (act && pos < ef::kMaxActive) ra.rf.dc->ent[pos] = make_int4(tabv[i].x, off[i], cnt[i], tabv[i].y);
      base += __popc(m);
    }
    ok = ok && base <= ef::kMaxActive;
    if (lane == 0) {
      if (ok) ra.rf.dc->n_active = base;
      __threadfence();
      *ra.rf.fast_word = ok ? ra.rf.seq : 0u;
      if (stamp) stamp[5] = ok ? 1ull : 0ull;
    }
  }
  if (ra.host_done) {  // publish (non-fast configurations)
    if (lane < N) ra.host_sel[lane] = e;
    if (ra.host_mask && lane == 0) {
      ra.host_mask[0] = mlo;
      ra.host_mask[1] = mhi;
    }
    for (int i = lane; i < B * M; i += 32) ra.host_logits[i] = __ldcg(logits + i);
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
      *reinterpret_cast<volatile uint32_t*>(ra.host_done) = 1u;
      if (stamp) stamp[3] = gtimer();
    }
  }
}

// Previous layer's combine folded into the router (small batches): every CTA
// recomputes h + sum_r w*y (+ g*ys) and the rmsnorm scale for its tokens into
// shared memory; the last CTA writes h and x back once all CTAs have read h.
struct CombArgs {
  float* h;  // null: x comes from global memory as usual
  float* x_out;
  const float* y;
  const int32_t* inv;
  const float* wts;
  const float* ys;
  const float* gate_logit;
  int k;
  float eps;
  unsigned long long* stamp;
};
constexpr int kCombSmemMax = 128 * 1024;

template <typename WT, int MAXB>
__global__ void __launch_bounds__(256) router_route_kernel(const float* __restrict__ x,
                                                           const WT* __restrict__ w, int rows,
                                                           int d, float* __restrict__ logits,
                                                           unsigned long long* stamp,
                                                           RouteArgs ra, CombArgs cb) {
  constexpr int V = WTraits<WT>::kPer16;
  const int B = ra.B, M = ra.M;
  const int t0 = blockIdx.y * MAXB;
  const int nb = min(MAXB, B - t0);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // UN 16-byte chunks in flight per lane (a 4096-wide bf16 row in one round trip at B=1)
  constexpr int UN = MAXB == 1 ? 16 : 8;
  // the router weights are constant: the first chunk group of this warp's row
  // is loaded before waiting on the previous kernel, so its HBM latency
  // overlaps the tail of the previous layer's FFN
  uint4 wv0[UN];
  const bool sg_row = ra.sgate_w && warp == ra.rows_main;
  const WT* wrow = sg_row ? reinterpret_cast<const WT*>(ra.sgate_w) : w + (int64_t)warp * d;
  if (warp < rows) {
#pragma unroll
    for (int u = 0; u < UN; ++u)
      if (lane * V + u * 32 * V < d) wv0[u] = ld_stream16(wrow + lane * V + u * 32 * V);
  }
  // this layer's slot-table row is final once the previous kernel has started
  // (written by the previous layer's gate warp, two kernels back)
  int2 tabv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) tabv[i] = make_int2(-1, 0);
  if (ra.rf.dc && threadIdx.x < 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < M) tabv[i] = ra.rf.tab[lane + 32 * i];
  }
  pdl_wait();
  pdl_trigger();  // a tiny grid: let the FFN's CTAs be scheduled behind it
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    *stamp = gtimer();
    stamp[8] = clock64();  // slot 15: SM clock at start (phase breakdown, same SM)
    unsigned dep = 0;
#pragma unroll
    for (int u = 0; u < UN; ++u) dep ^= wv0[u].x ^ wv0[u].w;
    stamp[7] = clock64() + (dep == 0x9e3779b9u ? 1 : 0);  // slot 14: weights arrived
  }
  extern __shared__ float hs[];  // [nb][d] combined, un-normalised rows (cb.h only)
  __shared__ float invn_s[MAXB];
  __shared__ float red[32];
  const bool comb = cb.h != nullptr;
  if (comb) {
    for (int t = 0; t < nb; ++t) {
      const float ss = combine_row(t0 + t, cb.h, hs + t * d, cb.y, cb.inv, cb.wts, cb.ys,
                                   cb.gate_logit, d, cb.k, red);
      if (threadIdx.x == 0) invn_s[t] = 1.0f / sqrtf(ss / (float)d + cb.eps);
    }
    __syncthreads();
  }
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) stamp[5] = clock64();
  if (warp < rows) {
    const WT* wr = wrow;
    float acc[MAXB];
#pragma unroll
    for (int t = 0; t < MAXB; ++t) acc[t] = 0.f;
    for (int c0 = lane * V; c0 < d; c0 += UN * 32 * V) {
      uint4 wv[UN];
      const bool first = c0 == lane * V;
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int c = c0 + u * 32 * V;
        // out-of-range chunks must be zero: 0 * (stale register) could be NaN
        wv[u] = c >= d ? make_uint4(0, 0, 0, 0) : first ? wv0[u] : ld_stream16(wr + c);
      }
#pragma unroll
      for (int t = 0; t < MAXB; ++t) {
        if (t < nb) {
          const float sc = comb ? invn_s[t] : 1.f;
          // groups of 4 chunks: all x loads of a group first (no branches between
          // them), 4 independent accumulators, then a fixed-order fold
#pragma unroll
          for (int g = 0; g < UN; g += 4) {
            float4 xa[4][V / 4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = c0 + (g + u) * 32 * V;
#pragma unroll
              for (int q = 0; q < V / 4; ++q) {
                float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c < d) {
                  if (comb) {  // x = v * invn, the same fp32 product the combine stores
                    xv = reinterpret_cast<const float4*>(hs + t * d + c)[q];
                    xv.x *= sc;
                    xv.y *= sc;
                    xv.z *= sc;
                    xv.w *= sc;
                  } else {
                    xv = __ldg(reinterpret_cast<const float4*>(x + (int64_t)(t0 + t) * d + c) + q);
                  }
                }
                xa[u][q] = xv;
              }
            }
            float part[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float f[V];
              WTraits<WT>::unpack(wv[g + u], f);
              float p = 0.f;
#pragma unroll
              for (int q = 0; q < V / 4; ++q) {
                p = fmaf(f[4 * q + 0], xa[u][q].x, p);
                p = fmaf(f[4 * q + 1], xa[u][q].y, p);
                p = fmaf(f[4 * q + 2], xa[u][q].z, p);
                p = fmaf(f[4 * q + 3], xa[u][q].w, p);
              }
              part[u] = p;
            }
            acc[t] += (part[0] + part[1]) + (part[2] + part[3]);
          }
        }
      }
    }
    const int r = warp / M, m = warp % M;
#pragma unroll
    for (int t = 0; t < MAXB; ++t) {
      if (t < nb) {
        float sum = warp_sum(acc[t]);
        if (lane == 0) {
          if (sg_row)
            ra.sgl_out[t0 + t] = sum;
          else
            logits[((int64_t)r * B + t0 + t) * M + m] = sum;
        }
      }
    }
  }
  __shared__ RouteSmem sm;
  __shared__ int last;
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) stamp[6] = clock64();
  // ticket: only the logits writers (lane 0 of each row warp) fence their
  // stores; the last CTA's thread 0 fences after the ticket, and the route
  // reads the logits through L2 (__ldcg)
  if (lane == 0 && warp < rows) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(ra.counter, 1) == (int)(gridDim.x * gridDim.y) - 1;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;

  if (comb) {  // every CTA has read h: publish h and x for the rest of the layer
    for (int t = 0; t < nb; ++t) {
      const int tt = t0 + t;
      for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const float v = hs[t * d + i];
        cb.h[(int64_t)tt * d + i] = v;
        cb.x_out[(int64_t)tt * d + i] = v * invn_s[t];
      }
    }
    if (cb.stamp && threadIdx.x == 0) *cb.stamp = gtimer();
  }
  if (threadIdx.x == 0) *ra.counter = 0;  // ready for the next launch
  if (B * ra.k <= 32 && B <= (int)(blockDim.x >> 5) && (!ra.host_done || ra.rows_main == M)) {
    route_small(logits, ra, tabv, ra.stamp_route);
    return;
  }
  route_body(sm, logits, B, M, ra.k, ra.mode, ra.bias, ra.mlo, ra.mhi, ra.topup_U, ra.mask_out,
             ra.sel, ra.wts, ra.counts, ra.offsets, ra.perm, ra.inv, ra.host_mask, ra.host_sel,
             ra.host_logits, ra.host_done, ra.stamp_route, ra.rows_main * B);
  if (ra.rf.dc && (threadIdx.x >> 5) == 0)
    resolve_fast(ra.rf, ra.counts, ra.offsets, M, ra.stamp_route ? ra.stamp_route + 5 : nullptr);
}

// B = 1 variant: one CTA per router row, its 4 warps splitting the row, so
// each SM reads the hidden vector once (the warp-per-row kernel is bound by
// shared-memory bandwidth at B = 1: 8 warps x 16 KB per SM, tools/router_lab.cu)
// and the rows spread over R*M SMs.  Same ticket / route / combine contract.
template <typename WT>
__global__ void __launch_bounds__(256) router_route_row_kernel(const float* __restrict__ x,
                                                               const WT* __restrict__ w, int rows,
                                                               int d, float* __restrict__ logits,
                                                               unsigned long long* stamp,
                                                               RouteArgs ra, CombArgs cb) {
  constexpr int V = WTraits<WT>::kPer16;
  constexpr int UQ = 8;  // 16-byte chunks per lane in flight
  const int M = ra.M;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int row = blockIdx.x;
  const int span = d / 8;  // 8 warps split the row
  const int cb0 = wid * span + lane * V;
  const bool sg_row = ra.sgate_w && row == ra.rows_main;
  const WT* wr = sg_row ? reinterpret_cast<const WT*>(ra.sgate_w) : w + (int64_t)row * d;
  uint4 wv0[UQ];
#pragma unroll
  for (int u = 0; u < UQ; ++u)
    wv0[u] = u * 32 * V < span ? ld_stream16(wr + cb0 + u * 32 * V) : make_uint4(0, 0, 0, 0);
  int2 tabv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) tabv[i] = make_int2(-1, 0);
  if (ra.rf.dc && threadIdx.x < 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < M) tabv[i] = ra.rf.tab[lane + 32 * i];
  }
  pdl_wait();
  pdl_trigger();
  if (stamp && blockIdx.x == 0 && threadIdx.x == 0) {
    *stamp = gtimer();
    stamp[8] = clock64();
    stamp[7] = clock64();
  }
  extern __shared__ float hs[];
  __shared__ float red[32], part[8];
  __shared__ float invn_s;
  __shared__ int last;
  const bool comb = cb.h != nullptr;
  if (comb) {
    // 256 threads x 4 float4 passes: a 4096-wide row in one round of loads
    const float ss = combine_row<4>(0, cb.h, hs, cb.y, cb.inv, cb.wts, cb.ys, cb.gate_logit, d,
                                    cb.k, red);
    if (threadIdx.x == 0) invn_s = 1.0f / sqrtf(ss / (float)d + cb.eps);
    __syncthreads();
  }
  if (stamp && blockIdx.x == 0 && threadIdx.x == 0) stamp[5] = clock64();
  const float sc = comb ? invn_s : 1.f;
  float p[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c0 = 0; c0 < span; c0 += UQ * 32 * V) {
#pragma unroll
    for (int u = 0; u < UQ; ++u) {
      const int cc = c0 + u * 32 * V;
      if (cc < span) {
        const uint4 wq = c0 == 0 ? wv0[u] : ld_stream16(wr + cb0 + cc);
        float f[V];
        WTraits<WT>::unpack(wq, f);
        const int c = cb0 + cc;
#pragma unroll
        for (int q = 0; q < V / 4; ++q) {
          float4 xv;
          if (comb) {
            xv = reinterpret_cast<const float4*>(hs + c)[q];
            xv.x *= sc;
            xv.y *= sc;
            xv.z *= sc;
            xv.w *= sc;
          } else {
            xv = __ldg(reinterpret_cast<const float4*>(x + c) + q);
          }
          p[u & 3] = fmaf(f[4 * q + 0], xv.x, p[u & 3]);
          p[u & 3] = fmaf(f[4 * q + 1], xv.y, p[u & 3]);
          p[u & 3] = fmaf(f[4 * q + 2], xv.z, p[u & 3]);
          p[u & 3] = fmaf(f[4 * q + 3], xv.w, p[u & 3]);
        }
      }
    }
  }
  float acc = warp_sum((p[0] + p[1]) + (p[2] + p[3]));
  if (lane == 0) part[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    const float v = ((part[0] + part[1]) + (part[2] + part[3])) +
                    ((part[4] + part[5]) + (part[6] + part[7]));
    if (sg_row)
      ra.sgl_out[0] = v;
    else
      logits[row] = v;  // B = 1: [r][0][m] = row
    if (stamp && blockIdx.x == 0) stamp[6] = clock64();
    __threadfence();
    last = atomicAdd(ra.counter, 1) == (int)gridDim.x - 1;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;
  if (comb) {  // every CTA has read h: publish h and x for the rest of the layer
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      const float v = hs[i];
      cb.h[i] = v;
      cb.x_out[i] = v * invn_s;
    }
    if (cb.stamp && threadIdx.x == 0) *cb.stamp = gtimer();
  }
  if (threadIdx.x == 0) *ra.counter = 0;
  route_small(logits, ra, tabv, ra.stamp_route);
}

namespace ef {
int router_route_fused(cudaStream_t st, const float* x, const void* w, int dtype, int R, int B,
                       int d, int M, float* logits, unsigned long long* stamp_router, int k,
                       int mode, float bias, uint64_t mlo, uint64_t mhi, int topup_U,
                       uint64_t* mask_out, uint64_t* host_mask, int32_t* sel, float* wts,
                       int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv,
                       int32_t* host_sel, float* host_logits, uint32_t* host_done,
                       unsigned long long* stamp_route, int* counter, const CombineIn* ci,
                       const RouteFast* rf, const void* sgate_w, float* sgl_out) {
  EF_CHECK_ARG(M <= 128 && k <= 16 && B >= 1, "bad fused route shape");
  RouteArgs ra{B, M, k, mode, bias, mlo, mhi, topup_U, mask_out, host_mask, sel, counts, offsets,
               perm, inv, host_sel, wts, host_logits, host_done, stamp_route, counter,
               rf ? *rf : RouteFast{}, sgate_w, sgl_out, R * M};
  CombArgs cb{};
  size_t smem = 0;
  if (ci) {
    EF_CHECK_ARG(B <= 8 && (size_t)B * d * 4 <= (size_t)kCombSmemMax,
                 "combine-in-router needs B*d*4 <= 128 KiB");
    // the previous layer's y / inv / wts are read before route_body of this
    // layer overwrites inv / wts (only the last CTA routes)
    cb = CombArgs{ci->h, const_cast<float*>(x), ci->y, ci->y_slot_order ? nullptr : inv, wts,
                  ci->ys, ci->gate_logit, k, ci->eps, ci->stamp};
    smem = (size_t)B * d * 4;
  }
  const int rows = R * M + (sgate_w ? 1 : 0), threads = 256;
  const int blocks = (rows * 32 + threads - 1) / threads;
  const int vq = dtype == EF_BF16 ? 8 : 4;
  if (B == 1 && d % (8 * 32 * vq) == 0 && k <= 32 && (!host_done || R == 1)) {
    if (dtype == EF_BF16)
      EF_CUDA_RET(launch_k(router_route_row_kernel<__nv_bfloat16>, dim3(rows), dim3(256), smem, st,
                           x, (const __nv_bfloat16*)w, rows, d, logits, stamp_router, ra, cb));
    else
      EF_CUDA_RET(launch_k(router_route_row_kernel<float>, dim3(rows), dim3(256), smem, st, x,
                           (const float*)w, rows, d, logits, stamp_router, ra, cb));
    return EF_OK;
  }
  if (dtype == EF_BF16) {
    if (B == 1)
      EF_CUDA_RET(launch_k(router_route_kernel<__nv_bfloat16, 1>, dim3(blocks, 1), dim3(threads), smem, st, x,
                           (const __nv_bfloat16*)w, rows, d, logits, stamp_router, ra, cb));
    else
      EF_CUDA_RET(launch_k(router_route_kernel<__nv_bfloat16, 8>, dim3(blocks, (B + 7) / 8), dim3(threads), smem, st, x,
                           (const __nv_bfloat16*)w, rows, d, logits, stamp_router, ra, cb));
  } else {
    if (B == 1)
      EF_CUDA_RET(launch_k(router_route_kernel<float, 1>, dim3(blocks, 1), dim3(threads), smem, st, x,
                           (const float*)w, rows, d, logits, stamp_router, ra, cb));
    else
      EF_CUDA_RET(launch_k(router_route_kernel<float, 8>, dim3(blocks, (B + 7) / 8), dim3(threads), smem, st, x,
                           (const float*)w, rows, d, logits, stamp_router, ra, cb));
  }
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}
}  // namespace ef

extern "C" int ef_route_permute(void* stream, const float* logits, int B, int M, int k, int mode,
                                float bias, uint64_t mlo, uint64_t mhi, int32_t* sel, float* wts,
                                int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv) {
  EF_CHECK_ARG(M >= 1 && M <= 128 && k >= 1 && k <= 16 && k <= M && B >= 0, "bad route shape");
  EF_CHECK_ARG(mode == EF_ROUTE_MIXTRAL || mode == EF_ROUTE_SOFTMAX_TOPK, "bad routing mode");
  route_permute_kernel<<<1, kRouteThreads, 0, S(stream)>>>(logits, B, M, k, mode, bias, mlo, mhi,
                                                           0, sel, wts, counts, offsets, perm,
                                                           inv, nullptr, nullptr, nullptr,
                                                           nullptr, nullptr, 0);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// ============================================================ (d) decode expert FFN
using ef::kMaxActive;
using ef::DevCtrl;
using ef::HostCtrl;
struct ActiveList {
  const char* w[kMaxActive];  // expert weight base ([W1|W3|W2])
  int32_t p0[kMaxActive];     // first permuted row (also output row)
  int32_t n[kMaxActive];      // rows
};

// Input-vector loaders (one 16-byte weight chunk = V columns).
template <typename WT>
struct XGather {  // T(x[perm[p]/k]) — expert input, cast to the weight dtype
  const float* x;
  const int32_t* perm;
  int k, d;
  bool identity;  // shared expert: row p reads token p - id_base
  int id_base;
  // expert parallelism: token t lives in rank t / tpr's block of the
  // all-gathered routing buffer, rank_stride floats apart (tpr 0: contiguous)
  int tpr = 0;
  int64_t rank_stride = 0;
  __device__ inline const float* row(int p) const {
    int t = identity ? p - id_base : perm[p] / k;
    if (tpr) return x + (int64_t)(t / tpr) * rank_stride + (int64_t)(t % tpr) * d;
    return x + (int64_t)t * d;
  }
  __device__ inline void load(const float* r, int c, float* out) const {
    constexpr int V = WTraits<WT>::kPer16;
    const float4* p = reinterpret_cast<const float4*>(r + c);
#pragma unroll
    for (int q = 0; q < V / 4; ++q) {
      float4 v = __ldg(p + q);
      out[4 * q + 0] = WTraits<WT>::cast(v.x);
      out[4 * q + 1] = WTraits<WT>::cast(v.y);
      out[4 * q + 2] = WTraits<WT>::cast(v.z);
      out[4 * q + 3] = WTraits<WT>::cast(v.w);
    }
  }
};

template <typename WT>
struct XAct {  // act[p] (already in the weight dtype)
  const WT* act;
  int ff;
  __device__ inline const WT* row(int p) const { return act + (int64_t)p * ff; }
  __device__ inline void load(const WT* r, int c, float* out) const {
    WTraits<WT>::unpack(__ldg(reinterpret_cast<const uint4*>(r + c)), out);
  }
};

// rows x cols matrix A (and B when DUAL) streamed once per token chunk; each
// warp owns R consecutive output rows; lanes stride the columns in 16 B.
// Engine pipeline control (pipeline.h): the gate kernel copies the host's
// per-layer decision into DevCtrl; entries are {slot, p0, rows, need_seq}; a
// slot is usable once ready[slot] >= need_seq (set by the copy stream after
// the swap-in lands).
struct CtrlSrc {
  const DevCtrl* ctrl;
  const char* slab;
  int64_t stride;
  const volatile uint32_t* ready;
  unsigned long long* stats;  // per layer: [0] gate enter [1] go [2] max wait [3] ffn start [4] ffn end
  bool wait_ready;            // first kernel of the pair waits for the copies
};

// ~10 s at 2 GHz: a spin this long means the host side died; fail loudly
// instead of hanging the GPU.
constexpr long long kSpinTimeoutCycles = 20000000000LL;
constexpr int kStatsPerLayer = 16;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Kernel fusions of the engine's decode pipeline (split FFN path):
//  * gate in the up kernel: warp 0 of CTA (0,0) waits for the host's go flag
//    and copies the decision into DevCtrl, then raises a device flag the
//    other CTAs wait on (one PCIe round trip, no separate gate launch);
//  (the combine is folded into the next layer's router instead, see
//   router_route_kernel: a last-CTA combine here serialised on one SM and
//   its registers cost the down GEMV occupancy)
struct FuseArgs {
  volatile HostCtrl* hc;
  DevCtrl* dc;
  volatile unsigned* dflag;
  unsigned seq;
  ef::GateIO io;
  // down kernel: write y in (token, rank) slot order, y[perm[p]], so the
  // combine needs no inverse-permutation lookup before loading y
  const int32_t* y_perm;
};

__device__ __forceinline__ uint2 ld_acquire_sys_v2_(const volatile void* p) {
  uint2 v;
  asm volatile("ld.acquire.sys.global.v2.u32 {%0,%1}, [%2];"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ int4 ld_volatile_v4_(const volatile void* p) {
  int4 v;
  asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const volatile unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One full warp: publish the route to the host, wait for go, copy the
// decision (unless the route kernel resolved every slot on the device), then
// copy the next layer's slot-table row for that kernel's fast path.
__device__ void gate_duty(volatile HostCtrl* hc, DevCtrl* dc, unsigned long long* stats,
                          volatile unsigned* dflag, unsigned seq, const ef::GateIO& io) {
  const int lane = threadIdx.x & 31;
  if (stats && lane == 0) stats[0] = globaltimer();
  if (io.host_done) {  // selection + every scored logits row -> mapped host memory
    for (int f = lane; f < io.n_sel; f += 32) io.host_sel[f] = __ldcg(io.sel_src + f);
    for (int i = lane; i < io.n_pub; i += 32) io.host_logits[i] = __ldcg(io.logits_src + i);
    if (io.host_mask && lane < 2) io.host_mask[lane] = __ldcg(io.mask_src + lane);
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
      *reinterpret_cast<volatile uint32_t*>(io.host_done) = 1u;
      if (stats) stats[9] = globaltimer();
    }
  }
  const bool fast = io.fast_word && *reinterpret_cast<const volatile unsigned*>(io.fast_word) == seq;
  if (fast) {  // the route kernel resolved every slot: nothing to wait for
    if (stats && lane == 0) stats[1] = stats[8] = globaltimer();
    __syncwarp();
    return;
  }
  // slow path: the host's decision; go carries the layer's launch sequence
  // number (monotonic), so no reset is needed
  uint2 gn = make_uint2(0, 0);
  if (lane == 0) {
    const long long c0 = clock64();
    for (;;) {
      gn = ld_acquire_sys_v2_(&hc->go);
      if ((int)(gn.x - seq) >= 0) break;
      __nanosleep(64);
      if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
    }
    if (stats) stats[1] = globaltimer();
  }
  const int n = __shfl_sync(0xffffffffu, (int)gn.y, 0);
  for (int i = lane; i < n; i += 32) dc->ent[i] = ld_volatile_v4_(&hc->ent[i]);
  __syncwarp();
  if (lane == 0) {
    dc->n_active = n;
    __threadfence();
    if (dflag) *dflag = seq;
    if (stats) stats[8] = globaltimer();
  }
  __syncwarp();
}

template <typename WT, int NT, int R, bool DUAL, typename XL, int U = 1>
__global__ void __launch_bounds__(128, NT <= 2 ? (DUAL ? 8 : 16) : 1) ffn_gemv_kernel(ActiveList al, CtrlSrc cs, FuseArgs fz,
                                                       int64_t offA, int64_t offB, int rows,
                                                       int cols, XL xl, WT* act_out, float* y_out,
                                                       int out_ld) {
  constexpr int V = WTraits<WT>::kPer16;
  constexpr int WARPS = 4;
  const int a = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int n_all, p0;
  const char* wbase;
  pdl_wait();
  // down projection: the next kernel is the small router grid, schedule it early;
  // gate/up: trigger only at the end (down CTAs must not take the slots of the
  // second wave of gate/up CTAs)
  if (!DUAL) pdl_trigger();
  if (fz.hc) {  // fused gate (up kernel): column 0 of the grid is the gate, not FFN work
    if (blockIdx.x == 0) {
      if (blockIdx.y == 0 && wid == 0) gate_duty(fz.hc, fz.dc, cs.stats, fz.dflag, fz.seq, fz.io);
      return;
    }
    if (threadIdx.x == 0) {
      const bool fast = fz.io.fast_word &&
                        *reinterpret_cast<const volatile unsigned*>(fz.io.fast_word) == fz.seq;
      const long long c0 = clock64();
      while (!fast && ld_acquire_gpu(fz.dflag) < fz.seq) {
        __nanosleep(64);
        if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
      }
    }
    __syncthreads();
  }
  if (cs.ctrl) {
    __shared__ int4 e_sh;
    if (threadIdx.x == 0) {
      // timeline stamps: the earliest CTAs of the grid define the start, one
      // atomic per CTA for the end (thousands of same-address atomics per
      // launch would serialise in L2)
      const bool early = blockIdx.x < 3;
      if (cs.wait_ready && cs.stats && early) atomicMin(&cs.stats[10], globaltimer());
      int4 e = make_int4(0, 0, 0, 0);
      if (a < __ldcg(&cs.ctrl->n_active)) e = __ldcg(&cs.ctrl->ent[a]);
      if (cs.wait_ready && e.z > 0) {
        unsigned long long t0 = globaltimer();
        unsigned need = (unsigned)e.w;
        if (cs.ready[e.x] < need) {
          const long long c0 = clock64();  // SM cycles: monotonic, used for the timeout
          while (cs.ready[e.x] < need) {
            __nanosleep(256);
            if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
          }
          unsigned long long t1 = globaltimer();
          if (t1 > t0) atomicMax(&cs.stats[2], t1 - t0);
        }
        if (early) atomicMin(&cs.stats[3], globaltimer());
      }
      e_sh = e;
    }
    __syncthreads();
    int4 e = e_sh;
    n_all = e.z;
    p0 = e.y;
    wbase = cs.slab + (int64_t)e.x * cs.stride;
  } else {
    n_all = al.n[a];
    p0 = al.p0[a];
    wbase = al.w[a];
  }
  const int j0 = ((blockIdx.x - (fz.hc ? 1 : 0)) * WARPS + wid) * R;
  // no early return: the fused combine counts every CTA of the grid
  const bool work = n_all > 0 && j0 < rows;
  const WT* A = reinterpret_cast<const WT*>(wbase + offA);
  const WT* Bm = reinterpret_cast<const WT*>(wbase + offB);
  const uint64_t pol = l2_evict_first_policy();

  for (int tc = 0; work && tc < n_all; tc += NT) {
    const int nt = min(NT, n_all - tc);
    float accA[R][NT], accB[R][NT];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int t = 0; t < NT; ++t) accA[r][t] = accB[r][t] = 0.f;

    decltype(xl.row(0)) xr[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) xr[t] = xl.row(p0 + tc + (t < nt ? t : 0));

    // U column chunks x R rows (x2 when DUAL) of 16-byte loads in flight per lane
    for (int c0 = lane * V; c0 < cols; c0 += 32 * V * U) {
      uint4 wa[U][R], wb[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * 32 * V;
        if (c < cols) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            int j = min(j0 + r, rows - 1);
            wa[u][r] = ld_stream16_ef(A + (int64_t)j * cols + c, pol);
            if (DUAL) wb[u][r] = ld_stream16_ef(Bm + (int64_t)j * cols + c, pol);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * 32 * V;
        if (c < cols) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (t < nt) {
              float xv[V];
              xl.load(xr[t], c, xv);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                float f[V];
                WTraits<WT>::unpack(wa[u][r], f);
#pragma unroll
                for (int q = 0; q < V; ++q) accA[r][t] = fmaf(f[q], xv[q], accA[r][t]);
                if (DUAL) {
                  WTraits<WT>::unpack(wb[u][r], f);
#pragma unroll
                  for (int q = 0; q < V; ++q) accB[r][t] = fmaf(f[q], xv[q], accB[r][t]);
                }
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (t < nt) {
          float g = warp_sum(accA[r][t]);
          float u = DUAL ? warp_sum(accB[r][t]) : 0.f;
          int j = j0 + r;
          if (lane == 0 && j < rows) {
            int64_t row = p0 + tc + t;
            if (DUAL) {
              float s = g / (1.0f + expf(-g));
              WTraits<WT>::store(act_out + row * out_ld + j, s * u);
            } else {
              y_out[(fz.y_perm ? (int64_t)__ldg(fz.y_perm + row) : row) * out_ld + j] = g;
            }
          }
        }
      }
    }
  }
  if (work && cs.ctrl && !DUAL && cs.stats && threadIdx.x == 0)
    atomicMax(&cs.stats[4], globaltimer());
  if (DUAL) pdl_trigger();
}

// ------------------------------------------------------------ (d) decode FFN on mma.sync
// Tensor-core decode FFN (bf16): one warp owns 16 output rows of one expert
// and streams them ONCE for all of the expert's tokens (8-token n-tiles,
// mma.sync.m16n8k16, fp32 accumulators in registers) — the GEMV kernel above
// re-streams an expert per 8-token chunk and runs out of FMA throughput past
// a few tokens.  The shared expert(s) ride in the same launch as extra work
// units (identity token map), so a layer's whole FFN is one gate/up launch
// and one down launch.  Weights: 16-byte L1-bypassing evict-first loads; k
// is permuted inside each 32-wide block (thread tq holds k 8tq..8tq+7 of its
// rows and of its token's x/act row) so every load is 16 B and A and B use
// the same permutation.
struct FfnMmaArgs {
  // routed entries: DevCtrl (engine) or an explicit list (tests / bench)
  const DevCtrl* ctrl;
  ActiveList al;
  int n_list;  // entries in `al` when ctrl is null
  const char* slab;
  int64_t stride;
  const volatile uint32_t* ready;
  unsigned long long* stats;
  bool wait_ready;
  // shared expert blob [W1 sff x d | W3 sff x d | W2 d x sff] (null: none),
  // its tokens are rows 0..B-1 of x / act_s
  const __nv_bfloat16* shared_w;
  int sff, B;
  // tensors
  const float* x;          // [B, d] fp32 (up)
  int tpr;                 // expert parallelism: tokens per rank block of x (0: contiguous)
  int64_t rank_stride;     //   floats between rank blocks
  const int32_t* perm;     // permuted row -> flat (token, rank) slot
  int k, d, ff;
  __nv_bfloat16* act;      // [rows, ff]  routed act (up out / down in)
  __nv_bfloat16* act_s;    // [B, sff]    shared act
  float* y;                // [slots, d]  routed out, row y_perm[p] (slot order) or p
  float* ys;               // [B, d]      shared out
  const int32_t* y_perm;
  int max_active, routed_units, shared_units;  // units = 16-row warp tiles
};

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1,
                                               uint32_t a2, uint32_t a3, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 8 consecutive fp32 -> 4 bf16x2 (RNE): the expert input T(x)
__device__ __forceinline__ uint4 ld_x8_bf16(const float* p) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  return make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                    pack_bf16x2(b.z, b.w));
}


// One warp: rows [r0, r0+16) of matrix A (and B when UP: W3 at +ff rows) of
// one expert over K columns, tokens n (rows p0.. of the permuted order or the
// shared expert's identity rows).
// One CTA = one 16-row unit of one expert: its 4 warps split the reduction
// dimension K in 4 (contiguous quarters), each streams its 16 x K/4 slice of
// A (and of W3 when UP) once for all of the expert's tokens (NT 8-token
// n-tiles per pass; more tokens loop over passes, the weights then come
// from L2), and the partial fp32 fragments are summed in a fixed warp order
// through shared memory before warp 0's epilogue (deterministic).  Split-K
// keeps ~4x more warps streaming than a whole-K warp tile at decode batch.
template <bool UP, int NT, int WARPS>
__device__ void mma_unit(const FfnMmaArgs& a, const __nv_bfloat16* W, int rows_total, int K,
                         int r0, int p0, int n, bool shared, uint64_t pol, float* red) {
  constexpr int kMmaWarps = WARPS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  // this warp's k range, in whole 32-wide blocks
  const int nkb = K / 32;
  const int kb0 = (nkb * wid) / kMmaWarps * 32, kb1 = (nkb * (wid + 1)) / kMmaWarps * 32;
  const __nv_bfloat16* A0 = W + (int64_t)(r0 + g) * K + 8 * tq;
  const __nv_bfloat16* A1 = A0 + (int64_t)8 * K;
  const int64_t offB = (int64_t)rows_total * K;  // W3 behind W1 (UP)
  for (int t0 = 0; t0 < n; t0 += 8 * NT) {
    const int nt = min(NT, (n - t0 + 7) / 8);
    const float* xr[NT];
    const __nv_bfloat16* br[NT];
    bool ok[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int p = t0 + 8 * j + g;
      ok[j] = j < nt && p < n;
      const int pp = ok[j] ? p : 0;
      if (UP) {
        const int tok = shared ? pp : __ldg(a.perm + p0 + pp) / a.k;
        xr[j] = (a.tpr ? a.x + (int64_t)(tok / a.tpr) * a.rank_stride + (int64_t)(tok % a.tpr) * a.d
                       : a.x + (int64_t)tok * a.d) + 8 * tq;
        br[j] = nullptr;
      } else {
        br[j] = (shared ? a.act_s + (int64_t)pp * a.sff : a.act + (int64_t)(p0 + pp) * a.ff) +
                8 * tq;
        xr[j] = nullptr;
      }
    }
    float c1[NT][4], c3[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) c1[j][q] = c3[j][q] = 0.f;
    constexpr int U = UP ? 4 : 8;  // 32-wide k blocks in flight per iteration
    for (int kb = kb0; kb < kb1; kb += 32 * U) {
      uint4 w1[U][2], w3[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kb + 32 * u;
        if (kk < kb1) {
          w1[u][0] = ld_stream16_ef(A0 + kk, pol);
          w1[u][1] = ld_stream16_ef(A1 + kk, pol);
          if (UP) {
            w3[u][0] = ld_stream16_ef(A0 + offB + kk, pol);
            w3[u][1] = ld_stream16_ef(A1 + offB + kk, pol);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = kb + 32 * u;
        if (kk >= kb1) break;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          if (j >= nt) break;
          uint4 bv = make_uint4(0, 0, 0, 0);
          if (ok[j])
            bv = UP ? ld_x8_bf16(xr[j] + kk) : __ldg(reinterpret_cast<const uint4*>(br[j] + kk));
          mma_bf16_16816(c1[j], w1[u][0].x, w1[u][1].x, w1[u][0].y, w1[u][1].y, bv.x, bv.y);
          mma_bf16_16816(c1[j], w1[u][0].z, w1[u][1].z, w1[u][0].w, w1[u][1].w, bv.z, bv.w);
          if (UP) {
            mma_bf16_16816(c3[j], w3[u][0].x, w3[u][1].x, w3[u][0].y, w3[u][1].y, bv.x, bv.y);
            mma_bf16_16816(c3[j], w3[u][0].z, w3[u][1].z, w3[u][0].w, w3[u][1].w, bv.z, bv.w);
          }
        }
      }
    }
    // split-K reduction: warps 1..3 park their fragments, warp 0 adds them in order
    constexpr int NV = (UP ? 8 : 4) * NT;  // floats per thread
    if (wid > 0) {
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          red[((wid - 1) * NV + j * 4 + q) * 32 + lane] = c1[j][q];
          if (UP) red[((wid - 1) * NV + 4 * NT + j * 4 + q) * 32 + lane] = c3[j][q];
        }
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
      for (int w = 1; w < kMmaWarps; ++w)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            c1[j][q] += red[((w - 1) * NV + j * 4 + q) * 32 + lane];
            if (UP) c3[j][q] += red[((w - 1) * NV + 4 * NT + j * 4 + q) * 32 + lane];
          }
      // epilogue: c[q] = (row g + 8*(q>>1), token 2tq + (q&1)) of each n-tile
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if (j >= nt) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = t0 + 8 * j + 2 * tq + (q & 1);
          if (p >= n) continue;
          const int row = r0 + g + 8 * (q >> 1);
          if (UP) {
            const float gg = c1[j][q], uu = c3[j][q];
            const float sv = gg / (1.0f + expf(-gg)) * uu;
            if (shared)
              a.act_s[(int64_t)p * a.sff + row] = __float2bfloat16_rn(sv);
            else
              a.act[(int64_t)(p0 + p) * a.ff + row] = __float2bfloat16_rn(sv);
          } else {
            if (shared)
              a.ys[(int64_t)p * a.d + row] = c1[j][q];
            else
              a.y[(a.y_perm ? (int64_t)__ldg(a.y_perm + p0 + p) : (int64_t)(p0 + p)) * a.d +
                  row] = c1[j][q];
          }
        }
      }
    }
    __syncthreads();  // red is reused by the next pass
  }
}

// CTA size: 4 warps split K for gate/up (W1 and W3 in flight), 8 for down
template <bool UP>
struct MmaWarps {
  static constexpr int value = UP ? 4 : 8;
};

template <bool UP, int NT>
__global__ void __launch_bounds__(MmaWarps<UP>::value * 32) ffn_mma_kernel(FfnMmaArgs a, FuseArgs fz) {
  constexpr int kMmaWarps = MmaWarps<UP>::value;
  __shared__ float red[(kMmaWarps - 1) * (UP ? 8 : 4) * NT * 32];
  __shared__ int4 e_sh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pdl_wait();
  if (!UP) pdl_trigger();  // the next kernel is the small router grid
  if (fz.hc && blockIdx.x == 0) {  // fused gate: CTA 0 is the gate (see ffn_gemv_kernel)
    if (wid == 0) gate_duty(fz.hc, fz.dc, a.stats, fz.dflag, fz.seq, fz.io);
    return;
  }
  const int u = blockIdx.x - (fz.hc ? 1 : 0);  // this CTA's 16-row unit
  const uint64_t pol = l2_evict_first_policy();
  if (u < a.shared_units) {  // shared expert: always resident, needs no decision
    const int rows = UP ? a.sff : a.d;
    const __nv_bfloat16* W = a.shared_w + (UP ? 0 : 2LL * a.sff * a.d);
    mma_unit<UP, NT, kMmaWarps>(a, W, rows, UP ? a.d : a.sff, u * 16, 0, a.B, true, pol, red);
    if (UP) pdl_trigger();
    return;
  }
  const int ru = u - a.shared_units;
  const int ei = ru / a.routed_units, sub = ru % a.routed_units;
  if (threadIdx.x == 0) {
    if (fz.hc) {  // routed work waits for the layer's decision
      const bool fast = fz.io.fast_word &&
                        *reinterpret_cast<const volatile unsigned*>(fz.io.fast_word) == fz.seq;
      const long long c0 = clock64();
      while (!fast && ld_acquire_gpu(fz.dflag) < fz.seq) {
        __nanosleep(64);
        if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
      }
    }
    int4 e = make_int4(0, 0, 0, 0);
    if (a.ctrl) {
      if (ei < a.max_active && ei < __ldcg(&a.ctrl->n_active)) e = __ldcg(&a.ctrl->ent[ei]);
    } else if (ei < a.n_list) {
      e = make_int4(ei, a.al.p0[ei], a.al.n[ei], 0);
    }
    if (a.ctrl && a.wait_ready && e.z > 0) {
      const bool early = ru < 4;  // the first routed units stamp the FFN start
      if (a.stats && early) atomicMin(&a.stats[10], globaltimer());
      const unsigned need = (unsigned)e.w;
      if (a.ready[e.x] < need) {
        const unsigned long long t0 = globaltimer();
        const long long c0 = clock64();
        while (a.ready[e.x] < need) {
          __nanosleep(256);
          if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
        }
        const unsigned long long t1 = globaltimer();
        if (a.stats && t1 > t0) atomicMax(&a.stats[2], t1 - t0);
      }
      if (a.stats && early) atomicMin(&a.stats[3], globaltimer());
    }
    e_sh = e;
  }
  __syncthreads();
  const int4 e = e_sh;
  if (e.z <= 0) {
    if (UP) pdl_trigger();
    return;
  }
  const char* wbase = a.ctrl ? a.slab + (int64_t)e.x * a.stride : a.al.w[e.x];
  const __nv_bfloat16* W =
      reinterpret_cast<const __nv_bfloat16*>(wbase) + (UP ? 0 : 2LL * a.ff * a.d);
  mma_unit<UP, NT, kMmaWarps>(a, W, UP ? a.ff : a.d, UP ? a.d : a.ff, sub * 16, e.y, e.z, false, pol, red);
  if (!UP && a.ctrl && a.stats && threadIdx.x == 0) atomicMax(&a.stats[4], globaltimer());
  if (UP) pdl_trigger();
}

template <int NT>
static int launch_ffn_mma_nt(cudaStream_t st, FfnMmaArgs a, const FuseArgs& fz_up,
                             const FuseArgs& fz_dn) {
  a.routed_units = a.ff / 16;
  a.shared_units = a.shared_w ? a.sff / 16 : 0;
  const int n_ent = a.ctrl ? a.max_active : a.n_list;
  const int up_ctas = a.shared_units + n_ent * a.routed_units + (fz_up.hc ? 1 : 0);
  EF_CUDA_RET(launch_k(ffn_mma_kernel<true, NT>, dim3(up_ctas), dim3(MmaWarps<true>::value * 32),
                       0, st, a, fz_up));
  FfnMmaArgs b = a;
  b.wait_ready = false;
  b.routed_units = a.d / 16;
  b.shared_units = a.shared_w ? a.d / 16 : 0;
  const int dn_ctas = b.shared_units + n_ent * b.routed_units;
  EF_CUDA_RET(launch_k(ffn_mma_kernel<false, NT>, dim3(dn_ctas), dim3(MmaWarps<false>::value * 32),
                       0, st, b, fz_dn));
  return EF_OK;
}

// Launch the pair for `max_tok` tokens per expert at most (the batch: a
// token picks an expert once): 8-token n-tiles, up to 4 per pass.
static int launch_ffn_mma(cudaStream_t st, FfnMmaArgs a, const FuseArgs& fz_up,
                          const FuseArgs& fz_dn, int max_tok) {
  if (max_tok <= 8) return launch_ffn_mma_nt<1>(st, a, fz_up, fz_dn);
  if (max_tok <= 16) return launch_ffn_mma_nt<2>(st, a, fz_up, fz_dn);
  return launch_ffn_mma_nt<4>(st, a, fz_up, fz_dn);
}

// The tensor-core decode FFN serves bf16 experts whose dimensions are
// multiples of 32 (every SURVEY §8 shape); EF_FFN_MMA=0 selects the GEMV pair
// (A/B comparisons, fp32 engines always use it).
namespace ef {
bool ffn_mma_enabled(int dtype, int d, int ff, int sff, int max_tok) {
  static const int env = [] {
    const char* v = getenv("EF_FFN_MMA");
    return v ? atoi(v) : 1;
  }();
  if (env == 0 || dtype != EF_BF16 || d % 32 || ff % 32 || sff % 32) return false;
  // auto: the GEMV pair streams a lone token's experts faster (tools/ffn_mma_lab.py,
  // profiles/r02_ffn_lab.txt); from 2 tokens per expert, or to fold a shared
  // expert into the layer's launches, the tensor-core pair
  return env == 2 || max_tok > 1 || sff > 0;
}
}  // namespace ef

// Decode GEMV tilings (tools/ffn_lab.cu sweep on B200, Mixtral shapes):
// gate/up: 2 rows x 2 column chunks per warp (8 x 16 B in flight per lane,
// few distinct DRAM rows per warp) ran at 6.5 TB/s vs 5.5 TB/s for 4 x 1;
// down: 1 row x 2 chunks with act through the read-only path, 6.2 TB/s.
constexpr int kUpR = 2, kUpU = 2, kDnR = 1, kDnU = 2;

template <typename WT, int NT>
static void launch_ffn_nt(cudaStream_t st, const ActiveList& al, const CtrlSrc& cs, int n_active,
                          int d, int ff, const XGather<WT>& xg, WT* act, float* y,
                          const FuseArgs& fz_up, const FuseArgs& fz_dn) {
  constexpr int WARPS = 4;
  const int64_t es = sizeof(WT);
  if (d <= 2048 && NT == 1) {
    // short rows (Qwen / DeepSeek experts, d = 2048): one row x 4 chunks per
    // warp keeps more warps streaming (tools/ffn_lab.cu -DQWEN: 4.47 vs 3.73 TB/s)
    dim3 gu((ff + WARPS - 1) / WARPS + (fz_up.hc ? 1 : 0), n_active);
    launch_k(ffn_gemv_kernel<WT, NT, 1, true, XGather<WT>, 4>, gu, dim3(128), 0, st, al, cs, fz_up,
             (int64_t)0, (int64_t)ff * d * es, ff, d, xg, act, (float*)nullptr, ff);
  } else {
    constexpr int R = kUpR;
    dim3 gu((ff + WARPS * R - 1) / (WARPS * R) + (fz_up.hc ? 1 : 0), n_active);
    launch_k(ffn_gemv_kernel<WT, NT, R, true, XGather<WT>, kUpU>, gu, dim3(128), 0, st, al, cs,
             fz_up, (int64_t)0, (int64_t)ff * d * es, ff, d, xg, act, (float*)nullptr, ff);
  }
  // down projection: one W2 row per warp (d rows only: more rows per warp
  // left SMs idle on Mixtral's 4096 x 14336 W2)
  constexpr int RD = kDnR, UD = kDnU;
  dim3 gd((d + WARPS * RD - 1) / (WARPS * RD), n_active);
  XAct<WT> xa{act, ff};
  CtrlSrc cs2 = cs;
  cs2.wait_ready = false;
  launch_k(ffn_gemv_kernel<WT, NT, RD, false, XAct<WT>, UD>, gd, dim3(128), 0, st, al, cs2, fz_dn,
           2 * (int64_t)ff * d * es, (int64_t)0, d, ff, xa, (WT*)nullptr, y, d);
}

template <typename WT>
static void launch_ffn(cudaStream_t st, const ActiveList& al, const CtrlSrc& cs, int n_active,
                       int max_rows, int d, int ff, const XGather<WT>& xg, WT* act, float* y,
                       const FuseArgs& fu = FuseArgs{}, const FuseArgs& fd = FuseArgs{}) {
  if (max_rows <= 1)
    launch_ffn_nt<WT, 1>(st, al, cs, n_active, d, ff, xg, act, y, fu, fd);
  else if (max_rows <= 2)
    launch_ffn_nt<WT, 2>(st, al, cs, n_active, d, ff, xg, act, y, fu, fd);
  else if (max_rows <= 4)
    launch_ffn_nt<WT, 4>(st, al, cs, n_active, d, ff, xg, act, y, fu, fd);
  else
    launch_ffn_nt<WT, 8>(st, al, cs, n_active, d, ff, xg, act, y, fu, fd);
}

namespace ef {
// Internal entry used by the engine: weight bases are explicit pointers.
int expert_ffn_ptrs(cudaStream_t st, const float* x, const int32_t* perm, int k, bool identity,
                    const char* const* wbase, const int32_t* p0, const int32_t* nrows,
                    int n_active, int d, int ff, int dtype, void* act, float* y) {
  EF_CHECK_ARG(n_active >= 0 && n_active <= kMaxActive, "too many active experts");
  EF_CHECK_ARG(d % 8 == 0 && ff % 8 == 0, "d and ff must be multiples of 8");
  if (n_active == 0) return EF_OK;
  ActiveList al;
  int max_rows = 0;
  for (int i = 0; i < n_active; ++i) {
    al.w[i] = wbase[i];
    al.p0[i] = p0[i];
    al.n[i] = nrows[i];
    max_rows = std::max(max_rows, nrows[i]);
  }
  if (max_rows == 0) return EF_OK;
  if (!identity && ffn_mma_enabled(dtype, d, ff, 0, max_rows)) {
    FfnMmaArgs a{};
    a.al = al;
    a.n_list = n_active;
    a.x = x;
    a.perm = perm;
    a.k = k;
    a.d = d;
    a.ff = ff;
    a.act = (__nv_bfloat16*)act;
    a.y = y;
    return launch_ffn_mma(st, a, FuseArgs{}, FuseArgs{}, max_rows);
  }
  CtrlSrc cs{};
  if (dtype == EF_BF16) {
    XGather<__nv_bfloat16> xg{x, perm, k, d, identity, identity ? p0[0] : 0};
    launch_ffn<__nv_bfloat16>(st, al, cs, n_active, max_rows, d, ff, xg, (__nv_bfloat16*)act, y);
  } else {
    XGather<float> xg{x, perm, k, d, identity, identity ? p0[0] : 0};
    launch_ffn<float>(st, al, cs, n_active, max_rows, d, ff, xg, (float*)act, y);
  }
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// Engine pipeline with the gate folded into the up kernel and (optionally)
// the combine folded into the down kernel.
int expert_ffn_fused(cudaStream_t st, const float* x, const int32_t* perm, int k, const char* slab,
                     int64_t stride, void* hctrl_dev, void* dctrl, volatile unsigned* dflag,
                     unsigned seq, const uint32_t* ready, unsigned long long* stats, int max_active,
                     int max_rows, int d, int ff, int dtype, void* act, float* y,
                     const GateIO* io, const SharedFfn* sh) {
  EF_CHECK_ARG(max_active >= 1 && max_active <= kMaxActive, "too many active experts");
  ActiveList al{};
  CtrlSrc cs{reinterpret_cast<const DevCtrl*>(dctrl), slab, stride, ready, stats, true};
  FuseArgs fu{reinterpret_cast<volatile HostCtrl*>(hctrl_dev), reinterpret_cast<DevCtrl*>(dctrl),
              dflag, seq, io ? *io : GateIO{}, nullptr};
  FuseArgs fd{};
  fd.y_perm = perm;  // y in slot order (the engine's combine reads it without inv)
  if (ffn_mma_enabled(dtype, d, ff, sh ? sh->sff : 0, max_rows)) {
    FfnMmaArgs a{};
    a.ctrl = reinterpret_cast<const DevCtrl*>(dctrl);
    a.slab = slab;
    a.stride = stride;
    a.ready = ready;
    a.stats = stats;
    a.wait_ready = true;
    if (sh) {
      a.shared_w = reinterpret_cast<const __nv_bfloat16*>(sh->w);
      a.sff = sh->sff;
      a.B = sh->B;
      a.act_s = reinterpret_cast<__nv_bfloat16*>(sh->act);
      a.ys = sh->y;
    }
    a.x = x;
    a.perm = perm;
    a.k = k;
    a.d = d;
    a.ff = ff;
    a.act = (__nv_bfloat16*)act;
    a.y = y;
    a.y_perm = perm;
    a.max_active = max_active;
    return launch_ffn_mma(st, a, fu, FuseArgs{}, std::max(max_rows, sh ? sh->B : 0));
  }
  EF_CHECK_ARG(!sh, "the shared expert rides in the tensor-core FFN launch only");
  if (dtype == EF_BF16) {
    XGather<__nv_bfloat16> xg{x, perm, k, d, false, 0};
    launch_ffn<__nv_bfloat16>(st, al, cs, max_active, max_rows, d, ff, xg, (__nv_bfloat16*)act, y,
                              fu, fd);
  } else {
    XGather<float> xg{x, perm, k, d, false, 0};
    launch_ffn<float>(st, al, cs, max_active, max_rows, d, ff, xg, (float*)act, y, fu, fd);
  }
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}


// ============================================================ expert parallelism
// Decode step split over G ranks (engine.cu ep_step_on).  Per
// layer each rank routes its own B tokens, then:
//   dispatch  ep_pack_kernel writes the rank's routing block
//             [x B*d | logits Rm*B*M | sel B*k | wts B*k] (4-byte words) and
//             one all-gather gives every rank every block;
//   owner     ep_owner_kernel selects the (token, rank) slots routed to the
//             experts this rank owns, in (local expert, global slot) order —
//             the stable permutation of the single-GPU route — publishes the
//             global selection and logits rows to the host for the shard's
//             scheduler, and builds the home combine index;
//   FFN       the decode GEMV pair reads the owned slots' x rows straight
//             from the gathered blocks and writes y in global slot order, which
//             is already the all-to-all layout (chunk g = rank g's B*k slots);
//   combine   after the all-to-all, rank-order combine of y rows from their
//             owners: y[(owner * B + t) * k + r], owner = e * G / M.
__global__ void ep_pack_kernel(const float* __restrict__ x, const float* __restrict__ logits,
                               const int32_t* __restrict__ sel, const float* __restrict__ wts,
                               int64_t nx, int64_t nl, int nk, float* __restrict__ out) {
  const int64_t n = nx + nl + 2 * (int64_t)nk;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v;
    if (i < nx) v = x[i];
    else if (i < nx + nl) v = logits[i - nx];
    else if (i < nx + nl + nk) v = __int_as_float(sel[i - nx - nl]);
    else v = wts[i - nx - nl - nk];
    out[i] = v;
  }
}

struct EpOwnerArgs {
  const float* recv;      // [G][W] gathered routing blocks
  int64_t W;              // block stride (4-byte words)
  int G, B, k, M, d, Rm, R, rank, e0, Ms;
  int32_t* counts;        // [Ms]
  int32_t* offsets;       // [Ms + 1]
  int32_t* perm;          // [G*B*k] owned global slots, stable by (local expert, slot)
  int32_t* home_idx;      // [B*k] y row of each local (token, rank) slot after the all-to-all
  int32_t* host_sel;      // [G*B*k] mapped
  float* host_logits;     // [R][G*B][M] mapped
  volatile uint32_t* host_done;
};

__global__ void __launch_bounds__(1024) ep_owner_kernel(EpOwnerArgs a) {
  __shared__ int cnt[kMaxExperts];
  __shared__ int off[kMaxExperts + 1];
  const int tid = threadIdx.x;
  const int N = a.G * a.B * a.k;
  const int64_t sel_off = (int64_t)a.B * a.d + (int64_t)a.Rm * a.B * a.M;
  auto sel_of = [&](int f) {  // global slot f = (g*B + t)*k + r
    const int g = f / (a.B * a.k), rem = f % (a.B * a.k);
    return __float_as_int(__ldcg(a.recv + (int64_t)g * a.W + sel_off + rem));
  };
  for (int j = tid; j < a.Ms; j += blockDim.x) cnt[j] = 0;
  __syncthreads();
  for (int f = tid; f < N; f += blockDim.x) {
    const int e = sel_of(f);
    if (e >= a.e0 && e < a.e0 + a.Ms) atomicAdd(&cnt[e - a.e0], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int j = 0; j < a.Ms; ++j) {
      off[j] = run;
      a.counts[j] = cnt[j];
      a.offsets[j] = run;
      run += cnt[j];
    }
    a.offsets[a.Ms] = run;
  }
  __syncthreads();
  for (int f = tid; f < N; f += blockDim.x) {
    const int e = sel_of(f);
    if (e < a.e0 || e >= a.e0 + a.Ms) continue;
    int before = 0;  // stable: earlier slots of the same expert
    for (int f2 = 0; f2 < f; ++f2) before += sel_of(f2) == e;
    a.perm[off[e - a.e0] + before] = f;
  }
  for (int i = tid; i < a.B * a.k; i += blockDim.x) {
    const int e = __float_as_int(__ldcg(a.recv + (int64_t)a.rank * a.W + sel_off + i));
    const int o = e * a.G / a.M;
    a.home_idx[i] = o * a.B * a.k + i;
  }
  // publish the global selection and the R scored logits rows of every token
  if (a.host_sel)
    for (int f = tid; f < N; f += blockDim.x) a.host_sel[f] = sel_of(f);
  const int GB = a.G * a.B;
  for (int64_t i = tid; a.host_logits && i < (int64_t)a.R * GB * a.M; i += blockDim.x) {
    const int rr = (int)(i / ((int64_t)GB * a.M));
    const int rem = (int)(i % ((int64_t)GB * a.M));
    const int tg = rem / a.M, m = rem % a.M;
    const int g = tg / a.B, t = tg % a.B;
    a.host_logits[i] =
        __ldcg(a.recv + (int64_t)g * a.W + (int64_t)a.B * a.d + ((int64_t)rr * a.B + t) * a.M + m);
  }
  __threadfence_system();
  __syncthreads();
  if (tid == 0) *a.host_done = 1u;
}

int ep_pack(cudaStream_t st, const float* x, const float* logits, const int32_t* sel,
            const float* wts, int B, int d, int Rm, int M, int k, float* out) {
  const int64_t nx = (int64_t)B * d, nl = (int64_t)Rm * B * M;
  const int64_t n = nx + nl + 2LL * B * k;
  const int blocks = (int)std::min<int64_t>(148, (n + 255) / 256);
  ep_pack_kernel<<<blocks, 256, 0, st>>>(x, logits, sel, wts, nx, nl, B * k, out);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

int ep_owner(cudaStream_t st, const float* recv, int64_t W, int G, int B, int k, int M, int d,
             int Rm, int R, int rank, int e0, int Ms, int32_t* counts, int32_t* offsets,
             int32_t* perm, int32_t* home_idx, int32_t* host_sel, float* host_logits,
             uint32_t* host_done) {
  EF_CHECK_ARG(Ms >= 1 && Ms <= kMaxExperts && M <= kMaxExperts, "bad expert-parallel shard");
  EpOwnerArgs a{recv, W, G, B, k, M, d, Rm, R, rank, e0, Ms, counts, offsets, perm, home_idx,
                host_sel, host_logits, host_done};
  ep_owner_kernel<<<1, 1024, 0, st>>>(a);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// owner-side routed FFN of the expert-parallel step: x rows from the
// gathered blocks (row stride W floats per rank), y in global slot order
int expert_ffn_ep(cudaStream_t st, const float* recv, int64_t W, int B, const int32_t* perm, int k,
                  const char* slab, int64_t stride, const void* dctrl, const uint32_t* ready,
                  unsigned long long* stats, int max_active, int max_rows, int d, int ff,
                  int dtype, void* act, float* y) {
  EF_CHECK_ARG(max_active >= 1 && max_active <= kMaxActive, "too many active experts");
  if (ffn_mma_enabled(dtype, d, ff, 0, max_rows)) {
    FfnMmaArgs a{};
    a.ctrl = reinterpret_cast<const DevCtrl*>(dctrl);
    a.slab = slab;
    a.stride = stride;
    a.ready = ready;
    a.stats = stats;
    a.wait_ready = true;
    a.x = recv;
    a.tpr = B;
    a.rank_stride = W;
    a.perm = perm;
    a.k = k;
    a.d = d;
    a.ff = ff;
    a.act = (__nv_bfloat16*)act;
    a.y = y;
    a.y_perm = perm;
    a.max_active = max_active;
    return launch_ffn_mma(st, a, FuseArgs{}, FuseArgs{}, max_rows);
  }
  ActiveList al{};
  CtrlSrc cs{reinterpret_cast<const DevCtrl*>(dctrl), slab, stride, ready, stats, true};
  FuseArgs fd{};
  fd.y_perm = perm;
  if (dtype == EF_BF16) {
    XGather<__nv_bfloat16> xg{recv, perm, k, d, false, 0, B, W};
    launch_ffn<__nv_bfloat16>(st, al, cs, max_active, max_rows, d, ff, xg, (__nv_bfloat16*)act, y,
                              FuseArgs{}, fd);
  } else {
    XGather<float> xg{recv, perm, k, d, false, 0, B, W};
    launch_ffn<float>(st, al, cs, max_active, max_rows, d, ff, xg, (float*)act, y, FuseArgs{}, fd);
  }
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// Engine pipeline: slots / rows come from the gate-copied DevCtrl at run time.
int expert_ffn_ctrl(cudaStream_t st, const float* x, const int32_t* perm, int k, const char* slab,
                    int64_t stride, const void* dctrl, const uint32_t* ready,
                    unsigned long long* stats, int max_active, int max_rows, int d, int ff,
                    int dtype, void* act, float* y, const SharedFfn* sh) {
  EF_CHECK_ARG(max_active >= 1 && max_active <= kMaxActive, "too many active experts");
  if (ffn_mma_enabled(dtype, d, ff, sh ? sh->sff : 0, max_rows)) {
    FfnMmaArgs a{};
    a.ctrl = reinterpret_cast<const DevCtrl*>(dctrl);
    a.slab = slab;
    a.stride = stride;
    a.ready = ready;
    a.stats = stats;
    a.wait_ready = true;
    if (sh) {
      a.shared_w = reinterpret_cast<const __nv_bfloat16*>(sh->w);
      a.sff = sh->sff;
      a.B = sh->B;
      a.act_s = reinterpret_cast<__nv_bfloat16*>(sh->act);
      a.ys = sh->y;
    }
    a.x = x;
    a.perm = perm;
    a.k = k;
    a.d = d;
    a.ff = ff;
    a.act = (__nv_bfloat16*)act;
    a.y = y;
    a.max_active = max_active;
    return launch_ffn_mma(st, a, FuseArgs{}, FuseArgs{}, std::max(max_rows, sh ? sh->B : 0));
  }
  EF_CHECK_ARG(!sh, "the shared expert rides in the tensor-core FFN launch only");
  ActiveList al{};
  CtrlSrc cs{reinterpret_cast<const DevCtrl*>(dctrl), slab, stride, ready, stats, true};
  if (dtype == EF_BF16) {
    XGather<__nv_bfloat16> xg{x, perm, k, d, false, 0};
    launch_ffn<__nv_bfloat16>(st, al, cs, max_active, max_rows, d, ff, xg, (__nv_bfloat16*)act, y);
  } else {
    XGather<float> xg{x, perm, k, d, false, 0};
    launch_ffn<float>(st, al, cs, max_active, max_rows, d, ff, xg, (float*)act, y);
  }
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// ------------------------------------------------------------ pipeline glue
__device__ __forceinline__ uint2 ld_acquire_sys_v2(const volatile void* p) {
  uint2 v;
  asm volatile("ld.acquire.sys.global.v2.u32 {%0,%1}, [%2];"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ int4 ld_volatile_v4(const volatile void* p) {
  int4 v;
  asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// One warp: spin on the host's go flag (8-byte acquire load returns go and
// n_active together), copy the decision with one 16-byte PCIe read per entry.
__global__ void gate_kernel(volatile HostCtrl* hc, DevCtrl* dc, unsigned long long* stats) {
  const int lane = threadIdx.x;
  uint2 gn = make_uint2(0, 0);
  if (lane == 0) {
    stats[0] = globaltimer();
    const long long c0 = clock64();
    for (;;) {
      gn = ld_acquire_sys_v2(&hc->go);
      if (gn.x != 0u) break;
      __nanosleep(64);
      if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");  // host died: fail loudly
    }
    stats[1] = globaltimer();
  }
  const int n = __shfl_sync(0xffffffffu, (int)gn.y, 0);
  for (int i = lane; i < n; i += 32) dc->ent[i] = ld_volatile_v4(&hc->ent[i]);
  __syncwarp();
  if (lane == 0) {
    dc->n_active = n;
    hc->go = 0u;  // consumed; the host sets it again for the next token's layer
    stats[8] = globaltimer();
  }
}

int launch_gate(cudaStream_t st, void* host_ctrl_dev, void* dctrl, unsigned long long* stats) {
  gate_kernel<<<1, 32, 0, st>>>(reinterpret_cast<HostCtrl*>(host_ctrl_dev),
                                reinterpret_cast<DevCtrl*>(dctrl), stats);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

__global__ void init_stats_kernel(unsigned long long* stats, int L) {
  for (int i = threadIdx.x; i < L * kStatsPerLayer; i += blockDim.x)
    stats[i] = (i % kStatsPerLayer == 3 || i % kStatsPerLayer == 10) ? ~0ull : 0ull;
}

int launch_init_stats(cudaStream_t st, unsigned long long* stats, int L) {
  init_stats_kernel<<<1, 256, 0, st>>>(stats, L);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

int launch_route_publish(cudaStream_t st, const float* logits, int B, int M, int k, int mode,
                         float bias, uint64_t mlo, uint64_t mhi, int topup_U, int32_t* sel,
                         float* wts, int32_t* counts, int32_t* offsets, int32_t* perm,
                         int32_t* inv, uint64_t* host_mask, int32_t* host_sel, float* host_logits,
                         uint32_t* host_done, unsigned long long* stamp, int n_pub) {
  route_permute_kernel<<<1, kRouteThreads, 0, st>>>(
      logits, B, M, k, mode, bias, mlo, mhi, topup_U, sel, wts, counts, offsets, perm, inv,
      host_mask, host_sel, host_logits, host_done, stamp, n_pub);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

}  // namespace ef

extern "C" int ef_expert_ffn_decode(void* stream, const float* x, const int32_t* perm, int k,
                                    const void* slab, int64_t stride, const int32_t* act_slot,
                                    const int32_t* act_off, const int32_t* act_rows,
                                    int n_active, int d, int ff, int dtype, void* act, float* y) {
  EF_CHECK_ARG(n_active <= kMaxActive, "too many active experts");
  const char* w[kMaxActive];
  for (int i = 0; i < n_active; ++i)
    w[i] = reinterpret_cast<const char*>(slab) + (int64_t)act_slot[i] * stride;
  return ef::expert_ffn_ptrs(S(stream), x, perm, k, false, w, act_off, act_rows, n_active, d, ff,
                             dtype, act, y);
}

// ============================================================ (c) permute gather (prefill)
// x_perm[p] = T(x[perm[p] / k]) as bf16 rows for the grouped GEMM's A operand.
__global__ void gather_rows_bf16_kernel(const float* __restrict__ x, const int32_t* __restrict__ perm,
                                        int k, int d, int n, __nv_bfloat16* __restrict__ out) {
  const int p = blockIdx.x;
  if (p >= n) return;
  const float* src = x + (int64_t)(perm[p] / k) * d;
  __nv_bfloat16* dst = out + (int64_t)p * d;
  for (int i = threadIdx.x * 2; i < d; i += blockDim.x * 2) {
    float2 v = *reinterpret_cast<const float2*>(src + i);
    *reinterpret_cast<__nv_bfloat162*>(dst + i) = __floats2bfloat162_rn(v.x, v.y);
  }
}

extern "C" int ef_gather_rows_bf16(void* stream, const float* x, const int32_t* perm, int k, int d,
                                   int n, void* out) {
  EF_CHECK_ARG(n >= 0 && d % 2 == 0 && k >= 1, "bad gather shape");
  if (n == 0) return EF_OK;
  gather_rows_bf16_kernel<<<n, 256, 0, S(stream)>>>(x, perm, k, d, n, (__nv_bfloat16*)out);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

// ============================================================ (c) combine + norm
__global__ void __launch_bounds__(256) combine_kernel(float* __restrict__ h, float* __restrict__ x,
                               const float* __restrict__ y, const int32_t* __restrict__ inv,
                               const float* __restrict__ wts, const float* __restrict__ ys,
                               const float* __restrict__ gate_logit, int d, int k, float eps,
                               unsigned long long* stamp) {
  __shared__ float red[32];
  combine_token(blockIdx.x, h, x, y, inv, wts, ys, gate_logit, d, k, eps, red);
  if (stamp && threadIdx.x == 0) atomicMax(stamp, gtimer());
}

namespace ef {
int combine_stamped(cudaStream_t st, float* h, float* x, const float* y, const int32_t* inv,
                    const float* wts, const float* ys, const float* gate_logit, int B, int d, int k,
                    float eps, unsigned long long* stamp) {
  if (B == 0) return EF_OK;
  combine_kernel<<<B, 256, 0, st>>>(h, x, y, inv, wts, ys, gate_logit, d, k, eps, stamp);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}
}  // namespace ef

extern "C" int ef_combine(void* stream, float* h, float* x, const float* y, const int32_t* inv,
                          const float* wts, const float* ys, const float* gate_logit, int B,
                          int d, int k, float eps) {
  EF_CHECK_ARG(B >= 0 && d > 0 && k >= 1, "bad combine shape");
  if (B == 0) return EF_OK;
  combine_kernel<<<B, 256, 0, S(stream)>>>(h, x, y, inv, wts, ys, gate_logit, d, k, eps, nullptr);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

namespace ef {
// Under CUDA lazy module loading the first launch of a kernel may wait for
// the device to go idle; the pipeline's gate kernel spins until the host
// publishes a decision, so every kernel the pipeline launches is loaded up
// front, while the device is idle.
template <typename T>
static void preload(T* fn, int& n) {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(fn)) == cudaSuccess) ++n;
}

template <typename WT>
static void preload_dtype(int& n) {
  preload(router_kernel<WT, 1>, n);
  preload(router_kernel<WT, 8>, n);
  preload(router_route_kernel<WT, 1>, n);
  preload(router_route_kernel<WT, 8>, n);
  preload(router_route_row_kernel<WT>, n);
  cudaFuncSetAttribute(router_route_row_kernel<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kCombSmemMax);
  cudaFuncSetAttribute(router_route_kernel<WT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kCombSmemMax);
  cudaFuncSetAttribute(router_route_kernel<WT, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kCombSmemMax);
  preload(ffn_gemv_kernel<WT, 1, kUpR, true, XGather<WT>, kUpU>, n);
  preload(ffn_gemv_kernel<WT, 1, 1, true, XGather<WT>, 4>, n);
  preload(ffn_gemv_kernel<WT, 2, kUpR, true, XGather<WT>, kUpU>, n);
  preload(ffn_gemv_kernel<WT, 4, kUpR, true, XGather<WT>, kUpU>, n);
  preload(ffn_gemv_kernel<WT, 8, kUpR, true, XGather<WT>, kUpU>, n);
  preload(ffn_gemv_kernel<WT, 1, kDnR, false, XAct<WT>, kDnU>, n);
  preload(ffn_gemv_kernel<WT, 2, kDnR, false, XAct<WT>, kDnU>, n);
  preload(ffn_gemv_kernel<WT, 4, kDnR, false, XAct<WT>, kDnU>, n);
  preload(ffn_gemv_kernel<WT, 8, kDnR, false, XAct<WT>, kDnU>, n);
}

// Host-buffer I/O for MoEEngine.step_host(): the hidden state is read from /
// written to pinned host memory by SMs (zero-copy), not by a copy engine: an
// H2D cudaMemcpy would queue behind an in-flight 352 MB expert swap-in on the
// shared copy engine (profiles/r01_copy_lab.txt).
__global__ void host_io_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n,
                               int to_host) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4;
       i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<float4*>(dst)[i] = __ldcv(reinterpret_cast<const float4*>(src) + i);
  for (int64_t i = (n / 4) * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcv(src + i);
  if (to_host) __threadfence_system();
}

int launch_host_io(cudaStream_t st, const float* src, float* dst, int64_t n, bool to_host) {
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>(32, (n / 4 + threads - 1) / threads + 1);
  host_io_kernel<<<blocks, threads, 0, st>>>(src, dst, n, to_host ? 1 : 0);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

int preload_pipeline_kernels() {
  int n = 0;
  preload_dtype<__nv_bfloat16>(n);
  preload_dtype<float>(n);
  preload(route_permute_kernel, n);
  preload(gate_kernel, n);
  preload(init_stats_kernel, n);
  preload(rmsnorm_kernel, n);
  preload(combine_kernel, n);
  preload(host_io_kernel, n);
  preload(ep_pack_kernel, n);
  preload(ffn_mma_kernel<true, 1>, n);
  preload(ffn_mma_kernel<false, 1>, n);
  preload(ffn_mma_kernel<true, 2>, n);
  preload(ffn_mma_kernel<false, 2>, n);
  preload(ffn_mma_kernel<true, 4>, n);
  preload(ffn_mma_kernel<false, 4>, n);
  preload(ep_owner_kernel, n);
  return n;
}
}  // namespace ef

#include "decode_layer.cuh"
