// Decode-FFN design lab (not part of the product): batch-1 SwiGLU expert FFN
// on Mixtral shapes (d=4096, ff=14336, bf16), two experts per launch pair,
// rotating over 16 experts (5.6 GB) so every launch streams from HBM.
// Times gate/up GEMV, down GEMV and the pair, for several tilings, with and
// without programmatic dependent launch (PDL) + L2 prefetch of W2.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/ffn_lab tools/ffn_lab.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

#ifdef QWEN  // Qwen1.5-MoE / DeepSeek-V2-Lite expert shape, 4 routed experts (top-4 at B=1)
constexpr int D = 2048, FF = 1408, E = 64, NA = 4;
#else
constexpr int D = 4096, FF = 14336, E = 16, NA = 2;
#endif

__device__ __forceinline__ uint4 ldw(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
__device__ __forceinline__ float wsum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float dot8(uint4 w, float4 a, float4 b, float acc) {
  acc = fmaf(lo(w.x), a.x, acc);
  acc = fmaf(hi(w.x), a.y, acc);
  acc = fmaf(lo(w.y), a.z, acc);
  acc = fmaf(hi(w.y), a.w, acc);
  acc = fmaf(lo(w.z), b.x, acc);
  acc = fmaf(hi(w.z), b.y, acc);
  acc = fmaf(lo(w.w), b.z, acc);
  acc = fmaf(hi(w.w), b.w, acc);
  return acc;
}

struct Args {
  const __nv_bfloat16* w;  // [E][3][..] W1 | W3 | W2
  int e0;                  // experts e0, e0+1 (mod E)
  const float* x;          // [D]
  __nv_bfloat16* act;      // [NA][FF]
  float* y;                // [NA][D]
};

template <int R, int U, int WARPS, bool PDL>
__global__ void __launch_bounds__(WARPS * 32) up_k(Args a) {
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int e = (a.e0 + blockIdx.y) % E;
  const __nv_bfloat16* W1 = a.w + (int64_t)e * 3 * FF * D;
  const __nv_bfloat16* W3 = W1 + (int64_t)FF * D;
  const int j0 = (blockIdx.x * WARPS + wid) * R;
  if (j0 >= FF) return;
  float ag[R], au[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ag[r] = au[r] = 0.f;
  for (int c0 = lane * 8; c0 < D; c0 += 32 * 8 * U) {
    uint4 g[U][R], u[U][R];
#pragma unroll
    for (int v = 0; v < U; ++v)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        g[v][r] = ldw(W1 + (int64_t)(j0 + r) * D + c0 + v * 256);
        u[v][r] = ldw(W3 + (int64_t)(j0 + r) * D + c0 + v * 256);
      }
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const float4* xp = reinterpret_cast<const float4*>(a.x + c0 + v * 256);
      float4 x0 = __ldg(xp), x1 = __ldg(xp + 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ag[r] = dot8(g[v][r], x0, x1, ag[r]);
        au[r] = dot8(u[v][r], x0, x1, au[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float gg = wsum(ag[r]), uu = wsum(au[r]);
    if (lane == 0) a.act[blockIdx.y * FF + j0 + r] = __float2bfloat16_rn(gg / (1.f + __expf(-gg)) * uu);
  }
}

// gate/up with a grid-stride loop over row blocks (grid = resident capacity):
// no ragged last wave
template <int R, int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) up_gs(Args a, int nblocks) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int blk = blockIdx.x; blk < nblocks * NA; blk += gridDim.x) {
    const int ea = blk / nblocks, bx = blk % nblocks;
    const int e = (a.e0 + ea) % E;
    const __nv_bfloat16* W1 = a.w + (int64_t)e * 3 * FF * D;
    const __nv_bfloat16* W3 = W1 + (int64_t)FF * D;
    const int j0 = (bx * WARPS + wid) * R;
    float ag[R], au[R];
#pragma unroll
    for (int r = 0; r < R; ++r) ag[r] = au[r] = 0.f;
    for (int c0 = lane * 8; c0 < D; c0 += 32 * 8 * U) {
      uint4 g[U][R], u[U][R];
#pragma unroll
      for (int v = 0; v < U; ++v)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          g[v][r] = ldw(W1 + (int64_t)(j0 + r) * D + c0 + v * 256);
          u[v][r] = ldw(W3 + (int64_t)(j0 + r) * D + c0 + v * 256);
        }
#pragma unroll
      for (int v = 0; v < U; ++v) {
        const float4* xp = reinterpret_cast<const float4*>(a.x + c0 + v * 256);
        float4 x0 = __ldg(xp), x1 = __ldg(xp + 1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ag[r] = dot8(g[v][r], x0, x1, ag[r]);
          au[r] = dot8(u[v][r], x0, x1, au[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float gg = wsum(ag[r]), uu = wsum(au[r]);
      if (lane == 0)
        a.act[ea * FF + j0 + r] = __float2bfloat16_rn(gg / (1.f + __expf(-gg)) * uu);
    }
  }
}

template <int R, int U, int WARPS, bool PDL, bool LDG = false>
__global__ void __launch_bounds__(WARPS * 32) down_k(Args a) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int e = (a.e0 + blockIdx.y) % E;
  const __nv_bfloat16* W2 = a.w + (int64_t)e * 3 * FF * D + 2LL * FF * D;
  const int i0 = (blockIdx.x * WARPS + wid) * R;
  if (PDL) {
    if (i0 < D && lane < R) {  // stream this warp's W2 rows into L2 while gate/up finishes
      const void* p = W2 + (int64_t)(i0 + lane) * FF;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(FF * 2) : "memory");
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (i0 >= D) return;
  const __nv_bfloat16* xa = a.act + blockIdx.y * FF;
  float acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.f;
  for (int c0 = lane * 8; c0 < FF; c0 += 32 * 8 * U) {
    uint4 w[U][R];
#pragma unroll
    for (int v = 0; v < U; ++v)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (c0 + v * 256 < FF) w[v][r] = ldw(W2 + (int64_t)(i0 + r) * FF + c0 + v * 256);
#pragma unroll
    for (int v = 0; v < U; ++v) {
      if (c0 + v * 256 < FF) {
        uint4 xv = LDG ? __ldg(reinterpret_cast<const uint4*>(xa + c0 + v * 256))
                       : __ldcg(reinterpret_cast<const uint4*>(xa + c0 + v * 256));
        float4 x0 = make_float4(lo(xv.x), hi(xv.x), lo(xv.y), hi(xv.y));
        float4 x1 = make_float4(lo(xv.z), hi(xv.z), lo(xv.w), hi(xv.w));
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = dot8(w[v][r], x0, x1, acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float s = wsum(acc[r]);
    if (lane == 0) a.y[blockIdx.y * D + i0 + r] = s;
  }
}

// down projection with each W2 row split over KS warps (smaller work units,
// better SM balance); fixed-order smem reduction.  act staged once in smem.
template <int KS, int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) down_sk(Args a) {
  __shared__ float part[WARPS];
  __shared__ __align__(16) __nv_bfloat16 xs[FF];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int e = (a.e0 + blockIdx.y) % E;
  const __nv_bfloat16* W2 = a.w + (int64_t)e * 3 * FF * D + 2LL * FF * D;
  const __nv_bfloat16* xa = a.act + blockIdx.y * FF;
  for (int i = threadIdx.x * 8; i < FF; i += WARPS * 32 * 8)
    *reinterpret_cast<uint4*>(xs + i) = __ldg(reinterpret_cast<const uint4*>(xa + i));
  __syncthreads();
  const int row = blockIdx.x * (WARPS / KS) + wid / KS;
  const int ks = wid % KS;
  constexpr int SPAN = FF / KS;
  float acc = 0.f;
  const __nv_bfloat16* wr = W2 + (int64_t)row * FF + ks * SPAN;
  const __nv_bfloat16* xr = xs + ks * SPAN;
  for (int c0 = lane * 8; c0 < SPAN; c0 += 32 * 8 * U) {
    uint4 w[U];
#pragma unroll
    for (int v = 0; v < U; ++v)
      if (c0 + v * 256 < SPAN) w[v] = ldw(wr + c0 + v * 256);
#pragma unroll
    for (int v = 0; v < U; ++v) {
      if (c0 + v * 256 < SPAN) {
        uint4 xv = *reinterpret_cast<const uint4*>(xr + c0 + v * 256);
        float4 x0 = make_float4(lo(xv.x), hi(xv.x), lo(xv.y), hi(xv.y));
        float4 x1 = make_float4(lo(xv.z), hi(xv.z), lo(xv.w), hi(xv.w));
        acc = dot8(w[v], x0, x1, acc);
      }
    }
  }
  acc = wsum(acc);
  if (lane == 0) part[wid] = acc;
  __syncthreads();
  if (threadIdx.x < WARPS / KS) {
    float s = 0.f;
    for (int q = 0; q < KS; ++q) s += part[threadIdx.x * KS + q];
    a.y[blockIdx.y * D + blockIdx.x * (WARPS / KS) + threadIdx.x] = s;
  }
}

// Persistent fused FFN: one launch, CTAs claim tiles from a counter in the
// order [up tiles of every expert][down tiles of every expert]; a down tile of
// expert e waits until all of e's up tiles have published their act rows.
struct PArgs {
  const __nv_bfloat16* w;
  int e0;
  const float* x;
  __nv_bfloat16* act;
  float* y;
  int* ctr;  // [0] tile ticket, [1 + e] finished up tiles of expert e
};
template <int UPR, int UPU, int DNU>
__global__ void __launch_bounds__(128, 8) persist_k(PArgs a) {
  constexpr int WARPS = 4;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int up_rows_per_tile = WARPS * UPR, dn_rows_per_tile = WARPS;
  constexpr int up_tiles = FF / up_rows_per_tile, dn_tiles = D / dn_rows_per_tile;
  constexpr int total = NA * (up_tiles + dn_tiles);
  __shared__ int tile_s;
  for (;;) {
    if (threadIdx.x == 0) tile_s = atomicAdd(&a.ctr[0], 1);
    __syncthreads();
    const int tile = tile_s;
    __syncthreads();
    if (tile >= total) break;
    if (tile < NA * up_tiles) {
      const int ea = tile / up_tiles, tb = tile % up_tiles;
      const int e = (a.e0 + ea) % E;
      const __nv_bfloat16* W1 = a.w + (int64_t)e * 3 * FF * D;
      const __nv_bfloat16* W3 = W1 + (int64_t)FF * D;
      const int j0 = (tb * WARPS + wid) * UPR;
      float ag[UPR], au[UPR];
#pragma unroll
      for (int r = 0; r < UPR; ++r) ag[r] = au[r] = 0.f;
      for (int c0 = lane * 8; c0 < D; c0 += 32 * 8 * UPU) {
        uint4 g[UPU][UPR], u[UPU][UPR];
#pragma unroll
        for (int v = 0; v < UPU; ++v)
#pragma unroll
          for (int r = 0; r < UPR; ++r) {
            g[v][r] = ldw(W1 + (int64_t)(j0 + r) * D + c0 + v * 256);
            u[v][r] = ldw(W3 + (int64_t)(j0 + r) * D + c0 + v * 256);
          }
#pragma unroll
        for (int v = 0; v < UPU; ++v) {
          const float4* xp = reinterpret_cast<const float4*>(a.x + c0 + v * 256);
          float4 x0 = __ldg(xp), x1 = __ldg(xp + 1);
#pragma unroll
          for (int r = 0; r < UPR; ++r) {
            ag[r] = dot8(g[v][r], x0, x1, ag[r]);
            au[r] = dot8(u[v][r], x0, x1, au[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < UPR; ++r) {
        float gg = wsum(ag[r]), uu = wsum(au[r]);
        if (lane == 0)
          a.act[ea * FF + j0 + r] = __float2bfloat16_rn(gg / (1.f + __expf(-gg)) * uu);
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(&a.ctr[1 + ea], 1);
    } else {
      const int t2 = tile - NA * up_tiles;
      const int ea = t2 / dn_tiles, tb = t2 % dn_tiles;
      if (threadIdx.x == 0) {
        while (atomicAdd(&a.ctr[1 + ea], 0) < up_tiles) __nanosleep(100);
      }
      __syncthreads();
      const int e = (a.e0 + ea) % E;
      const __nv_bfloat16* W2 = a.w + (int64_t)e * 3 * FF * D + 2LL * FF * D;
      const int i0 = tb * WARPS + wid;
      const __nv_bfloat16* xa = a.act + ea * FF;
      float acc = 0.f;
      for (int c0 = lane * 8; c0 < FF; c0 += 32 * 8 * DNU) {
        uint4 wv[DNU];
#pragma unroll
        for (int v = 0; v < DNU; ++v)
          if (c0 + v * 256 < FF) wv[v] = ldw(W2 + (int64_t)i0 * FF + c0 + v * 256);
#pragma unroll
        for (int v = 0; v < DNU; ++v)
          if (c0 + v * 256 < FF) {
            uint4 xv = __ldcg(reinterpret_cast<const uint4*>(xa + c0 + v * 256));
            float4 x0 = make_float4(lo(xv.x), hi(xv.x), lo(xv.y), hi(xv.y));
            float4 x1 = make_float4(lo(xv.z), hi(xv.z), lo(xv.w), hi(xv.w));
            acc = dot8(wv[v], x0, x1, acc);
          }
      }
      acc = wsum(acc);
      if (lane == 0) a.y[ea * D + i0] = acc;
    }
  }
}

__global__ void fill_k(__nv_bfloat16* w, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)(i * 2654435761u);
    w[i] = __float2bfloat16_rn(((h >> 8) & 0xffff) / 65536.f - 0.5f);
  }
}

using KFn = void (*)(Args);

struct Up {
  const char* name;
  KFn fn;
  int rows_per_cta;
  int threads;
};

template <int R, int U, int W, bool P>
Up mk_up(const char* n) {
  return Up{n, up_k<R, U, W, P>, R * W, W * 32};
}
template <int R, int U, int W, bool P, bool G = false>
Up mk_dn(const char* n) {
  return Up{n, down_k<R, U, W, P, G>, R * W, W * 32};
}
template <int KS, int U, int W>
Up mk_sk(const char* n) {
  return Up{n, down_sk<KS, U, W>, W / KS, W * 32};
}

static void launch(KFn fn, int rows, int per, int threads, Args a, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t c{};
  c.gridDim = dim3((rows + per - 1) / per, NA);
  c.blockDim = dim3(threads);
  c.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = at;
  c.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&c, fn, a));
}

int main() {
  __nv_bfloat16* w;
  const int64_t per = 3LL * FF * D;
  CK(cudaMalloc(&w, per * E * 2));
  fill_k<<<2048, 256>>>(w, per * E);
  float *x, *y;
  __nv_bfloat16* act;
  CK(cudaMalloc(&x, D * 4));
  CK(cudaMalloc(&y, NA * D * 4));
  CK(cudaMalloc(&act, NA * FF * 2));
  std::vector<float> hx(D);
  for (int i = 0; i < D; ++i) hx[i] = (i % 17) * 0.01f - 0.08f;
  CK(cudaMemcpy(x, hx.data(), D * 4, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double up_bytes = 2.0 * FF * D * 2 * NA, dn_bytes = 1.0 * FF * D * 2 * NA;
  const int IT = 48;

  auto time_it = [&](auto&& body) {
    for (int i = 0; i < 4; ++i) body(i);
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < IT; ++i) body(i);
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms * 1e3 / IT;  // us per iteration
  };

#ifdef QWEN
  std::vector<Up> ups = {
      mk_up<2, 2, 4, false>("up R2 U2 W4 (engine)"), mk_up<1, 4, 4, false>("up R1 U4 W4"),
      mk_up<1, 2, 4, false>("up R1 U2 W4"),          mk_up<1, 4, 2, false>("up R1 U4 W2"),
      mk_up<1, 8, 4, false>("up R1 U8 W4"),          mk_up<1, 2, 2, false>("up R1 U2 W2"),
  };
  std::vector<Up> dns = {
      mk_dn<1, 2, 4, false, true>("down R1 U2 W4 ldg (engine)"), mk_dn<1, 1, 4, false, true>("down R1 U1 W4 ldg"),
      mk_dn<1, 4, 4, false, true>("down R1 U4 W4 ldg"),          mk_dn<1, 2, 2, false, true>("down R1 U2 W2 ldg"),
      mk_dn<1, 1, 2, false, true>("down R1 U1 W2 ldg"),          mk_dn<2, 1, 4, false, true>("down R2 U1 W4 ldg"),
  };
#else
  std::vector<Up> ups = {
      mk_up<4, 1, 4, false>("up R4 U1 W4 (engine)"), mk_up<2, 2, 4, false>("up R2 U2 W4"),
      mk_up<2, 2, 2, false>("up R2 U2 W2"),          mk_up<2, 2, 8, false>("up R2 U2 W8"),
      mk_up<1, 2, 4, false>("up R1 U2 W4"),          mk_up<2, 1, 4, false>("up R2 U1 W4"),
      mk_up<1, 4, 4, false>("up R1 U4 W4"),          mk_up<2, 3, 4, false>("up R2 U3 W4"),
      mk_up<1, 2, 8, false>("up R1 U2 W8"),          mk_up<2, 2, 16, false>("up R2 U2 W16"),
  };
  std::vector<Up> dns = {
      mk_dn<1, 4, 4, false>("down R1 U4 W4 (engine)"),     mk_dn<1, 2, 4, false>("down R1 U2 W4"),
      mk_dn<1, 4, 4, false, true>("down R1 U4 W4 ldg"),    mk_dn<1, 2, 4, false, true>("down R1 U2 W4 ldg"),
      mk_dn<2, 2, 4, false, true>("down R2 U2 W4 ldg"),    mk_dn<1, 1, 4, false, true>("down R1 U1 W4 ldg"),
      mk_dn<1, 2, 8, false, true>("down R1 U2 W8 ldg"),    mk_dn<2, 1, 4, false, true>("down R2 U1 W4 ldg"),
      mk_sk<2, 2, 8>("down splitK2 U2 W8 smem"),          mk_sk<4, 2, 8>("down splitK4 U2 W8 smem"),
      mk_sk<2, 4, 8>("down splitK2 U4 W8 smem"),          mk_sk<4, 1, 16>("down splitK4 U1 W16 smem"),
      mk_sk<7, 1, 14>("down splitK7 U1 W14 smem"),        mk_sk<2, 2, 16>("down splitK2 U2 W16 smem"),
  };
#endif
  for (auto& u : ups) {
    float t = time_it([&](int i) {
      launch(u.fn, FF, u.rows_per_cta, u.threads, Args{w, (2 * i) % E, x, act, y}, s, false);
    });
    printf("%-28s %8.1f us %7.0f GB/s\n", u.name, t, up_bytes / t * 1e-3);
  }
  for (auto& dn : dns) {
    float t = time_it([&](int i) {
      launch(dn.fn, D, dn.rows_per_cta, dn.threads, Args{w, (2 * i) % E, x, act, y}, s, false);
    });
    printf("%-28s %8.1f us %7.0f GB/s\n", dn.name, t, dn_bytes / t * 1e-3);
  }
  // pairs: engine tiling, with and without PDL + W2 prefetch
  struct Pair {
    const char* name;
    Up u, d;
    bool pdl;
  };
#ifdef QWEN
  std::vector<Pair> pairs = {
      {"pair engine", mk_up<2, 2, 4, false>(""), mk_dn<1, 2, 4, false, true>(""), false},
      {"pair R1U4 + R1U2", mk_up<1, 4, 4, false>(""), mk_dn<1, 2, 4, false, true>(""), false},
      {"pair R1U4W2 + R1U1W2", mk_up<1, 4, 2, false>(""), mk_dn<1, 1, 2, false, true>(""), false},
  };
#else
  std::vector<Pair> pairs = {
      {"pair engine", mk_up<4, 1, 4, false>(""), mk_dn<1, 4, 4, false>(""), false},
      {"pair R2U2 + R1U2ldg", mk_up<2, 2, 4, false>(""), mk_dn<1, 2, 4, false, true>(""), false},
      {"pair R2U2 + sk2U2W8", mk_up<2, 2, 4, false>(""), mk_sk<2, 2, 8>(""), false},
      {"pair R2U2 + sk4U2W8", mk_up<2, 2, 4, false>(""), mk_sk<4, 2, 8>(""), false},
  };
#endif
  for (auto& p : pairs) {
    float t = time_it([&](int i) {
      Args a{w, (2 * i) % E, x, act, y};
      launch(p.u.fn, FF, p.u.rows_per_cta, p.u.threads, a, s, false);
      launch(p.d.fn, D, p.d.rows_per_cta, p.d.threads, a, s, p.pdl);
    });
    printf("%-28s %8.1f us %7.0f GB/s\n", p.name, t, (up_bytes + dn_bytes) / t * 1e-3);
  }
  // grid-stride gate/up (grid = resident capacity)
  for (int per_sm : {8, 7, 6}) {
    float t = time_it([&](int i) {
      constexpr int R = 2, W = 4;
      up_gs<R, 2, W><<<148 * per_sm, W * 32, 0, s>>>(Args{w, (2 * i) % E, x, act, y}, FF / (R * W));
    });
    printf("up grid-stride %d/SM           %8.1f us %7.0f GB/s\n", per_sm, t, up_bytes / t * 1e-3);
  }
  // persistent fused variant
  int* ctr;
  CK(cudaMalloc(&ctr, 64 * sizeof(int)));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto persist_time = [&](auto kern, const char* name, int per_sm) {
    float t = time_it([&](int i) {
      CK(cudaMemsetAsync(ctr, 0, 64 * sizeof(int), s));
      kern<<<sms * per_sm, 128, 0, s>>>(PArgs{w, (2 * i) % E, x, act, y, ctr});
    });
    printf("%-28s %8.1f us %7.0f GB/s\n", name, t, (up_bytes + dn_bytes) / t * 1e-3);
  };
#ifndef QWEN
  persist_time(persist_k<2, 2, 2>, "persist 8/SM up2x2 dn2", 8);
  persist_time(persist_k<2, 2, 2>, "persist 6/SM up2x2 dn2", 6);
  persist_time(persist_k<2, 2, 4>, "persist 8/SM up2x2 dn4", 8);
  persist_time(persist_k<1, 4, 2>, "persist 8/SM up1x4 dn2", 8);
#else
  persist_time(persist_k<1, 4, 2>, "persist 8/SM up1x4 dn2", 8);
#endif
  // isolated pair (sync between iterations, as in the engine where each layer
  // is gated by the host): launch latency and ramp included
  for (auto& p : pairs) {
    double tot = 0;
    for (int i = 0; i < 24; ++i) {
      Args a{w, (2 * i) % E, x, act, y};
      CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(e0, s));
      launch(p.u.fn, FF, p.u.rows_per_cta, p.u.threads, a, s, false);
      launch(p.d.fn, D, p.d.rows_per_cta, p.d.threads, a, s, p.pdl);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (i >= 4) tot += ms * 1e3;
    }
    double t = tot / 20;
    printf("isolated %-19s %8.1f us %7.0f GB/s\n", p.name, t, (up_bytes + dn_bytes) / t * 1e-3);
  }
  return 0;
}
