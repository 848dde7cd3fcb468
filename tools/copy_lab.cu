// H2D expert-copy interference lab (not part of the product).  Measures how a
// concurrent 352 MB host->device expert copy slows (a) the decode FFN GEMV
// pair and (b) a control round trip (kernel launch + one mapped-host-memory
// read), for several copy mechanisms:
//   none | copy engine, one memcpy | copy engine, 4 MB chunks |
//   SM pull kernel (few CTAs, bounded bytes in flight, low-priority stream)
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/copy_lab tools/copy_lab.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr int D = 4096, FF = 14336, E = 8, NA = 2;
constexpr int64_t BLOB = 3LL * FF * D * 2;

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

template <int R = 2, int U = 2>
__global__ void __launch_bounds__(128) up_k(const __nv_bfloat16* w, int e0, const float* x,
                                            __nv_bfloat16* act) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int e = (e0 + blockIdx.y) % E;
  const __nv_bfloat16* W1 = w + (int64_t)e * 3 * FF * D;
  const __nv_bfloat16* W3 = W1 + (int64_t)FF * D;
  const int j0 = (blockIdx.x * 4 + wid) * R;
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
      const float4* xp = reinterpret_cast<const float4*>(x + c0 + v * 256);
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
      act[blockIdx.y * FF + j0 + r] = __float2bfloat16_rn(gg / (1.f + __expf(-gg)) * uu);
  }
}

template <int U = 2>
__global__ void __launch_bounds__(128) down_k(const __nv_bfloat16* w, int e0,
                                              const __nv_bfloat16* act, float* y) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int e = (e0 + blockIdx.y) % E;
  const __nv_bfloat16* W2 = w + (int64_t)e * 3 * FF * D + 2LL * FF * D;
  const int i0 = blockIdx.x * 4 + wid;
  const __nv_bfloat16* xa = act + blockIdx.y * FF;
  float acc = 0.f;
  for (int c0 = lane * 8; c0 < FF; c0 += 32 * 8 * U) {
    uint4 wv[U];
#pragma unroll
    for (int v = 0; v < U; ++v)
      if (c0 + v * 256 < FF) wv[v] = ldw(W2 + (int64_t)i0 * FF + c0 + v * 256);
#pragma unroll
    for (int v = 0; v < U; ++v)
      if (c0 + v * 256 < FF) {
        uint4 xv = __ldg(reinterpret_cast<const uint4*>(xa + c0 + v * 256));
        float4 x0 = make_float4(lo(xv.x), hi(xv.x), lo(xv.y), hi(xv.y));
        float4 x1 = make_float4(lo(xv.z), hi(xv.z), lo(xv.w), hi(xv.w));
        acc = dot8(wv[v], x0, x1, acc);
      }
  }
  acc = wsum(acc);
  if (lane == 0) y[blockIdx.y * D + i0] = acc;
}

// control round trip: read one word of mapped host memory and record it
__global__ void ctrl_k(const volatile uint32_t* host_word, uint32_t* out) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(host_word) : "memory");
  *out = v;
}

// SM pull copy: each CTA streams its share of the blob from mapped pinned host
// memory with IN 16-byte loads in flight per thread.
template <int IN>
__global__ void __launch_bounds__(256) pull_k(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                              int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * IN;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * IN + threadIdx.x; base < n16;
       base += stride) {
    uint4 v[IN];
#pragma unroll
    for (int u = 0; u < IN; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < n16) v[u] = __ldcv(src + i);
    }
#pragma unroll
    for (int u = 0; u < IN; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < n16) __stcg(dst + i, v[u]);
    }
  }
}

__global__ void fill_k(__nv_bfloat16* w, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __float2bfloat16_rn(((uint32_t)(i * 2654435761u) >> 20) / 4096.f - 0.5f);
}

int main() {
  int lo_prio, hi_prio;
  CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  __nv_bfloat16* w;
  CK(cudaMalloc(&w, BLOB * E));
  fill_k<<<2048, 256>>>(w, BLOB / 2 * E);
  char* slab;
  CK(cudaMalloc(&slab, BLOB));
  char* host;
  CK(cudaHostAlloc(&host, BLOB, cudaHostAllocMapped));
  for (int64_t i = 0; i < BLOB; i += 4096) host[i] = (char)i;
  char* host_dev;
  CK(cudaHostGetDevicePointer((void**)&host_dev, host, 0));
  uint32_t* hword;
  CK(cudaHostAlloc(&hword, 64, cudaHostAllocMapped));
  *hword = 7;
  uint32_t* hword_dev;
  CK(cudaHostGetDevicePointer((void**)&hword_dev, hword, 0));
  char *small_h, *small_hd, *small_d;
  CK(cudaHostAlloc(&small_h, 16384, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&small_hd, small_h, 0));
  CK(cudaMalloc(&small_d, 16384));
  float *x, *y;
  __nv_bfloat16* act;
  uint32_t* out;
  CK(cudaMalloc(&x, D * 4));
  CK(cudaMalloc(&y, NA * D * 4));
  CK(cudaMalloc(&act, NA * FF * 2));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(x, 0, D * 4));
  cudaStream_t s, cs;
  CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi_prio));
  CK(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, lo_prio));
  cudaEvent_t e0, e1, c0, c1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&c0));
  CK(cudaEventCreate(&c1));
  CK(cudaDeviceSynchronize());

  auto start_copy = [&](int mode) {
    CK(cudaEventRecord(c0, cs));
    if (mode == 1) {
      CK(cudaMemcpyAsync(slab, host, BLOB, cudaMemcpyHostToDevice, cs));
    } else if (mode == 2) {
      for (int64_t o = 0; o < BLOB; o += 4 << 20)
        CK(cudaMemcpyAsync(slab + o, host + o, std::min<int64_t>(4 << 20, BLOB - o),
                           cudaMemcpyHostToDevice, cs));
    } else if (mode >= 3) {
      const int ctas = mode == 3 ? 8 : mode == 4 ? 16 : 32;
      pull_k<2><<<ctas, 256, 0, cs>>>((const uint4*)host_dev, (uint4*)slab, BLOB / 16);
    }
    CK(cudaEventRecord(c1, cs));
  };
  const char* names[] = {"no copy", "CE memcpy 352MB", "CE 4MB chunks", "pull 8 CTAs",
                         "pull 16 CTAs", "pull 32 CTAs"};
  for (int mode = 0; mode < 6; ++mode) {
    start_copy(mode);
    // while the copy runs: alternate FFN pairs and control round trips
    double ffn_us = 0, ctrl_us = 0, small_us = 0, zc_us = 0, ffn2_us = 0, ffn3_us = 0;
    int n_ffn = 0, n_ctrl = 0, n_small = 0, n_zc = 0;
    for (int it = 0; it < 40; ++it) {
      CK(cudaEventRecord(e0, s));
      up_k<<<dim3(FF / 8, NA), 128, 0, s>>>(w, (2 * it) % E, x, act);
      down_k<<<dim3(D / 4, NA), 128, 0, s>>>(w, (2 * it) % E, act, y);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 2) ffn_us += ms * 1e3, ++n_ffn;
      // deeper-pipelined variant: 2 rows x 4 chunks up, 4 chunks down
      CK(cudaEventRecord(e0, s));
      up_k<2, 4><<<dim3(FF / 8, NA), 128, 0, s>>>(w, (2 * it + 1) % E, x, act);
      down_k<4><<<dim3(D / 4, NA), 128, 0, s>>>(w, (2 * it + 1) % E, act, y);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 2) ffn2_us += ms * 1e3;
      CK(cudaEventRecord(e0, s));
      up_k<4, 2><<<dim3(FF / 16, NA), 128, 0, s>>>(w, (2 * it) % E, x, act);
      down_k<8><<<dim3(D / 4, NA), 128, 0, s>>>(w, (2 * it) % E, act, y);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 2) ffn3_us += ms * 1e3;
      CK(cudaEventRecord(e0, s));
      ctrl_k<<<1, 32, 0, s>>>(hword_dev, out);
      ctrl_k<<<1, 32, 0, s>>>(hword_dev, out);
      ctrl_k<<<1, 32, 0, s>>>(hword_dev, out);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 2) ctrl_us += ms * 1e3 / 3, ++n_ctrl;
      // small H2D copy (16 KB, a B=1 hidden state) on the compute stream
      CK(cudaEventRecord(e0, s));
      CK(cudaMemcpyAsync(small_d, small_h, 16384, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 2) small_us += ms * 1e3, ++n_small;
      // the same 16 KB pulled by a kernel from mapped host memory
      CK(cudaEventRecord(e0, s));
      pull_k<1><<<4, 256, 0, s>>>((const uint4*)small_hd, (uint4*)small_d, 1024);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 2) zc_us += ms * 1e3, ++n_zc;
      if (mode && cudaEventQuery(c1) == cudaSuccess) break;
    }
    CK(cudaEventSynchronize(c1));
    float cms = 0;
    CK(cudaEventElapsedTime(&cms, c0, c1));
    printf("%-18s deep ffn (up 2x4, down 4) %7.1f us  (up 4x2, down 8) %7.1f us\n", names[mode],
           n_ffn ? ffn2_us / n_ffn : 0.0, n_ffn ? ffn3_us / n_ffn : 0.0);
    printf("%-18s ffn pair %7.1f us  ctrl kernel %6.2f us  16KB memcpy %7.1f us  16KB zero-copy "
           "kernel %6.1f us  copy %7.2f ms (%5.1f GB/s)  samples %d\n",
           names[mode], n_ffn ? ffn_us / n_ffn : 0.0, n_ctrl ? ctrl_us / n_ctrl : 0.0,
           n_small ? small_us / n_small : 0.0, n_zc ? zc_us / n_zc : 0.0, cms,
           mode ? BLOB / (cms * 1e6) : 0.0, n_ffn);
  }
  return 0;
}
