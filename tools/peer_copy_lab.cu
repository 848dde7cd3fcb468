// Peer-tier copy lab: does a device-to-device expert copy need SMs?
//
// The engine's routed FFN may occupy every SM while it spins on the ready flag
// of a slot being filled; the fill must therefore run on a copy engine.  This
// lab launches a kernel that holds all SMs and spins (bounded by a 2 s timeout)
// until a flag published by a 4-byte H2D copy queued behind the expert copy,
// for each way of issuing a same-device copy.  "timeout" means the copy needed
// SMs (it only ran after the spinners gave up).  Also times each variant alone.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/peer_copy_lab tools/peer_copy_lab.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void spin(volatile uint32_t* flag, uint32_t want, int* timed_out, uint64_t* waited) {
  if (threadIdx.x == 0) {
    uint64_t t0 = gtime();
    while (*flag != want) {
      if (gtime() - t0 > 2000000000ull) {
        atomicExch(timed_out, 1);
        break;
      }
    }
    if (blockIdx.x == 0) *waited = gtime() - t0;
  }
  __syncthreads();
}

enum Mode { PEER = 0, D2D = 1 };
static const char* names[] = {"cudaMemcpyPeerAsync (same device)", "cudaMemcpyAsync D2D"};

static cudaError_t issue(int mode, void* dst, void* src, size_t n, cudaStream_t s) {
  if (mode == PEER) return cudaMemcpyPeerAsync(dst, 0, src, 0, n, s);
  return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s);
}

int main() {
  const size_t n = 352321536;  // one Mixtral-8x7B expert, bf16
  char *src, *dst;
  uint32_t* flag;
  int* tout;
  uint64_t* waited;
  uint32_t* hflag;
  CK(cudaMalloc(&src, n));
  CK(cudaMalloc(&dst, n));
  CK(cudaMemset(src, 1, n));
  CK(cudaMalloc(&flag, 4));
  CK(cudaMemset(flag, 0, 4));
  CK(cudaMallocManaged(&tout, 4));
  CK(cudaMallocManaged(&waited, 8));
  CK(cudaHostAlloc(&hflag, 4, cudaHostAllocDefault));
  int sms = 0, per = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spin, 128, 0));
  cudaStream_t cs, ks;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  printf("SMs %d, spinner blocks/SM %d\n", sms, per);
  uint32_t seq = 0;
  for (int mode = 0; mode < 2; ++mode) {
    // alone: bandwidth
    for (int w = 0; w < 2; ++w) CK(issue(mode, dst, src, n, cs));
    CK(cudaEventRecord(a, cs));
    for (int r = 0; r < 5; ++r) CK(issue(mode, dst, src, n, cs));
    CK(cudaEventRecord(b, cs));
    CK(cudaStreamSynchronize(cs));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    // under a kernel holding every SM
    *tout = 0;
    *waited = 0;
    ++seq;
    CK(cudaDeviceSynchronize());
    spin<<<sms * per, 128, 0, ks>>>(flag, seq, tout, waited);
    CK(cudaGetLastError());
    CK(issue(mode, dst, src, n, cs));
    *hflag = seq;
    CK(cudaMemcpyAsync(flag, hflag, 4, cudaMemcpyHostToDevice, cs));
    CK(cudaDeviceSynchronize());
    printf("%-48s alone %.1f GB/s (copy+read+write %.1f GB/s) | under full-SM spinner: %s, "
           "flag after %.3f ms\n",
           names[mode], n * 5 / (ms * 1e-3) / 1e9, 2.0 * n * 5 / (ms * 1e-3) / 1e9,
           *tout ? "TIMEOUT (copy needs SMs)" : "ok (copy engine)", *waited / 1e6);
  }
  return 0;
}
