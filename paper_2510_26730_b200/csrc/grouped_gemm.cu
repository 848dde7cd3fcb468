// grouped_gemm.cu — (d) prefill expert FFN: TMA + tcgen05 grouped GEMM for sm_100a.
//
// One persistent launch computes every (expert, m-tile, n-tile) tile of a
// grouped GEMM  C[rows_e, N] = A[rows_e, K] · B_eᵀ  where A is the permuted
// token matrix (bf16, K-contiguous) and B_e an expert's weight matrix inside
// the slot-indirected HBM slab (bf16 [N, K], K-contiguous) — the slab is
// viewed as one 2-D tensor so a single TMA descriptor reaches every slot.
//
//   warp 0      TMA producer (one elected lane): A and B tiles, 128B swizzle,
//               STAGES-deep smem ring guarded by full/empty mbarriers
//   warp 1      MMA issuer (one lane): tcgen05.mma.cta_group::1.kind::f16,
//               M=128 N=128 K=16 per instruction, fp32 accumulators in TMEM,
//               double-buffered so the epilogue of tile i overlaps tile i+1
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> global
//               DUAL: B holds W1 and W3 rows; act = bf16(silu(h) * u)
//               else: y = fp32 accumulator
// Tiles are ordered (expert, n-tile, m-tile) so CTAs running concurrently
// share an expert's weight tile through L2.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/expertflow.h"

namespace ef {
extern thread_local std::string g_last_error;
}

namespace efg {

constexpr int BM = 128, BN = 128, BK = 64;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  const long long c0 = clock64();
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    // a pipeline bug must fail loudly, never hang the GPU (~10 s at 2 GHz)
    if (!done && clock64() - c0 > 20000000000LL) asm volatile("trap;");
  } while (!done);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major, 128-byte-swizzled operand tile (rows of 64 bf16): SBO = 1024 B
// between 8-row groups, LBO unused (1), version 1 (sm100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t start = (smem_u32(p) & 0x3FFFFu) >> 4;
  return start | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: D=f32, A=B=bf16, both K-major, N=BN, M=BM.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

template <bool DUAL>
struct Cfg {
  static constexpr int B_TILE = DUAL ? 2 * B_BYTES : B_BYTES;
  static constexpr int STAGE = A_BYTES + B_TILE;
  static constexpr int STAGES = DUAL ? 4 : 6;
  static constexpr int ACC_COLS = DUAL ? 2 * BN : BN;  // fp32 columns per accumulator buffer
  static constexpr int TMEM_COLS = 2 * ACC_COLS;       // double buffered (power of 2)
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

// tiles[i] = {a_row0, b_row0 (first weight row of the expert), m_valid, n0}
template <bool DUAL>
__global__ void __launch_bounds__(192, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const int4* __restrict__ tiles,
                        int n_tiles, int K, int dual_off, void* __restrict__ out, int out_ld) {
  using C = Cfg<DUAL>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_sh)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_sh;
  const int kblocks = K / BK;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int4 tl = tiles[t];
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full[stage], C::STAGE);
          tma_load_2d(sa, &tmA, &full[stage], kb * BK, tl.x);
          tma_load_2d(sb, &tmB, &full[stage], kb * BK, tl.y + tl.w);
          if (DUAL) tma_load_2d(sb + B_BYTES, &tmB, &full[stage], kb * BK, tl.y + dual_off + tl.w);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * C::ACC_COLS;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint8_t* sa = smem + stage * C::STAGE;
          const uint8_t* sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = smem_desc_sw128(sa) + (uint64_t)(2 * k);
            const uint64_t bd = smem_desc_sw128(sb) + (uint64_t)(2 * k);
            const uint32_t accum = (kb | k) ? 1u : 0u;
            umma_f16(d0, ad, bd, accum);
            if (DUAL) umma_f16(d0 + BN, ad, smem_desc_sw128(sb + B_BYTES) + (uint64_t)(2 * k), accum);
          }
          umma_commit(&empty[stage]);  // frees the smem stage when these MMAs retire
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {  // ---------------- epilogue warps 2..5
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int4 tl = tiles[t];
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * C::ACC_COLS;
      const bool valid = row < tl.z;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t h[16], u[16];
        tmem_ld16(taddr + c, h);
        if (DUAL) tmem_ld16(taddr + BN + c, u);
        tmem_wait_ld();
        if (valid) {
          const int64_t o = (int64_t)(tl.x + row) * out_ld + tl.w + c;
          if (DUAL) {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(out) + o;
            uint32_t packed[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              float g0 = __uint_as_float(h[2 * i]), g1 = __uint_as_float(h[2 * i + 1]);
              float v0 = g0 / (1.0f + expf(-g0)) * __uint_as_float(u[2 * i]);
              float v1 = g1 / (1.0f + expf(-g1)) * __uint_as_float(u[2 * i + 1]);
              __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
              packed[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
            d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
          } else {
            float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              d4[i] = make_float4(__uint_as_float(h[4 * i]), __uint_as_float(h[4 * i + 1]),
                                  __uint_as_float(h[4 * i + 2]), __uint_as_float(h[4 * i + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(C::TMEM_COLS));
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor [rows, cols] with row pitch `pitch_elems`, box 64 x 128, 128B swizzle.
static bool make_tmap(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols,
                      int64_t pitch_elems) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(pitch_elems * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool DUAL>
static int launch(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, const int4* tiles,
                  int n_tiles, int K, int dual_off, void* out, int out_ld) {
  using C = Cfg<DUAL>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(grouped_gemm_kernel<DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::SMEM) != cudaSuccess)
      return EF_ECUDA;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = std::min(n_tiles, sms);
  if (grid < 1) return EF_OK;
  grouped_gemm_kernel<DUAL><<<grid, 192, C::SMEM, st>>>(ta, tb, tiles, n_tiles, K, dual_off, out,
                                                         out_ld);
  return EF_OK;
}

}  // namespace efg

// C ABI (include/expertflow.h).  tiles: device int4[n_tiles].
extern "C" int ef_grouped_gemm_bf16(void* stream, const void* A, int64_t a_rows, int K,
                                    const void* B, int64_t b_rows, int64_t b_pitch,
                                    const void* tiles, int n_tiles, int dual, int dual_off,
                                    void* out, int out_ld) {
  using namespace efg;
  if (K % BK != 0 || K <= 0) {
    ef::g_last_error = "K must be a positive multiple of 64";
    return EF_EINVAL;
  }
  if (out_ld % 16 != 0) {
    ef::g_last_error = "output leading dimension must be a multiple of 16";
    return EF_EINVAL;
  }
  CUtensorMap ta, tb;
  if (!make_tmap(&ta, A, a_rows, K, K) || !make_tmap(&tb, B, b_rows, K, b_pitch)) {
    ef::g_last_error = "cuTensorMapEncodeTiled failed (alignment / driver entry point)";
    return EF_ECUDA;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc = dual ? launch<true>(st, ta, tb, reinterpret_cast<const int4*>(tiles), n_tiles, K,
                               dual_off, out, out_ld)
                : launch<false>(st, ta, tb, reinterpret_cast<const int4*>(tiles), n_tiles, K, 0,
                                out, out_ld);
  if (rc != EF_OK) return rc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ef::g_last_error = std::string("grouped_gemm launch: ") + cudaGetErrorString(e);
    return EF_ECUDA;
  }
  return EF_OK;
}
