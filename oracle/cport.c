/* oracle/cport.c — CPU port of the canonical MoE decode-layer arithmetic.
 *
 * TEST AND BASELINE INFRASTRUCTURE (see oracle/__init__.py): used by tests/
 * as a checked restatement and by bench.py's cpu_baseline leg and
 * `--impl reference` arm as the CPU implementation of the path timed beside
 * the GPU.  Never linked into, loaded by or called from the product.
 *
 * The reference (/root/reference/pkg/src/moesim) has no layer arithmetic: it
 * charges a constant T_l per layer (engine.py:263, :606).  The
 * semantics restated here are those of oracle/numerics.py:
 *   weights  element i of a tensor = fp32(int24(mix64(key + (i+1)*GOLDEN)) - 2^23) * scale,
 *            rounded to bf16 (round-to-nearest-even)       — numerics.fill_uniform / to_bf16
 *   expert   y = W2 . T(silu(W1 . xe) * (W3 . xe)), fp32 accumulation, T = bf16 rounding
 *                                                          — numerics.swiglu
 * Weights stay in bf16 in host RAM (the expert blob layout of the HBM slab,
 * [W1 ff x d | W3 ff x d | W2 d x ff]) and are widened on the fly, so the CPU
 * streams the same bytes per token as the GPU.  OpenMP over output rows.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint16_t f32_to_bf16(float v) {
  uint32_t b;
  memcpy(&b, &v, 4);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

static inline float bf16_to_f32(uint16_t h) {
  uint32_t b = (uint32_t)h << 16;
  float v;
  memcpy(&v, &b, 4);
  return v;
}

/* numerics.fill_uniform + to_bf16 (engine weights, ef_fill_uniform on device) */
void cp_fill_bf16(uint16_t* dst, int64_t n, uint64_t key, float scale, int64_t offset) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = mix64(key + (uint64_t)(offset + i + 1) * GOLDEN);
    int32_t u = (int32_t)(h >> 40) - 8388608;
    dst[i] = f32_to_bf16((float)u * scale);
  }
}

/* 16 independent fp32 partial sums (vectorisable without reassociation
   flags), folded in a fixed order */
__attribute__((target_clones("avx512f", "avx2", "default")))
float dot_bf16(const uint16_t* w, const float* x, int n) {
  float acc[16] = {0};
  int i = 0;
  for (; i + 16 <= n; i += 16)
    for (int k = 0; k < 16; ++k) acc[k] += bf16_to_f32(w[i + k]) * x[i + k];
  for (; i < n; ++i) acc[i & 15] += bf16_to_f32(w[i]) * x[i];
  float s = 0.f;
  for (int k = 0; k < 16; ++k) s += acc[k];
  return s;
}

__attribute__((target_clones("avx512f", "avx2", "default")))
float dot_f32(const float* w, const float* x, int n) {
  float acc[16] = {0};
  int i = 0;
  for (; i + 16 <= n; i += 16)
    for (int k = 0; k < 16; ++k) acc[k] += w[i + k] * x[i + k];
  for (; i < n; ++i) acc[i & 15] += w[i] * x[i];
  float s = 0.f;
  for (int k = 0; k < 16; ++k) s += acc[k];
  return s;
}

/* Y[t][r] = sum_c W[r][c] * X[t][c]; W bf16 (dtype 1) or fp32 (dtype 0), rows x cols */
void cp_gemv(const void* W, int dtype, int rows, int cols, const float* X, int n, float* Y) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int t = 0; t < n; ++t)
      Y[(int64_t)t * rows + r] =
          dtype ? dot_bf16((const uint16_t*)W + (int64_t)r * cols, X + (int64_t)t * cols, cols)
                : dot_f32((const float*)W + (int64_t)r * cols, X + (int64_t)t * cols, cols);
}

/* One SwiGLU expert on n rows: xe[n][d] (already in the weight dtype's
   values), blob = [W1 | W3 | W2]; act scratch [n][ff]; y[n][d]. */
void cp_swiglu(const void* blob, int dtype, int d, int ff, const float* xe, int n, float* act,
               float* y) {
  const int64_t nf = (int64_t)ff * d;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < ff; ++j) {
    for (int t = 0; t < n; ++t) {
      float g, u;
      if (dtype) {
        const uint16_t* w = (const uint16_t*)blob;
        g = dot_bf16(w + (int64_t)j * d, xe + (int64_t)t * d, d);
        u = dot_bf16(w + nf + (int64_t)j * d, xe + (int64_t)t * d, d);
      } else {
        const float* w = (const float*)blob;
        g = dot_f32(w + (int64_t)j * d, xe + (int64_t)t * d, d);
        u = dot_f32(w + nf + (int64_t)j * d, xe + (int64_t)t * d, d);
      }
      float a = g / (1.0f + expf(-g)) * u;
      act[(int64_t)t * ff + j] = dtype ? bf16_to_f32(f32_to_bf16(a)) : a;
    }
  }
#pragma omp parallel for schedule(static)
  for (int i = 0; i < d; ++i)
    for (int t = 0; t < n; ++t)
      y[(int64_t)t * d + i] =
          dtype ? dot_bf16((const uint16_t*)blob + 2 * nf + (int64_t)i * ff, act + (int64_t)t * ff, ff)
                : dot_f32((const float*)blob + 2 * nf + (int64_t)i * ff, act + (int64_t)t * ff, ff);
}

int cp_num_threads(void) {
  int n = 1;
#pragma omp parallel
  {
#pragma omp single
    n = omp_get_num_threads();
  }
  return n;
}
