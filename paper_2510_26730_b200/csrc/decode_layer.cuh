// decode_layer.cuh — the persistent decode layer kernel (included by kernels.cu,
// whose device helpers it uses).
//
// One launch per MoE layer replaces the three-kernel pipeline (router_route,
// gate/up, down) for batches of up to 8 tokens.  A fixed grid of one
// 512-thread CTA per SM runs four independent 4-warp WORKERS; each worker
// takes work items from the layer's queue (one atomicAdd) in this order:
//
//   [router rows]  (worker 0 of each CTA, claimed before the PDL wait so the
//                  row's weights are prefetched into shared memory with
//                  cp.async while the previous layer drains) one row of the
//                  layer's router, a pre-gate row of a later layer or the
//                  shared-expert gate, for every token; the worker that
//                  finishes the last row (ticket) ROUTES: top-k with the
//                  cache-aware bias, routing weights, stable permutation,
//                  device-side slot resolution from the slot-table row passed
//                  in the launch, the global routing outputs, and the
//                  selection + scored rows published to the host as tagged
//                  8-byte words (no system fence: under an expert swap-in a
//                  fence.sys costs ~14 us); on an unresolved layer it waits
//                  for the host's decision block (fused gate)
//   [shared up]    16-row gate/up units of the shared expert(s): no routing
//                  dependency, so they stream while the router and route run
//   [routed up]    16-row gate/up units of each decision entry.  A worker's
//                  first routed item waits for the router ticket and routes
//                  the layer ITSELF from the logits (the same deterministic
//                  code as the routing worker, so bit-identical), instead of
//                  waiting for the routing worker's stores and flag — two
//                  fewer dependent memory round trips, each several us while
//                  the shared expert saturates HBM; then it waits for its
//                  slot's copy to land (ready[slot] >= fill seq)
//   [shared down]  16-row down units of the shared expert (wait: all shared up)
//   [routed down]  16-row down units of each entry (wait: that entry's up units)
//
// An item only ever waits on items dispensed before it, which are held by
// running workers, so the kernel makes progress whatever the number of
// resident CTAs.  No kernel boundary separates the router from the FFN or
// gate/up from down, and the dynamic queue has no wave quantisation.
//
// Every CTA first recomputes the previous layer's combine + residual +
// rmsnorm for all B tokens into shared memory (fp32 rows and the bf16 expert
// input T(x)); the routing worker writes h and x back.  Layer outputs that the
// next layer's prologue reads (h, y, ys, routing weights, shared-gate logits)
// are double-buffered by layer parity, so no CTA can overwrite a value another
// CTA of the same launch still has to read.
//
// Weight units are mma.sync.m16n8k16 tiles (bf16 in, fp32 accumulate): each
// of a worker's 4 warps streams one quarter of the reduction dimension of 16
// output rows with 16-byte L1-bypassing evict-first loads (k permuted within
// each 32-wide block so every load is 16 B and the B operand uses the same
// permutation), and the partial fragments are summed in a fixed warp order
// (deterministic).  The up epilogue fuses SiLU(gate) * up -> bf16.

namespace {

constexpr int kDlThreads = 512;  // 4 workers x 4 warps
constexpr int kDlWorkers = 4;
constexpr int kDlMaxB = 8;

struct DlArgs {
  int B, d, ff, sff, M, k, mode;
  int rows_main, n_rows;  // R*M router rows (+1: shared gate)
  int dp, dpb;            // shared-memory row strides: fp32 / bf16 elements
  float eps;
  int has_prev;
  const float* h_src;
  float* h_dst;
  float* x_out;
  const float* y_prev;
  const float* wts_prev;
  const float* ys_prev;
  const float* sgl_prev;
  unsigned long long* comb_stamp;
  const __nv_bfloat16* w_router;
  const __nv_bfloat16* w_sgate;
  float* logits;
  float* sgl_out;
  float bias;
  uint64_t mlo, mhi;
  int topup_U;
  uint64_t* mask_out;
  int32_t *sel, *counts, *offsets, *perm, *inv;
  float* wts_out;
  ef::RouteFast rf;
  volatile HostCtrl* hc;
  ef::GateIO io;
  const char* slab;
  int64_t stride;
  const volatile uint32_t* ready;
  const __nv_bfloat16* shared_w;
  __nv_bfloat16* act;
  __nv_bfloat16* act_s;
  float* y_out;
  float* ys_out;
  int max_active;
  ef::LayerSync* sync;
  unsigned long long* stats;
  unsigned long long* pub;  // tagged publish words {seq | value << 32} (null: none)
  int hold;                 // shared-expert units wait for the router ticket
  int parity;               // router-claim counter of this step
  int x_first;              // h / x written before the host publish
  int kinter;               // unit k blocks interleaved across the worker's warps
  int udepth;               // loads in flight per warp (dl_unit)
  unsigned long long* trace;  // EF_MEGA_TRACE: per work item {start, end} ns (null: off)
  // item ranges
  int i_shu, i_rup, i_shd, i_rdn, i_end;
  int su, ru, sd, rd;  // 16-row units: shared up, routed up (per entry), shared down, routed down
};

__device__ __forceinline__ void wbar(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}
struct WorkerBar {
  int id;
  __device__ void operator()() const { wbar(id); }
};

struct DlRoute {  // one worker's view of the layer's routing
  int32_t sel[128];
  float wts[128];
  int32_t perm[128];
  int4 ent[ef::kMaxActive];
  int n_active, ok;
};
struct DlSmem {
  DlRoute lr[kDlWorkers];
  float red[kDlWorkers][3 * 8 * 32];  // split-K partials (warps 1..3 of a worker)
  float rred[kDlWorkers][4][kDlMaxB]; // router row partials
  float invn[kDlMaxB];
  float bsum[kDlMaxB][kDlThreads / 32];
  int item[kDlWorkers];
  int4 ent[kDlWorkers];
  int last[kDlWorkers];
  int row[kDlWorkers];
  TopupSmem ts;
};

// One 16-row unit of an expert matrix for n <= 8 tokens (one 8-wide n-tile).
// UP: rows r0.. of W1 and W3 (W3 at rows_total rows behind W1), K = d, the B
// operand is T(x) from shared memory; epilogue act = bf16(silu(g) * u).
// Down: rows r0.. of W2, K = ff (or sff), B operand = act rows (L2), fp32 out.
template <bool UP, int U>
__device__ __noinline__ void dl_unit_u(const DlArgs& a, DlSmem& sm, const __nv_bfloat16* xb,
                                        const __nv_bfloat16* W, int rows_total, int K, int r0,
                                        int p0, int n, bool shared, uint64_t pol,
                                        const int32_t* perm) {
  const int lane = threadIdx.x & 31, wl = (threadIdx.x >> 5) & 3, wk = threadIdx.x >> 7;
  const int g = lane >> 2, tq = lane & 3;
  const int nkb = K / 32;
  const int kb0 = (nkb * wl) / 4 * 32, kb1 = (nkb * (wl + 1)) / 4 * 32;
  const __nv_bfloat16* A0 = W + (int64_t)(r0 + g) * K + 8 * tq;
  const __nv_bfloat16* A1 = A0 + (int64_t)8 * K;
  const int64_t offB = (int64_t)rows_total * K;
  const bool ok = g < n;
  const __nv_bfloat16* br;
  if (UP) {
    const int tok = !ok ? 0 : shared ? g : perm[p0 + g] / a.k;
    br = xb + tok * a.dpb + 8 * tq;
  } else {
    const int gg = ok ? g : 0;
    br = (shared ? a.act_s + (int64_t)gg * a.sff : a.act + (int64_t)(p0 + gg) * a.ff) + 8 * tq;
  }
  float c1[4] = {0.f, 0.f, 0.f, 0.f}, c3[4] = {0.f, 0.f, 0.f, 0.f};
  // U: 32-wide k blocks in flight per warp and iteration
  // the operands of one 32-wide k block: rows g / g+8 of W1 (and W3), token g's B column
  auto block = [&](int kk, uint4& a0, uint4& a1, uint4& b0, uint4& b1, uint4& bv) {
    a0 = ld_stream16_ef(A0 + kk, pol);
    a1 = ld_stream16_ef(A1 + kk, pol);
    if (UP) {
      b0 = ld_stream16_ef(A0 + offB + kk, pol);
      b1 = ld_stream16_ef(A1 + offB + kk, pol);
    }
    bv = make_uint4(0, 0, 0, 0);
    if (ok) bv = UP ? *reinterpret_cast<const uint4*>(br + kk) : __ldcg(reinterpret_cast<const uint4*>(br + kk));
  };
  auto mma = [&](const uint4& a0, const uint4& a1, const uint4& b0, const uint4& b1, const uint4& bv) {
    mma_bf16_16816(c1, a0.x, a1.x, a0.y, a1.y, bv.x, bv.y);
    mma_bf16_16816(c1, a0.z, a1.z, a0.w, a1.w, bv.z, bv.w);
    if (UP) {
      mma_bf16_16816(c3, b0.x, b1.x, b0.y, b1.y, bv.x, bv.y);
      mma_bf16_16816(c3, b0.z, b1.z, b0.w, b1.w, bv.z, bv.w);
    }
  };
  // k blocks of this warp: a contiguous quarter of K, or (kinter) every 4th
  // block, so the worker's 4 warps together read 4*U consecutive blocks of
  // each row per iteration (longer contiguous DRAM runs)
  const int kfirst = a.kinter ? 32 * wl : kb0, kend = a.kinter ? 32 * nkb : kb1;
  const int ustep = a.kinter ? 128 : 32;
  int kb = kfirst;
  // full groups of U blocks: every load of the group issued before the first mma
#pragma unroll 1
  for (; kb + (U - 1) * ustep < kend; kb += U * ustep) {
    uint4 w1[U][2], w3[U][2], bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) block(kb + u * ustep, w1[u][0], w1[u][1], w3[u][0], w3[u][1], bv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) mma(w1[u][0], w1[u][1], w3[u][0], w3[u][1], bv[u]);
  }
#pragma unroll 1
  for (; kb + ustep < kend; kb += 2 * ustep) {  // remainder: pairs of blocks in flight
    uint4 a0, a1, b0, b1, v0, c0, c1_, d0, d1, v1;
    block(kb, a0, a1, b0, b1, v0);
    block(kb + ustep, c0, c1_, d0, d1, v1);
    mma(a0, a1, b0, b1, v0);
    mma(c0, c1_, d0, d1, v1);
  }
  if (kb < kend) {  // last single block
    uint4 a0, a1, b0, b1, bv;
    block(kb, a0, a1, b0, b1, bv);
    mma(a0, a1, b0, b1, bv);
  }
  // split-K reduction in a fixed warp order: warps 1..3 park, warp 0 adds
  constexpr int NV = UP ? 8 : 4;
  float* red = sm.red[wk];
  if (wl > 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[((wl - 1) * NV + q) * 32 + lane] = c1[q];
      if (UP) red[((wl - 1) * NV + 4 + q) * 32 + lane] = c3[q];
    }
  }
  wbar(1 + wk);
  if (wl == 0) {
#pragma unroll
    for (int w = 1; w < 4; ++w)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        c1[q] += red[((w - 1) * NV + q) * 32 + lane];
        if (UP) c3[q] += red[((w - 1) * NV + 4 + q) * 32 + lane];
      }
    // c[q] = (row g + 8*(q>>1), token 2tq + (q&1))
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = 2 * tq + (q & 1);
      if (p >= n) continue;
      const int row = r0 + g + 8 * (q >> 1);
      if (UP) {
        const float gg = c1[q], uu = c3[q];
        const float sv = gg / (1.0f + expf(-gg)) * uu;
        if (shared)
          a.act_s[(int64_t)p * a.sff + row] = __float2bfloat16_rn(sv);
        else
          a.act[(int64_t)(p0 + p) * a.ff + row] = __float2bfloat16_rn(sv);
      } else {
        if (shared)
          a.ys_out[(int64_t)p * a.d + row] = c1[q];
        else
          a.y_out[(int64_t)perm[p0 + p] * a.d + row] = c1[q];  // slot order
      }
    }
    __threadfence();  // the unit's outputs before its completion count
  }
  wbar(1 + wk);
}

// a.udepth selects the 32-wide k blocks in flight per warp and iteration:
// 2 (default) U = 1 gate/up (4 x 16 B per lane), 2 down; 0: U = 2 / 3;
// 1: U = 4 / 6.  With ~600 workers streaming, fewer loads in flight per
// warp keep the same HBM throughput at a lower queueing latency, which
// shortens every dependent phase of the layer (B200, tok/s for depth
// 1 / 0 / 2: Qwen B=1 671 / 676 / 701, Qwen B=8 2204 / 2321 / 2313,
// DeepSeek B=1 552 / 569 / 565).
template <bool UP>
__device__ __forceinline__ void dl_unit(const DlArgs& a, DlSmem& sm, const __nv_bfloat16* xb,
                                        const __nv_bfloat16* W, int rows_total, int K, int r0,
                                        int p0, int n, bool shared, uint64_t pol,
                                        const int32_t* perm) {
  if (a.udepth == 1)
    dl_unit_u<UP, UP ? 4 : 6>(a, sm, xb, W, rows_total, K, r0, p0, n, shared, pol, perm);
  else if (a.udepth == 2)
    dl_unit_u<UP, UP ? 1 : 2>(a, sm, xb, W, rows_total, K, r0, p0, n, shared, pol, perm);
  else
    dl_unit_u<UP, UP ? 2 : 3>(a, sm, xb, W, rows_total, K, r0, p0, n, shared, pol, perm);
}

// One router row (layer row, pre-gate row or shared gate) for all B tokens:
// the 4 warps split the row, x = hs * invn from shared memory.
__device__ const __nv_bfloat16* dl_row_ptr(const DlArgs& a, int row) {
  return a.w_sgate && row == a.rows_main ? a.w_sgate : a.w_router + (int64_t)row * a.d;
}
// wsm: the row already in shared memory (prefetched), else streamed from HBM
__device__ __noinline__ void dl_router_row(const DlArgs& a, DlSmem& sm, const float* hs, int row,
                                           const __nv_bfloat16* wsm) {
  const int lane = threadIdx.x & 31, wl = (threadIdx.x >> 5) & 3, wk = threadIdx.x >> 7;
  const int tw = threadIdx.x & 127;
  const bool sg = a.w_sgate && row == a.rows_main;
  const __nv_bfloat16* wr = dl_row_ptr(a, row);
  const int span = a.d / 4, c00 = wl * span;
  float acc[kDlMaxB];
#pragma unroll
  for (int t = 0; t < kDlMaxB; ++t) acc[t] = 0.f;
  constexpr int UQ = 8;
  for (int c0 = lane * 8; c0 < span; c0 += UQ * 256) {
    uint4 wv[UQ];
#pragma unroll
    for (int u = 0; u < UQ; ++u)
      wv[u] = c0 + u * 256 >= span ? make_uint4(0, 0, 0, 0)
              : wsm ? *reinterpret_cast<const uint4*>(wsm + c00 + c0 + u * 256)
                    : ld_stream16(wr + c00 + c0 + u * 256);
#pragma unroll
    for (int u = 0; u < UQ; ++u) {
      const int c = c00 + c0 + u * 256;
      if (c0 + u * 256 >= span) break;
      float f[8];
      WTraits<__nv_bfloat16>::unpack(wv[u], f);
#pragma unroll
      for (int t = 0; t < kDlMaxB; ++t) {
        if (t >= a.B) break;
        const float sc = sm.invn[t];
        const float4 x0 = *reinterpret_cast<const float4*>(hs + t * a.dp + c);
        const float4 x1 = *reinterpret_cast<const float4*>(hs + t * a.dp + c + 4);
        float p = 0.f;
        p = fmaf(f[0], x0.x * sc, p);
        p = fmaf(f[1], x0.y * sc, p);
        p = fmaf(f[2], x0.z * sc, p);
        p = fmaf(f[3], x0.w * sc, p);
        p = fmaf(f[4], x1.x * sc, p);
        p = fmaf(f[5], x1.y * sc, p);
        p = fmaf(f[6], x1.z * sc, p);
        p = fmaf(f[7], x1.w * sc, p);
        acc[t] += p;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < kDlMaxB; ++t) {
    if (t >= a.B) break;
    const float s = warp_sum(acc[t]);
    if (lane == 0) sm.rred[wk][wl][t] = s;
  }
  wbar(1 + wk);
  if (tw < a.B) {
    const int t = tw;
    const float v = (sm.rred[wk][0][t] + sm.rred[wk][1][t]) + (sm.rred[wk][2][t] + sm.rred[wk][3][t]);
    if (sg) {
      a.sgl_out[t] = v;
    } else {
      const int r = row / a.M, m = row % a.M;
      a.logits[((int64_t)r * a.B + t) * a.M + m] = v;
    }
    __threadfence();
  }
  wbar(1 + wk);  // the row's logits are fenced before the ticket
}

// Top-k of every token (warp wl takes tokens wl, wl+4) into sel / wts
// (shared or global), then warp 0 sorts the N = B*k <= 128 (token, rank)
// slots by expert (stable) and resolves each active expert's slot from the
// launch's slot-table row.  Outputs: perm (and inv / counts / offsets when
// non-null), the decision entries {slot, first row, rows, fill seq} in
// ascending expert order, their count, and whether every expert resolved.
// All four warps must call it; deterministic, so every worker that routes
// gets the same answer as the routing worker.
__device__ void dl_sort_resolve(const DlArgs& a, const int32_t* sel_sh, int32_t* perm, int32_t* inv,
                                int32_t* counts, int32_t* offsets, int4* ent, int* n_active,
                                int* ok_out) {
  const int tw = threadIdx.x & 127, lane = tw & 31, wl = tw >> 5;
  const int M = a.M, N = a.B * a.k;
  if (wl != 0) return;
  int es[4], pos[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = lane + 32 * i;
    es[i] = f < N ? sel_sh[f] : 0x7fffffff;
    pos[i] = 0;
  }
  for (int j = 0; j < N; ++j) {
    const int ej = sel_sh[j];
#pragma unroll
    for (int i = 0; i < 4; ++i) pos[i] += (ej < es[i]) || (ej == es[i] && j < lane + 32 * i);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = lane + 32 * i;
    if (f < N) {
      if (inv) inv[f] = pos[i];
      perm[pos[i]] = f;
    }
  }
  int cnt[4], off[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) cnt[i] = off[i] = 0;
  for (int j = 0; j < N; ++j) {
    const int ej = sel_sh[j];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      cnt[i] += ej == lane + 32 * i;
      off[i] += ej < lane + 32 * i;
    }
  }
  if (counts) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = lane + 32 * i;
      if (x < M) {
        counts[x] = cnt[i];
        offsets[x] = off[i];
      }
    }
    if (lane == 0) offsets[M] = N;
  }
  int base = 0;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int x = lane + 32 * i;
    const bool act = x < M && cnt[i] > 0;
    const int2 t = act ? a.rf.tab[x] : make_int2(-1, 0);
    ok = ok && !__any_sync(0xffffffffu, act && t.x < 0);
    const unsigned m = __ballot_sync(0xffffffffu, act);
    const int p = base + __popc(m & ((1u << lane) - 1u));
    if (act && p < ef::kMaxActive) ent[p] = make_int4(t.x, off[i], cnt[i], t.y);
    base += __popc(m);
  }
  ok = ok && base <= ef::kMaxActive;
  if (lane == 0) {
    *n_active = base;
    *ok_out = ok ? 1 : 0;
  }
  __syncwarp();
}

// Publish the layer's mask, selection and scored logits rows to the host as
// tagged words {seq | value << 32} (single-copy-atomic 8-byte stores): the
// host accepts the block once every word carries this launch's seq, so no
// system-scope fence is needed.  One warp.
__device__ void dl_publish(const DlArgs& a, uint64_t mlo, uint64_t mhi) {
  const int lane = threadIdx.x & 31;
  const unsigned long long tag = a.rf.seq;
  volatile unsigned long long* p = a.pub;
  const int N = a.B * a.k, R = a.rows_main * a.B;
  if (lane < 4) {
    const uint64_t m = lane < 2 ? mlo : mhi;
    const uint32_t v = (lane & 1) ? (uint32_t)(m >> 32) : (uint32_t)m;
    p[lane] = tag | ((unsigned long long)v << 32);
  }
  for (int f = lane; f < N; f += 32)
    p[4 + f] = tag | ((unsigned long long)(uint32_t)__ldcg(a.sel + f) << 32);
  for (int i = lane; i < R; i += 32)
    p[4 + N + i] = tag | ((unsigned long long)__float_as_uint(__ldcg(a.logits + i)) << 32);
  if (a.stats && lane == 0) a.stats[9] = gtimer();
}

// The route, by the worker that finished the last router row: this layer's
// h and x, the global routing outputs (the next layer's combine and the host
// read them), device-side slot resolution, the host publish, and on an
// unresolved layer the wait for the host's decision block.
__device__ __noinline__ void dl_route(const DlArgs& a, DlSmem& sm, const float* hs) {
  const int tw = threadIdx.x & 127, lane = tw & 31, wl = tw >> 5, wk = threadIdx.x >> 7;
  const int B = a.B, M = a.M, k = a.k;
  unsigned long long* st = a.stats;
  if (st && tw == 0) st[6] = gtimer();
  uint64_t mlo = a.mlo, mhi = a.mhi;
  if (a.topup_U > 0) topup_mask(sm.ts, a.logits, B, M, k, a.topup_U, mlo, mhi, tw, 128, WorkerBar{1 + wk});
  DlRoute& lr = sm.lr[wk];
  for (int t = wl; t < B; t += 4)
    topk_token(a.logits + (int64_t)t * M, M, k, a.mode, a.bias, mlo, mhi, a.sel + t * k,
               a.wts_out + t * k, lr.sel + t * k);
  wbar(1 + wk);
  dl_sort_resolve(a, lr.sel, a.perm, a.inv, a.counts, a.offsets, a.rf.dc->ent, &lr.n_active, &lr.ok);
  const unsigned seq = a.rf.seq;
  if (wl == 0) {
    const bool ok = lr.ok != 0;
    if (lane == 0) {
      if (ok) a.rf.dc->n_active = lr.n_active;
      if (!ok && !a.hc) a.rf.dc->n_active = 0;  // standalone: nothing the host could resolve
      if (a.mask_out) {
        a.mask_out[0] = mlo;
        a.mask_out[1] = mhi;
      }
      __threadfence();
      *a.rf.fast_word = ok ? seq : 0u;
      if (st) st[11] = ok ? 1ull : 0ull;
      if (ok || !a.hc) {  // workers waiting on the global decision may start
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&a.sync->route), "r"(seq) : "memory");
        if (st) st[13] = gtimer();
      }
    }
    // publish first unless the host records x_l (it copies x once it has the selection)
    if (a.pub && !a.x_first) dl_publish(a, mlo, mhi);
  }
  wbar(1 + wk);
  // this layer's h and x (every CTA computed the same rows)
  for (int i = tw * 4; i < B * a.d; i += 128 * 4) {
    const int t = i / a.d, c = i % a.d;
    const float4 v = *reinterpret_cast<const float4*>(hs + t * a.dp + c);
    const float sc = sm.invn[t];
    *reinterpret_cast<float4*>(a.h_dst + i) = v;
    *reinterpret_cast<float4*>(a.x_out + i) = make_float4(v.x * sc, v.y * sc, v.z * sc, v.w * sc);
  }
  if (a.x_first) __threadfence();
  if (a.comb_stamp && tw == 0) *a.comb_stamp = gtimer();
  if (a.x_first) wbar(1 + wk);
  if (wl == 0) {
    if (a.pub && a.x_first) dl_publish(a, mlo, mhi);
    // on an unresolved layer: wait for the host's decision block (gate_duty
    // raises sync->route = seq once it is copied); io.host_done is null, so
    // gate_duty does not publish again
    if (a.hc) gate_duty(a.hc, a.rf.dc, st, reinterpret_cast<volatile unsigned*>(&a.sync->route), seq, a.io);
  }
}

// A worker's own routing of the layer: after the router ticket, from the
// logits, exactly as dl_route computes it (bit-identical).  lr.ok = 0 when
// the bias mask needs a top-up or an expert is not resident: the worker then
// takes the global decision (dl_route_global) before its routed items.
__device__ __noinline__ void dl_route_local(const DlArgs& a, DlSmem& sm) {
  const int tw = threadIdx.x & 127, wl = tw >> 5, wk = threadIdx.x >> 7;
  DlRoute& lr = sm.lr[wk];
  if (tw == 0) {
    const long long c0 = clock64();
    while (ld_acquire_gpu(reinterpret_cast<const volatile unsigned*>(&a.sync->ticket)) <
           (unsigned)a.n_rows) {
      __nanosleep(32);
      if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
    }
    lr.ok = 0;
  }
  wbar(1 + wk);
  if (a.topup_U == 0) {
    for (int t = wl; t < a.B; t += 4)
      topk_token(a.logits + (int64_t)t * a.M, a.M, a.k, a.mode, a.bias, a.mlo, a.mhi,
                 lr.sel + t * a.k, lr.wts + t * a.k, nullptr);
    wbar(1 + wk);
    dl_sort_resolve(a, lr.sel, lr.perm, nullptr, nullptr, nullptr, lr.ent, &lr.n_active, &lr.ok);
  }
  wbar(1 + wk);
}
// The global decision (the routing worker's, or the host's on an unresolved
// layer): wait for it, then take its entries and permutation.
__device__ __noinline__ void dl_route_global(const DlArgs& a, DlSmem& sm) {
  const int tw = threadIdx.x & 127, wk = threadIdx.x >> 7;
  DlRoute& lr = sm.lr[wk];
  const unsigned seq = a.rf.seq;
  if (tw == 0) {
    const long long c0 = clock64();
    while (ld_acquire_gpu(&a.sync->route) != seq) {
      __nanosleep(32);
      if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
    }
  }
  wbar(1 + wk);
  const int n = min(__ldcg(&a.rf.dc->n_active), a.max_active);
  for (int i = tw; i < n; i += 128) lr.ent[i] = __ldcg(&a.rf.dc->ent[i]);
  for (int i = tw; i < a.B * a.k; i += 128) lr.perm[i] = __ldcg(a.perm + i);
  if (tw == 0) {
    lr.n_active = n;
    lr.ok = 1;
  }
  wbar(1 + wk);
}

// Prologue of every CTA: v = h + sum_r w_r y_r (rank order) + g * ys of the
// previous layer (just h at layer 0) into shared memory, its rmsnorm scale,
// and the expert input T(x) = bf16(v * invn) — the same fp32 product the
// router uses.
__device__ __noinline__ void dl_prologue(const DlArgs& a, DlSmem& sm, float* hs, __nv_bfloat16* xb) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // every token's loads in flight together (one L2 round trip per 2048 columns)
  float ss[kDlMaxB];
#pragma unroll
  for (int t = 0; t < kDlMaxB; ++t) {
    ss[t] = 0.f;
    if (t >= a.B) continue;
    float g = 1.f, wr[16];
    if (a.has_prev) {
      g = a.sgl_prev ? 1.0f / (1.0f + expf(-__ldcg(a.sgl_prev + t))) : 1.f;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < a.k) wr[r] = __ldcg(a.wts_prev + t * a.k + r);
    }
    for (int i = tid * 4; i < a.d; i += kDlThreads * 4) {
      const float4 hv = __ldcg(reinterpret_cast<const float4*>(a.h_src + (int64_t)t * a.d + i));
      float4 v = hv;
      if (a.has_prev) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (r >= a.k) break;
          const float4 yv =
              __ldcg(reinterpret_cast<const float4*>(a.y_prev + ((int64_t)t * a.k + r) * a.d + i));
          acc.x = fmaf(wr[r], yv.x, acc.x);
          acc.y = fmaf(wr[r], yv.y, acc.y);
          acc.z = fmaf(wr[r], yv.z, acc.z);
          acc.w = fmaf(wr[r], yv.w, acc.w);
        }
        if (a.ys_prev) {
          const float4 sv = __ldcg(reinterpret_cast<const float4*>(a.ys_prev + (int64_t)t * a.d + i));
          acc.x = fmaf(g, sv.x, acc.x);
          acc.y = fmaf(g, sv.y, acc.y);
          acc.z = fmaf(g, sv.z, acc.z);
          acc.w = fmaf(g, sv.w, acc.w);
        }
        v = make_float4(hv.x + acc.x, hv.y + acc.y, hv.z + acc.z, hv.w + acc.w);
      }
      *reinterpret_cast<float4*>(hs + t * a.dp + i) = v;
      ss[t] += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
  }
  // per-token sums of squares: warp shuffles, then a fixed order over the 16 warps
#pragma unroll
  for (int t = 0; t < kDlMaxB; ++t) {
    if (t >= a.B) break;
    const float v = warp_sum(ss[t]);
    if (lane == 0) sm.bsum[t][wid] = v;
  }
  __syncthreads();
  if (tid < a.B) {
    float v = 0.f;
    for (int w = 0; w < kDlThreads / 32; ++w) v += sm.bsum[tid][w];
    sm.invn[tid] = 1.0f / sqrtf(v / (float)a.d + a.eps);
  }
  __syncthreads();
  for (int i = tid * 4; i < a.B * a.d; i += kDlThreads * 4) {
    const int t = i / a.d, c = i % a.d;
    const float4 v = *reinterpret_cast<const float4*>(hs + t * a.dp + c);
    const float sc = sm.invn[t];
    uint2 o;
    o.x = pack_bf16x2(v.x * sc, v.y * sc);
    o.y = pack_bf16x2(v.z * sc, v.w * sc);
    *reinterpret_cast<uint2*>(xb + t * a.dpb + c) = o;
  }
  __syncthreads();
}

// Claim the next router row of this launch.  The claim counters alternate
// by step parity and each is zeroed one step before its use (see
// launch_zero_sync), so a claim may be made before the PDL wait.
__device__ __forceinline__ int dl_claim_row(const DlArgs& a) {
  return atomicAdd(&a.sync->rq[a.parity], 1);
}

__global__ void __launch_bounds__(kDlThreads, 1) decode_layer_kernel(const __grid_constant__ DlArgs a) {
  extern __shared__ __align__(16) unsigned char dl_smem_raw[];
  __shared__ DlSmem sm;
  float* hs = reinterpret_cast<float*>(dl_smem_raw);
  __nv_bfloat16* xb = reinterpret_cast<__nv_bfloat16*>(hs + a.B * a.dp);
  const int tid = threadIdx.x, tw = tid & 127, wk = tid >> 7;
  // every worker claims a router row and prefetches the row's (constant)
  // weights into its shared-memory buffer while the previous layer drains
  __nv_bfloat16* rw = reinterpret_cast<__nv_bfloat16*>(xb + a.B * a.dpb) + wk * a.d;
  if (tw == 0) sm.row[wk] = dl_claim_row(a);
  wbar(1 + wk);
  if (sm.row[wk] < a.n_rows) {
    const __nv_bfloat16* wr = dl_row_ptr(a, sm.row[wk]);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(rw);
    for (int c = tw; c < a.d / 8; c += 128)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * c), "l"(wr + 8 * c)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  pdl_wait();
  pdl_trigger();
  unsigned long long* st = a.stats;
  if (st && blockIdx.x == 0 && tid == 0) st[7] = gtimer();

  dl_prologue(a, sm, hs, xb);
  if (st && blockIdx.x == 0 && tid == 0) st[12] = gtimer();

  // ---- router rows; the worker that finishes the last one routes
  {
    int row = sm.row[wk];
    bool first = true;
    while (row < a.n_rows) {
      if (first) asm volatile("cp.async.wait_all;" ::: "memory");
      wbar(1 + wk);
      if (a.trace && tw == 0) a.trace[2 * row] = gtimer();
      dl_router_row(a, sm, hs, row, first ? rw : nullptr);
      if (a.trace && tw == 0) a.trace[2 * row + 1] = gtimer();
      first = false;
      if (tw == 0) {
        const int done = atomicAdd(&a.sync->ticket, 1);
        sm.last[wk] = done == a.n_rows - 1;
        if (done == a.n_rows - 1) __threadfence();
        // more rows than workers: keep claiming (the common case claims once)
        sm.row[wk] = a.n_rows > (int)gridDim.x * kDlWorkers ? dl_claim_row(a) : a.n_rows;
      }
      wbar(1 + wk);
      if (sm.last[wk]) dl_route(a, sm, hs);
      row = sm.row[wk];
      wbar(1 + wk);
    }
  }

  // ---- FFN work items
  const uint64_t pol = l2_evict_first_policy();
  bool routed = false;  // this worker has routed the layer itself (sm.lr[wk])
  DlRoute& lr = sm.lr[wk];
  int prev_it = -1;
  for (;;) {
    if (tw == 0) {
      if (a.trace && prev_it >= 0) a.trace[2 * (a.n_rows + prev_it) + 1] = gtimer();
      sm.item[wk] = atomicAdd(&a.sync->q, 1);
    }
    wbar(1 + wk);
    const int it = sm.item[wk];
    wbar(1 + wk);  // item slot read by every thread before it can be rewritten
    if (it >= a.i_end) break;
    prev_it = it;
    if (a.trace && tw == 0) a.trace[2 * (a.n_rows + it)] = gtimer();
    if (it < a.i_rup) {  // ---- shared gate/up unit (no routing dependency)
      const int u = it - a.i_shu;
      if (a.hold && !routed) {  // route first, so the routing runs on a quiet memory system
        dl_route_local(a, sm);
        routed = true;
      }
      if (st && u == 0 && tw == 0) atomicMin(&st[3], gtimer());  // the FFN window starts here
      dl_unit<true>(a, sm, xb, a.shared_w, a.sff, a.d, u * 16, 0, a.B, true, pol, nullptr);
      if (tw == 0) {
        atomicAdd(&a.sync->sh_up, 1);
        if (st) atomicMax(&st[15], gtimer());
      }
      continue;
    }
    if (it < a.i_shd || it >= a.i_rdn) {  // ---- routed unit (up or down)
      const bool up = it < a.i_shd;
      const int r = up ? it - a.i_rup : it - a.i_rdn;
      const int per = up ? a.ru : a.rd;
      const int ei = r / per, sub = r % per;
      if (!routed) {
        dl_route_local(a, sm);
        routed = true;
      }
      if (!lr.ok) dl_route_global(a, sm);
      if (ei >= lr.n_active) continue;
      const int4 e = lr.ent[ei];
      if (tw == 0) {
        if (up) {
          const bool first = sub == 0;
          if (st && first) atomicMin(&st[10], gtimer());
          if (a.ready && a.ready[e.x] < (unsigned)e.w) {
            const unsigned long long t0 = gtimer();
            const long long c0 = clock64();
            while (a.ready[e.x] < (unsigned)e.w) {
              __nanosleep(128);
              if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
            }
            const unsigned long long t1 = gtimer();
            if (st && t1 > t0) atomicMax(&st[2], t1 - t0);
          }
          if (st && first) atomicMin(&st[3], gtimer());
        } else {  // down: every gate/up unit of this entry has finished
          const long long c0 = clock64();
          while (ld_acquire_gpu(reinterpret_cast<const volatile unsigned*>(&a.sync->up[ei])) <
                 (unsigned)a.ru) {
            __nanosleep(32);
            if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
          }
        }
      }
      wbar(1 + wk);
      const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(a.slab + (int64_t)e.x * a.stride);
      if (up) {
        dl_unit<true>(a, sm, xb, W, a.ff, a.d, sub * 16, e.y, e.z, false, pol, lr.perm);
        if (tw == 0) {
          atomicAdd(&a.sync->up[ei], 1);
          if (st) atomicMax(&st[14], gtimer());
        }
      } else {
        dl_unit<false>(a, sm, xb, W + 2LL * a.ff * a.d, a.d, a.ff, sub * 16, e.y, e.z, false, pol,
                       lr.perm);
        if (st && tw == 0) atomicMax(&st[4], gtimer());
      }
      continue;
    }
    // ---- shared down unit
    const int u = it - a.i_shd;
    if (tw == 0) {
      const long long c0 = clock64();
      while (ld_acquire_gpu(reinterpret_cast<const volatile unsigned*>(&a.sync->sh_up)) <
             (unsigned)a.su) {
        __nanosleep(32);
        if (clock64() - c0 > kSpinTimeoutCycles) asm volatile("trap;");
      }
    }
    wbar(1 + wk);
    dl_unit<false>(a, sm, xb, a.shared_w + 2LL * a.sff * a.d, a.d, a.sff, u * 16, 0, a.B, true, pol,
                   nullptr);
    if (st && tw == 0) atomicMax(&st[4], gtimer());
  }
}

// h_dst = h_src + sum_r w_r y_r (rank order, y in slot order) + g * ys: the
// last layer's combine (no next rmsnorm); the same arithmetic as the prologue.
__global__ void final_combine_kernel(const float* __restrict__ h_src, float* __restrict__ h_dst,
                                     const float* __restrict__ y, const float* __restrict__ wts,
                                     const float* __restrict__ ys, const float* __restrict__ sgl,
                                     int d, int k) {
  pdl_wait();
  const int t = blockIdx.x;
  const float g = sgl ? 1.0f / (1.0f + expf(-sgl[t])) : 1.f;
  for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
    const float4 hv = *reinterpret_cast<const float4*>(h_src + (int64_t)t * d + i);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < k; ++r) {
      const float w = wts[t * k + r];
      const float4 yv = *reinterpret_cast<const float4*>(y + ((int64_t)t * k + r) * d + i);
      acc.x = fmaf(w, yv.x, acc.x);
      acc.y = fmaf(w, yv.y, acc.y);
      acc.z = fmaf(w, yv.z, acc.z);
      acc.w = fmaf(w, yv.w, acc.w);
    }
    if (ys) {
      const float4 sv = *reinterpret_cast<const float4*>(ys + (int64_t)t * d + i);
      acc.x = fmaf(g, sv.x, acc.x);
      acc.y = fmaf(g, sv.y, acc.y);
      acc.z = fmaf(g, sv.z, acc.z);
      acc.w = fmaf(g, sv.w, acc.w);
    }
    *reinterpret_cast<float4*>(h_dst + (int64_t)t * d + i) =
        make_float4(hv.x + acc.x, hv.y + acc.y, hv.z + acc.z, hv.w + acc.w);
  }
}

// At the start of a step: zero every LayerSync field except the router-claim
// counter of this step's parity (zeroed one step earlier: a layer kernel
// claims before its PDL wait, when this kernel's writes need not be visible
// yet); the other parity's counter is zeroed for the next step.
__global__ void zero_sync_kernel(int* p, int n, int parity) {
  constexpr int W = (int)(sizeof(ef::LayerSync) / 4);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (i % W != parity) p[i] = 0;
}

// fp32 rows, bf16 expert input, and one router-row prefetch buffer per worker
size_t dl_dyn_smem(int B, int d) {
  return (size_t)B * (d + 4) * 4 + (size_t)B * (d + 32) * 2 + (size_t)kDlWorkers * d * 2;
}
constexpr size_t kDlDynSmemMax = 176 * 1024;

}  // namespace

namespace ef {
bool decode_layer_supported(int dtype, int d, int ff, int sff, int M, int k, int B) {
  const char* ev = getenv("EF_MEGA");  // read per step: tests switch it per engine
  const int env = ev ? atoi(ev) : 1;
  if (env == 0 || dtype != EF_BF16) return false;
  // measured on B200: the persistent layer wins where a shared expert streams
  // while the router and route run (Qwen / DeepSeek shapes, +8-10 %); without
  // one (Mixtral) the classic router / gate-up / down pipeline is faster
  // (220 vs 205 tok/s), so EF_MEGA=2 forces it there
  if (sff == 0 && env != 2) return false;
  if (B < 1 || B > kDlMaxB || M > 128 || k > 16 || B * k > 128) return false;
  if (d % 256 || ff % 32 || sff % 32) return false;
  return dl_dyn_smem(B, d) <= kDlDynSmemMax;
}

int launch_decode_layer(cudaStream_t st, const DecodeLayerIn& in) {
  EF_CHECK_ARG(decode_layer_supported(EF_BF16, in.d, in.ff, in.sff, in.M, in.k, in.B),
               "shape not supported by the persistent decode layer");
  EF_CHECK_ARG(in.max_active >= 1 && in.max_active <= kMaxActive, "bad max_active");
  static int grid = 0;
  const size_t smem = dl_dyn_smem(in.B, in.d);
  if (!grid) {
    EF_CUDA_RET(cudaFuncSetAttribute(decode_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kDlDynSmemMax));
    int dev = 0, sms = 0, per = 0;
    EF_CUDA_RET(cudaGetDevice(&dev));
    EF_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    EF_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_layer_kernel, kDlThreads,
                                                              kDlDynSmemMax));
    grid = sms * std::max(per, 1);
  }
  DlArgs a{};
  a.B = in.B;
  a.d = in.d;
  a.ff = in.ff;
  a.sff = in.sff;
  a.M = in.M;
  a.k = in.k;
  a.mode = in.mode;
  a.rows_main = in.R * in.M;
  a.n_rows = a.rows_main + (in.sgate ? 1 : 0);
  a.dp = in.d + 4;
  a.dpb = in.d + 32;  // bf16 rows 64 B apart mod 128: conflict-free 16-B loads
  a.eps = in.eps;
  a.has_prev = in.has_prev ? 1 : 0;
  a.h_src = in.h_src;
  a.h_dst = in.h_dst;
  a.x_out = in.x_out;
  a.y_prev = in.y_prev;
  a.wts_prev = in.wts_prev;
  a.ys_prev = in.ys_prev;
  a.sgl_prev = in.sgl_prev;
  a.comb_stamp = in.comb_stamp;
  a.w_router = reinterpret_cast<const __nv_bfloat16*>(in.w_router);
  a.w_sgate = in.sgate ? reinterpret_cast<const __nv_bfloat16*>(in.w_sgate) : nullptr;
  a.logits = in.logits;
  a.sgl_out = in.sgl_out;
  a.bias = in.bias;
  a.mlo = in.mlo;
  a.mhi = in.mhi;
  a.topup_U = in.topup_U;
  a.mask_out = in.mask_out;
  a.sel = in.sel;
  a.counts = in.counts;
  a.offsets = in.offsets;
  a.perm = in.perm;
  a.inv = in.inv;
  a.wts_out = in.wts_out;
  a.rf = in.rf;
  a.hc = reinterpret_cast<volatile HostCtrl*>(in.hc_dev);
  a.io = in.io;
  a.slab = in.slab;
  a.stride = in.stride;
  a.ready = in.ready;
  a.shared_w = reinterpret_cast<const __nv_bfloat16*>(in.shared_w);
  a.act = reinterpret_cast<__nv_bfloat16*>(in.act);
  a.act_s = reinterpret_cast<__nv_bfloat16*>(in.act_s);
  a.y_out = in.y_out;
  a.ys_out = in.ys_out;
  a.max_active = in.max_active;
  a.sync = in.sync;
  a.stats = in.stats;
  a.pub = reinterpret_cast<unsigned long long*>(in.pub);
  static const int hold = [] {
    const char* v = getenv("EF_MEGA_HOLD");
    return v ? atoi(v) : 0;
  }();
  a.hold = hold;
  a.parity = in.parity;
  a.x_first = in.x_before_publish ? 1 : 0;
  static const int kinter = [] {
    const char* v = getenv("EF_MEGA_KINTER");
    return v ? atoi(v) : 0;
  }();
  a.kinter = kinter;
  static const int udepth = [] {
    const char* v = getenv("EF_MEGA_UDEPTH");
    return v ? atoi(v) : 2;
  }();
  a.udepth = udepth;
  a.trace = reinterpret_cast<unsigned long long*>(in.trace);
  a.su = in.sff / 16;
  a.ru = in.ff / 16;
  a.sd = in.sff ? in.d / 16 : 0;
  a.rd = in.d / 16;
  a.i_shu = 0;  // router rows are claimed separately (dl_claim_row)
  a.i_rup = a.i_shu + a.su;
  a.i_shd = a.i_rup + in.max_active * a.ru;
  a.i_rdn = a.i_shd + a.sd;
  a.i_end = a.i_rdn + in.max_active * a.rd;
  EF_CUDA_RET(launch_k(decode_layer_kernel, dim3(grid), dim3(kDlThreads), smem, st, a));
  return EF_OK;
}

int launch_final_combine(cudaStream_t st, const float* h_src, float* h_dst, const float* y,
                         const float* wts, const float* ys, const float* sgl, int B, int d, int k) {
  EF_CUDA_RET(launch_k(final_combine_kernel, dim3(B), dim3(256), 0, st, h_src, h_dst, y, wts, ys,
                       sgl, d, k));
  return EF_OK;
}

int launch_zero_sync(cudaStream_t st, LayerSync* sync, int L, int parity) {
  const int n = (int)(sizeof(LayerSync) / 4) * L;
  zero_sync_kernel<<<1, 1024, 0, st>>>(reinterpret_cast<int*>(sync), n, parity);
  EF_CUDA_RET(cudaGetLastError());
  return EF_OK;
}

int preload_decode_layer() {
  int n = 0;
  preload(decode_layer_kernel, n);
  preload(final_combine_kernel, n);
  preload(zero_sync_kernel, n);
  cudaFuncSetAttribute(decode_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kDlDynSmemMax);
  return n;
}
}  // namespace ef
