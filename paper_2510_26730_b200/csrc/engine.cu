// engine.cu — the MoE decode engine: HBM expert-cache slab with a physical
// slot table, pinned host store, dedicated copy stream with events, and the
// scheduler Stepper (simcore.h) driving it.
//
// Decision parity: the Stepper runs the reference's per-layer loop
// (engine.py:566-659) on a LOGICAL integer-ns clock, so the hit / miss /
// admit / evict trace, predictions and step sizes are exactly the oracle's
// for the routing the GPU produced.  Data movement is PHYSICAL: every
// logical transfer start issues one cudaMemcpyAsync of the expert blob into a
// free HBM slot on the copy stream; the expert FFN of a layer waits (stream
// wait on the copy's event) only for the slots it reads, so swap-ins overlap
// compute and the measured wait is the physical expert stall.
//
// Slot safety: a slot freed by an eviction is reused by a later copy only
// after the last kernel that read it (per-layer reader event), and slots read
// by the current layer stay pinned until that layer's kernels are enqueued.
// The slab therefore holds capacity + staging slots.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/expertflow.h"
#include "capi_util.h"
#include "simcore.h"

namespace ef {
int expert_ffn_ptrs(cudaStream_t st, const float* x, const int32_t* perm, int k, bool identity,
                    const char* const* wbase, const int32_t* p0, const int32_t* nrows,
                    int n_active, int d, int ff, int dtype, void* act, float* y);
}

using namespace ef;

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) throw CudaErr(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)
#define CKS(expr)                                                          \
  do {                                                                     \
    int _s = (expr);                                                       \
    if (_s != EF_OK) throw CudaErr(std::string(#expr) + ": " + g_last_error); \
  } while (0)

// fp64 softmax of fp32 logits: glibc exp, sequential sum (
// oracle/numerics.py softmax64) and the token-weighted batch gate
// (workload.py:215-223 with one group per token).
static void batch_gate(const float* logits, int B, int M, double* out) {
  std::vector<double> mixed(M, 0.0), ex(M);
  const double w = 1.0 / (double)B;
  for (int t = 0; t < B; ++t) {
    const float* lg = logits + (int64_t)t * M;
    double mx = (double)lg[0];
    for (int e = 1; e < M; ++e) mx = std::max(mx, (double)lg[e]);
    double s = 0.0;
    for (int e = 0; e < M; ++e) {
      ex[e] = std::exp((double)lg[e] - mx);
      s += ex[e];
    }
    for (int e = 0; e < M; ++e) {
      double p = ex[e] / s;
      double wp = w * p;
      mixed[e] = mixed[e] + wp;
    }
  }
  double s = 0.0;
  for (int e = 0; e < M; ++e) s += mixed[e];
  for (int e = 0; e < M; ++e) out[e] = mixed[e] / s;
}

struct ef_engine {
  ef_engine_cfg cfg{};
  SimConfig simcfg;
  std::unique_ptr<CallbackHooks> hooks;
  std::unique_ptr<Stepper> st;

  int64_t esz = 2, stride = 0, sstride = 0;  // element size, expert / shared slot bytes
  int P = 0;                                  // physical slots
  int Rmax = 1;
  // device
  char* slab = nullptr;
  void* router_w = nullptr;  // [L][M][d]
  char* shared_w = nullptr;  // [L] x sstride
  void* sgate_w = nullptr;   // [L][d]
  float *x_d = nullptr, *logits_d = nullptr, *sgl_d = nullptr, *wts_d = nullptr, *y_d = nullptr,
        *ys_d = nullptr;
  int32_t *sel_d = nullptr, *counts_d = nullptr, *offsets_d = nullptr, *perm_d = nullptr,
          *inv_d = nullptr;
  void *act_d = nullptr, *acts_d = nullptr;
  // host pinned
  float* logits_h = nullptr;
  int32_t* sel_h = nullptr;
  std::vector<char*> store;  // per layer: M * stride bytes
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> fill_ev;     // per physical slot: last copy into it
  std::vector<int> fill_recorded;
  std::vector<cudaEvent_t> reader_ring;  // per-layer "kernels done" events
  std::vector<int> reader_of;            // per slot: ring index of last reader (-1)
  int ring_next = 0;
  std::vector<cudaEvent_t> stall_a, stall_b;  // per layer (timing)
  // slot table
  std::vector<int32_t> phys_of;  // [L*M] -> slot or -1
  std::deque<int> free_slots;
  std::vector<char> pinned;
  std::vector<int> pinned_list, deferred_free;
  int inflight_slot = -1;
  std::vector<int> layer_use;  // [M] -> slot used by the current layer (-1)
  struct RoutingRec {
    std::vector<float> logits;
    std::vector<int32_t> sel;
    int R, B;
    uint64_t mlo, mhi;
  };
  std::vector<RoutingRec> rlog;
  // stats
  int64_t steps = 0, copies = 0, copy_bytes = 0, launches = 0, preload_copies = 0,
          d2h_bytes = 0;
  double stall_ms = 0, host_ms = 0, ffn_ms = 0, step_ms = 0;

  struct Mirror : Observer {
    ef_engine* e;
    void on_transfer_start(uint64_t key, int prio) override { e->issue_copy(key, false); }
    void on_admit(uint64_t key) override {
      if (e->inflight_slot < 0) throw RuntimeErr("admit without a landed transfer");
      e->phys_of[e->idx(key)] = e->inflight_slot;
      e->inflight_slot = -1;
    }
    void on_evict(uint64_t key) override {
      int s = e->phys_of[e->idx(key)];
      e->phys_of[e->idx(key)] = -1;
      if (s < 0) return;
      if (e->pinned[s])
        e->deferred_free.push_back(s);
      else
        e->free_slots.push_back(s);
    }
    void on_preload(uint64_t key) override { e->issue_copy(key, true); }
    void on_group_run(int layer, const std::vector<uint64_t>& demand) override {
      for (uint64_t k : demand) {
        int s = e->phys_of[e->idx(k)];
        if (s < 0) throw RuntimeErr("group runs with a non-resident expert");
        if (!e->pinned[s]) {
          e->pinned[s] = 1;
          e->pinned_list.push_back(s);
        }
        e->layer_use[eid_expert(k)] = s;
      }
    }
  } mirror;

  int64_t idx(uint64_t key) const {
    return (int64_t)eid_layer(key) * cfg.M + eid_expert(key);
  }

  void issue_copy(uint64_t key, bool preload) {
    if (free_slots.empty())
      throw RuntimeErr("no free physical expert slot (raise staging_slots)");
    int s = free_slots.front();
    free_slots.pop_front();
    if (reader_of[s] >= 0) CK(cudaStreamWaitEvent(copy_stream, reader_ring[reader_of[s]], 0));
    const char* src = store[eid_layer(key)] + (int64_t)eid_expert(key) * stride;
    CK(cudaMemcpyAsync(slab + (int64_t)s * stride, src, stride, cudaMemcpyHostToDevice,
                       copy_stream));
    CK(cudaEventRecord(fill_ev[s], copy_stream));
    fill_recorded[s] = 1;
    ++copies;
    copy_bytes += stride;
    if (preload) {
      ++preload_copies;
      phys_of[idx(key)] = s;
    } else {
      inflight_slot = s;
    }
  }

  void init_weights();
  void step(cudaStream_t stream, float* h, int B, const std::vector<int64_t>& tokens);
  ~ef_engine();
};

void ef_engine::init_weights() {
  const int L = cfg.L, M = cfg.M, d = cfg.d, ff = cfg.ff;
  const int dt = cfg.dtype;
  auto scale_for = [](double fan_in) { return (float)(std::sqrt(3.0 / fan_in) / 8388608.0); };
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // router and shared weights are always resident
  for (int l = 0; l < L; ++l) {
    CKS(ef_fill_uniform(s, (char*)router_w + (int64_t)l * M * d * esz, dt, (int64_t)M * d,
                        ef_stream_key(cfg.seed, l, 0, 3), scale_for(d), 0));
    if (cfg.shared_ff) {
      int64_t sff = cfg.shared_ff;
      char* base = shared_w + (int64_t)l * sstride;
      CKS(ef_fill_uniform(s, base, dt, sff * d, ef_stream_key(cfg.seed, l, 0, 4), scale_for(d), 0));
      CKS(ef_fill_uniform(s, base + sff * d * esz, dt, sff * d, ef_stream_key(cfg.seed, l, 0, 5),
                          scale_for(d), 0));
      CKS(ef_fill_uniform(s, base + 2 * sff * d * esz, dt, sff * d,
                          ef_stream_key(cfg.seed, l, 0, 6), scale_for((double)sff), 0));
      if (cfg.shared_gate)
        CKS(ef_fill_uniform(s, (char*)sgate_w + (int64_t)l * d * esz, dt, d,
                            ef_stream_key(cfg.seed, l, 0, 7), scale_for(d), 0));
    }
  }
  // experts: generate on device (two staging buffers), copy into the pinned store
  char* stage[2];
  cudaEvent_t done[2];
  for (int i = 0; i < 2; ++i) {
    CK(cudaMalloc(&stage[i], stride));
    CK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
  }
  int64_t nff = (int64_t)ff * d;
  int it = 0;
  for (int l = 0; l < L; ++l) {
    for (int e = 0; e < M; ++e, ++it) {
      char* st = stage[it & 1];
      if (it >= 2) CK(cudaEventSynchronize(done[it & 1]));
      CKS(ef_fill_uniform(s, st, dt, nff, ef_stream_key(cfg.seed, l, e, 0), scale_for(d), 0));
      CKS(ef_fill_uniform(s, st + nff * esz, dt, nff, ef_stream_key(cfg.seed, l, e, 1),
                          scale_for(d), 0));
      CKS(ef_fill_uniform(s, st + 2 * nff * esz, dt, nff, ef_stream_key(cfg.seed, l, e, 2),
                          scale_for(ff), 0));
      CK(cudaMemcpyAsync(store[l] + (int64_t)e * stride, st, 3 * nff * esz, cudaMemcpyDeviceToHost,
                         s));
      CK(cudaEventRecord(done[it & 1], s));
    }
  }
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < 2; ++i) {
    cudaFree(stage[i]);
    cudaEventDestroy(done[i]);
  }
  cudaStreamDestroy(s);
}

ef_engine::~ef_engine() {
  if (copy_stream) cudaStreamSynchronize(copy_stream);
  cudaDeviceSynchronize();
  for (auto ev : fill_ev) cudaEventDestroy(ev);
  for (auto ev : reader_ring) cudaEventDestroy(ev);
  for (auto ev : stall_a) cudaEventDestroy(ev);
  for (auto ev : stall_b) cudaEventDestroy(ev);
  for (void* p : {(void*)slab, router_w, (void*)shared_w, sgate_w, (void*)x_d, (void*)logits_d,
                  (void*)sgl_d, (void*)wts_d, (void*)y_d, (void*)ys_d, (void*)sel_d,
                  (void*)counts_d, (void*)offsets_d, (void*)perm_d, (void*)inv_d, act_d, acts_d})
    if (p) cudaFree(p);
  if (logits_h) cudaFreeHost(logits_h);
  if (sel_h) cudaFreeHost(sel_h);
  for (char* p : store)
    if (p) cudaFreeHost(p);
  if (copy_stream) cudaStreamDestroy(copy_stream);
}

void ef_engine::step(cudaStream_t stream, float* h, int B, const std::vector<int64_t>& tokens_in) {
  using clk = std::chrono::steady_clock;
  const int L = cfg.L, M = cfg.M, k = cfg.top_k, d = cfg.d;
  if (B < 1 || B > cfg.max_batch) throw ValueError("batch size outside [1, max_batch]");
  std::vector<int64_t> tokens = tokens_in;
  if (tokens.empty()) tokens.push_back(-(int64_t)(steps + 1));  // unique prediction-cache key
  cudaEvent_t t_begin, t_end;
  CK(cudaEventCreate(&t_begin));
  CK(cudaEventCreate(&t_end));
  CK(cudaEventRecord(t_begin, stream));
  CKS(ef_rmsnorm(stream, h, x_d, B, d, 1e-6f));
  ++launches;
  std::vector<double> gate(M);
  std::vector<int64_t> gsizes(B, 1);
  double host_acc = 0;
  for (int l = 0; l < L; ++l) {
    // (b) how many future router matrices to score at this layer
    int R = 1;
    if (l == 0)  // the boundary state of a new token is set after its layer-0 routing
      R = Rmax;
    else
      R = 1 + std::min(st->planned_horizon(l), Rmax - 1);
    R = std::min(R, L - l);
    // cache-aware bias mask: residency before this layer's step
    uint64_t mlo = 0, mhi = 0;
    if (cfg.routing_bias != 0.f)
      for (int e = 0; e < M; ++e)
        if (st->resident(l, e)) (e < 64 ? mlo : mhi) |= 1ull << (e & 63);
    CKS(ef_router_logits(stream, x_d, (char*)router_w + (int64_t)l * M * d * esz, cfg.dtype, R, B,
                         d, M, logits_d));
    ++launches;
    if (cfg.shared_ff && cfg.shared_gate) {
      CKS(ef_router_logits(stream, x_d, (char*)sgate_w + (int64_t)l * d * esz, cfg.dtype, 1, B, d,
                           1, sgl_d));
      ++launches;
    }
    CKS(ef_route_permute(stream, logits_d, B, M, k, cfg.route_mode, cfg.routing_bias, mlo, mhi,
                         sel_d, wts_d, counts_d, offsets_d, perm_d, inv_d));
    ++launches;
    CK(cudaMemcpyAsync(logits_h, logits_d, (size_t)R * B * M * sizeof(float),
                       cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(sel_h, sel_d, (size_t)B * k * sizeof(int32_t), cudaMemcpyDeviceToHost,
                       stream));
    d2h_bytes += (int64_t)R * B * M * 4 + (int64_t)B * k * 4;
    CK(cudaStreamSynchronize(stream));
    auto h0 = clk::now();
    // ---- scheduler view of this layer's routing (workload.py:161-179 contract)
    LayerRouting r;
    r.gate.resize(M);
    batch_gate(logits_h, B, M, r.gate.data());
    std::set<int> uni;
    r.group_actual.resize(B);
    for (int t = 0; t < B; ++t) {
      std::vector<int> g(sel_h + t * k, sel_h + (t + 1) * k);
      std::sort(g.begin(), g.end());
      for (int e : g) uni.insert(e);
      r.group_actual[t] = g;
    }
    r.actual.assign(uni.begin(), uni.end());
    if (cfg.record_routing)
      rlog.push_back(RoutingRec{std::vector<float>(logits_h, logits_h + (int64_t)R * B * M),
                                std::vector<int32_t>(sel_h, sel_h + B * k), R, B, mlo, mhi});
    const int Rl = R;
    hooks->pregate_fn = [this, Rl, B, M](int layer, int hz, double* out) {
      if (hz >= Rl) throw RuntimeErr("pre-gate horizon beyond the scored router rows");
      batch_gate(logits_h + (int64_t)hz * B * M, B, M, out);
    };
    if (l == 0) st->begin_token(tokens, gsizes, r);
    std::fill(layer_use.begin(), layer_use.end(), -1);
    st->begin_layer(l);
    st->run_layer(l, r);
    host_acc += std::chrono::duration<double, std::milli>(clk::now() - h0).count();

    // ---- (d) expert FFN over the slots the scheduler resolved
    std::vector<int> cnt(M, 0);
    for (int i = 0; i < B * k; ++i) cnt[sel_h[i]]++;
    std::vector<const char*> wb;
    std::vector<int32_t> p0, nr;
    int run = 0;
    if (cfg.timing) CK(cudaEventRecord(stall_a[l], stream));
    for (int e = 0; e < M; ++e) {
      if (cnt[e]) {
        int s = layer_use[e];
        if (s < 0) throw RuntimeErr("routed expert has no resolved slot");
        if (fill_recorded[s]) CK(cudaStreamWaitEvent(stream, fill_ev[s], 0));
        wb.push_back(slab + (int64_t)s * stride);
        p0.push_back(run);
        nr.push_back(cnt[e]);
      }
      run += cnt[e];
    }
    if (cfg.timing) CK(cudaEventRecord(stall_b[l], stream));
    CKS(expert_ffn_ptrs(stream, x_d, perm_d, k, false, wb.data(), p0.data(), nr.data(),
                        (int)wb.size(), d, cfg.ff, cfg.dtype, act_d, y_d));
    launches += 2;
    const float* ys = nullptr;
    if (cfg.shared_ff) {
      const char* sw = shared_w + (int64_t)l * sstride;
      int32_t z = 0, nb = B;
      CKS(expert_ffn_ptrs(stream, x_d, perm_d, k, true, &sw, &z, &nb, 1, d, cfg.shared_ff,
                          cfg.dtype, acts_d, ys_d));
      launches += 2;
      ys = ys_d;
    }
    CKS(ef_combine(stream, h, x_d, y_d, inv_d, wts_d, ys,
                   (cfg.shared_ff && cfg.shared_gate) ? sgl_d : nullptr, B, d, k, 1e-6f));
    ++launches;
    // release the layer's slots behind a reader event
    int ri = ring_next;
    ring_next = (ring_next + 1) % (int)reader_ring.size();
    CK(cudaEventRecord(reader_ring[ri], stream));
    for (int s : pinned_list) {
      reader_of[s] = ri;
      pinned[s] = 0;
    }
    pinned_list.clear();
    for (int s : deferred_free) free_slots.push_back(s);
    deferred_free.clear();
  }
  st->end_token();
  CK(cudaEventRecord(t_end, stream));
  CK(cudaEventSynchronize(t_end));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, t_begin, t_end));
  step_ms += ms;
  if (cfg.timing) {
    for (int l = 0; l < L; ++l) {
      float a = 0;
      CK(cudaEventElapsedTime(&a, stall_a[l], stall_b[l]));
      stall_ms += a;
    }
  }
  cudaEventDestroy(t_begin);
  cudaEventDestroy(t_end);
  host_ms += host_acc;
  ++steps;
}

extern "C" int ef_engine_create(const ef_engine_cfg* cfg, const ef_sim_cfg* sim,
                                const ef_ladder_cfg* ladder, ef_engine** out) {
  EF_TRY({
    auto e = std::make_unique<ef_engine>();
    e->cfg = *cfg;
    const ef_engine_cfg& c = e->cfg;
    if (c.L < 1 || c.M < 1 || c.M > 128 || c.top_k < 1 || c.top_k > 16 || c.top_k > c.M)
      throw ValueError("unsupported model shape (M <= 128, top_k <= 16)");
    if (c.d % 256 != 0 || c.ff % 8 != 0 || (c.shared_ff && c.shared_ff % 8 != 0))
      throw ValueError("d must be a multiple of 256 and ff of 8");
    if (c.dtype != EF_BF16 && c.dtype != EF_F32) throw ValueError("dtype must be bf16 or f32");
    if (c.max_batch < 1 || c.max_batch * c.top_k > 1024) throw ValueError("bad max_batch");
    if (c.staging_slots < 1) throw ValueError("staging_slots must be >= 1");
    e->esz = c.dtype == EF_BF16 ? 2 : 4;
    e->stride = 3LL * c.d * c.ff * e->esz;
    e->sstride = 3LL * c.d * c.shared_ff * e->esz;
    e->simcfg = sim_config_from(sim);
    if (e->simcfg.L != c.L || e->simcfg.M != c.M || e->simcfg.top_k != c.top_k)
      throw ValueError("scheduler and engine shapes differ");
    if (e->simcfg.expert_size != e->stride)
      throw ValueError("scheduler expert_size_bytes must equal the expert blob size");
    if (e->simcfg.policy.predictor == 3)
      throw ValueError("the oracle predictor needs future routing; it exists only in simulate()");
    e->hooks = std::make_unique<CallbackHooks>(ladder);
    e->st = std::make_unique<Stepper>(e->simcfg, e->hooks.get());
    e->mirror.e = e.get();
    e->st->set_observer(&e->mirror);
    int64_t cap = e->st->cache().capacity();
    e->P = (int)(cap + c.staging_slots);
    int pol_max = e->simcfg.policy.max_step >= 0 ? e->simcfg.policy.max_step : std::max(1, c.L - 1);
    e->Rmax = 1 + std::min(pol_max, c.L - 1);
    if (e->simcfg.policy.strategy == 2) e->Rmax = 1 + std::min(e->simcfg.policy.interval, c.L - 1);
    if (e->simcfg.policy.strategy == 1) e->Rmax = std::min(2, c.L);
    if (e->simcfg.policy.strategy == 0) e->Rmax = 1;

    CK(cudaSetDevice(c.device));
    const int B = c.max_batch, M = c.M, k = c.top_k, d = c.d;
    CK(cudaMalloc(&e->slab, (size_t)e->P * e->stride));
    CK(cudaMalloc(&e->router_w, (size_t)c.L * M * d * e->esz));
    if (c.shared_ff) {
      CK(cudaMalloc(&e->shared_w, (size_t)c.L * e->sstride));
      CK(cudaMalloc(&e->sgate_w, (size_t)c.L * d * e->esz));
      CK(cudaMalloc(&e->acts_d, (size_t)B * c.shared_ff * e->esz));
      CK(cudaMalloc(&e->ys_d, (size_t)B * d * 4));
    }
    CK(cudaMalloc(&e->x_d, (size_t)B * d * 4));
    CK(cudaMalloc(&e->logits_d, (size_t)e->Rmax * B * M * 4));
    CK(cudaMalloc(&e->sgl_d, (size_t)B * 4));
    CK(cudaMalloc(&e->wts_d, (size_t)B * k * 4));
    CK(cudaMalloc(&e->sel_d, (size_t)B * k * 4));
    CK(cudaMalloc(&e->counts_d, (size_t)M * 4));
    CK(cudaMalloc(&e->offsets_d, (size_t)(M + 1) * 4));
    CK(cudaMalloc(&e->perm_d, (size_t)B * k * 4));
    CK(cudaMalloc(&e->inv_d, (size_t)B * k * 4));
    CK(cudaMalloc(&e->act_d, (size_t)B * k * c.ff * e->esz));
    CK(cudaMalloc(&e->y_d, (size_t)B * k * d * 4));
    CK(cudaHostAlloc(&e->logits_h, (size_t)e->Rmax * B * M * 4, cudaHostAllocDefault));
    CK(cudaHostAlloc(&e->sel_h, (size_t)B * k * 4, cudaHostAllocDefault));
    e->store.assign(c.L, nullptr);
    for (int l = 0; l < c.L; ++l)
      CK(cudaHostAlloc(&e->store[l], (size_t)M * e->stride, cudaHostAllocDefault));
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CK(cudaStreamCreateWithPriority(&e->copy_stream, cudaStreamNonBlocking, prio_hi));
    e->fill_ev.resize(e->P);
    e->fill_recorded.assign(e->P, 0);
    e->reader_of.assign(e->P, -1);
    e->pinned.assign(e->P, 0);
    for (auto& ev : e->fill_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->reader_ring.resize(std::max(64, 2 * c.L));
    for (auto& ev : e->reader_ring) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (c.timing) {
      e->stall_a.resize(c.L);
      e->stall_b.resize(c.L);
      for (auto& ev : e->stall_a) CK(cudaEventCreate(&ev));
      for (auto& ev : e->stall_b) CK(cudaEventCreate(&ev));
    }
    e->phys_of.assign((size_t)c.L * M, -1);
    e->layer_use.assign(M, -1);
    for (int s = 0; s < e->P; ++s) e->free_slots.push_back(s);
    e->init_weights();
    *out = e.release();
  });
}

extern "C" void ef_engine_destroy(ef_engine* e) { delete e; }

extern "C" int ef_engine_step(ef_engine* e, void* stream, float* h, int B, const int64_t* tokens,
                              int n_tokens) {
  EF_TRY({
    std::vector<int64_t> t;
    if (tokens && n_tokens > 0) t.assign(tokens, tokens + n_tokens);
    e->step(reinterpret_cast<cudaStream_t>(stream), h, B, t);
  });
}

extern "C" int ef_engine_metrics(ef_engine* e, int64_t* ints, int32_t n, double* bw) {
  EF_TRY({ sim_metrics_out(*e->st, ints, n, bw); });
}
extern "C" int ef_engine_output(ef_engine* e, int32_t kind, int64_t* buf, int64_t max_len,
                                int64_t* n) {
  EF_TRY({
    std::vector<int64_t> o = sim_output(*e->st, kind);
    *n = (int64_t)o.size();
    for (int64_t i = 0; i < (int64_t)o.size() && i < max_len; ++i) buf[i] = o[i];
  });
}
extern "C" int ef_engine_event_details(ef_engine* e, char* buf, int64_t max_len, int64_t* n) {
  EF_TRY({
    std::string d = sim_event_details(*e->st);
    *n = (int64_t)d.size();
    if (buf && max_len > 0) std::memcpy(buf, d.data(), std::min<int64_t>(max_len, *n));
  });
}

extern "C" int ef_engine_stats(ef_engine* e, double* out, int n) {
  EF_TRY({
    double v[13] = {(double)e->steps,         (double)e->copies,
                    (double)e->copy_bytes,    e->stall_ms,
                    (double)e->P,             (double)e->st->cache().capacity(),
                    (double)e->cfg.staging_slots, (double)e->launches,
                    e->host_ms,               e->ffn_ms,
                    e->step_ms,               (double)e->preload_copies,
                    (double)e->d2h_bytes};
    for (int i = 0; i < n && i < 13; ++i) out[i] = v[i];
  });
}

extern "C" int ef_engine_ptr(ef_engine* e, int which, void** out) {
  EF_TRY({
    void* p[10] = {e->slab,   e->router_w, e->shared_w, e->logits_d, e->sel_d,
                   e->wts_d,  e->perm_d,   e->inv_d,    e->y_d,      e->x_d};
    if (which < 0 || which >= 10) throw ValueError("unknown pointer id");
    *out = p[which];
  });
}

extern "C" int ef_engine_routing_log(ef_engine* e, int64_t index, float* logits,
                                     int64_t max_logits, int32_t* sel, int64_t max_sel,
                                     int32_t* R, int32_t* B, uint64_t* mlo, uint64_t* mhi,
                                     int64_t* n_entries) {
  EF_TRY({
    *n_entries = (int64_t)e->rlog.size();
    if (index < 0) return EF_OK;
    if (index >= (int64_t)e->rlog.size()) throw ValueError("routing log index out of range");
    const auto& r = e->rlog[index];
    *R = r.R;
    *B = r.B;
    *mlo = r.mlo;
    *mhi = r.mhi;
    if (logits)
      std::memcpy(logits, r.logits.data(),
                  sizeof(float) * std::min<int64_t>(max_logits, (int64_t)r.logits.size()));
    if (sel)
      std::memcpy(sel, r.sel.data(),
                  sizeof(int32_t) * std::min<int64_t>(max_sel, (int64_t)r.sel.size()));
  });
}

extern "C" int ef_engine_slot_of(ef_engine* e, int32_t layer, int32_t expert, int32_t* slot) {
  EF_TRY({
    if (layer < 0 || layer >= e->cfg.L || expert < 0 || expert >= e->cfg.M)
      throw ValueError("expert id out of range");
    *slot = e->phys_of[(int64_t)layer * e->cfg.M + expert];
  });
}
