// pipeline.h — host/device control blocks of the engine's flag-gated decode
// pipeline (engine.cu) and the launchers in kernels.cu.
//
// Per layer: the route kernel publishes (sel, row-0 logits, done=1) into
// mapped host memory; the host runs the scheduler step and writes a HostCtrl
// (slots, rows, copy sequence numbers, next layer's bias mask) then go=1; the
// gate kernel copies it to DevCtrl, resets go and lets the routed FFN run.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ef {
constexpr int kMaxActive = 80;
extern bool g_use_pdl;  // launch decode kernels with programmatic dependent launch
constexpr int kStats = 16;  // per-layer device timeline slots (see engine.cu dump)

struct HostCtrl {
  volatile uint32_t go;
  int32_t n_active;
  uint64_t mask[2];    // cache-aware bias mask for THIS layer's routing
  int4 ent[kMaxActive];  // {slot, p0, rows, need_seq}
};

struct DevCtrl {
  int32_t n_active, pad[3];
  int4 ent[kMaxActive];
};

// Device-side slot resolution by the route kernel (see resolve_fast).
constexpr int kMaxTab = 128;
struct RouteFast {
  DevCtrl* dc;          // this layer's decision block
  unsigned* fast_word;  // set to seq when every routed expert resolved, else 0
  unsigned seq;
  // this layer's slot table row {slot, fill seq} (slot -1: not resident),
  // passed by value in the launch: the host enqueues the router after it has
  // decided the previous layer, so the row is final and needs no PCIe read
  int2 tab[kMaxTab];
};
// Extra duties of the fused gate warp (up kernel CTA 0, warp 0).
struct GateIO {
  const unsigned* fast_word;  // == seq: decision already on the device; the gate neither
                              // waits for the host nor copies its decision
  const int32_t* sel_src;     // publish sel[n_sel] and logits rows[n_pub] to the host
  const float* logits_src;
  int n_sel, n_pub;
  int32_t* host_sel;
  float* host_logits;
  uint32_t* host_done;
  int M;
  const uint64_t* mask_src;  // the layer's final bias mask (route kernel, after top-up)
  uint64_t* host_mask;
};
struct HostOut {  // followed by sel[B*k] int32 and logits[B*M] f32
  volatile uint32_t done;
  uint32_t pad0;
  uint64_t mask[2];  // final cache-aware bias mask the route kernel selected on
  uint32_t pad[10];
};

// shared expert(s) of a layer riding in the routed FFN launch (tensor-core path)
struct SharedFfn {
  const char* w;  // [W1 sff x d | W3 sff x d | W2 d x sff] bf16
  int sff, B;
  void* act;      // [B, sff] bf16
  float* y;       // [B, d]
};
bool ffn_mma_enabled(int dtype, int d, int ff, int sff, int max_tok);
int expert_ffn_ptrs(cudaStream_t st, const float* x, const int32_t* perm, int k, bool identity,
                    const char* const* wbase, const int32_t* p0, const int32_t* nrows,
                    int n_active, int d, int ff, int dtype, void* act, float* y);
int expert_ffn_ctrl(cudaStream_t st, const float* x, const int32_t* perm, int k, const char* slab,
                    int64_t stride, const void* dctrl, const uint32_t* ready,
                    unsigned long long* stats, int max_active, int max_rows, int d, int ff,
                    int dtype, void* act, float* y, const SharedFfn* sh = nullptr);
int launch_gate(cudaStream_t st, void* host_ctrl_dev, void* dctrl, unsigned long long* stats);
int launch_init_stats(cudaStream_t st, unsigned long long* stats, int L);
int preload_pipeline_kernels();
int launch_route_publish(cudaStream_t st, const float* logits, int B, int M, int k, int mode,
                         float bias, uint64_t mlo, uint64_t mhi, int topup_U, int32_t* sel,
                         float* wts, int32_t* counts, int32_t* offsets, int32_t* perm,
                         int32_t* inv, uint64_t* host_mask, int32_t* host_sel, float* host_logits,
                         uint32_t* host_done, unsigned long long* stamp, int n_pub);
int router_logits_stamped(cudaStream_t st, const float* x, const void* w, int dtype, int R, int B,
                          int d, int M, float* logits, unsigned long long* stamp);
int combine_stamped(cudaStream_t st, float* h, float* x, const float* y, const int32_t* inv,
                    const float* wts, const float* ys, const float* gate_logit, int B, int d, int k,
                    float eps, unsigned long long* stamp);
// Fused decode pipeline (default for the split FFN): router + route in one
// kernel (the last CTA routes; optionally the previous layer's combine +
// rmsnorm first), gate folded into the up kernel.
// The previous layer's combine, folded into router_route_fused (x is then
// both the router input and, rewritten by the last CTA, the layer's x).
struct CombineIn {
  float* h;
  const float* y;
  const float* ys;
  const float* gate_logit;
  float eps;
  unsigned long long* stamp;
  bool y_slot_order;  // y rows indexed by (token, rank) slot (fused FFN), not by inv
};
// zero-copy hidden-state I/O between pinned host memory and HBM (SM loads/stores)
int launch_host_io(cudaStream_t st, const float* src, float* dst, int64_t n, bool to_host);
int router_route_fused(cudaStream_t st, const float* x, const void* w, int dtype, int R, int B,
                       int d, int M, float* logits, unsigned long long* stamp_router, int k,
                       int mode, float bias, uint64_t mlo, uint64_t mhi, int topup_U,
                       uint64_t* mask_out, uint64_t* host_mask, int32_t* sel, float* wts,
                       int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv,
                       int32_t* host_sel, float* host_logits, uint32_t* host_done,
                       unsigned long long* stamp_route, int* counter,
                       const CombineIn* comb = nullptr, const RouteFast* rf = nullptr,
                       const void* sgate_w = nullptr, float* sgl_out = nullptr);
int expert_ffn_fused(cudaStream_t st, const float* x, const int32_t* perm, int k, const char* slab,
                     int64_t stride, void* hctrl_dev, void* dctrl, volatile unsigned* dflag,
                     unsigned seq, const uint32_t* ready, unsigned long long* stats, int max_active,
                     int max_rows, int d, int ff, int dtype, void* act, float* y,
                     const GateIO* io = nullptr, const SharedFfn* sh = nullptr);
// ---- persistent decode layer (decode_layer.cuh): one launch per layer runs the
// previous layer's combine + rmsnorm, the router rows, the route, and the
// shared + routed expert FFN (gate/up, then down) as a dataflow of work items
// over a fixed grid (one 512-thread CTA per SM, four 4-warp workers each).
struct LayerSync {  // per layer, zeroed at the start of every step (rq: see launch_zero_sync)
  int rq[2];        // router row claims, by step parity
  int q;            // next work item
  int ticket;       // router rows finished
  unsigned route;   // == launch seq: the decision block is final
  int sh_up;        // shared-expert gate/up units finished
  int up[kMaxActive];  // routed gate/up units finished, per decision entry
  int pad[10];
};
struct DecodeLayerIn {
  int B, d, ff, sff, M, k, mode, R;  // R router matrices (layer + pre-gate rows)
  bool sgate;                        // one more router row: the shared expert's gate
  float eps;
  // hidden state: h_dst = h_src (+ previous layer's MoE output); x_out = rmsnorm(h_dst)
  const float* h_src;
  float* h_dst;
  float* x_out;
  bool has_prev;
  const float* y_prev;    // [B*k, d] slot order
  const float* wts_prev;  // [B*k]
  const float* ys_prev;   // [B, d] shared-expert output (null: none)
  const float* sgl_prev;  // [B] shared-gate logits (null: ungated)
  unsigned long long* comb_stamp;
  // router
  const void* w_router;  // [R*M, d] (rows of layers l .. l+R-1)
  const void* w_sgate;   // [d]
  float* logits;         // [R][B][M]
  float* sgl_out;        // [B]
  // route
  float bias;
  uint64_t mlo, mhi;
  int topup_U;
  uint64_t* mask_out;
  int32_t *sel, *counts, *offsets, *perm, *inv;
  float* wts_out;
  RouteFast rf;
  void* hc_dev;  // HostCtrl of the layer (null: standalone, every expert must resolve)
  GateIO io;     // host publishing (io.host_done null: none)
  // FFN
  const char* slab;
  int64_t stride;
  const uint32_t* ready;  // null: no copy waits
  const void* shared_w;
  void* act;
  void* act_s;
  float* y_out;
  float* ys_out;
  int max_active;
  LayerSync* sync;
  unsigned long long* stats;
  void* pub;  // mapped host words of the tagged publish (null: none)
  int parity; // router-claim counter of this step (launch_zero_sync)
  bool x_before_publish;  // write h / x before the host publish (the host records x)
  void* trace;  // EF_MEGA_TRACE: per work item {start, end} ns, [router rows | queue items]
};
bool decode_layer_supported(int dtype, int d, int ff, int sff, int M, int k, int B);
int launch_decode_layer(cudaStream_t st, const DecodeLayerIn& in);
int launch_final_combine(cudaStream_t st, const float* h_src, float* h_dst, const float* y,
                         const float* wts, const float* ys, const float* sgl, int B, int d, int k);
int launch_zero_sync(cudaStream_t st, LayerSync* sync, int L, int parity);
int preload_decode_layer();
// expert parallelism (kernels.cu "expert parallelism" section)
int ep_pack(cudaStream_t st, const float* x, const float* logits, const int32_t* sel,
            const float* wts, int B, int d, int Rm, int M, int k, float* out);
int ep_owner(cudaStream_t st, const float* recv, int64_t W, int G, int B, int k, int M, int d,
             int Rm, int R, int rank, int e0, int Ms, int32_t* counts, int32_t* offsets,
             int32_t* perm, int32_t* home_idx, int32_t* host_sel, float* host_logits,
             uint32_t* host_done);
int expert_ffn_ep(cudaStream_t st, const float* recv, int64_t W, int B, const int32_t* perm, int k,
                  const char* slab, int64_t stride, const void* dctrl, const uint32_t* ready,
                  unsigned long long* stats, int max_active, int max_rows, int d, int ff,
                  int dtype, void* act, float* y);
}  // namespace ef
