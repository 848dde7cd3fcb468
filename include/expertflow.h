/*
 * expertflow.h — C ABI of the B200-native ExpertFlow hot path
 * (libexpertflow.so, built from paper_2510_26730_b200/csrc).
 *
 * Plain pointers, sizes and opaque handles only; no torch types.  Device
 * pointers are CUDA device addresses (e.g. torch.Tensor.data_ptr()), streams
 * are cudaStream_t passed as void*.  Every entry point returns an int status:
 *   EF_OK (0), EF_EINVAL (-22, maps to ValueError), EF_ERUNTIME (-1, maps to
 *   RuntimeError, e.g. the reference's no-forward-progress guard),
 *   EF_ECUDA (-5, CUDA failure, RuntimeError), EF_ENOMEM (-12).
 * ef_last_error() returns a thread-local message for the last failure.
 *
 * Each function names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/moesim).  The reference is pure Python; its
 * "FFI" for this path is the Python call surface, so the binding a
 * maintainer adds is a ctypes stub.
 */
#ifndef EXPERTFLOW_H
#define EXPERTFLOW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EF_OK 0
#define EF_ERUNTIME (-1)
#define EF_ECUDA (-5)
#define EF_ENOMEM (-12)
#define EF_EINVAL (-22)

#define EF_TIER_HIGH 1 /* memory.py:24 TIER_HIGH */
#define EF_TIER_LOW 0  /* memory.py:25 TIER_LOW  */

/* cache event kinds (memory.py:63-65, :83-85) */
#define EF_EV_MISS 0
#define EF_EV_HIT 1
#define EF_EV_ADMIT 2
#define EF_EV_EVICT 3

const char* ef_last_error(void);
int ef_abi_version(void);

/* ------------------------------------------------------------------ */
/* Decision primitives                                                */
/* ------------------------------------------------------------------ */

/* scheduler.py:36-53 expected_expert_count */
int ef_expected_expert_count(const double* probs, int m, double cum_threshold, int* out_count);
/* scheduler.py:56-60 top_experts: ascending indices of the `count` best */
int ef_top_experts(const double* probs, int m, int count, int* out_sel);
/* scheduler.py:63-74 swap_in_latency */
int ef_swap_in_latency(int64_t n, int64_t size, int64_t bw, int64_t* out_ns);
/* scheduler.py:77-105 compute_step, exact-integer bandwidth path */
int ef_compute_step_int(int64_t n_e, int64_t size, int64_t bw, int64_t layer_ns, int min_step,
                        int max_step, int* out_step);
/* scheduler.py:77-105 compute_step, float-bandwidth path (math.ceil of a double) */
int ef_compute_step_float(int64_t n_e, int64_t size, double bw, int64_t layer_ns, int min_step,
                          int max_step, int* out_step);

/* scheduler.py:108-163 StepState / on_stall / on_overfetch */
typedef struct ef_step_state {
  int32_t current, max_step, min_step, stall_count, overfetch_count, stall_threshold,
      overfetch_threshold;
} ef_step_state;
int ef_step_validate(const ef_step_state* s);
int ef_step_on_stall(ef_step_state* s);
int ef_step_on_overfetch(ef_step_state* s);

/* ------------------------------------------------------------------ */
/* ExpertCache — memory.py:28-156 (two-tier LRU) + slot table          */
/* ------------------------------------------------------------------ */
typedef struct ef_cache ef_cache;
int ef_cache_create(int64_t capacity_bytes, int64_t expert_size_bytes, int record_events,
                    ef_cache** out);
void ef_cache_destroy(ef_cache* c);
int ef_cache_access(ef_cache* c, int32_t layer, int32_t expert, int64_t now, int* out_hit);
/* victims written as (layer, expert) pairs; *n_victims may exceed max_victims (then truncated) */
int ef_cache_admit(ef_cache* c, int32_t layer, int32_t expert, int tier, int64_t now,
                   int32_t* victims, int max_victims, int* n_victims);
/* pred: n_pred (layer, expert) pairs */
int ef_cache_reassign_tiers(ef_cache* c, const int32_t* pred, int n_pred, int64_t recent_window,
                            int64_t now);
/* tier: EF_TIER_* or -1 when absent */
int ef_cache_query(ef_cache* c, int32_t layer, int32_t expert, int* tier, int64_t* last_access);
/* out: capacity_experts, size, hits, misses, admissions, evictions */
int ef_cache_counters(ef_cache* c, int64_t out[6]);
/* resident pairs in (layer, expert) order */
int ef_cache_resident(ef_cache* c, int32_t* pairs, int max_pairs, int* n);
/* events as rows (now, kind, layer, expert); returns -1 count when recording is off */
int ef_cache_events(ef_cache* c, int64_t* rows, int64_t max_rows, int64_t* n);

/* ------------------------------------------------------------------ */
/* TransferQueue — memory.py:183-202; BandwidthEstimator — :205-236    */
/* ------------------------------------------------------------------ */
typedef struct ef_tqueue ef_tqueue;
int ef_tqueue_create(ef_tqueue** out);
void ef_tqueue_destroy(ef_tqueue* q);
int ef_tqueue_enqueue(ef_tqueue* q, int32_t layer, int32_t expert, int priority, int64_t* out_seq);
/* *found = 0 when empty */
int ef_tqueue_next(ef_tqueue* q, int32_t* layer, int32_t* expert, int* priority, int64_t* seq,
                   int* found);
int ef_tqueue_len(ef_tqueue* q, int64_t* n);

/* Physical transfer engine (xfer.cu): expert copies pinned host -> HBM issued in
   TransferQueue order (MISS 0 before PREFETCH 1, FIFO within a class; memory.py:184-202)
   on a dedicated high-priority copy stream, at most max_inflight outstanding (1 = the
   reference's serial link, engine.py:328-354), each bracketed by CUDA events; measured
   rates feed a BandwidthEstimator (alpha 0.25, memory.py:205-236).  Replaces the
   reference's logical _pump/_advance_to transfer start/finish for a caller running its
   own scheduler. */
typedef struct ef_xfer ef_xfer;
int ef_xfer_create(int32_t device, int32_t max_inflight, ef_xfer** out);
void ef_xfer_destroy(ef_xfer* x);
/* queue one copy; *ticket identifies it (0, 1, 2, ... in submission order) */
int ef_xfer_submit(ef_xfer* x, int32_t layer, int32_t expert, int32_t priority,
                   const void* src_host, void* dst_dev, int64_t bytes, int64_t* ticket);
/* issue queued copies while fewer than max_inflight are outstanding */
int ef_xfer_pump(ef_xfer* x, int32_t* issued);
/* tickets completed since the last poll, in completion order (pumps first) */
int ef_xfer_poll(ef_xfer* x, int64_t* tickets, int32_t max, int32_t* n);
/* block the host until `ticket` has landed (pumping as copies complete) */
int ef_xfer_wait(ef_xfer* x, int64_t ticket);
/* make `stream` wait on the device for an issued `ticket` (no host block) */
int ef_xfer_stream_wait(ef_xfer* x, int64_t ticket, void* stream);
/* measured bandwidth EWMA in bytes/s (0 before the first completion), copies completed */
int ef_xfer_bandwidth(ef_xfer* x, double* bytes_per_s, int64_t* completed);

typedef struct ef_bw ef_bw;
int ef_bw_create(int has_initial, double initial, double alpha, ef_bw** out);
void ef_bw_destroy(ef_bw* b);
int ef_bw_observe(ef_bw* b, int64_t bytes, int64_t elapsed_ns, double* out_estimate);
int ef_bw_estimate(ef_bw* b, double* out);

/* ------------------------------------------------------------------ */
/* PredictionCache (scheduler.py:194-221) with encoded int64 values    */
/* ------------------------------------------------------------------ */
typedef struct ef_pcache ef_pcache;
int ef_pcache_create(int capacity, ef_pcache** out);
void ef_pcache_destroy(ef_pcache* p);
/* key = (tokens[n_tokens], layer, step); value = int64 blob (encoding owned by caller) */
int ef_pcache_get(ef_pcache* p, const int64_t* tokens, int n_tokens, int64_t layer, int64_t step,
                  int64_t* val, int64_t max_val, int64_t* n_val, int* found);
int ef_pcache_put(ef_pcache* p, const int64_t* tokens, int n_tokens, int64_t layer, int64_t step,
                  const int64_t* val, int64_t n_val);
int ef_pcache_stats(ef_pcache* p, int64_t out[3]); /* hits, misses, len */

/* ------------------------------------------------------------------ */
/* Forest inference — predictor.py:195-232, :312-359, :608-632         */
/* ------------------------------------------------------------------ */
typedef struct ef_forest ef_forest;
/* flat node arrays for all trees concatenated; tree_off[n_trees+1] node offsets;
   value[n_nodes*num_outputs] (leaf rows; ignored for interior nodes) */
int ef_forest_create(int n_trees, const int64_t* tree_off, const int32_t* feature,
                     const double* threshold, const int32_t* left, const int32_t* right,
                     const double* value, int32_t feature_len, int32_t num_outputs, int residual,
                     ef_forest** out);
void ef_forest_destroy(ef_forest* f);
int ef_forest_predict(ef_forest* f, const double* features, const double* baseline /*nullable*/,
                      double* out_scores);
/* predictor.py:113-128 inference_features; table row-major [vocab][embed_dim];
   history given as (layer, n, experts...) records */
int ef_inference_features(const double* table, int64_t vocab, int32_t embed_dim, int32_t L,
                          int32_t M, const int64_t* tokens, int n_tokens, int32_t step,
                          int32_t target, const int32_t* hist, int64_t hist_len, double* out);

/* Prediction ladder — scheduler.py:247-309.  Callbacks stand in for the
   reference's duck-typed plug points (PredictionQuery.pregate, forest). */
typedef int (*ef_pregate_cb)(void* user, int32_t layer, int32_t horizon, double* probs_out);
typedef int (*ef_forest_cb)(void* user, const double* features, int32_t n_features,
                            const double* baseline /*nullable*/, double* scores_out);
typedef struct ef_ladder_cfg {
  int32_t L, M, top_k;
  double cum_threshold;
  /* forest: exactly one of native / callback, or neither */
  ef_forest* forest;
  ef_forest_cb forest_cb;
  void* forest_user;
  int32_t forest_feature_len;
  const double* table; /* embedding table for features (required with a forest) */
  int64_t vocab;
  int32_t embed_dim;
  ef_pregate_cb pregate_cb; /* nullable */
  void* pregate_user;
} ef_ladder_cfg;
/* out: (target, n, experts...) records, *n_out int64 written */
int ef_predict_experts(const ef_ladder_cfg* cfg, ef_pcache* cache, const int64_t* tokens,
                       int n_tokens, int32_t layer, int32_t step, const double* router_probs,
                       const int32_t* known, int64_t known_len, int64_t* out, int64_t max_out,
                       int64_t* n_out);

/* engine.py:192-209 route_batch.  groups: (gid, n, experts...) records over one layer;
   resident: M-bit mask as bytes.  order/deferred receive group ids. */
int ef_route_batch(const int32_t* groups, int64_t groups_len, const uint8_t* resident_mask,
                   int32_t M, int32_t* order, int32_t* deferred, int32_t* n_groups,
                   int32_t* n_deferred);

/* ------------------------------------------------------------------ */
/* Scheduler stepper — engine.py:240-716 (_Sim / simulate), steppable  */
/* ------------------------------------------------------------------ */
typedef struct ef_sim ef_sim;
typedef struct ef_sim_cfg {
  int32_t L, M, top_k;
  int64_t expert_size_bytes, link_bw, device_memory_bytes, layer_ns;
  /* PolicyConfig, engine.py:95-142 */
  int32_t strategy;  /* 0 static 1 reactive 2 fixed_interval 3 adaptive */
  int32_t predictor; /* 0 none 1 pregate 2 forest 3 oracle */
  int32_t interval, cache_aware_routing, cold_start_preload;
  double cum_threshold;
  int32_t stall_threshold, overfetch_threshold, min_step, max_step /* -1 = L-1 */,
      recent_window /* -1 = S */;
  int32_t prediction_cache_capacity;
  int32_t emit_events;
  uint64_t seed;
  /* 1: bandwidth feedback into S: each adaptive boundary re-bases
     the step on the current bandwidth estimate — the logical EWMA in ef_sim, the
     copy engine's measured transfer times in ef_engine.  0 (parity mode): S is
     computed once, as the reference does (engine.py:545-556). */
  int32_t bw_feedback;
} ef_sim_cfg;
int ef_sim_create(const ef_sim_cfg* cfg, const ef_ladder_cfg* ladder, ef_sim** out);
void ef_sim_destroy(ef_sim* s);
/* One token (= one trace, ActivationTrace workload.py:161-179):
   gates[L*M] fp64, actual: (n, experts...) per layer, groups: per layer
   (n_groups, [n, experts...]*), group_sizes[n_groups]. */
int ef_sim_run_token(ef_sim* s, const int64_t* tokens, int n_tokens, const double* gates,
                     const int32_t* actual, int64_t actual_len, const int32_t* groups,
                     int64_t groups_len, const int64_t* group_sizes, int32_t n_groups);
/* SimMetrics scalars (engine.py:157-189), fixed order documented in simcore.h */
int ef_sim_metrics(ef_sim* s, int64_t* ints, int32_t n_ints, double* bw_estimate);
/* variable-length outputs; kind: 0 step_history(2/row) 1 per_layer 2 samples 3 events 4 cache events */
int ef_sim_output(ef_sim* s, int32_t kind, int64_t* buf, int64_t max_len, int64_t* n);
/* event detail strings, '\n' separated, in sorted event order */
int ef_sim_event_details(ef_sim* s, char* buf, int64_t max_len, int64_t* n);

/* ------------------------------------------------------------------ */
/* Device kernels (sm_100a).  Graph-capturable: no allocation, no sync */
/* ------------------------------------------------------------------ */
/* dtype codes */
#define EF_F32 0
#define EF_BF16 1
/* routing conventions */
#define EF_ROUTE_MIXTRAL 0 /* softmax over the k selected logits */
#define EF_ROUTE_SOFTMAX_TOPK 1 /* softmax over all M, gathered, no renorm */

/* counter-based synthetic weights (oracle/numerics.py fill_uniform) */
int ef_fill_uniform(void* stream, void* dst, int dtype, int64_t n, uint64_t key, float scale,
                    int64_t offset);
uint64_t ef_stream_key(uint64_t seed, int32_t layer, int32_t expert, int32_t mat);

/* x[B,d] = rmsnorm(h[B,d]) (fp32) */
int ef_rmsnorm(void* stream, const float* h, float* x, int B, int d, float eps);
/* (a)+(b): logits[R, B, M] fp32 = x[B,d] . W[rows]^T for R router matrices
   starting at w (stacked [R, M, d] of dtype) */
int ef_router_logits(void* stream, const float* x, const void* w, int dtype, int R, int B, int d,
                     int M, float* logits);
/* (a) epilogue + (c): top-k keyed on logits (+bias*resident), routing weights,
   stable permutation.  sel[B,k], wts[B,k], counts[M], offsets[M+1], perm[B*k], inv[B*k] */
int ef_route_permute(void* stream, const float* logits, int B, int M, int k, int mode,
                     float bias, uint64_t resident_mask_lo, uint64_t resident_mask_hi,
                     int32_t* sel, float* wts, int32_t* counts, int32_t* offsets,
                     int32_t* perm, int32_t* inv);
/* (d) decode expert FFN over a slot-indirected slab.
   Active list: n_active entries of (slot, row_offset, n_rows) into perm.
   Slot s holds [W1 ff*d | W3 ff*d | W2 d*ff] at slab + s*slot_stride_bytes.
   Row p of the permuted batch reads x[perm[p]/k]; output y[p, d] fp32.
   act is scratch [rows_total, ff] of dtype. */
int ef_expert_ffn_decode(void* stream, const float* x, const int32_t* perm, int k,
                         const void* slab, int64_t slot_stride_bytes, const int32_t* act_slot,
                         const int32_t* act_off, const int32_t* act_rows, int n_active, int d,
                         int ff, int dtype, void* act, float* y);
/* (c) unpermute + weighted combine (rank order) + optional shared expert +
   residual + next rmsnorm:  h[t] += sum_r wts[t,r]*y[inv[t,r]] + g_t*ys[t];
   x = rmsnorm(h).  ys/shared_gate nullable. */
int ef_combine(void* stream, float* h, float* x, const float* y, const int32_t* inv,
               const float* wts, const float* ys, const float* shared_gate_logit, int B, int d,
               int k, float eps);

/* (c) prefill permute gather: out[p] = bf16(x[perm[p] / k]) rows, x fp32 [*, d] */
int ef_gather_rows_bf16(void* stream, const float* x, const int32_t* perm, int k, int d, int n,
                        void* out);
/* (d) prefill expert FFN: TMA + tcgen05 grouped GEMM (grouped_gemm.cu).
   C[rows, N] = A[rows, K] . B_e^T per tile; A bf16 [a_rows, K] K-contiguous;
   B bf16 view [b_rows, K] with row pitch b_pitch elements (the slab viewed as
   one tensor).  tiles: DEVICE int4[n_tiles] = {a_row0, b_row0, m_valid, n0}
   (128-row m-tiles, 128-column n-tiles, K % 64 == 0).  dual: B rows
   b_row0+n0.. are W1 and b_row0+dual_off+n0.. are W3; out = bf16
   silu(A.W1^T) * (A.W3^T).  Otherwise out = fp32 A.B^T.  out_ld in elements. */
int ef_grouped_gemm_bf16(void* stream, const void* A, int64_t a_rows, int K, const void* B,
                         int64_t b_rows, int64_t b_pitch, const void* tiles, int n_tiles, int dual,
                         int dual_off, void* out, int out_ld);

/* ------------------------------------------------------------------ */
/* Expert parallelism: collectives of the EP decode step */
/* ------------------------------------------------------------------ */
#define EF_COLL_ALLGATHER 0 /* recv[g*bytes..] = rank g's send[0..bytes) */
#define EF_COLL_ALLTOALL 1  /* recv[g*bytes..] = rank g's send[me*bytes..) */
/* host transport of the EP collectives (device buffers, ordered on `stream`;
   return 0 on success).  The NCCL transport is built in; a callback lets G
   processes share one GPU in tests (NCCL refuses two ranks on one device). */
typedef int (*ef_collective_cb)(void* user, int op, void* dev_send, void* dev_recv,
                                int64_t bytes, void* stream);
/* 128-byte NCCL unique id for an EP group (rank 0 creates, all pass it) */
int ef_ep_nccl_unique_id(void* out128);
typedef struct ef_ep_comm ef_ep_comm;
/* an EP group handle: nccl_id128 non-null -> NCCL; else cb (world 1: local copies) */
int ef_ep_comm_create(int world, int rank, const void* nccl_id128, ef_collective_cb cb,
                      void* user, ef_ep_comm** out);
void ef_ep_comm_destroy(ef_ep_comm* c);
/* dispatch (replaces the reference's single-process routing hand-off,
   engine.py:573-581, for G ranks): pack this rank's routing block
   [x B*d f32 | logits Rm*B*M f32 | sel B*k i32 | wts B*k f32] into `send`
   (block_words 4-byte words, >= the block) and all-gather every rank's block
   into recv[G][block_words]. */
int ef_ep_dispatch(ef_ep_comm* c, void* stream, const float* x, const float* logits,
                   const int32_t* sel, const float* wts, int B, int d, int Rm, int M, int k,
                   int64_t block_words, float* send, float* recv);
/* owner side: the (token, rank) slots of all G*B tokens routed to the Ms experts
   [e0, e0+Ms) this rank owns, stable by (local expert, global slot) -> counts[Ms],
   offsets[Ms+1], perm[<= G*B*k]; home_idx[B*k] = row of each local slot in the
   all-to-all output (owner*B*k + t*k + r) */
int ef_ep_owner(void* stream, const float* recv, int64_t block_words, int G, int B, int k, int M,
                int d, int Rm, int rank, int e0, int Ms, int32_t* counts, int32_t* offsets,
                int32_t* perm, int32_t* home_idx);
/* combine: all-to-all of y rows in global slot order (y_slots [G*B*k][d] f32,
   chunk g = rank g's slots) into y_recv, then the rank-order weighted combine
   h[t] += sum_r wts[t,r]*y_recv[home_idx[t*k+r]] (+ g_t*ys[t]); x = rmsnorm(h)
   (x nullable).  Same arithmetic and order as ef_combine. */
int ef_ep_combine(ef_ep_comm* c, void* stream, const float* y_slots, float* y_recv,
                  const int32_t* home_idx, const float* wts, const float* ys,
                  const float* shared_gate_logit, int B, int d, int k, float* h, float* x);

/* the shard's scheduler view of one layer's global routing (logits [GB][M] of all
   G ranks' tokens, sel [GB][k]): gate[Ms] = the fp64 batch gate (bias 0, sequential
   sums) restricted to the owned experts and renormalised; groups[GB][k] = each
   token's owned experts as local ids ascending (-1 padded); actual[Ms] = their
   ascending union (-1 padded, *n_actual entries).  The routing contract of
   workload.py:161-179 per shard. */
int ef_ep_shard_view(const float* logits, const int32_t* sel, int GB, int M, int k, int G,
                     int rank, double* gate, int32_t* groups, int32_t* actual, int32_t* n_actual);

/* ------------------------------------------------------------------ */
/* MoE decode engine: slab + pinned host store + copy streams + stepper */
/* ------------------------------------------------------------------ */
typedef struct ef_engine ef_engine;
typedef struct ef_engine_cfg {
  int32_t L, M, top_k, d, ff, dtype, route_mode, max_batch;
  int32_t shared_ff, shared_gate; /* 0 = no shared expert */
  int64_t budget_slots;           /* logical cache capacity in experts */
  int32_t staging_slots;          /* extra physical slots (landing + pinned), >= 1 */
  float routing_bias;             /* cache-aware logit bias (0 = off) */
  uint64_t seed;
  int32_t device;
  int32_t timing; /* record per-layer stall events (physical stall %) */
  int32_t record_routing; /* keep every layer's logits / selection for parity checks */
  int32_t max_prefill;    /* > 0: allocate prefill buffers for up to this many tokens (bf16) */
  const char* host_store_shm; /* non-null: pinned host expert store in POSIX shared memory of
                                 this name, shared by the processes of one node */
  int32_t host_store_attach;  /* 1: attach to a store another process created and filled */
  int32_t peer_device;        /* device holding the peer pool (may equal `device`) */
  int64_t peer_pool_experts;  /* N: pool size in experts; 0 turns the tier off */
  /* Peer-HBM miss tier (the reference models one host link,
     SPEC.md:557): home copies of N experts (the first N flat ids l*M+e, or the
     list below) live in a pool on the peer device; a swap-in of one of them is a
     cudaMemcpyPeerAsync over NVLink instead of the host copy.  Tiers change
     only latency, never which experts are requested or admitted.  A pool on
     the engine's own device is a test-only stand-in (EF_PEER_SAME_DEVICE=1):
     same-device copies run on SMs and can deadlock a GPU-filling FFN. */
  const int32_t* peer_pool_ids; /* optional [N] flat expert ids (l*M+e) in pool order; null:
                                   the first N experts.  Expert-parallel placement: the home
                                   copies of one rank's owned experts (ep.peer_pool_ids) */
  const void* peer_ipc_handle; /* non-null: 64-byte cudaIpcMemHandle_t of a pool another
                                  process (one process per GPU) created and filled on
                                  peer_device (ef_engine_peer_pool_handle); opened, not
                                  allocated or filled */
  /* Expert parallelism: ep_world > 0 makes this engine rank
     ep_rank of an ep_world-rank group.  It owns experts [ep_rank*M/G, +M/G) of every
     layer (G | M): its slab, pinned host store and scheduler (ef_sim_cfg with
     M/G experts, top_k min(k, M/G), the shard's budget) cover only those; every step
     routes its own B tokens, all-gathers the routing blocks, runs its experts for all
     G*B tokens and all-to-alls the outputs back (ep_step).  Transport: ep_nccl_id
     (NCCL), else ep_collective (callback), else (world 1) local copies.  Decode only,
     routing_bias must be 0. */
  int32_t ep_world;
  int32_t ep_rank;
  const void* ep_nccl_id;
  ef_collective_cb ep_collective;
  void* ep_user;
  /* peer pool modes (see peer_device above): 1 = allocate and fill the pool on this
     engine's own device for OTHER processes only (this engine's misses never read it;
     export with ef_engine_peer_pool_handle).  Pool ids are global flat ids l*M + e. */
  int32_t peer_pool_export;
  uint64_t peer_ipc_layout_hash; /* the exporter's layout hash, checked when opening */
} ef_engine_cfg;
int ef_engine_create(const ef_engine_cfg* cfg, const ef_sim_cfg* sim, const ef_ladder_cfg* ladder,
                     ef_engine** out);
void ef_engine_destroy(ef_engine* e);
/* one decode step: h[B,d] fp32 device in/out, on `stream` */
int ef_engine_step(ef_engine* e, void* stream, float* h, int B, const int64_t* tokens,
                   int n_tokens);
/* prefill: T <= max_prefill tokens h[T,d] (fp32 device, in place) through every
   layer as one scheduler step (one routing group per token); the expert FFNs run
   on the tcgen05/TMA grouped GEMM (ef_grouped_gemm_bf16), synchronously per layer */
int ef_engine_prefill(ef_engine* e, void* stream, float* h, int T, const int64_t* tokens,
                      int n_tokens);
/* the same step with the hidden state in pinned host memory: h_in[B,d] is read
   and h_out[B,d] written (may alias) by SM loads/stores over PCIe, ordered on
   `stream` (h_out is complete when the stream reaches the step's end); never
   queues behind an expert swap-in on the copy engine */
int ef_engine_step_host(ef_engine* e, void* stream, const float* h_in, float* h_out, int B,
                        const int64_t* tokens, int n_tokens);
/* scheduler outputs of the engine's stepper: same layouts as ef_sim_* */
int ef_engine_metrics(ef_engine* e, int64_t* ints, int32_t n_ints, double* bw_estimate);
int ef_engine_output(ef_engine* e, int32_t kind, int64_t* buf, int64_t max_len, int64_t* n);
int ef_engine_event_details(ef_engine* e, char* buf, int64_t max_len, int64_t* n);
/* physical counters, in order: steps, copies, copy_bytes, stall_ms, phys_slots,
   logical_capacity, staging_slots, kernel_launches, host_decision_ms, ffn_ms, step_ms,
   preload_copies, d2h_bytes, ffn_bytes (routed expert weight bytes streamed), ffn_launches,
   gate_wait_ms (GPU time spent waiting for the host's per-layer decision),
   fast_layers (layers whose routed FFN started from the device-side slot table,
   without waiting for the host), peer_copies, peer_bytes (swap-ins served by the
   peer-HBM tier), prefetch_admitted / prefetch_used / prefetch_wasted (experts admitted
   by a PREFETCH transfer; routed to by a later layer before eviction; evicted unused),
   bw_physical_Bps (EWMA, alpha 0.25, of the measured expert-copy rates; copy-stream
   events), bw_physical_transfers (copies folded into it), layer_kernel_steps (decode
   steps run on the persistent one-launch-per-layer kernel) */
int ef_engine_stats(ef_engine* e, double* out, int n);
/* device pointers for tests: 0 slab, 1 router weights, 2 shared, 3 logits, 4 sel, 5 wts,
   6 perm, 7 inv, 8 y, 9 x */
int ef_engine_ptr(ef_engine* e, int which, void** out);
/* export this engine's peer pool (allocated on its own device: export-only mode, or
   the same-device test mode) as a 64-byte cudaIpcMemHandle_t plus the pool's layout
   hash (expert bytes + global ids), for the engine of another process to open
   through ef_engine_cfg.peer_ipc_handle / peer_ipc_layout_hash */
int ef_engine_peer_pool_handle(ef_engine* e, void* handle64, uint64_t* layout_hash);
/* routing log entry `index` (one per executed layer, in order): R scored router
   matrices of logits [R][B][M] fp32, sel [B][k], cache-aware bias mask.  Pass
   null buffers to query sizes; *n_entries = log length. */
int ef_engine_routing_log(ef_engine* e, int64_t index, float* logits, int64_t max_logits,
                          int32_t* sel, int64_t max_sel, int32_t* R, int32_t* B,
                          uint64_t* mask_lo, uint64_t* mask_hi, int64_t* n_entries);
/* routing-log recording between steps: 0 off, 1 logits + selection + router input x
   (ef_engine_cfg.record_routing = 1 at creation), 2 logits + selection only (no device
   copy on the step's path); entries append to the log */
int ef_engine_set_record(ef_engine* e, int32_t mode);
/* a fresh scheduler (policy / logical clock of `sim`, same shape) and cache-aware
   routing bias on the same slab, weights and host store: every slot is emptied, the
   routing log cleared; physical counters keep accumulating */
int ef_engine_reset(ef_engine* e, const ef_sim_cfg* sim, float routing_bias);
/* the router input x_l [B][d] fp32 of routing log entry `index`, as the GPU
   computed it (copied off the device when the layer was decided), and the token
   count the cache-aware bias mask's top-up rule used (0: prefill).  Null x
   queries *n_x.  For parity checks of every scored router row. */
int ef_engine_routing_x(ef_engine* e, int64_t index, float* x, int64_t max_x, int64_t* n_x,
                        int32_t* mask_tokens);
/* physical slot of (layer, expert) or -1 */
int ef_engine_slot_of(ef_engine* e, int32_t layer, int32_t expert, int32_t* slot);

#ifdef __cplusplus
}
#endif
#endif /* EXPERTFLOW_H */
