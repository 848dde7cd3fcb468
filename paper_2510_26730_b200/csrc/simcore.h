// simcore.h — C++17 host runtime of the ExpertFlow decision path.
//
// B200-native redesign of the reference's single-threaded Python scheduler
// (/root/reference/pkg/src/moesim/{scheduler,memory,engine}.py):
//   * ExpertCache: O(1) two-tier LRU with intrusive per-tier lists ordered by
//     touch sequence (memory.py:28-156), plus event log.
//   * TransferQueue / BandwidthEstimator (memory.py:169-236).
//   * prediction ladder + LRU prediction cache (scheduler.py:194-309).
//   * Stepper: the per-layer loop of engine.py:566-659 on a logical
//     integer-ns clock, steppable per layer and persistent across tokens,
//     with an Observer hook the physical engine uses to mirror transfer
//     starts / admissions / evictions onto HBM slots and copy streams.
// All floating-point arithmetic follows the reference's fp64 operation order
// (compiled with -ffp-contract=off) so decisions are bit-exact.
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <functional>
#include <vector>

namespace ef {

constexpr int64_t kNsPerSec = 1000000000LL;
constexpr double kCumEps = 1e-9;  // scheduler.py:24

struct ValueError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline uint64_t eid_key(int32_t layer, int32_t expert) {
  return (uint64_t(uint32_t(layer)) << 32) | uint32_t(expert);
}
inline int32_t eid_layer(uint64_t k) { return int32_t(k >> 32); }
inline int32_t eid_expert(uint64_t k) { return int32_t(k & 0xffffffffu); }

// ---------------------------------------------------------------- primitives
std::vector<int> desc_order(const double* p, int m);
int expected_expert_count(const double* p, int m, double thr);
std::vector<int> top_experts(const double* p, int m, int count);
int64_t swap_in_latency(int64_t n, int64_t size, int64_t bw);
int compute_step_int(int64_t n_e, int64_t size, int64_t bw, int64_t layer_ns, int lo, int hi);
int compute_step_float(int64_t n_e, int64_t size, double bw, int64_t layer_ns, int lo, int hi);
// correctly rounded double of num/den for non-negative 128-bit num, den > 0
double exact_div(unsigned __int128 num, uint64_t den);

struct StepState {
  int current = 1, max_step = 1, min_step = 1, stall_count = 0, overfetch_count = 0,
      stall_threshold = 3, overfetch_threshold = 3;
  void validate() const;
  void on_stall();
  void on_overfetch();
};

// ---------------------------------------------------------------- cache
enum Tier : int { kLow = 0, kHigh = 1 };
enum CacheEv : int { kEvMiss = 0, kEvHit = 1, kEvAdmit = 2, kEvEvict = 3 };

struct CacheEvent {
  int64_t now;
  int kind;
  uint64_t key;
};

class ExpertCache {
 public:
  ExpertCache(int64_t capacity_bytes, int64_t expert_size, bool record_events);
  bool contains(uint64_t k) const { return nodes_.count(k) != 0; }
  size_t size() const { return nodes_.size(); }
  int64_t capacity() const { return capacity_; }
  bool access(uint64_t k, int64_t now);
  // returns victims in eviction order
  std::vector<uint64_t> admit(uint64_t k, int tier, int64_t now);
  void reassign_tiers(const std::vector<uint64_t>& predicted_sorted, int64_t window, int64_t now);
  int tier_of(uint64_t k) const;  // -1 absent
  int64_t last_access(uint64_t k) const;
  std::vector<uint64_t> resident_sorted() const;
  int64_t hits = 0, misses = 0, admissions = 0, evictions = 0;
  bool recording() const { return record_; }
  const std::vector<CacheEvent>& events() const { return events_; }

 private:
  struct Node {
    uint64_t key;
    int tier;
    int64_t touch, last;
    Node *prev = nullptr, *next = nullptr;
  };
  struct List {
    Node *head = nullptr, *tail = nullptr;
  };
  void unlink(Node* n);
  void append(Node* n, int tier);
  void log(int64_t now, int kind, uint64_t k) {
    if (record_) events_.push_back({now, kind, k});
  }
  int64_t capacity_;
  int64_t seq_ = 0;
  bool record_;
  List lists_[2];
  // nodes live in pooled chunks (locality for the tier walks of
  // reassign_tiers), recycled through a free list
  static constexpr int kChunk = 1024;
  std::vector<std::unique_ptr<Node[]>> chunks_;
  std::vector<Node*> free_;
  std::vector<Node*> order_;  // reassign_tiers scratch
  Node* alloc_node();
  std::unordered_map<uint64_t, Node*> nodes_;
  std::vector<CacheEvent> events_;
};

// ---------------------------------------------------------------- queue / bw
struct TransferRequest {
  uint64_t key;
  int prio;
  int64_t seq;
};
class TransferQueue {
 public:
  TransferRequest enqueue(uint64_t k, int prio);
  bool next(TransferRequest* out);
  size_t size() const { return heap_.size(); }

 private:
  std::vector<TransferRequest> heap_;
  int64_t seq_ = 0;
};

class BandwidthEstimator {
 public:
  BandwidthEstimator(bool has_initial, double initial, double alpha);
  double observe(int64_t bytes, int64_t ns);
  double estimate() const;

 private:
  double alpha_, est_ = 0.0;
  bool has_est_, observed_ = false;
};

// ---------------------------------------------------------------- prediction
using Blob = std::vector<int64_t>;
class PredictionCache {
 public:
  explicit PredictionCache(int capacity);
  const Blob* get(const std::vector<int64_t>& tokens, int64_t layer, int64_t step);
  void put(const std::vector<int64_t>& tokens, int64_t layer, int64_t step, Blob v);
  int64_t hits = 0, misses = 0;
  size_t size() const { return map_.size(); }

 private:
  struct Key {
    std::vector<int64_t> tokens;
    int64_t layer, step;
    bool operator==(const Key& o) const {
      return layer == o.layer && step == o.step && tokens == o.tokens;
    }
  };
  struct KeyHash {
    size_t operator()(const Key& k) const;
  };
  int capacity_;
  std::list<std::pair<Key, Blob>> lru_;  // front = least recent
  std::unordered_map<Key, std::list<std::pair<Key, Blob>>::iterator, KeyHash> map_;
};

struct Forest {
  int n_trees = 0, feature_len = 0, num_outputs = 0;
  bool residual = false;
  std::vector<int64_t> tree_off;
  std::vector<int32_t> feature, left, right;
  std::vector<double> threshold, value;
  void predict(const double* x, const double* baseline, double* out) const;
};

void inference_features(const double* table, int64_t vocab, int embed_dim, int L, int M,
                        const std::vector<int64_t>& tokens, int step, int target,
                        const std::map<int, std::vector<int>>& history, double* out);

// Plug points of the ladder (scheduler.py:238, :261-262).
struct LadderHooks {
  virtual ~LadderHooks() = default;
  virtual bool has_pregate() const = 0;
  virtual void pregate(int layer, int h, double* out) = 0;  // fp64 [M]
  virtual bool has_forest() const = 0;
  virtual void forest_scores(const double* feats, int nfeat, const double* baseline,
                             double* out) = 0;
  virtual int forest_feature_len() const = 0;
  // features: pooled embedding etc. (predictor.py:113-128)
  virtual void features(const std::vector<int64_t>& tokens, int step, int target,
                        const std::map<int, std::vector<int>>& hist, double* out) = 0;
};

using Horizon = std::vector<std::pair<int, std::vector<int>>>;
Blob encode_horizon(const Horizon& h);
Horizon decode_horizon(const Blob& b);

Horizon predict_experts(LadderHooks& hooks, PredictionCache& cache,
                        const std::vector<int64_t>& tokens, int layer, int step,
                        const double* router_probs, int M, int top_k, double cum_threshold,
                        const std::map<int, std::vector<int>>& known);

// ---------------------------------------------------------------- stepper
struct Policy {
  int strategy = 0;   // 0 static 1 reactive 2 fixed_interval 3 adaptive
  int predictor = 0;  // 0 none 1 pregate 2 forest 3 oracle
  int interval = 0;
  bool cache_aware_routing = false, preload = false;
  double cum_threshold = 0.9;
  int stall_threshold = 3, overfetch_threshold = 3, min_step = 1, max_step = -1,
      recent_window = -1, prediction_cache_capacity = 4096;
  uint64_t seed = 0;
};

struct SimConfig {
  int L = 1, M = 1, top_k = 1;
  int64_t expert_size = 1, link_bw = 1, device_memory = 1, layer_ns = 1;
  bool emit_events = false;
  bool bw_feedback = false;  // ef_sim_cfg.bw_feedback
  Policy policy;
};

// Per-layer router output as the scheduler sees it (workload.py:161-179).
struct LayerRouting {
  std::vector<double> gate;                  // fp64 batch gate [M]
  std::vector<int> actual;                   // ascending union
  std::vector<std::vector<int>> group_actual;  // per group, ascending
};

struct TokenInput {
  std::vector<int64_t> tokens;
  std::vector<int64_t> group_sizes;
  // routing for all L layers (trace-driven), or filled layer by layer
  std::vector<LayerRouting> layers;
};

// Physical mirror hooks (all optional).
struct Observer {
  virtual ~Observer() = default;
  virtual void on_transfer_start(uint64_t key, int prio) {}
  virtual void on_transfer_end(uint64_t key) {}  // admitted (HIGH) right after
  virtual void on_admit(uint64_t key) {}
  virtual void on_evict(uint64_t key) {}
  virtual void on_preload(uint64_t key) {}
  virtual void on_group_run(int layer, const std::vector<uint64_t>& demand) {}
};

struct SimEventRec {
  int64_t time;
  int kind;
  int64_t seq;
  std::string detail;
};
enum SimEv { kTransferStart = 0, kTransferEnd, kPrefetchIssue, kStall, kOverfetch, kLayerStart,
             kLayerEnd };

struct LayerRecord {
  int layer;
  int64_t start_ns, end_ns, stall_ns;
  int step;
  std::vector<int> predicted, actual;
  int demand_misses;
};
struct SampleRec {
  std::vector<int64_t> tokens;
  int layer;
  std::vector<int> predicted, actual;
  int step;
};

struct Metrics {
  int64_t total_time_ns = 0, compute_ns = 0, waiting_ns = 0, cache_miss_ns = 0, prefetch_ns = 0,
          cold_start_ns = 0, hits = 0, misses = 0, admissions = 0, evictions = 0,
          stall_events = 0, overfetch_events = 0, prediction_cache_hits = 0,
          prediction_cache_misses = 0, final_step = 0, n_selected = 0, n_total = 0;
  double bandwidth_estimate = 0.0;
};

class Stepper {
 public:
  Stepper(const SimConfig& cfg, LadderHooks* hooks);
  // Token API: begin_token(tokens, group_sizes, gate0, actual0) must come
  // after layer 0's routing is known; then for l in 0..L-1:
  //   begin_layer(l); run_layer(l, routing[l]); then end_token().
  void begin_token(const std::vector<int64_t>& tokens, const std::vector<int64_t>& group_sizes,
                   const LayerRouting& layer0);
  void begin_layer(int l);
  void run_layer(int l, const LayerRouting& r);
  void end_token();
  // Convenience: whole token from a trace (simulate()).
  void run_token(const TokenInput& in);

  // horizon (clipped) that layer l's boundary will issue, 0 if none;
  // valid after end of layer l-1 (or begin_token for l = 0)
  int planned_horizon(int l) const;
  bool resident(int32_t layer, int32_t expert) const {
    return cache_.contains(eid_key(layer, expert));
  }
  const ExpertCache& cache() const { return cache_; }
  Metrics metrics() const;
  const std::vector<std::pair<int, int>>& step_history() const { return step_history_; }
  const std::vector<LayerRecord>& layer_records() const { return records_; }
  const std::vector<SampleRec>& samples() const { return samples_; }
  std::vector<SimEventRec> sorted_events() const;
  void set_observer(Observer* o) { obs_ = o; }
  // Bandwidth feedback into S ("observed transfer times update
  // the bandwidth estimate C_s, informing subsequent skip-distance
  // calculations"; the reference computes S once, engine.py:545-556, and never
  // feeds its EWMA back — SURVEY Appendix A Q2).  When a source is set, every
  // adaptive boundary re-bases the step: S = compute_step(N_e(this layer's
  // gate), E_s, source(), T_l, min, max), then stall / overfetch feedback
  // continues from it.  Off by default (parity mode).
  void set_bw_feedback(std::function<double()> src) { bw_src_ = std::move(src); }
  double logical_bw_estimate() const { return estimator_.estimate(); }
  void set_oracle_future(const std::vector<LayerRouting>* f) { oracle_future_ = f; }
  int64_t clock() const { return clock_; }
  int64_t per_expert_ns() const { return per_expert_ns_; }
  int64_t layer_ns() const { return cfg_.layer_ns; }
  int step_in_effect() const;
  int tokens_run() const { return tokens_run_; }

 private:
  std::vector<uint64_t> hot_scratch_;
  std::function<double()> bw_src_;
  struct Inflight {
    uint64_t key;
    int prio;
    int bucket;  // 0 cold 1 miss 2 prefetch
    int64_t start, end;
  };
  struct HorizonRec {
    int first;
    int64_t issue_ns;
    std::set<uint64_t> missing;
    int64_t last_arrival;
    bool checked = false;
  };
  void emit(int64_t t, int kind, std::string detail);
  void request(uint64_t k, int prio, int bucket);
  void pump(int64_t t);
  void advance_to(int64_t t);
  int64_t wait_until_resident(const std::vector<uint64_t>& req, int64_t t);
  void consume(const std::vector<uint64_t>& req);
  int bucket_now() const { return now_ == 0 ? 0 : 1; }
  Horizon predict_targets(int layer, int step);
  void issue_horizon(int layer, int step);
  void boundary(int layer);
  void check_overfetch(int layer, int64_t first_exec);

  SimConfig cfg_;
  LadderHooks* hooks_;
  Observer* obs_ = nullptr;
  const std::vector<LayerRouting>* oracle_future_ = nullptr;
  int max_step_;
  int64_t per_expert_ns_;
  ExpertCache cache_;
  TransferQueue queue_;
  std::unordered_map<uint64_t, TransferRequest> queued_;
  std::unordered_map<int64_t, int> bucket_of_;
  bool has_inflight_ = false;
  Inflight inflight_{};
  int64_t link_free_ = 0;
  BandwidthEstimator estimator_;
  PredictionCache pcache_;
  Metrics m_;
  int64_t n_selected_ = 0, n_total_ = 0;
  std::vector<SimEventRec> events_;
  int64_t event_seq_ = 0;
  int64_t clock_ = 0, now_ = 0;
  bool has_state_ = false;
  StepState state_;
  std::unordered_map<uint64_t, std::deque<int64_t>> unconsumed_;
  int64_t consumed_ns_ = 0;
  int tokens_run_ = 0;
  int64_t miss_guard_ = 0, miss_guard_limit_;
  // per token
  std::vector<int64_t> tokens_, group_sizes_;
  std::vector<LayerRouting> seen_;  // routing of executed layers this token
  std::map<int, std::pair<std::vector<int>, int>> predicted_;
  std::vector<std::unique_ptr<HorizonRec>> horizons_;
  std::unordered_map<uint64_t, HorizonRec*> horizon_by_expert_;
  int next_boundary_ = 0;
  // per layer (begin_layer -> run_layer)
  int64_t t0_ = 0;
  std::vector<std::pair<int, int>> step_history_;
  std::vector<LayerRecord> records_;
  std::vector<SampleRec> samples_;
};

}  // namespace ef
