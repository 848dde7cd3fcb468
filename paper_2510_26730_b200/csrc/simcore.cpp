// simcore.cpp — decision path of the ExpertFlow hot path (see simcore.h).
// Reference citations are relative to /root/reference/pkg/src/moesim.
#include "simcore.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <numeric>

namespace ef {

// =================================================================== primitives

std::vector<int> desc_order(const double* p, int m) {
  // np.argsort(-p, kind="stable") (workload.py:184, scheduler.py:47, :59)
  std::vector<int> idx(m);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [p](int a, int b) { return p[a] > p[b]; });
  return idx;
}

int expected_expert_count(const double* p, int m, double thr) {
  // scheduler.py:36-53
  if (!(thr > 0.0 && thr <= 1.0)) throw ValueError("cum_threshold must lie in (0, 1]");
  std::vector<int> order = desc_order(p, m);
  double total = 0.0;
  for (int c = 0; c < m; ++c) {
    total += p[order[c]];
    if (total >= thr - kCumEps) return c + 1;
  }
  return m;
}

std::vector<int> top_experts(const double* p, int m, int count) {
  // scheduler.py:56-60
  std::vector<int> order = desc_order(p, m);
  if (count < 0) count = 0;
  if (count > m) count = m;
  std::vector<int> out(order.begin(), order.begin() + count);
  std::sort(out.begin(), out.end());
  return out;
}

int64_t swap_in_latency(int64_t n, int64_t size, int64_t bw) {
  // scheduler.py:63-74
  if (n < 0) throw ValueError("num_experts must be >= 0");
  if (bw < 1) throw ValueError("bandwidth must be >= 1 byte/s");
  __int128 numer = (__int128)n * size * kNsPerSec;
  __int128 q = (numer + bw - 1) / bw;
  return (int64_t)q;
}

static void check_step_args(int64_t n_e, int64_t layer_ns, int lo, int hi) {
  if (layer_ns < 1) throw ValueError("layer_compute_ns must be >= 1");
  if (!(1 <= lo && lo <= hi)) throw ValueError("bad step bounds");
  if (n_e < 0) throw ValueError("num_experts must be >= 0");
}

int compute_step_int(int64_t n_e, int64_t size, int64_t bw, int64_t layer_ns, int lo, int hi) {
  // scheduler.py:96-101 (exact rational ceiling)
  check_step_args(n_e, layer_ns, lo, hi);
  if (bw < 1) throw ValueError("bandwidth must be >= 1 byte/s");
  unsigned __int128 numer = (unsigned __int128)n_e * (uint64_t)size * (uint64_t)kNsPerSec;
  unsigned __int128 den = (unsigned __int128)(uint64_t)bw * (uint64_t)layer_ns;
  unsigned __int128 raw = (numer + den - 1) / den;
  if (raw > (unsigned __int128)hi) return hi;
  return std::max(lo, (int)raw);
}

int compute_step_float(int64_t n_e, int64_t size, double bw, int64_t layer_ns, int lo, int hi) {
  // scheduler.py:102-105: math.ceil(int / (float * int)).  Python converts the
  // integer numerator to the nearest double; __floattidf rounds the same way.
  check_step_args(n_e, layer_ns, lo, hi);
  if (!(bw > 0)) throw ValueError("bandwidth must be positive");
  __int128 numer = (__int128)n_e * size * kNsPerSec;
  double q = (double)numer / (bw * (double)layer_ns);
  double raw = std::ceil(q);
  if (raw > (double)hi) return hi;
  return std::max(lo, (int)raw);
}

static int bitlen128(unsigned __int128 v) {
  int n = 0;
  while (v) {
    ++n;
    v >>= 1;
  }
  return n;
}

double exact_div(unsigned __int128 num, uint64_t den) {
  // Python's int / int: the correctly rounded quotient (memory.py:230).
  if (num == 0) return 0.0;
  int s = std::max(0, 64 + bitlen128(den) - bitlen128(num));
  unsigned __int128 sh = num << s;
  unsigned __int128 q = sh / den, r = sh % den;
  if (r) q |= 1;  // sticky bit below the rounding position (q has >= 64 bits)
  return std::ldexp((double)q, -s);
}

void StepState::validate() const {
  // scheduler.py:125-139
  if (!(1 <= min_step && min_step <= max_step)) throw ValueError("bad step bounds");
  if (!(min_step <= current && current <= max_step)) throw ValueError("step outside bounds");
  if (stall_threshold < 1 || overfetch_threshold < 1)
    throw ValueError("feedback thresholds must be >= 1");
  if (!(0 <= stall_count && stall_count < stall_threshold))
    throw ValueError("stall_count out of range");
  if (!(0 <= overfetch_count && overfetch_count < overfetch_threshold))
    throw ValueError("overfetch_count out of range");
}

void StepState::on_stall() {  // scheduler.py:142-151
  if (++stall_count >= stall_threshold) {
    stall_count = 0;
    current = std::min(current + 1, max_step);
  }
}

void StepState::on_overfetch() {  // scheduler.py:154-163
  if (++overfetch_count >= overfetch_threshold) {
    overfetch_count = 0;
    current = std::max(current - 1, min_step);
  }
}

// =================================================================== cache

ExpertCache::ExpertCache(int64_t capacity_bytes, int64_t expert_size, bool record_events)
    : record_(record_events) {
  // memory.py:36-61
  if (expert_size < 1) throw ValueError("expert_size_bytes must be >= 1");
  capacity_ = capacity_bytes / expert_size;
  if (capacity_ < 1) throw ValueError("capacity cannot hold one expert");
}

ExpertCache::Node* ExpertCache::alloc_node() {
  if (free_.empty()) {
    chunks_.emplace_back(new Node[kChunk]);
    Node* c = chunks_.back().get();
    for (int i = kChunk - 1; i >= 0; --i) free_.push_back(c + i);
  }
  Node* n = free_.back();
  free_.pop_back();
  *n = Node{};
  return n;
}

void ExpertCache::unlink(Node* n) {
  List& l = lists_[n->tier];
  (n->prev ? n->prev->next : l.head) = n->next;
  (n->next ? n->next->prev : l.tail) = n->prev;
  n->prev = n->next = nullptr;
}

void ExpertCache::append(Node* n, int tier) {
  List& l = lists_[tier];
  n->tier = tier;
  n->prev = l.tail;
  n->next = nullptr;
  (l.tail ? l.tail->next : l.head) = n;
  l.tail = n;
}

bool ExpertCache::access(uint64_t k, int64_t now) {
  // memory.py:94-104
  auto it = nodes_.find(k);
  if (it == nodes_.end()) {
    ++misses;
    log(now, kEvMiss, k);
    return false;
  }
  Node* n = it->second;
  unlink(n);
  append(n, kHigh);
  n->touch = seq_++;
  n->last = now;
  ++hits;
  log(now, kEvHit, k);
  return true;
}

std::vector<uint64_t> ExpertCache::admit(uint64_t k, int tier, int64_t now) {
  // memory.py:106-129
  if (tier != kLow && tier != kHigh) throw ValueError("unknown tier");
  auto it = nodes_.find(k);
  if (it != nodes_.end()) {  // re-admission only re-places
    Node* n = it->second;
    unlink(n);
    append(n, tier);
    n->touch = seq_++;
    n->last = now;
    return {};
  }
  std::vector<uint64_t> victims;
  while ((int64_t)nodes_.size() >= capacity_) {
    Node* v = lists_[kLow].head ? lists_[kLow].head : lists_[kHigh].head;
    uint64_t vk = v->key;
    unlink(v);
    nodes_.erase(vk);
    free_.push_back(v);
    ++evictions;
    log(now, kEvEvict, vk);
    victims.push_back(vk);
  }
  Node* node = alloc_node();
  node->key = k;
  node->touch = seq_++;
  node->last = now;
  append(node, tier);
  nodes_.emplace(k, node);
  ++admissions;
  log(now, kEvAdmit, k);
  return victims;
}

void ExpertCache::reassign_tiers(const std::vector<uint64_t>& predicted, int64_t window,
                                 int64_t now) {
  // predicted: sorted, unique keys
  // memory.py:137-156: global touch order, then split by the new tier.
  if (window < 0) throw ValueError("recent_window must be >= 0");
  std::vector<Node*>& order = order_;
  order.clear();
  order.reserve(nodes_.size());
  Node* a = lists_[kLow].head;
  Node* b = lists_[kHigh].head;
  while (a || b) {
    if (!b || (a && a->touch < b->touch)) {
      order.push_back(a);
      a = a->next;
    } else {
      order.push_back(b);
      b = b->next;
    }
  }
  lists_[kLow] = List{};
  lists_[kHigh] = List{};
  for (Node* n : order) {
    bool hot = (now - n->last < window) ||
               std::binary_search(predicted.begin(), predicted.end(), n->key);
    n->prev = n->next = nullptr;
    append(n, hot ? kHigh : kLow);
  }
}

int ExpertCache::tier_of(uint64_t k) const {
  auto it = nodes_.find(k);
  return it == nodes_.end() ? -1 : it->second->tier;
}

int64_t ExpertCache::last_access(uint64_t k) const {
  auto it = nodes_.find(k);
  return it == nodes_.end() ? -1 : it->second->last;
}

std::vector<uint64_t> ExpertCache::resident_sorted() const {
  std::vector<uint64_t> out;
  out.reserve(nodes_.size());
  for (auto& kv : nodes_) out.push_back(kv.first);
  std::sort(out.begin(), out.end());
  return out;
}

// =================================================================== queue / bw

static bool req_less(const TransferRequest& a, const TransferRequest& b) {
  return a.prio != b.prio ? a.prio < b.prio : a.seq < b.seq;
}

TransferRequest TransferQueue::enqueue(uint64_t k, int prio) {
  // memory.py:192-195
  TransferRequest r{k, prio, seq_++};
  heap_.push_back(r);
  std::push_heap(heap_.begin(), heap_.end(),
                 [](const TransferRequest& a, const TransferRequest& b) { return req_less(b, a); });
  return r;
}

bool TransferQueue::next(TransferRequest* out) {
  // memory.py:197-200
  if (heap_.empty()) return false;
  std::pop_heap(heap_.begin(), heap_.end(),
                [](const TransferRequest& a, const TransferRequest& b) { return req_less(b, a); });
  *out = heap_.back();
  heap_.pop_back();
  return true;
}

BandwidthEstimator::BandwidthEstimator(bool has_initial, double initial, double alpha)
    : alpha_(alpha), est_(initial), has_est_(has_initial) {
  if (!(alpha > 0.0 && alpha <= 1.0)) throw ValueError("alpha must lie in (0, 1]");
}

double BandwidthEstimator::observe(int64_t bytes, int64_t ns) {
  // memory.py:226-236
  if (ns < 1) throw ValueError("elapsed_ns must be >= 1");
  if (bytes < 0) throw ValueError("transferred_bytes must be >= 0");
  double rate = exact_div((unsigned __int128)(uint64_t)bytes * (uint64_t)kNsPerSec, (uint64_t)ns);
  if (!observed_) {
    est_ = rate;
    observed_ = true;
    has_est_ = true;
  } else {
    double a = alpha_ * rate;
    double b = (1.0 - alpha_) * est_;
    est_ = a + b;
  }
  return est_;
}

double BandwidthEstimator::estimate() const {
  if (!has_est_) throw RuntimeErr("no estimate: no prior and nothing observed yet");
  return est_;
}

// =================================================================== prediction

size_t PredictionCache::KeyHash::operator()(const Key& k) const {
  uint64_t h = 0x9E3779B97F4A7C15ULL ^ (uint64_t)k.layer * 0x100000001B3ULL ^ (uint64_t)k.step;
  for (int64_t t : k.tokens) h = (h ^ (uint64_t)t) * 0x100000001B3ULL + 0x9E37;
  return (size_t)h;
}

PredictionCache::PredictionCache(int capacity) : capacity_(capacity) {
  if (capacity < 1) throw ValueError("capacity must be >= 1");
}

const Blob* PredictionCache::get(const std::vector<int64_t>& tokens, int64_t layer, int64_t step) {
  // scheduler.py:206-213
  auto it = map_.find(Key{tokens, layer, step});
  if (it == map_.end()) {
    ++misses;
    return nullptr;
  }
  lru_.splice(lru_.end(), lru_, it->second);
  ++hits;
  return &it->second->second;
}

void PredictionCache::put(const std::vector<int64_t>& tokens, int64_t layer, int64_t step,
                          Blob v) {
  // scheduler.py:215-221
  Key key{tokens, layer, step};
  auto it = map_.find(key);
  if (it != map_.end()) {
    it->second->second = std::move(v);
    lru_.splice(lru_.end(), lru_, it->second);
  } else {
    lru_.emplace_back(key, std::move(v));
    map_.emplace(std::move(key), std::prev(lru_.end()));
  }
  while ((int)map_.size() > capacity_) {
    map_.erase(lru_.front().first);
    lru_.pop_front();
  }
}

void Forest::predict(const double* x, const double* baseline, double* out) const {
  // predictor.py:327-349 (tree walk :225-232)
  std::vector<double> acc(num_outputs, 0.0);
  for (int t = 0; t < n_trees; ++t) {
    int64_t base = tree_off[t];
    int64_t n = 0;
    while (feature[base + n] != -1) {
      n = (x[feature[base + n]] <= threshold[base + n]) ? left[base + n] : right[base + n];
    }
    const double* leaf = &value[(base + n) * num_outputs];
    for (int j = 0; j < num_outputs; ++j) acc[j] += leaf[j];
  }
  for (int j = 0; j < num_outputs; ++j) acc[j] /= (double)n_trees;
  if (residual) {
    if (!baseline) throw ValueError("residual model needs a baseline distribution");
    for (int j = 0; j < num_outputs; ++j) out[j] = baseline[j] + acc[j];
  } else {
    for (int j = 0; j < num_outputs; ++j) out[j] = acc[j];
  }
}

void inference_features(const double* table, int64_t vocab, int embed_dim, int L, int M,
                        const std::vector<int64_t>& tokens, int step, int target,
                        const std::map<int, std::vector<int>>& history, double* out) {
  // predictor.py:76-128: [pooled embedding, step, target, history bits]
  if (tokens.empty()) throw ValueError("no tokens");
  for (int j = 0; j < embed_dim; ++j) out[j] = 0.0;
  for (int64_t t : tokens) {
    if (t < 0 || t >= vocab) throw ValueError("token id out of range for the embedding table");
    const double* row = table + t * embed_dim;
    for (int j = 0; j < embed_dim; ++j) out[j] += row[j];
  }
  for (int j = 0; j < embed_dim; ++j) out[j] /= (double)tokens.size();
  out[embed_dim] = (double)step;
  out[embed_dim + 1] = (double)target;
  double* bits = out + embed_dim + 2;
  std::fill(bits, bits + (int64_t)L * M, 0.0);
  for (auto& kv : history) {
    int layer = kv.first;
    if (layer >= 0 && layer < target && target - 1 - layer < L) {
      for (int e : kv.second) bits[(int64_t)(target - 1 - layer) * M + e] = 1.0;
    }
  }
}

Blob encode_horizon(const Horizon& h) {
  Blob b;
  b.push_back((int64_t)h.size());
  for (auto& t : h) {
    b.push_back(t.first);
    b.push_back((int64_t)t.second.size());
    for (int e : t.second) b.push_back(e);
  }
  return b;
}

Horizon decode_horizon(const Blob& b) {
  Horizon h;
  size_t p = 0;
  int64_t n = b.at(p++);
  for (int64_t i = 0; i < n; ++i) {
    int target = (int)b.at(p++);
    int64_t c = b.at(p++);
    std::vector<int> ex;
    for (int64_t j = 0; j < c; ++j) ex.push_back((int)b.at(p++));
    h.emplace_back(target, std::move(ex));
  }
  return h;
}

// numpy's pairwise float64 sum of a contiguous vector (numpy
// umath/loops_utils.h pairwise_sum), used by ``mass.sum()`` at scheduler.py:285.
static double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;  // numpy starts from -0.0 / 0.0; identical for n >= 1 here
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

Horizon predict_experts(LadderHooks& hooks, PredictionCache& cache,
                        const std::vector<int64_t>& tokens, int layer, int step,
                        const double* router_probs, int M, int top_k, double cum_threshold,
                        const std::map<int, std::vector<int>>& known) {
  // scheduler.py:247-309
  if (const Blob* hit = cache.get(tokens, layer, step)) return decode_horizon(*hit);
  Horizon out;
  std::map<int, std::vector<int>> prev = known;
  std::vector<double> pg(M), scores(M), mass(M);
  std::vector<double> feats;
  for (int h = 1; h <= step; ++h) {
    int target = layer + h;
    bool have_pg = hooks.has_pregate();
    if (have_pg) hooks.pregate(layer, h, pg.data());
    std::vector<int> chosen;
    if (hooks.has_forest()) {
      feats.assign(hooks.forest_feature_len(), 0.0);
      hooks.features(tokens, step, target, prev, feats.data());
      hooks.forest_scores(feats.data(), (int)feats.size(), have_pg ? pg.data() : nullptr,
                          scores.data());
      for (int e = 0; e < M; ++e) mass[e] = scores[e] > 0.0 ? scores[e] : 0.0;
      double total = np_pairwise_sum(mass.data(), M);
      int n_sel;
      if (total > 0) {
        std::vector<double> norm(M);
        for (int e = 0; e < M; ++e) norm[e] = mass[e] / total;
        n_sel = expected_expert_count(norm.data(), M, cum_threshold);
      } else if (have_pg) {
        n_sel = expected_expert_count(pg.data(), M, cum_threshold);
      } else {
        n_sel = expected_expert_count(router_probs, M, cum_threshold);
      }
      chosen = top_experts(scores.data(), M, n_sel);
    } else if (have_pg) {
      chosen = top_experts(pg.data(), M, expected_expert_count(pg.data(), M, cum_threshold));
    } else {
      if (top_k < 1) throw ValueError("fallback prediction needs model for top_k");
      chosen = top_experts(router_probs, M, top_k);
    }
    out.emplace_back(target, chosen);
    prev[target] = chosen;
  }
  cache.put(tokens, layer, step, encode_horizon(out));
  return out;
}

// =================================================================== stepper

static const char* kPrioName[3] = {"miss", "prefetch", "evict"};

Stepper::Stepper(const SimConfig& cfg, LadderHooks* hooks)
    : cfg_(cfg),
      hooks_(hooks),
      max_step_(cfg.policy.max_step >= 0 ? cfg.policy.max_step : std::max(1, cfg.L - 1)),
      per_expert_ns_(swap_in_latency(1, cfg.expert_size, cfg.link_bw)),  // engine.py:266
      cache_(cfg.device_memory, cfg.expert_size, cfg.emit_events),
      estimator_(true, (double)cfg.link_bw, 0.25),                      // engine.py:278
      pcache_(cfg.policy.prediction_cache_capacity),
      miss_guard_limit_(16LL * cfg.L * cfg.M + 256) {                    // engine.py:299
  if (cfg.layer_ns < 1) throw ValueError("layer compute time rounds below 1 ns");
  const Policy& p = cfg.policy;
  if (p.strategy < 0 || p.strategy > 3) throw ValueError("unknown strategy");
  if (p.predictor < 0 || p.predictor > 3) throw ValueError("unknown predictor");
  if (p.strategy == 2 && p.interval < 1) throw ValueError("fixed_interval needs interval >= 1");
  if (p.strategy == 0 && p.predictor != 0) throw ValueError("static strategy takes no predictor");
  if (!(1 <= p.min_step && p.min_step <= max_step_)) throw ValueError("bad step bounds");
}

void Stepper::emit(int64_t t, int kind, std::string detail) {
  if (!cfg_.emit_events) return;
  events_.push_back({t, kind, event_seq_++, std::move(detail)});
}

void Stepper::request(uint64_t k, int prio, int bucket) {
  // engine.py:311-326
  if (cache_.contains(k)) return;
  if (has_inflight_ && inflight_.key == k) return;
  auto it = queued_.find(k);
  if (it != queued_.end() && prio >= it->second.prio) return;
  TransferRequest r = queue_.enqueue(k, prio);
  queued_[k] = r;
  bucket_of_[r.seq] = bucket;
  pump(clock_);
}

void Stepper::pump(int64_t t) {
  // engine.py:328-354
  while (!has_inflight_) {
    TransferRequest r;
    if (!queue_.next(&r)) return;
    auto it = queued_.find(r.key);
    if (it == queued_.end() || it->second.seq != r.seq) {  // superseded
      bucket_of_.erase(r.seq);
      continue;
    }
    queued_.erase(it);
    if (cache_.contains(r.key)) {
      bucket_of_.erase(r.seq);
      continue;
    }
    int64_t start = std::max(t, link_free_);
    int bucket = bucket_of_.at(r.seq);
    bucket_of_.erase(r.seq);
    inflight_ = Inflight{r.key, r.prio, bucket, start, start + per_expert_ns_};
    has_inflight_ = true;
    if (obs_) obs_->on_transfer_start(r.key, r.prio);
    if (cfg_.emit_events) {
      char buf[96];
      snprintf(buf, sizeof buf, "expert=%d:%d priority=%s", eid_layer(r.key), eid_expert(r.key),
               kPrioName[r.prio]);
      emit(start, kTransferStart, buf);
    }
  }
}

void Stepper::advance_to(int64_t t) {
  // engine.py:356-381
  while (has_inflight_ && inflight_.end <= t) {
    Inflight tr = inflight_;
    has_inflight_ = false;
    link_free_ = tr.end;
    int64_t dur = tr.end - tr.start;
    estimator_.observe(cfg_.expert_size, dur);
    if (obs_) obs_->on_transfer_end(tr.key);
    std::vector<uint64_t> victims = cache_.admit(tr.key, kHigh, now_);
    if (obs_) {
      for (uint64_t v : victims) obs_->on_evict(v);
      obs_->on_admit(tr.key);
    }
    unconsumed_[tr.key].push_back(dur);
    if (tr.bucket == 0)
      m_.cold_start_ns += dur;
    else if (tr.bucket == 1)
      m_.cache_miss_ns += dur;
    else
      m_.prefetch_ns += dur;
    auto hz = horizon_by_expert_.find(tr.key);
    if (hz != horizon_by_expert_.end() && hz->second->missing.count(tr.key)) {
      hz->second->missing.erase(tr.key);
      hz->second->last_arrival = std::max(hz->second->last_arrival, tr.end);
    }
    if (cfg_.emit_events) {
      char buf[64];
      snprintf(buf, sizeof buf, "expert=%d:%d", eid_layer(tr.key), eid_expert(tr.key));
      emit(tr.end, kTransferEnd, buf);
    }
    pump(tr.end);
  }
}

int64_t Stepper::wait_until_resident(const std::vector<uint64_t>& req, int64_t t) {
  // engine.py:383-402
  for (;;) {
    advance_to(t);
    std::vector<uint64_t> missing;
    for (uint64_t k : req)
      if (!cache_.contains(k)) missing.push_back(k);
    if (missing.empty()) return t;
    std::sort(missing.begin(), missing.end());
    for (uint64_t k : missing) {
      request(k, 0, bucket_now());
      ++miss_guard_;
    }
    if (miss_guard_ > miss_guard_limit_)
      throw RuntimeErr(
          "no forward progress: device memory too small to hold a routing group's experts "
          "alongside in-flight prefetches");
    if (!has_inflight_) pump(t);
    if (!has_inflight_) throw RuntimeErr("missing experts but idle link");
    t = std::max(t, inflight_.end);
  }
}

void Stepper::consume(const std::vector<uint64_t>& req) {
  // engine.py:404-408
  std::vector<uint64_t> s = req;
  std::sort(s.begin(), s.end());
  for (uint64_t k : s) {
    auto it = unconsumed_.find(k);
    if (it != unconsumed_.end() && !it->second.empty()) {
      consumed_ns_ += it->second.front();
      it->second.pop_front();
    }
  }
}

namespace {
struct NoHooks : LadderHooks {
  bool has_pregate() const override { return false; }
  void pregate(int, int, double*) override {}
  bool has_forest() const override { return false; }
  void forest_scores(const double*, int, const double*, double*) override {}
  int forest_feature_len() const override { return 0; }
  void features(const std::vector<int64_t>&, int, int, const std::map<int, std::vector<int>>&,
                double*) override {}
};
// Restricts the caller's hooks to what a policy's predictor may use
// (engine.py:420-428).
struct PolicyHooks : LadderHooks {
  LadderHooks* base;
  bool pregate_on, forest_on;
  bool has_pregate() const override { return pregate_on && base && base->has_pregate(); }
  void pregate(int l, int h, double* out) override { base->pregate(l, h, out); }
  bool has_forest() const override { return forest_on && base && base->has_forest(); }
  void forest_scores(const double* f, int n, const double* b, double* o) override {
    base->forest_scores(f, n, b, o);
  }
  int forest_feature_len() const override { return base->forest_feature_len(); }
  void features(const std::vector<int64_t>& t, int s, int tg,
                const std::map<int, std::vector<int>>& h, double* o) override {
    base->features(t, s, tg, h, o);
  }
};
}  // namespace

Horizon Stepper::predict_targets(int layer, int step) {
  // engine.py:412-449
  if (cfg_.policy.predictor == 3) {  // oracle
    if (!oracle_future_) throw ValueError("oracle predictor needs the trace's future routing");
    Horizon h;
    for (int t = layer + 1; t <= layer + step; ++t) h.emplace_back(t, (*oracle_future_)[t].actual);
    return h;
  }
  PolicyHooks ph;
  ph.base = hooks_;
  ph.pregate_on = cfg_.policy.predictor == 1 || cfg_.policy.predictor == 2;
  ph.forest_on = cfg_.policy.predictor == 2;
  if (ph.forest_on && !ph.has_forest()) throw ValueError("forest predictor needs a trained model");
  std::map<int, std::vector<int>> known;
  for (int x = 0; x <= layer; ++x) known[x] = seen_[x].actual;
  return predict_experts(ph, pcache_, tokens_, layer, step, seen_[layer].gate.data(), cfg_.M,
                         cfg_.top_k, cfg_.policy.cum_threshold, known);
}

void Stepper::issue_horizon(int layer, int step) {
  // engine.py:451-482
  step = std::min(step, cfg_.L - 1 - layer);
  if (step < 1) return;
  Horizon targets = predict_targets(layer, step);
  if (targets.empty()) return;
  auto hz = std::make_unique<HorizonRec>();
  hz->first = targets[0].first;
  hz->issue_ns = clock_;
  hz->last_arrival = clock_;
  for (auto& tg : targets) {
    predicted_[tg.first] = {tg.second, step};
    for (int e : tg.second) {
      uint64_t k = eid_key(tg.first, e);
      if (!cache_.contains(k)) {
        if (!queued_.count(k) && !(has_inflight_ && inflight_.key == k)) request(k, 1, 2);
        hz->missing.insert(k);
        horizon_by_expert_[k] = hz.get();
      }
    }
  }
  if (cfg_.emit_events) {
    char buf[96];
    snprintf(buf, sizeof buf, "layer=%d targets=%d..%d step=%d", layer, targets.front().first,
             targets.back().first, step);
    emit(clock_, kPrefetchIssue, buf);
  }
  horizons_.push_back(std::move(hz));
}

int Stepper::planned_horizon(int l) const {
  const Policy& p = cfg_.policy;
  int step = 0;
  if (p.strategy == 1)
    step = 1;
  else if (p.strategy == 2)
    step = (l % p.interval == 0) ? p.interval : 0;
  else if (p.strategy == 3)
    step = (l == next_boundary_ && has_state_) ? state_.current : 0;
  return std::max(0, std::min(step, cfg_.L - 1 - l));
}

void Stepper::boundary(int layer) {
  // engine.py:484-499
  const Policy& p = cfg_.policy;
  if (p.strategy == 0) return;
  if (p.strategy == 1) {
    issue_horizon(layer, 1);
  } else if (p.strategy == 2) {
    if (layer % p.interval == 0) issue_horizon(layer, p.interval);
  } else if (layer == next_boundary_) {
    if (bw_src_ && has_state_) {
      const Policy& pp = cfg_.policy;
      const int n_e = expected_expert_count(seen_[layer].gate.data(), cfg_.M, pp.cum_threshold);
      state_.current = compute_step_float(n_e, cfg_.expert_size, bw_src_(), cfg_.layer_ns,
                                          pp.min_step, max_step_);
    }
    int step = state_.current;
    issue_horizon(layer, step);
    next_boundary_ = layer + step;  // unclipped (Appendix A Q7)
  }
}

void Stepper::check_overfetch(int layer, int64_t first_exec) {
  // engine.py:501-517
  for (auto& hz : horizons_) {
    if (hz->first != layer || hz->checked) continue;
    hz->checked = true;
    if (!hz->missing.empty()) continue;
    int64_t margin = first_exec - hz->last_arrival;
    if (margin > cfg_.layer_ns) {
      ++m_.overfetch_events;
      if (cfg_.emit_events) {
        char buf[96];
        snprintf(buf, sizeof buf, "layer=%d margin_ns=%lld", layer, (long long)margin);
        emit(first_exec, kOverfetch, buf);
      }
      if (has_state_) state_.on_overfetch();
    }
  }
}

int Stepper::step_in_effect() const {
  // engine.py:532-541
  switch (cfg_.policy.strategy) {
    case 3:
      return state_.current;
    case 2:
      return cfg_.policy.interval;
    case 1:
      return 1;
    default:
      return 0;
  }
}

void Stepper::begin_token(const std::vector<int64_t>& tokens,
                          const std::vector<int64_t>& group_sizes, const LayerRouting& layer0) {
  tokens_ = tokens;
  group_sizes_ = group_sizes;
  miss_guard_ = 0;  // engine.py:299's guard covers one trace (one token); re-armed per token
  if (tokens_run_ == 0) {
    const Policy& p = cfg_.policy;
    if (p.strategy == 3) {  // engine.py:545-563
      int n_e = expected_expert_count(layer0.gate.data(), cfg_.M, p.cum_threshold);
      int s0 = compute_step_float(n_e, cfg_.expert_size, estimator_.estimate(), cfg_.layer_ns,
                                  p.min_step, max_step_);
      state_ = StepState{s0, max_step_, p.min_step, 0, 0, p.stall_threshold,
                         p.overfetch_threshold};
      state_.validate();
      has_state_ = true;
    }
    if (p.preload) {  // engine.py:521-530
      for (int e : layer0.actual) {
        uint64_t k = eid_key(0, e);
        std::vector<uint64_t> victims = cache_.admit(k, kHigh, 0);
        if (obs_) {
          for (uint64_t v : victims) obs_->on_evict(v);
          obs_->on_preload(k);
        }
      }
      m_.cold_start_ns =
          swap_in_latency((int64_t)layer0.actual.size(), cfg_.expert_size, cfg_.link_bw);
    }
  }
  predicted_.clear();
  horizons_.clear();
  horizon_by_expert_.clear();
  next_boundary_ = 0;
  seen_.clear();
}

void Stepper::begin_layer(int l) {
  // engine.py:567-571
  now_ = (int64_t)tokens_run_ * cfg_.L + l;
  t0_ = clock_;
  advance_to(t0_);
  if (cfg_.emit_events) emit(t0_, kLayerStart, "layer=" + std::to_string(l));
  step_history_.emplace_back(l, step_in_effect());
}

void Stepper::run_layer(int l, const LayerRouting& r) {
  // engine.py:573-659
  seen_.push_back(r);
  if ((int)seen_.size() != l + 1) throw ValueError("layers must run in order");
  std::vector<uint64_t> missing;
  for (int e : r.actual) {
    uint64_t k = eid_key(l, e);
    if (!cache_.access(k, now_)) missing.push_back(k);
  }
  for (uint64_t k : missing) request(k, 0, bucket_now());
  boundary(l);
  auto pit = predicted_.find(l);
  if (pit != predicted_.end()) {  // engine.py:585-596
    const std::vector<int>& pred = pit->second.first;
    // |set(pred) & set(actual)| and |set(actual)| with expert bit masks (M <= 128
    // on the engine path; wider models fall back to sorted vectors)
    std::vector<int> a(r.actual.begin(), r.actual.end()), pv(pred.begin(), pred.end());
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    std::sort(pv.begin(), pv.end());
    pv.erase(std::unique(pv.begin(), pv.end()), pv.end());
    int sel = 0;
    for (int e : pv) sel += std::binary_search(a.begin(), a.end(), e);
    n_selected_ += sel;
    n_total_ += (int64_t)a.size();
    samples_.push_back(SampleRec{tokens_, l, pred, r.actual, pit->second.second});
  }
  // groups and routing order (engine.py:598-606)
  int ng = (int)r.group_actual.size();
  if ((int)group_sizes_.size() != ng) throw ValueError("group count mismatch");
  std::vector<std::vector<uint64_t>> demand(ng);
  for (int g = 0; g < ng; ++g)
    for (int e : r.group_actual[g]) demand[g].push_back(eid_key(l, e));
  std::vector<int> order;
  if (cfg_.policy.cache_aware_routing) {  // route_batch engine.py:192-209
    std::vector<int> late;
    for (int g = 0; g < ng; ++g) {
      bool ready = true;
      for (uint64_t k : demand[g]) ready = ready && cache_.contains(k);
      (ready ? order : late).push_back(g);
    }
    order.insert(order.end(), late.begin(), late.end());
  } else {
    for (int g = 0; g < ng; ++g) order.push_back(g);
  }
  // _group_durations engine.py:212-219
  int64_t tot_tokens = 0;
  for (int64_t s : group_sizes_) tot_tokens += s;
  std::vector<int64_t> durs(ng);
  int64_t used = 0;
  for (int g = 0; g < ng; ++g) {
    durs[g] = (int64_t)((__int128)cfg_.layer_ns * group_sizes_[g] / tot_tokens);
    used += durs[g];
  }
  for (int64_t g = 0; g < cfg_.layer_ns - used; ++g) durs[g] += 1;

  int64_t chain = t0_, stall = 0;
  for (size_t pos = 0; pos < order.size(); ++pos) {  // engine.py:608-622
    int g = order[pos];
    std::vector<uint64_t> dem(demand[g]);
    std::sort(dem.begin(), dem.end());
    dem.erase(std::unique(dem.begin(), dem.end()), dem.end());
    int64_t avail = wait_until_resident(dem, chain);
    if (pos == 0) check_overfetch(l, avail);
    if (avail > chain) {
      int64_t gap = avail - chain;
      stall += gap;
      if (cfg_.emit_events) {
        char buf[96];
        snprintf(buf, sizeof buf, "layer=%d gap_ns=%lld", l, (long long)gap);
        emit(chain, kStall, buf);
      }
      chain = avail;
    }
    if (obs_) obs_->on_group_run(l, dem);
    consume(dem);
    chain += durs[g];
    advance_to(chain);
  }
  m_.waiting_ns += stall;  // engine.py:624-629
  m_.compute_ns += cfg_.layer_ns;
  if (stall > 0) {
    ++m_.stall_events;
    if (has_state_) state_.on_stall();
  }
  if (cfg_.policy.strategy == 3) {  // engine.py:631-644
    int64_t window = cfg_.policy.recent_window >= 0 ? cfg_.policy.recent_window : state_.current;
    hot_scratch_.clear();
    for (auto& kv : predicted_)
      if (kv.first > l)
        for (int e : kv.second.first) hot_scratch_.push_back(eid_key(kv.first, e));
    std::sort(hot_scratch_.begin(), hot_scratch_.end());
    hot_scratch_.erase(std::unique(hot_scratch_.begin(), hot_scratch_.end()), hot_scratch_.end());
    cache_.reassign_tiers(hot_scratch_, window, now_);
  }
  if (cfg_.emit_events) emit(chain, kLayerEnd, "layer=" + std::to_string(l));
  LayerRecord rec;
  rec.layer = l;
  rec.start_ns = t0_;
  rec.end_ns = chain;
  rec.stall_ns = stall;
  rec.step = step_in_effect();
  if (pit != predicted_.end()) rec.predicted = pit->second.first;
  rec.actual = r.actual;
  rec.demand_misses = (int)missing.size();
  records_.push_back(std::move(rec));
  clock_ = chain;
}

void Stepper::end_token() {
  ++tokens_run_;
  // engine.py:677-689 conservation
  if (clock_ != m_.compute_ns + m_.waiting_ns) throw RuntimeErr("timeline conservation violated");
  if (consumed_ns_ > clock_) throw RuntimeErr("work conservation violated");
}

void Stepper::run_token(const TokenInput& in) {
  if ((int)in.layers.size() != cfg_.L) throw ValueError("trace has wrong number of layers");
  set_oracle_future(&in.layers);
  begin_token(in.tokens, in.group_sizes, in.layers[0]);
  for (int l = 0; l < cfg_.L; ++l) {
    begin_layer(l);
    run_layer(l, in.layers[l]);
  }
  end_token();
  set_oracle_future(nullptr);
}

Metrics Stepper::metrics() const {
  Metrics m = m_;
  m.total_time_ns = clock_;
  m.hits = cache_.hits;
  m.misses = cache_.misses;
  m.admissions = cache_.admissions;
  m.evictions = cache_.evictions;
  m.prediction_cache_hits = pcache_.hits;
  m.prediction_cache_misses = pcache_.misses;
  m.bandwidth_estimate = estimator_.estimate();
  m.final_step = step_in_effect();
  m.n_selected = n_selected_;
  m.n_total = n_total_;
  return m;
}

std::vector<SimEventRec> Stepper::sorted_events() const {
  // engine.py:72-92 (time, EVENT_RANK, seq); kinds are numbered by rank
  std::vector<SimEventRec> ev = events_;
  std::sort(ev.begin(), ev.end(), [](const SimEventRec& a, const SimEventRec& b) {
    if (a.time != b.time) return a.time < b.time;
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.seq < b.seq;
  });
  return ev;
}

}  // namespace ef
