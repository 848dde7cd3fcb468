// capi_host.cpp — extern "C" boundary for the host-side decision path
// (include/expertflow.h).  Status codes instead of exceptions; a
// thread-local message for ef_last_error().
#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "../../include/expertflow.h"
#include "capi_util.h"
#include "simcore.h"

using namespace ef;

namespace ef {
thread_local std::string g_last_error;
}  // namespace ef

extern "C" const char* ef_last_error(void) { return ef::g_last_error.c_str(); }
extern "C" int ef_abi_version(void) { return 1; }

// ------------------------------------------------------------------ primitives
extern "C" int ef_expected_expert_count(const double* probs, int m, double thr, int* out) {
  EF_TRY({
    if (m < 1 || !probs || !out) throw ValueError("empty distribution");
    *out = expected_expert_count(probs, m, thr);
  });
}

extern "C" int ef_top_experts(const double* probs, int m, int count, int* out) {
  EF_TRY({
    std::vector<int> v = top_experts(probs, m, count);
    std::memcpy(out, v.data(), v.size() * sizeof(int));
  });
}

extern "C" int ef_swap_in_latency(int64_t n, int64_t size, int64_t bw, int64_t* out) {
  EF_TRY({ *out = swap_in_latency(n, size, bw); });
}

extern "C" int ef_compute_step_int(int64_t n_e, int64_t size, int64_t bw, int64_t layer_ns,
                                   int lo, int hi, int* out) {
  EF_TRY({ *out = compute_step_int(n_e, size, bw, layer_ns, lo, hi); });
}

extern "C" int ef_compute_step_float(int64_t n_e, int64_t size, double bw, int64_t layer_ns,
                                     int lo, int hi, int* out) {
  EF_TRY({ *out = compute_step_float(n_e, size, bw, layer_ns, lo, hi); });
}

static StepState to_state(const ef_step_state* s) {
  return StepState{s->current,         s->max_step,       s->min_step,           s->stall_count,
                   s->overfetch_count, s->stall_threshold, s->overfetch_threshold};
}
static void from_state(const StepState& t, ef_step_state* s) {
  s->current = t.current;
  s->stall_count = t.stall_count;
  s->overfetch_count = t.overfetch_count;
}

extern "C" int ef_step_validate(const ef_step_state* s) { EF_TRY({ to_state(s).validate(); }); }
extern "C" int ef_step_on_stall(ef_step_state* s) {
  EF_TRY({
    StepState t = to_state(s);
    t.on_stall();
    from_state(t, s);
  });
}
extern "C" int ef_step_on_overfetch(ef_step_state* s) {
  EF_TRY({
    StepState t = to_state(s);
    t.on_overfetch();
    from_state(t, s);
  });
}

// ------------------------------------------------------------------ cache
struct ef_cache {
  ExpertCache c;
};

extern "C" int ef_cache_create(int64_t capacity_bytes, int64_t expert_size, int record,
                               ef_cache** out) {
  EF_TRY({ *out = new ef_cache{ExpertCache(capacity_bytes, expert_size, record != 0)}; });
}
extern "C" void ef_cache_destroy(ef_cache* c) { delete c; }

static void check_id(int32_t layer, int32_t expert) {
  if (layer < 0 || expert < 0) throw ValueError("negative expert id");
}

extern "C" int ef_cache_access(ef_cache* c, int32_t layer, int32_t expert, int64_t now,
                               int* hit) {
  EF_TRY({
    check_id(layer, expert);
    *hit = c->c.access(eid_key(layer, expert), now) ? 1 : 0;
  });
}

extern "C" int ef_cache_admit(ef_cache* c, int32_t layer, int32_t expert, int tier, int64_t now,
                              int32_t* victims, int max_victims, int* n_victims) {
  EF_TRY({
    check_id(layer, expert);
    std::vector<uint64_t> v = c->c.admit(eid_key(layer, expert), tier, now);
    *n_victims = (int)v.size();
    for (int i = 0; i < (int)v.size() && i < max_victims; ++i) {
      victims[2 * i] = eid_layer(v[i]);
      victims[2 * i + 1] = eid_expert(v[i]);
    }
  });
}

extern "C" int ef_cache_reassign_tiers(ef_cache* c, const int32_t* pred, int n_pred,
                                       int64_t window, int64_t now) {
  EF_TRY({
    std::vector<uint64_t> s;
    for (int i = 0; i < n_pred; ++i) s.push_back(eid_key(pred[2 * i], pred[2 * i + 1]));
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    c->c.reassign_tiers(s, window, now);
  });
}

extern "C" int ef_cache_query(ef_cache* c, int32_t layer, int32_t expert, int* tier,
                              int64_t* last) {
  EF_TRY({
    uint64_t k = eid_key(layer, expert);
    *tier = c->c.tier_of(k);
    *last = c->c.last_access(k);
  });
}

extern "C" int ef_cache_counters(ef_cache* c, int64_t out[6]) {
  EF_TRY({
    out[0] = c->c.capacity();
    out[1] = (int64_t)c->c.size();
    out[2] = c->c.hits;
    out[3] = c->c.misses;
    out[4] = c->c.admissions;
    out[5] = c->c.evictions;
  });
}

extern "C" int ef_cache_resident(ef_cache* c, int32_t* pairs, int max_pairs, int* n) {
  EF_TRY({
    std::vector<uint64_t> r = c->c.resident_sorted();
    *n = (int)r.size();
    for (int i = 0; i < (int)r.size() && i < max_pairs; ++i) {
      pairs[2 * i] = eid_layer(r[i]);
      pairs[2 * i + 1] = eid_expert(r[i]);
    }
  });
}

extern "C" int ef_cache_events(ef_cache* c, int64_t* rows, int64_t max_rows, int64_t* n) {
  EF_TRY({
    if (!c->c.recording()) {
      *n = -1;
      return EF_OK;
    }
    const auto& ev = c->c.events();
    *n = (int64_t)ev.size();
    for (int64_t i = 0; i < (int64_t)ev.size() && i < max_rows; ++i) {
      rows[4 * i] = ev[i].now;
      rows[4 * i + 1] = ev[i].kind;
      rows[4 * i + 2] = eid_layer(ev[i].key);
      rows[4 * i + 3] = eid_expert(ev[i].key);
    }
  });
}

// ------------------------------------------------------------------ queue / bw
struct ef_tqueue {
  TransferQueue q;
};
extern "C" int ef_tqueue_create(ef_tqueue** out) { EF_TRY({ *out = new ef_tqueue(); }); }
extern "C" void ef_tqueue_destroy(ef_tqueue* q) { delete q; }
extern "C" int ef_tqueue_enqueue(ef_tqueue* q, int32_t layer, int32_t expert, int prio,
                                 int64_t* seq) {
  EF_TRY({
    if (prio < 0 || prio > 2) throw ValueError("unknown priority");
    *seq = q->q.enqueue(eid_key(layer, expert), prio).seq;
  });
}
extern "C" int ef_tqueue_next(ef_tqueue* q, int32_t* layer, int32_t* expert, int* prio,
                              int64_t* seq, int* found) {
  EF_TRY({
    TransferRequest r;
    *found = q->q.next(&r) ? 1 : 0;
    if (*found) {
      *layer = eid_layer(r.key);
      *expert = eid_expert(r.key);
      *prio = r.prio;
      *seq = r.seq;
    }
  });
}
extern "C" int ef_tqueue_len(ef_tqueue* q, int64_t* n) { EF_TRY({ *n = (int64_t)q->q.size(); }); }

struct ef_bw {
  BandwidthEstimator b;
};
extern "C" int ef_bw_create(int has_initial, double initial, double alpha, ef_bw** out) {
  EF_TRY({ *out = new ef_bw{BandwidthEstimator(has_initial != 0, initial, alpha)}; });
}
extern "C" void ef_bw_destroy(ef_bw* b) { delete b; }
extern "C" int ef_bw_observe(ef_bw* b, int64_t bytes, int64_t ns, double* out) {
  EF_TRY({ *out = b->b.observe(bytes, ns); });
}
extern "C" int ef_bw_estimate(ef_bw* b, double* out) { EF_TRY({ *out = b->b.estimate(); }); }

// ------------------------------------------------------------------ prediction cache
struct ef_pcache {
  PredictionCache p;
};
extern "C" int ef_pcache_create(int capacity, ef_pcache** out) {
  EF_TRY({ *out = new ef_pcache{PredictionCache(capacity)}; });
}
extern "C" void ef_pcache_destroy(ef_pcache* p) { delete p; }
extern "C" int ef_pcache_get(ef_pcache* p, const int64_t* tokens, int n_tokens, int64_t layer,
                             int64_t step, int64_t* val, int64_t max_val, int64_t* n_val,
                             int* found) {
  EF_TRY({
    std::vector<int64_t> t(tokens, tokens + n_tokens);
    const Blob* b = p->p.get(t, layer, step);
    *found = b ? 1 : 0;
    *n_val = b ? (int64_t)b->size() : 0;
    if (b)
      for (int64_t i = 0; i < (int64_t)b->size() && i < max_val; ++i) val[i] = (*b)[i];
  });
}
extern "C" int ef_pcache_put(ef_pcache* p, const int64_t* tokens, int n_tokens, int64_t layer,
                             int64_t step, const int64_t* val, int64_t n_val) {
  EF_TRY({
    p->p.put(std::vector<int64_t>(tokens, tokens + n_tokens), layer, step,
             Blob(val, val + n_val));
  });
}
extern "C" int ef_pcache_stats(ef_pcache* p, int64_t out[3]) {
  EF_TRY({
    out[0] = p->p.hits;
    out[1] = p->p.misses;
    out[2] = (int64_t)p->p.size();
  });
}

// ------------------------------------------------------------------ forest
struct ef_forest {
  Forest f;
};
extern "C" int ef_forest_create(int n_trees, const int64_t* tree_off, const int32_t* feature,
                                const double* threshold, const int32_t* left,
                                const int32_t* right, const double* value, int32_t feature_len,
                                int32_t num_outputs, int residual, ef_forest** out) {
  EF_TRY({
    if (n_trees < 1) throw ValueError("forest needs at least one tree");
    auto* f = new ef_forest();
    Forest& F = f->f;
    F.n_trees = n_trees;
    F.feature_len = feature_len;
    F.num_outputs = num_outputs;
    F.residual = residual != 0;
    F.tree_off.assign(tree_off, tree_off + n_trees + 1);
    int64_t nn = tree_off[n_trees];
    F.feature.assign(feature, feature + nn);
    F.left.assign(left, left + nn);
    F.right.assign(right, right + nn);
    F.threshold.assign(threshold, threshold + nn);
    F.value.assign(value, value + nn * num_outputs);
    for (int64_t i = 0; i < nn; ++i)
      if (F.feature[i] >= feature_len) {
        delete f;
        throw ValueError("forest split feature out of range");
      }
    *out = f;
  });
}
extern "C" void ef_forest_destroy(ef_forest* f) { delete f; }
extern "C" int ef_forest_predict(ef_forest* f, const double* x, const double* base,
                                 double* out) {
  EF_TRY({ f->f.predict(x, base, out); });
}

static std::map<int, std::vector<int>> parse_hist(const int32_t* h, int64_t len) {
  std::map<int, std::vector<int>> m;
  int64_t p = 0;
  while (p < len) {
    int layer = h[p++];
    int n = h[p++];
    std::vector<int> v(h + p, h + p + n);
    p += n;
    m[layer] = v;
  }
  return m;
}

extern "C" int ef_inference_features(const double* table, int64_t vocab, int32_t embed_dim,
                                     int32_t L, int32_t M, const int64_t* tokens, int n_tokens,
                                     int32_t step, int32_t target, const int32_t* hist,
                                     int64_t hist_len, double* out) {
  EF_TRY({
    inference_features(table, vocab, embed_dim, L, M,
                       std::vector<int64_t>(tokens, tokens + n_tokens), step, target,
                       parse_hist(hist, hist_len), out);
  });
}

// ------------------------------------------------------------------ ladder hooks
namespace ef {
CallbackHooks::CallbackHooks(const ef_ladder_cfg* c) {
  if (c) cfg = *c;
  else std::memset(&cfg, 0, sizeof cfg);
}
bool CallbackHooks::has_pregate() const { return cfg.pregate_cb != nullptr || pregate_fn; }
void CallbackHooks::pregate(int layer, int h, double* out) {
  if (pregate_fn) {
    pregate_fn(layer, h, out);
    return;
  }
  if (cfg.pregate_cb(cfg.pregate_user, layer, h, out) != 0)
    throw RuntimeErr("pregate callback failed");
}
bool CallbackHooks::has_forest() const { return cfg.forest || cfg.forest_cb; }
void CallbackHooks::forest_scores(const double* f, int n, const double* b, double* out) {
  if (cfg.forest) {
    cfg.forest->f.predict(f, b, out);
    return;
  }
  if (cfg.forest_cb(cfg.forest_user, f, n, b, out) != 0)
    throw RuntimeErr("forest callback failed");
}
int CallbackHooks::forest_feature_len() const {
  return cfg.forest ? cfg.forest->f.feature_len : cfg.forest_feature_len;
}
void CallbackHooks::features(const std::vector<int64_t>& tokens, int step, int target,
                             const std::map<int, std::vector<int>>& hist, double* out) {
  if (!cfg.table) throw ValueError("forest prediction needs table and model");
  inference_features(cfg.table, cfg.vocab, cfg.embed_dim, cfg.L, cfg.M, tokens, step, target,
                     hist, out);
}
}  // namespace ef

extern "C" int ef_predict_experts(const ef_ladder_cfg* cfg, ef_pcache* cache,
                                  const int64_t* tokens, int n_tokens, int32_t layer,
                                  int32_t step, const double* router_probs, const int32_t* known,
                                  int64_t known_len, int64_t* out, int64_t max_out,
                                  int64_t* n_out) {
  EF_TRY({
    CallbackHooks hooks(cfg);
    if (hooks.has_forest() && !cfg->table) throw ValueError("forest prediction needs table and model");
    Horizon h = predict_experts(hooks, cache->p, std::vector<int64_t>(tokens, tokens + n_tokens),
                                layer, step, router_probs, cfg->M, cfg->top_k,
                                cfg->cum_threshold, parse_hist(known, known_len));
    Blob b = encode_horizon(h);
    *n_out = (int64_t)b.size();
    for (int64_t i = 0; i < (int64_t)b.size() && i < max_out; ++i) out[i] = b[i];
  });
}

extern "C" int ef_route_batch(const int32_t* groups, int64_t len, const uint8_t* mask, int32_t M,
                              int32_t* order, int32_t* deferred, int32_t* n_groups,
                              int32_t* n_deferred) {
  EF_TRY({
    std::vector<int32_t> ready, late;
    int64_t p = 0;
    while (p < len) {
      int32_t gid = groups[p++];
      int32_t n = groups[p++];
      bool ok = true;
      for (int i = 0; i < n; ++i) {
        int32_t e = groups[p + i];
        if (e < 0 || e >= M) throw ValueError("expert out of range");
        ok = ok && mask[e];
      }
      p += n;
      (ok ? ready : late).push_back(gid);
    }
    *n_groups = (int32_t)(ready.size() + late.size());
    *n_deferred = (int32_t)late.size();
    int i = 0;
    for (int32_t g : ready) order[i++] = g;
    for (int32_t g : late) order[i++] = g;
    for (size_t j = 0; j < late.size(); ++j) deferred[j] = late[j];
  });
}

// ------------------------------------------------------------------ sim
struct ef_sim {
  std::unique_ptr<CallbackHooks> hooks;
  std::unique_ptr<Stepper> st;
  int L, M;
};

namespace ef {
SimConfig sim_config_from(const ef_sim_cfg* c) {
  SimConfig s;
  s.L = c->L;
  s.M = c->M;
  s.top_k = c->top_k;
  s.expert_size = c->expert_size_bytes;
  s.link_bw = c->link_bw;
  s.device_memory = c->device_memory_bytes;
  s.layer_ns = c->layer_ns;
  s.emit_events = c->emit_events != 0;
  s.bw_feedback = c->bw_feedback != 0;
  Policy& p = s.policy;
  p.strategy = c->strategy;
  p.predictor = c->predictor;
  p.interval = c->interval;
  p.cache_aware_routing = c->cache_aware_routing != 0;
  p.preload = c->cold_start_preload != 0;
  p.cum_threshold = c->cum_threshold;
  p.stall_threshold = c->stall_threshold;
  p.overfetch_threshold = c->overfetch_threshold;
  p.min_step = c->min_step;
  p.max_step = c->max_step;
  p.recent_window = c->recent_window;
  p.prediction_cache_capacity = c->prediction_cache_capacity;
  p.seed = c->seed;
  if (s.L < 1 || s.M < 1 || s.top_k < 1 || s.top_k > s.M) throw ValueError("invalid model spec");
  return s;
}
}  // namespace ef

extern "C" int ef_sim_create(const ef_sim_cfg* cfg, const ef_ladder_cfg* ladder, ef_sim** out) {
  EF_TRY({
    auto s = std::make_unique<ef_sim>();
    s->hooks = std::make_unique<CallbackHooks>(ladder);
    SimConfig sc = sim_config_from(cfg);
    if (sc.policy.predictor == 2 && (!s->hooks->has_forest() || !ladder->table))
      throw ValueError("forest predictor needs a trained model and table");
    s->st = std::make_unique<Stepper>(sc, s->hooks.get());
    if (sc.bw_feedback) {
      Stepper* st = s->st.get();
      st->set_bw_feedback([st] { return st->logical_bw_estimate(); });
    }
    s->L = cfg->L;
    s->M = cfg->M;
    *out = s.release();
  });
}
extern "C" void ef_sim_destroy(ef_sim* s) { delete s; }

extern "C" int ef_sim_run_token(ef_sim* s, const int64_t* tokens, int n_tokens,
                                const double* gates, const int32_t* actual, int64_t actual_len,
                                const int32_t* groups, int64_t groups_len,
                                const int64_t* group_sizes, int32_t n_groups) {
  EF_TRY({
    TokenInput in;
    in.tokens.assign(tokens, tokens + n_tokens);
    in.group_sizes.assign(group_sizes, group_sizes + n_groups);
    in.layers.resize(s->L);
    int64_t pa = 0, pg = 0;
    for (int l = 0; l < s->L; ++l) {
      LayerRouting& r = in.layers[l];
      r.gate.assign(gates + (int64_t)l * s->M, gates + (int64_t)(l + 1) * s->M);
      if (pa >= actual_len || pg >= groups_len) throw ValueError("truncated trace");
      int n = actual[pa++];
      r.actual.assign(actual + pa, actual + pa + n);
      pa += n;
      int ng = groups[pg++];
      if (ng != n_groups) throw ValueError("group count mismatch");
      r.group_actual.resize(ng);
      for (int g = 0; g < ng; ++g) {
        int c = groups[pg++];
        r.group_actual[g].assign(groups + pg, groups + pg + c);
        pg += c;
      }
    }
    s->st->run_token(in);
  });
}

namespace ef {
void sim_metrics_out(const Stepper& st, int64_t* ints, int n, double* bw) {
  Metrics m = st.metrics();
  int64_t v[17] = {m.total_time_ns,   m.compute_ns,   m.waiting_ns,    m.cache_miss_ns,
                   m.prefetch_ns,     m.cold_start_ns, m.hits,         m.misses,
                   m.admissions,      m.evictions,    m.stall_events,  m.overfetch_events,
                   m.prediction_cache_hits, m.prediction_cache_misses, m.final_step,
                   m.n_selected,      m.n_total};
  for (int i = 0; i < n && i < 17; ++i) ints[i] = v[i];
  if (bw) *bw = m.bandwidth_estimate;
}

std::vector<int64_t> sim_output(const Stepper& st, int kind) {
  std::vector<int64_t> o;
  if (kind == 0) {
    for (auto& p : st.step_history()) {
      o.push_back(p.first);
      o.push_back(p.second);
    }
  } else if (kind == 1) {
    for (auto& r : st.layer_records()) {
      o.insert(o.end(), {r.layer, r.start_ns, r.end_ns, r.stall_ns, r.step, r.demand_misses});
      o.push_back((int64_t)r.predicted.size());
      o.insert(o.end(), r.predicted.begin(), r.predicted.end());
      o.push_back((int64_t)r.actual.size());
      o.insert(o.end(), r.actual.begin(), r.actual.end());
    }
  } else if (kind == 2) {
    for (auto& s : st.samples()) {
      o.push_back(s.layer);
      o.push_back(s.step);
      o.push_back((int64_t)s.tokens.size());
      o.insert(o.end(), s.tokens.begin(), s.tokens.end());
      o.push_back((int64_t)s.predicted.size());
      o.insert(o.end(), s.predicted.begin(), s.predicted.end());
      o.push_back((int64_t)s.actual.size());
      o.insert(o.end(), s.actual.begin(), s.actual.end());
    }
  } else if (kind == 3) {
    for (auto& e : st.sorted_events()) o.insert(o.end(), {e.time, (int64_t)e.kind, e.seq});
  } else if (kind == 4) {
    if (st.cache().recording())
      for (auto& e : st.cache().events())
        o.insert(o.end(), {e.now, (int64_t)e.kind, (int64_t)eid_layer(e.key),
                           (int64_t)eid_expert(e.key)});
  } else {
    throw ValueError("unknown output kind");
  }
  return o;
}

std::string sim_event_details(const Stepper& st) {
  std::string s;
  for (auto& e : st.sorted_events()) {
    s += e.detail;
    s += '\n';
  }
  return s;
}
}  // namespace ef

extern "C" int ef_sim_metrics(ef_sim* s, int64_t* ints, int32_t n, double* bw) {
  EF_TRY({ sim_metrics_out(*s->st, ints, n, bw); });
}
extern "C" int ef_sim_output(ef_sim* s, int32_t kind, int64_t* buf, int64_t max_len, int64_t* n) {
  EF_TRY({
    std::vector<int64_t> o = sim_output(*s->st, kind);
    *n = (int64_t)o.size();
    for (int64_t i = 0; i < (int64_t)o.size() && i < max_len; ++i) buf[i] = o[i];
  });
}
extern "C" int ef_sim_event_details(ef_sim* s, char* buf, int64_t max_len, int64_t* n) {
  EF_TRY({
    std::string d = sim_event_details(*s->st);
    *n = (int64_t)d.size();
    if (buf && max_len > 0) std::memcpy(buf, d.data(), std::min<int64_t>(max_len, *n));
  });
}
