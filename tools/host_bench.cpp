// Host decision cost of the engine's scheduler (not part of the product):
// the Stepper driven layer by layer like engine.cu's step loop, Mixtral-8x7B
// shape at a 40% budget, adaptive horizon + pre-gate predictor, routing
// biased toward resident experts.  Prints us per layer and per token.
//   g++ -O2 -std=c++17 -I paper_2510_26730_b200/csrc -o tools/host_bench \
//       tools/host_bench.cpp paper_2510_26730_b200/csrc/simcore.cpp
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>

#include "simcore.h"

using namespace ef;

struct Hooks : LadderHooks {
  int M;
  std::mt19937_64 rng{7};
  explicit Hooks(int m) : M(m) {}
  bool has_pregate() const override { return true; }
  void pregate(int, int, double* out) override {
    double s = 0;
    for (int e = 0; e < M; ++e) s += (out[e] = 0.01 + (rng() % 1000) * 1e-5);
    for (int j = 0; j < 2; ++j) {
      int e = rng() % M;
      out[e] += 0.45;
      s += 0.45;
    }
    for (int e = 0; e < M; ++e) out[e] /= s;
  }
  bool has_forest() const override { return false; }
  void forest_scores(const double*, int, const double*, double*) override {}
  int forest_feature_len() const override { return 0; }
  void features(const std::vector<int64_t>&, int, int, const std::map<int, std::vector<int>>&,
                double*) override {}
};

int main(int argc, char** argv) {
  const int L = 32, M = 8, k = 2, tokens = argc > 1 ? atoi(argv[1]) : 200;
  SimConfig c;
  c.L = L;
  c.M = M;
  c.top_k = k;
  c.expert_size = 3LL * 4096 * 14336 * 2;
  c.link_bw = 55'000'000'000LL;
  c.device_memory = c.expert_size * 102;
  c.layer_ns = 145'000;
  c.policy.strategy = 3;
  c.policy.predictor = 1;
  Hooks hooks(M);
  Stepper st(c, &hooks);
  std::mt19937_64 rng(1);
  double layer_us = 0, token_us = 0;
  int n_layers = 0;
  for (int t = 0; t < tokens; ++t) {
    auto t0 = std::chrono::steady_clock::now();
    for (int l = 0; l < L; ++l) {
      auto a = std::chrono::steady_clock::now();
      LayerRouting r;
      r.gate.assign(M, 0.0);
      // prefer resident experts (cache-aware routing with a large bias)
      std::vector<int> pick;
      for (int e = 0; e < M && (int)pick.size() < k; ++e)
        if (st.resident(l, (e + (int)(rng() % M)) % M)) pick.push_back((e + (int)(rng() % M)) % M);
      while ((int)pick.size() < k) {
        int e = rng() % M;
        bool dup = false;
        for (int p : pick) dup |= p == e;
        if (!dup) pick.push_back(e);
      }
      if (pick[0] == pick[1]) pick[1] = (pick[0] + 1) % M;
      std::sort(pick.begin(), pick.end());
      double s = 0;
      for (int e = 0; e < M; ++e) s += (r.gate[e] = 0.01 + (rng() % 100) * 1e-4);
      for (int p : pick) s += 0.45, r.gate[p] += 0.45;
      for (int e = 0; e < M; ++e) r.gate[e] /= s;
      r.actual = pick;
      r.group_actual = {pick};
      if (l == 0) st.begin_token({(int64_t)t}, {1}, r);
      st.begin_layer(l);
      st.run_layer(l, r);
      (void)st.planned_horizon(std::min(l + 1, L - 1));
      layer_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a)
                      .count();
      ++n_layers;
    }
    st.end_token();
    token_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                    .count();
  }
  printf("tokens %d  us/layer %.2f  us/token %.1f\n", tokens, layer_us / n_layers,
         token_us / tokens);
  return 0;
}
