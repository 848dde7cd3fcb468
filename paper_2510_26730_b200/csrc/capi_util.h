// capi_util.h — exception -> status mapping shared by the C-ABI files.
#pragma once
#include <functional>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "../../include/expertflow.h"
#include "simcore.h"

namespace ef {
extern thread_local std::string g_last_error;
struct CudaErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// LadderHooks backed by the C-ABI ladder config (native forest or callbacks).
struct CallbackHooks : LadderHooks {
  explicit CallbackHooks(const ef_ladder_cfg* c);
  ef_ladder_cfg cfg;
  std::function<void(int, int, double*)> pregate_fn;  // engine-internal provider
  bool has_pregate() const override;
  void pregate(int layer, int h, double* out) override;
  bool has_forest() const override;
  void forest_scores(const double* f, int n, const double* b, double* out) override;
  int forest_feature_len() const override;
  void features(const std::vector<int64_t>& tokens, int step, int target,
                const std::map<int, std::vector<int>>& hist, double* out) override;
};

SimConfig sim_config_from(const ef_sim_cfg* c);
void sim_metrics_out(const Stepper& st, int64_t* ints, int n, double* bw);
std::vector<int64_t> sim_output(const Stepper& st, int kind);
std::string sim_event_details(const Stepper& st);
}  // namespace ef

#define EF_TRY(...)                                   \
  do {                                                \
    try {                                             \
      __VA_ARGS__;                                    \
      return EF_OK;                                   \
    } catch (const ef::ValueError& e) {               \
      ef::g_last_error = e.what();                    \
      return EF_EINVAL;                               \
    } catch (const ef::RuntimeErr& e) {               \
      ef::g_last_error = e.what();                    \
      return EF_ERUNTIME;                             \
    } catch (const ef::CudaErr& e) {                  \
      ef::g_last_error = e.what();                    \
      return EF_ECUDA;                                \
    } catch (const std::bad_alloc&) {                 \
      ef::g_last_error = "out of host memory";        \
      return EF_ENOMEM;                               \
    } catch (const std::exception& e) {               \
      ef::g_last_error = e.what();                    \
      return EF_ERUNTIME;                             \
    }                                                 \
  } while (0)
