// Host plan helpers of the subsequence pipeline (include/sppo_pipeline.h).
#include "../../include/sppo_pipeline.h"
#include "internal.h"

#include <algorithm>
#include <vector>

extern "C" {

sppo_status sppo_msp_phases(int32_t pp, int32_t n, int32_t stage, int8_t* phase_out, int32_t* left_sp,
                            int32_t* right_sp) {
  if (!phase_out || !left_sp || !right_sp) return (sppo_status)sppo::api_fail(SPPO_E_ARG, "msp_phases: NULL output");
  if (pp < 1 || pp > n || stage < 0 || stage >= pp)
    return (sppo_status)sppo::api_fail(SPPO_E_SHAPE, "msp_phases: need 1 <= pp (%d) <= n (%d), 0 <= stage (%d) < pp",
                                       pp, n, stage);
  const int left_end = pp - 1 - stage;  // Left = [0, left_end), Steady = [left_end, n - stage), Right = [n - stage, n)
  for (int x = 0; x < n; ++x)
    phase_out[x] = (int8_t)(x < left_end ? SPPO_MSP_LEFT : (x < n - stage ? SPPO_MSP_STEADY : SPPO_MSP_RIGHT));
  if (left_end > 0) {
    left_sp[0] = stage;
    left_sp[1] = pp - 1;
  } else {
    left_sp[0] = 1;
    left_sp[1] = 0;
  }
  if (stage > 0) {
    right_sp[0] = 0;
    right_sp[1] = stage;
  } else {
    right_sp[0] = 1;
    right_sp[1] = 0;
  }
  return SPPO_OK;
}

sppo_status sppo_pipeline_bubble(int32_t pp, int32_t n, double* ratio_out) {
  if (!ratio_out) return (sppo_status)sppo::api_fail(SPPO_E_ARG, "pipeline_bubble: NULL output");
  if (pp < 1 || n < 1) return (sppo_status)sppo::api_fail(SPPO_E_SHAPE, "pipeline_bubble: pp, n must be >= 1");
  *ratio_out = (double)(pp - 1) / (double)n;
  return SPPO_OK;
}

sppo_status sppo_pipeline_makespan(int32_t pp, int32_t n, const double* t_fwd, const double* t_bwd,
                                   double* makespan_out) {
  if (!t_fwd || !t_bwd || !makespan_out)
    return (sppo_status)sppo::api_fail(SPPO_E_ARG, "pipeline_makespan: NULL argument");
  if (pp < 1 || n < 1) return (sppo_status)sppo::api_fail(SPPO_E_SHAPE, "pipeline_makespan: pp, n must be >= 1");
  std::vector<double> prev(n, 0.0), cur(n, 0.0), fend_last(pp, 0.0);
  // forward wavefront: cur[i] = end of fwd(i) at stage s
  for (int s = 0; s < pp; ++s) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) {
      const double start = std::max(t, s > 0 ? prev[i] : 0.0);
      t = start + t_fwd[i];
      cur[i] = t;
    }
    fend_last[s] = cur[n - 1];
    prev.swap(cur);
  }
  // backward wavefront from the last stage down
  double span = 0.0;
  for (int s = pp - 1; s >= 0; --s) {
    double t = fend_last[s];
    for (int i = n - 1; i >= 0; --i) {
      const double start = std::max(t, s + 1 < pp ? prev[i] : 0.0);
      t = start + t_bwd[i];
      cur[i] = t;
    }
    span = std::max(span, cur[0]);
    prev.swap(cur);
  }
  *makespan_out = span;
  return SPPO_OK;
}

}  // extern "C"
