// Host plan helpers of the subsequence pipeline (include/sppo_pipeline.h).
#include "../../include/sppo_pipeline.h"
#include "internal.h"

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

}  // extern "C"
