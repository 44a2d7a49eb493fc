/*
 * sppo_pipeline.h — host plan helpers of the subsequence pipeline across
 * stages.  Pure functions: no device work, no ctx.
 *
 * P:282-287 [§3.3 "Inevitable bubble overhead"]: with p pipeline stages and N
 * subsequences, t_b = (p-1) F(N)/N and R_b = (p-1)/N ("when p=4 and N=16, the
 * bubble ratio reaches ... 3/16").
 * P:420-455 [§6.2 Multiplexing Sequence Partition]: the forward of stage i has
 * a Left-SP, a Steady and a Right-SP phase; subsequence ids and the GPU ranges
 * that run the two SP phases follow the Definitions, read through the paper's
 * worked example (Table; reading L18 in DESIGN.md — the Definition's
 * inclusive bounds overlap, the Table's do not):
 *   Left = {0 .. PP-2-i}, Steady = {PP-1-i .. N-1-i}, Right = {N-i .. N-1},
 *   Left-SP range = {i .. PP-1} (if Left non-empty), Right-SP range = {0 .. i}
 *   (if Right non-empty).
 * Errors: SPPO_E_ARG for NULL outputs, SPPO_E_SHAPE unless 1 <= pp <= n and
 * 0 <= stage < pp.
 */
#ifndef SPPO_PIPELINE_H_
#define SPPO_PIPELINE_H_

#include <stdint.h>

#include "sppo.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { SPPO_MSP_LEFT = 0, SPPO_MSP_STEADY = 1, SPPO_MSP_RIGHT = 2 };

/* phase_out[x] (x = 0..n-1) = SPPO_MSP_* of subsequence x at stage `stage`;
 * left_sp[2], right_sp[2] = inclusive stage ranges {lo, hi}, lo > hi = empty. */
sppo_status sppo_msp_phases(int32_t pp, int32_t n, int32_t stage, int8_t* phase_out, int32_t* left_sp,
                            int32_t* right_sp);

/* Makespan of one step of the subsequence pipeline: pp stages
 * with identical per-chunk times t_fwd[i], t_bwd[i] (host arrays, n entries);
 * stage s runs fwd(i) for i = 0..n-1, each after stage s-1's fwd(i), then
 * bwd(i) for i = n-1..0, each after stage s+1's bwd(i) (the last stage starts
 * its backward after its last forward).  With uniform times this is
 * (pp-1+n)/n * F(n).  Writes the makespan (same unit as the inputs). */
sppo_status sppo_pipeline_makespan(int32_t pp, int32_t n, const double* t_fwd, const double* t_bwd,
                                   double* makespan_out);

/* R_b = (pp - 1) / n. */
sppo_status sppo_pipeline_bubble(int32_t pp, int32_t n, double* ratio_out);

#ifdef __cplusplus
}
#endif
#endif /* SPPO_PIPELINE_H_ */
