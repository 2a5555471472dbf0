/*
 * masw_probe.h -- measurement helpers of libmasw.so (not part of the forward model).
 *
 * The FP64 roofline denominator: MEASURED_PEAKS.json has no FP64 entry, so bench.py
 * measures it on the box with a dependent-chain-free DFMA microbenchmark (SURVEY.md §8(d)
 * "Peak").  Nominal: 148 SMs x 64 FP64 FMA/clk x 2 flop x f_clk (37.2 TFLOP/s at 1965 MHz).
 */
#ifndef MASW_PROBE_H
#define MASW_PROBE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Runs a DFMA-only kernel (every SM, 8 independent FMA chains per thread) for about
 * `target_ms` on `device` (-1 = current) and reports the achieved fp64 TFLOP/s
 * (2 flops per DFMA) and the kernel time.  Returns 0 or a MASW_E_* code. */
int masw_probe_fp64_peak(int32_t device, double target_ms, double *tflops_out, double *ms_out);

#ifdef __cplusplus
}
#endif
#endif
