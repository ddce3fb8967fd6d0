// Internal host-side declarations: one launcher per kernel family.  Every
// launcher enqueues on `s`, never synchronises, and returns the launch error.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace gecc {

enum { CURVE_SM2 = 0, CURVE_SECP = 1 };

cudaError_t launch_field_op(int curve, int field, int op, size_t n, const uint32_t* a,
                            const uint32_t* b, uint32_t* out, cudaStream_t s);
cudaError_t run_microbench(int which, int iters, int sm_count, double* ops_per_clk_per_sm,
                           double* seconds, double* total_ops, cudaStream_t s);

}  // namespace gecc
