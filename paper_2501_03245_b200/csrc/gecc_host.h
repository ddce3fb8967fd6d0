// Internal host-side declarations: one launcher per kernel family.  Every
// launcher enqueues on `s`, never synchronises, and returns the launch error.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#ifndef GECC_WG
#define GECC_WG 16  // fixed-base window width in bits (table = 17 x 2^15 x 64 B = 34 MiB)
#endif

namespace gecc {

enum { CURVE_SM2 = 0, CURVE_SECP = 1, CURVE_BLS381 = 2, CURVE_BLS377 = 3 };  // BLS12-381 / BLS12-377 G1: 12-limb coordinates
inline bool curve_is_bls(int curve) { return curve == CURVE_BLS381 || curve == CURVE_BLS377; }
inline int curve_limbs(int curve) { return curve_is_bls(curve) ? 12 : 8; }

cudaError_t launch_field_op(int curve, int field, int op, size_t n, const uint32_t* a,
                            const uint32_t* b, uint32_t* out, cudaStream_t s);
cudaError_t run_microbench(int which, int iters, int sm_count, double* ops_per_clk_per_sm,
                           double* seconds, double* total_ops, cudaStream_t s);

size_t gtable_words();
// lazy_plain: the table of the byte-record kernels on secp256k1 (plain coordinates);
// otherwise Montgomery-form coordinates (column-buffer kernels; SM2 uses it for both)
cudaError_t build_gtable(int curve, bool lazy_plain, uint32_t* tab, uint32_t* bases_scratch,
                         cudaStream_t s);
// the same table for an arbitrary base point (x, y: 8 Montgomery-form limbs each, device memory);
// flags[0] is set when the point is not on the curve (the table content is then meaningless)
cudaError_t build_base_table(int curve, const uint32_t* xy_dev, uint32_t* tab, uint32_t* bases_scratch,
                             uint32_t* flags, cudaStream_t s);
// sum of `parts` affine points, each packed as x[L] y[L] inf (2L + 1 words); the sum is written in
// the same packing to `out` (may alias parts[0]) -- the local additions of the MSM exchange
cudaError_t launch_point_fold(int curve, int parts, const uint32_t* packed, uint32_t* out, cudaStream_t s);
// packed (2L + 1 words) <-> separate x / y / inf buffers of one point
cudaError_t launch_point_pack(int curve, const uint32_t* x, const uint32_t* y, const uint8_t* inf,
                              uint32_t* packed, cudaStream_t s);
cudaError_t launch_point_unpack(int curve, const uint32_t* packed, uint32_t* x, uint32_t* y, uint8_t* inf,
                                cudaStream_t s);

// lane_scratch: verify_scratch_bytes(scratch_lanes) bytes of device memory for the per-lane
// point tables; batches larger than scratch_lanes are processed in pieces
size_t verify_scratch_bytes(size_t lanes);
cudaError_t launch_verify(int curve, size_t n, const uint8_t* dig, const uint8_t* pub,
                          const uint8_t* sig, const uint32_t* gtab, uint8_t* res,
                          uint32_t* lane_scratch, size_t scratch_lanes, cudaStream_t s);
cudaError_t launch_secret_range(int curve, size_t n, const uint8_t* sec, uint32_t* flags, cudaStream_t s);
cudaError_t launch_sign(int curve, size_t n, const uint8_t* dig, const uint8_t* sec, uint64_t seed,
                        uint64_t lane_base, const uint32_t* gtab, uint8_t* sig, int32_t* status,
                        uint32_t* flags, cudaStream_t s, bool uniform = false);
// one attempt per lane with caller-supplied 32-byte nonces; status 5 = replace the nonce
cudaError_t launch_sign_nonces(int curve, size_t n, const uint8_t* dig, const uint8_t* sec,
                               const uint8_t* nonces, const uint32_t* gtab, uint8_t* sig, int32_t* status,
                               uint32_t* flags, cudaStream_t s, bool uniform = false);
cudaError_t launch_keygen(int curve, size_t n, uint64_t seed, uint64_t lane_base,
                          const uint32_t* gtab, uint8_t* sec, uint8_t* pub, cudaStream_t s, bool uniform = false);
cudaError_t launch_ecdh(int curve, size_t n, const uint8_t* sec, const uint8_t* peers,
                        uint8_t* shared, int32_t* status, uint32_t* flags, uint32_t* lane_scratch,
                        size_t scratch_lanes, cudaStream_t s, bool uniform = false);
cudaError_t launch_fpmul(int curve, size_t n, const uint32_t* k, const uint32_t* gtab, uint32_t* ox,
                         uint32_t* oy, uint8_t* oinf, cudaStream_t s);
// lane_scratch must cover all n lanes (verify_scratch_bytes(n))
cudaError_t launch_upmul(int curve, size_t n, const uint32_t* k, const uint32_t* px,
                         const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                         uint8_t* oinf, uint32_t* lane_scratch, cudaStream_t s);

// 0 auto (by batch size), 1 chunked (one inversion per thread), 2 cooperative (one per block)
void set_batch_form(int form);
cudaError_t launch_batch_invert(int curve, int field, size_t n, const uint32_t* in, uint32_t* out,
                                cudaStream_t s);
cudaError_t launch_batch_invert_secp_lazy(size_t n, const uint32_t* in, uint32_t* out, cudaStream_t s);
// optional second stream + two events: large batches run as two overlapping halves when given
struct BatchAux {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t launch_batch_padd(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                              const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                              cudaStream_t s, void* scratch = nullptr, BatchAux aux = BatchAux());
// scratch of the tiled batch_padd form (tile totals); without it the single-launch forms run
size_t batch_padd_scratch_bytes(size_t n);
cudaError_t launch_batch_pdbl(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                              cudaStream_t s);


cudaError_t launch_seeded_scalars(int curve, size_t n, uint64_t seed, uint64_t tag, uint32_t* out,
                                  cudaStream_t s);
cudaError_t launch_padd_jacobian(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                                 const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                                 const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                                 cudaStream_t s);
cudaError_t launch_pmul_serial(int curve, size_t n, const uint32_t* k, const uint32_t* px,
                               const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                               uint8_t* oinf, cudaStream_t s);

// MSM: scratch must hold msm_scratch_bytes(n) bytes of device memory
size_t msm_scratch_bytes(size_t n, int curve);
void set_msm_form(int form);  // 0 default (batch-affine), 1 mixed-Jacobian slices, 2 batch-affine tree
// optional second stream + two events: the tree levels run as two overlapping halves when given
struct MsmAux {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t launch_msm(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                       const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                       uint8_t* oinf, void* scratch, cudaStream_t s, int* launches,
                       cudaEvent_t points_ready = nullptr,  // waited for before the first read of px / py
                       MsmAux aux = MsmAux());

}  // namespace gecc
