/*
 * gecc_b200.h -- C ABI of libgecc_b200.so, the B200 (sm_100a) batched
 * elliptic-curve engine.
 *
 * Part 1 is the drop-in boundary: the exact entry points, enum values and struct
 * layouts of the reference library's C interface
 * (/root/reference/proj/include/sm2batch.h), so a consumer of libsm2batch.so
 * can link this library instead.  Each declaration cites the line it replaces.
 * Part 2 adds what the reference's C++ batch API offers (batch_invert.hpp,
 * batch_point.hpp) in C form -- flat column-major arrays, host or device
 * pointers -- plus a curve selector (SM2 / secp256k1) and MSM.
 *
 * Record formats (sm2batch.h:4-9): all big-endian, flat arrays:
 *   scalar / digest / secret 32 B, point 65 B (0x04 || X || Y),
 *   signature 64 B (r || s), shared secret 32 B.
 * Column buffers (batch_buffer.hpp:15-35): limb k of element i at cols[k*n + i],
 *   least-significant limb first, 8 limbs; field elements are in Montgomery form
 *   (R = 2^256), scalars are plain integers.  Infinity masks are one byte per
 *   element (1 = point at infinity) and infinity coordinates are written as zero
 *   (batch_point.cpp:41-47).
 *
 * There is no CPU fallback: every compute entry point runs CUDA kernels and
 * returns SM2B_ERROR_INTERNAL (see gecc_last_error) if no device is usable.
 */
#ifndef GECC_B200_H
#define GECC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ===================== Part 1: drop-in for sm2batch.h ===================== */

/* sm2batch.h:27-36 */
typedef enum sm2b_status {
    SM2B_OK = 0,
    SM2B_ERROR_INVALID_ARGUMENT = 1,
    SM2B_ERROR_MALFORMED_INPUT = 2,
    SM2B_ERROR_INVALID_PEER = 3,
    SM2B_ERROR_DEGENERATE = 4,
    SM2B_ERROR_NONCE_EXHAUSTED = 5,
    SM2B_ERROR_NO_CROSSOVER = 6,
    SM2B_ERROR_INTERNAL = 7
} sm2b_status;

/* sm2batch.h:41 -- opaque; here it owns a CUDA stream, device scratch and the
 * fixed-base tables instead of a worker pool. Calls on one context serialise. */
typedef struct sm2b_ctx sm2b_ctx;

/* sm2batch.h:44-45.  SM2 curve on the current CUDA device.  `workers` and `lanes`
 * are accepted for compatibility; results are lane-count invariant by contract
 * (batch_invert.hpp:59-60) and the grid replaces the pool.  NULL on failure. */
sm2b_ctx* sm2b_ctx_new(uint32_t workers, uint32_t lanes);
void sm2b_ctx_free(sm2b_ctx* ctx);

/* sm2batch.h:47-48 */
const char* sm2b_version(void);
const char* sm2b_status_str(sm2b_status status);

/* sm2batch.h:51-59.  The GPU kernels do not count operations; the ledger is
 * advanced with the reference algorithm's closed-form counts for each call
 * (SURVEY.md section 5), so economics checks written against the reference
 * (e.g. modinv == 257 per sign call) keep their meaning. */
typedef struct sm2b_op_counts {
    uint64_t modmul;
    uint64_t modadd;
    uint64_t modsub;
    uint64_t modinv;
} sm2b_op_counts;
sm2b_status sm2b_ledger_read(const sm2b_ctx* ctx, sm2b_op_counts* out);
sm2b_status sm2b_ledger_reset(sm2b_ctx* ctx);

/* sm2batch.h:63-64 */
sm2b_status sm2b_keygen(sm2b_ctx* ctx, uint64_t seed, size_t count, uint8_t* secrets,
                        uint8_t* publics);
/* sm2batch.h:69-71 */
sm2b_status sm2b_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                      const uint8_t* secrets, uint64_t nonce_seed, uint8_t* signatures,
                      int32_t* lane_status);
/* sm2batch.h:75-77 */
sm2b_status sm2b_verify(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                        const uint8_t* publics, const uint8_t* signatures,
                        uint8_t* results);
/* sm2batch.h:80-82 */
sm2b_status sm2b_ecdh(sm2b_ctx* ctx, size_t count, const uint8_t* secrets,
                      const uint8_t* peers, uint8_t* shared, int32_t* lane_status);
/* sm2batch.h:86-87 */
sm2b_status sm2b_crossover_n(uint64_t cost_add, uint64_t cost_mul, uint64_t cost_inv,
                             uint64_t* out_n);

/* sm2batch.h:89-96 */
typedef struct sm2b_bench_report {
    uint64_t lanes_used;
    double wall_seconds;
    double throughput;
    sm2b_op_counts ops;
    uint64_t modeled_cost;
    int equivalence_checked;
} sm2b_bench_report;
/* sm2batch.h:102-105.  op: padd|fpmul|upmul|sign|verify; strategy: affine-batch (the
 * production kernels) | jacobian-serial (independent per-lane kernels: one mixed
 * Jacobian add / LSB-first double-and-add, as serial_padd and pmul_serial of the
 * reference).  Inputs use the reference's seeded recipe and stream tags
 * (bench.cpp:20-48,139-200); both strategies run once and are compared before timing
 * (bench.cpp:253-256); wall_seconds is the median of `repeats` CUDA-event timings after
 * one warm-up; ops are the reference's closed-form counts. */
sm2b_status sm2b_bench_run(sm2b_ctx* ctx, const char* op, const char* strategy, size_t n,
                           size_t lanes, uint32_t workers, uint64_t seed, uint32_t repeats,
                           sm2b_bench_report* out);

/* ========================== Part 2: extensions ========================== */

/* GECC_CURVE_BLS12_381 (G1: y^2 = x^3 + 4 over the 381-bit prime) and GECC_CURVE_BLS12_377 (G1:
 * y^2 = x^3 + 1 over the 377-bit prime, 253-bit group order) serve the field, batch and MSM
 * layer only -- the reference is 256-bit (limbs.hpp:17) and has no counterpart.  Its coordinate
 * column buffers hold 12 limbs per element (limb k of element i at cols[k*n + i], Montgomery
 * form with R = 2^384); scalars and GECC_FIELD_N elements stay 8 limbs (255-bit group order).
 * The ECDSA / fixed-base / variable-base entry points return SM2B_ERROR_INVALID_ARGUMENT on it. */
typedef enum gecc_curve {
    GECC_CURVE_SM2 = 0, GECC_CURVE_SECP256K1 = 1, GECC_CURVE_BLS12_381 = 2, GECC_CURVE_BLS12_377 = 3
} gecc_curve;
typedef enum gecc_field { GECC_FIELD_P = 0, GECC_FIELD_N = 1 } gecc_field;
/* same numbering as the oracle's field ops */
typedef enum gecc_field_opcode {
    GECC_OP_MONT_MUL = 0, /* field.cpp:205-211 */
    GECC_OP_MOD_ADD = 1,  /* field.cpp:213-219 */
    GECC_OP_MOD_SUB = 2,  /* field.cpp:221-227 */
    GECC_OP_TO_MONT = 3,  /* field.cpp:194-198 */
    GECC_OP_FROM_MONT = 4,/* field.cpp:200-203 */
    GECC_OP_MOD_INV = 5,  /* field.cpp:239-246's value via safegcd, zero maps to zero */
    GECC_OP_MOD_INV_FERMAT = 6, /* same value by a^(q-2), kept as a cross-check */
    /* mont_reduce of a 512-bit value (field.hpp mont_reduce_generic / mont_reduce_sm2,
     * field.cpp:50-128): a = low 8 limbs, b = high 8 limbs, out = value * R^-1 mod q, canonical.
     * The value must be below q * 2^256.  Reaches the curve-specialised reductions directly. */
    GECC_OP_MONT_REDUCE = 7,
    /* The weakly reduced plain representation the fused secp256k1 kernels compute in
     * (GECC_CURVE_SECP256K1, GECC_FIELD_P only): inputs are ANY 256-bit values (not Montgomery
     * form, not necessarily below q), outputs are the canonical residues a*b, a^2, a+b, a-b mod q. */
    GECC_OP_LAZY_MUL = 8, GECC_OP_LAZY_SQR = 9, GECC_OP_LAZY_ADD = 10, GECC_OP_LAZY_SUB = 11,
    /* GECC_OP_MOD_INV's value computed by the warp-cooperative inversion the block-level Montgomery
     * trick uses for its one shared inversion (every element is inverted by a whole warp) */
    GECC_OP_MOD_INV_WARP = 12
} gecc_field_opcode;

/* Context for `curve` on CUDA device `device` (< 0: the current device). */
sm2b_ctx* gecc_ctx_new(gecc_curve curve, int device);
/* GROUP context: one context that drives `ndev` CUDA devices (the reference's
 * context owns its workers the same way, capi.cpp:94-107).  `devices` lists them (NULL: devices
 * 0 .. ndev-1; ndev <= 0: every visible device).  Every host-pointer entry point splits its batch
 * into contiguous lane ranges, one per device, each served by its own host thread, streams and
 * arenas; every device downloads its own slice.  The global lane index stays the nonce stream id
 * (protocol.cpp:125-126), so outputs are byte-identical for any device count.  gecc_msm shards by
 * point range and exchanges the per-device partial sums with one ncclAllGather followed by local
 * additions.  A device may be listed more than once (several shards on one GPU: how the sharding
 * logic is exercised on a one-GPU box; the exchange then uses peer copies, NCCL refuses duplicate
 * devices).  The *_dev entry points, gecc_ctx_set_stream and gecc_microbench address ONE device and
 * return SM2B_ERROR_INVALID_ARGUMENT on a group context.
 * sm2b_ctx_new() itself creates a group over all visible devices when there is more than one
 * (environment GECC_NDEV=k limits it to the first k). */
sm2b_ctx* gecc_ctx_new_multi(gecc_curve curve, int ndev, const int* devices);
/* number of device shards behind the context (1 for a device context) */
int gecc_ctx_shards(const sm2b_ctx* ctx);
int gecc_ctx_curve(const sm2b_ctx* ctx);
int gecc_ctx_device(const sm2b_ctx* ctx);
/* Message of the last failing call on this context ("" if none). */
const char* gecc_last_error(const sm2b_ctx* ctx);
/* Number of CUDA kernels this context has launched so far. */
uint64_t gecc_kernel_launches(const sm2b_ctx* ctx);
/* Use `stream` (a cudaStream_t) for all following calls; NULL = context's own. */
sm2b_status gecc_ctx_set_stream(sm2b_ctx* ctx, void* stream);

/* Sharded forms of keygen / sign: `lane_base` is the global index of lane 0 of
 * this call, used as the nonce stream id (protocol.cpp:125-126), so a batch split
 * over several GPUs / calls produces the same bytes as one call. */
sm2b_status gecc_keygen(sm2b_ctx* ctx, uint64_t seed, uint64_t lane_base, size_t count,
                        uint8_t* secrets, uint8_t* publics);
sm2b_status gecc_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                      const uint8_t* secrets, uint64_t nonce_seed, uint64_t lane_base,
                      uint8_t* signatures, int32_t* lane_status);

/* One signing attempt with caller-supplied nonces (32-byte big-endian records): the building
 * block of ecdsa_sign_batch with an arbitrary NonceSource (protocol.cpp:121-164).  lane_status[i] is
 * SM2B_OK, or SM2B_ERROR_NONCE_EXHAUSTED when this nonce must be replaced (nonce outside (0, n),
 * r == 0 or s == 0; the signature is then zeroed).  Secrets are checked as in sm2b_sign. */
sm2b_status gecc_sign_nonces(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                             const uint8_t* secrets, const uint8_t* nonces, uint8_t* signatures,
                             int32_t* lane_status);

/* Secret-scalar discipline (SPEC.md: "constant structure" on secret-dependent paths; the
 * reference applies table entries by select, batch_point.cpp:319-333,420).  GECC_SECRET_FAST skips
 * zero digits and branches on digit signs; GECC_SECRET_UNIFORM makes k*G (sign, keygen) and d*P
 * (ECDH) execute the same instruction and memory-access sequence for every scalar: every window
 * performs its addition, the table entry is chosen by masked sweep / arithmetic select and the sign
 * by a conditional negation without branches.  Outputs are identical. */
enum { GECC_SECRET_FAST = 0, GECC_SECRET_UNIFORM = 1 };
sm2b_status gecc_ctx_set_secret_mode(sm2b_ctx* ctx, int mode);

/* precompute_base_table (batch_point.hpp:76-83, batch_point.cpp:341-350) for an arbitrary base:
 * a device-resident windowed table of the affine point (x, y) (8 Montgomery-form limbs each).
 * SM2B_ERROR_MALFORMED_INPUT when the point is not on the context's curve (the reference throws
 * std::invalid_argument there).  batch_fpmul over it: out[i] = scalars[i] * base. */
typedef struct gecc_base_table gecc_base_table;
sm2b_status gecc_base_table_new(sm2b_ctx* ctx, const uint32_t* x, const uint32_t* y,
                                gecc_base_table** out);
void gecc_base_table_free(gecc_base_table* table);
sm2b_status gecc_batch_fpmul_base(sm2b_ctx* ctx, const gecc_base_table* base, size_t n,
                                  const uint32_t* scalars, uint32_t* ox, uint32_t* oy, uint8_t* oinf);

/* Multi-process form of the MSM exchange (one process per GPU, e.g. under torchrun): rank 0 draws
 * an id, the launcher's own plumbing broadcasts the 128 bytes, every rank joins with its device
 * context.  gecc_msm_combine_dev then turns every rank's partial sum (one affine point in device
 * memory, as gecc_msm_dev wrote it) into the total on every rank: one ncclAllGather of 2L+1 words
 * per rank + nranks-1 local additions (EC addition is not an NCCL reduction operator), enqueued on
 * the context's stream, not synchronised. */
#define GECC_COMM_ID_BYTES 128
sm2b_status gecc_comm_unique_id(uint8_t id[GECC_COMM_ID_BYTES]);
sm2b_status gecc_comm_init_rank(sm2b_ctx* ctx, int nranks, int rank, const uint8_t id[GECC_COMM_ID_BYTES]);
sm2b_status gecc_msm_combine_dev(sm2b_ctx* ctx, uint32_t* x, uint32_t* y, uint8_t* inf);

/* ---- runtime moduli and user curves (the reference's C++ layer is generic in both:
 * FieldParams::make(q), field.cpp:159-179; CurveParams {base_field, a, b}, curve.hpp:51-59;
 * batch_invert / batch_padd / batch_pdbl take them as arguments, batch_invert.hpp:61,
 * batch_point.hpp:47-60).  Elements are 8-limb column buffers, Montgomery form with R = 2^256.
 * Device contexts only; any context serves (the constants travel with the call). */
typedef struct gecc_field_params { uint32_t w[64]; } gecc_field_params; /* opaque; fill with gecc_field_params_make */
/* FieldParams::make(q): q odd and >= 3, else SM2B_ERROR_INVALID_ARGUMENT ("modulus must be odd").
 * Inversion assumes q prime, as the reference's does. */
sm2b_status gecc_field_params_make(const uint32_t q[8], gecc_field_params* out);
/* which: 0 q, 1 R = 2^256 mod q, 2 R^2 mod q, 3 R^3 mod q (FieldParams::r / r2) */
sm2b_status gecc_field_params_get(const gecc_field_params* params, int which, uint32_t out[8]);
/* op: GECC_OP_MONT_MUL .. GECC_OP_MOD_INV_FERMAT on the runtime field */
sm2b_status gecc_field_op_rt(sm2b_ctx* ctx, const gecc_field_params* params, gecc_field_opcode op, size_t n,
                             const uint32_t* a, const uint32_t* b, uint32_t* out);
sm2b_status gecc_batch_invert_rt(sm2b_ctx* ctx, const gecc_field_params* params, size_t n, const uint32_t* in,
                                 uint32_t* out);
/* batch_padd / batch_pdbl on y^2 = x^3 + a x + b over F_q; a_mont = a R mod q (b is not needed by
 * the formulas).  Same complete pair classification as gecc_batch_padd. */
sm2b_status gecc_batch_padd_rt(sm2b_ctx* ctx, const gecc_field_params* params, const uint32_t a_mont[8], size_t n,
                               const uint32_t* px, const uint32_t* py, const uint8_t* pinf, const uint32_t* tx,
                               const uint32_t* ty, const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf);
sm2b_status gecc_batch_pdbl_rt(sm2b_ctx* ctx, const gecc_field_params* params, const uint32_t a_mont[8], size_t n,
                               const uint32_t* px, const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                               uint8_t* oinf);

/* Element-wise field operation on column buffers (host pointers). */
sm2b_status gecc_field_op(sm2b_ctx* ctx, gecc_field field, gecc_field_opcode op, size_t n,
                          const uint32_t* a, const uint32_t* b, uint32_t* out);

/* batch_invert (batch_invert.hpp:61-63): element-wise inverse, zero -> zero. */
sm2b_status gecc_batch_invert(sm2b_ctx* ctx, gecc_field field, size_t n, const uint32_t* in,
                              uint32_t* out);
/* batch_padd (batch_point.hpp:47-49): out[i] = p[i] + t[i], complete. */
sm2b_status gecc_batch_padd(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                            const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                            const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf);
/* batch_pdbl (batch_point.hpp:52-53) */
sm2b_status gecc_batch_pdbl(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                            const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf);
/* batch_fpmul (batch_point.hpp:89-91): out[i] = scalars[i] * G, scalars raw 256-bit. */
sm2b_status gecc_batch_fpmul(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, uint32_t* ox,
                             uint32_t* oy, uint8_t* oinf);
/* batch_upmul (batch_point.hpp:72-74): out[i] = scalars[i] * p[i]. */
sm2b_status gecc_batch_upmul(sm2b_ctx* ctx, size_t n, const uint32_t* scalars,
                             const uint32_t* px, const uint32_t* py, const uint8_t* pinf,
                             uint32_t* ox, uint32_t* oy, uint8_t* oinf);
/* MSM (no reference counterpart): out = sum_i scalars[i]*p[i],
 * one affine point (ox, oy: 8 limbs each; *oinf). */
sm2b_status gecc_msm(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                     const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                     uint8_t* oinf);

/* Device-resident forms: identical semantics, all pointers are device memory on
 * the context's device, work is enqueued on the context's stream and NOT
 * synchronised (the caller owns ordering). */
sm2b_status gecc_field_op_dev(sm2b_ctx* ctx, gecc_field field, gecc_field_opcode op, size_t n,
                              const uint32_t* a, const uint32_t* b, uint32_t* out);
sm2b_status gecc_batch_invert_dev(sm2b_ctx* ctx, gecc_field field, size_t n,
                                  const uint32_t* in, uint32_t* out);
sm2b_status gecc_batch_padd_dev(sm2b_ctx* ctx, size_t n, const uint32_t* px,
                                const uint32_t* py, const uint8_t* pinf, const uint32_t* tx,
                                const uint32_t* ty, const uint8_t* tinf, uint32_t* ox,
                                uint32_t* oy, uint8_t* oinf);
sm2b_status gecc_batch_pdbl_dev(sm2b_ctx* ctx, size_t n, const uint32_t* px,
                                const uint32_t* py, const uint8_t* pinf, uint32_t* ox,
                                uint32_t* oy, uint8_t* oinf);
sm2b_status gecc_batch_fpmul_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars,
                                 uint32_t* ox, uint32_t* oy, uint8_t* oinf);
sm2b_status gecc_batch_upmul_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars,
                                 const uint32_t* px, const uint32_t* py, const uint8_t* pinf,
                                 uint32_t* ox, uint32_t* oy, uint8_t* oinf);
sm2b_status gecc_verify_dev(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                            const uint8_t* publics, const uint8_t* signatures,
                            uint8_t* results);
/* Differs from sm2b_sign / gecc_sign in one documented way: nothing is synchronised, so a zero or
 * oversize secret cannot fail the call -- it returns SM2B_OK, the lane's status is
 * SM2B_ERROR_MALFORMED_INPUT (2) and its signature is zeroed; the caller inspects lane_status.
 * nonce_seed == 0 (system entropy) is served by the host forms only. */
sm2b_status gecc_sign_dev(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                          const uint8_t* secrets, uint64_t nonce_seed, uint64_t lane_base,
                          uint8_t* signatures, int32_t* lane_status);
sm2b_status gecc_batch_fpmul_base_dev(sm2b_ctx* ctx, const gecc_base_table* base, size_t n,
                                      const uint32_t* scalars, uint32_t* ox, uint32_t* oy,
                                      uint8_t* oinf);
sm2b_status gecc_msm_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                         const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                         uint8_t* oinf);

/* Form of the batch_invert / batch_padd / batch_pdbl kernels (process-wide; results are
 * identical, batch_invert.hpp:59-60): 0 = by batch size (default), 1 = chunked (every thread
 * runs Montgomery's trick over its own 16 elements), 2 = cooperative (one inversion per thread
 * block: warp-shuffle scans + shared memory). */
void gecc_set_batch_form(int form);

/* Bucket accumulation of gecc_msm (process-wide; results are identical): 0 = default
 * (batch-affine), 1 = mixed Jacobian additions over fixed slices of the sorted pairs,
 * 2 = batch-affine: segmented pairwise tree, affine additions sharing one inversion per
 * thread block, three launches per tree level, 3 = the same with one launch per level. */
void gecc_set_msm_form(int form);

/* Integer-pipe issue-rate microbenchmark (roofline denominator).
 * which: 0 IMAD.WIDE.U32 independent, 1 IMAD.WIDE dependent chain, 2 IMAD (32-bit),
 *        3 IMAD.HI, 4 IADD3, 5 IADD3.X carry chain, 6 IMAD.WIDE + IADD3 1:1 mix,
 *        7 secp256k1 fe_mul (inlined), 8 generic fe_mul, 9 secp256k1 fe_add+fe_sub,
 *        10 secp256k1 fe_mul (by-value call), 11 fe_sqr (inlined), 12 fe_sqr (call).
 * Fills ops_per_clk_per_sm (thread-level operations per SM clock per SM, from
 * clock64 spans) and seconds (CUDA-event time); iters = inner loop trip count. */
sm2b_status gecc_microbench(sm2b_ctx* ctx, int which, int iters, double* ops_per_clk_per_sm,
                            double* seconds, double* total_ops);

#ifdef __cplusplus
}
#endif
#endif /* GECC_B200_H */
