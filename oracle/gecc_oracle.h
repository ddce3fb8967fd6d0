/* TEST INFRASTRUCTURE ONLY.
 *
 * gecc_oracle -- a plain-C, single-threaded CPU restatement of the reference's
 * batched elliptic-curve path (sm2batch 1.0.0 under /root/reference/proj), with
 * the curve made a parameter so that the same algorithm also runs on secp256k1.
 *
 * Parity status:
 *   - SM2 (curve 0): PINNED.  Every entry point is checked against the compiled,
 *     unmodified reference (oracle/_ref) and against committed golden vectors
 *     generated from it (tests/golden/, tests/test_oracle_*.py).
 *   - secp256k1 (curve 1) field / point / batch kernels: PINNED against the
 *     reference's own generic-q kernels run on a hand-built CurveParams.
 *   - secp256k1 ECDSA glue: the reference hard-wires SM2's n in its protocol
 *     layer, so there is no reference output for it; it is pinned against the
 *     same restated glue driving the reference's kernels (oracle/ref_shim.cpp)
 *     and the independent Python-int textbook oracle (oracle/pyec.py).
 *   - MSM: no reference implementation exists ("parity unpinned" for MSM); the
 *     oracle is the definition sum_i s_i * P_i built from pmul_serial.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU arm may load this
 * library.  The product (libgecc_b200.so) never links or calls it.
 *
 * Layout conventions (identical to the product's C ABI):
 *   "cols"  : column-major limbs, limb k of element i at cols[k*n + i], LSW first
 *             (batch_buffer.hpp:15-35).  Field elements in cols are in Montgomery
 *             form (R = 2^256) unless stated otherwise; scalars are plain.
 *   "inf"   : one byte per element, 1 = point at infinity.
 *   records : big-endian bytes as in sm2batch.h:4-9.
 */
#ifndef GECC_ORACLE_H
#define GECC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GO_CURVE_SM2 = 0, GO_CURVE_SECP256K1 = 1 };
enum { GO_FIELD_P = 0, GO_FIELD_N = 1 };

/* field.cpp:159-179 -- returns q_inv; q, r, r2 are 8 limbs each */
uint32_t go_field_params(int curve, int which, uint32_t* q, uint32_t* r, uint32_t* r2);
/* a, b, Gx, Gy in Montgomery form */
void go_curve_params(int curve, uint32_t* a, uint32_t* b, uint32_t* gx, uint32_t* gy);

/* op: 0 mont_mul 1 mod_add 2 mod_sub 3 to_mont 4 from_mont 5 mod_inv (0 -> 0) */
int go_field_op(int curve, int which, int op, size_t n, const uint32_t* a,
                const uint32_t* b, uint32_t* out);
/* c16: 16 columns per element; route 0 generic SOS, 1 SM2 add/sub-only */
int go_mont_reduce(int curve, int which, int sm2_route, size_t n, const uint32_t* c16,
                   uint32_t* out);

int go_batch_invert(int curve, int which, size_t n, const uint32_t* in, uint32_t* out,
                    size_t lanes);
int go_batch_padd(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                  const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                  const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                  size_t lanes);
int go_batch_pdbl(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                  const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                  size_t lanes);
int go_batch_fpmul(int curve, size_t n, const uint32_t* scalars, uint32_t* ox,
                   uint32_t* oy, uint8_t* oinf, size_t lanes);
int go_batch_upmul(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                   const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                   uint8_t* oinf, size_t lanes);
int go_pmul_serial(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                   const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                   uint8_t* oinf);
/* sum_i scalars[i]*P[i] (definition; affine result, Montgomery form) */
int go_msm(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
           const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
           uint8_t* oinf);

void go_nonce(int curve, uint64_t seed, uint64_t stream, uint32_t attempt, uint8_t* out32);

/* byte-record entry points; return an sm2b_status value (sm2batch.h:27-36) */
int go_keygen(int curve, uint64_t seed, uint64_t lane_base, size_t count,
              uint8_t* secrets, uint8_t* publics, size_t lanes);
int go_sign(int curve, size_t count, const uint8_t* digests, const uint8_t* secrets,
            uint64_t nonce_seed, uint64_t lane_base, uint8_t* signatures,
            int32_t* lane_status, size_t lanes);
int go_verify(int curve, size_t count, const uint8_t* digests, const uint8_t* publics,
              const uint8_t* signatures, uint8_t* results, size_t lanes);
int go_ecdh(int curve, size_t count, const uint8_t* secrets, const uint8_t* peers,
            uint8_t* shared, int32_t* lane_status, size_t lanes);

/* operation ledger of the calling thread (field.hpp:19-47): modmul, modadd, modsub, modinv */
void go_ledger_read(uint64_t out[4]);
void go_ledger_reset(void);

#ifdef __cplusplus
}
#endif
#endif
