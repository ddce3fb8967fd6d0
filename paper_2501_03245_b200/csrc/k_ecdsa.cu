// Fused ECDSA kernels: one thread = one lane; wire records are decoded, checked,
// processed and re-encoded on the GPU, nothing but the records touches HBM
// (reference path: capi.cpp:145-261 host loops + protocol.cpp:106-263, which
// re-reads all point state from memory for each of 256 bit steps).
#include <cstdlib>
#include <cstring>

#include "gecc_batch.cuh"
#include "gecc_ecdsa.cuh"
#include "gecc_host.h"

namespace gecc {

#ifndef GECC_VERIFY_BLOCKS
#define GECC_VERIFY_BLOCKS 6      // blocks per SM (x 128 lanes): measured 4 / 5 / 6 = 22.70 / 22.10 / 22.03 ms per 2^20 (secp256k1)
#endif
#ifndef GECC_VERIFY_BLOCKS_SM2
#define GECC_VERIFY_BLOCKS_SM2 5  // SM2 (lazy field): 4 / 5 / 6 = 37.4 / 36.6 / 36.6 ms
#endif
constexpr int VERIFY_THREADS = 128;  // x 512 B of lane table = 64 KiB shared memory per block
constexpr int SIGN_THREADS = 128;

// THREADS x BLOCKS_PER_SM is the occupancy knob: the lane tables need 512 B of shared
// memory per lane, so at most 454 lanes (14 warps) fit an SM whatever the block shape.
template <class C, int THREADS, int BLOCKS_PER_SM>
__global__ void __launch_bounds__(THREADS, BLOCKS_PER_SM)
k_verify(size_t n, const uint8_t* __restrict__ dig, const uint8_t* __restrict__ pub,
         const uint8_t* __restrict__ sig, const uint32_t* __restrict__ gtab,
         uint8_t* __restrict__ res) {
    extern __shared__ uint32_t lane_tables[];
    const size_t i = blockIdx.x * (size_t)THREADS + threadIdx.x;
    if (i >= n) return;
    GTable<GECC_WG> gt{gtab};
    LaneTable qt{lane_tables + threadIdx.x, THREADS};
    res[i] = verify_lane<C, GECC_WG>(dig + 32 * i, pub + 65 * i, sig + 64 * i, gt, qt);
}

// Lane tables in global memory (512 B per lane, read back through L2): no shared memory,
// so residency is limited by registers only.
template <class C, int THREADS, int BLOCKS_PER_SM>
__global__ void __launch_bounds__(THREADS, BLOCKS_PER_SM)
k_verify_gtab(size_t n, const uint8_t* __restrict__ dig, const uint8_t* __restrict__ pub,
              const uint8_t* __restrict__ sig, const uint32_t* __restrict__ gtab,
              uint32_t* __restrict__ lane_tables, uint8_t* __restrict__ res) {
    const size_t i = blockIdx.x * (size_t)THREADS + threadIdx.x;
    if (i >= n) return;
    GTable<GECC_WG> gt{gtab};
    LaneTable qt{lane_tables + i * 128, 1};
#if defined(GECC_VERIFY_REGS)
    res[i] = verify_lane<C, GECC_WG>(dig + 32 * i, pub + 65 * i, sig + 64 * i, gt, qt);
#else
    // accumulator and temporaries of the ladder: 8 slots x 32 B per lane of shared memory
    const PointSlots S = block_point_slots<THREADS>();
    res[i] = verify_lane<C, GECC_WG>(dig + 32 * i, pub + 65 * i, sig + 64 * i, gt, qt, &S);
#endif
}

// flags[0] is set when any secret is zero or >= n: the whole call is malformed
// (capi.cpp:181-184) and the host discards the outputs.  Each thread signs SIGN_K
// consecutive lanes and shares the two inversions among them (sign_lanes).
#ifndef GECC_SIGN_SMALL_LOG2
#define GECC_SIGN_SMALL_LOG2 18
#endif
constexpr int SIGN_K_SMALL = 4;
constexpr size_t SIGN_SMALL_MAX = (size_t)1 << GECC_SIGN_SMALL_LOG2;
constexpr int SIGN_K = GECC_SIGN_K;  // gecc_ecdsa.cuh: measured 4 / 8 / 16 lanes per thread = 2.87 / 2.76 / 3.09 ms per 2^20

#ifndef GECC_SIGN_BLOCKS
#define GECC_SIGN_BLOCKS 4
#endif
template <class C, bool UNIFORM, int SIGN_K = GECC_SIGN_K>
__global__ void __launch_bounds__(SIGN_THREADS, GECC_SIGN_BLOCKS)
k_sign(size_t n, const uint8_t* __restrict__ dig, const uint8_t* __restrict__ sec, uint64_t seed,
       uint64_t lane_base, const uint32_t* __restrict__ gtab, uint8_t* __restrict__ sig,
       int32_t* __restrict__ status, uint32_t* __restrict__ flags) {
    const size_t i0 = (blockIdx.x * (size_t)SIGN_THREADS + threadIdx.x) * SIGN_K;
    if (UNIFORM && i0 >= n) return;  // the fast mode meets block-wide barriers below: no early exit there
    GTable<GECC_WG> gt{gtab};
    // accumulator and temporaries of the fixed-base additions rest in shared memory (PointSlots)
    const PointSlots S = block_point_slots<SIGN_THREADS>();
    const PointSlots* slots = UNIFORM ? nullptr : &S;
    fe e[SIGN_K], d[SIGN_K];
    bool all_ok = i0 + SIGN_K <= n;
    // 32- and 64-byte records on 16-byte boundaries: vector loads / stores (uniform over the launch)
    const bool al_in = ptr_aligned16(dig) && ptr_aligned16(sec), al_out = ptr_aligned16(sig);
#pragma unroll 1
    for (int j = 0; j < SIGN_K && i0 + j < n; ++j) {
        d[j] = be32_load_a(sec + 32 * (i0 + j), al_in);
        e[j] = scalar_reduce_once<typename C::Fn>(be32_load_a(dig + 32 * (i0 + j), al_in));
        if (!scalar_in_range<typename C::Fn>(d[j])) all_ok = false;
    }
    if constexpr (!UNIFORM) {
        // The two inversions of a group (its denominators mod p, its nonces mod n) are shared by the
        // whole BLOCK: warp-shuffle scans over the 128 group totals and one warp-cooperative safegcd
        // each (coop_block_inverse) instead of two safegcd chains per thread.  Every thread of the
        // block takes part; a thread without a full valid group contributes 1.
        __shared__ uint32_t sm_scan[2 * 8 * (SIGN_THREADS / 32)];
        const typename C::Fp fp{};
        const typename C::Fn fn{};
        SignGroup<SIGN_K> g;
        fe tz = fe_one(fp), tk = fe_one(fn);
        if (all_ok) {
            sign_lanes_walk<C, GECC_WG, SIGN_K, false>(seed, lane_base + i0, gt, slots, g);
            tz = g.pz[SIGN_K - 1];
            tk = g.pk[SIGN_K - 1];
        }
        const fe iz = coop_block_inverse<decltype(fp), SIGN_THREADS>(fp, tz, sm_scan);
        __syncthreads();  // sm_scan is reused
        // the Montgomery-domain inverse of the residue tk is R^2 / tk; one reduction makes it R / tk
        const fe ik = fe_from_mont(fn, coop_block_inverse<decltype(fn), SIGN_THREADS>(fn, tk, sm_scan));
        if (all_ok) {
            int st[SIGN_K];
            sign_lanes_finish<C, GECC_WG, SIGN_K, false>(e, d, seed, lane_base + i0, gt, sig + 64 * i0, st, al_out, slots, g, iz, ik);
#pragma unroll
            for (int j = 0; j < SIGN_K; ++j) status[i0 + j] = st[j];
            return;
        }
        if (i0 >= n) return;
    } else if (all_ok) {
        int st[SIGN_K];
        sign_lanes<C, GECC_WG, SIGN_K, UNIFORM>(e, d, seed, lane_base + i0, gt, sig + 64 * i0, st, al_out, slots);
#pragma unroll
        for (int j = 0; j < SIGN_K; ++j) status[i0 + j] = st[j];
        return;
    }
    // ragged tail or a malformed secret in this group: lane by lane
#pragma unroll 1
    for (int j = 0; j < SIGN_K && i0 + j < n; ++j) {
        const size_t i = i0 + j;
        if (!scalar_in_range<typename C::Fn>(d[j])) {
            atomicOr(flags, 1u);
            status[i] = 2;
            for (int b = 0; b < 64; ++b) sig[64 * i + b] = 0;
            continue;
        }
        status[i] = sign_lane<C, GECC_WG, UNIFORM>(e[j], d[j], seed, lane_base + i, gt, sig + 64 * i, 0, slots);
    }
}

// One attempt per lane with caller-supplied nonces (gecc_sign_nonces; the step that
// ecdsa_sign_batch repeats for the lanes still pending, protocol.cpp:121-164).
template <class C, bool UNIFORM>
__global__ void __launch_bounds__(SIGN_THREADS)
k_sign_nonces(size_t n, const uint8_t* __restrict__ dig, const uint8_t* __restrict__ sec,
              const uint8_t* __restrict__ nonces, const uint32_t* __restrict__ gtab,
              uint8_t* __restrict__ sig, int32_t* __restrict__ status, uint32_t* __restrict__ flags) {
    const size_t i = blockIdx.x * (size_t)SIGN_THREADS + threadIdx.x;
    if (i >= n) return;
    GTable<GECC_WG> gt{gtab};
    const fe d = be32_load(sec + 32 * i);
    if (!scalar_in_range<typename C::Fn>(d)) {
        atomicOr(flags, 1u);
        status[i] = 2;
        for (int b = 0; b < 64; ++b) sig[64 * i + b] = 0;
        return;
    }
    const fe e = scalar_reduce_once<typename C::Fn>(be32_load(dig + 32 * i));
    status[i] = sign_lane_nonce<C, GECC_WG, UNIFORM>(e, d, be32_load(nonces + 32 * i), gt, sig + 64 * i);
}

// Range check of all secrets of a call (capi.cpp:181-184: one bad secret fails the WHOLE call
// before any output is written).  Run right after the secrets are uploaded, so that the host
// knows the verdict early and can stream the signatures out while later chunks still sign.
template <class C>
__global__ void __launch_bounds__(256)
k_secret_range(size_t n, const uint8_t* __restrict__ sec, uint32_t* __restrict__ flags) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!scalar_in_range<typename C::Fn>(be32_load(sec + 32 * i))) atomicOr(flags, 1u);
}

// capi.cpp:145-169: secret = nonce stream (lane, attempt 0), public = secret * G
template <class C, bool UNIFORM>
__global__ void __launch_bounds__(SIGN_THREADS)
k_keygen(size_t n, uint64_t seed, uint64_t lane_base, const uint32_t* __restrict__ gtab,
         uint8_t* __restrict__ sec, uint8_t* __restrict__ pub) {
    const size_t i = blockIdx.x * (size_t)SIGN_THREADS + threadIdx.x;
    const typename C::Fp f{};
    GTable<GECC_WG> gt{gtab};
    if constexpr (UNIFORM) {  // constant structure: every lane inverts its own Z with the branch-free rounds
        if (i >= n) return;
        fe d = nonce_scalar<typename C::Fn>(seed, lane_base + i, 0);
        be32_store(sec + 32 * i, d);
        jac r = fixed_base_mul_mode<C, GECC_WG, true>(d, gt, nullptr);
        encode_point<C>(pub + 65 * i, jac_to_aff_with<C>(r, fe_inv(f, r.Z)));
    } else {
        // the block's Z coordinates share ONE inversion (warp-shuffle scans + the warp-cooperative
        // safegcd of coop_block_inverse) instead of one safegcd per lane; lanes past n carry 1
        __shared__ uint32_t sm_scan[2 * C::Fp::N * (SIGN_THREADS / 32)];
        const bool live = i < n;
        jac r = jac_infinity<C>();
        fe z = fe_one(f);
        if (live) {
            fe d = nonce_scalar<typename C::Fn>(seed, lane_base + i, 0);
            be32_store(sec + 32 * i, d);
            const PointSlots S = block_point_slots<SIGN_THREADS>();
            r = fixed_base_mul_mode<C, GECC_WG, false>(d, gt, &S);
            z = r.Z;  // never zero for 0 < d < n
        }
        const fe zinv = coop_block_inverse<decltype(f), SIGN_THREADS>(f, z, sm_scan);
        if (live) encode_point<C>(pub + 65 * i, jac_to_aff_with<C>(r, zinv));
    }
}

// capi.cpp:230-261 + protocol.cpp:224-263.  status: 0 ok, 3 invalid peer,
// 4 degenerate; a secret >= n flags the whole call malformed.
template <class C, bool UNIFORM>
__global__ void __launch_bounds__(VERIFY_THREADS, 4)
k_ecdh(size_t n, const uint8_t* __restrict__ sec, const uint8_t* __restrict__ peers,
       uint8_t* __restrict__ shared, int32_t* __restrict__ status, uint32_t* __restrict__ flags,
       uint32_t* __restrict__ lane_tables) {
    const size_t i = blockIdx.x * (size_t)VERIFY_THREADS + threadIdx.x;
    if (i >= n) return;
    const typename C::Fp f{};
    LaneTable qt{lane_tables + i * 128, 1};
    for (int b = 0; b < 32; ++b) shared[32 * i + b] = 0;
    fe d = be32_load(sec + 32 * i);
    if (!fe_lt_modulus(typename C::Fn{}, d)) {  // Scalar::checked: zero is allowed here
        atomicOr(flags, 1u);
        status[i] = 2;
        return;
    }
    aff p;
    if (!decode_point<C>(peers + 65 * i, &p)) {
        status[i] = 3;
        return;
    }
    const PointSlots S = block_point_slots<VERIFY_THREADS>();
    jac r;
    if constexpr (UNIFORM) {
        build_lane_table<C>(p, qt);
        r = var_base_mul_uniform<C>(d, qt);
    } else {
        var_base_mul_point_slots<C>(d, p, qt, S);
        r = S.load_point();
    }
    if (jac_is_inf<C>(r)) {
        status[i] = 4;
        return;
    }
    fe zinv = fe_inv(f, r.Z);
    be32_store(shared + 32 * i, fe_from_mont(f, fe_mul(f, r.X, fe_sqr(f, zinv))));
    status[i] = 0;
}

// ---- column-buffer forms of the two multiplication kernels (batch_point.hpp:72-91)
template <class C>
__device__ __forceinline__ void store_affine(const jac& r, uint32_t* ox, uint32_t* oy,
                                             uint8_t* oinf, size_t n, size_t i) {
    const typename C::Fp f{};
    if (jac_is_inf<C>(r)) {  // infinity coordinates are normalised to zero (batch_point.cpp:41-47)
        col_store(ox, n, i, fe_zero());
        col_store(oy, n, i, fe_zero());
        oinf[i] = 1;
        return;
    }
    aff a = jac_to_aff_with<C>(r, fe_inv(f, r.Z));
    col_store(ox, n, i, a.x);
    col_store(oy, n, i, a.y);
    oinf[i] = 0;
}

template <class C>
__global__ void __launch_bounds__(SIGN_THREADS)
k_fpmul(size_t n, const uint32_t* __restrict__ k, const uint32_t* __restrict__ gtab,
        uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    const size_t i = blockIdx.x * (size_t)SIGN_THREADS + threadIdx.x;
    if (i >= n) return;
    GTable<GECC_WG> gt{gtab};
    const PointSlots S = block_point_slots<SIGN_THREADS>();
    store_affine<C>(fixed_base_mul_mode<C, GECC_WG, false>(col_load(k, n, i), gt, &S), ox, oy, oinf, n, i);
}

template <class C>
__global__ void __launch_bounds__(VERIFY_THREADS, 4)
k_upmul(size_t n, const uint32_t* __restrict__ k, const uint32_t* __restrict__ px,
        const uint32_t* __restrict__ py, const uint8_t* __restrict__ pinf,
        uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf,
        uint32_t* __restrict__ lane_tables) {
    const size_t i = blockIdx.x * (size_t)VERIFY_THREADS + threadIdx.x;
    if (i >= n) return;
    LaneTable qt{lane_tables + i * 128, 1};
    if (pinf && pinf[i]) {  // infinity input stays infinity (test_batch_point.cpp:231,244)
        store_affine<C>(jac_infinity<C>(), ox, oy, oinf, n, i);
        return;
    }
    aff p{col_load(px, n, i), col_load(py, n, i)};
    const PointSlots S = block_point_slots<VERIFY_THREADS>();
    var_base_mul_point_slots<C>(col_load(k, n, i), p, qt, S);
    store_affine<C>(S.load_point(), ox, oy, oinf, n, i);
}

// ---- sm2b_bench_run support (bench.cpp:20-62): seeded inputs and the "jacobian-serial"
// strategy as independent per-lane kernels
template <class C>
__global__ void __launch_bounds__(256)
k_seeded_scalars(size_t n, uint64_t seed, uint64_t tag, uint32_t* __restrict__ out) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    col_store(out, n, i, nonce_scalar<typename C::Fn>(seed, tag + i, 0));  // bench.cpp:20-28
}

// serial_padd (bench.cpp:50-60): one mixed Jacobian addition per lane, normalised to affine
template <class C>
__global__ void __launch_bounds__(SIGN_THREADS)
k_padd_jacobian(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx,
                const uint32_t* __restrict__ ty, const uint8_t* __restrict__ tinf,
                uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    const size_t i = blockIdx.x * (size_t)SIGN_THREADS + threadIdx.x;
    if (i >= n) return;
    const typename C::Fp f{};
    jac acc = jac_infinity<C>();
    if (!(pinf && pinf[i])) {
        acc.X = col_load(px, n, i);
        acc.Y = col_load(py, n, i);
        acc.Z = fe_one(f);
    }
    if (!(tinf && tinf[i])) acc = jac_madd<C>(acc, aff{col_load(tx, n, i), col_load(ty, n, i)});
    store_affine<C>(acc, ox, oy, oinf, n, i);
}

// pmul_serial (curve.cpp:176-185): LSB-first double-and-add, no tables, no recoding --
// deliberately a different algorithm from k_fpmul / k_upmul so that comparing them is a
// real equivalence check.  px == nullptr multiplies the generator.
template <class C>
__global__ void __launch_bounds__(SIGN_THREADS)
k_pmul_serial(size_t n, const uint32_t* __restrict__ k, const uint32_t* __restrict__ px,
              const uint32_t* __restrict__ py, const uint8_t* __restrict__ pinf,
              uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    const size_t i = blockIdx.x * (size_t)SIGN_THREADS + threadIdx.x;
    if (i >= n) return;
    const typename C::Fp f{};
    fe s = col_load(k, n, i);
    jac acc = jac_infinity<C>(), run = jac_infinity<C>();
    if (!px) {
        aff g = curve_g<C>();
        run.X = g.x; run.Y = g.y; run.Z = fe_one(f);
    } else if (!(pinf && pinf[i])) {
        run.X = col_load(px, n, i); run.Y = col_load(py, n, i); run.Z = fe_one(f);
    }
#pragma unroll 1
    for (int b = 0; b < 256; ++b) {
        if ((s.w[b >> 5] >> (b & 31)) & 1u) acc = jac_add<C>(acc, run);
        run = jac_dbl<C>(run);
    }
    store_affine<C>(acc, ox, oy, oinf, n, i);
}

// ---------------------------------------------------------------- launchers
static int blocks_for(size_t n, int threads) { return (int)((n + threads - 1) / threads); }

#define GECC_BY_CURVE(curve, EXPR_SECP, EXPR_SM2) \
    do {                                          \
        if ((curve) == CURVE_SECP) { EXPR_SECP; } \
        else { EXPR_SM2; }                        \
    } while (0)
// The byte-record (ECDSA / keygen / ECDH) kernels run secp256k1 in the lazy plain
// representation (SecpLCurve, its own fixed-base table); the column-buffer kernels keep
// the reference's Montgomery form (SecpCurve) because that is their I/O contract.
using SecpEcdsaCurve = SecpLCurve;
// SM2 likewise computes on its weakly reduced Montgomery field inside the byte-record kernels
// (Sm2LCurve: same Montgomery form and the same fixed-base table, carry / borrow folds instead of
// trial subtractions); the column-buffer kernels keep the canonical field.
using Sm2EcdsaCurve = Sm2LCurve;

template <class C, int THREADS, int BLOCKS_PER_SM>
static cudaError_t launch_verify_t(size_t n, const uint8_t* dig, const uint8_t* pub, const uint8_t* sig,
                                   const uint32_t* gtab, uint8_t* res, cudaStream_t s) {
    const size_t smem = (size_t)THREADS * 8 * 16 * sizeof(uint32_t);
    cudaError_t e = cudaFuncSetAttribute(k_verify<C, THREADS, BLOCKS_PER_SM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_verify<C, THREADS, BLOCKS_PER_SM><<<blocks_for(n, THREADS), THREADS, smem, s>>>(n, dig, pub, sig, gtab, res);
    return cudaGetLastError();
}

// Production shape: lane tables in global memory, 128 threads x 4 blocks per SM (16 warps,
// 128 registers): measured 26.6 ms per 2^20 against 28.9 ms for the shared-memory shape
// (12 warps; 512 B of shared memory per lane caps an SM at 14 warps).  The resident lanes'
// tables (148 x 512 lanes x 512 B = 39 MB) stay in the 126 MB L2; each entry is one 64-byte
// vector read.  GECC_VERIFY_SHAPE=smem selects the shared-memory kernel for comparison.
size_t verify_scratch_bytes(size_t lanes) { return lanes * 512; }

cudaError_t launch_verify(int curve, size_t n, const uint8_t* dig, const uint8_t* pub,
                          const uint8_t* sig, const uint32_t* gtab, uint8_t* res,
                          uint32_t* lane_scratch, size_t scratch_lanes, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    static const bool use_smem = [] {
        const char* v = getenv("GECC_VERIFY_SHAPE");
        return v && !strcmp(v, "smem");
    }();
    if (use_smem || !lane_scratch || scratch_lanes == 0) {
        if (curve == CURVE_SECP) return launch_verify_t<SecpEcdsaCurve, 128, 3>(n, dig, pub, sig, gtab, res, s);
        return launch_verify_t<Sm2EcdsaCurve, 128, 3>(n, dig, pub, sig, gtab, res, s);
    }
    // kernels on one stream run back to back, so consecutive pieces may reuse the scratch
    // 4 blocks per SM (128 registers) measured best: 3 / 4 / 5 / 6 blocks = 26.4 / 25.5 / 27.1 / 29.2 ms
    for (size_t at = 0; at < n; at += scratch_lanes) {
        const size_t m = n - at < scratch_lanes ? n - at : scratch_lanes;
        const int b = blocks_for(m, 128);
        const size_t slot_bytes = 0;  // the ladder's slots are a static shared array of the kernel (32 KB per block)
        if (curve == CURVE_SECP)
            k_verify_gtab<SecpEcdsaCurve, 128, GECC_VERIFY_BLOCKS><<<b, 128, slot_bytes, s>>>(m, dig + 32 * at, pub + 65 * at, sig + 64 * at,
                                                                             gtab, lane_scratch, res + at);
        else
            k_verify_gtab<Sm2EcdsaCurve, 128, GECC_VERIFY_BLOCKS_SM2><<<b, 128, slot_bytes, s>>>(m, dig + 32 * at, pub + 65 * at, sig + 64 * at, gtab,
                                                                       lane_scratch, res + at);
    }
    return cudaGetLastError();
}

cudaError_t launch_secret_range(int curve, size_t n, const uint8_t* sec, uint32_t* flags, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned b = (unsigned)((n + 255) / 256);
    if (curve == CURVE_SECP) k_secret_range<SecpEcdsaCurve><<<b, 256, 0, s>>>(n, sec, flags);
    else k_secret_range<Sm2Curve><<<b, 256, 0, s>>>(n, sec, flags);
    return cudaGetLastError();
}

#define GECC_BY_CURVE_MODE_SMEM(curve, uniform, KERNEL, GRID, THREADS, SMEM, ...)                  \
    do {                                                                                           \
        if ((curve) == CURVE_SECP) {                                                               \
            if (uniform) KERNEL<SecpEcdsaCurve, true><<<GRID, THREADS, SMEM, s>>>(__VA_ARGS__);    \
            else KERNEL<SecpEcdsaCurve, false><<<GRID, THREADS, SMEM, s>>>(__VA_ARGS__);           \
        } else {                                                                                   \
            if (uniform) KERNEL<Sm2EcdsaCurve, true><<<GRID, THREADS, SMEM, s>>>(__VA_ARGS__);     \
            else KERNEL<Sm2EcdsaCurve, false><<<GRID, THREADS, SMEM, s>>>(__VA_ARGS__);            \
        }                                                                                          \
    } while (0)
#define GECC_BY_CURVE_MODE(curve, uniform, KERNEL, GRID, THREADS, ...) \
    GECC_BY_CURVE_MODE_SMEM(curve, uniform, KERNEL, GRID, THREADS, 0, __VA_ARGS__)

cudaError_t launch_sign(int curve, size_t n, const uint8_t* dig, const uint8_t* sec, uint64_t seed,
                        uint64_t lane_base, const uint32_t* gtab, uint8_t* sig, int32_t* status,
                        uint32_t* flags, cudaStream_t s, bool uniform) {
    if (n == 0) return cudaSuccess;
    // lanes per thread: SIGN_K (8) shares the two inversions best; a launch that would leave the chip
    // half empty at 8 (the chunks of the host pipeline, small batches) takes 4 and twice the blocks
    if (!uniform && n <= SIGN_SMALL_MAX) {
        const int b = blocks_for((n + SIGN_K_SMALL - 1) / SIGN_K_SMALL, SIGN_THREADS);
        if (curve == CURVE_SECP)
            k_sign<SecpEcdsaCurve, false, SIGN_K_SMALL><<<b, SIGN_THREADS, 0, s>>>(n, dig, sec, seed, lane_base, gtab, sig, status, flags);
        else
            k_sign<Sm2EcdsaCurve, false, SIGN_K_SMALL><<<b, SIGN_THREADS, 0, s>>>(n, dig, sec, seed, lane_base, gtab, sig, status, flags);
        return cudaGetLastError();
    }
    const int b = blocks_for((n + SIGN_K - 1) / SIGN_K, SIGN_THREADS);
    GECC_BY_CURVE_MODE(curve, uniform, k_sign, b, SIGN_THREADS, n, dig, sec, seed, lane_base, gtab, sig, status, flags);
    return cudaGetLastError();
}

cudaError_t launch_sign_nonces(int curve, size_t n, const uint8_t* dig, const uint8_t* sec,
                               const uint8_t* nonces, const uint32_t* gtab, uint8_t* sig, int32_t* status,
                               uint32_t* flags, cudaStream_t s, bool uniform) {
    if (n == 0) return cudaSuccess;
    const int b = blocks_for(n, SIGN_THREADS);
    GECC_BY_CURVE_MODE(curve, uniform, k_sign_nonces, b, SIGN_THREADS, n, dig, sec, nonces, gtab, sig, status, flags);
    return cudaGetLastError();
}

cudaError_t launch_keygen(int curve, size_t n, uint64_t seed, uint64_t lane_base,
                          const uint32_t* gtab, uint8_t* sec, uint8_t* pub, cudaStream_t s, bool uniform) {
    if (n == 0) return cudaSuccess;
    const int b = blocks_for(n, SIGN_THREADS);
    GECC_BY_CURVE_MODE(curve, uniform, k_keygen, b, SIGN_THREADS, n, seed, lane_base, gtab, sec, pub);
    return cudaGetLastError();
}

cudaError_t launch_ecdh(int curve, size_t n, const uint8_t* sec, const uint8_t* peers,
                        uint8_t* shared, int32_t* status, uint32_t* flags, uint32_t* lane_scratch,
                        size_t scratch_lanes, cudaStream_t s, bool uniform) {
    if (n == 0) return cudaSuccess;
    if (!lane_scratch || scratch_lanes == 0) return cudaErrorInvalidValue;
    for (size_t at = 0; at < n; at += scratch_lanes) {
        const size_t m = n - at < scratch_lanes ? n - at : scratch_lanes;
        const int b = blocks_for(m, VERIFY_THREADS);
        GECC_BY_CURVE_MODE(curve, uniform, k_ecdh, b, VERIFY_THREADS, m, sec + 32 * at, peers + 65 * at,
                           shared + 32 * at, status + at, flags, lane_scratch);
    }
    return cudaGetLastError();
}

cudaError_t launch_fpmul(int curve, size_t n, const uint32_t* k, const uint32_t* gtab, uint32_t* ox,
                         uint32_t* oy, uint8_t* oinf, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int b = blocks_for(n, SIGN_THREADS);
    GECC_BY_CURVE(curve,
        (k_fpmul<SecpCurve><<<b, SIGN_THREADS, 0, s>>>(n, k, gtab, ox, oy, oinf)),
        (k_fpmul<Sm2Curve><<<b, SIGN_THREADS, 0, s>>>(n, k, gtab, ox, oy, oinf)));
    return cudaGetLastError();
}

// column buffers are indexed k*n + i, so pieces are not contiguous: the scratch must cover n
cudaError_t launch_upmul(int curve, size_t n, const uint32_t* k, const uint32_t* px,
                         const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                         uint8_t* oinf, uint32_t* lane_scratch, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (!lane_scratch) return cudaErrorInvalidValue;
    const int b = blocks_for(n, VERIFY_THREADS);
    GECC_BY_CURVE(curve,
        (k_upmul<SecpCurve><<<b, VERIFY_THREADS, 0, s>>>(n, k, px, py, pinf, ox, oy, oinf, lane_scratch)),
        (k_upmul<Sm2Curve><<<b, VERIFY_THREADS, 0, s>>>(n, k, px, py, pinf, ox, oy, oinf, lane_scratch)));
    return cudaGetLastError();
}

cudaError_t launch_seeded_scalars(int curve, size_t n, uint64_t seed, uint64_t tag, uint32_t* out,
                                  cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int b = blocks_for(n, 256);
    GECC_BY_CURVE(curve, (k_seeded_scalars<SecpCurve><<<b, 256, 0, s>>>(n, seed, tag, out)),
                  (k_seeded_scalars<Sm2Curve><<<b, 256, 0, s>>>(n, seed, tag, out)));
    return cudaGetLastError();
}
cudaError_t launch_padd_jacobian(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                                 const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                                 const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                                 cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int b = blocks_for(n, SIGN_THREADS);
    GECC_BY_CURVE(curve,
        (k_padd_jacobian<SecpCurve><<<b, SIGN_THREADS, 0, s>>>(n, px, py, pinf, tx, ty, tinf, ox, oy, oinf)),
        (k_padd_jacobian<Sm2Curve><<<b, SIGN_THREADS, 0, s>>>(n, px, py, pinf, tx, ty, tinf, ox, oy, oinf)));
    return cudaGetLastError();
}
cudaError_t launch_pmul_serial(int curve, size_t n, const uint32_t* k, const uint32_t* px,
                               const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                               uint8_t* oinf, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int b = blocks_for(n, SIGN_THREADS);
    GECC_BY_CURVE(curve,
        (k_pmul_serial<SecpCurve><<<b, SIGN_THREADS, 0, s>>>(n, k, px, py, pinf, ox, oy, oinf)),
        (k_pmul_serial<Sm2Curve><<<b, SIGN_THREADS, 0, s>>>(n, k, px, py, pinf, ox, oy, oinf)));
    return cudaGetLastError();
}

}  // namespace gecc
