// Shared device helpers of the batched-affine kernels (k_batch.cu, k_msm.cu):
// the complete pair classification of batch_padd (batch_point.cpp:91-111), the
// chord / tangent finish (batch_point.cpp:124-170) and the block-level Montgomery
// trick (warp-shuffle scans + shared memory, one inversion per thread block).
#pragma once
#include <type_traits>
#include "gecc_curve.cuh"
#include "gecc_dev.cuh"
#include "gecc_modinv.cuh"

namespace gecc {

enum : uint32_t { K_GENERIC = 0, K_TANGENT, K_INFINITY, K_COPY_LEFT, K_COPY_RIGHT };

// secp256k1 column buffers hold Montgomery representatives x~ = x R (the reference's I/O contract),
// but R = 2^256 = c (mod p) is tiny, so the affine formulas can run on the PLAIN weakly reduced
// field directly on the representatives, without ever converting:
//   lambda   = (y1~ - y2~) / (x1~ - x2~)            the factors R cancel: the plain slope
//   x3~      = c lambda^2 - x1~ - x2~                 one multiplication by c = 2^32 + 977 (a fold)
//   y3~      = lambda (x1~ - x3~) - y1~               already scaled
//   tangent  : lambda = 3 (x~^2 R^-1) / (2 y~)        one more product, on doubling lanes only
// Montgomery's trick runs on the plain denominators d~ (their plain inverses are what lambda
// needs).  Products cost 72 wide multiplies with a shallow fold instead of the word-serial
// Montgomery reduction, additions fold a carry instead of compare-and-select; results are made
// canonical when they are stored.
struct SecpMLCurve : SecpLCurve {
    static constexpr bool mont_reps = true;
    GECC_HD static constexpr uint32_t rinv(int i) {  // (2^256)^-1 mod p
        constexpr uint32_t t[8] = {0x0868192Au, 0xD838091Du, 0xDC24A059u, 0xBCB223FEu, 0x95F2B761u, 0x9C46C2C2u, 0x15538399u, 0xC9BD1905u};
        return t[i];
    }
};
template <class C, class = void>
struct curve_mont_reps : std::false_type {};
template <class C>
struct curve_mont_reps<C, std::void_t<decltype(C::mont_reps)>> : std::bool_constant<C::mont_reps> {};

// a * 2^256 mod p = a * c, weakly reduced: the product fold applied to (a : 0)
__device__ __forceinline__ fe lazy_times_r(const fe& a) {
    uint32_t t[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        t[i] = 0;
        t[8 + i] = a.w[i];
    }
    return redc_secp_lazy(t);
}

// classification + denominator of one pair (batch_point.cpp:91-111)
template <class C>
__device__ __forceinline__ uint32_t classify_pair(const cfe<C>& px, const cfe<C>& py, bool pinf,
                                                  const cfe<C>& tx, const cfe<C>& ty, bool tinf, cfe<C>* d) {
    const typename C::Fp f{};
    if (pinf && tinf) return K_INFINITY;
    if (pinf) return K_COPY_RIGHT;
    if (tinf) return K_COPY_LEFT;
    if (fe_eq(f, px, tx)) {  // field-aware: a weakly reduced field compares mod q
        if (fe_eq(f, py, ty) && !fe_is_zero(f, py)) {
            *d = fe_dbl(f, py);
            return K_TANGENT;
        }
        return K_INFINITY;  // inverse pair (covers y == 0)
    }
    *d = fe_sub(f, px, tx);
    return K_GENERIC;
}

template <class C>
__device__ __forceinline__ void finish_lambda(const cfe<C>& lam, const cfe<C>& x1, const cfe<C>& x2,
                                              const cfe<C>& y1, cfe<C>* xr, cfe<C>* yr) {
    const typename C::Fp f{};
    if constexpr (curve_mont_reps<C>::value) {
        cfe<C> x3 = fe_sub(f, fe_sub(f, lazy_times_r(fe_sqr(f, lam)), x1), x2);
        *yr = lazy_canon(f, fe_sub(f, fe_mul(f, lam, fe_sub(f, x1, x3)), y1));
        *xr = lazy_canon(f, x3);
    } else {
        *xr = fe_sub(f, fe_sub(f, fe_sqr(f, lam), x1), x2);
        *yr = fe_sub(f, fe_mul(f, lam, fe_sub(f, x1, *xr)), y1);
    }
}
template <class C>
__device__ __forceinline__ cfe<C> tangent_numerator(const cfe<C>& x) {  // 3x^2 + a
    const typename C::Fp f{};
    cfe<C> x2 = fe_sqr(f, x);
    if constexpr (curve_mont_reps<C>::value) {  // x~^2 R^-1 = x^2 R
        cfe<C> ri;
#pragma unroll
        for (int i = 0; i < 8; ++i) ri.w[i] = C::rinv(i);
        x2 = fe_mul(f, x2, ri);
    }
    cfe<C> num = fe_add(f, fe_dbl(f, x2), x2);
    if (C::a_kind == A_ZERO) return num;
    return fe_add(f, num, curve_a<C>());
}

template <int N>
__device__ __forceinline__ feN<N> fe_shfl_up(const feN<N>& v, int d) {
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = __shfl_up_sync(0xFFFFFFFFu, v.w[i], d);
    return r;
}
template <int N>
__device__ __forceinline__ feN<N> fe_shfl_down(const feN<N>& v, int d) {
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = __shfl_down_sync(0xFFFFFFFFu, v.w[i], d);
    return r;
}
template <int N>
__device__ __forceinline__ feN<N> fe_shfl(const feN<N>& v, int src) {
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = __shfl_sync(0xFFFFFFFFu, v.w[i], src);
    return r;
}
// inclusive prefix product P and inclusive suffix product Q of t over the 32 lanes of a warp
template <class F>
__device__ __forceinline__ void warp_scan_products(const F& f, const fel<F>& t, int lane, int width,
                                                   fel<F>* P, fel<F>* Q) {
    using fe = fel<F>;
    *P = t;
    *Q = t;
#pragma unroll 1
    for (int d = 1; d < width; d <<= 1) {
        fe m = fe_mul(f, *P, fe_shfl_up(*P, d));
        *P = fe_select(lane >= d, m, *P);
        fe m2 = fe_mul(f, *Q, fe_shfl_down(*Q, d));
        *Q = fe_select(lane + d < 32, m2, *Q);
    }
}
// t != 0 on every thread of the block (all COOP_THREADS threads must call).  Returns t^-1.
// sm: 2 * (COOP_THREADS / 32) field elements (2 * F::N * COOP_THREADS / 32 words) of shared
// memory, word-major.
template <class F, int COOP_THREADS>
__device__ fel<F> coop_block_inverse(const F& f, const fel<F>& t, uint32_t* sm) {
    using fe = fel<F>;
    constexpr int NL = F::N;
    constexpr int NW = COOP_THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const fe one = fe_one(f);
    fe P, Q;
    warp_scan_products(f, t, lane, 32, &P, &Q);
    fe E = fe_select(lane == 0, one, fe_shfl_up(P, 1));    // exclusive prefix
    fe S = fe_select(lane == 31, one, fe_shfl_down(Q, 1)); // exclusive suffix
    if constexpr (NW == 1) {  // a block of one warp: the warp total is inverted directly
        fe total;
#pragma unroll
        for (int i = 0; i < NL; ++i) total.w[i] = __shfl_sync(0xFFFFFFFFu, P.w[i], 31);
        return fe_mul(f, fe_mul(f, fe_inv_warp(f, total), E), S);  // all 32 lanes hold the total: cooperative inversion
    }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < NL; ++i) sm[i * NW + warp] = P.w[i];
    }
    __syncthreads();
    // the block's one inversion is run by a warp that ROTATES with the block index: warp w always
    // sits on sub-partition w % 4, and with several blocks per SM the inversions (long chains of
    // dependent instructions) would otherwise all queue on sub-partition 0
    if (warp == (int)(blockIdx.x % NW)) {
        fe w = one;
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < NL; ++i) w.w[i] = sm[i * NW + lane];
        }
        fe PP, QQ;
        warp_scan_products(f, w, lane, NW, &PP, &QQ);  // lanes >= NW hold one
        fe total;
#pragma unroll
        for (int i = 0; i < NL; ++i) total.w[i] = __shfl_sync(0xFFFFFFFFu, PP.w[i], NW - 1);
        const fe inv = fe_inv_warp(f, total);  // the block's single inversion: warp 0 runs it cooperatively
        fe EE = fe_select(lane == 0, one, fe_shfl_up(PP, 1));
        fe SS = fe_select(lane == 31, one, fe_shfl_down(QQ, 1));
        fe wi = fe_mul(f, fe_mul(f, inv, EE), SS);
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < NL; ++i) sm[(NL + i) * NW + lane] = wi.w[i];
        }
    }
    __syncthreads();
    fe wi;
#pragma unroll
    for (int i = 0; i < NL; ++i) wi.w[i] = sm[(NL + i) * NW + warp];
    return fe_mul(f, fe_mul(f, wi, E), S);
}

// product of every other thread's t in the block (returned) and the block total (*total, valid
// on thread 0 only).  sm: 2 * F::N * (THREADS / 32) words.
template <class F, int THREADS>
__device__ fel<F> block_others_product(const F& f, const fel<F>& t, uint32_t* sm, fel<F>* total) {
    using fe = fel<F>;
    constexpr int NL = F::N;
    constexpr int NW = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const fe one = fe_one(f);
    fe P, Q;
    warp_scan_products(f, t, lane, 32, &P, &Q);
    fe E = fe_select(lane == 0, one, fe_shfl_up(P, 1));
    fe S = fe_select(lane == 31, one, fe_shfl_down(Q, 1));
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < NL; ++i) sm[i * NW + warp] = P.w[i];
    }
    __syncthreads();
    if (warp == 0) {
        fe w = one;
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < NL; ++i) w.w[i] = sm[i * NW + lane];
        }
        fe PP, QQ;
        warp_scan_products(f, w, lane, NW, &PP, &QQ);
        fe EE = fe_select(lane == 0, one, fe_shfl_up(PP, 1));
        fe SS = fe_select(lane == 31, one, fe_shfl_down(QQ, 1));
        fe ab = fe_mul(f, EE, SS);  // product of the other warps' totals
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < NL; ++i) sm[(NL + i) * NW + lane] = ab.w[i];
        }
        if (lane == 0) *total = QQ;  // lane 0's inclusive suffix = all warps
    }
    __syncthreads();
    fe ab;
#pragma unroll
    for (int i = 0; i < NL; ++i) ab.w[i] = sm[(NL + i) * NW + warp];
    return fe_mul(f, fe_mul(f, ab, E), S);
}

}  // namespace gecc
