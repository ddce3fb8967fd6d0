// Batch inversion and batched affine point addition / doubling over column
// buffers: the GPU form of batch_invert (batch_invert.cpp:91-126), batch_padd
// (batch_point.cpp:68-173) and batch_pdbl (batch_point.cpp:175-231).
//
// Montgomery's trick, gather/apply/scatter: every thread owns a *strided* chunk
// (elements t, t+T, t+2T, ... so each limb load of a warp is one coalesced 128-B
// line), multiplies its denominators into a running product (compress), inverts
// the chunk product once (apply) and unwinds (scatter), finishing the chord /
// tangent formulas in the same sweep.  Prefix products live in the output buffer
// until they are consumed, so no extra scratch array exists.  Results do not
// depend on how elements are grouped (batch_invert.hpp:59-60), so they equal the
// reference's for any LanePlan.
#include "gecc_curve.cuh"
#include "gecc_dev.cuh"
#include "gecc_modinv.cuh"
#include "gecc_host.h"

namespace gecc {

constexpr int BATCH_THREADS = 128;

// zero -> zero, neighbours unaffected (batch_invert.cpp:31-47, 70-89)
template <class F>
__global__ void __launch_bounds__(BATCH_THREADS)
k_batch_invert(size_t n, size_t T, const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
    const F f{};
    const size_t t = blockIdx.x * (size_t)BATCH_THREADS + threadIdx.x;
    if (t >= T || t >= n) return;
    fe acc = fe_one(f);
    size_t last = t;
#pragma unroll 1
    for (size_t i = t; i < n; i += T) {
        fe v = col_load(in, n, i);
        if (!fe_is_zero(v)) acc = fe_mul(f, acc, v);
        col_store(out, n, i, acc);  // prefix product through element i
        last = i;
    }
    fe inv = fe_inv(f, acc);
#pragma unroll 1
    for (size_t i = last;; i -= T) {
        fe v = col_load(in, n, i);
        const bool zero = fe_is_zero(v);
        fe prev = i >= T + t ? col_load(out, n, i - T) : fe_one(f);
        fe r = fe_mul(f, inv, prev);
        if (!zero) inv = fe_mul(f, inv, v);
        col_store(out, n, i, zero ? fe_zero() : r);
        if (i < T + t) break;
    }
}

enum : uint32_t { K_GENERIC = 0, K_TANGENT, K_INFINITY, K_COPY_LEFT, K_COPY_RIGHT };

// classification + denominator of one pair (batch_point.cpp:91-111)
template <class C>
__device__ __forceinline__ uint32_t classify_pair(const fe& px, const fe& py, bool pinf,
                                                  const fe& tx, const fe& ty, bool tinf, fe* d) {
    const typename C::Fp f{};
    if (pinf && tinf) return K_INFINITY;
    if (pinf) return K_COPY_RIGHT;
    if (tinf) return K_COPY_LEFT;
    if (fe_eq(px, tx)) {
        if (fe_eq(py, ty) && !fe_is_zero(py)) {
            *d = fe_dbl(f, py);
            return K_TANGENT;
        }
        return K_INFINITY;  // inverse pair (covers y == 0)
    }
    *d = fe_sub(f, px, tx);
    return K_GENERIC;
}

template <class C>
__device__ __forceinline__ void finish_lambda(const fe& lam, const fe& x1, const fe& x2,
                                              const fe& y1, fe* xr, fe* yr) {
    const typename C::Fp f{};
    *xr = fe_sub(f, fe_sub(f, fe_sqr(f, lam), x1), x2);
    *yr = fe_sub(f, fe_mul(f, lam, fe_sub(f, x1, *xr)), y1);
}
template <class C>
__device__ __forceinline__ fe tangent_numerator(const fe& x) {  // 3x^2 + a
    const typename C::Fp f{};
    fe x2 = fe_sqr(f, x);
    fe num = fe_add(f, fe_dbl(f, x2), x2);
    if (C::a_kind == A_ZERO) return num;
    return fe_add(f, num, curve_a<C>());
}

template <class C>
__global__ void __launch_bounds__(BATCH_THREADS)
k_batch_padd(size_t n, size_t T, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
             const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx,
             const uint32_t* __restrict__ ty, const uint8_t* __restrict__ tinf,
             uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    const typename C::Fp f{};
    const size_t t = blockIdx.x * (size_t)BATCH_THREADS + threadIdx.x;
    if (t >= T || t >= n) return;
    fe acc = fe_one(f);
    size_t last = t;
    // compress: running product of the denominators, parked in ox
#pragma unroll 1
    for (size_t i = t; i < n; i += T) {
        fe ax = col_load(px, n, i), bx = col_load(tx, n, i);
        const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
        fe d = fe_one(f);
        if (!ai && !bi && fe_eq(ax, bx)) {  // y is only needed when the x's collide
            fe ay = col_load(py, n, i), by = col_load(ty, n, i);
            classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
        } else if (!ai && !bi) {
            d = fe_sub(f, ax, bx);
        }
        acc = fe_mul(f, acc, d);
        col_store(ox, n, i, acc);
        last = i;
    }
    fe inv = fe_inv(f, acc);
    // scatter + DCWPA: recover each inverse and finish the formulas (batch_point.cpp:124-170)
#pragma unroll 1
    for (size_t i = last;; i -= T) {
        fe ax = col_load(px, n, i), ay = col_load(py, n, i);
        fe bx = col_load(tx, n, i), by = col_load(ty, n, i);
        const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
        fe d = fe_one(f);
        const uint32_t kind = classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
        fe prev = i >= T + t ? col_load(ox, n, i - T) : fe_one(f);
        fe dinv = fe_mul(f, inv, prev);
        inv = fe_mul(f, inv, d);
        fe xr = fe_zero(), yr = fe_zero();
        uint8_t rinf = 0;
        if (kind == K_GENERIC) {
            fe lam = fe_mul(f, fe_sub(f, ay, by), dinv);
            finish_lambda<C>(lam, ax, bx, ay, &xr, &yr);
        } else if (kind == K_TANGENT) {
            fe lam = fe_mul(f, tangent_numerator<C>(ax), dinv);
            finish_lambda<C>(lam, ax, ax, ay, &xr, &yr);
        } else if (kind == K_COPY_LEFT) {
            xr = ax; yr = ay;
        } else if (kind == K_COPY_RIGHT) {
            xr = bx; yr = by;
        } else {
            rinf = 1;
        }
        col_store(ox, n, i, xr);
        col_store(oy, n, i, yr);
        oinf[i] = rinf;
        if (i < T + t) break;
    }
}

template <class C>
__global__ void __launch_bounds__(BATCH_THREADS)
k_batch_pdbl(size_t n, size_t T, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
             const uint8_t* __restrict__ pinf, uint32_t* __restrict__ ox,
             uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    const typename C::Fp f{};
    const size_t t = blockIdx.x * (size_t)BATCH_THREADS + threadIdx.x;
    if (t >= T || t >= n) return;
    fe acc = fe_one(f);
    size_t last = t;
#pragma unroll 1
    for (size_t i = t; i < n; i += T) {
        fe ay = col_load(py, n, i);
        const bool degenerate = (pinf && pinf[i]) || fe_is_zero(ay);
        if (!degenerate) acc = fe_mul(f, acc, fe_dbl(f, ay));
        col_store(ox, n, i, acc);
        last = i;
    }
    fe inv = fe_inv(f, acc);
#pragma unroll 1
    for (size_t i = last;; i -= T) {
        fe ax = col_load(px, n, i), ay = col_load(py, n, i);
        const bool degenerate = (pinf && pinf[i]) || fe_is_zero(ay);
        fe prev = i >= T + t ? col_load(ox, n, i - T) : fe_one(f);
        fe dinv = fe_mul(f, inv, prev);
        fe xr = fe_zero(), yr = fe_zero();
        if (!degenerate) {
            inv = fe_mul(f, inv, fe_dbl(f, ay));
            fe lam = fe_mul(f, tangent_numerator<C>(ax), dinv);
            finish_lambda<C>(lam, ax, ax, ay, &xr, &yr);
        }
        col_store(ox, n, i, xr);
        col_store(oy, n, i, yr);
        oinf[i] = degenerate ? 1 : 0;
        if (i < T + t) break;
    }
}

// threads: enough to fill the chip, at most one element short of ~CHUNK per thread
static size_t pick_threads(size_t n) {
    const size_t CHUNK = 16, cap = (size_t)148 * 16 * BATCH_THREADS;
    size_t T = (n + CHUNK - 1) / CHUNK;
    if (T > cap) T = cap;
    if (T < 1) T = 1;
    return (T + BATCH_THREADS - 1) / BATCH_THREADS * BATCH_THREADS;
}

cudaError_t launch_batch_invert(int curve, int field, size_t n, const uint32_t* in, uint32_t* out,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t T = pick_threads(n);
    const int b = (int)(T / BATCH_THREADS);
    if (curve == CURVE_SECP) {
        if (field == 0) k_batch_invert<SecpP><<<b, BATCH_THREADS, 0, s>>>(n, T, in, out);
        else k_batch_invert<SecpN><<<b, BATCH_THREADS, 0, s>>>(n, T, in, out);
    } else {
        if (field == 0) k_batch_invert<Sm2P><<<b, BATCH_THREADS, 0, s>>>(n, T, in, out);
        else k_batch_invert<Sm2N><<<b, BATCH_THREADS, 0, s>>>(n, T, in, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_batch_padd(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                              const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                              cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t T = pick_threads(n);
    const int b = (int)(T / BATCH_THREADS);
    if (curve == CURVE_SECP)
        k_batch_padd<SecpCurve><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
    else
        k_batch_padd<Sm2Curve><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
    return cudaGetLastError();
}

cudaError_t launch_batch_pdbl(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                              cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t T = pick_threads(n);
    const int b = (int)(T / BATCH_THREADS);
    if (curve == CURVE_SECP)
        k_batch_pdbl<SecpCurve><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, ox, oy, oinf);
    else
        k_batch_pdbl<Sm2Curve><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, ox, oy, oinf);
    return cudaGetLastError();
}

}  // namespace gecc
