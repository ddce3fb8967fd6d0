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
#include <cstdlib>
#include "gecc_batch.cuh"
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

template <class C, int MINB>
__global__ void __launch_bounds__(BATCH_THREADS, MINB)
k_batch_padd(size_t n, size_t T, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
             const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx,
             const uint32_t* __restrict__ ty, const uint8_t* __restrict__ tinf,
             uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    const typename C::Fp f{};
    const size_t t = blockIdx.x * (size_t)BATCH_THREADS + threadIdx.x;
    if (t >= T || t >= n) return;
    fe acc = fe_one(f);
    size_t last = t;
    // compress: running product of the denominators, parked in ox.  The next pair's x
    // coordinates are requested before the current product so the loads overlap the multiply.
    fe ax = col_load(px, n, t), bx = col_load(tx, n, t);
#pragma unroll 1
    for (size_t i = t; i < n; i += T) {
        fe nax = ax, nbx = bx;
        if (i + T < n) {
            nax = col_load(px, n, i + T);
            nbx = col_load(tx, n, i + T);
        }
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
        ax = nax;
        bx = nbx;
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

// ---------------------------------------------------------------- block-cooperative form
// Montgomery's trick with ONE inversion per thread block (section 3.3's prefix-product
// tree, mapped to the SM): a thread folds the denominators of its COOP_K elements into a local
// prefix product (registers); the per-thread totals are scanned inside each warp with shuffles
// (inclusive prefix and inclusive suffix, 5 steps each); the 8 warp totals meet in shared
// memory, warp 0 scans them the same way, inverts the block product once and hands every warp
// the inverse of its own total; thread j then gets the inverse of its total as
//     winv[warp] * (exclusive prefix)_j * (exclusive suffix)_j
// and unwinds its local prefix products.  Elements of a tile are interleaved (element
// tile + k * COOP_THREADS + tid), so every limb load of a warp is one 128-byte line.
// Compared with the chunked kernels above this exposes n / COOP_K threads instead of n / 16:
// it is the form used while the batch is too small to fill the chip with 16-element chunks.
constexpr int COOP_K = 4;  // elements per thread of the default form; small batches take fewer (coop_k)

template <class F, int COOP_THREADS, int COOP_K = 4>
__global__ void __launch_bounds__(COOP_THREADS, COOP_THREADS == 128 ? 4 : 1)
k_batch_invert_coop(size_t n, const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
    using fe = fel<F>;
    constexpr int NL = F::N;
    __shared__ uint32_t sm[2 * NL * (COOP_THREADS / 32)];
    const F f{};
    const size_t tile = (size_t)blockIdx.x * (COOP_THREADS * COOP_K) + threadIdx.x;
    fe lp[COOP_K];
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 0; k < COOP_K; ++k) {
        const size_t i = tile + (size_t)k * COOP_THREADS;
        if (i < n) {
            fe v = col_load<NL>(in, n, i);
            if (!fe_is_zero(f, v)) acc = fe_mul(f, acc, v);
        }
        lp[k] = acc;
    }
    fe inv = coop_block_inverse<decltype(f), COOP_THREADS>(f, acc, sm);
#pragma unroll
    for (int k = COOP_K - 1; k >= 0; --k) {
        const size_t i = tile + (size_t)k * COOP_THREADS;
        if (i < n) {
            fe v = col_load<NL>(in, n, i);
            const bool zero = fe_is_zero(f, v);
            fe r = k > 0 ? fe_mul(f, inv, lp[k > 0 ? k - 1 : 0]) : inv;
            if (!zero && k > 0) inv = fe_mul(f, inv, v);
            col_store(out, n, i, zero ? fe_zero_n<NL>() : r);
        }
    }
}

template <class C, int COOP_THREADS, int COOP_K = 4>
__global__ void __launch_bounds__(COOP_THREADS, COOP_THREADS == 128 ? 4 : 1)
k_batch_padd_coop(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                  const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx,
                  const uint32_t* __restrict__ ty, const uint8_t* __restrict__ tinf,
                  uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    __shared__ uint32_t sm[2 * NL * (COOP_THREADS / 32)];
    const typename C::Fp f{};
    const size_t tile = (size_t)blockIdx.x * (COOP_THREADS * COOP_K) + threadIdx.x;
    fe lp[COOP_K];
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 0; k < COOP_K; ++k) {
        const size_t i = tile + (size_t)k * COOP_THREADS;
        if (i < n) {
            fe ax = col_load<NL>(px, n, i), bx = col_load<NL>(tx, n, i);
            const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
            fe d = fe_one(f);
            if (!ai && !bi && fe_eq(ax, bx)) {
                fe ay = col_load<NL>(py, n, i), by = col_load<NL>(ty, n, i);
                classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
            } else if (!ai && !bi) {
                d = fe_sub(f, ax, bx);
            }
            acc = fe_mul(f, acc, d);
        }
        lp[k] = acc;
    }
    fe inv = coop_block_inverse<decltype(f), COOP_THREADS>(f, acc, sm);
#pragma unroll
    for (int k = COOP_K - 1; k >= 0; --k) {
        const size_t i = tile + (size_t)k * COOP_THREADS;
        if (i < n) {
            fe ax = col_load<NL>(px, n, i), ay = col_load<NL>(py, n, i);
            fe bx = col_load<NL>(tx, n, i), by = col_load<NL>(ty, n, i);
            const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
            fe d = fe_one(f);
            const uint32_t kind = classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
            fe dinv = k > 0 ? fe_mul(f, inv, lp[k > 0 ? k - 1 : 0]) : inv;
            if (k > 0) inv = fe_mul(f, inv, d);
            fe xr = fe_zero_n<NL>(), yr = fe_zero_n<NL>();
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
        }
    }
}

template <class C, int COOP_THREADS, int COOP_K = 4>
__global__ void __launch_bounds__(COOP_THREADS, COOP_THREADS == 128 ? 4 : 1)
k_batch_pdbl_coop(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                  const uint8_t* __restrict__ pinf, uint32_t* __restrict__ ox,
                  uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    __shared__ uint32_t sm[2 * NL * (COOP_THREADS / 32)];
    const typename C::Fp f{};
    const size_t tile = (size_t)blockIdx.x * (COOP_THREADS * COOP_K) + threadIdx.x;
    fe lp[COOP_K];
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 0; k < COOP_K; ++k) {
        const size_t i = tile + (size_t)k * COOP_THREADS;
        if (i < n) {
            fe ay = col_load<NL>(py, n, i);
            const bool degenerate = (pinf && pinf[i]) || fe_is_zero(ay);
            if (!degenerate) acc = fe_mul(f, acc, fe_dbl(f, ay));
        }
        lp[k] = acc;
    }
    fe inv = coop_block_inverse<decltype(f), COOP_THREADS>(f, acc, sm);
#pragma unroll
    for (int k = COOP_K - 1; k >= 0; --k) {
        const size_t i = tile + (size_t)k * COOP_THREADS;
        if (i < n) {
            fe ax = col_load<NL>(px, n, i), ay = col_load<NL>(py, n, i);
            const bool degenerate = (pinf && pinf[i]) || fe_is_zero(ay);
            fe dinv = k > 0 ? fe_mul(f, inv, lp[k > 0 ? k - 1 : 0]) : inv;
            fe xr = fe_zero_n<NL>(), yr = fe_zero_n<NL>();
            if (!degenerate) {
                if (k > 0) inv = fe_mul(f, inv, fe_dbl(f, ay));
                fe lam = fe_mul(f, tangent_numerator<C>(ax), dinv);
                finish_lambda<C>(lam, ax, ax, ay, &xr, &yr);
            }
            col_store(ox, n, i, xr);
            col_store(oy, n, i, yr);
            oinf[i] = degenerate ? 1 : 0;
        }
    }
}

// ---------------------------------------------------------------- tiled form (three launches)
// The single-launch cooperative kernels make a whole block wait for one warp's inversion
// (~36 us of dependent divsteps), which only pays while the batch is small.  The tiled form
// splits the same block-level trick at the inversion:
//   k_padd_fwd  : per tile of TILED_THREADS * K pairs -- local prefix products (parked in ox,
//                 which is free until the last launch), warp-shuffle scans, cross-warp scan in
//                 shared memory; every thread keeps the product of ALL OTHER totals of its tile
//                 (parked in oy at its first element) and the tile total goes to `totals`;
//   batch_invert: the n / tile totals are inverted by the kernels above (a batch 1000x smaller);
//   k_padd_bwd  : thread total^-1 = tile total^-1 * others, unwind, chord / tangent formulas.
// Per pair: (6K + 8)/K products (K = 8: 7) and no inversion work to speak of; the chunked form
// spends ~875 of its ~2000 instructions per pair inside safegcd at 16 pairs per thread.
constexpr int TILED_THREADS = 256;

template <class C, int K>
__global__ void __launch_bounds__(TILED_THREADS)
k_padd_fwd(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
           const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx,
           const uint32_t* __restrict__ ty, const uint8_t* __restrict__ tinf,
           uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint32_t* __restrict__ totals,
           size_t tiles) {
    __shared__ uint32_t sm[16 * (TILED_THREADS / 32)];
    const typename C::Fp f{};
    const size_t first = (size_t)blockIdx.x * (TILED_THREADS * K) + threadIdx.x;
    fe acc = fe_one(f);
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
        const size_t i = first + (size_t)k * TILED_THREADS;
        if (i < n) {
            fe ax = col_load(px, n, i), bx = col_load(tx, n, i);
            const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
            fe d = fe_one(f);
            if (!ai && !bi && fe_eq(ax, bx)) {
                fe ay = col_load(py, n, i), by = col_load(ty, n, i);
                classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
            } else if (!ai && !bi) {
                d = fe_sub(f, ax, bx);
            }
            acc = fe_mul(f, acc, d);
            col_store(ox, n, i, acc);  // local prefix product through element k
        }
    }
    fe total;
    fe others = block_others_product<decltype(f), TILED_THREADS>(f, acc, sm, &total);
    if (first < n) col_store(oy, n, first, others);
    if (threadIdx.x == 0) col_store(totals, tiles, blockIdx.x, total);
}

template <class C, int K>
__global__ void __launch_bounds__(TILED_THREADS, 2)
k_padd_bwd(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
           const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx,
           const uint32_t* __restrict__ ty, const uint8_t* __restrict__ tinf,
           uint32_t* __restrict__ ox, uint32_t* __restrict__ oy, uint8_t* __restrict__ oinf,
           const uint32_t* __restrict__ total_inv, size_t tiles) {
    const typename C::Fp f{};
    const size_t first = (size_t)blockIdx.x * (TILED_THREADS * K) + threadIdx.x;
    if (first >= n) return;
    fe inv = fe_mul(f, col_load(total_inv, tiles, blockIdx.x), col_load(oy, n, first));
    int last = K - 1;
    while (first + (size_t)last * TILED_THREADS >= n) --last;
#pragma unroll 1
    for (int k = last; k >= 0; --k) {
        const size_t i = first + (size_t)k * TILED_THREADS;
        fe ax = col_load(px, n, i), ay = col_load(py, n, i);
        fe bx = col_load(tx, n, i), by = col_load(ty, n, i);
        const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
        fe d = fe_one(f);
        const uint32_t kind = classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
        fe dinv = inv;
        if (k > 0) {
            dinv = fe_mul(f, inv, col_load(ox, n, i - TILED_THREADS));
            inv = fe_mul(f, inv, d);
        }
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
    }
}

// ---------------------------------------------------------------- fused form (three launches, recompute)
// The tiled form above parks every prefix product in the output buffer (64 B written and 64 B read
// back per pair) and re-reads both x coordinates a third time.  Here the forward launch keeps
// nothing but the tile total and each thread's "product of all other totals"; the backward launch
// RECOMPUTES the thread's K prefix products (one more product per pair instead of 128 B of HBM
// traffic), holds them in shared memory (word-interleaved by thread: conflict-free), and unwinds.
//   fwd : 1 + 14/K products per pair, reads x1, x2 (64 B per pair)
//   bwd : 1 + 1/K + 2 + 3 products per pair, reads x1, x2 (L2), y1, y2, writes x3, y3, flag
// HBM traffic ~ 257 B per pair against 385 B for the tiled form.  Elements [begin, end) of column
// buffers with row pitch n: large batches run as two halves on two streams, so that the inversion
// of one half's tile totals (one warp, pure latency) hides behind the other half's launches.
#ifndef GECC_PADD_PF
#define GECC_PADD_PF 1  // pairs of prefetch distance in the forward launch
#endif
template <int NL>
__device__ __forceinline__ void prefetch_cols(const uint32_t* __restrict__ cols, size_t n, size_t i) {
#pragma unroll
    for (int k = 0; k < NL; ++k) asm volatile("prefetch.global.L1 [%0];" ::"l"(cols + (size_t)k * n + i));
}

template <class C>
__device__ __forceinline__ cfe<C> padd_denominator(size_t n, size_t i, const uint32_t* __restrict__ px,
                                                   const uint32_t* __restrict__ py, const uint8_t* __restrict__ pinf,
                                                   const uint32_t* __restrict__ tx, const uint32_t* __restrict__ ty,
                                                   const uint8_t* __restrict__ tinf) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    const typename C::Fp f{};
    fe ax = col_load<NL>(px, n, i), bx = col_load<NL>(tx, n, i);
    const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
    fe d = fe_one(f);
    if (!ai && !bi && fe_eq(ax, bx)) {  // y is only needed when the x's collide
        fe ay = col_load<NL>(py, n, i), by = col_load<NL>(ty, n, i);
        classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
    } else if (!ai && !bi) {
        d = fe_sub(f, ax, bx);
    }
    return d;
}

template <class C, int K, int THREADS>
__global__ void __launch_bounds__(THREADS)
k_padd_fused_fwd(size_t n, size_t begin, size_t end, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                 const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx, const uint32_t* __restrict__ ty,
                 const uint8_t* __restrict__ tinf, uint32_t* __restrict__ totals, uint32_t* __restrict__ others,
                 size_t tiles) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    __shared__ uint32_t sm[2 * NL * (THREADS / 32)];
    const typename C::Fp f{};
    const size_t first = begin + (size_t)blockIdx.x * (THREADS * K) + threadIdx.x;
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 1; k < GECC_PADD_PF; ++k) {
        if (k < K && first + (size_t)k * THREADS < end) {
            prefetch_cols<NL>(px, n, first + (size_t)k * THREADS);
            prefetch_cols<NL>(tx, n, first + (size_t)k * THREADS);
        }
    }
    if (first < end) acc = padd_denominator<C>(n, first, px, py, pinf, tx, ty, tinf);
#pragma unroll 1
    for (int k = 1; k < K; ++k) {
        const size_t i = first + (size_t)k * THREADS;
        if (k + GECC_PADD_PF < K && i + (size_t)GECC_PADD_PF * THREADS < end) {  // lines of the pair GECC_PADD_PF ahead are requested before this pair's product
            prefetch_cols<NL>(px, n, i + (size_t)GECC_PADD_PF * THREADS);
            prefetch_cols<NL>(tx, n, i + (size_t)GECC_PADD_PF * THREADS);
        }
        if (i < end) acc = fe_mul(f, acc, padd_denominator<C>(n, i, px, py, pinf, tx, ty, tinf));
    }
    fe total;
    fe oth = block_others_product<decltype(f), THREADS>(f, acc, sm, &total);
    col_store(others, tiles * THREADS, (size_t)blockIdx.x * THREADS + threadIdx.x, oth);
    if (threadIdx.x == 0) col_store(totals, tiles, blockIdx.x, total);
}

template <class C, int K, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
k_padd_fused_bwd(size_t n, size_t begin, size_t end, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                 const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx, const uint32_t* __restrict__ ty,
                 const uint8_t* __restrict__ tinf, uint32_t* __restrict__ ox, uint32_t* __restrict__ oy,
                 uint8_t* __restrict__ oinf, const uint32_t* __restrict__ total_inv,
                 const uint32_t* __restrict__ others, size_t tiles) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    extern __shared__ uint32_t pre[];  // prefix products 0 .. K-2: word (k * NL + w) of thread t at [(k * NL + w) * THREADS + t]
    const typename C::Fp f{};
    const size_t first = begin + (size_t)blockIdx.x * (THREADS * K) + threadIdx.x;
    if (first >= end) return;
    fe inv = fe_mul(f, col_load<NL>(total_inv, tiles, blockIdx.x),
                    col_load<NL>(others, tiles * THREADS, (size_t)blockIdx.x * THREADS + threadIdx.x));
    int last = K - 1;
    while (first + (size_t)last * THREADS >= end) --last;
    {   // recompute the prefix products of this thread's denominators
        fe acc = padd_denominator<C>(n, first, px, py, pinf, tx, ty, tinf);
#pragma unroll 1
        for (int k = 0; k < last; ++k) {
            if (k + 2 <= last) {
                prefetch_cols<NL>(px, n, first + (size_t)(k + 2) * THREADS);
                prefetch_cols<NL>(tx, n, first + (size_t)(k + 2) * THREADS);
            } else {  // the unwind starts at the last pair: its y coordinates come from HBM
                prefetch_cols<NL>(py, n, first + (size_t)last * THREADS);
                prefetch_cols<NL>(ty, n, first + (size_t)last * THREADS);
            }
#pragma unroll
            for (int w = 0; w < NL; ++w) pre[(size_t)(k * NL + w) * THREADS + threadIdx.x] = acc.w[w];
            acc = fe_mul(f, acc, padd_denominator<C>(n, first + (size_t)(k + 1) * THREADS, px, py, pinf, tx, ty, tinf));
        }
    }
#pragma unroll 1
    for (int k = last; k >= 0; --k) {
        const size_t i = first + (size_t)k * THREADS;
        if (k > 0) {
            prefetch_cols<NL>(py, n, i - THREADS);
            prefetch_cols<NL>(ty, n, i - THREADS);
        }
        fe ax = col_load<NL>(px, n, i), ay = col_load<NL>(py, n, i);
        fe bx = col_load<NL>(tx, n, i), by = col_load<NL>(ty, n, i);
        const bool ai = pinf && pinf[i], bi = tinf && tinf[i];
        fe d = fe_one(f);
        const uint32_t kind = classify_pair<C>(ax, ay, ai, bx, by, bi, &d);
        fe dinv = inv;
        if (k > 0) {
            fe prev;
#pragma unroll
            for (int w = 0; w < NL; ++w) prev.w[w] = pre[(size_t)((k - 1) * NL + w) * THREADS + threadIdx.x];
            dinv = fe_mul(f, inv, prev);
            inv = fe_mul(f, inv, d);
        }
        fe xr = fe_zero_n<NL>(), yr = fe_zero_n<NL>();
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
    }
}

// Form selection: the cooperative kernels while 16-element chunks would leave the chip
// under-filled, the chunked kernels beyond.  gecc_set_batch_form pins one form (tests, sweeps):
// 0 auto, 1 chunked (16 per thread), 2 cooperative 256 threads, 3 chunked at 6 blocks per SM,
// 4 cooperative 128 threads, 5 cooperative 32 threads (one inversion per warp),
// 6 / 7 tiled with 8 / 4 pairs per thread (batch_padd only; needs the context's scratch).
static size_t g_coop_max_n = (size_t)1 << 18;
static int g_batch_form = 0;
void set_batch_form(int form) { g_batch_form = form; }
static int pick_form(size_t n, bool tiled_ok = false) {
    if (g_batch_form >= 6) return tiled_ok ? g_batch_form : (n <= g_coop_max_n ? 4 : 1);
    if (g_batch_form) return g_batch_form;
    // measured on B200 (profiles/r01f_sweep.json): cooperative/128 wins up to 2^18 pairs
    // (0.054 ms vs 0.083 ms); beyond, the fused three-launch form (batch_padd with scratch only)
    if (n <= g_coop_max_n) return 4;
    return tiled_ok ? 8 : 1;
}
// fused form: K pairs per thread, FUSED_THREADS threads per tile
#ifndef GECC_FUSED_THREADS
#define GECC_FUSED_THREADS 128
#endif
#ifndef GECC_FUSED_MINB
#define GECC_FUSED_MINB 4
#endif
constexpr int FUSED_THREADS = GECC_FUSED_THREADS;
constexpr int FUSED_MINB = GECC_FUSED_MINB;
static size_t fused_tiles(size_t n, int K) { return (n + (size_t)FUSED_THREADS * K - 1) / ((size_t)FUSED_THREADS * K); }
// tile totals, their inverses (tiled / fused forms) and the per-thread "others" products (fused)
size_t batch_padd_scratch_bytes(size_t n) {
    const size_t tiles = (n + (size_t)TILED_THREADS * 4 - 1) / ((size_t)TILED_THREADS * 4);
    // fused form: two sets (the two halves) of totals | inverses | others; K = 8 has the most tiles
    const size_t half_tiles = fused_tiles(n, 8) / 2 + 2;
    const size_t tot_words = (half_tiles * 8 + 63) & ~(size_t)63;
    const size_t fused = 2 * (2 * tot_words + half_tiles * FUSED_THREADS * 8) * 4;
    const size_t tiled = 2 * tiles * 32 + 512;
    return (fused > tiled ? fused : tiled) + 1024;
}
static int coop_threads(int form) { return form == 2 ? 256 : form == 4 ? 128 : form == 5 ? 32 : 0; }
static unsigned coop_blocks(size_t n, int threads, int k = COOP_K) {
    return (unsigned)((n + (size_t)threads * k - 1) / ((size_t)threads * k));
}
// elements per thread: small batches spread over more blocks (the chain of dependent products and
// memory round trips per thread is what their time consists of)
static int coop_k(size_t n) { return n <= ((size_t)1 << 15) ? 1 : n <= ((size_t)1 << 17) ? 2 : 4; }
// threads: enough to fill the chip, at most one element short of ~CHUNK per thread
static size_t pick_threads(size_t n, int form) {
    const size_t CHUNK = 16, cap = (size_t)148 * (form == 3 ? 24 : 16) * BATCH_THREADS;
    size_t T = (n + CHUNK - 1) / CHUNK;
    if (T > cap) T = cap;
    if (T < 1) T = 1;
    return (T + BATCH_THREADS - 1) / BATCH_THREADS * BATCH_THREADS;
}
#define COOP_DISPATCH(threads, KERNEL, ...)                                                       \
    do {                                                                                          \
        const int ck__ = threads == 128 ? coop_k(n) : COOP_K;                                     \
        const unsigned cb__ = coop_blocks(n, threads, ck__);                                      \
        if (threads == 256) KERNEL(256, 4)<<<cb__, 256, 0, s>>>(__VA_ARGS__);                     \
        else if (threads == 128 && ck__ == 1) KERNEL(128, 1)<<<cb__, 128, 0, s>>>(__VA_ARGS__);   \
        else if (threads == 128 && ck__ == 2) KERNEL(128, 2)<<<cb__, 128, 0, s>>>(__VA_ARGS__);   \
        else if (threads == 128) KERNEL(128, 4)<<<cb__, 128, 0, s>>>(__VA_ARGS__);                \
        else KERNEL(32, 4)<<<cb__, 32, 0, s>>>(__VA_ARGS__);                                      \
    } while (0)

cudaError_t launch_batch_invert(int curve, int field, size_t n, const uint32_t* in, uint32_t* out,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (curve_is_bls(curve)) {  // 12-limb base fields / their 8-limb scalar fields: cooperative form
        if (field == 0 && n <= ((size_t)1 << 15)) {  // small batches (the MSM's level totals): one element per thread
            const unsigned c1 = coop_blocks(n, 128, 1);
            if (curve == CURVE_BLS381) k_batch_invert_coop<Bls381P, 128, 1><<<c1, 128, 0, s>>>(n, in, out);
            else k_batch_invert_coop<Bls377P, 128, 1><<<c1, 128, 0, s>>>(n, in, out);
            return cudaGetLastError();
        }
        const unsigned cb = coop_blocks(n, 128);
        if (curve == CURVE_BLS381) {
            if (field == 0) k_batch_invert_coop<Bls381P, 128><<<cb, 128, 0, s>>>(n, in, out);
            else k_batch_invert_coop<Bls381R, 128><<<cb, 128, 0, s>>>(n, in, out);
        } else {
            if (field == 0) k_batch_invert_coop<Bls377P, 128><<<cb, 128, 0, s>>>(n, in, out);
            else k_batch_invert_coop<Bls377R, 128><<<cb, 128, 0, s>>>(n, in, out);
        }
        return cudaGetLastError();
    }
    const int form = pick_form(n);
    if (const int ct = coop_threads(form)) {
        if (curve == CURVE_SECP && field == 0) {
#define KT_(t, k) k_batch_invert_coop<SecpP, t, k>
            COOP_DISPATCH(ct, KT_, n, in, out);
#undef KT_
        } else if (curve == CURVE_SECP) {
#define KT_(t, k) k_batch_invert_coop<SecpN, t, k>
            COOP_DISPATCH(ct, KT_, n, in, out);
#undef KT_
        } else if (field == 0) {
#define KT_(t, k) k_batch_invert_coop<Sm2P, t, k>
            COOP_DISPATCH(ct, KT_, n, in, out);
#undef KT_
        } else {
#define KT_(t, k) k_batch_invert_coop<Sm2N, t, k>
            COOP_DISPATCH(ct, KT_, n, in, out);
#undef KT_
        }
        return cudaGetLastError();
    }
    const size_t T = pick_threads(n, form);
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

// block totals of the MSM tree when it runs on the lazy plain secp256k1 field (plain in, plain out)
cudaError_t launch_batch_invert_secp_lazy(size_t n, const uint32_t* in, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    // the totals of a tree level / a fused batch_padd half: a few thousand elements whose inversion is pure
    // latency -- one element per thread (the shortest chain) while that still fits one wave
    if (n <= ((size_t)1 << 15)) k_batch_invert_coop<SecpPL, 128, 1><<<coop_blocks(n, 128, 1), 128, 0, s>>>(n, in, out);
    else k_batch_invert_coop<SecpPL, 128><<<coop_blocks(n, 128), 128, 0, s>>>(n, in, out);
    return cudaGetLastError();
}

// one range [begin, end) of the fused form on stream s
template <class C, int K>
static cudaError_t fused_range(int curve, size_t n, size_t begin, size_t end, const uint32_t* px, const uint32_t* py,
                               const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty, const uint8_t* tinf,
                               uint32_t* ox, uint32_t* oy, uint8_t* oinf, uint32_t* totals, uint32_t* total_inv,
                               uint32_t* others, cudaStream_t s) {
    const size_t m = end - begin;
    const size_t tiles = fused_tiles(m, K);
    const size_t smem = (size_t)(K - 1) * 8 * FUSED_THREADS * sizeof(uint32_t);
    if (smem > 48 * 1024)  // per device: set on every launch (a context may be one of several devices')
        cudaFuncSetAttribute(k_padd_fused_bwd<C, K, FUSED_THREADS, FUSED_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_padd_fused_fwd<C, K, FUSED_THREADS><<<(unsigned)tiles, FUSED_THREADS, 0, s>>>(n, begin, end, px, py, pinf, tx, ty, tinf,
                                                                                  totals, others, tiles);
    // tile totals: plain residues on the lazy secp256k1 field, Montgomery form otherwise
    if (cudaError_t e = curve_mont_reps<C>::value ? launch_batch_invert_secp_lazy(tiles, totals, total_inv, s)
                                                  : launch_batch_invert(curve, 0, tiles, totals, total_inv, s))
        return e;
    k_padd_fused_bwd<C, K, FUSED_THREADS, FUSED_MINB><<<(unsigned)tiles, FUSED_THREADS, smem, s>>>(
        n, begin, end, px, py, pinf, tx, ty, tinf, ox, oy, oinf, total_inv, others, tiles);
    return cudaGetLastError();
}

template <class C, int K>
static cudaError_t fused_padd(int curve, size_t n, const uint32_t* px, const uint32_t* py, const uint8_t* pinf,
                              const uint32_t* tx, const uint32_t* ty, const uint8_t* tinf, uint32_t* ox, uint32_t* oy,
                              uint8_t* oinf, void* scratch, cudaStream_t s, const BatchAux& aux) {
    // scratch: two sets (one per part) of totals | total_inv | others, carved by each part's tile count
    const size_t tile_pairs = (size_t)FUSED_THREADS * K;
    uint32_t* base = (uint32_t*)scratch;
    const bool split = aux.stream && aux.fork && aux.join && n >= ((size_t)1 << 18);
    if (!split) {  // one range: the whole scratch is one set, sized by the full tile count
        const size_t all_words = (fused_tiles(n, K) * 8 + 63) & ~(size_t)63;
        return fused_range<C, K>(curve, n, 0, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, base, base + all_words,
                                 base + 2 * all_words, s);
    }
    // two parts on two streams: each part is fwd -> invert -> bwd; the inversion of one part (a
    // single warp's latency) overlaps the other part's launches
    // (GECC_PADD_SPLIT: percent of the tiles in the first part, an experiment knob; 25 ... 75 measured within
    // 171 ... 182 us at 2^20 with the optimum at the default; delaying the second part's forward launch until the
    // first part's has finished -- so that inversion and forward launch overlap by construction -- measured 184 us)
    static const int split_pct = getenv("GECC_PADD_SPLIT") ? atoi(getenv("GECC_PADD_SPLIT")) : 50;
    const size_t tiles = fused_tiles(n, K);
    size_t tiles0 = tiles * (size_t)split_pct / 100;
    if (tiles0 < 1) tiles0 = 1;
    if (tiles0 >= tiles) tiles0 = tiles - 1;
    const size_t mid = tiles0 * tile_pairs;
    const size_t tot0 = (tiles0 * 8 + 63) & ~(size_t)63, tot1 = ((tiles - tiles0) * 8 + 63) & ~(size_t)63;
    uint32_t* set0 = base;
    uint32_t* set1 = base + 2 * tot0 + tiles0 * FUSED_THREADS * 8;
    cudaError_t e = cudaEventRecord(aux.fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(aux.stream, aux.fork, 0);
    if (e == cudaSuccess)
        e = fused_range<C, K>(curve, n, 0, mid, px, py, pinf, tx, ty, tinf, ox, oy, oinf, set0, set0 + tot0, set0 + 2 * tot0, s);
    if (e == cudaSuccess)
        e = fused_range<C, K>(curve, n, mid, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, set1, set1 + tot1, set1 + 2 * tot1,
                              aux.stream);
    if (e == cudaSuccess) e = cudaEventRecord(aux.join, aux.stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, aux.join, 0);
    return e;
}

cudaError_t launch_batch_padd(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                              const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                              cudaStream_t s, void* scratch, BatchAux aux) {
    if (n == 0) return cudaSuccess;
    if (curve == CURVE_BLS381) {
        k_batch_padd_coop<Bls381Curve, 128><<<coop_blocks(n, 128), 128, 0, s>>>(n, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
        return cudaGetLastError();
    }
    if (curve == CURVE_BLS377) {
        k_batch_padd_coop<Bls377Curve, 128><<<coop_blocks(n, 128), 128, 0, s>>>(n, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
        return cudaGetLastError();
    }
    const int form = pick_form(n, scratch != nullptr);
    if (form >= 8) {  // fused: 8 = eight pairs per thread, 9 = sixteen
        if (curve == CURVE_SECP) {
            if (form == 8) return fused_padd<SecpMLCurve, 8>(curve, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, scratch, s, aux);
            return fused_padd<SecpMLCurve, 16>(curve, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, scratch, s, aux);
        }
        if (form == 8) return fused_padd<Sm2Curve, 8>(curve, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, scratch, s, aux);
        return fused_padd<Sm2Curve, 16>(curve, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, scratch, s, aux);
    }
    if (form >= 6) {
        const int K = form == 6 ? 8 : 4;
        const size_t tiles = (n + (size_t)TILED_THREADS * K - 1) / ((size_t)TILED_THREADS * K);
        uint32_t* totals = (uint32_t*)scratch;
        uint32_t* total_inv = totals + ((tiles * 8 + 63) & ~(size_t)63);
        const unsigned b = (unsigned)tiles;
#define TILED_(CURVE, KK)                                                                              \
    k_padd_fwd<CURVE, KK><<<b, TILED_THREADS, 0, s>>>(n, px, py, pinf, tx, ty, tinf, ox, oy, totals, tiles); \
    if (cudaError_t e = launch_batch_invert(curve, 0, tiles, totals, total_inv, s)) return e;           \
    k_padd_bwd<CURVE, KK><<<b, TILED_THREADS, 0, s>>>(n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, total_inv, tiles)
        if (curve == CURVE_SECP) {
            if (K == 8) { TILED_(SecpCurve, 8); } else { TILED_(SecpCurve, 4); }
        } else {
            if (K == 8) { TILED_(Sm2Curve, 8); } else { TILED_(Sm2Curve, 4); }
        }
#undef TILED_
        return cudaGetLastError();
    }
    if (const int ct = coop_threads(form)) {
        if (curve == CURVE_SECP) {
#define KT_(t, k) k_batch_padd_coop<SecpMLCurve, t, k>
            COOP_DISPATCH(ct, KT_, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
#undef KT_
        } else {
#define KT_(t, k) k_batch_padd_coop<Sm2Curve, t, k>
            COOP_DISPATCH(ct, KT_, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
#undef KT_
        }
        return cudaGetLastError();
    }
    const size_t T = pick_threads(n, form);
    const int b = (int)(T / BATCH_THREADS);
    if (form == 3) {  // experimental: 6 blocks per SM (80 registers)
        if (curve == CURVE_SECP)
            k_batch_padd<SecpCurve, 6><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
        else
            k_batch_padd<Sm2Curve, 6><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
    } else if (curve == CURVE_SECP)
        k_batch_padd<SecpCurve, 4><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
    else
        k_batch_padd<Sm2Curve, 4><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
    return cudaGetLastError();
}

cudaError_t launch_batch_pdbl(int curve, size_t n, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                              cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (curve == CURVE_BLS381) {
        k_batch_pdbl_coop<Bls381Curve, 128><<<coop_blocks(n, 128), 128, 0, s>>>(n, px, py, pinf, ox, oy, oinf);
        return cudaGetLastError();
    }
    if (curve == CURVE_BLS377) {
        k_batch_pdbl_coop<Bls377Curve, 128><<<coop_blocks(n, 128), 128, 0, s>>>(n, px, py, pinf, ox, oy, oinf);
        return cudaGetLastError();
    }
    const int form = pick_form(n);
    if (const int ct = coop_threads(form)) {
        if (curve == CURVE_SECP) {
#define KT_(t, k) k_batch_pdbl_coop<SecpMLCurve, t, k>
            COOP_DISPATCH(ct, KT_, n, px, py, pinf, ox, oy, oinf);
#undef KT_
        } else {
#define KT_(t, k) k_batch_pdbl_coop<Sm2Curve, t, k>
            COOP_DISPATCH(ct, KT_, n, px, py, pinf, ox, oy, oinf);
#undef KT_
        }
        return cudaGetLastError();
    }
    const size_t T = pick_threads(n, form);
    const int b = (int)(T / BATCH_THREADS);
    if (curve == CURVE_SECP)
        k_batch_pdbl<SecpCurve><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, ox, oy, oinf);
    else
        k_batch_pdbl<Sm2Curve><<<b, BATCH_THREADS, 0, s>>>(n, T, px, py, pinf, ox, oy, oinf);
    return cudaGetLastError();
}

}  // namespace gecc
