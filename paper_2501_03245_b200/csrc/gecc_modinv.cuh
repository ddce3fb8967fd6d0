// Modular inversion by Bernstein-Yang division steps ("safegcd", Bernstein & Yang,
// "Fast constant-time gcd computation and modular inversion", TCHES 2019), in the
// signed 30-bit-limb organisation that is common for 32-bit targets: 20 rounds of 30
// branch-free divsteps on the low limbs, each followed by one 2x2 matrix update of
// (f, g) and, modulo q, of (d, e).  Every lane of a warp executes the identical
// instruction sequence (no data-dependent branches), which is what a SIMT machine
// needs; a Fermat exponentiation costs 256 squarings + ~80 products instead.
//
// The reference inverts by Fermat (mod_inv_fermat, field.cpp:239-246) and checks it
// against an extended-Euclid oracle (tests/test_field.cpp:203-225): the residue is
// unique, so the result bits are identical whichever way it is computed.
//
//   safegcd_inverse(f, x)  : x^-1 mod q for a plain residue 0 < x < q (0 -> 0)
//   fe_inv(f, a)           : Montgomery-form inverse of a Montgomery-form element:
//                            (aR)^-1 * R^3 * R^-1 = a^-1 R
#pragma once
#include "gecc_field.cuh"

namespace gecc {

template <int L>
struct s30n {
    int32_t v[L];  // value = sum v[i] 2^(30 i); limbs in (-2^30, 2^30) except the top one
};
using s30 = s30n<9>;  // 256-bit fields; the 381-bit field uses 13 limbs
struct trans2x2 {
    int32_t u, v, q, r;
};

// N 32-bit limbs -> L 30-bit limbs (the shifts are compile-time constants after unrolling)
template <int N, int L>
GECC_HD s30n<L> s30_from_limbs(const uint32_t* w) {
    s30n<L> r;
    const uint32_t M30 = 0x3FFFFFFFu;
#pragma unroll
    for (int i = 0; i < L; ++i) {
        const int bit = 30 * i, wi = bit >> 5, sh = bit & 31;
        uint32_t v = w[wi] >> sh;
        if (sh > 2 && wi + 1 < N) v |= w[wi + 1] << (32 - sh);
        r.v[i] = (int32_t)(v & M30);
    }
    return r;
}
template <int N, int L>
GECC_HD void s30_to_limbs(uint32_t* w, const s30n<L>& a) {  // a normalised: limbs in [0, 2^30)
    const uint32_t* v = reinterpret_cast<const uint32_t*>(a.v);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const int bit = 32 * k, li = bit / 30, off = bit % 30;
        uint32_t x = v[li] >> off;
        if (li + 1 < L) x |= v[li + 1] << (30 - off);
        if (60 - off < 32 && li + 2 < L) x |= v[li + 2] << (60 - off);
        w[k] = x;
    }
}

// 30 division steps on the low limbs; zeta = -(delta + 1/2).  Returns the new zeta
// and the transition matrix t with t * [f, g] = 2^30 * [f', g'].
GECC_HD int32_t divsteps_30(int32_t zeta, uint32_t f0, uint32_t g0, trans2x2* t) {
    uint32_t u = 1, v = 0, q = 0, r = 1;
    uint32_t f = f0, g = g0;
#pragma unroll 6
    for (int i = 0; i < 30; ++i) {
        const uint32_t c1 = (uint32_t)(zeta >> 31);  // all ones when zeta < 0
        const uint32_t c2 = 0u - (g & 1u);           // all ones when g is odd
        const uint32_t c12 = c1 & c2;                // swap happens when zeta < 0 and g odd
        // g += (+-f) & c2 with -f = (f ^ c1) - c1:  ((f ^ c1) - c1) & c2 == ((f ^ c1) & c2) - c12, so each
        // update is one three-input logic operation and one three-input add (21 instead of 27 per step)
        g = g + ((f ^ c1) & c2) - c12;
        q = q + ((u ^ c1) & c2) - c12;
        r = r + ((v ^ c1) & c2) - c12;
        zeta = (int32_t)(((uint32_t)zeta ^ c12) - 1u);
        f += g & c12;
        u += q & c12;
        v += r & c12;
        g >>= 1;
        u <<= 1;
        v <<= 1;
    }
    t->u = (int32_t)u;
    t->v = (int32_t)v;
    t->q = (int32_t)q;
    t->r = (int32_t)r;
    return zeta;
}

// c + a * b, signed 32 x 32 -> 64: ONE instruction on the device (IMAD.WIDE); the C expression
// (int64)a * b + c compiles to an unsigned wide multiply plus two sign corrections.
GECC_HD int64_t mac_s32(int32_t a, int32_t b, int64_t c) {
#if defined(__CUDA_ARCH__)
    int64_t r;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
    return r;
#else
    return (int64_t)a * b + c;
#endif
}

// (f, g) <- t * (f, g) / 2^30 (exact)
template <int L>
GECC_HD void update_fg_30(s30n<L>* f, s30n<L>* g, const trans2x2& t) {
    const int32_t M30 = 0x3FFFFFFF;
    const int32_t u = t.u, v = t.v, q = t.q, r = t.r;
    int64_t cf = mac_s32(u, f->v[0], mac_s32(v, g->v[0], 0));
    int64_t cg = mac_s32(q, f->v[0], mac_s32(r, g->v[0], 0));
    cf >>= 30;
    cg >>= 30;
#pragma unroll
    for (int i = 1; i < L; ++i) {
        const int32_t fi = f->v[i], gi = g->v[i];
        cf = mac_s32(u, fi, mac_s32(v, gi, cf));
        cg = mac_s32(q, fi, mac_s32(r, gi, cg));
        f->v[i - 1] = (int32_t)cf & M30;
        cf >>= 30;
        g->v[i - 1] = (int32_t)cg & M30;
        cg >>= 30;
    }
    f->v[L - 1] = (int32_t)cf;
    g->v[L - 1] = (int32_t)cg;
}

// (d, e) <- t * (d, e) / 2^30 mod q: a multiple of q is added first so that the
// low 30 bits vanish and the division is exact.  d, e stay in (-2q, q).
template <class F, int L>
GECC_HD void update_de_30(const F& f, s30n<L>* d, s30n<L>* e, const trans2x2& t) {
    const int32_t M30 = 0x3FFFFFFF;
    const int32_t u = t.u, v = t.v, q = t.q, r = t.r;
    const int32_t sd = d->v[L - 1] >> 31, se = e->v[L - 1] >> 31;
    int32_t md = (t.u & sd) + (t.v & se);
    int32_t me = (t.q & sd) + (t.r & se);
    int64_t cd = mac_s32(u, d->v[0], mac_s32(v, e->v[0], 0));
    int64_t ce = mac_s32(q, d->v[0], mac_s32(r, e->v[0], 0));
    md -= (int32_t)((f.qinv30() * (uint32_t)cd + (uint32_t)md) & (uint32_t)M30);
    me -= (int32_t)((f.qinv30() * (uint32_t)ce + (uint32_t)me) & (uint32_t)M30);
    cd = mac_s32((int32_t)f.q30(0), md, cd);
    ce = mac_s32((int32_t)f.q30(0), me, ce);
    cd >>= 30;
    ce >>= 30;
#pragma unroll
    for (int i = 1; i < L; ++i) {
        const int32_t di = d->v[i], ei = e->v[i];
        cd = mac_s32(u, di, mac_s32(v, ei, mac_s32((int32_t)f.q30(i), md, cd)));
        ce = mac_s32(q, di, mac_s32(r, ei, mac_s32((int32_t)f.q30(i), me, ce)));
        d->v[i - 1] = (int32_t)cd & M30;
        cd >>= 30;
        e->v[i - 1] = (int32_t)ce & M30;
        ce >>= 30;
    }
    d->v[L - 1] = (int32_t)cd;
    e->v[L - 1] = (int32_t)ce;
}

// r in (-2q, q) -> [0, q), negated first when sign < 0
template <class F, int L>
GECC_HD void normalize_30(const F& f, s30n<L>* r, int32_t sign) {
    const int32_t M30 = 0x3FFFFFFF;
    int32_t cond_add = r->v[L - 1] >> 31;
#pragma unroll
    for (int i = 0; i < L; ++i) r->v[i] += (int32_t)f.q30(i) & cond_add;
    const int32_t cond_negate = sign >> 31;
#pragma unroll
    for (int i = 0; i < L; ++i) r->v[i] = (r->v[i] ^ cond_negate) - cond_negate;
#pragma unroll
    for (int i = 0; i < L - 1; ++i) {
        r->v[i + 1] += r->v[i] >> 30;
        r->v[i] &= M30;
    }
    cond_add = r->v[L - 1] >> 31;
#pragma unroll
    for (int i = 0; i < L; ++i) r->v[i] += (int32_t)f.q30(i) & cond_add;
#pragma unroll
    for (int i = 0; i < L - 1; ++i) {
        r->v[i + 1] += r->v[i] >> 30;
        r->v[i] &= M30;
    }
}

// x^-1 mod q, x a plain residue in [0, q); 0 -> 0.  Limb and round counts per field size
// (half-delta divsteps: 590 suffice for 256-bit moduli, 879 for 381-bit ones; extra rounds
// leave the result unchanged once g has reached zero).
template <class F>
GECC_HD_CALL fel<F> safegcd_inverse(const F& fld, const fel<F>& x) {
    GECC_COUNT(safegcd, F);
    constexpr int N = F::N, L = N == 8 ? 9 : (32 * N + 29) / 30, ROUNDS = N == 8 ? 20 : (49 * N + 16) / 17 + 1;
    s30n<L> d, e, f, g;
#pragma unroll
    for (int i = 0; i < L; ++i) {
        d.v[i] = 0;
        e.v[i] = 0;
        f.v[i] = (int32_t)fld.q30(i);
    }
    e.v[0] = 1;
    g = s30_from_limbs<N, L>(x.w);
    int32_t zeta = -1;
#pragma unroll 1
    for (int round = 0; round < ROUNDS; ++round) {
        trans2x2 t;
        zeta = divsteps_30(zeta, (uint32_t)f.v[0], (uint32_t)g.v[0], &t);
        update_de_30(fld, &d, &e, t);
        update_fg_30(&f, &g, t);
    }
    // g == 0 now and f == +-gcd == +-1 (or f == +-q when x == 0, where d == 0)
    normalize_30(fld, &d, f.v[L - 1]);
    fel<F> r;
    s30_to_limbs<N, L>(r.w, d);
    return r;
}

// ---------------------------------------------------------------- variable-time form
// The same recurrence run for LATENCY instead of uniformity, for the places where one warp inverts
// one PUBLIC value that all of its lanes share (the block total of Montgomery's trick: every lane
// holds the same number, so data-dependent control flow does not diverge): whole runs of zero bits
// of g are shifted out at once (count-trailing-zeros), up to six low bits of g are cancelled per
// iteration with w = -g / f mod 2^k (f (f^2 - 2) == -1/f mod 64 for odd f), and the rounds stop as
// soon as g is zero.  Classic divsteps (delta starts at 1; eta = -delta).  Never used on secrets.
GECC_HD int ctz32_nz(uint32_t x) {  // x != 0
#if defined(__CUDA_ARCH__)
    return __ffs((int)x) - 1;
#else
    return __builtin_ctz(x);
#endif
}
GECC_HD int32_t divsteps_30_var(int32_t eta, uint32_t f0, uint32_t g0, trans2x2* t) {
    uint32_t u = 1, v = 0, q = 0, r = 1;
    uint32_t f = f0, g = g0;
    uint32_t nf = f * (f * f - 2u);  // -1/f mod 64
    int i = 30;
    for (;;) {
        const int zeros = ctz32_nz(g | (0xFFFFFFFFu << i));  // sentinel: at most i
        g >>= zeros;
        u <<= zeros;
        v <<= zeros;
        eta -= zeros;
        i -= zeros;
        if (i == 0) break;
        if (eta < 0) {  // g is odd here: (f, g) <- (g, -f)
            eta = -eta;
            uint32_t tmp = f; f = g; g = 0u - tmp;
            tmp = u; u = q; q = 0u - tmp;
            tmp = v; v = r; r = 0u - tmp;
            nf = f * (f * f - 2u);
        }
        // cancel the low min(eta + 1, i, 6) bits of g: no more than i are left in this round and the
        // sign of eta flips after eta + 1
        const int limit = (eta + 1) > i ? i : (eta + 1);
        const uint32_t m = (0xFFFFFFFFu >> (32 - limit)) & 63u;
        const uint32_t w = (g * nf) & m;
        g += f * w;
        q += u * w;
        r += v * w;
    }
    t->u = (int32_t)u;
    t->v = (int32_t)v;
    t->q = (int32_t)q;
    t->r = (int32_t)r;
    return eta;
}
template <class F>
GECC_HD_CALL fel<F> safegcd_inverse_var(const F& fld, const fel<F>& x) {
    GECC_COUNT(safegcd, F);
    constexpr int N = F::N, L = N == 8 ? 9 : (32 * N + 29) / 30;
    constexpr int MAX_ROUNDS = N == 8 ? 25 : 37;  // 724 / 1086 classic divsteps bound the worst case
    s30n<L> d, e, f, g;
#pragma unroll
    for (int i = 0; i < L; ++i) {
        d.v[i] = 0;
        e.v[i] = 0;
        f.v[i] = (int32_t)fld.q30(i);
    }
    e.v[0] = 1;
    g = s30_from_limbs<N, L>(x.w);
    int32_t eta = -1;
#pragma unroll 1
    for (int round = 0; round < MAX_ROUNDS; ++round) {
        int32_t nz = 0;
#pragma unroll
        for (int i = 0; i < L; ++i) nz |= g.v[i];
        if (nz == 0) break;
        trans2x2 t;
        eta = divsteps_30_var(eta, (uint32_t)f.v[0], (uint32_t)g.v[0], &t);
        update_de_30(fld, &d, &e, t);
        update_fg_30(&f, &g, t);
    }
    normalize_30(fld, &d, f.v[L - 1]);
    fel<F> r;
    s30_to_limbs<N, L>(r.w, d);
    return r;
}
// ---------------------------------------------------------------- latency-scheduled form
// One warp inverting one value is a chain of dependent instructions: 30 divsteps (each ~5 dependent
// operations on g) and then the matrix applied to 4 x L limbs, round after round.  Only the LOW TWO
// limbs of f and g decide the next round's matrix, so the rounds are software-pipelined: the next
// matrix is computed from the freshly updated low limbs in the SAME straight-line block as the rest
// of this round's update of f, g, d, e -- two independent instruction streams that the scheduler
// interleaves.  Same branch-free recurrence and round count as safegcd_inverse (one extra, unused,
// divsteps block at the end); EARLY_EXIT additionally stops once g is zero (data-dependent: for
// warp-uniform public values only).
GECC_HD int32_t divsteps_30_flat(int32_t zeta, uint32_t f0, uint32_t g0, trans2x2* t) {
    uint32_t u = 1, v = 0, q = 0, r = 1;
    uint32_t f = f0, g = g0;
#pragma unroll
    for (int i = 0; i < 30; ++i) {
        uint32_t c1 = (uint32_t)(zeta >> 31);
        uint32_t c2 = 0u - (g & 1u);
        uint32_t x = (f ^ c1) - c1;
        uint32_t y = (u ^ c1) - c1;
        uint32_t z = (v ^ c1) - c1;
        g += x & c2;
        q += y & c2;
        r += z & c2;
        c1 &= c2;
        zeta = (int32_t)(((uint32_t)zeta ^ c1) - 1u);
        f += g & c1;
        u += q & c1;
        v += r & c1;
        g >>= 1;
        u <<= 1;
        v <<= 1;
    }
    t->u = (int32_t)u;
    t->v = (int32_t)v;
    t->q = (int32_t)q;
    t->r = (int32_t)r;
    return zeta;
}
template <bool EARLY_EXIT, class F>
GECC_HD_CALL fel<F> safegcd_inverse_sched(const F& fld, const fel<F>& x) {
    GECC_COUNT(safegcd, F);
    constexpr int N = F::N, L = N == 8 ? 9 : (32 * N + 29) / 30, ROUNDS = N == 8 ? 20 : (49 * N + 16) / 17 + 1;
    const int32_t M30 = 0x3FFFFFFF;
    s30n<L> d, e, f, g;
#pragma unroll
    for (int i = 0; i < L; ++i) {
        d.v[i] = 0;
        e.v[i] = 0;
        f.v[i] = (int32_t)fld.q30(i);
    }
    e.v[0] = 1;
    g = s30_from_limbs<N, L>(x.w);
    trans2x2 t;
    int32_t zeta = divsteps_30_flat(-1, (uint32_t)f.v[0], (uint32_t)g.v[0], &t);
#pragma unroll 1
    for (int round = 0; round < ROUNDS; ++round) {
        // limb 0 of t * (f, g) / 2^30 from limbs 0 and 1 (the same arithmetic update_fg_30 does)
        const int64_t u = t.u, v = t.v, q = t.q, r = t.r;
        int64_t cf = u * f.v[0] + v * g.v[0];
        int64_t cg = q * f.v[0] + r * g.v[0];
        cf >>= 30;
        cg >>= 30;
        cf += u * f.v[1] + v * g.v[1];
        cg += q * f.v[1] + r * g.v[1];
        trans2x2 tn;
        const int32_t zn = divsteps_30_flat(zeta, (uint32_t)((int32_t)cf & M30), (uint32_t)((int32_t)cg & M30), &tn);
        update_de_30(fld, &d, &e, t);
        update_fg_30(&f, &g, t);
        t = tn;
        zeta = zn;
        if (EARLY_EXIT) {
            int32_t nz = 0;
#pragma unroll
            for (int i = 0; i < L; ++i) nz |= g.v[i];
            if (nz == 0) break;
        }
    }
    normalize_30(fld, &d, f.v[L - 1]);
    fel<F> res;
    s30_to_limbs<N, L>(res.w, d);
    return res;
}

#if defined(__CUDACC__)
#ifndef GECC_WARP_INV_VAR
#define GECC_WARP_INV_VAR false
#endif
// ---------------------------------------------------------------- warp-cooperative form
// One value inverted by a whole warp (every lane passes the SAME x; all 32 lanes must call).  A
// single thread's inversion is ~24 000 dependent-ish instructions; here the two halves of the warp
// split the work that does not sit on the critical chain:
//   * the transition matrix: lanes 0-15 track its first column (u, q), lanes 16-31 the second
//     (v, r) -- the same recurrence from different start values, 7 operations per divstep instead
//     of 14 -- and swap the columns with four shuffles per round;
//   * the big updates: lanes 0-15 hold (f, g), lanes 16-31 hold (d, e).  Both run the ONE routine
//     "(A, B) <- t (A, B) + (md, me) q, shifted down 30 bits" (md = me = 0 on the f, g half), with
//     signed wide multiply-adds (mad.wide.s32: one instruction per product; the C form compiles to
//     three);
//   * the next round's f0, g0 come back from lane 0 by shuffle; the rounds stop when g is zero
//     (uniform: the value is shared), the result leaves lanes 16-31 by shuffle.
// Same recurrence, same value as safegcd_inverse.  Public values only (early exit).
// VAR: the divsteps of a round by count-trailing-zeros runs and 6-bit cancellation (divsteps_30_var)
// instead of 30 branch-free steps -- a third of the instructions, data-dependent trip count.
template <bool VAR, class F>
__device__ __noinline__ fel<F> safegcd_inverse_warp(const F& fld, const fel<F>& x) {
    constexpr int N = F::N, L = N == 8 ? 9 : (32 * N + 29) / 30;
    constexpr int ROUNDS = VAR ? (N == 8 ? 25 : 37) : (N == 8 ? 20 : (49 * N + 16) / 17 + 1);
    const int32_t M30 = 0x3FFFFFFF;
    const unsigned FULL = 0xFFFFFFFFu;
    const bool de = (threadIdx.x & 16) != 0;  // this lane's half: (d, e) / second column
    s30n<L> A, B;                             // (f, g) or (d, e)
    {
        const s30n<L> g = s30_from_limbs<N, L>(x.w);
#pragma unroll
        for (int i = 0; i < L; ++i) {
            A.v[i] = de ? 0 : (int32_t)fld.q30(i);
            B.v[i] = de ? (i == 0 ? 1 : 0) : g.v[i];
        }
    }
    int32_t zeta = -1;
    uint32_t f0 = fld.q30(0), g0 = (uint32_t)__shfl_sync(FULL, B.v[0], 0);
#pragma unroll 1
    for (int round = 0; round < ROUNDS; ++round) {
        // 30 divsteps; this lane's column (a, b) of the matrix
        uint32_t a = de ? 0u : 1u, b = de ? 1u : 0u;
        uint32_t f = f0, g = g0;
        if constexpr (VAR) {  // zeta holds eta = -delta of the classic divsteps here
            uint32_t nf = f * (f * f - 2u);
            int i = 30;
            for (;;) {
                const int zeros = ctz32_nz(g | (0xFFFFFFFFu << i));
                g >>= zeros;
                a <<= zeros;
                zeta -= zeros;
                i -= zeros;
                if (i == 0) break;
                if (zeta < 0) {
                    zeta = -zeta;
                    uint32_t tmp = f; f = g; g = 0u - tmp;
                    tmp = a; a = b; b = 0u - tmp;
                    nf = f * (f * f - 2u);
                }
                const int limit = (zeta + 1) > i ? i : (zeta + 1);
                const uint32_t w = (g * nf) & (0xFFFFFFFFu >> (32 - limit)) & 63u;
                g += f * w;
                b += a * w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 30; ++i) {
                const uint32_t c1 = (uint32_t)(zeta >> 31);
                const uint32_t c2 = 0u - (g & 1u);
                const uint32_t c12 = c1 & c2;
                g = g + ((f ^ c1) & c2) - c12;   // see divsteps_30
                b = b + ((a ^ c1) & c2) - c12;
                zeta = (int32_t)(((uint32_t)zeta ^ c12) - 1u);
                f += g & c12;
                a += b & c12;
                g >>= 1;
                a <<= 1;
            }
        }
        const int32_t u = (int32_t)__shfl_sync(FULL, a, 0), q = (int32_t)__shfl_sync(FULL, b, 0);
        const int32_t v = (int32_t)__shfl_sync(FULL, a, 16), r = (int32_t)__shfl_sync(FULL, b, 16);
        // (A, B) <- (t (A, B) + (md, me) q) / 2^30; md = me = 0 on the (f, g) half (update_fg_30),
        // the modular correction of update_de_30 on the other
        const int32_t sa = A.v[L - 1] >> 31, sb = B.v[L - 1] >> 31;
        int32_t md = (u & sa) + (v & sb);
        int32_t me = (q & sa) + (r & sb);
        int64_t ca = mac_s32(u, A.v[0], mac_s32(v, B.v[0], 0));
        int64_t cb = mac_s32(q, A.v[0], mac_s32(r, B.v[0], 0));
        md -= (int32_t)((fld.qinv30() * (uint32_t)ca + (uint32_t)md) & (uint32_t)M30);
        me -= (int32_t)((fld.qinv30() * (uint32_t)cb + (uint32_t)me) & (uint32_t)M30);
        md = de ? md : 0;
        me = de ? me : 0;
        ca = mac_s32((int32_t)fld.q30(0), md, ca);
        cb = mac_s32((int32_t)fld.q30(0), me, cb);
        ca >>= 30;
        cb >>= 30;
#pragma unroll
        for (int i = 1; i < L; ++i) {
            const int32_t ai = A.v[i], bi = B.v[i];
            ca = mac_s32(u, ai, mac_s32(v, bi, mac_s32((int32_t)fld.q30(i), md, ca)));
            cb = mac_s32(q, ai, mac_s32(r, bi, mac_s32((int32_t)fld.q30(i), me, cb)));
            A.v[i - 1] = (int32_t)ca & M30;
            ca >>= 30;
            B.v[i - 1] = (int32_t)cb & M30;
            cb >>= 30;
        }
        A.v[L - 1] = (int32_t)ca;
        B.v[L - 1] = (int32_t)cb;
        int32_t nz = 0;
#pragma unroll
        for (int i = 0; i < L; ++i) nz |= B.v[i];
        f0 = (uint32_t)__shfl_sync(FULL, A.v[0], 0);
        g0 = (uint32_t)__shfl_sync(FULL, B.v[0], 0);
        if (__shfl_sync(FULL, nz, 0) == 0) break;  // g == 0: uniform over the warp
    }
    // d (lanes 16-31), negated when f (lanes 0-15) ended at -1
    const int32_t fsign = __shfl_sync(FULL, A.v[L - 1], 0);
    normalize_30(fld, &A, fsign);
    fel<F> res;
    s30_to_limbs<N, L>(res.w, A);
#pragma unroll
    for (int i = 0; i < N; ++i) res.w[i] = __shfl_sync(FULL, res.w[i], 16);
    return res;
}
// Montgomery-form inverse of a value shared by the whole warp (all 32 lanes call with the same a)
template <class F>
__device__ __forceinline__ fel<F> fe_inv_warp(const F& f, const fel<F>& a) {
    if constexpr (F::kind == KIND_SECP_LAZY) return safegcd_inverse_warp<GECC_WARP_INV_VAR>(f, lazy_canon(f, a));
    if constexpr (F::kind == KIND_SM2_LAZY) {
        fe r3l;
#pragma unroll
        for (int i = 0; i < 8; ++i) r3l.w[i] = f.r3(i);
        return fe_mul(f, safegcd_inverse_warp<GECC_WARP_INV_VAR>(f, weak_canon(f, a)), r3l);
    }
    fel<F> r3;
#pragma unroll
    for (int i = 0; i < F::N; ++i) r3.w[i] = f.r3(i);
    return fe_mul(f, safegcd_inverse_warp<GECC_WARP_INV_VAR>(f, a), r3);
}
#endif

// Montgomery-form inverse, variable time: for warp-uniform public values only (see above)
template <class F>
GECC_HD fel<F> fe_inv_var(const F& f, const fel<F>& a) {
    if constexpr (F::kind == KIND_SECP_LAZY) return safegcd_inverse_var(f, lazy_canon(f, a));
    if constexpr (F::kind == KIND_SM2_LAZY) {
        fe r3l;
#pragma unroll
        for (int i = 0; i < 8; ++i) r3l.w[i] = f.r3(i);
        return fe_mul(f, safegcd_inverse_var(f, weak_canon(f, a)), r3l);
    }
    fel<F> r3;
#pragma unroll
    for (int i = 0; i < F::N; ++i) r3.w[i] = f.r3(i);
    return fe_mul(f, safegcd_inverse_var(f, a), r3);
}

// Montgomery-form inverse of a Montgomery-form element (zero -> zero).
template <class F>
GECC_HD fel<F> fe_inv(const F& f, const fel<F>& a) {
    if constexpr (F::kind == KIND_SECP_LAZY) return safegcd_inverse(f, lazy_canon(f, a));  // plain in, plain out
    if constexpr (F::kind == KIND_SM2_LAZY) {  // weakly reduced Montgomery in, Montgomery out
        fe r3l;
#pragma unroll
        for (int i = 0; i < 8; ++i) r3l.w[i] = f.r3(i);
        return fe_mul(f, safegcd_inverse(f, weak_canon(f, a)), r3l);
    }
    fel<F> r3;
#pragma unroll
    for (int i = 0; i < F::N; ++i) r3.w[i] = f.r3(i);
    return fe_mul(f, safegcd_inverse(f, a), r3);
}

}  // namespace gecc
