// Per-lane (one thread = one signature / one scalar) building blocks of the fused
// ECDSA kernels.  All of it is __host__ __device__ so tests/hostsim can run the
// exact logic on the CPU.
//
// Reference behaviour being reproduced (values, not operation sequence):
//   nonce_scalar      DeterministicNonceSource::scalar_for + draw_scalar
//                     (protocol.cpp:13-34, 67-75), n parameterised
//   fixed_base_mul    batch_fpmul's result  s*G      (batch_point.cpp:358-426)
//   var_base_mul      batch_upmul's result  s*P      (batch_point.cpp:236-339)
//   sign_lane         one lane of ecdsa_sign_batch   (protocol.cpp:121-164)
//   verify_lane       one lane of ecdsa_verify_batch (protocol.cpp:184-220) +
//                     the C-ABI decoding rules (capi.cpp:207-226)
// The reference walks 256 bits with one shared inversion per bit; here each lane
// keeps a Jacobian accumulator in registers: s*G is WG-bit signed windows over a
// precomputed table of d*2^(WG*j)*G (no doublings), s*P is 4-bit signed windows
// over an 8-entry affine table of the lane's own point kept in shared memory.
#pragma once
#include "gecc_curve.cuh"
#include "gecc_dev.cuh"
#include "gecc_modinv.cuh"

// lanes signed by one thread of k_sign (they share one inversion mod p and one mod n)
#ifndef GECC_SIGN_K
#define GECC_SIGN_K 8
#endif

namespace gecc {

// ------------------------------------------------------------ scalars
GECC_HD fe u256_add(const fe& a, const fe& b, uint32_t* carry) {
    fe r;
    r.w[0] = add_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) r.w[i] = addc_cc(a.w[i], b.w[i]);
    *carry = addc(0, 0);
    return r;
}
GECC_HD fe u256_sub(const fe& a, const fe& b) {
    fe r;
    r.w[0] = sub_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) r.w[i] = subc_cc(a.w[i], b.w[i]);
    return r;
}
// v mod n for v < 2n: one conditional subtraction (Scalar::reduce, curve.cpp:22-27)
template <class Fn>
GECC_HD fe scalar_reduce_once(const fe& v) {
    const Fn f{};
    fe n = fe_modulus(f);
    return u256_lt(v, n) ? v : u256_sub(v, n);
}
// 0 < v < n (scalar_in_range, protocol.cpp:41-44)
template <class Fn>
GECC_HD bool scalar_in_range(const fe& v) {
    return !fe_is_zero(v) && fe_lt_modulus(Fn{}, v);
}

// k (already below n) or n - k, whichever is below 2^255 (n > 2^255 on every curve here), and
// whether it was flipped: k G = -((n - k) G).  A scalar below 2^255 leaves the top window of the
// signed recoding without a carry, so the fixed-base walk needs no addition of 2^256 G (one in
// two scalars otherwise): the caller negates every digit instead.
template <class Fn>
GECC_HD fe scalar_fold_half(const fe& k, bool* flipped) {
    *flipped = (k.w[7] >> 31) != 0;
    return *flipped ? u256_sub(fe_modulus(Fn{}), k) : k;
}

GECC_HD uint64_t splitmix64(uint64_t* x) {  // protocol.cpp:13-19
    *x += 0x9E3779B97F4A7C15ull;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
template <class Fn>
GECC_HD fe nonce_scalar(uint64_t seed, uint64_t stream, uint32_t attempt) {
    uint64_t state = seed;
    (void)splitmix64(&state);
    state ^= 0xA3EC647659359ACDull * (stream + 1);
    (void)splitmix64(&state);
    state ^= 0xC2B2AE3D27D4EB4Full * ((uint64_t)attempt + 1);
    for (;;) {
        fe raw;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            uint64_t v = splitmix64(&state);
            raw.w[i] = (uint32_t)v;
            raw.w[i + 1] = (uint32_t)(v >> 32);
        }
        if (scalar_in_range<Fn>(raw)) return raw;
    }
}

// Signed fixed-window recoding: k = sum_j (win_j(k + C) - 2^(W-1)) 2^(W j) + carry 2^256
// with C = sum_j 2^(W-1) 2^(W j); every digit lies in [-2^(W-1), 2^(W-1)-1] and can be
// read MSB-first without a dependent carry sweep.  W must divide 256.
template <int W>
struct Recoded {
    fe biased;       // (k + C) mod 2^256
    uint32_t carry;  // digit of the extra top window (0 or 1)
};
template <int W>
GECC_HD Recoded<W> recode_signed(const fe& k) {
    fe c;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t v = 0;
#pragma unroll
        for (int b = W - 1; b < 32; b += W) v |= 1u << b;
        c.w[i] = v;
    }
    static_assert(32 % W == 0 || W == 16, "window must tile the 32-bit limbs");
    Recoded<W> r;
    r.biased = u256_add(k, c, &r.carry);
    return r;
}
template <int W>
GECC_HD int recoded_digit(const Recoded<W>& r, int j) {  // j-th window, signed
    int bit = j * W;
    uint32_t v = (r.biased.w[bit >> 5] >> (bit & 31)) & ((1u << W) - 1u);
    return (int)v - (1 << (W - 1));
}

// ------------------------------------------------------------ fixed base
// Table layout (built by k_tables.cu): entry (j, d), d = 1 .. 2^(WG-1), holds the
// affine Montgomery point d * 2^(WG*j) * G as 16 words x[0..7] y[0..7] at
// tab[(j * 2^(WG-1) + d - 1) * 16].  Windows j = 0 .. 256/WG (the last one only
// ever uses d = 1).
template <int WG>
struct GTable {
    const uint32_t* tab;
    static constexpr int windows = 256 / WG + 1;
    static constexpr int per_window = 1 << (WG - 1);
    // requests the 64-byte row (j, d) ahead of its use: the rows are gathered at random from a
    // table that lives in L2, one per window, and each gather otherwise sits in the dependency chain
    GECC_HD void prefetch(int j, int d) const {
#if defined(__CUDA_ARCH__)
        const uint32_t* p = tab + ((size_t)j * per_window + (size_t)(d - 1)) * 16;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 8));
#else
        (void)j; (void)d;
#endif
    }
    GECC_HD aff load(int j, int d) const {  // d >= 1
        const uint32_t* p = tab + ((size_t)j * per_window + (size_t)(d - 1)) * 16;
        aff r;
#if defined(__CUDA_ARCH__)
        const uint4* q = reinterpret_cast<const uint4*>(p);
        uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), e = __ldg(q + 3);
        r.x.w[0] = a.x; r.x.w[1] = a.y; r.x.w[2] = a.z; r.x.w[3] = a.w;
        r.x.w[4] = b.x; r.x.w[5] = b.y; r.x.w[6] = b.z; r.x.w[7] = b.w;
        r.y.w[0] = c.x; r.y.w[1] = c.y; r.y.w[2] = c.z; r.y.w[3] = c.w;
        r.y.w[4] = e.x; r.y.w[5] = e.y; r.y.w[6] = e.z; r.y.w[7] = e.w;
#else
        for (int i = 0; i < 8; ++i) {
            r.x.w[i] = p[i];
            r.y.w[i] = p[8 + i];
        }
#endif
        return r;
    }
};

// k * G for any 256-bit k (the value of k mod n times G, like the reference's
// bit ladder on an unreduced scalar, acceptance.cpp:288-291).
template <class C, int WG>
GECC_HD jac fixed_base_mul(const fe& k_raw, const GTable<WG>& tab, const jac* start = nullptr) {
    const typename C::Fp f{};
    bool flip;
    fe k = scalar_fold_half<typename C::Fn>(scalar_reduce_once<typename C::Fn>(k_raw), &flip);
    Recoded<WG> rc = recode_signed<WG>(k);
    // `start`: the additions continue into an existing accumulator (start + k G): the verify
    // lane adds u1 G onto u2 Q this way, which saves the separate complete addition at the end
    jac acc = start ? *start : jac_infinity<C>();
    auto digit = [&](int j) { return j == 256 / WG ? (int)rc.carry : recoded_digit<WG>(rc, j); };
#pragma unroll 1
    for (int j = 0; j <= 256 / WG; ++j) {
        if (j < 256 / WG) {  // the next window's row is on its way while this window's addition runs
            const int dn = digit(j + 1);
            if (dn != 0) tab.prefetch(j + 1, dn < 0 ? -dn : dn);
        }
        int d = digit(j);
        if (d == 0) continue;
        aff t = tab.load(j, d < 0 ? -d : d);
        if ((d < 0) != flip) t.y = fe_neg(f, t.y);
        acc = jac_madd<C>(acc, t);
    }
    return acc;
}

// ---- constant-structure forms (GECC_SECRET_UNIFORM, SPEC.md "constant structure"; the
// reference applies every table entry by select, batch_point.cpp:319-333,420).  The sequence of
// instructions and of table ROWS touched does not depend on the scalar: every window performs its
// addition, a zero digit adds a dummy entry whose result is discarded by an arithmetic select,
// signs are applied by masked negation.  What stays data dependent is only the exceptional-relation
// branch inside the complete addition (accumulator equal to +- the addend), which a windowed
// recoding of a scalar below n reaches with negligible probability and which is kept so that the
// result is correct for EVERY input.
template <int N>
GECC_HD feN<N> fe_cmov(uint32_t m, const feN<N>& a, const feN<N>& b) {  // m all ones -> a, zero -> b
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = (a.w[i] & m) | (b.w[i] & ~m);
    return r;
}
// p + q with  keep == all ones -> p returned unchanged (the addition is still executed);
// p at infinity is handled by select, not by an early return.
template <class C>
GECC_HD_CALL cjac<C> jac_madd_uniform(const cjac<C>& p, const caff<C>& q, uint32_t keep) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    const typename C::Fp f{};
    const uint32_t pinf = jac_is_inf<C>(p) ? 0xFFFFFFFFu : 0u;
    fe z1z1 = fe_sqr(f, p.Z);
    fe u2 = fe_mul(f, q.x, z1z1);
    fe s2 = fe_mul(f, q.y, fe_mul(f, z1z1, p.Z));
    fe h = fe_sub(f, u2, p.X);
    fe rr = fe_sub(f, s2, p.Y);
    jac r;
    if (!pinf && fe_is_zero(f, h)) {  // accumulator == +-q: see the note above
        r = fe_is_zero(f, rr) ? jac_dbl<C>(p) : jac_infinity<C>();
    } else {
        fe hh = fe_sqr(f, h);
        fe hhh = fe_mul(f, hh, h);
        fe v = fe_mul(f, p.X, hh);
        r.X = fe_sub(f, fe_sub(f, fe_sub(f, fe_sqr(f, rr), hhh), v), v);
        r.Y = fe_sub(f, fe_mul(f, rr, fe_sub(f, v, r.X)), fe_mul(f, p.Y, hhh));
        r.Z = fe_mul(f, p.Z, h);
    }
    jac o;
    o.X = fe_cmov(keep, p.X, fe_cmov(pinf, q.x, r.X));
    o.Y = fe_cmov(keep, p.Y, fe_cmov(pinf, q.y, r.Y));
    o.Z = fe_cmov(keep, p.Z, fe_cmov(pinf, fe_one(f), r.Z));
    return o;
}

// k * G, constant structure: 17 window additions + the removal of the 2^256 G the accumulator
// starts from, always executed.  Table rows are gathered by address (one 64-byte row per window
// whatever the digit; digit 0 gathers row 1 and discards the sum).
template <class C, int WG>
GECC_HD jac fixed_base_mul_uniform(const fe& k_raw, const GTable<WG>& tab) {
    const typename C::Fp f{};
    fe k = scalar_reduce_once<typename C::Fn>(k_raw);
    Recoded<WG> rc = recode_signed<WG>(k);
    const aff top = tab.load(256 / WG, 1);  // 2^256 G
    jac acc;
    acc.X = top.x; acc.Y = top.y; acc.Z = fe_one(f);
#pragma unroll 1
    for (int j = 0; j < 256 / WG; ++j) {
        const int d = recoded_digit<WG>(rc, j);
        const int s = d >> 31;                       // all ones when d < 0
        const int mag = (d ^ s) - s;                 // |d|
        const uint32_t zero = mag == 0 ? 0xFFFFFFFFu : 0u;
        aff t = tab.load(j, mag + (int)(zero & 1u));  // row 1 stands in for the zero digit
        t.y = fe_cmov((uint32_t)s, fe_neg(f, t.y), t.y);
        acc = jac_madd_uniform<C>(acc, t, zero);
    }
    // acc = 2^256 G + sum_j d_j 2^(WG j) G; the true top digit is rc.carry: take 2^256 G off when it is 0
    aff mt = top;
    mt.y = fe_neg(f, mt.y);
    return jac_madd_uniform<C>(acc, mt, rc.carry ? 0xFFFFFFFFu : 0u);
}

// ------------------------------------------------------------ variable base
// 8-entry table of the lane's own point, entry e (0..7) = (e+1) * P, affine.
// `base` points at this lane's first word; consecutive words of one entry are
// `stride` words apart (stride = blockDim.x in shared memory: conflict-free,
// 1 on the host).
template <class C>
struct RowSrc;
struct LaneTable {
    uint32_t* base;
    int stride;
    template <class C>
    GECC_HD RowSrc<C> row(int e, bool neg, bool endo) const;  // entry e as a row source (defined below)
    GECC_HD void store(int e, const aff& p) const {
#if defined(__CUDA_ARCH__)
        if (stride == 1) {  // table in global memory, 64 B per entry, 16-byte aligned by construction
            uint4* q = reinterpret_cast<uint4*>(base + e * 16);
            q[0] = make_uint4(p.x.w[0], p.x.w[1], p.x.w[2], p.x.w[3]);
            q[1] = make_uint4(p.x.w[4], p.x.w[5], p.x.w[6], p.x.w[7]);
            q[2] = make_uint4(p.y.w[0], p.y.w[1], p.y.w[2], p.y.w[3]);
            q[3] = make_uint4(p.y.w[4], p.y.w[5], p.y.w[6], p.y.w[7]);
            return;
        }
#endif
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            base[(size_t)(e * 16 + i) * stride] = p.x.w[i];
            base[(size_t)(e * 16 + 8 + i) * stride] = p.y.w[i];
        }
    }
    GECC_HD fe load_x(int e) const { return load_half(e, 0); }
    GECC_HD fe load_y(int e) const { return load_half(e, 8); }
    GECC_HD fe load_half(int e, int off) const {  // one coordinate of entry e
        fe v;
#if defined(__CUDA_ARCH__)
        if (stride == 1) {
            const uint4* q = reinterpret_cast<const uint4*>(base + e * 16 + off);
            const uint4 a = q[0], b = q[1];
            v.w[0] = a.x; v.w[1] = a.y; v.w[2] = a.z; v.w[3] = a.w;
            v.w[4] = b.x; v.w[5] = b.y; v.w[6] = b.z; v.w[7] = b.w;
            return v;
        }
#endif
#pragma unroll
        for (int i = 0; i < 8; ++i) v.w[i] = base[(size_t)(e * 16 + off + i) * stride];
        return v;
    }
    GECC_HD aff load(int e) const {
        aff p;
#if defined(__CUDA_ARCH__)
        if (stride == 1) {
            const uint4* q = reinterpret_cast<const uint4*>(base + e * 16);
            uint4 a = q[0], b = q[1], c = q[2], d = q[3];
            p.x.w[0] = a.x; p.x.w[1] = a.y; p.x.w[2] = a.z; p.x.w[3] = a.w;
            p.x.w[4] = b.x; p.x.w[5] = b.y; p.x.w[6] = b.z; p.x.w[7] = b.w;
            p.y.w[0] = c.x; p.y.w[1] = c.y; p.y.w[2] = c.z; p.y.w[3] = c.w;
            p.y.w[4] = d.x; p.y.w[5] = d.y; p.y.w[6] = d.z; p.y.w[7] = d.w;
            return p;
        }
#endif
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            p.x.w[i] = base[(size_t)(e * 16 + i) * stride];
            p.y.w[i] = base[(size_t)(e * 16 + 8 + i) * stride];
        }
        return p;
    }
};

// entry `e` by a sweep over all eight rows (no secret-dependent address)
GECC_HD aff lane_table_sweep(const LaneTable& tab, int e) {
    aff r;
    r.x = fe_zero();
    r.y = fe_zero();
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
        const aff t = tab.load(i);
        const uint32_t m = i == e ? 0xFFFFFFFFu : 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            r.x.w[w] |= t.x.w[w] & m;
            r.y.w[w] |= t.y.w[w] & m;
        }
    }
    return r;
}

// Builds {1..8} * P in affine form with ONE field inversion (Montgomery's trick
// over the seven Jacobian Z's).  P must be finite and on the curve.
template <class C>
GECC_HD void build_lane_table(const aff& p, const LaneTable& tab) {
    const typename C::Fp f{};
    jac m[8];
    m[0].X = p.x; m[0].Y = p.y; m[0].Z = fe_one(f);
    m[1] = jac_dbl<C>(m[0]);
    m[2] = jac_madd<C>(m[1], p);
    m[3] = jac_dbl<C>(m[1]);
    m[4] = jac_madd<C>(m[3], p);
    m[5] = jac_dbl<C>(m[2]);
    m[6] = jac_madd<C>(m[5], p);
    m[7] = jac_dbl<C>(m[3]);
    // prefix products of Z_1..Z_7 (none is zero: the group has prime order > 8)
    fe pre[8];
    pre[1] = m[1].Z;
#pragma unroll
    for (int i = 2; i < 8; ++i) pre[i] = fe_mul(f, pre[i - 1], m[i].Z);
    fe inv = fe_inv(f, pre[7]);
    tab.store(0, p);
#pragma unroll
    for (int i = 7; i >= 1; --i) {
        fe zi = i > 1 ? fe_mul(f, inv, pre[i - 1]) : inv;
        if (i > 1) inv = fe_mul(f, inv, m[i].Z);
        tab.store(i, jac_to_aff_with<C>(m[i], zi));
    }
}

// The same table WITHOUT the inversion, for curves with a = 0: the eight multiples are brought to a
// COMMON denominator Zc = Z_1 ... Z_7 (entry i scaled by s_i = Zc / Z_i: x' = X_i s_i^2, y' = Y_i s_i^3)
// and (x', y') are used as AFFINE points of the isomorphic curve y^2 = x^3 + b Zc^6 -- the doubling
// and mixed-addition formulas of an a = 0 curve do not contain b, and the endomorphism is
// (x', y') -> (beta x', y') there as well.  A ladder run on these entries gives (X', Y', Z'), which is
// the point (X', Y', Z' Zc) of the original curve: one multiplication instead of ~19 000 instructions
// of inversion per table.  Returns Zc.  (The trick of "effective affine" tables; P finite, on the curve.)
template <class C>
GECC_HD fe build_lane_table_isomorphic(const aff& p, const LaneTable& tab) {
    static_assert(C::a_kind == A_ZERO, "the isomorphic curve keeps the formulas only when a = 0");
    const typename C::Fp f{};
    jac m[8];
    m[0].X = p.x; m[0].Y = p.y; m[0].Z = fe_one(f);
    m[1] = jac_dbl<C>(m[0]);
    m[2] = jac_madd<C>(m[1], p);
    m[3] = jac_dbl<C>(m[1]);
    m[4] = jac_madd<C>(m[3], p);
    m[5] = jac_dbl<C>(m[2]);
    m[6] = jac_madd<C>(m[5], p);
    m[7] = jac_dbl<C>(m[3]);
    // prefix / suffix products of Z_1 .. Z_7 (none is zero: the group has prime order > 8)
    fe pre[8], suf[9];
    pre[1] = m[1].Z;
#pragma unroll
    for (int i = 2; i < 8; ++i) pre[i] = fe_mul(f, pre[i - 1], m[i].Z);
    suf[7] = m[7].Z;
#pragma unroll
    for (int i = 6; i >= 2; --i) suf[i] = fe_mul(f, suf[i + 1], m[i].Z);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const fe s = i == 0 ? pre[7] : i == 1 ? suf[2] : i == 7 ? pre[6] : fe_mul(f, pre[i - 1], suf[i + 1]);
        const fe s2 = fe_sqr(f, s);
        tab.store(i, aff{fe_mul(f, m[i].X, s2), fe_mul(f, m[i].Y, fe_mul(f, s2, s))});
    }
    return pre[7];
}

// ---- GLV split for curves with the endomorphism phi(x, y) = (beta x, y) = lambda (x, y)
// (secp256k1; Gallant-Lambert-Vanstone 2001).  k = k1 + k2 lambda (mod n) with
// |k1|, |k2| < 2^129, by rounding k onto the lattice basis (a1, b1), (a2, b2):
//   c1 = round(k g1 / 2^384), c2 = round(k g2 / 2^384)
//   k1 = k - c1 a1 - c2 a2,   k2 = c1 (-b1) - c2 b2        (exact integers)
// The ladder then needs 132 doublings instead of 256.
struct GlvSplit {
    fe m1, m2;        // magnitudes (upper limbs zero)
    bool neg1, neg2;  // signs
};

// out[na+nb] = a[na] * b[nb], small schoolbook on 64-bit accumulators
template <int NA, int NB>
GECC_HD void mul_small(uint32_t* out, const uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int i = 0; i < NA + NB; ++i) out[i] = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
        uint64_t carry = 0;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            uint64_t t = (uint64_t)a[i] * b[j] + out[i + j] + carry;
            out[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
        out[i + NB] = (uint32_t)carry;
    }
}
// r[N] = a[N] - b[N]; returns true when the result is negative, in which case r = b - a
// (branch-free: the sign of a GLV half is a function of the secret scalar in sign / keygen / ECDH)
template <int N>
GECC_HD bool sub_abs(uint32_t* r, const uint32_t* a, const uint32_t* b) {
    r[0] = sub_cc(a[0], b[0]);
#pragma unroll
    for (int i = 1; i < N; ++i) r[i] = subc_cc(a[i], b[i]);
    const uint32_t m = subc(0, 0);  // all ones when a < b
    // two's complement negation under the mask: (r ^ m) + (m & 1)
    r[0] = add_cc(r[0] ^ m, m & 1u);
#pragma unroll
    for (int i = 1; i < N; ++i) r[i] = addc_cc(r[i] ^ m, 0);
    return m != 0;
}

template <class C>
GECC_HD GlvSplit glv_split(const fe& k) {
    uint32_t g[8], t[16], c1[5], c2[5];
    // c = (k g + 2^383) >> 384
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = C::glv_g1(i);
    mul_wide8(t, k.w, g);
    c1[0] = add_cc(t[12], t[11] >> 31);
    c1[1] = addc_cc(t[13], 0);
    c1[2] = addc_cc(t[14], 0);
    c1[3] = addc_cc(t[15], 0);
    c1[4] = addc(0, 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = C::glv_g2(i);
    mul_wide8(t, k.w, g);
    c2[0] = add_cc(t[12], t[11] >> 31);
    c2[1] = addc_cc(t[13], 0);
    c2[2] = addc_cc(t[14], 0);
    c2[3] = addc_cc(t[15], 0);
    c2[4] = addc(0, 0);
    uint32_t a1[4], a2[5], mb1[4], b2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a1[i] = C::glv_a1(i);
        mb1[i] = C::glv_minus_b1(i);
        b2[i] = C::glv_b2(i);
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) a2[i] = C::glv_a2(i);
    // k1 = k - (c1 a1 + c2 a2), 10-limb arithmetic
    uint32_t p1[10], p2[10], s[10], kk[10], d[10];
    mul_small<5, 4>(p1, c1, a1);
    p1[9] = 0;
    mul_small<5, 5>(p2, c2, a2);
    s[0] = add_cc(p1[0], p2[0]);
#pragma unroll
    for (int i = 1; i < 10; ++i) s[i] = addc_cc(p1[i], p2[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) kk[i] = k.w[i];
    kk[8] = kk[9] = 0;
    GlvSplit r;
    r.neg1 = sub_abs<10>(d, kk, s);
#pragma unroll
    for (int i = 0; i < 8; ++i) r.m1.w[i] = d[i];
    // k2 = c1 (-b1) - c2 b2, 9-limb arithmetic
    uint32_t u1[9], u2[9], e[9];
    mul_small<5, 4>(u1, c1, mb1);
    mul_small<5, 4>(u2, c2, b2);
    r.neg2 = sub_abs<9>(e, u1, u2);
#pragma unroll
    for (int i = 0; i < 8; ++i) r.m2.w[i] = e[i];
    return r;
}

// k * P, P finite and on the curve, any 256-bit k (k mod n is what is computed).
template <class C>
GECC_HD jac var_base_mul(const fe& k_raw, const LaneTable& tab) {
    const typename C::Fp f{};
    fe k = scalar_reduce_once<typename C::Fn>(k_raw);
    jac acc = jac_infinity<C>();
    if constexpr (C::has_glv) {
        const GlvSplit sp = glv_split<C>(k);
        const Recoded<4> r1 = recode_signed<4>(sp.m1), r2 = recode_signed<4>(sp.m2);
        fe beta;
#pragma unroll
        for (int i = 0; i < 8; ++i) beta.w[i] = C::beta(i);
        // magnitudes are below 2^129: windows 0..32 plus the recoding carry in window 33
#pragma unroll 1
        for (int j = 33; j >= 0; --j) {
            if (j != 33) {
                acc = jac_dbl<C>(acc);
                acc = jac_dbl<C>(acc);
                acc = jac_dbl<C>(acc);
                acc = jac_dbl<C>(acc);
            }
            int d1 = recoded_digit<4>(r1, j), d2 = recoded_digit<4>(r2, j);
            if (sp.neg1) d1 = -d1;
            if (sp.neg2) d2 = -d2;
            if (d1 != 0) {
                aff t = tab.load((d1 < 0 ? -d1 : d1) - 1);
                if (d1 < 0) t.y = fe_neg(f, t.y);
                acc = jac_madd<C>(acc, t);
            }
            if (d2 != 0) {  // phi(d P) = (beta x, y)
                aff t = tab.load((d2 < 0 ? -d2 : d2) - 1);
                t.x = fe_mul(f, t.x, beta);
                if (d2 < 0) t.y = fe_neg(f, t.y);
                acc = jac_madd<C>(acc, t);
            }
        }
        return acc;
    } else {
        Recoded<4> rc = recode_signed<4>(k);
        if (rc.carry) {
            aff t = tab.load(0);
            acc.X = t.x; acc.Y = t.y; acc.Z = fe_one(f);
        }
#pragma unroll 1
        for (int j = 63; j >= 0; --j) {
            acc = jac_dbl<C>(acc);
            acc = jac_dbl<C>(acc);
            acc = jac_dbl<C>(acc);
            acc = jac_dbl<C>(acc);
            int d = recoded_digit<4>(rc, j);
            if (d != 0) {
                aff t = tab.load((d < 0 ? -d : d) - 1);
                if (d < 0) t.y = fe_neg(f, t.y);
                acc = jac_madd<C>(acc, t);
            }
        }
        return acc;
    }
}

// k * P, constant structure (the scalar is the secret of ECDH): every window doubles four times
// and performs its addition(s); entries come from a sweep over the whole lane table.
template <class C>
GECC_HD jac var_base_mul_uniform(const fe& k_raw, const LaneTable& tab) {
    const typename C::Fp f{};
    fe k = scalar_reduce_once<typename C::Fn>(k_raw);
    jac acc = jac_infinity<C>();
    auto step = [&](int d, bool endo) {
        const int s = d >> 31;
        const int mag = (d ^ s) - s;
        const uint32_t zero = mag == 0 ? 0xFFFFFFFFu : 0u;
        aff t = lane_table_sweep(tab, mag - 1 + (int)(zero & 1u));
        if constexpr (C::has_glv) {
            if (endo) {  // public choice: which half of the split this digit belongs to
                fe beta;
#pragma unroll
                for (int i = 0; i < 8; ++i) beta.w[i] = C::beta(i);
                t.x = fe_mul(f, t.x, beta);
            }
        }
        t.y = fe_cmov((uint32_t)s, fe_neg(f, t.y), t.y);
        acc = jac_madd_uniform<C>(acc, t, zero);
    };
    if constexpr (C::has_glv) {
        const GlvSplit sp = glv_split<C>(k);
        const Recoded<4> r1 = recode_signed<4>(sp.m1), r2 = recode_signed<4>(sp.m2);
        const int n1 = sp.neg1 ? -1 : 0, n2 = sp.neg2 ? -1 : 0;
#pragma unroll 1
        for (int j = 33; j >= 0; --j) {
            if (j != 33) {
                acc = jac_dbl<C>(acc);
                acc = jac_dbl<C>(acc);
                acc = jac_dbl<C>(acc);
                acc = jac_dbl<C>(acc);
            }
            const int d1 = recoded_digit<4>(r1, j), d2 = recoded_digit<4>(r2, j);
            step((d1 ^ n1) - n1, false);
            step((d2 ^ n2) - n2, true);
        }
    } else {
        Recoded<4> rc = recode_signed<4>(k);
        step((int)rc.carry, false);  // top digit: 0 or 1
#pragma unroll 1
        for (int j = 63; j >= 0; --j) {
            acc = jac_dbl<C>(acc);
            acc = jac_dbl<C>(acc);
            acc = jac_dbl<C>(acc);
            acc = jac_dbl<C>(acc);
            step(recoded_digit<4>(rc, j), false);
        }
    }
    return acc;
}

// ------------------------------------------------------------ accumulator at rest in shared memory
// The verify ladder (132 doublings + ~80 mixed additions per signature) spends ~13 % of its
// instructions moving registers around the two product calls and ~4 % spilling the accumulator:
// every value that lives across a call has to be copied out of the argument registers.  Here the
// accumulator and the formulas' temporaries REST in per-thread shared-memory slots (16-byte
// granules, granule g of slot s of thread t at [(2 s + g) * stride + t]: conflict-free LDS.128 /
// STS.128); an operand is loaded straight into the argument registers where it is consumed and a
// result is stored straight from the return registers, so nothing is live across a call but
// addresses.  Same formulas, same values as jac_dbl / jac_madd.
struct PointSlots {
    enum { SX = 0, SY, SZ, S1, S2, S3, S4, S5, COUNT };
#if defined(__CUDA_ARCH__)
    uint32_t addr;    // shared-window byte address of this thread's granule 0 of slot 0
    uint32_t pitch;   // bytes between consecutive granules of one thread (16 * threads per block)
    __device__ __forceinline__ fe ld(int s) const {
        fe r;
        const uint32_t a = addr + (uint32_t)(2 * s) * pitch;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]) : "r"(a));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]) : "r"(a + pitch));
        return r;
    }
    __device__ __forceinline__ void st(int s, const fe& v) const {
        const uint32_t a = addr + (uint32_t)(2 * s) * pitch;
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]) : "memory");
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a + pitch), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7]) : "memory");
    }
#else
    fe* slots;  // COUNT elements (host-sim)
    fe ld(int s) const { return slots[s]; }
    void st(int s, const fe& v) const { slots[s] = v; }
#endif
    GECC_HD jac load_point() const { return jac{ld(SX), ld(SY), ld(SZ)}; }
    GECC_HD void store_point(const jac& p) const {
        st(SX, p.X);
        st(SY, p.Y);
        st(SZ, p.Z);
    }
};

template <class C>
GECC_HD_CALL void jac_dbl_slots(const PointSlots S) {
    using P = PointSlots;
    const typename C::Fp f{};
    if constexpr (C::a_kind == A_ZERO) {  // dbl-2009-l, as jac_dbl
        S.st(P::S1, fe_sqr(f, S.ld(P::SX)));                                   // A
        S.st(P::S2, fe_sqr(f, S.ld(P::SY)));                                   // B
        S.st(P::S3, fe_sqr(f, S.ld(P::S2)));                                   // C
        {
            const fe T = fe_sqr(f, fe_add(f, S.ld(P::SX), S.ld(P::S2)));
            S.st(P::S4, fe_dbl(f, fe_sub(f, fe_sub(f, T, S.ld(P::S1)), S.ld(P::S3))));  // D
        }
        S.st(P::SZ, fe_dbl(f, fe_mul(f, S.ld(P::SY), S.ld(P::SZ))));           // Z3 = 2 Y Z
        {
            const fe A = S.ld(P::S1);
            S.st(P::S1, fe_add(f, fe_dbl(f, A), A));                           // E = 3A
        }
        {
            const fe F = fe_sqr(f, S.ld(P::S1));
            S.st(P::SX, fe_sub(f, F, fe_dbl(f, S.ld(P::S4))));                 // X3 = F - 2D
        }
        {
            const fe M = fe_mul(f, S.ld(P::S1), fe_sub(f, S.ld(P::S4), S.ld(P::SX)));
            S.st(P::SY, fe_sub(f, M, fe_mul8(f, S.ld(P::S3))));                // Y3 = E (D - X3) - 8C
        }
    } else if constexpr (C::a_kind == A_MINUS3) {  // dbl-2001-b, as jac_dbl
        S.st(P::S1, fe_sqr(f, S.ld(P::SZ)));                                   // delta
        S.st(P::S2, fe_sqr(f, S.ld(P::SY)));                                   // gamma
        S.st(P::S3, fe_mul(f, S.ld(P::SX), S.ld(P::S2)));                      // beta
        {
            const fe X = S.ld(P::SX), d = S.ld(P::S1);
            const fe t = fe_mul(f, fe_sub(f, X, d), fe_add(f, X, d));
            S.st(P::S4, fe_add(f, fe_dbl(f, t), t));                           // alpha
        }
        // Z3 = 2 Y Z as a product: (Y + Z)^2 - gamma - delta trades the multiply for a square and three
        // additions, which is MORE instructions on a field whose reduction is additions
        S.st(P::SZ, fe_dbl(f, fe_mul(f, S.ld(P::SY), S.ld(P::SZ))));
        {
            const fe a2 = fe_sqr(f, S.ld(P::S4));
            const fe beta4 = fe_dbl(f, fe_dbl(f, S.ld(P::S3)));
            const fe X3 = fe_sub(f, a2, fe_dbl(f, beta4));
            S.st(P::SX, X3);
            S.st(P::S3, fe_sub(f, beta4, X3));                                 // 4 beta - X3
        }
        S.st(P::S2, fe_mul8(f, fe_sqr(f, S.ld(P::S2))));                       // 8 gamma^2
        S.st(P::SY, fe_sub(f, fe_mul(f, S.ld(P::S4), S.ld(P::S3)), S.ld(P::S2)));
    } else {
        S.store_point(jac_dbl<C>(S.load_point()));
    }
}

// A 64-byte table row x[8] y[8] (a lane-table entry or a fixed-base table entry; `stride` words
// between consecutive words: 1 for rows in global memory), optionally mapped by the endomorphism
// (x -> beta x) and / or negated.  The coordinates are reloaded where the formulas consume them.
template <class C>
struct RowSrc {
    const uint32_t* row;
    int stride;
    bool neg, endo;
    GECC_HD fe half(int off) const {
        fe v;
#if defined(__CUDA_ARCH__)
        if (stride == 1) {
            const uint4* q = reinterpret_cast<const uint4*>(row + off);
            const uint4 a = __ldg(q), b = __ldg(q + 1);
            v.w[0] = a.x; v.w[1] = a.y; v.w[2] = a.z; v.w[3] = a.w;
            v.w[4] = b.x; v.w[5] = b.y; v.w[6] = b.z; v.w[7] = b.w;
            return v;
        }
#endif
#pragma unroll
        for (int i = 0; i < 8; ++i) v.w[i] = row[(size_t)(off + i) * stride];
        return v;
    }
    GECC_HD fe x() const {
        fe v = half(0);
        if constexpr (C::has_glv) {
            if (endo) {
                fe beta;
#pragma unroll
                for (int i = 0; i < 8; ++i) beta.w[i] = C::beta(i);
                v = fe_mul(typename C::Fp{}, v, beta);
            }
        }
        return v;
    }
    GECC_HD fe y() const {
        const fe v = half(8);
        return neg ? fe_neg(typename C::Fp{}, v) : v;
    }
    GECC_HD aff point() const { return aff{x(), y()}; }
};

template <class C>
GECC_HD RowSrc<C> LaneTable::row(int e, bool neg, bool endo) const {
    return RowSrc<C>{base + (size_t)e * 16 * stride, stride, neg, endo};
}

// acc += q, q finite and affine, given as a row source.  Complete, as jac_madd.
template <class C>
GECC_HD_CALL void jac_madd_slots(const PointSlots S, const RowSrc<C> src) {
    using P = PointSlots;
    const typename C::Fp f{};
    {
        const fe Z = S.ld(P::SZ);
        if (fe_is_zero(f, Z)) {  // accumulator at infinity
            const aff q = src.point();
            S.st(P::SX, q.x);
            S.st(P::SY, q.y);
            S.st(P::SZ, fe_one(f));
            return;
        }
        S.st(P::S1, fe_sqr(f, Z));                                             // Z^2
    }
    bool h_zero;
    {
        const fe h = fe_sub(f, fe_mul(f, src.x(), S.ld(P::S1)), S.ld(P::SX));  // u2 - X
        h_zero = fe_is_zero(f, h);
        S.st(P::S2, h);
    }
    {
        const fe zzz = fe_mul(f, S.ld(P::S1), S.ld(P::SZ));
        S.st(P::S3, fe_sub(f, fe_mul(f, src.y(), zzz), S.ld(P::SY)));          // r = s2 - Y
    }
    if (h_zero) {  // accumulator == +-q: the complete formulas
        S.store_point(jac_madd<C>(S.load_point(), src.point()));
        return;
    }
    S.st(P::S1, fe_sqr(f, S.ld(P::S2)));                                       // hh
    S.st(P::S4, fe_mul(f, S.ld(P::S1), S.ld(P::S2)));                          // hhh
    S.st(P::S5, fe_mul(f, S.ld(P::SX), S.ld(P::S1)));                          // v = X hh
    {
        const fe r2 = fe_sqr(f, S.ld(P::S3));
        const fe v = S.ld(P::S5);
        S.st(P::SX, fe_sub(f, fe_sub(f, fe_sub(f, r2, S.ld(P::S4)), v), v));   // X3 = r^2 - hhh - 2v
    }
    S.st(P::S4, fe_mul(f, S.ld(P::SY), S.ld(P::S4)));                          // Y hhh
    S.st(P::SY, fe_sub(f, fe_mul(f, S.ld(P::S3), fe_sub(f, S.ld(P::S5), S.ld(P::SX))), S.ld(P::S4)));
    S.st(P::SZ, fe_mul(f, S.ld(P::SZ), S.ld(P::S2)));                          // Z3 = Z h
}

// acc += q with the accumulator AFFINE (Z == 1: the second addition of a fixed-base walk, whose
// first one only places a table row): 4M + 2S instead of 8M + 3S.  Complete (falls back on +-q).
template <class C>
GECC_HD_CALL void jac_mmadd_slots(const PointSlots S, const RowSrc<C> src) {
    using P = PointSlots;
    const typename C::Fp f{};
    {
        const fe h = fe_sub(f, src.x(), S.ld(P::SX));                          // x2 - X
        if (fe_is_zero(f, h)) {
            jac_madd_slots<C>(S, src);
            return;
        }
        S.st(P::S2, h);
    }
    S.st(P::S3, fe_sub(f, src.y(), S.ld(P::SY)));                              // r = y2 - Y
    S.st(P::S1, fe_sqr(f, S.ld(P::S2)));                                       // hh
    S.st(P::S4, fe_mul(f, S.ld(P::S1), S.ld(P::S2)));                          // hhh
    S.st(P::S5, fe_mul(f, S.ld(P::SX), S.ld(P::S1)));                          // v = X hh
    {
        const fe r2 = fe_sqr(f, S.ld(P::S3));
        const fe v = S.ld(P::S5);
        S.st(P::SX, fe_sub(f, fe_sub(f, fe_sub(f, r2, S.ld(P::S4)), v), v));   // X3 = r^2 - hhh - 2v
    }
    S.st(P::S4, fe_mul(f, S.ld(P::SY), S.ld(P::S4)));                          // Y hhh
    S.st(P::SY, fe_sub(f, fe_mul(f, S.ld(P::S3), fe_sub(f, S.ld(P::S5), S.ld(P::SX))), S.ld(P::S4)));
    S.st(P::SZ, S.ld(P::S2));                                                  // Z3 = h
}

// ---- the same additions on (X, Y, ZZ, ZZZ) = (X, Y, Z^2, Z^3): a walk made of mixed additions only
// never needs Z itself (ZZ3 = ZZ PP, ZZZ3 = ZZZ PPP), which saves the squaring of Z in every
// addition: 8M + 2S.  Slots: SX, SY, SZ = ZZ, S1 = ZZZ; infinity is ZZ == 0.  Complete.
template <class C>
GECC_HD_CALL void zz_madd_slots(const PointSlots S, const RowSrc<C> src) {
    using P = PointSlots;
    const typename C::Fp f{};
    if (fe_is_zero(f, S.ld(P::SZ))) {  // accumulator at infinity: place the row
        const aff q = src.point();
        S.st(P::SX, q.x);
        S.st(P::SY, q.y);
        S.st(P::SZ, fe_one(f));
        S.st(P::S1, fe_one(f));
        return;
    }
    bool p_zero;
    {
        const fe p = fe_sub(f, fe_mul(f, src.x(), S.ld(P::SZ)), S.ld(P::SX));  // P = x2 ZZ - X
        p_zero = fe_is_zero(f, p);
        S.st(P::S2, p);
    }
    S.st(P::S3, fe_sub(f, fe_mul(f, src.y(), S.ld(P::S1)), S.ld(P::SY)));      // R = y2 ZZZ - Y
    if (p_zero) {  // accumulator == +-q
        if (fe_is_zero(f, S.ld(P::S3))) {  // == q: the tangent at the affine point
            const aff q = src.point();
            const jac d = jac_dbl<C>(jac{q.x, q.y, fe_one(f)});
            const fe zz = fe_sqr(f, d.Z);
            S.st(P::SX, d.X);
            S.st(P::SY, d.Y);
            S.st(P::SZ, zz);
            S.st(P::S1, fe_mul(f, zz, d.Z));
        } else {
            S.st(P::SZ, fe_zero());
            S.st(P::S1, fe_zero());
        }
        return;
    }
    S.st(P::S4, fe_sqr(f, S.ld(P::S2)));                                       // PP
    S.st(P::S5, fe_mul(f, S.ld(P::S2), S.ld(P::S4)));                          // PPP
    S.st(P::S2, fe_mul(f, S.ld(P::SX), S.ld(P::S4)));                          // Q = X PP
    S.st(P::SZ, fe_mul(f, S.ld(P::SZ), S.ld(P::S4)));                          // ZZ3
    S.st(P::S1, fe_mul(f, S.ld(P::S1), S.ld(P::S5)));                          // ZZZ3
    {
        const fe r2 = fe_sqr(f, S.ld(P::S3));
        const fe q = S.ld(P::S2);
        S.st(P::SX, fe_sub(f, fe_sub(f, fe_sub(f, r2, S.ld(P::S5)), q), q));   // X3 = R^2 - PPP - 2Q
    }
    S.st(P::S4, fe_mul(f, S.ld(P::SY), S.ld(P::S5)));                          // Y PPP
    S.st(P::SY, fe_sub(f, fe_mul(f, S.ld(P::S3), fe_sub(f, S.ld(P::S2), S.ld(P::SX))), S.ld(P::S4)));
}
// the accumulator affine (ZZ == ZZZ == 1, the state right after a row was placed): 4M + 2S
template <class C>
GECC_HD_CALL void zz_mmadd_slots(const PointSlots S, const RowSrc<C> src) {
    using P = PointSlots;
    const typename C::Fp f{};
    {
        const fe p = fe_sub(f, src.x(), S.ld(P::SX));
        if (fe_is_zero(f, p)) {
            zz_madd_slots<C>(S, src);
            return;
        }
        S.st(P::S2, p);
    }
    S.st(P::S3, fe_sub(f, src.y(), S.ld(P::SY)));                              // R
    S.st(P::SZ, fe_sqr(f, S.ld(P::S2)));                                       // ZZ3 = PP
    S.st(P::S1, fe_mul(f, S.ld(P::S2), S.ld(P::SZ)));                          // ZZZ3 = PPP
    S.st(P::S2, fe_mul(f, S.ld(P::SX), S.ld(P::SZ)));                          // Q = X PP
    {
        const fe r2 = fe_sqr(f, S.ld(P::S3));
        const fe q = S.ld(P::S2);
        S.st(P::SX, fe_sub(f, fe_sub(f, fe_sub(f, r2, S.ld(P::S1)), q), q));
    }
    S.st(P::S4, fe_mul(f, S.ld(P::SY), S.ld(P::S1)));                          // Y PPP
    S.st(P::SY, fe_sub(f, fe_mul(f, S.ld(P::S3), fe_sub(f, S.ld(P::S2), S.ld(P::SX))), S.ld(P::S4)));
}

// var_base_mul with the accumulator in the slots (result left there)
template <class C>
GECC_HD void var_base_mul_slots(const fe& k_raw, const LaneTable& tab, const PointSlots S) {
    const typename C::Fp f{};
    const fe k = scalar_reduce_once<typename C::Fn>(k_raw);
    S.store_point(jac_infinity<C>());
    if constexpr (C::has_glv) {
        const GlvSplit sp = glv_split<C>(k);
        const Recoded<4> r1 = recode_signed<4>(sp.m1), r2 = recode_signed<4>(sp.m2);
#pragma unroll 1
        for (int j = 33; j >= 0; --j) {
            if (j != 33) {
                jac_dbl_slots<C>(S);
                jac_dbl_slots<C>(S);
                jac_dbl_slots<C>(S);
                jac_dbl_slots<C>(S);
            }
            int d1 = recoded_digit<4>(r1, j), d2 = recoded_digit<4>(r2, j);
            if (sp.neg1) d1 = -d1;
            if (sp.neg2) d2 = -d2;
            if (d1 != 0) jac_madd_slots<C>(S, tab.template row<C>((d1 < 0 ? -d1 : d1) - 1, d1 < 0, false));
            if (d2 != 0) jac_madd_slots<C>(S, tab.template row<C>((d2 < 0 ? -d2 : d2) - 1, d2 < 0, true));
        }
    } else {
        const Recoded<4> rc = recode_signed<4>(k);
        if (rc.carry) {
            const aff t = tab.load(0);
            S.store_point(jac{t.x, t.y, fe_one(f)});
        }
#pragma unroll 1
        for (int j = 63; j >= 0; --j) {
            jac_dbl_slots<C>(S);
            jac_dbl_slots<C>(S);
            jac_dbl_slots<C>(S);
            jac_dbl_slots<C>(S);
            const int d = recoded_digit<4>(rc, j);
            if (d != 0) jac_madd_slots<C>(S, tab.template row<C>((d < 0 ? -d : d) - 1, d < 0, false));
        }
    }
}
// k * P, P finite and on the curve, table built here: the route the kernels take (table on the
// isomorphic curve when a = 0 -- no inversion; result in the slots, on the curve itself)
template <class C>
GECC_HD void var_base_mul_point_slots(const fe& k, const aff& P, const LaneTable& tab, const PointSlots S) {
    if constexpr (C::a_kind == A_ZERO) {
        const fe zc = build_lane_table_isomorphic<C>(P, tab);
        var_base_mul_slots<C>(k, tab, S);
        S.st(PointSlots::SZ, fe_mul(typename C::Fp{}, S.ld(PointSlots::SZ), zc));
    } else {
        build_lane_table<C>(P, tab);
        var_base_mul_slots<C>(k, tab, S);
    }
}
// the accumulator in the slots += k G (fixed_base_mul with `start`)
// fresh: the accumulator is known to be at infinity (k G alone): the first addition places its
// row, the second one runs on an affine accumulator
template <class C, int WG>
GECC_HD void fixed_base_add_slots(const fe& k_raw, const GTable<WG>& tab, const PointSlots S, bool fresh = false) {
    int placed = fresh ? 0 : 2;
    bool flip;
    const fe k = scalar_fold_half<typename C::Fn>(scalar_reduce_once<typename C::Fn>(k_raw), &flip);
    const Recoded<WG> rc = recode_signed<WG>(k);
    auto digit = [&](int j) { return j == 256 / WG ? (int)rc.carry : recoded_digit<WG>(rc, j); };
#pragma unroll 1
    for (int j = 0; j <= 256 / WG; ++j) {
        if (j < 256 / WG) {
            const int dn = digit(j + 1);
            if (dn != 0) tab.prefetch(j + 1, dn < 0 ? -dn : dn);
        }
        const int d = digit(j);
        if (d == 0) continue;
        const RowSrc<C> row{tab.tab + ((size_t)j * GTable<WG>::per_window + (size_t)((d < 0 ? -d : d) - 1)) * 16, 1, (d < 0) != flip, false};
        if (placed == 1) jac_mmadd_slots<C>(S, row);
        else jac_madd_slots<C>(S, row);  // places the row while the accumulator is at infinity
        if (placed < 2) ++placed;
    }
}

// x(k G) as a fraction X / ZZ (what a signature needs of the nonce point): the walk of
// fixed_base_add_slots from infinity on (X, Y, ZZ, ZZZ).  ZZ == 0 for k == 0 (mod n) only.
template <class C, int WG>
GECC_HD void fixed_base_x_slots(const fe& k_raw, const GTable<WG>& tab, const PointSlots S, fe* X, fe* ZZ) {
    bool flip;
    const fe k = scalar_fold_half<typename C::Fn>(scalar_reduce_once<typename C::Fn>(k_raw), &flip);
    const Recoded<WG> rc = recode_signed<WG>(k);
    auto digit = [&](int j) { return j == 256 / WG ? (int)rc.carry : recoded_digit<WG>(rc, j); };
    S.st(PointSlots::SZ, fe_zero());
    int placed = 0;
#pragma unroll 1
    for (int j = 0; j <= 256 / WG; ++j) {
        if (j < 256 / WG) {
            const int dn = digit(j + 1);
            if (dn != 0) tab.prefetch(j + 1, dn < 0 ? -dn : dn);
        }
        const int d = digit(j);
        if (d == 0) continue;
        const RowSrc<C> row{tab.tab + ((size_t)j * GTable<WG>::per_window + (size_t)((d < 0 ? -d : d) - 1)) * 16, 1, (d < 0) != flip, false};
        if (placed == 1) zz_mmadd_slots<C>(S, row);
        else zz_madd_slots<C>(S, row);
        if (placed < 2) ++placed;
    }
    *X = S.ld(PointSlots::SX);
    *ZZ = S.ld(PointSlots::SZ);
}

template <class C, int WG, bool UNIFORM>
GECC_HD jac fixed_base_mul_mode(const fe& k, const GTable<WG>& tab, const PointSlots* slots = nullptr) {
    if constexpr (UNIFORM) return fixed_base_mul_uniform<C, WG>(k, tab);
    else {
        if (slots) {  // accumulator at rest in shared memory (see PointSlots)
            slots->store_point(jac_infinity<C>());
            fixed_base_add_slots<C, WG>(k, tab, *slots, true);
            return slots->load_point();
        }
        return fixed_base_mul<C, WG>(k, tab);
    }
}
template <class C, bool UNIFORM>
GECC_HD jac var_base_mul_mode(const fe& k, const LaneTable& tab, const PointSlots* slots = nullptr) {
    if constexpr (UNIFORM) return var_base_mul_uniform<C>(k, tab);
    else {
        if (slots) {
            var_base_mul_slots<C>(k, tab, *slots);
            return slots->load_point();
        }
        return var_base_mul<C>(k, tab);
    }
}
#if defined(__CUDACC__)
// this thread's slots in a static shared array of the calling kernel (1-D blocks of THREADS)
template <int THREADS>
__device__ __forceinline__ PointSlots block_point_slots() {
    __shared__ uint4 mem[2 * PointSlots::COUNT * THREADS];
    return PointSlots{(uint32_t)__cvta_generic_to_shared(mem + threadIdx.x), 16u * THREADS};
}
#endif

// ------------------------------------------------------------ point codec
// 65-byte record 0x04 || X || Y -> affine Montgomery point; false when the tag,
// range or curve check fails (decode_point, curve.cpp:203-217).
template <class C>
GECC_HD bool decode_point(const uint8_t* rec, aff* out) {
    const typename C::Fp f{};
    if (rec[0] != 0x04) return false;
    fe x = be32_load(rec + 1), y = be32_load(rec + 33);
    if (!fe_lt_modulus(f, x) || !fe_lt_modulus(f, y)) return false;
    out->x = fe_to_mont(f, x);
    out->y = fe_to_mont(f, y);
    return aff_on_curve<C>(*out);
}
template <class C>
GECC_HD void encode_point(uint8_t* rec, const aff& p) {  // curve.cpp:192-201
    const typename C::Fp f{};
    rec[0] = 0x04;
    be32_store(rec + 1, fe_from_mont(f, p.x));
    be32_store(rec + 33, fe_from_mont(f, p.y));
}

// ------------------------------------------------------------ ECDSA lanes
enum { LANE_OK = 0, LANE_NONCE_EXHAUSTED = 5 };  // sm2b_status values

// One lane of ecdsa_sign_batch: e already reduced mod n, 0 < d < n.
// Writes r || s (64 bytes) or zeros; returns the lane status.
// One signing attempt with the nonce k (0 < k < n), e_m and d_m in Montgomery form mod n
// (the body of the retry loop, protocol.cpp:133-160).  False when r == 0 or s == 0.
template <class C, int WG, bool UNIFORM = false>
GECC_HD bool sign_attempt(const fe& e_m, const fe& d_m, const fe& k, const GTable<WG>& gt, uint8_t* sig64,
                          bool aligned = false, const PointSlots* slots = nullptr) {
    const typename C::Fp fp{};
    const typename C::Fn fn{};
    jac R = fixed_base_mul_mode<C, WG, UNIFORM>(k, gt, slots);
    if (jac_is_inf<C>(R)) return false;                   // cannot happen for 0 < k < n
    fe zinv = fe_inv(fp, R.Z);
    fe x = fe_from_mont(fp, fe_mul(fp, R.X, fe_sqr(fp, zinv)));
    fe r = scalar_reduce_once<typename C::Fn>(x);         // coord_mod_n, protocol.cpp:37-39
    if (fe_is_zero(r)) return false;
    fe kinv_m = fe_to_mont(fn, safegcd_inverse(fn, k));
    fe r_m = fe_to_mont(fn, r);
    fe s_m = fe_mul(fn, kinv_m, fe_add(fn, e_m, fe_mul(fn, r_m, d_m)));
    fe s = fe_from_mont(fn, s_m);
    if (fe_is_zero(s)) return false;
    be32_store_a(sig64, r, aligned);
    be32_store_a(sig64 + 32, s, aligned);
    return true;
}

template <class C, int WG, bool UNIFORM = false>
GECC_HD int sign_lane(const fe& e, const fe& d, uint64_t seed, uint64_t stream,
                      const GTable<WG>& gt, uint8_t* sig64, uint32_t first_attempt = 0, const PointSlots* slots = nullptr) {
    const typename C::Fn fn{};
    fe e_m = fe_to_mont(fn, e);
    fe d_m = fe_to_mont(fn, d);
#pragma unroll 1
    for (uint32_t attempt = first_attempt; attempt < 8; ++attempt) {  // protocol.cpp:121
        fe k = nonce_scalar<typename C::Fn>(seed, stream, attempt);
        if (sign_attempt<C, WG, UNIFORM>(e_m, d_m, k, gt, sig64, false, slots)) return LANE_OK;
    }
    for (int i = 0; i < 64; ++i) sig64[i] = 0;
    return LANE_NONCE_EXHAUSTED;
}

// One attempt with a caller-supplied nonce (gecc_sign_nonces): LANE_OK, or LANE_NONCE_EXHAUSTED
// when the nonce has to be replaced (outside (0, n), r == 0 or s == 0).
template <class C, int WG, bool UNIFORM = false>
GECC_HD int sign_lane_nonce(const fe& e, const fe& d, const fe& k, const GTable<WG>& gt, uint8_t* sig64,
                            const PointSlots* slots = nullptr) {
    const typename C::Fn fn{};
    if (scalar_in_range<typename C::Fn>(k) &&
        sign_attempt<C, WG, UNIFORM>(fe_to_mont(fn, e), fe_to_mont(fn, d), k, gt, sig64, false, slots))
        return LANE_OK;
    for (int i = 0; i < 64; ++i) sig64[i] = 0;
    return LANE_NONCE_EXHAUSTED;
}

// K lanes signed by one thread: the K nonce points are computed first, then ONE inversion
// mod p (for the K Jacobian Z's) and ONE inversion mod n (for the K nonces) are shared by
// Montgomery's trick -- the same idea the reference applies across a whole batch
// (protocol.cpp:133-136 + batch_invert), applied here inside a thread so that no
// cross-thread traffic is needed.  A lane that has to retry (r == 0 or s == 0, probability
// ~2^-255 unless forced) falls back to sign_lane from attempt 1, which reproduces the
// reference's per-lane retry sequence exactly.
// the state of a group between its two phases: nonce-point fractions, nonces, prefix products
template <int K>
struct SignGroup {
    fe X[K], Z[K], km[K], pz[K], pk[K];
};
// phase 1: the K nonce points and the running products of their denominators and of the nonces
template <class C, int WG, int K, bool UNIFORM = false>
GECC_HD void sign_lanes_walk(uint64_t seed, uint64_t stream0, const GTable<WG>& gt, const PointSlots* slots,
                             SignGroup<K>& g) {
    const typename C::Fp fp{};
    const typename C::Fn fn{};
    const bool zz_walk = !UNIFORM && slots != nullptr;
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
        fe k = nonce_scalar<typename C::Fn>(seed, stream0 + j, 0);
        if (zz_walk) {  // only x = X / ZZ is needed: the walk on (X, Y, ZZ, ZZZ), Z[j] holds ZZ
            fixed_base_x_slots<C, WG>(k, gt, *slots, &g.X[j], &g.Z[j]);
        } else {
            jac R = fixed_base_mul_mode<C, WG, UNIFORM>(k, gt, slots);
            g.X[j] = R.X;
            g.Z[j] = R.Z;  // never zero for 0 < k < n
        }
        // the nonces stay PLAIN in the Montgomery products mod n: p_j = k_0 ... k_j / R^j, so the
        // inverse of the last one, brought to Montgomery form, is I_j = R^(j+1) / (k_0 ... k_j) for
        // j = K - 1, and the unwinding yields k_j^-1 R (Montgomery form) from I_j p_(j-1) / R
        // and I_(j-1) from I_j k_j / R -- no conversion of the nonces
        g.km[j] = k;
        g.pz[j] = j ? fe_mul(fp, g.pz[j - 1], g.Z[j]) : g.Z[j];
        g.pk[j] = j ? fe_mul(fn, g.pk[j - 1], g.km[j]) : g.km[j];
    }
}
// phase 2: iz = pz[K-1]^-1 (representation of the field), ik = R / pk[K-1] mod n (the plain inverse
// of the residue pk[K-1], in Montgomery form); unwinds both and writes the signatures
template <class C, int WG, int K, bool UNIFORM = false>
GECC_HD void sign_lanes_finish(const fe* e, const fe* d, uint64_t seed, uint64_t stream0, const GTable<WG>& gt,
                               uint8_t* sig64, int* status, bool aligned, const PointSlots* slots,
                               const SignGroup<K>& g, fe iz, fe ik) {
    const typename C::Fp fp{};
    const typename C::Fn fn{};
    const bool zz_walk = !UNIFORM && slots != nullptr;
#pragma unroll 1
    for (int j = K - 1; j >= 0; --j) {
        fe zinv = j ? fe_mul(fp, iz, g.pz[j - 1]) : iz;
        fe kinv_m = j ? fe_mul(fn, ik, g.pk[j - 1]) : ik;
        if (j) {
            iz = fe_mul(fp, iz, g.Z[j]);
            ik = fe_mul(fn, ik, g.km[j]);
        }
        uint8_t* out = sig64 + 64 * j;
        fe x = fe_from_mont(fp, fe_mul(fp, g.X[j], zz_walk ? zinv : fe_sqr(fp, zinv)));
        fe r = scalar_reduce_once<typename C::Fn>(x);
        fe s = fe_zero();
        if (!fe_is_zero(r)) {  // s = k^-1 (e + r d): (r)(d R) / R is r d plain, (k^-1 R)(e + r d) / R is s plain
            s = fe_mul(fn, kinv_m, fe_add(fn, e[j], fe_mul(fn, r, fe_to_mont(fn, d[j]))));
        }
        if (fe_is_zero(r) || fe_is_zero(s)) {  // retry with fresh nonces (protocol.cpp:142-160)
            status[j] = sign_lane<C, WG, UNIFORM>(e[j], d[j], seed, stream0 + j, gt, out, 1, slots);
            continue;
        }
        be32_store_a(out, r, aligned);
        be32_store_a(out + 32, s, aligned);
        status[j] = LANE_OK;
    }
}
template <class C, int WG, int K, bool UNIFORM = false>
GECC_HD void sign_lanes(const fe* e, const fe* d, uint64_t seed, uint64_t stream0,
                        const GTable<WG>& gt, uint8_t* sig64, int* status, bool aligned = false,
                        const PointSlots* slots = nullptr) {
    const typename C::Fp fp{};
    const typename C::Fn fn{};
    SignGroup<K> g;
    sign_lanes_walk<C, WG, K, UNIFORM>(seed, stream0, gt, slots, g);
    const fe iz = fe_inv(fp, g.pz[K - 1]);                                   // (Z_0 ... Z_{K-1})^-1
    const fe ik = fe_to_mont(fn, safegcd_inverse(fn, g.pk[K - 1]));
    sign_lanes_finish<C, WG, K, UNIFORM>(e, d, seed, stream0, gt, sig64, status, aligned, slots, g, iz, ik);
}

// One lane of sm2b_verify: raw records in, 0/1 out.
template <class C, int WG>
GECC_HD uint8_t verify_lane(const uint8_t* digest32, const uint8_t* pub65, const uint8_t* sig64,
                            const GTable<WG>& gt, const LaneTable& qt, const PointSlots* slots = nullptr) {
    const typename C::Fp fp{};
    const typename C::Fn fn{};
    fe r = be32_load(sig64), s = be32_load(sig64 + 32);
    if (!scalar_in_range<typename C::Fn>(r) || !scalar_in_range<typename C::Fn>(s)) return 0;
    aff Q;
    if (!decode_point<C>(pub65, &Q)) return 0;
    fe e = scalar_reduce_once<typename C::Fn>(be32_load(digest32));   // capi.cpp:81-88
    fe w_m = fe_to_mont(fn, safegcd_inverse(fn, s));                   // s^-1 (Montgomery form)
    fe u1 = fe_mul(fn, e, w_m);                                        // e * w, plain
    fe u2 = fe_mul(fn, r, w_m);
    jac R;
    if (slots) {  // the ladder with its accumulator at rest in shared memory
        var_base_mul_point_slots<C>(u2, Q, qt, *slots);
        fixed_base_add_slots<C, WG>(u1, gt, *slots);
        R = slots->load_point();
    } else {
        build_lane_table<C>(Q, qt);
        jac B = var_base_mul<C>(u2, qt);
        R = fixed_base_mul<C, WG>(u1, gt, &B);   // u2 Q + u1 G: mixed additions are complete
    }
    if (jac_is_inf<C>(R)) return 0;
    // x(R) mod n == r  <=>  X == r Z^2  or  (r + n < p and X == (r + n) Z^2)
    fe zz = fe_sqr(fp, R.Z);
    if (fe_eq(fp, R.X, fe_mul(fp, fe_to_mont(fp, r), zz))) return 1;
    uint32_t carry;
    fe rn = u256_add(r, fe_modulus(fn), &carry);
    if (carry == 0 && fe_lt_modulus(fp, rn) && fe_eq(fp, R.X, fe_mul(fp, fe_to_mont(fp, rn), zz)))
        return 1;
    return 0;
}

}  // namespace gecc
