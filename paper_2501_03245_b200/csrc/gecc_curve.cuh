// Short-Weierstrass point arithmetic y^2 = x^3 + a x + b over a 256-bit prime
// field, one point per thread, coordinates in Montgomery form.
//
// The reference keeps points affine and shares one inversion per batch step
// (batch_point.cpp); its serial ground truth is Jacobian (curve.cpp:109-185).
// The GPU ladders here are per-thread Jacobian with complete case handling, so
// every output *value* equals the reference's (points are unique; only the
// representation inside a kernel differs).  Affine conversion happens once at
// kernel exit.
//
//   jac_dbl   : a = 0    -> 2M + 5S ("dbl-2009-l")
//               a = -3   -> 4M + 4S ("dbl-2001-b" with Z3 = 2 Y Z)
//               generic  -> the reference's own formula, curve.cpp:109-127
//   jac_madd  : Jacobian + affine, 8M + 3S, the reference's mixed path
//               (curve.cpp:136-141,152-166), complete
//   jac_add   : Jacobian + Jacobian, 12M + 4S (curve.cpp:142-166), complete
#pragma once
#include "gecc_field.cuh"

namespace gecc {

template <int N>
struct jacN {
    feN<N> X, Y, Z;  // Z == 0 <=> point at infinity
};
template <int N>
struct affN {
    feN<N> x, y;
};
using jac = jacN<8>;
using aff = affN<8>;
template <class C>
using cfe = feN<C::Fp::N>;   // coordinate type of curve C
template <class C>
using cjac = jacN<C::Fp::N>;
template <class C>
using caff = affN<C::Fp::N>;

template <class C>
GECC_HD cjac<C> jac_infinity() {
    cjac<C> r;
    r.X = fe_one(typename C::Fp{});
    r.Y = r.X;
    r.Z = fe_zero_n<C::Fp::N>();
    return r;
}
// Z == 0 (mod q).  Infinity is always *written* as the exact zero, but a weakly reduced
// field may also hold q itself, so the test is the field's own.
template <class C>
GECC_HD bool jac_is_inf(const cjac<C>& p) {
    return fe_is_zero(typename C::Fp{}, p.Z);
}

template <class C>
GECC_HD cfe<C> curve_a() {
    cfe<C> r;
#pragma unroll
    for (int i = 0; i < C::Fp::N; ++i) r.w[i] = C::a(i);
    return r;
}
template <class C>
GECC_HD cfe<C> curve_b() {
    cfe<C> r;
#pragma unroll
    for (int i = 0; i < C::Fp::N; ++i) r.w[i] = C::b(i);
    return r;
}
template <class C>
GECC_HD caff<C> curve_g() {
    caff<C> g;
#pragma unroll
    for (int i = 0; i < C::Fp::N; ++i) {
        g.x.w[i] = C::gx(i);
        g.y.w[i] = C::gy(i);
    }
    return g;
}

// y^2 == x^3 + a x + b (curve.cpp:62-70)
template <class C>
GECC_HD bool aff_on_curve(const caff<C>& p) {
    using fe = cfe<C>;
    const typename C::Fp f{};
    fe lhs = fe_sqr(f, p.y);
    fe rhs = fe_mul(f, fe_sqr(f, p.x), p.x);
    if (C::a_kind == A_MINUS3) {
        fe x3 = fe_add(f, fe_dbl(f, p.x), p.x);
        rhs = fe_sub(f, rhs, x3);
    } else if (C::a_kind != A_ZERO) {
        rhs = fe_add(f, rhs, fe_mul(f, curve_a<C>(), p.x));
    }
    rhs = fe_add(f, rhs, curve_b<C>());
    return fe_eq(f, lhs, rhs);
}

template <class C>
GECC_HD_CALL cjac<C> jac_dbl(const cjac<C>& p) {
    using fe = cfe<C>;
    const typename C::Fp f{};
    cjac<C> r;
    if (C::a_kind == A_ZERO) {
        fe A = fe_sqr(f, p.X);
        fe B = fe_sqr(f, p.Y);
        fe Cc = fe_sqr(f, B);
        fe t = fe_add(f, p.X, B);
        fe D = fe_sub(f, fe_sub(f, fe_sqr(f, t), A), Cc);
        D = fe_dbl(f, D);                       // 2((X+B)^2 - A - C)
        fe E = fe_add(f, fe_dbl(f, A), A);      // 3A
        fe F = fe_sqr(f, E);
        r.X = fe_sub(f, F, fe_dbl(f, D));
        fe C8 = fe_mul8(f, Cc);
        r.Y = fe_sub(f, fe_mul(f, E, fe_sub(f, D, r.X)), C8);
        r.Z = fe_dbl(f, fe_mul(f, p.Y, p.Z));
    } else if (C::a_kind == A_MINUS3) {
        fe delta = fe_sqr(f, p.Z);
        fe gamma = fe_sqr(f, p.Y);
        fe beta = fe_mul(f, p.X, gamma);
        fe t = fe_mul(f, fe_sub(f, p.X, delta), fe_add(f, p.X, delta));
        fe alpha = fe_add(f, fe_dbl(f, t), t);
        fe beta4 = fe_dbl(f, fe_dbl(f, beta));
        r.X = fe_sub(f, fe_sqr(f, alpha), fe_dbl(f, beta4));
        r.Z = fe_dbl(f, fe_mul(f, p.Y, p.Z));  // 2 Y Z: fewer instructions than (Y + Z)^2 - gamma - delta here
        fe g2 = fe_sqr(f, gamma);
        fe g8 = fe_mul8(f, g2);
        r.Y = fe_sub(f, fe_mul(f, alpha, fe_sub(f, beta4, r.X)), g8);
    } else {
        fe yy = fe_sqr(f, p.Y);
        fe yy2 = fe_dbl(f, yy);
        fe s4 = fe_dbl(f, fe_mul(f, p.X, yy2));
        fe c8 = fe_dbl(f, fe_sqr(f, yy2));
        fe xx = fe_sqr(f, p.X);
        fe zz2 = fe_sqr(f, fe_sqr(f, p.Z));
        fe m = fe_add(f, fe_add(f, fe_dbl(f, xx), xx), fe_mul(f, curve_a<C>(), zz2));
        r.X = fe_sub(f, fe_sub(f, fe_sqr(f, m), s4), s4);
        r.Y = fe_sub(f, fe_mul(f, m, fe_sub(f, s4, r.X)), c8);
        r.Z = fe_dbl(f, fe_mul(f, p.Y, p.Z));
    }
    // infinity (Z = 0) stays infinity: Z3 = 2 Y Z = 0.  Y = 0 (a 2-torsion point)
    // also gives Z3 = 0, matching curve.cpp:110-112.
    return r;
}

// The same doubling with the products inlined: for the few places where ONE warp runs a long chain
// of dependent doublings (window combine of the MSM) -- there the cost is latency, and the
// independent products of one doubling interleave once they are visible to the scheduler.
template <class C>
GECC_HD cjac<C> jac_dbl_flat(const cjac<C>& p) {
    using fe = cfe<C>;
    const typename C::Fp f{};
    cjac<C> r;
    if (C::a_kind == A_ZERO) {
        fe A = fe_sqr_inl(f, p.X);
        fe B = fe_sqr_inl(f, p.Y);
        fe Cc = fe_sqr_inl(f, B);
        fe t = fe_add(f, p.X, B);
        fe D = fe_sub(f, fe_sub(f, fe_sqr_inl(f, t), A), Cc);
        D = fe_dbl(f, D);                       // 2((X+B)^2 - A - C)
        fe E = fe_add(f, fe_dbl(f, A), A);      // 3A
        fe F = fe_sqr_inl(f, E);
        r.X = fe_sub(f, F, fe_dbl(f, D));
        fe C8 = fe_mul8(f, Cc);
        r.Y = fe_sub(f, fe_mul_inl(f, E, fe_sub(f, D, r.X)), C8);
        r.Z = fe_dbl(f, fe_mul_inl(f, p.Y, p.Z));
    } else if (C::a_kind == A_MINUS3) {
        fe delta = fe_sqr_inl(f, p.Z);
        fe gamma = fe_sqr_inl(f, p.Y);
        fe beta = fe_mul_inl(f, p.X, gamma);
        fe t = fe_mul_inl(f, fe_sub(f, p.X, delta), fe_add(f, p.X, delta));
        fe alpha = fe_add(f, fe_dbl(f, t), t);
        fe beta4 = fe_dbl(f, fe_dbl(f, beta));
        r.X = fe_sub(f, fe_sqr_inl(f, alpha), fe_dbl(f, beta4));
        fe yz = fe_add(f, p.Y, p.Z);
        r.Z = fe_sub(f, fe_sub(f, fe_sqr_inl(f, yz), gamma), delta);
        fe g2 = fe_sqr_inl(f, gamma);
        fe g8 = fe_mul8(f, g2);
        r.Y = fe_sub(f, fe_mul_inl(f, alpha, fe_sub(f, beta4, r.X)), g8);
    } else {
        fe yy = fe_sqr_inl(f, p.Y);
        fe yy2 = fe_dbl(f, yy);
        fe s4 = fe_dbl(f, fe_mul_inl(f, p.X, yy2));
        fe c8 = fe_dbl(f, fe_sqr_inl(f, yy2));
        fe xx = fe_sqr_inl(f, p.X);
        fe zz2 = fe_sqr_inl(f, fe_sqr_inl(f, p.Z));
        fe m = fe_add(f, fe_add(f, fe_dbl(f, xx), xx), fe_mul_inl(f, curve_a<C>(), zz2));
        r.X = fe_sub(f, fe_sub(f, fe_sqr_inl(f, m), s4), s4);
        r.Y = fe_sub(f, fe_mul_inl(f, m, fe_sub(f, s4, r.X)), c8);
        r.Z = fe_dbl(f, fe_mul_inl(f, p.Y, p.Z));
    }
    // infinity (Z = 0) stays infinity: Z3 = 2 Y Z = 0.  Y = 0 (a 2-torsion point)
    // also gives Z3 = 0, matching curve.cpp:110-112.
    return r;
}

// p + (x2, y2), (x2, y2) finite.  Handles p = infinity, p = q (doubling) and
// p = -q (infinity) -- curve.cpp:129-167 with t.Z == 1.
template <class C>
GECC_HD_CALL cjac<C> jac_madd(const cjac<C>& p, const caff<C>& q) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    const typename C::Fp f{};
    if (jac_is_inf<C>(p)) {
        jac r;
        r.X = q.x;
        r.Y = q.y;
        r.Z = fe_one(f);
        return r;
    }
    fe z1z1 = fe_sqr(f, p.Z);
    fe u2 = fe_mul(f, q.x, z1z1);
    fe s2 = fe_mul(f, q.y, fe_mul(f, z1z1, p.Z));
    fe h = fe_sub(f, u2, p.X);
    fe rr = fe_sub(f, s2, p.Y);
    if (fe_is_zero(f, h)) {
        if (fe_is_zero(f, rr)) return jac_dbl<C>(p);
        return jac_infinity<C>();
    }
    fe hh = fe_sqr(f, h);
    fe hhh = fe_mul(f, hh, h);
    fe v = fe_mul(f, p.X, hh);
    jac r;
    r.X = fe_sub(f, fe_sub(f, fe_sub(f, fe_sqr(f, rr), hhh), v), v);
    r.Y = fe_sub(f, fe_mul(f, rr, fe_sub(f, v, r.X)), fe_mul(f, p.Y, hhh));
    r.Z = fe_mul(f, p.Z, h);
    return r;
}

// complete Jacobian + Jacobian (curve.cpp:142-166)
template <class C>
GECC_HD_CALL cjac<C> jac_add(const cjac<C>& p, const cjac<C>& q) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    const typename C::Fp f{};
    if (jac_is_inf<C>(p)) return q;
    if (jac_is_inf<C>(q)) return p;
    fe z1z1 = fe_sqr(f, p.Z);
    fe z2z2 = fe_sqr(f, q.Z);
    fe u1 = fe_mul(f, p.X, z2z2);
    fe u2 = fe_mul(f, q.X, z1z1);
    fe s1 = fe_mul(f, p.Y, fe_mul(f, z2z2, q.Z));
    fe s2 = fe_mul(f, q.Y, fe_mul(f, z1z1, p.Z));
    fe h = fe_sub(f, u2, u1);
    fe rr = fe_sub(f, s2, s1);
    if (fe_is_zero(f, h)) {
        if (fe_is_zero(f, rr)) return jac_dbl<C>(p);
        return jac_infinity<C>();
    }
    fe hh = fe_sqr(f, h);
    fe hhh = fe_mul(f, hh, h);
    fe v = fe_mul(f, u1, hh);
    jac r;
    r.X = fe_sub(f, fe_sub(f, fe_sub(f, fe_sqr(f, rr), hhh), v), v);
    r.Y = fe_sub(f, fe_mul(f, rr, fe_sub(f, v, r.X)), fe_mul(f, s1, hhh));
    r.Z = fe_mul(f, fe_mul(f, p.Z, q.Z), h);
    return r;
}

// (X/Z^2, Y/Z^3) given zinv = Z^-1 (curve.cpp:169-174)
template <class C>
GECC_HD caff<C> jac_to_aff_with(const cjac<C>& p, const cfe<C>& zinv) {
    using fe = cfe<C>;
    using aff = caff<C>;
    const typename C::Fp f{};
    fe zi2 = fe_sqr(f, zinv);
    aff r;
    r.x = fe_mul(f, p.X, zi2);
    r.y = fe_mul(f, p.Y, fe_mul(f, zi2, zinv));
    return r;
}

template <class C>
GECC_HD caff<C> aff_neg(const caff<C>& p) {
    caff<C> r;
    r.x = p.x;
    r.y = fe_neg(typename C::Fp{}, p.y);
    return r;
}

}  // namespace gecc
