// 256-bit Montgomery field arithmetic, one element per thread, 8 x 32-bit limbs in
// registers, built on the carry-chain primitives of gecc_prims.cuh.
//
// Semantics follow the reference's field layer (proj/src/field.cpp):
//   fe_mul   == mont_mul  (field.cpp:205-211): a*b*2^-256 mod q, canonical (< q)
//   fe_add   == mod_add   (field.cpp:24-29,213-219)
//   fe_sub   == mod_sub   (field.cpp:31-35,221-227)
//   fe_to_mont / fe_from_mont (field.cpp:194-203)
//   fe_inv   == mod_inv_fermat's *value* (field.cpp:239-246); computed differently
//               (windowed Fermat or safegcd) -- the residue is unique.
// All outputs are canonical, so results are bit-identical to the reference no
// matter which reduction route computes them (the reference itself checks its
// two routes against each other, tests/test_field.cpp:166-169).
//
// A field is a type F with accessors q(i), r(i), r2(i), ninv(i), qm2(i), qinv32 and
// a `kind`.  Compile-time fields (gecc_consts.cuh) fold to immediates after
// unrolling; FieldRT carries runtime constants for arbitrary odd 256-bit moduli
// (the reference's FieldParams::make(q), field.cpp:159-179).
#pragma once
#include <type_traits>

#include "gecc_consts.cuh"

namespace gecc {

// N x 32-bit limbs, least significant first.  fe (8 limbs) is the 256-bit element every
// reference-facing kernel uses; 12 limbs carry the 381-bit base field of BLS12-381.
template <int N>
struct feN {
    uint32_t w[N];
};
using fe = feN<8>;
template <class F>
using fel = feN<F::N>;  // element type of field F

struct FieldRT {
    static constexpr int N = 8;
    static constexpr int kind = KIND_GENERIC;
    uint32_t q_[8], r_[8], r2_[8], ninv_[8], qm2_[8], r3_[8], q30_[9];
    uint32_t qinv32, qinv30_;
    GECC_HD uint32_t q(int i) const { return q_[i]; }
    GECC_HD uint32_t r(int i) const { return r_[i]; }
    GECC_HD uint32_t r2(int i) const { return r2_[i]; }
    GECC_HD uint32_t ninv(int i) const { return ninv_[i]; }
    GECC_HD uint32_t qm2(int i) const { return qm2_[i]; }
    GECC_HD uint32_t r3(int i) const { return r3_[i]; }
    GECC_HD uint32_t q30(int i) const { return q30_[i]; }
    GECC_HD uint32_t qinv30() const { return qinv30_; }
};

// ---------------------------------------------------------------- basics
template <int N>
GECC_HD feN<N> fe_zero_n() {
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = 0;
    return r;
}
GECC_HD fe fe_zero() { return fe_zero_n<8>(); }
template <class F>
GECC_HD fel<F> fe_one(const F& f) {  // Montgomery one = R mod q
    fel<F> r;
#pragma unroll
    for (int i = 0; i < F::N; ++i) r.w[i] = f.r(i);
    return r;
}
template <class F>
GECC_HD fel<F> fe_modulus(const F& f) {
    fel<F> r;
#pragma unroll
    for (int i = 0; i < F::N; ++i) r.w[i] = f.q(i);
    return r;
}
template <int N>
GECC_HD bool fe_is_zero(const feN<N>& a) {
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) acc |= a.w[i];
    return acc == 0;
}
template <int N>
GECC_HD bool fe_eq(const feN<N>& a, const feN<N>& b) {
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) acc |= a.w[i] ^ b.w[i];
    return acc == 0;
}
template <int N>
GECC_HD feN<N> fe_select(bool c, const feN<N>& a, const feN<N>& b) {  // c ? a : b
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = c ? a.w[i] : b.w[i];
    return r;
}
// a < b as unsigned integers (limbs.hpp:115-122)
template <int N>
GECC_HD bool u256_lt(const feN<N>& a, const feN<N>& b) {
    sub_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < N; ++i) subc_cc(a.w[i], b.w[i]);
    return subc(0, 0) != 0;
}
template <class F>
GECC_HD bool fe_lt_modulus(const F& f, const fel<F>& a) {
    return u256_lt(a, fe_modulus(f));
}

// ---------------------------------------------------------------- lazy secp256k1 field
// KIND_SECP_LAZY: elements are plain residues (no Montgomery factor) that are only
// WEAKLY reduced -- any 256-bit value, congruent mod q = 2^256 - c, c = 2^32 + 977.
// 2^256 == c (mod q), so an overflow of 2^256 is folded back by adding c and a borrow by
// subtracting c; there is no compare-and-select.  Canonical form is produced only where a
// value leaves the field layer (bytes, equality with a canonical constant, inversion).
template <class F>
GECC_HD fe lazy_canon(const F&, const fe& a) {  // a -> a mod q in [0, q)
    fe s;
    s.w[0] = add_cc(a.w[0], 977u);
    s.w[1] = addc_cc(a.w[1], 1u);
#pragma unroll
    for (int i = 2; i < 8; ++i) s.w[i] = addc_cc(a.w[i], 0);
    const uint32_t over = addc(0, 0);  // a + c >= 2^256  <=>  a >= q
    return fe_select(over != 0, s, a);
}
// a == 0 (mod q) for a weakly reduced a: a is 0 or q
template <class F>
GECC_HD bool lazy_is_zero(const F& f, const fe& a) {
    uint32_t z = 0, e = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        z |= a.w[i];
        e |= a.w[i] ^ f.q(i);
    }
    return z == 0 || e == 0;
}
// r = (carry : a) folded once more: a + carry * c (carry is 0 or 1).  Only the two low limbs
// change unless the addition carries out of limb 1 (probability ~2^-31): the ripple through
// limbs 2..7 and the (rarer still) second wrap sit behind a branch no warp normally takes.
GECC_HD fe lazy_fold_carry(const fe& a, uint32_t carry) {
    fe r = a;
    const uint32_t m = 0u - carry;
    r.w[0] = add_cc(a.w[0], m & 977u);
    r.w[1] = addc_cc(a.w[1], carry);
    if (addc(0, 0)) {
        r.w[2] = add_cc(a.w[2], 1u);
#pragma unroll
        for (int i = 3; i < 8; ++i) r.w[i] = addc_cc(a.w[i], 0);
        if (addc(0, 0)) {  // only when a >= 2^256 - c: the wrapped value is below c, adding c cannot wrap
            r.w[0] = add_cc(r.w[0], 977u);
            r.w[1] = addc_cc(r.w[1], 1u);
#pragma unroll
            for (int i = 2; i < 8; ++i) r.w[i] = addc_cc(r.w[i], 0);
        }
    }
    return r;
}
// (a << K) mod q for K = 1..3, weakly reduced: funnel shifts (no carry chain) and the K bits
// shifted out folded back as t * c, t < 8.
template <int K>
GECC_HD fe lazy_shl(const fe& a) {
    static_assert(K >= 1 && K <= 3, "small shifts only");
    const uint32_t t = a.w[7] >> (32 - K);
    fe r;
    r.w[0] = a.w[0] << K;
#pragma unroll
    for (int i = 1; i < 8; ++i) r.w[i] = (a.w[i] << K) | (a.w[i - 1] >> (32 - K));
    const uint32_t lo = r.w[0], hi = r.w[1];
    r.w[0] = add_cc(lo, t * 977u);
    r.w[1] = addc_cc(hi, t);
    if (addc(0, 0)) {  // carry out of limb 1: rare
        r.w[2] = add_cc(r.w[2], 1u);
#pragma unroll
        for (int i = 3; i < 8; ++i) r.w[i] = addc_cc(r.w[i], 0);
        if (addc(0, 0)) {  // wrapped past 2^256: what is left is below t * c, one more c cannot wrap
            r.w[0] = add_cc(r.w[0], 977u);
            r.w[1] = addc_cc(r.w[1], 1u);
#pragma unroll
            for (int i = 2; i < 8; ++i) r.w[i] = addc_cc(r.w[i], 0);
        }
    }
    return r;
}
GECC_HD fe lazy_add(const fe& a, const fe& b) {
    fe s;
    s.w[0] = add_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) s.w[i] = addc_cc(a.w[i], b.w[i]);
    return lazy_fold_carry(s, addc(0, 0));
}
GECC_HD fe lazy_sub(const fe& a, const fe& b) {
    fe d;
    d.w[0] = sub_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) d.w[i] = subc_cc(a.w[i], b.w[i]);
    const uint32_t k = subc(0, 0) & 1u;  // borrowed: d = a - b + 2^256 == a - b + c, so take c off
    fe r = d;
    r.w[0] = sub_cc(d.w[0], (0u - k) & 977u);
    r.w[1] = subc_cc(d.w[1], k);
    if (subc(0, 0)) {  // borrow out of limb 1 (probability ~2^-31): ripple, and the rarer second wrap
        r.w[2] = sub_cc(d.w[2], 1u);
#pragma unroll
        for (int i = 3; i < 8; ++i) r.w[i] = subc_cc(d.w[i], 0);
        if (subc(0, 0)) {  // only when d < c: wrapped once more, take c off again (cannot wrap a third time)
            r.w[0] = sub_cc(r.w[0], 977u);
            r.w[1] = subc_cc(r.w[1], 1u);
#pragma unroll
            for (int i = 2; i < 8; ++i) r.w[i] = subc_cc(r.w[i], 0);
        }
    }
    return r;
}
// 512-bit t -> weakly reduced 256-bit value == t (mod q):
//   v = t_lo + t_hi * 977 + (t_hi << 32)          (10 limbs, top part V < 2^33 + 2^10)
//   w = v_lo + V * 977 + (V << 32)                 (carry <= 1)
//   r = w + carry * c
// 8 wide multiplies + 2, everything else carry chains; no dependent multiplier sequence.
GECC_HD fe redc_secp_lazy(const uint32_t* t) {
    uint32_t s[10], o[8];
    // even limbs of t_hi: products sit on aligned pairs of s -> one chain of four IMAD.WIDE
    s[0] = mad_lo_cc(t[8], 977u, t[0]);
    s[1] = madc_hi_cc(t[8], 977u, t[1]);
#pragma unroll
    for (int i = 2; i < 8; i += 2) {
        s[i] = madc_lo_cc(t[8 + i], 977u, t[i]);
        s[i + 1] = madc_hi_cc(t[8 + i], 977u, t[i + 1]);
    }
    s[8] = addc(0, 0);
    // odd limbs: four independent wide products, one limb to the left
#pragma unroll
    for (int i = 1; i < 8; i += 2) {
        o[i - 1] = mul_lo(t[8 + i], 977u);
        o[i] = mul_hi(t[8 + i], 977u);
    }
    s[1] = add_cc(s[1], o[0]);
#pragma unroll
    for (int i = 1; i < 7; ++i) s[i + 1] = addc_cc(s[i + 1], o[i]);
    s[8] = addc(s[8], o[7]);  // <= 1 + 976 + 1: no carry out
    s[1] = add_cc(s[1], t[8]);
#pragma unroll
    for (int i = 1; i < 8; ++i) s[i + 1] = addc_cc(s[i + 1], t[8 + i]);
    s[9] = addc(0, 0);
    // fold V = s[9] : s[8]
    const uint32_t lo977 = mul_lo(s[8], 977u);
    const uint32_t hi977 = mul_hi(s[8], 977u) + s[9] * 977u;
    fe r;
    r.w[0] = add_cc(s[0], lo977);
    r.w[1] = addc_cc(s[1], hi977);
    r.w[2] = addc_cc(s[2], s[9]);
#pragma unroll
    for (int i = 3; i < 8; ++i) r.w[i] = addc_cc(s[i], 0);
    uint32_t carry = addc(0, 0);
    r.w[1] = add_cc(r.w[1], s[8]);
#pragma unroll
    for (int i = 2; i < 8; ++i) r.w[i] = addc_cc(r.w[i], 0);
    carry = addc(carry, 0);  // total carry is 0 or 1 (w < 2^256 + 2^67)
    // w >= 2^256 leaves a tiny remainder (below 2^67), so adding c touches limbs 0..2 only and
    // cannot wrap again
    r.w[0] = add_cc(r.w[0], (0u - carry) & 977u);
    r.w[1] = addc_cc(r.w[1], carry);
    r.w[2] = addc(r.w[2], 0);
    return r;
}

// ---------------------------------------------------------------- lazy SM2 field
// KIND_SM2_LAZY: the SM2 prime in MONTGOMERY form (R = 2^256: the constants and tables of Sm2P
// serve), elements only WEAKLY reduced -- any 256-bit value congruent to the element.  2^256 == c
// (mod q) with c = 2^256 - q = 2^224 + 2^96 - 2^64 + 1 = limbs {1, 0, 0xFFFFFFFF, 0, 0, 0, 0, 1}: a
// carry out of an addition is folded back by adding c under a mask and a borrow by subtracting it
// (one more 8-limb chain instead of a trial subtraction and a select), a second wrap (probability
// 2^-32) sits behind a branch.  The Montgomery reduction ends with the same fold instead of the
// conditional subtraction.  Canonical form only where a value leaves the field layer.
template <class F>
GECC_HD fe weak_canon(const F& f, const fe& a) {  // a in [0, 2^256) -> a mod q (q > 2^255: one subtraction)
    fe d;
    d.w[0] = sub_cc(a.w[0], f.q(0));
#pragma unroll
    for (int i = 1; i < 8; ++i) d.w[i] = subc_cc(a.w[i], f.q(i));
    const uint32_t borrow = subc(0, 0);
    return fe_select(borrow == 0, d, a);
}
GECC_HD fe sm2l_fold_carry(const fe& s, uint32_t k) {  // (k : s) -> s + k c, k = 0 or 1
    const uint32_t m = 0u - k;
    fe r;
    r.w[0] = add_cc(s.w[0], k);
    r.w[1] = addc_cc(s.w[1], 0);
    r.w[2] = addc_cc(s.w[2], m);
#pragma unroll
    for (int i = 3; i < 7; ++i) r.w[i] = addc_cc(s.w[i], 0);
    r.w[7] = addc_cc(s.w[7], k);
    if (addc(0, 0)) {  // s >= q and k: what is left is below c, one more c cannot wrap
        r.w[0] = add_cc(r.w[0], 1u);
        r.w[1] = addc_cc(r.w[1], 0);
        r.w[2] = addc_cc(r.w[2], 0xFFFFFFFFu);
#pragma unroll
        for (int i = 3; i < 7; ++i) r.w[i] = addc_cc(r.w[i], 0);
        r.w[7] = addc_cc(r.w[7], 1u);
    }
    return r;
}
GECC_HD fe sm2l_add(const fe& a, const fe& b) {
    fe s;
    s.w[0] = add_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) s.w[i] = addc_cc(a.w[i], b.w[i]);
    return sm2l_fold_carry(s, addc(0, 0));
}
GECC_HD fe sm2l_sub(const fe& a, const fe& b) {
    fe d;
    d.w[0] = sub_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) d.w[i] = subc_cc(a.w[i], b.w[i]);
    const uint32_t k = subc(0, 0) & 1u;  // borrowed: d = a - b + 2^256 == a - b + c, so take c off
    const uint32_t m = 0u - k;
    fe r;
    r.w[0] = sub_cc(d.w[0], k);
    r.w[1] = subc_cc(d.w[1], 0);
    r.w[2] = subc_cc(d.w[2], m);
#pragma unroll
    for (int i = 3; i < 7; ++i) r.w[i] = subc_cc(d.w[i], 0);
    r.w[7] = subc_cc(d.w[7], k);
    if (subc(0, 0)) {  // d < c and k: wrapped once more, take c off again (cannot wrap a third time)
        r.w[0] = sub_cc(r.w[0], 1u);
        r.w[1] = subc_cc(r.w[1], 0);
        r.w[2] = subc_cc(r.w[2], 0xFFFFFFFFu);
#pragma unroll
        for (int i = 3; i < 7; ++i) r.w[i] = subc_cc(r.w[i], 0);
        r.w[7] = subc_cc(r.w[7], 1u);
    }
    return r;
}
template <class F>
constexpr bool field_is_weak_v = F::kind == KIND_SECP_LAZY || F::kind == KIND_SM2_LAZY;

// field-aware predicates: canonical fields compare limbs, the lazy field compares mod q
template <class F>
GECC_HD bool fe_is_zero(const F& f, const fel<F>& a) {
    if constexpr (field_is_weak_v<F>) return lazy_is_zero(f, a);
    else return fe_is_zero(a);
}

// ---------------------------------------------------------------- add / sub
template <class F>
GECC_HD fel<F> fe_add(const F& f, const fel<F>& a, const fel<F>& b) {
    if constexpr (F::kind == KIND_SECP_LAZY) return lazy_add(a, b);
    if constexpr (F::kind == KIND_SM2_LAZY) return sm2l_add(a, b);
    constexpr int N = F::N;
    fel<F> s, d;
    s.w[0] = add_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < N; ++i) s.w[i] = addc_cc(a.w[i], b.w[i]);
    uint32_t top = addc(0, 0);
    d.w[0] = sub_cc(s.w[0], f.q(0));
#pragma unroll
    for (int i = 1; i < N; ++i) d.w[i] = subc_cc(s.w[i], f.q(i));
    uint32_t borrow = subc(0, 0);  // 0xFFFFFFFF when s < q
    // s >= q  <=>  carried out of 2^(32N), or no borrow
    return fe_select(top != 0 || borrow == 0, d, s);
}
template <class F>
GECC_HD fel<F> fe_sub(const F& f, const fel<F>& a, const fel<F>& b) {
    if constexpr (F::kind == KIND_SECP_LAZY) return lazy_sub(a, b);
    if constexpr (F::kind == KIND_SM2_LAZY) return sm2l_sub(a, b);
    constexpr int N = F::N;
    fel<F> d, e;
    d.w[0] = sub_cc(a.w[0], b.w[0]);
#pragma unroll
    for (int i = 1; i < N; ++i) d.w[i] = subc_cc(a.w[i], b.w[i]);
    uint32_t borrow = subc(0, 0);
    e.w[0] = add_cc(d.w[0], f.q(0));
#pragma unroll
    for (int i = 1; i < N; ++i) e.w[i] = addc_cc(d.w[i], f.q(i));
    return fe_select(borrow != 0, e, d);
}
template <class F>
GECC_HD bool fe_eq(const F& f, const fel<F>& a, const fel<F>& b) {
    if constexpr (F::kind == KIND_SECP_LAZY) return lazy_is_zero(f, lazy_sub(a, b));
    else if constexpr (F::kind == KIND_SM2_LAZY) return lazy_is_zero(f, sm2l_sub(a, b));
    else return fe_eq(a, b);
}
template <class F>
GECC_HD fel<F> fe_neg(const F& f, const fel<F>& a) {
    return fe_sub(f, fe_zero_n<F::N>(), a);
}
template <class F>
GECC_HD fel<F> fe_dbl(const F& f, const fel<F>& a) {
    if constexpr (F::kind == KIND_SECP_LAZY) return lazy_shl<1>(a);
    else return fe_add(f, a, a);
}
template <class F>
GECC_HD fel<F> fe_mul8(const F& f, const fel<F>& a) {  // 8 a
    if constexpr (F::kind == KIND_SECP_LAZY) return lazy_shl<3>(a);
    else return fe_dbl(f, fe_dbl(f, fe_dbl(f, a)));
}

// ---------------------------------------------------------------- products
// Full 16-limb product.  Products a[j]*b[i] whose position i+j is even are
// accumulated in e[], odd ones in o[] (o is one limb to the left), so that every
// lo/hi pair sits on an aligned register pair and each row is two carry chains of
// IMAD.WIDE.U32(.X).  64 wide multiply-adds + 8 carry folds + 15 merge adds.
// unmerged form: a*b = sum e[k] 2^(32k) + sum o[k] 2^(32(k+1))
template <int N>
GECC_HD void mul_wide_eo(uint32_t* e, uint32_t* o, const uint32_t* a, const uint32_t* b) {
    static_assert(N % 2 == 0, "even/odd layout needs an even limb count");
#pragma unroll
    for (int k = 0; k < 2 * N; ++k) e[k] = o[k] = 0;
    {   // row 0 meets only zeros: plain wide products, no carry chain
        const uint32_t b0 = b[0];
#pragma unroll
        for (int j = 0; j < N; j += 2) {
            const uint64_t pe = (uint64_t)a[j] * b0, po = (uint64_t)a[j + 1] * b0;
            e[j] = (uint32_t)pe;
            e[j + 1] = (uint32_t)(pe >> 32);
            o[j] = (uint32_t)po;
            o[j + 1] = (uint32_t)(po >> 32);
        }
    }
#pragma unroll
    for (int i = 1; i < N; ++i) {
        const uint32_t bi = b[i];
        if ((i & 1) == 0) {
            e[i] = mad_lo_cc(a[0], bi, e[i]);
            e[i + 1] = madc_hi_cc(a[0], bi, e[i + 1]);
#pragma unroll
            for (int j = 2; j < N; j += 2) {
                e[i + j] = madc_lo_cc(a[j], bi, e[i + j]);
                e[i + j + 1] = madc_hi_cc(a[j], bi, e[i + j + 1]);
            }
            e[i + N] = addc(e[i + N], 0);
            o[i] = mad_lo_cc(a[1], bi, o[i]);
            o[i + 1] = madc_hi_cc(a[1], bi, o[i + 1]);
#pragma unroll
            for (int j = 3; j < N; j += 2) {
                o[i + j - 1] = madc_lo_cc(a[j], bi, o[i + j - 1]);
                o[i + j] = madc_hi_cc(a[j], bi, o[i + j]);
            }
        } else {
            o[i - 1] = mad_lo_cc(a[0], bi, o[i - 1]);
            o[i] = madc_hi_cc(a[0], bi, o[i]);
#pragma unroll
            for (int j = 2; j < N; j += 2) {
                o[i + j - 1] = madc_lo_cc(a[j], bi, o[i + j - 1]);
                o[i + j] = madc_hi_cc(a[j], bi, o[i + j]);
            }
            o[i + N - 1] = addc(o[i + N - 1], 0);
            e[i + 1] = mad_lo_cc(a[1], bi, e[i + 1]);
            e[i + 2] = madc_hi_cc(a[1], bi, e[i + 2]);
#pragma unroll
            for (int j = 3; j < N; j += 2) {
                e[i + j] = madc_lo_cc(a[j], bi, e[i + j]);
                e[i + j + 1] = madc_hi_cc(a[j], bi, e[i + j + 1]);
            }
        }
    }
}
template <int N>
GECC_HD void mul_wide_n(uint32_t* t, const uint32_t* a, const uint32_t* b) {
    uint32_t e[2 * N], o[2 * N];
    mul_wide_eo<N>(e, o, a, b);
    t[0] = e[0];
    t[1] = add_cc(e[1], o[0]);
#pragma unroll
    for (int k = 2; k < 2 * N; ++k) t[k] = addc_cc(e[k], o[k - 1]);
}

GECC_HD void mul_wide8(uint32_t* t, const uint32_t* a, const uint32_t* b) { mul_wide_n<8>(t, a, b); }

// Low N limbs of a*b (used only by the generic REDC).
template <int N>
GECC_HD void mul_low_n(uint32_t* r, const uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int k = 0; k < N; ++k) r[k] = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const uint32_t bi = b[i];
        r[i] = mad_lo_cc(a[0], bi, r[i]);
#pragma unroll
        for (int j = 1; j < N - i; ++j) r[i + j] = madc_lo_cc(a[j], bi, r[i + j]);
        if (i < N - 1) {
            r[i + 1] = mad_hi_cc(a[0], bi, r[i + 1]);
#pragma unroll
            for (int j = 1; j < N - 1 - i; ++j) r[i + j + 1] = madc_hi_cc(a[j], bi, r[i + j + 1]);
        }
    }
}

GECC_HD void mul_low8(uint32_t* r, const uint32_t* a, const uint32_t* b) { mul_low_n<8>(r, a, b); }

// Full 2N-limb square: the N(N-1)/2 off-diagonal products once (same even/odd carry-chain
// layout as mul_wide8), doubled by a one-bit funnel shift, plus the 8 diagonal
// squares in one chain: 36 wide multiply-adds instead of 64.
template <int N>
GECC_HD void sqr_wide_n(uint32_t* t, const uint32_t* a) {
    uint32_t e[2 * N], o[2 * N];
#pragma unroll
    for (int k = 0; k < 2 * N; ++k) e[k] = o[k] = 0;
#pragma unroll
    for (int i = 0; i < N - 1; ++i) {
        const uint32_t ai = a[i];
        // s = i + j even: j = i+2, i+4, ...  -> e[s], e[s+1]
        if (i + 2 < N) {
            e[2 * i + 2] = mad_lo_cc(a[i + 2], ai, e[2 * i + 2]);
            e[2 * i + 3] = madc_hi_cc(a[i + 2], ai, e[2 * i + 3]);
#pragma unroll
            for (int j = i + 4; j < N; j += 2) {
                e[i + j] = madc_lo_cc(a[j], ai, e[i + j]);
                e[i + j + 1] = madc_hi_cc(a[j], ai, e[i + j + 1]);
            }
            // chain ended at index i + jl + 1 with jl the last j used; fold the carry
            const int jl = ((N - 1 - i) % 2 == 0) ? N - 1 : N - 2;  // last j with i + j even
            if (i + jl + 2 < 2 * N) e[i + jl + 2] = addc(e[i + jl + 2], 0);
        }
        // s = i + j odd: j = i+1, i+3, ...  -> o[s-1], o[s]
        o[2 * i] = mad_lo_cc(a[i + 1], ai, o[2 * i]);
        o[2 * i + 1] = madc_hi_cc(a[i + 1], ai, o[2 * i + 1]);
#pragma unroll
        for (int j = i + 3; j < N; j += 2) {
            o[i + j - 1] = madc_lo_cc(a[j], ai, o[i + j - 1]);
            o[i + j] = madc_hi_cc(a[j], ai, o[i + j]);
        }
        {
            const int jl = ((N - 1 - i) % 2 == 1) ? N - 1 : N - 2;  // last j with i + j odd
            if (i + jl + 1 < 2 * N) o[i + jl + 1] = addc(o[i + jl + 1], 0);
        }
    }
    // off-diagonal sum S = e + (o << 32)
    uint32_t sd[2 * N];
    sd[0] = e[0];
    sd[1] = add_cc(e[1], o[0]);
#pragma unroll
    for (int k = 2; k < 2 * N; ++k) sd[k] = addc_cc(e[k], o[k - 1]);
    // 2S, then + diagonal squares
    uint32_t dbl[2 * N];
    dbl[0] = sd[0] << 1;
#pragma unroll
    for (int k = 1; k < 2 * N; ++k) dbl[k] = (sd[k] << 1) | (sd[k - 1] >> 31);
    t[0] = mad_lo_cc(a[0], a[0], dbl[0]);
    t[1] = madc_hi_cc(a[0], a[0], dbl[1]);
#pragma unroll
    for (int i = 1; i < N; ++i) {
        t[2 * i] = madc_lo_cc(a[i], a[i], dbl[2 * i]);
        t[2 * i + 1] = madc_hi_cc(a[i], a[i], dbl[2 * i + 1]);
    }
}

GECC_HD void sqr_wide8(uint32_t* t, const uint32_t* a) { sqr_wide_n<8>(t, a); }

// ---------------------------------------------------------------- reductions
// r = (top:r) - q if (top:r) >= q
template <class F>
GECC_HD fel<F> final_sub(const F& f, const fel<F>& r, uint32_t top) {
    fel<F> d;
    d.w[0] = sub_cc(r.w[0], f.q(0));
#pragma unroll
    for (int i = 1; i < F::N; ++i) d.w[i] = subc_cc(r.w[i], f.q(i));
    uint32_t borrow = subc(0, 0);
    return fe_select(top != 0 || borrow == 0, d, r);
}

#if defined(__CUDACC__)
static __constant__ uint32_t gecc_opaque_zero_word = 0;
#endif
GECC_HD uint32_t opaque_zero() {
#if defined(__CUDA_ARCH__)
    return gecc_opaque_zero_word;
#else
    return 0;
#endif
}

// Word-serial Montgomery reduction for any odd q on the UNMERGED even/odd product (reference:
// reduce_generic_raw, field.cpp:50-78 -- the same word-by-word elimination and the same value).
// Step i takes the low word of what is left at position i, L = e[i] + o[i-1] + carry, the
// multiplier m = L * (-q^-1 mod 2^32), and adds m * q * 2^(32 i) with the SAME two aligned
// IMAD.WIDE carry chains a product row uses (row i of "q times m"), so the reduction costs N^2
// wide multiplies + N 32-bit ones instead of the N(N+1)/2 + N^2 of a two-product REDC.  The
// chains end in words that may already be full, so their carry-outs are collected in cc[] (by
// position) and enter the final merge of the high half.
template <class F>
GECC_HD fel<F> redc_ws_eo(const F& f, uint32_t* e, uint32_t* o) {
    constexpr int N = F::N;
    uint32_t cc[N + 1];  // cc[k]: carries into position N + k
#pragma unroll
    for (int k = 0; k <= N; ++k) cc[k] = 0;
    uint32_t c = 0;      // carry into position i from the eliminated positions below
    // q[0] and -q^-1 mod 2^32 offset by a word of constant memory (zero) that ptxas cannot fold:
    // when they are 1 and -1 (BLS12-377) it rewrites the multiplier as a negation and the first
    // product of every chain as an addition, and then no longer pairs the chains into IMAD.WIDE
    // (611 instead of 469 instructions per 12-limb product)
    const uint32_t q0 = f.q(0) + opaque_zero(), qinv = f.qinv32 + opaque_zero();
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const uint32_t below = i ? o[i - 1] : 0u;
        const uint32_t m = (e[i] + below + c) * qinv;
        if ((i & 1) == 0) {
            e[i] = mad_lo_cc(q0, m, e[i]);
            e[i + 1] = madc_hi_cc(q0, m, e[i + 1]);
#pragma unroll
            for (int j = 2; j < N; j += 2) {
                e[i + j] = madc_lo_cc(f.q(j), m, e[i + j]);
                e[i + j + 1] = madc_hi_cc(f.q(j), m, e[i + j + 1]);
            }
            cc[i] = addc(cc[i], 0);
            o[i] = mad_lo_cc(f.q(1), m, o[i]);
            o[i + 1] = madc_hi_cc(f.q(1), m, o[i + 1]);
#pragma unroll
            for (int j = 3; j < N; j += 2) {
                o[i + j - 1] = madc_lo_cc(f.q(j), m, o[i + j - 1]);
                o[i + j] = madc_hi_cc(f.q(j), m, o[i + j]);
            }
            cc[i + 1] = addc(cc[i + 1], 0);
        } else {
            o[i - 1] = mad_lo_cc(q0, m, o[i - 1]);
            o[i] = madc_hi_cc(q0, m, o[i]);
#pragma unroll
            for (int j = 2; j < N; j += 2) {
                o[i + j - 1] = madc_lo_cc(f.q(j), m, o[i + j - 1]);
                o[i + j] = madc_hi_cc(f.q(j), m, o[i + j]);
            }
            cc[i] = addc(cc[i], 0);
            e[i + 1] = mad_lo_cc(f.q(1), m, e[i + 1]);
            e[i + 2] = madc_hi_cc(f.q(1), m, e[i + 2]);
#pragma unroll
            for (int j = 3; j < N; j += 2) {
                e[i + j] = madc_lo_cc(f.q(j), m, e[i + j]);
                e[i + j + 1] = madc_hi_cc(f.q(j), m, e[i + j + 1]);
            }
            cc[i + 1] = addc(cc[i + 1], 0);
        }
        // position i now sums to 0 mod 2^32; what it carries into position i + 1:
        const uint32_t s1 = add_cc(e[i], i ? o[i - 1] : 0u);
        const uint32_t k1 = addc(0, 0);
        add_cc(s1, c);
        c = addc(k1, 0);
    }
    // high half: e[N + k] + o[N + k - 1] + cc[k] (+ c at k = 0)
    fel<F> r;
    r.w[0] = add_cc(e[N], o[N - 1]);
#pragma unroll
    for (int k = 1; k < N; ++k) r.w[k] = addc_cc(e[N + k], o[N + k - 1]);
    uint32_t top = addc(cc[N], 0);
    r.w[0] = add_cc(r.w[0], c);
#pragma unroll
    for (int k = 1; k < N; ++k) r.w[k] = addc_cc(r.w[k], 0);
    top = addc(top, 0);
    r.w[0] = add_cc(r.w[0], cc[0]);
#pragma unroll
    for (int k = 1; k < N; ++k) r.w[k] = addc_cc(r.w[k], cc[k]);
    top = addc(top, 0);
    return final_sub(f, r, top);
}
// the same from a merged 2N-limb value
template <class F>
GECC_HD fel<F> redc_ws(const F& f, const uint32_t* t) {
    constexpr int N = F::N;
    uint32_t e[2 * N], o[2 * N];
#pragma unroll
    for (int k = 0; k < 2 * N; ++k) {
        e[k] = t[k];
        o[k] = 0;
    }
    return redc_ws_eo(f, e, o);
}

// Generic REDC for any odd q (reference: reduce_generic_raw, field.cpp:50-78, same
// value): m = t_lo * (-q^-1) mod 2^256, result = (t + m*q) / 2^256, one final
// subtraction.  Two more products instead of a word-serial sweep: no dependent
// chain of 8 multiplier words.
template <class F>
GECC_HD fel<F> redc_generic(const F& f, const uint32_t* t) {
    constexpr int N = F::N;
    uint32_t ninv[N], q[N], m[N], u[2 * N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        ninv[i] = f.ninv(i);
        q[i] = f.q(i);
    }
    mul_low_n<N>(m, t, ninv);
    mul_wide_n<N>(u, m, q);
    // t_lo + u_lo == 0 mod 2^(32N): it carries exactly when t_lo != 0
    uint32_t nz = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) nz |= t[i];
    add_cc(nz != 0 ? 1u : 0u, 0xFFFFFFFFu);
    fel<F> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = addc_cc(t[N + i], u[N + i]);
    uint32_t top = addc(0, 0);
    return final_sub(f, r, top);
}

// secp256k1 base field, q = 2^256 - c with c = 2^32 + 977.  Word-serial REDC where
// m_i * q = m_i * 2^256 - m_i * c, so each step needs one low multiply (m_i) and
// one high multiply (m_i * 977); D carries the running amount still to be
// subtracted from the next limb.  Result = t_hi + M - D, then one conditional
// subtraction done as "+ c with carry-out".  16 multiplies instead of 72.
template <class F>
GECC_HD fe redc_secp(const F& f, const uint32_t* t) {
    uint32_t m[8];
    uint32_t dlo = 0, dhi = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t v = sub_cc(t[i], dlo);
        uint32_t bmask = subc(0, 0);           // 0xFFFFFFFF on borrow (sub family only:
                                               // a sub-produced flag must never feed addc)
        m[i] = mul_lo(v, F::qinv32);           // m_i * 977 == v mod 2^32
        uint32_t ph = mul_hi(m[i], 977u);
        uint32_t tmp = dhi + ph - bmask;       // dhi + hi(m_i*977) + borrow (no overflow)
        dlo = add_cc(tmp, m[i]);               // + m_i from the 2^32 term of c
        dhi = addc(0, 0);
    }
    fe r;
    r.w[0] = add_cc(t[8], m[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) r.w[i] = addc_cc(t[8 + i], m[i]);
    uint32_t top = addc(0, 0);
    r.w[0] = sub_cc(r.w[0], dlo);
    r.w[1] = subc_cc(r.w[1], dhi);
#pragma unroll
    for (int i = 2; i < 8; ++i) r.w[i] = subc_cc(r.w[i], 0);
    top = subc(top, 0);
    // (top:r) >= q  <=>  (top:r) + c >= 2^256
    fe s;
    s.w[0] = add_cc(r.w[0], 977u);
    s.w[1] = addc_cc(r.w[1], 1u);
#pragma unroll
    for (int i = 2; i < 8; ++i) s.w[i] = addc_cc(r.w[i], 0);
    uint32_t over = addc(top, 0);
    (void)f;
    return fe_select(over != 0, s, r);
}

// SM2 base field (SCA-256), q = 2^256 - 2^224 - 2^96 + 2^64 - 1, q_inv32 == 1: the
// Montgomery multiplier of every eliminated word is the word itself and
//   m q = m 2^256 - m 2^224 - m 2^96 + m 2^64 - m
// is single-word signed contributions, so the whole reduction is additions and
// subtractions (reference: reduce_sm2_impl, field.cpp:88-128; same two-words-per-pass
// schedule).  Pass j eliminates t[j], t[j+1] (m0, m1); their combined deltas are
//   +m0 @ j+2,  +m1 - m0 @ j+3,  -m1 @ j+4,  -m0 @ j+7,  +m0 - m1 @ j+8,  +m1 @ j+9
// applied as one add chain and one sub chain that run to the top word.  No multiply.
template <class F>
GECC_HD fe redc_sm2(const F& f, const uint32_t* tin) {
    uint32_t t[17];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = tin[i];
    t[16] = 0;
    // FOUR words per pass (two passes instead of the reference's four two-word passes, same value):
    // the multipliers of words j+2, j+3 are what words j, j+1 leave there,
    //   m2 = t[j+2] + m0            (the add chain's first step)
    //   m3 = t[j+3] + m1 + carry - m0
    // and from position j+4 on every position receives at most one positive and one negative term of
    // the four eliminations, so ONE add chain and ONE sub chain apply them all:
    //   +m0 +m1 +m2 +m3 @ j+2 .. j+5 and @ j+8 .. j+11;  -m0 @ j+3, j+7; -m1 @ j+4, j+8; -m2 @ j+5, j+9; -m3 @ j+6, j+10
    // 52 chain operations per reduction instead of 92, and half the depth.
#pragma unroll
    for (int j = 0; j < 8; j += 4) {
        const uint32_t m0 = t[j], m1 = t[j + 1];
        const uint32_t m2 = add_cc(t[j + 2], m0);
        const uint32_t u3 = addc_cc(t[j + 3], m1);
        const uint32_t m3 = u3 - m0;  // plain subtraction: leaves the carry flag of the chain alone
        t[j + 4] = addc_cc(t[j + 4], m2);
        t[j + 5] = addc_cc(t[j + 5], m3);
#pragma unroll
        for (int w = j + 6; w < 17; ++w) {
            const uint32_t d = (w == j + 8) ? m0 : (w == j + 9) ? m1 : (w == j + 10) ? m2 : (w == j + 11) ? m3 : 0u;
            t[w] = addc_cc(t[w], d);
        }
        sub_cc(u3, m0);  // position j+3 again, for its borrow (the word itself is eliminated)
#pragma unroll
        for (int w = j + 4; w < 17; ++w) {
            const uint32_t d = (w == j + 4 || w == j + 8) ? m1 : (w == j + 5 || w == j + 9) ? m2
                             : (w == j + 6 || w == j + 10) ? m3 : (w == j + 7) ? m0 : 0u;
            t[w] = subc_cc(t[w], d);
        }
    }
    fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.w[i] = t[8 + i];
    if constexpr (F::kind == KIND_SM2_LAZY) {
        // weakly reduced inputs: the value is below 2^256 + q, so t[16] is 0 or 1 and folding it
        // (+ c under a mask) cannot wrap: what is left of a set top word is below q
        const uint32_t k = t[16], m = 0u - k;
        fe o;
        o.w[0] = add_cc(r.w[0], k);
        o.w[1] = addc_cc(r.w[1], 0);
        o.w[2] = addc_cc(r.w[2], m);
#pragma unroll
        for (int i = 3; i < 7; ++i) o.w[i] = addc_cc(r.w[i], 0);
        o.w[7] = addc(r.w[7], k);
        return o;
    } else {
        return final_sub(f, r, t[16]);
    }
}

template <class F>
GECC_HD fel<F> redc(const F& f, const uint32_t* t) {
    if constexpr (F::kind == KIND_SECP_P) return redc_secp(f, t);
    else if constexpr (F::kind == KIND_SECP_LAZY) return redc_secp_lazy(t);
    else if constexpr (F::kind == KIND_SM2_P || F::kind == KIND_SM2_LAZY) return redc_sm2(f, t);
    else return redc_ws(f, t);
}

// ---------------------------------------------------------------- mul / sqr
#if defined(GECC_COUNT_OPS) && !defined(__CUDA_ARCH__)
// test-only instrumentation (tests/hostsim): executed products per field kind,
// used to derive the analytic work-per-lane figures quoted in DESIGN.md / bench.py
struct OpCounters {
    unsigned long long mul[3], sqr[3], safegcd[3];
};
inline OpCounters& op_counters() {
    static OpCounters c = {};
    return c;
}
#define GECC_COUNT(what, F) (op_counters().what[F::kind == KIND_GENERIC ? 0 : 1]++)
#else
#define GECC_COUNT(what, F) ((void)0)
#endif

template <class F>
GECC_HD fel<F> fe_mul_inl(const F& f, const fel<F>& a, const fel<F>& b) {
    GECC_COUNT(mul, F);
    if constexpr (F::kind == KIND_GENERIC) {  // reduce the unmerged product: no merge pass in between
        uint32_t e[2 * F::N], o[2 * F::N];
        mul_wide_eo<F::N>(e, o, a.w, b.w);
        return redc_ws_eo(f, e, o);
    }
    uint32_t t[2 * F::N];
    mul_wide_n<F::N>(t, a.w, b.w);
    return redc(f, t);
}
template <class F>
GECC_HD fel<F> fe_sqr_inl(const F& f, const fel<F>& a) {
    GECC_COUNT(sqr, F);
    uint32_t t[2 * F::N];
    sqr_wide_n<F::N>(t, a.w);
    return redc(f, t);
}
// On the device the two products are real functions with by-value arguments: the
// ABI passes the 16 + 8 limbs in registers (no stack traffic), and the hot code
// of a whole ECDSA kernel shrinks to these two bodies plus glue, which is what
// keeps it inside the instruction caches (round-1 ncu: with everything inlined the
// top stall of k_verify was no_instruction).  Runtime fields stay inline.
#if defined(__CUDA_ARCH__) && !defined(GECC_INLINE_FIELD)
#if defined(GECC_PRODUCTS_SMEM)
// experiment: operands and result travel through per-thread shared-memory slots (16-byte granules,
// granule g of thread t at [g * 256 + t]: conflict-free LDS.128 / STS.128) instead of the register
// ABI -- no argument / result register moves around the call.  1-D blocks of <= 256 threads, N = 8.
template <class F>
__device__ __forceinline__ uint4* product_slots() {
    __shared__ uint4 slots[6 * 256];
    return slots + threadIdx.x;
}
__device__ __forceinline__ void slot_store(uint4* s, int g, const uint32_t* w) {
    s[g * 256] = make_uint4(w[0], w[1], w[2], w[3]);
    s[(g + 1) * 256] = make_uint4(w[4], w[5], w[6], w[7]);
}
__device__ __forceinline__ void slot_load(const uint4* s, int g, uint32_t* w) {
    const uint4 a = s[g * 256], b = s[(g + 1) * 256];
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}
template <class F>
__device__ __noinline__ void fe_mul_smem() {
    uint4* s = product_slots<F>();
    fel<F> a, b;
    slot_load(s, 0, a.w);
    slot_load(s, 2, b.w);
    const fel<F> r = fe_mul_inl(F{}, a, b);
    slot_store(s, 4, r.w);
}
template <class F>
__device__ __noinline__ void fe_sqr_smem() {
    uint4* s = product_slots<F>();
    fel<F> a;
    slot_load(s, 0, a.w);
    const fel<F> r = fe_sqr_inl(F{}, a);
    slot_store(s, 4, r.w);
}
template <class F>
__device__ __forceinline__ fel<F> fe_mul_call(const fel<F>& a, const fel<F>& b) {
    if constexpr (F::N != 8) return fe_mul_inl(F{}, a, b);
    uint4* s = product_slots<F>();
    slot_store(s, 0, a.w);
    slot_store(s, 2, b.w);
    fe_mul_smem<F>();
    fel<F> r;
    slot_load(s, 4, r.w);
    return r;
}
template <class F>
__device__ __forceinline__ fel<F> fe_sqr_call(const fel<F>& a) {
    if constexpr (F::N != 8) return fe_sqr_inl(F{}, a);
    uint4* s = product_slots<F>();
    slot_store(s, 0, a.w);
    fe_sqr_smem<F>();
    fel<F> r;
    slot_load(s, 4, r.w);
    return r;
}
#elif defined(GECC_PRODUCTS_BY_REF)
// experiment: operands and result through local memory (LSU pipe) instead of register moves
template <class F>
__device__ __noinline__ void fe_mul_ref(fel<F>* r, const fel<F>* a, const fel<F>* b) {
    *r = fe_mul_inl(F{}, *a, *b);
}
template <class F>
__device__ __noinline__ void fe_sqr_ref(fel<F>* r, const fel<F>* a) {
    *r = fe_sqr_inl(F{}, *a);
}
template <class F>
__device__ __forceinline__ fel<F> fe_mul_call(const fel<F>& a, const fel<F>& b) {
    fel<F> r;
    fe_mul_ref<F>(&r, &a, &b);
    return r;
}
template <class F>
__device__ __forceinline__ fel<F> fe_sqr_call(const fel<F>& a) {
    fel<F> r;
    fe_sqr_ref<F>(&r, &a);
    return r;
}
#else
template <class F>
__device__ __noinline__ fel<F> fe_mul_call(fel<F> a, fel<F> b) {
    return fe_mul_inl(F{}, a, b);
}
template <class F>
__device__ __noinline__ fel<F> fe_sqr_call(fel<F> a) {
    return fe_sqr_inl(F{}, a);
}
#endif
template <class F>
GECC_HD fel<F> fe_mul(const F& f, const fel<F>& a, const fel<F>& b) {
    if constexpr (std::is_empty<F>::value) return fe_mul_call<F>(a, b);
    else return fe_mul_inl(f, a, b);
}
template <class F>
GECC_HD fel<F> fe_sqr(const F& f, const fel<F>& a) {
    if constexpr (std::is_empty<F>::value) return fe_sqr_call<F>(a);
    else return fe_sqr_inl(f, a);
}
#else
template <class F>
GECC_HD fel<F> fe_mul(const F& f, const fel<F>& a, const fel<F>& b) {
    return fe_mul_inl(f, a, b);
}
template <class F>
GECC_HD fel<F> fe_sqr(const F& f, const fel<F>& a) {
    return fe_sqr_inl(f, a);
}
#endif
template <class F>
GECC_HD fel<F> fe_to_mont(const F& f, const fel<F>& a) {  // a * R
    if constexpr (F::kind == KIND_SECP_LAZY) return a;  // plain representation: R = 1
    fel<F> r2;
#pragma unroll
    for (int i = 0; i < F::N; ++i) r2.w[i] = f.r2(i);
    return fe_mul(f, a, r2);
}
template <class F>
GECC_HD fel<F> fe_from_mont(const F& f, const fel<F>& a) {  // a * R^-1
    if constexpr (F::kind == KIND_SECP_LAZY) return lazy_canon(f, a);  // leaves the field layer: canonical
    uint32_t t[2 * F::N];
#pragma unroll
    for (int i = 0; i < F::N; ++i) {
        t[i] = a.w[i];
        t[F::N + i] = 0;
    }
    if constexpr (F::kind == KIND_SM2_LAZY) return weak_canon(f, redc(f, t));
    else return redc(f, t);
}

// a^(q-2) in Montgomery form, 4-bit fixed window: 256 squarings + 64 + 14 products.
// Not unrolled on purpose (code size).  Zero maps to zero.
template <class F>
GECC_HD_CALL fel<F> fe_inv_fermat(const F& f, const fel<F>& a) {
    fel<F> tab[16];
    tab[0] = fe_one(f);
    tab[1] = a;
#pragma unroll 1
    for (int i = 2; i < 16; ++i) tab[i] = fe_mul(f, tab[i - 1], a);
    fel<F> r = fe_one(f);
#pragma unroll 1
    for (int k = 8 * F::N - 1; k >= 0; --k) {
        r = fe_sqr(f, r);
        r = fe_sqr(f, r);
        r = fe_sqr(f, r);
        r = fe_sqr(f, r);
        uint32_t nib = (f.qm2(k >> 3) >> ((k & 7) * 4)) & 15u;
        r = fe_mul(f, r, tab[nib]);
    }
    return r;
}

}  // namespace gecc
