// TEST-ONLY host simulator: compiles the product's __host__ __device__ limb code
// (paper_2501_03245_b200/csrc/*.cuh) with g++ so that the exact device logic can be
// exercised in the GPU-less authoring container.  gecc_prims.cuh emulates the
// PTX carry flag on the host.  Nothing here is reachable from libgecc_b200.so.
#include <cstddef>
#include <cstdint>

#include "gecc_field.cuh"
#include "gecc_modinv.cuh"

using namespace gecc;

namespace {
template <int N = 8>
feN<N> col_get(const uint32_t* c, size_t n, size_t i) {
    feN<N> v;
    for (int k = 0; k < N; ++k) v.w[k] = c[k * n + i];
    return v;
}
template <int N>
void col_set(uint32_t* c, size_t n, size_t i, const feN<N>& v) {
    for (int k = 0; k < N; ++k) c[k * n + i] = v.w[k];
}

template <class F>
int field_op_t(const F& f, int op, size_t n, const uint32_t* a, const uint32_t* b, uint32_t* out) {
    constexpr int N = F::N;
    for (size_t i = 0; i < n; ++i) {
        feN<N> x = col_get<N>(a, n, i), y = b ? col_get<N>(b, n, i) : fe_zero_n<N>(), r = fe_zero_n<N>();
        switch (op) {
            case 0: r = fe_mul(f, x, y); break;
            case 1: r = fe_add(f, x, y); break;
            case 2: r = fe_sub(f, x, y); break;
            case 3: r = fe_to_mont(f, x); break;
            case 4: r = fe_from_mont(f, x); break;
            case 5: r = fe_is_zero(x) ? x : fe_inv_fermat(f, x); break;
            case 6: r = fe_sqr(f, x); break;
            case 7: r = fe_inv(f, x); break;            // safegcd, Montgomery in/out
            case 8: r = safegcd_inverse(f, x); break;   // safegcd, plain in/out
            case 9: r = fe_dbl(f, x); break;            // 2x (shift form on the lazy field)
            case 10: r = fe_mul8(f, x); break;          // 8x
            case 11: r = fe_inv_var(f, x); break;       // variable-time safegcd, Montgomery in/out
            case 12: r = safegcd_inverse_var(f, x); break;  // variable-time safegcd, plain in/out
            case 13: r = safegcd_inverse_sched<false>(f, x); break;  // latency-scheduled, plain in/out
            case 14: r = safegcd_inverse_sched<true>(f, x); break;   // + early exit
            default: return 1;
        }
        col_set(out, n, i, r);
    }
    return 0;
}
}  // namespace

extern "C" {

// field: 0 SecpP 1 SecpN 2 Sm2P 3 Sm2N ; 4 = runtime field given by rt
int hs_field_op(int field, const FieldRT* rt, int op, size_t n, const uint32_t* a,
                const uint32_t* b, uint32_t* out) {
    switch (field) {
        case 0: return field_op_t(SecpP{}, op, n, a, b, out);
        case 1: return field_op_t(SecpN{}, op, n, a, b, out);
        case 2: return field_op_t(Sm2P{}, op, n, a, b, out);
        case 3: return field_op_t(Sm2N{}, op, n, a, b, out);
        case 4: return field_op_t(*rt, op, n, a, b, out);
        case 5: return field_op_t(SecpPL{}, op, n, a, b, out);  // lazy plain secp256k1 (outputs weakly reduced)
        case 10: return field_op_t(Sm2PL{}, op, n, a, b, out);  // lazy Montgomery SM2 (outputs weakly reduced)
        case 6: return field_op_t(Bls381P{}, op, n, a, b, out);  // 12 limbs
        case 7: return field_op_t(Bls381R{}, op, n, a, b, out);
        case 8: return field_op_t(Bls377P{}, op, n, a, b, out);  // 12 limbs
        case 9: return field_op_t(Bls377R{}, op, n, a, b, out);
    }
    return 1;
}

}  // extern "C"

// BLS12-381 G1 point formulas (12-limb coordinates): op 0 = P + Q through jac_madd / jac_add,
// 1 = 2P, 2 = k * P by double-and-add with mixed additions; affine Montgomery in and out.
#include "gecc_curve.cuh"
template <class C>
static int bls_point_op_t(int op, size_t n, const uint32_t* k, const uint32_t* px, const uint32_t* py,
                          const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty, const uint8_t* tinf,
                          uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    const typename C::Fp f{};
    for (size_t i = 0; i < n; ++i) {
        caff<C> p{col_get<12>(px, n, i), col_get<12>(py, n, i)};
        cjac<C> P = jac_infinity<C>();
        if (!pinf[i]) { P.X = p.x; P.Y = p.y; P.Z = fe_one(f); }
        cjac<C> r = jac_infinity<C>();
        if (op == 0) {
            caff<C> t{col_get<12>(tx, n, i), col_get<12>(ty, n, i)};
            cjac<C> T = jac_infinity<C>();
            if (!tinf[i]) { T.X = t.x; T.Y = t.y; T.Z = fe_one(f); }
            // exercise both routes: mixed when T is finite, and the general addition of two doubled-up points
            cjac<C> m = tinf[i] ? P : jac_madd<C>(P, t);
            cjac<C> g = jac_add<C>(jac_add<C>(P, T), jac_infinity<C>());
            if (jac_is_inf<C>(m) != jac_is_inf<C>(g)) return 2;
            r = g;
            if (!jac_is_inf<C>(m)) {  // the two routes must agree as affine points
                caff<C> am = jac_to_aff_with<C>(m, fe_inv(f, m.Z)), ag = jac_to_aff_with<C>(g, fe_inv(f, g.Z));
                if (!fe_eq(am.x, ag.x) || !fe_eq(am.y, ag.y)) return 3;
            }
        } else if (op == 1) {
            r = jac_dbl<C>(P);
        } else {
            feN<8> s = col_get<8>(k, n, i);
            for (int b = 255; b >= 0; --b) {
                r = jac_dbl<C>(r);
                if (!pinf[i] && ((s.w[b >> 5] >> (b & 31)) & 1)) r = jac_madd<C>(r, p);
            }
        }
        if (jac_is_inf<C>(r)) {
            col_set(ox, n, i, fe_zero_n<12>());
            col_set(oy, n, i, fe_zero_n<12>());
            oinf[i] = 1;
        } else {
            caff<C> a = jac_to_aff_with<C>(r, fe_inv(f, r.Z));
            col_set(ox, n, i, a.x);
            col_set(oy, n, i, a.y);
            oinf[i] = 0;
        }
    }
    return 0;
}
// curve: 2 = BLS12-381, 3 = BLS12-377
extern "C" int hs_bls_point_op(int curve, int op, size_t n, const uint32_t* k, const uint32_t* px, const uint32_t* py,
                               const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty, const uint8_t* tinf,
                               uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (curve == 3) return bls_point_op_t<Bls377Curve>(op, n, k, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
    return bls_point_op_t<Bls381Curve>(op, n, k, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
}

// ---------------------------------------------------------------------------
// ECDSA / point-multiplication lanes (gecc_ecdsa.cuh) run as plain host loops.
#include <vector>

#include "gecc_ecdsa.cuh"

namespace {

#ifndef HS_WG
#define HS_WG 4  // small fixed-base window so the host can build the table quickly
#endif

template <class C>
const std::vector<uint32_t>& host_gtable() {
    static std::vector<uint32_t> tab;
    if (!tab.empty()) return tab;
    using GT = GTable<HS_WG>;
    const typename C::Fp f{};
    tab.assign((size_t)GT::windows * GT::per_window * 16, 0);
    jac base;  // 2^(WG*j) * G
    aff g = curve_g<C>();
    base.X = g.x; base.Y = g.y; base.Z = fe_one(f);
    for (int j = 0; j < GT::windows; ++j) {
        aff b = jac_to_aff_with<C>(base, fe_inv(f, base.Z));
        jac acc = jac_infinity<C>();
        for (int d = 1; d <= GT::per_window; ++d) {
            acc = jac_madd<C>(acc, b);
            aff e = jac_to_aff_with<C>(acc, fe_inv(f, acc.Z));
            uint32_t* p = &tab[((size_t)j * GT::per_window + (d - 1)) * 16];
            for (int i = 0; i < 8; ++i) { p[i] = e.x.w[i]; p[8 + i] = e.y.w[i]; }
        }
        for (int k = 0; k < HS_WG; ++k) base = jac_dbl<C>(base);
    }
    return tab;
}

template <class C>
void store_point(const jac& r, uint32_t* ox, uint32_t* oy, uint8_t* oinf, size_t n, size_t i) {
    const typename C::Fp f{};
    if (jac_is_inf<C>(r)) {
        col_set(ox, n, i, fe_zero());
        col_set(oy, n, i, fe_zero());
        oinf[i] = 1;
        return;
    }
    aff a = jac_to_aff_with<C>(r, fe_inv(f, r.Z));
    col_set(ox, n, i, a.x);
    col_set(oy, n, i, a.y);
    oinf[i] = 0;
}

// 1: the constant-structure forms (GECC_SECRET_UNIFORM) of k*G, k*P, sign, keygen
static int g_uniform = 0;

template <class C>
int fpmul_t(size_t n, const uint32_t* k, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    GTable<HS_WG> gt{host_gtable<C>().data()};
    for (size_t i = 0; i < n; ++i)
        store_point<C>(g_uniform ? fixed_base_mul_uniform<C, HS_WG>(col_get(k, n, i), gt)
                                 : fixed_base_mul<C, HS_WG>(col_get(k, n, i), gt), ox, oy, oinf, n, i);
    return 0;
}
template <class C>
int upmul_t(size_t n, const uint32_t* k, const uint32_t* px, const uint32_t* py,
            const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    uint32_t lane[8 * 16];
    LaneTable lt{lane, 1};
    for (size_t i = 0; i < n; ++i) {
        if (pinf && pinf[i]) { store_point<C>(jac_infinity<C>(), ox, oy, oinf, n, i); continue; }
        aff p{col_get(px, n, i), col_get(py, n, i)};
        if (g_uniform) {
            build_lane_table<C>(p, lt);
            store_point<C>(var_base_mul_uniform<C>(col_get(k, n, i), lt), ox, oy, oinf, n, i);
            continue;
        }
        // the kernel's route (slots; lane table on the isomorphic curve when a = 0) ...
        fe slot_mem[PointSlots::COUNT];
        PointSlots S{slot_mem};
        var_base_mul_point_slots<C>(col_get(k, n, i), p, lt, S);
        store_point<C>(S.load_point(), ox, oy, oinf, n, i);
#if !defined(GECC_COUNT_OPS)
        {   // ... must give the point of the register route (affine table by one inversion)
            const typename C::Fp f{};
            build_lane_table<C>(p, lt);
            const jac a = S.load_point(), b = var_base_mul<C>(col_get(k, n, i), lt);
            if (jac_is_inf<C>(a) != jac_is_inf<C>(b)) return 78;
            if (!jac_is_inf<C>(a)) {  // X_a Z_b^2 == X_b Z_a^2 and Y_a Z_b^3 == Y_b Z_a^3
                const fe za2 = fe_sqr(f, a.Z), zb2 = fe_sqr(f, b.Z);
                if (!fe_eq(f, fe_mul(f, a.X, zb2), fe_mul(f, b.X, za2))) return 78;
                if (!fe_eq(f, fe_mul(f, a.Y, fe_mul(f, zb2, b.Z)), fe_mul(f, b.Y, fe_mul(f, za2, a.Z)))) return 78;
            }
        }
#endif
    }
    return 0;
}
template <class C>
int sign_t(size_t n, const uint8_t* dig, const uint8_t* sec, uint64_t seed, uint64_t base,
           uint8_t* sig, int32_t* st) {
    GTable<HS_WG> gt{host_gtable<C>().data()};
    constexpr int K = GECC_SIGN_K;  // same grouping as k_sign: shared inversions inside a group
    size_t i = 0;
    for (; i + K <= n; i += K) {
        fe e[K], d[K];
        int s4[K];
        for (int j = 0; j < K; ++j) {
            e[j] = scalar_reduce_once<typename C::Fn>(be32_load(dig + 32 * (i + j)));
            d[j] = be32_load(sec + 32 * (i + j));
        }
        if (g_uniform) sign_lanes<C, HS_WG, K, true>(e, d, seed, base + i, gt, sig + 64 * i, s4);
        else {  // through the shared-memory-slot form of the fixed-base additions, as k_sign runs it
            fe slot_mem[PointSlots::COUNT];
            PointSlots S{slot_mem};
            sign_lanes<C, HS_WG, K>(e, d, seed, base + i, gt, sig + 64 * i, s4, false, &S);
        }
        for (int j = 0; j < K; ++j) st[i + j] = s4[j];
    }
    for (; i < n; ++i) {
        fe e = scalar_reduce_once<typename C::Fn>(be32_load(dig + 32 * i));
        fe d = be32_load(sec + 32 * i);
        st[i] = g_uniform ? sign_lane<C, HS_WG, true>(e, d, seed, base + i, gt, sig + 64 * i)
                          : sign_lane<C, HS_WG>(e, d, seed, base + i, gt, sig + 64 * i);
    }
    return 0;
}
// one attempt per lane with explicit nonces (k_sign_nonces)
template <class C>
int sign_nonces_t(size_t n, const uint8_t* dig, const uint8_t* sec, const uint8_t* nonces, uint8_t* sig, int32_t* st) {
    GTable<HS_WG> gt{host_gtable<C>().data()};
    for (size_t i = 0; i < n; ++i) {
        fe e = scalar_reduce_once<typename C::Fn>(be32_load(dig + 32 * i));
        fe d = be32_load(sec + 32 * i);
        fe k = be32_load(nonces + 32 * i);
        st[i] = g_uniform ? sign_lane_nonce<C, HS_WG, true>(e, d, k, gt, sig + 64 * i)
                          : sign_lane_nonce<C, HS_WG>(e, d, k, gt, sig + 64 * i);
    }
    return 0;
}
template <class C>
int verify_t(size_t n, const uint8_t* dig, const uint8_t* pub, const uint8_t* sig, uint8_t* res) {
    GTable<HS_WG> gt{host_gtable<C>().data()};
    uint32_t lane[8 * 16];
    LaneTable lt{lane, 1};
    for (size_t i = 0; i < n; ++i) {
        // the lane as the GPU kernel runs it: the ladder's accumulator at rest in "shared memory" slots
        // (and, on a = 0 curves, the lane table on the isomorphic curve)
        fe slot_mem[PointSlots::COUNT];
        PointSlots S{slot_mem};
        res[i] = verify_lane<C, HS_WG>(dig + 32 * i, pub + 65 * i, sig + 64 * i, gt, lt, &S);
#if !defined(GECC_COUNT_OPS)
        // and with everything in registers (affine lane table by one inversion): must agree
        if (verify_lane<C, HS_WG>(dig + 32 * i, pub + 65 * i, sig + 64 * i, gt, lt) != res[i]) return 77;
#endif
    }
    return 0;
}
template <class C>
int keygen_t(size_t n, uint64_t seed, uint64_t base, uint8_t* sec, uint8_t* pub) {
    GTable<HS_WG> gt{host_gtable<C>().data()};
    const typename C::Fp f{};
    for (size_t i = 0; i < n; ++i) {
        fe d = nonce_scalar<typename C::Fn>(seed, base + i, 0);
        be32_store(sec + 32 * i, d);
        jac r = g_uniform ? fixed_base_mul_uniform<C, HS_WG>(d, gt) : fixed_base_mul<C, HS_WG>(d, gt);
        encode_point<C>(pub + 65 * i, jac_to_aff_with<C>(r, fe_inv(f, r.Z)));
    }
    return 0;
}
}  // namespace

extern "C" {
int hs_fpmul(int curve, size_t n, const uint32_t* k, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    return curve == 0 ? fpmul_t<Sm2Curve>(n, k, ox, oy, oinf) : curve == 3 ? fpmul_t<Sm2LCurve>(n, k, ox, oy, oinf) : curve == 2 ? fpmul_t<SecpLCurve>(n, k, ox, oy, oinf) : fpmul_t<SecpCurve>(n, k, ox, oy, oinf);
}
int hs_upmul(int curve, size_t n, const uint32_t* k, const uint32_t* px, const uint32_t* py,
             const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    return curve == 0 ? upmul_t<Sm2Curve>(n, k, px, py, pinf, ox, oy, oinf) : curve == 3 ? upmul_t<Sm2LCurve>(n, k, px, py, pinf, ox, oy, oinf) : curve == 2 ? upmul_t<SecpLCurve>(n, k, px, py, pinf, ox, oy, oinf) : upmul_t<SecpCurve>(n, k, px, py, pinf, ox, oy, oinf);
}
int hs_sign(int curve, size_t n, const uint8_t* dig, const uint8_t* sec, uint64_t seed,
            uint64_t base, uint8_t* sig, int32_t* st) {
    return curve == 0 ? sign_t<Sm2Curve>(n, dig, sec, seed, base, sig, st) : curve == 3 ? sign_t<Sm2LCurve>(n, dig, sec, seed, base, sig, st) : curve == 2 ? sign_t<SecpLCurve>(n, dig, sec, seed, base, sig, st) : sign_t<SecpCurve>(n, dig, sec, seed, base, sig, st);
}
int hs_verify(int curve, size_t n, const uint8_t* dig, const uint8_t* pub, const uint8_t* sig,
              uint8_t* res) {
    return curve == 0 ? verify_t<Sm2Curve>(n, dig, pub, sig, res) : curve == 3 ? verify_t<Sm2LCurve>(n, dig, pub, sig, res) : curve == 2 ? verify_t<SecpLCurve>(n, dig, pub, sig, res) : verify_t<SecpCurve>(n, dig, pub, sig, res);
}
void hs_set_uniform(int on) { g_uniform = on; }
int hs_sign_nonces(int curve, size_t n, const uint8_t* dig, const uint8_t* sec, const uint8_t* nonces,
                   uint8_t* sig, int32_t* st) {
    return curve == 0 ? sign_nonces_t<Sm2Curve>(n, dig, sec, nonces, sig, st) : curve == 3 ? sign_nonces_t<Sm2LCurve>(n, dig, sec, nonces, sig, st) : curve == 2 ? sign_nonces_t<SecpLCurve>(n, dig, sec, nonces, sig, st) : sign_nonces_t<SecpCurve>(n, dig, sec, nonces, sig, st);
}
int hs_keygen(int curve, size_t n, uint64_t seed, uint64_t base, uint8_t* sec, uint8_t* pub) {
    return curve == 0 ? keygen_t<Sm2Curve>(n, seed, base, sec, pub) : curve == 3 ? keygen_t<Sm2LCurve>(n, seed, base, sec, pub) : curve == 2 ? keygen_t<SecpLCurve>(n, seed, base, sec, pub) : keygen_t<SecpCurve>(n, seed, base, sec, pub);
}
}  // extern "C"

// The additions on shared-memory slots (jac_madd_slots, jac_mmadd_slots, and the (X, Y, ZZ, ZZZ)
// forms zz_madd_slots, zz_mmadd_slots) against jac_madd, for every pair (P_i, Q_i) with the
// accumulator = P_i affine, P_i rescaled by Z = lam_i, and infinity.  Pairs with P == +-Q exercise
// the exceptional branches.  Returns 0 or the number of the first failing check.
template <class C>
static int slot_adds_t(size_t n, const uint32_t* px, const uint32_t* py, const uint32_t* tx, const uint32_t* ty,
                       const uint32_t* lam) {
    const typename C::Fp f{};
    auto same = [&](const jac& a, const jac& b) {  // projective equality
        if (jac_is_inf<C>(a) || jac_is_inf<C>(b)) return jac_is_inf<C>(a) == jac_is_inf<C>(b);
        const fe za2 = fe_sqr(f, a.Z), zb2 = fe_sqr(f, b.Z);
        return fe_eq(f, fe_mul(f, a.X, zb2), fe_mul(f, b.X, za2)) &&
               fe_eq(f, fe_mul(f, a.Y, fe_mul(f, zb2, b.Z)), fe_mul(f, b.Y, fe_mul(f, za2, a.Z)));
    };
    auto same_zz = [&](const PointSlots& S, const jac& b) {  // (X, Y, ZZ, ZZZ) in the slots against b
        const fe zz = S.ld(PointSlots::SZ), zzz = S.ld(PointSlots::S1);
        if (fe_is_zero(f, zz) || jac_is_inf<C>(b)) return fe_is_zero(f, zz) == jac_is_inf<C>(b);
        const fe zb2 = fe_sqr(f, b.Z);
        return fe_eq(f, fe_mul(f, S.ld(PointSlots::SX), zb2), fe_mul(f, b.X, zz)) &&
               fe_eq(f, fe_mul(f, S.ld(PointSlots::SY), fe_mul(f, zb2, b.Z)), fe_mul(f, b.Y, zzz));
    };
    for (size_t i = 0; i < n; ++i) {
        const aff P{col_get(px, n, i), col_get(py, n, i)}, Q{col_get(tx, n, i), col_get(ty, n, i)};
        uint32_t row[16];
        for (int w = 0; w < 8; ++w) { row[w] = Q.x.w[w]; row[8 + w] = Q.y.w[w]; }
        const fe l = col_get(lam, n, i), l2 = fe_sqr(f, l);
        const jac accs[3] = {jac{P.x, P.y, fe_one(f)}, jac{fe_mul(f, P.x, l2), fe_mul(f, P.y, fe_mul(f, l2, l)), l},
                             jac_infinity<C>()};
        for (int neg = 0; neg < 2; ++neg) {
            aff q = Q;
            if (neg) q.y = fe_neg(f, q.y);
            const RowSrc<C> src{row, 1, neg != 0, false};
            for (int a = 0; a < 3; ++a) {
                const jac want = jac_madd<C>(accs[a], q);
                fe mem[PointSlots::COUNT];
                PointSlots S{mem};
                S.store_point(accs[a]);
                jac_madd_slots<C>(S, src);
                if (!same(S.load_point(), want)) return 100 + 10 * a + neg;
                if (a == 0) {
                    S.store_point(accs[a]);
                    jac_mmadd_slots<C>(S, src);
                    if (!same(S.load_point(), want)) return 200 + neg;
                }
                // (X, Y, ZZ, ZZZ)
                S.st(PointSlots::SX, accs[a].X);
                S.st(PointSlots::SY, accs[a].Y);
                S.st(PointSlots::SZ, fe_sqr(f, accs[a].Z));
                S.st(PointSlots::S1, fe_mul(f, fe_sqr(f, accs[a].Z), accs[a].Z));
                zz_madd_slots<C>(S, src);
                if (!same_zz(S, want)) return 300 + 10 * a + neg;
                if (a == 0) {
                    S.st(PointSlots::SX, P.x);
                    S.st(PointSlots::SY, P.y);
                    S.st(PointSlots::SZ, fe_one(f));
                    S.st(PointSlots::S1, fe_one(f));
                    zz_mmadd_slots<C>(S, src);
                    if (!same_zz(S, want)) return 400 + neg;
                }
            }
        }
    }
    return 0;
}
extern "C" int hs_slot_adds(int curve, size_t n, const uint32_t* px, const uint32_t* py, const uint32_t* tx,
                            const uint32_t* ty, const uint32_t* lam) {
    return curve == 0 ? slot_adds_t<Sm2Curve>(n, px, py, tx, ty, lam) : curve == 3 ? slot_adds_t<Sm2LCurve>(n, px, py, tx, ty, lam)
         : curve == 2 ? slot_adds_t<SecpLCurve>(n, px, py, tx, ty, lam) : slot_adds_t<SecpCurve>(n, px, py, tx, ty, lam);
}

// GLV split of secp256k1 scalars: out = m1 (8 limbs) | m2 (8 limbs) per element, signs in sg[2*i..]
extern "C" int hs_glv_split(size_t n, const uint32_t* k, uint32_t* m1, uint32_t* m2, uint8_t* sg) {
    for (size_t i = 0; i < n; ++i) {
        GlvSplit s = glv_split<SecpCurve>(col_get(k, n, i));
        col_set(m1, n, i, s.m1);
        col_set(m2, n, i, s.m2);
        sg[2 * i] = s.neg1;
        sg[2 * i + 1] = s.neg2;
    }
    return 0;
}

// executed-product counters: [mul_generic, mul_special, sqr_generic, sqr_special, safegcd_generic, safegcd_special]
extern "C" void hs_op_counts(unsigned long long* out, int reset) {
#if defined(GECC_COUNT_OPS)
    OpCounters& c = op_counters();
    out[0] = c.mul[0]; out[1] = c.mul[1]; out[2] = c.sqr[0]; out[3] = c.sqr[1];
    out[4] = c.safegcd[0]; out[5] = c.safegcd[1];
    if (reset) c = OpCounters{};
#else
    for (int i = 0; i < 6; ++i) out[i] = 0;
    (void)reset;
#endif
}
extern "C" int hs_window_bits(void) { return HS_WG; }

// raw Montgomery reduction of 16-limb inputs (c < q * 2^256), field ids as hs_field_op
template <class F>
static int redc_t(const F& f, size_t n, const uint32_t* c16, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t t[16];
        for (int k = 0; k < 16; ++k) t[k] = c16[k * n + i];
        const fe r = redc(f, t);
        // every reduction route must give the same canonical value (test_field.cpp:166-169):
        // the two-product REDC is kept as the cross-check of the specialised / word-serial ones
        if (!fe_eq(r, redc_generic(f, t))) return 2;
        col_set(out, n, i, r);
    }
    return 0;
}
extern "C" int hs_redc(int field, size_t n, const uint32_t* c16, uint32_t* out) {
    switch (field) {
        case 0: return redc_t(SecpP{}, n, c16, out);
        case 1: return redc_t(SecpN{}, n, c16, out);
        case 2: return redc_t(Sm2P{}, n, c16, out);
        case 3: return redc_t(Sm2N{}, n, c16, out);
    }
    return 1;
}
