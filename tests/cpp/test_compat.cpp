// Reads like the reference's tests/test_batch_point.cpp, written against
// include/gecc/sm2batch_compat.hpp: random points by batch_fpmul, the exceptional-lane
// fixture (indices 3, 7, 11, 19, 23, 31, 47 in n = 64; test_batch_point.cpp:70-100),
// "t all infinity returns p" (:102-112), size-mismatch errors (:306-322), and the checker
// is the C oracle (oracle/gecc_oracle.h), linked only into this test.
#include <cstdio>
#include <random>
#include <vector>

#include "gecc/sm2batch_compat.hpp"
#include "gecc_oracle.h"

using namespace sm2b;

static int failures = 0;
#define CHECK(cond)                                                     \
    do {                                                                \
        if (!(cond)) {                                                  \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                 \
        }                                                               \
    } while (0)

static std::vector<Scalar> random_scalars(std::mt19937_64& rng, std::size_t n) {
    std::vector<Scalar> s(n);
    for (auto& x : s) {
        for (int k = 0; k < 8; k += 2) {
            std::uint64_t v = rng();
            x.v.w[k] = (std::uint32_t)v;
            x.v.w[k + 1] = (std::uint32_t)(v >> 32);
        }
        x.v.w[7] &= 0x7FFFFFFFu;
    }
    return s;
}

static BatchPointBuffer oracle_padd(int curve, const BatchPointBuffer& p, const BatchPointBuffer& t) {
    BatchPointBuffer o = BatchPointBuffer::make(p.n);
    go_batch_padd(curve, p.n, p.x.data(), p.y.data(), p.infinity_mask.data(), t.x.data(), t.y.data(),
                  t.infinity_mask.data(), o.x.data(), o.y.data(), o.infinity_mask.data(), 4);
    return o;
}
static bool same(const CurveParams& c, const BatchPointBuffer& a, const BatchPointBuffer& b) {
    if (a.n != b.n) return false;
    for (std::size_t i = 0; i < a.n; ++i)
        if (!(a.get(c, i) == b.get(c, i))) return false;
    return true;
}

static void run(const CurveParams& C, int curve_id) {
    std::mt19937_64 rng(62 + curve_id);
    const std::size_t n = 64;
    auto ps = batch_fpmul(C, random_scalars(rng, n), sm2_base_table(), LanePlan::make(n, 8));
    auto ts = batch_fpmul(C, random_scalars(rng, n), sm2_base_table(), LanePlan::make(n, 8));

    auto neg = [&](const AffinePoint& p) {  // -p via the oracle's field subtraction
        AffinePoint r = p;
        std::uint32_t zero[8] = {0}, out[8];
        go_field_op(curve_id, 0, 2, 1, zero, p.y.w.data(), out);
        for (int k = 0; k < 8; ++k) r.y.w[k] = out[k];
        return r;
    };
    AffinePoint inf{{}, {}, true};
    ts.set(3, ps.get(C, 3));         // doubling pair
    ts.set(7, neg(ps.get(C, 7)));    // inverse pair
    ps.set(11, inf);                 // left infinity
    ts.set(19, inf);                 // right infinity
    ps.set(23, inf);
    ts.set(23, inf);                 // both
    ts.set(31, ps.get(C, 31));
    ps.set(47, inf);

    auto out = batch_padd(C, ps, ts, LanePlan::make(n, 4));
    CHECK(same(C, out, oracle_padd(curve_id, ps, ts)));
    CHECK(out.get(C, 7).infinity);
    CHECK(out.get(C, 23).infinity);
    auto dbl = batch_pdbl(C, ps, LanePlan::make(n, 4));
    CHECK(out.get(C, 3) == dbl.get(C, 3));

    // t all infinity returns p
    BatchPointBuffer all_inf = BatchPointBuffer::make(n);
    for (std::size_t i = 0; i < n; ++i) all_inf.set(i, inf);
    CHECK(same(C, batch_padd(C, ps, all_inf, LanePlan::make(n, 4)), ps));

    // size / plan mismatches throw std::invalid_argument
    bool threw = false;
    try { (void)batch_padd(C, ps, BatchPointBuffer::make(n - 1), LanePlan::make(n, 4)); }
    catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { (void)batch_padd(C, ps, ts, LanePlan::make(n + 1, 4)); }
    catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);

    // batch_invert: zero masking
    BatchColumnBuffer v = BatchColumnBuffer::make(40), want = BatchColumnBuffer::make(40);
    for (std::size_t i = 0; i < 40; ++i) v.set(i, (i % 13 == 0) ? Limbs256::zero() : ps.get(C, i).x);
    go_batch_invert(curve_id, 0, 40, v.data(), want.data(), 3);
    auto got = batch_invert(v, *C.base_field, LanePlan::make(40, 3));
    CHECK(got.cols == want.cols);

    // upmul against the serial ground truth; MSM against the definition
    auto ks = random_scalars(rng, n);
    auto up = batch_upmul(C, ks, ts, LanePlan::make(n, 4));
    BatchPointBuffer ser = BatchPointBuffer::make(n);
    auto kc = detail::scalar_columns(ks);
    go_pmul_serial(curve_id, n, kc.data(), ts.x.data(), ts.y.data(), ts.infinity_mask.data(), ser.x.data(),
                   ser.y.data(), ser.infinity_mask.data());
    CHECK(same(C, up, ser));
    // the same curve given at run time: FieldParams::make(q) + CurveParams::user(field, a, b)
    // (field.cpp:159-179, curve.hpp:51-59) must give the compiled-in kernels' results
    {
        Limbs256 q{}, a_mont{}, b_mont{}, gx{}, gy{}, r{}, r2{};
        go_field_params(curve_id, 0, q.w.data(), r.w.data(), r2.w.data());
        FieldParams fq = FieldParams::make(q);
        CHECK(fq.r == r);
        CHECK(fq.r2 == r2);
        go_curve_params(curve_id, a_mont.w.data(), b_mont.w.data(), gx.w.data(), gy.w.data());
        CurveParams U = CurveParams::user(fq, a_mont, b_mont, C);
        CHECK(same(C, batch_padd(U, ps, ts, LanePlan::make(n, 4)), out));
        CHECK(same(C, batch_pdbl(U, ps, LanePlan::make(n, 4)), dbl));
        auto inv_rt = batch_invert(v, U.field(), LanePlan::make(40, 3));
        CHECK(inv_rt.cols == want.cols);
        bool even_threw = false;
        Limbs256 even = q;
        even.w[0] &= ~1u;
        try { (void)FieldParams::make(even); }
        catch (const std::invalid_argument&) { even_threw = true; }
        CHECK(even_threw);
    }
    AffinePoint m = msm(C, ks, ts), mw;
    std::uint8_t winf = 0;
    go_msm(curve_id, n, kc.data(), ts.x.data(), ts.y.data(), ts.infinity_mask.data(), mw.x.w.data(), mw.y.w.data(), &winf);
    mw.infinity = winf != 0;
    CHECK(m == mw);
}

int main() {
    run(CurveParams::sm2(), 0);
    run(CurveParams::secp256k1(), 1);
    std::printf(failures ? "FAILED (%d)\n" : "compat tests passed%.0d\n", failures);
    return failures ? 1 : 0;
}
