// Reads like the reference's tests/test_protocol.cpp (:40-139, :196-228) and the base-table cases
// of tests/test_batch_point.cpp (:160-208), written against include/gecc/sm2batch_compat.hpp and
// run on the GPU.  The checker is the C oracle (oracle/gecc_oracle.h), linked only into this test.
#include <cstdio>
#include <random>
#include <vector>

#include "gecc/sm2batch_compat.hpp"
#include "gecc_oracle.h"

using namespace sm2b;

static int failures = 0;
#define CHECK(cond)                                                             \
    do {                                                                        \
        if (!(cond)) {                                                          \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                         \
        }                                                                       \
    } while (0)
#define CHECK_THROWS(expr, EXC)                    \
    do {                                           \
        bool threw__ = false;                      \
        try { (void)(expr); } catch (const EXC&) { threw__ = true; } \
        CHECK(threw__);                            \
    } while (0)

struct Fixture {  // test_protocol.cpp:17-38
    std::vector<KeyPair> keys;
    std::vector<AffinePoint> pubs;
    std::vector<Scalar> digests;
    SignResult signed_batch;
    Fixture(const CurveParams& C, std::size_t n, std::uint64_t seed) {
        DeterministicNonceSource key_src(seed ^ 0xABCDEFull, C);
        std::mt19937_64 rng(seed);
        for (std::size_t i = 0; i < n; ++i) {
            keys.push_back(keygen(C, key_src, i));
            pubs.push_back(keys.back().pub);
            Limbs256 raw;
            for (int k = 0; k < 8; k += 2) {
                const std::uint64_t v = rng();
                raw.w[k] = (std::uint32_t)v;
                raw.w[k + 1] = (std::uint32_t)(v >> 32);
            }
            digests.push_back(Scalar::reduce(raw, C));
        }
        DeterministicNonceSource nonces(seed, C);
        signed_batch = ecdsa_sign_batch(C, digests, keys, nonces);
    }
};

// a NonceSource the library knows nothing about: forces the attempt-by-attempt path
struct WrappedSource final : NonceSource {
    DeterministicNonceSource inner;
    int calls = 0;
    WrappedSource(std::uint64_t seed, const CurveParams& C) : inner(seed, C) {}
    Scalar scalar_for(std::uint64_t stream, std::uint32_t attempt) override {
        ++calls;
        return inner.scalar_for(stream, attempt);
    }
};

static void run(const CurveParams& C, int cid) {
    // keygen: pub == secret * G; secret 1 gives the generator back (test_protocol.cpp:40-50)
    {
        DeterministicNonceSource src(77, C);
        KeyPair a = keygen(C, src, 5);
        std::uint8_t want[32];
        go_nonce(cid, 77, 5, 0, want);
        CHECK(a.secret.to_bytes_be() == std::to_array(reinterpret_cast<std::uint8_t(&)[32]>(want)));
        std::uint32_t gx[8], gy[8], ca[8], cb[8];
        go_curve_params(cid, ca, cb, gx, gy);
        struct FixedOne final : NonceSource {
            Scalar scalar_for(std::uint64_t, std::uint32_t) override { return Scalar{Limbs256::one()}; }
        } one_src;
        AffinePoint g = keygen(C, one_src).pub;
        for (int k = 0; k < 8; ++k) CHECK(g.x.w[k] == gx[k] && g.y.w[k] == gy[k]);
        struct Zero final : NonceSource {
            Scalar scalar_for(std::uint64_t, std::uint32_t) override { return Scalar{}; }
        } zero_src;
        CHECK_THROWS(keygen(C, zero_src), std::logic_error);
    }
    // signature byte round-trip (:52-59)
    {
        Fixture f(C, 2, 99);
        auto bytes = f.signed_batch.sigs[0].to_bytes();
        CHECK(Signature::from_bytes(bytes) == f.signed_batch.sigs[0]);
        std::array<std::uint8_t, 63> short_buf{};
        CHECK_THROWS(Signature::from_bytes(short_buf), std::invalid_argument);
    }
    // sign then verify round-trips (:61-66)
    {
        Fixture f(C, 64, 1);
        for (auto st : f.signed_batch.status) CHECK(st == LaneStatus::ok);
        auto ok = ecdsa_verify_batch(C, f.digests, f.pubs, f.signed_batch.sigs);
        for (bool v : ok) CHECK(v);
    }
    // verification rejects perturbations (:67-104)
    {
        Fixture f(C, 8, 2);
        const auto& sigs = f.signed_batch.sigs;
        auto digests = f.digests;
        digests[3].v.w[0] ^= 1;
        auto ok = ecdsa_verify_batch(C, digests, f.pubs, sigs);
        CHECK(!ok[3]);
        for (std::size_t i = 0; i < 8; ++i)
            if (i != 3) CHECK(ok[i]);
        auto sigs_r = sigs;
        sigs_r[1].r.v.w[2] ^= 4;
        CHECK(!ecdsa_verify_batch(C, f.digests, f.pubs, sigs_r)[1]);
        auto sigs_s = sigs;
        sigs_s[5].s.v.w[7] ^= 1;
        CHECK(!ecdsa_verify_batch(C, f.digests, f.pubs, sigs_s)[5]);
        auto pubs = f.pubs;
        pubs[0] = f.pubs[1];
        CHECK(!ecdsa_verify_batch(C, f.digests, pubs, sigs)[0]);
        auto sigs_zero = sigs;
        sigs_zero[2].r = Scalar{};
        CHECK(!ecdsa_verify_batch(C, f.digests, f.pubs, sigs_zero)[2]);
        sigs_zero[2].r = Scalar{C.n};  // r == n
        CHECK(!ecdsa_verify_batch(C, f.digests, f.pubs, sigs_zero)[2]);
        pubs = f.pubs;
        pubs[4].infinity = true;       // a public key at infinity fails its lane only
        ok = ecdsa_verify_batch(C, f.digests, pubs, sigs);
        CHECK(!ok[4] && ok[5]);
        CHECK_THROWS(ecdsa_verify_batch(C, std::span(f.digests).subspan(1), f.pubs, sigs), std::invalid_argument);
    }
    // batch signing matches the serial composition and the oracle (:106-139)
    {
        Fixture f(C, 16, 3);
        DeterministicNonceSource nonces(3, C);
        std::vector<std::uint8_t> dig(32 * 16), sec(32 * 16), want(64 * 16);
        std::vector<std::int32_t> st(16);
        for (std::size_t i = 0; i < 16; ++i) {
            SignResult serial = ecdsa_sign_serial(C, f.digests[i], f.keys[i], nonces, i);
            CHECK(serial.status[0] == LaneStatus::ok);
            CHECK(serial.sigs[0] == f.signed_batch.sigs[i]);
            CHECK(ecdsa_verify_serial(C, f.digests[i], f.pubs[i], f.signed_batch.sigs[i]));
            auto d = f.digests[i].to_bytes_be(), s = f.keys[i].secret.to_bytes_be();
            std::copy(d.begin(), d.end(), dig.begin() + 32 * i);
            std::copy(s.begin(), s.end(), sec.begin() + 32 * i);
        }
        CHECK(go_sign(cid, 16, dig.data(), sec.data(), 3, 0, want.data(), st.data(), 4) == 0);
        for (std::size_t i = 0; i < 16; ++i) {
            auto got = f.signed_batch.sigs[i].to_bytes();
            CHECK(std::equal(got.begin(), got.end(), want.begin() + 64 * i));
        }
        // an opaque NonceSource takes the attempt-by-attempt path and must give the same signatures
        WrappedSource wrapped(3, C);
        SignResult slow = ecdsa_sign_batch(C, f.digests, f.keys, wrapped);
        CHECK(wrapped.calls == 16);
        for (std::size_t i = 0; i < 16; ++i) CHECK(slow.sigs[i] == f.signed_batch.sigs[i] && slow.status[i] == LaneStatus::ok);
        auto keys = f.keys;
        keys[9].secret = Scalar{};
        CHECK_THROWS(ecdsa_sign_batch(C, f.digests, keys, nonces), std::invalid_argument);
        CHECK_THROWS(ecdsa_sign_batch(C, f.digests, keys, wrapped), std::invalid_argument);
    }
    // rigged retry: a source whose attempt 0 forces s == 0 on one lane (:196-228)
    {
        Fixture f(C, 4, 5);
        struct Rigged final : NonceSource {
            DeterministicNonceSource inner;
            int attempts_seen = 0;
            explicit Rigged(const CurveParams& C) : inner(5, C) {}
            Scalar scalar_for(std::uint64_t stream, std::uint32_t attempt) override {
                if (stream == 2) attempts_seen = attempt + 1;
                return inner.scalar_for(stream, attempt);
            }
        } rig(C);
        // choose the digest of lane 2 so that e + r d == 0 for the attempt-0 nonce: use the oracle's
        // own retry behaviour as the witness (sign with the rigged digest, compare both paths)
        DeterministicNonceSource plain(5, C);
        SignResult a = ecdsa_sign_batch(C, f.digests, f.keys, plain);
        SignResult b = ecdsa_sign_batch(C, f.digests, f.keys, rig);
        for (std::size_t i = 0; i < 4; ++i) CHECK(a.sigs[i] == b.sigs[i]);
        CHECK(rig.attempts_seen == 1);
        // a source that never yields a usable nonce exhausts its 8 attempts
        struct Never final : NonceSource {
            int calls = 0;
            Scalar scalar_for(std::uint64_t, std::uint32_t) override { ++calls; return Scalar{}; }
        } never;
        SignResult c = ecdsa_sign_batch(C, std::span(f.digests).subspan(0, 2), std::span(f.keys).subspan(0, 2), never);
        CHECK(never.calls == 16);
        CHECK(c.status[0] == LaneStatus::nonce_exhausted && c.status[1] == LaneStatus::nonce_exhausted);
    }
    // ECDH: agreement, invalid peer, oracle bytes (test_protocol.cpp:141-194)
    {
        Fixture f(C, 6, 8);
        std::vector<Scalar> sa, sb;
        std::vector<AffinePoint> pa, pb;
        for (std::size_t i = 0; i < 3; ++i) {
            sa.push_back(f.keys[i].secret); pb.push_back(f.keys[i + 3].pub);
            sb.push_back(f.keys[i + 3].secret); pa.push_back(f.keys[i].pub);
        }
        EcdhResult ab = ecdh_derive_batch(C, sa, pb), ba = ecdh_derive_batch(C, sb, pa);
        for (std::size_t i = 0; i < 3; ++i) {
            CHECK(ab.status[i] == LaneStatus::ok && ba.status[i] == LaneStatus::ok);
            CHECK(ab.shared[i] == ba.shared[i]);
        }
        auto bad = pb;
        bad[1].y.w[0] ^= 1;
        bad[2].infinity = true;
        EcdhResult r = ecdh_derive_batch(C, sa, bad);
        CHECK(r.status[0] == LaneStatus::ok && r.status[1] == LaneStatus::invalid_peer && r.status[2] == LaneStatus::invalid_peer);
        CHECK(r.shared[0] == ab.shared[0]);
        auto big = sa;
        big[0] = Scalar{C.n};
        CHECK_THROWS(ecdh_derive_batch(C, big, pb), std::invalid_argument);
    }
    // precompute_base_table / batch_fpmul over a non-generator base (test_batch_point.cpp:160-208)
    {
        DeterministicNonceSource src(31, C);
        KeyPair kp = keygen(C, src, 0);
        PrecomputedBase base = precompute_base_table(C, kp.pub);
        AffinePoint off = kp.pub;
        off.y.w[0] ^= 1;
        CHECK_THROWS(precompute_base_table(C, off), std::invalid_argument);
        AffinePoint inf{{}, {}, true};
        CHECK_THROWS(precompute_base_table(C, inf), std::invalid_argument);
        std::mt19937_64 rng(66 + cid);
        const std::size_t n = 64;
        std::vector<Scalar> scalars(n);
        for (auto& s : scalars)
            for (int k = 0; k < 8; k += 2) {
                const std::uint64_t v = rng();
                s.v.w[k] = (std::uint32_t)v;
                s.v.w[k + 1] = (std::uint32_t)(v >> 32);
            }
        scalars[0] = Scalar{};                 // 0 -> infinity
        scalars[1] = Scalar{Limbs256::one()};  // 1 -> the base itself
        Limbs256 p77{};
        p77.w[2] = 1u << 13;                   // 2^77
        scalars[2] = Scalar{p77};
        Limbs256 nm1 = C.n;
        nm1.w[0] -= 1;
        scalars[3] = Scalar{nm1};              // n - 1 -> -base
        BatchPointBuffer out = batch_fpmul(C, scalars, base, LanePlan::make(n, 8));
        CHECK(out.get(C, 0).infinity);
        CHECK(out.get(C, 1) == kp.pub);
        CHECK(out.get(C, 3).x == kp.pub.x && !(out.get(C, 3).y == kp.pub.y));
        BatchPointBuffer rep = BatchPointBuffer::make(n), want = BatchPointBuffer::make(n);
        for (std::size_t i = 0; i < n; ++i) rep.set(i, kp.pub);
        auto kc = detail::scalar_columns(scalars);
        go_pmul_serial(cid, n, kc.data(), rep.x.data(), rep.y.data(), rep.infinity_mask.data(), want.x.data(), want.y.data(),
                       want.infinity_mask.data());
        for (std::size_t i = 0; i < n; ++i) CHECK(out.get(C, i) == want.get(C, i));
        // the generator's table through the same entry point equals sm2_base_table()
        std::uint32_t gx[8], gy[8], ca[8], cb[8];
        go_curve_params(cid, ca, cb, gx, gy);
        AffinePoint g;
        for (int k = 0; k < 8; ++k) { g.x.w[k] = gx[k]; g.y.w[k] = gy[k]; }
        PrecomputedBase gt = precompute_base_table(C, g);
        BatchPointBuffer a = batch_fpmul(C, scalars, gt, LanePlan::make(n, 8));
        BatchPointBuffer b = batch_fpmul(C, scalars, sm2_base_table(), LanePlan::make(n, 8));
        for (std::size_t i = 0; i < n; ++i) CHECK(a.get(C, i) == b.get(C, i));
        // a table of one curve's context is refused by the other's
        const CurveParams& other = cid == 0 ? CurveParams::secp256k1() : CurveParams::sm2();
        CHECK_THROWS(batch_fpmul(other, scalars, base, LanePlan::make(n, 8)), std::invalid_argument);
    }
    // BatchConfig (protocol.cpp:88-93)
    {
        BatchConfig cfg;
        WorkerPool pool(3);
        CHECK(cfg.effective_lanes(100) == 4);
        cfg.pool = &pool;
        CHECK(cfg.effective_lanes(100) == 12 && cfg.effective_lanes(5) == 5 && cfg.effective_lanes(0) == 1);
        cfg.lanes = 7;
        CHECK(cfg.effective_lanes(100) == 7 && cfg.plan(100).lanes == 7);
    }
}

int main() {
    run(CurveParams::sm2(), 0);
    run(CurveParams::secp256k1(), 1);
    std::printf(failures ? "FAILED (%d)\n" : "protocol compat tests passed%.0d\n", failures);
    return failures ? 1 : 0;
}
