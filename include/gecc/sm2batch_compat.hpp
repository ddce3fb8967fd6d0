// C++ mirror of the reference's batch API on top of the C ABI (gecc_b200.h).
//
// Same type and function names, argument meaning and error behaviour as
//   sm2batch/limbs.hpp        Limbs256
//   sm2batch/batch_buffer.hpp BatchColumnBuffer, BitMask           (:15-73)
//   sm2batch/batch_invert.hpp LanePlan, batch_invert               (:29-63)
//   sm2batch/batch_point.hpp  BatchPointBuffer, batch_padd/pdbl/upmul/fpmul (:26-91)
//   sm2batch/curve.hpp        Scalar, CurveParams (as a handle)
//   sm2batch/protocol.hpp     KeyPair, Signature, NonceSource, DeterministicNonceSource,
//                             SystemNonceSource, LaneStatus, BatchConfig, keygen,
//                             ecdsa_sign_batch / verify_batch, ecdh_derive_batch, *_serial (:14-124)
// so code written against the reference's C++ layer recompiles against this header
// and runs on the GPU.  Differences, all deliberate:
//   * CurveParams / FieldParams are handles onto an engine context (the constants
//     live on the device); CurveParams::sm2() and ::secp256k1() are provided.
//   * LanePlan and WorkerPool are accepted and ignored: results do not depend on the
//     lane count (batch_invert.hpp:59-60) and the CUDA grid replaces the pool.
//   * errors: size / plan mismatches throw std::invalid_argument exactly as the
//     reference (batch_point.cpp:71-74, batch_invert.cpp:94-95); a device failure
//     throws std::runtime_error with gecc_last_error().
// Header-only; link with -lgecc_b200.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../gecc_b200.h"

namespace sm2b {

struct Limbs256 {
    std::array<std::uint32_t, 8> w{};
    constexpr bool operator==(const Limbs256&) const = default;
    static constexpr Limbs256 zero() { return {}; }
    constexpr bool is_zero() const {
        std::uint32_t acc = 0;
        for (std::uint32_t x : w) acc |= x;
        return acc == 0;
    }
    constexpr unsigned bit(std::size_t i) const { return (w[i / 32] >> (i % 32)) & 1u; }
    static constexpr Limbs256 one() {
        Limbs256 v{};
        v.w[0] = 1;
        return v;
    }
};

// 32 big-endian bytes <-> limbs (limbs.cpp:5-27)
inline Limbs256 from_bytes_be(std::span<const std::uint8_t> b) {
    if (b.size() != 32) throw std::invalid_argument("from_bytes_be: expected 32 bytes");
    Limbs256 v;
    for (std::size_t i = 0; i < 8; ++i) {
        const std::uint8_t* s = b.data() + 4 * (7 - i);
        v.w[i] = (std::uint32_t(s[0]) << 24) | (std::uint32_t(s[1]) << 16) | (std::uint32_t(s[2]) << 8) | s[3];
    }
    return v;
}
inline std::array<std::uint8_t, 32> to_bytes_be(const Limbs256& v) {
    std::array<std::uint8_t, 32> out;
    for (std::size_t i = 0; i < 8; ++i) {
        std::uint8_t* d = out.data() + 4 * (7 - i);
        d[0] = std::uint8_t(v.w[i] >> 24);
        d[1] = std::uint8_t(v.w[i] >> 16);
        d[2] = std::uint8_t(v.w[i] >> 8);
        d[3] = std::uint8_t(v.w[i]);
    }
    return out;
}
// a < b as unsigned 256-bit integers (limbs.hpp:115-122)
inline bool less_than(const Limbs256& a, const Limbs256& b) {
    for (std::size_t i = 8; i-- > 0;)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
    return false;
}

// One flat allocation per buffer: column k is the slice [k*n, (k+1)*n), which is the
// layout the device consumes directly (no transposition on the way to the GPU).
struct BatchColumnBuffer {
    std::size_t n = 0;
    std::vector<std::uint32_t> cols;  // 8 * n words

    static BatchColumnBuffer make(std::size_t n) {
        BatchColumnBuffer b;
        b.n = n;
        b.cols.assign(8 * n, 0);
        return b;
    }
    Limbs256 get(std::size_t i) const {
        Limbs256 v;
        for (std::size_t k = 0; k < 8; ++k) v.w[k] = cols[k * n + i];
        return v;
    }
    void set(std::size_t i, const Limbs256& v) {
        for (std::size_t k = 0; k < 8; ++k) cols[k * n + i] = v.w[k];
    }
    const std::uint32_t* data() const { return cols.data(); }
    std::uint32_t* data() { return cols.data(); }
};

// one byte per element instead of packed bits: what the device entry points take
class BitMask {
public:
    BitMask() = default;
    explicit BitMask(std::size_t n) : bits_(n, 0) {}
    std::size_t size() const { return bits_.size(); }
    bool get(std::size_t i) const { return bits_[i] != 0; }
    void set(std::size_t i, bool v) { bits_[i] = v ? 1 : 0; }
    bool any() const {
        for (std::uint8_t b : bits_)
            if (b) return true;
        return false;
    }
    bool operator==(const BitMask&) const = default;
    const std::uint8_t* data() const { return bits_.data(); }
    std::uint8_t* data() { return bits_.data(); }

private:
    std::vector<std::uint8_t> bits_;
};

struct LanePlan {
    std::size_t total = 0;
    std::size_t lanes = 0;
    static LanePlan make(std::size_t total, std::size_t lanes) {  // batch_invert.cpp:8-29
        LanePlan p;
        p.total = total;
        p.lanes = total == 0 ? 0 : (lanes == 0 ? 1 : (lanes > total ? total : lanes));
        return p;
    }
};
class WorkerPool {  // accepted for source compatibility; the GPU grid does the work
public:
    explicit WorkerPool(unsigned workers) : workers_(workers ? workers : 1) {}
    unsigned workers() const { return workers_; }

private:
    unsigned workers_;
};

struct CurveParams;
struct Scalar {
    Limbs256 v{};
    bool operator==(const Scalar&) const = default;
    bool is_zero() const { return v.is_zero(); }
    unsigned bit(std::size_t i) const { return v.bit(i); }
    // curve.cpp:22-38 with the group order of `c` (the reference hard-wires SM2's n; the
    // one-argument forms below keep that meaning)
    static Scalar reduce(const Limbs256& raw, const CurveParams& c);
    static Scalar checked(const Limbs256& raw, const CurveParams& c);
    static Scalar reduce(const Limbs256& raw);
    static Scalar checked(const Limbs256& raw);
    static Scalar from_bytes_be(std::span<const std::uint8_t> bytes) { return reduce(sm2b::from_bytes_be(bytes)); }
    std::array<std::uint8_t, 32> to_bytes_be() const { return sm2b::to_bytes_be(v); }
};

class Engine {  // RAII owner of one sm2b_ctx
public:
    explicit Engine(gecc_curve curve, int device = -1) : ctx_(gecc_ctx_new(curve, device)) {
        if (!ctx_) throw std::runtime_error("gecc_ctx_new failed: no usable CUDA device (no CPU path)");
    }
    ~Engine() { sm2b_ctx_free(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    sm2b_ctx* ctx() const { return ctx_; }
    void check(sm2b_status st, const char* what) const {
        if (st == SM2B_OK) return;
        if (st == SM2B_ERROR_INTERNAL) throw std::runtime_error(std::string(what) + ": " + gecc_last_error(ctx_));
        throw std::invalid_argument(std::string(what) + ": " + sm2b_status_str(st));
    }

private:
    sm2b_ctx* ctx_;
};

using MontElement = Limbs256;  // a field element in Montgomery form (field.hpp)

struct FieldParams {  // handle: which field of which engine, or a runtime modulus (make)
    const Engine* engine = nullptr;
    gecc_field which = GECC_FIELD_P;
    // runtime modulus: FieldParams::make(q) (field.hpp / field.cpp:159-179).  The constants travel
    // with every call (gecc_*_rt); `engine` only names the device that runs it.
    std::shared_ptr<gecc_field_params> runtime;
    Limbs256 q{}, r{}, r2{};

    static FieldParams make(const Limbs256& modulus, const Engine* on = nullptr) {
        FieldParams f;
        f.runtime = std::make_shared<gecc_field_params>();
        if (gecc_field_params_make(modulus.w.data(), f.runtime.get()) != SM2B_OK)
            throw std::invalid_argument("modulus must be odd");  // field.cpp:160
        f.engine = on;
        f.q = modulus;
        gecc_field_params_get(f.runtime.get(), 1, f.r.w.data());
        gecc_field_params_get(f.runtime.get(), 2, f.r2.w.data());
        return f;
    }
    bool is_runtime() const { return runtime != nullptr; }
};

struct CurveParams {
    std::shared_ptr<Engine> engine;
    FieldParams base, order;
    const FieldParams* base_field = nullptr;   // F_q
    const FieldParams* order_field = nullptr;  // F_n
    gecc_curve id = GECC_CURVE_SM2;
    Limbs256 n{};                               // group order (plain integer)

    static const CurveParams& sm2() { return instance(GECC_CURVE_SM2); }
    static const CurveParams& secp256k1() { return instance(GECC_CURVE_SECP256K1); }

    // A user curve y^2 = x^3 + a x + b over F_q (curve.hpp:51-59: CurveParams is a plain aggregate
    // of a base field and the Montgomery-form coefficients).  batch_invert / batch_padd /
    // batch_pdbl serve it through the runtime-modulus kernels on the device of `like`'s engine;
    // the fixed-base, ECDSA and MSM layers need a compiled-in curve.
    MontElement a{}, b{};
    bool custom = false;
    static CurveParams user(const FieldParams& base_field_rt, const Limbs256& a_mont, const Limbs256& b_mont,
                            const CurveParams& like = sm2()) {
        if (!base_field_rt.is_runtime()) throw std::invalid_argument("CurveParams::user needs FieldParams::make(q)");
        CurveParams c;
        c.engine = like.engine;
        c.base = base_field_rt;
        c.base.engine = c.engine.get();
        c.order = c.base;
        c.base_field = c.order_field = nullptr;  // (the object is copied by value: use field())
        c.a = a_mont;
        c.b = b_mont;
        c.custom = true;
        return c;
    }
    const FieldParams& field() const { return base; }

private:
    static const CurveParams& instance(gecc_curve id) {
        static std::unique_ptr<CurveParams> inst[2];
        if (!inst[id]) {
            auto c = std::make_unique<CurveParams>();
            c->engine = std::make_shared<Engine>(id);
            c->base = {c->engine.get(), GECC_FIELD_P};
            c->order = {c->engine.get(), GECC_FIELD_N};
            c->base_field = &c->base;
            c->order_field = &c->order;
            c->id = id;
            // group orders: SM2 (GB/T 32918) and secp256k1 (SEC 2), least significant limb first
            static constexpr std::uint32_t kOrder[2][8] = {
                {0x39D54123u, 0x53BBF409u, 0x21C6052Bu, 0x7203DF6Bu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFEu},
                {0xD0364141u, 0xBFD25E8Cu, 0xAF48A03Bu, 0xBAAEDCE6u, 0xFFFFFFFEu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}};
            for (int k = 0; k < 8; ++k) c->n.w[k] = kOrder[id][k];
            inst[id] = std::move(c);
        }
        return *inst[id];
    }
};

struct AffinePoint {
    Limbs256 x, y;  // Montgomery form
    bool infinity = false;
    bool operator==(const AffinePoint& o) const {
        if (infinity || o.infinity) return infinity == o.infinity;
        return x == o.x && y == o.y;
    }
};

struct BatchPointBuffer {
    std::size_t n = 0;
    BatchColumnBuffer x, y;
    BitMask infinity_mask;

    static BatchPointBuffer make(std::size_t n) {
        BatchPointBuffer b;
        b.n = n;
        b.x = BatchColumnBuffer::make(n);
        b.y = BatchColumnBuffer::make(n);
        b.infinity_mask = BitMask(n);
        return b;
    }
    AffinePoint get(const CurveParams&, std::size_t i) const {
        return {x.get(i), y.get(i), infinity_mask.get(i)};
    }
    void set(std::size_t i, const AffinePoint& p) {  // batch_point.cpp:41-47
        x.set(i, p.infinity ? Limbs256::zero() : p.x);
        y.set(i, p.infinity ? Limbs256::zero() : p.y);
        infinity_mask.set(i, p.infinity);
    }
};

inline BatchColumnBuffer batch_invert(const BatchColumnBuffer& inputs, const FieldParams& field,
                                      const LanePlan& plan, WorkerPool* = nullptr) {
    if (plan.total != inputs.n) throw std::invalid_argument("batch_invert: plan does not match batch size");
    BatchColumnBuffer out = BatchColumnBuffer::make(inputs.n);
    if (field.is_runtime()) {
        const Engine* e = field.engine ? field.engine : CurveParams::sm2().engine.get();
        e->check(gecc_batch_invert_rt(e->ctx(), field.runtime.get(), inputs.n, inputs.data(), out.data()), "batch_invert");
        return out;
    }
    field.engine->check(gecc_batch_invert(field.engine->ctx(), field.which, inputs.n, inputs.data(), out.data()),
                        "batch_invert");
    return out;
}

inline BatchPointBuffer batch_padd(const CurveParams& c, const BatchPointBuffer& p, const BatchPointBuffer& t,
                                   const LanePlan& plan, WorkerPool* = nullptr) {
    if (p.n != t.n) throw std::invalid_argument("batch_padd: buffer sizes differ");
    if (plan.total != p.n) throw std::invalid_argument("batch_padd: plan does not match batch");
    BatchPointBuffer out = BatchPointBuffer::make(p.n);
    if (c.custom) {
        c.engine->check(gecc_batch_padd_rt(c.engine->ctx(), c.base.runtime.get(), c.a.w.data(), p.n, p.x.data(), p.y.data(),
                                           p.infinity_mask.data(), t.x.data(), t.y.data(), t.infinity_mask.data(),
                                           out.x.data(), out.y.data(), out.infinity_mask.data()),
                        "batch_padd");
        return out;
    }
    c.engine->check(gecc_batch_padd(c.engine->ctx(), p.n, p.x.data(), p.y.data(), p.infinity_mask.data(), t.x.data(),
                                    t.y.data(), t.infinity_mask.data(), out.x.data(), out.y.data(),
                                    out.infinity_mask.data()),
                    "batch_padd");
    return out;
}

inline BatchPointBuffer batch_pdbl(const CurveParams& c, const BatchPointBuffer& p, const LanePlan& plan,
                                   WorkerPool* = nullptr) {
    if (plan.total != p.n) throw std::invalid_argument("batch_pdbl: plan does not match batch");
    BatchPointBuffer out = BatchPointBuffer::make(p.n);
    if (c.custom) {
        c.engine->check(gecc_batch_pdbl_rt(c.engine->ctx(), c.base.runtime.get(), c.a.w.data(), p.n, p.x.data(), p.y.data(),
                                           p.infinity_mask.data(), out.x.data(), out.y.data(), out.infinity_mask.data()),
                        "batch_pdbl");
        return out;
    }
    c.engine->check(gecc_batch_pdbl(c.engine->ctx(), p.n, p.x.data(), p.y.data(), p.infinity_mask.data(),
                                    out.x.data(), out.y.data(), out.infinity_mask.data()),
                    "batch_pdbl");
    return out;
}

namespace detail {
inline std::vector<std::uint32_t> scalar_columns(std::span<const Scalar> s) {
    const std::size_t n = s.size();
    std::vector<std::uint32_t> cols(8 * n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t k = 0; k < 8; ++k) cols[k * n + i] = s[i].v.w[k];
    return cols;
}
}  // namespace detail

inline BatchPointBuffer batch_upmul(const CurveParams& c, std::span<const Scalar> scalars,
                                    const BatchPointBuffer& points, const LanePlan& plan, WorkerPool* = nullptr) {
    if (scalars.size() != points.n) throw std::invalid_argument("batch_upmul: scalar count mismatch");
    if (plan.total != points.n) throw std::invalid_argument("batch_upmul: plan does not match batch");
    BatchPointBuffer out = BatchPointBuffer::make(points.n);
    auto k = detail::scalar_columns(scalars);
    c.engine->check(gecc_batch_upmul(c.engine->ctx(), points.n, k.data(), points.x.data(), points.y.data(),
                                     points.infinity_mask.data(), out.x.data(), out.y.data(),
                                     out.infinity_mask.data()),
                    "batch_upmul");
    return out;
}

inline Scalar Scalar::reduce(const Limbs256& raw, const CurveParams& c) {  // one conditional subtraction
    if (less_than(raw, c.n)) return Scalar{raw};
    Limbs256 d;
    std::uint64_t borrow = 0;
    for (std::size_t i = 0; i < 8; ++i) {
        const std::uint64_t t = std::uint64_t(raw.w[i]) - c.n.w[i] - borrow;
        d.w[i] = std::uint32_t(t);
        borrow = (t >> 32) & 1u;
    }
    return Scalar{d};
}
inline Scalar Scalar::checked(const Limbs256& raw, const CurveParams& c) {
    if (!less_than(raw, c.n)) throw std::out_of_range("Scalar::checked: value not below the group order");
    return Scalar{raw};
}
inline Scalar Scalar::reduce(const Limbs256& raw) { return reduce(raw, CurveParams::sm2()); }
inline Scalar Scalar::checked(const Limbs256& raw) { return checked(raw, CurveParams::sm2()); }

// precompute_base_table (batch_point.hpp:76-83): a device-resident windowed table of an arbitrary
// on-curve point; the default-constructed value stands for the curve generator's table, which
// every context builds at creation (sm2_base_table()).
struct PrecomputedBase {
    std::shared_ptr<Engine> engine;          // context the table lives on
    std::shared_ptr<gecc_base_table> table;  // null: the generator
};
inline PrecomputedBase precompute_base_table(const CurveParams& c, const AffinePoint& g) {
    if (g.infinity) throw std::invalid_argument("precompute_base_table: point off curve");
    gecc_base_table* t = nullptr;
    const sm2b_status st = gecc_base_table_new(c.engine->ctx(), g.x.w.data(), g.y.w.data(), &t);
    if (st == SM2B_ERROR_MALFORMED_INPUT)  // batch_point.cpp:343-344
        throw std::invalid_argument("precompute_base_table: point off curve");
    c.engine->check(st, "precompute_base_table");
    return PrecomputedBase{c.engine, std::shared_ptr<gecc_base_table>(t, gecc_base_table_free)};
}
inline const PrecomputedBase& sm2_base_table() {
    static const PrecomputedBase b;
    return b;
}

inline BatchPointBuffer batch_fpmul(const CurveParams& c, std::span<const Scalar> scalars, const PrecomputedBase& base,
                                    const LanePlan& plan, WorkerPool* = nullptr) {
    if (plan.total != scalars.size()) throw std::invalid_argument("batch_fpmul: plan does not match batch");
    if (base.table && base.engine != c.engine)
        throw std::invalid_argument("batch_fpmul: the base table belongs to another curve context");
    BatchPointBuffer out = BatchPointBuffer::make(scalars.size());
    auto k = detail::scalar_columns(scalars);
    const sm2b_status st =
        base.table ? gecc_batch_fpmul_base(c.engine->ctx(), base.table.get(), scalars.size(), k.data(), out.x.data(),
                                           out.y.data(), out.infinity_mask.data())
                   : gecc_batch_fpmul(c.engine->ctx(), scalars.size(), k.data(), out.x.data(), out.y.data(),
                                      out.infinity_mask.data());
    c.engine->check(st, "batch_fpmul");
    return out;
}

// MSM entry point (no reference counterpart): sum_i scalars[i] * points[i]
inline AffinePoint msm(const CurveParams& c, std::span<const Scalar> scalars, const BatchPointBuffer& points) {
    if (scalars.size() != points.n) throw std::invalid_argument("msm: scalar count mismatch");
    auto k = detail::scalar_columns(scalars);
    AffinePoint r;
    std::uint8_t inf = 0;
    c.engine->check(gecc_msm(c.engine->ctx(), points.n, k.data(), points.x.data(), points.y.data(),
                             points.infinity_mask.data(), r.x.w.data(), r.y.w.data(), &inf),
                    "msm");
    r.infinity = inf != 0;
    return r;
}

// =========================================================================== protocol layer
// sm2batch/protocol.hpp:14-124 over the C ABI.  Digests arrive as scalars already reduced mod n;
// signatures are raw r || s.  The GPU kernels work on wire records (32 / 65 / 64 bytes), so this
// layer encodes scalars big-endian and takes points out of Montgomery form with one batched
// from_mont on the device.
struct KeyPair {
    Scalar secret;    // nonzero, < n
    AffinePoint pub;  // secret * G
};

struct Signature {
    Scalar r;
    Scalar s;
    bool operator==(const Signature&) const = default;
    std::array<std::uint8_t, 64> to_bytes() const {
        std::array<std::uint8_t, 64> out;
        const auto rb = r.to_bytes_be(), sb = s.to_bytes_be();
        std::copy(rb.begin(), rb.end(), out.begin());
        std::copy(sb.begin(), sb.end(), out.begin() + 32);
        return out;
    }
    static Signature from_bytes(std::span<const std::uint8_t> bytes) {  // raw values kept, verification rejects them
        if (bytes.size() != 64) throw std::invalid_argument("Signature::from_bytes: expected 64 bytes");
        Signature sig;
        sig.r.v = sm2b::from_bytes_be(bytes.subspan(0, 32));
        sig.s.v = sm2b::from_bytes_be(bytes.subspan(32, 32));
        return sig;
    }
};

class NonceSource {
public:
    virtual ~NonceSource() = default;
    virtual Scalar scalar_for(std::uint64_t stream, std::uint32_t attempt) = 0;
};

namespace detail {
inline std::uint64_t splitmix(std::uint64_t& x) {  // protocol.cpp:13-19
    x += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline Scalar draw_scalar(std::uint64_t state, const Limbs256& n) {  // protocol.cpp:21-34: reject 0 and >= n
    for (;;) {
        Limbs256 raw;
        for (std::size_t i = 0; i < 8; i += 2) {
            const std::uint64_t v = splitmix(state);
            raw.w[i] = std::uint32_t(v);
            raw.w[i + 1] = std::uint32_t(v >> 32);
        }
        if (!raw.is_zero() && less_than(raw, n)) return Scalar{raw};
    }
}
inline bool scalar_in_range(const Scalar& s, const Limbs256& n) { return !s.is_zero() && less_than(s.v, n); }
}  // namespace detail

// Pure function of (seed, stream, attempt) (protocol.cpp:67-75).  The curve argument selects the
// group order the draw is rejected against (the reference is SM2-only).
class DeterministicNonceSource final : public NonceSource {
public:
    explicit DeterministicNonceSource(std::uint64_t seed, const CurveParams& c = CurveParams::sm2())
        : seed_(seed), n_(c.n), curve_(c.id) {}
    Scalar scalar_for(std::uint64_t stream, std::uint32_t attempt) override {
        std::uint64_t state = seed_;
        (void)detail::splitmix(state);
        state ^= 0xA3EC647659359ACDull * (stream + 1);
        (void)detail::splitmix(state);
        state ^= 0xC2B2AE3D27D4EB4Full * (std::uint64_t(attempt) + 1);
        return detail::draw_scalar(state, n_);
    }
    std::uint64_t seed() const { return seed_; }
    gecc_curve curve() const { return curve_; }

private:
    std::uint64_t seed_;
    Limbs256 n_;
    gecc_curve curve_;
};

class SystemNonceSource final : public NonceSource {  // protocol.cpp:77-86
public:
    explicit SystemNonceSource(const CurveParams& c = CurveParams::sm2()) : n_(c.n) {
        std::random_device rd;
        base_[0] = (std::uint64_t(rd()) << 32) | rd();
        base_[1] = (std::uint64_t(rd()) << 32) | rd();
    }
    Scalar scalar_for(std::uint64_t, std::uint32_t) override {
        std::uint64_t state = base_[0] ^ (base_[1] + ++counter_ * 0x9E3779B97F4A7C15ull);
        return detail::draw_scalar(state, n_);
    }

private:
    std::uint64_t base_[2];
    std::uint64_t counter_ = 0;
    Limbs256 n_;
};

enum class LaneStatus : std::uint8_t { ok = 0, nonce_exhausted, invalid_peer, degenerate_result };

struct BatchConfig {  // accepted for source compatibility: lane counts do not change results
    std::size_t lanes = 0;
    WorkerPool* pool = nullptr;
    std::size_t effective_lanes(std::size_t n) const {  // protocol.cpp:88-93
        if (lanes != 0) return lanes;
        const std::size_t w = pool ? pool->workers() : 1, l = w * 4;
        return l < n ? l : (n == 0 ? 1 : n);
    }
    LanePlan plan(std::size_t n) const { return LanePlan::make(n, effective_lanes(n)); }
};

namespace detail {
inline LaneStatus lane_status_of(std::int32_t st) {
    switch (st) {
        case SM2B_OK: return LaneStatus::ok;
        case SM2B_ERROR_NONCE_EXHAUSTED: return LaneStatus::nonce_exhausted;
        case SM2B_ERROR_INVALID_PEER: return LaneStatus::invalid_peer;
        case SM2B_ERROR_DEGENERATE: return LaneStatus::degenerate_result;
    }
    throw std::runtime_error("unexpected lane status " + std::to_string(st));
}
inline std::vector<std::uint8_t> scalar_records(std::span<const Scalar> s) {
    std::vector<std::uint8_t> out(32 * s.size());
    for (std::size_t i = 0; i < s.size(); ++i) {
        const auto b = s[i].to_bytes_be();
        std::copy(b.begin(), b.end(), out.begin() + 32 * i);
    }
    return out;
}
// Montgomery-form affine points -> 65-byte records 0x04 || X || Y (curve.cpp:192-201): one batched
// from_mont per coordinate on the device.  A point at infinity has no uncompressed encoding; it
// becomes a record with tag 0x00, which every consumer rejects exactly where the reference does.
inline std::vector<std::uint8_t> point_records(const CurveParams& c, std::span<const AffinePoint> pts) {
    const std::size_t n = pts.size();
    std::vector<std::uint8_t> out(65 * n, 0);
    if (n == 0) return out;
    BatchColumnBuffer x = BatchColumnBuffer::make(n), y = BatchColumnBuffer::make(n);
    for (std::size_t i = 0; i < n; ++i) {
        x.set(i, pts[i].x);
        y.set(i, pts[i].y);
    }
    BatchColumnBuffer px = BatchColumnBuffer::make(n), py = BatchColumnBuffer::make(n);
    c.engine->check(gecc_field_op(c.engine->ctx(), GECC_FIELD_P, GECC_OP_FROM_MONT, n, x.data(), nullptr, px.data()), "from_mont");
    c.engine->check(gecc_field_op(c.engine->ctx(), GECC_FIELD_P, GECC_OP_FROM_MONT, n, y.data(), nullptr, py.data()), "from_mont");
    for (std::size_t i = 0; i < n; ++i) {
        if (pts[i].infinity) continue;
        out[65 * i] = 0x04;
        const auto xb = sm2b::to_bytes_be(px.get(i)), yb = sm2b::to_bytes_be(py.get(i));
        std::copy(xb.begin(), xb.end(), out.begin() + 65 * i + 1);
        std::copy(yb.begin(), yb.end(), out.begin() + 65 * i + 33);
    }
    return out;
}
}  // namespace detail

// keygen (protocol.cpp:95-100): d = nonces(stream, 0), pub = d * G
inline KeyPair keygen(const CurveParams& c, NonceSource& nonces, std::uint64_t stream = 0) {
    const Scalar d = nonces.scalar_for(stream, 0);
    if (!detail::scalar_in_range(d, c.n)) throw std::logic_error("keygen: nonce source broke its contract");
    const Scalar one[1] = {d};
    const BatchPointBuffer p = batch_fpmul(c, one, sm2_base_table(), LanePlan::make(1, 1));
    return {d, p.get(c, 0)};
}

struct SignResult {
    std::vector<Signature> sigs;  // valid where status[i] == ok
    std::vector<LaneStatus> status;
};

// ecdsa_sign_batch (protocol.cpp:106-168).  With the library's DeterministicNonceSource the whole
// call -- nonce derivation, R = k G, both inversions, up to 8 retries per lane -- is ONE fused GPU
// kernel (sm2b_sign's path, stream id = lane index).  Any other NonceSource is driven exactly as
// the reference drives it: attempt by attempt, nonces.scalar_for(lane, attempt) for the lanes
// still pending, one gecc_sign_nonces call per attempt.
// A secret outside (0, n) fails the call with std::invalid_argument (the reference's C ABI rule,
// capi.cpp:181-184; its C++ layer computes garbage there).
inline SignResult ecdsa_sign_batch(const CurveParams& c, std::span<const Scalar> digests,
                                   std::span<const KeyPair> keys, NonceSource& nonces, const BatchConfig& = {}) {
    if (digests.size() != keys.size()) throw std::invalid_argument("ecdsa_sign_batch: length mismatch");
    const std::size_t n = digests.size();
    SignResult out;
    out.sigs.resize(n);
    out.status.assign(n, LaneStatus::ok);
    if (n == 0) return out;
    std::vector<Scalar> secrets(n);
    for (std::size_t i = 0; i < n; ++i) secrets[i] = keys[i].secret;
    const auto dig = detail::scalar_records(digests), sec = detail::scalar_records(secrets);
    std::vector<std::uint8_t> sig(64 * n);
    std::vector<std::int32_t> st(n);
    auto* det = dynamic_cast<DeterministicNonceSource*>(&nonces);
    if (det && det->curve() == c.id && det->seed() != 0) {
        const sm2b_status rc = gecc_sign(c.engine->ctx(), n, dig.data(), sec.data(), det->seed(), 0, sig.data(), st.data());
        if (rc == SM2B_ERROR_MALFORMED_INPUT) throw std::invalid_argument("ecdsa_sign_batch: secret outside (0, n)");
        c.engine->check(rc, "ecdsa_sign_batch");
        for (std::size_t i = 0; i < n; ++i) {
            out.status[i] = detail::lane_status_of(st[i]);
            if (st[i] == SM2B_OK) out.sigs[i] = Signature::from_bytes(std::span<const std::uint8_t>(sig.data() + 64 * i, 64));
        }
        return out;
    }
    std::vector<std::size_t> pending(n);
    for (std::size_t i = 0; i < n; ++i) pending[i] = i;
    for (std::uint32_t attempt = 0; attempt < 8 && !pending.empty(); ++attempt) {  // protocol.cpp:121
        const std::size_t m = pending.size();
        std::vector<std::uint8_t> d(32 * m), s(32 * m), k(32 * m), sg(64 * m);
        std::vector<std::int32_t> ls(m);
        for (std::size_t i = 0; i < m; ++i) {
            const std::size_t lane = pending[i];
            std::copy(dig.begin() + 32 * lane, dig.begin() + 32 * lane + 32, d.begin() + 32 * i);
            std::copy(sec.begin() + 32 * lane, sec.begin() + 32 * lane + 32, s.begin() + 32 * i);
            const auto kb = nonces.scalar_for(lane, attempt).to_bytes_be();
            std::copy(kb.begin(), kb.end(), k.begin() + 32 * i);
        }
        const sm2b_status rc = gecc_sign_nonces(c.engine->ctx(), m, d.data(), s.data(), k.data(), sg.data(), ls.data());
        if (rc == SM2B_ERROR_MALFORMED_INPUT) throw std::invalid_argument("ecdsa_sign_batch: secret outside (0, n)");
        c.engine->check(rc, "ecdsa_sign_batch");
        std::vector<std::size_t> retry;
        for (std::size_t i = 0; i < m; ++i) {
            if (ls[i] == SM2B_OK) out.sigs[pending[i]] = Signature::from_bytes(std::span<const std::uint8_t>(sg.data() + 64 * i, 64));
            else retry.push_back(pending[i]);
        }
        pending.swap(retry);
    }
    for (std::size_t lane : pending) out.status[lane] = LaneStatus::nonce_exhausted;
    return out;
}

// ecdsa_verify_batch (protocol.cpp:170-222): range rules, w = s^-1, u1 G + u2 Q, x mod n == r --
// one fused GPU kernel per batch.  A public key at infinity or off the curve fails its lane.
inline std::vector<bool> ecdsa_verify_batch(const CurveParams& c, std::span<const Scalar> digests,
                                            std::span<const AffinePoint> publics, std::span<const Signature> sigs,
                                            const BatchConfig& = {}) {
    if (digests.size() != publics.size() || digests.size() != sigs.size())
        throw std::invalid_argument("ecdsa_verify_batch: length mismatch");
    const std::size_t n = digests.size();
    std::vector<bool> ok(n, false);
    if (n == 0) return ok;
    const auto dig = detail::scalar_records(digests);
    const auto pub = detail::point_records(c, publics);
    std::vector<std::uint8_t> sg(64 * n), res(n);
    for (std::size_t i = 0; i < n; ++i) {
        const auto b = sigs[i].to_bytes();
        std::copy(b.begin(), b.end(), sg.begin() + 64 * i);
    }
    c.engine->check(sm2b_verify(c.engine->ctx(), n, dig.data(), pub.data(), sg.data(), res.data()), "ecdsa_verify_batch");
    for (std::size_t i = 0; i < n; ++i) ok[i] = res[i] != 0;
    return ok;
}

struct EcdhResult {
    std::vector<std::array<std::uint8_t, 32>> shared;  // x-coordinate bytes
    std::vector<LaneStatus> status;
};

// ecdh_derive_batch (protocol.cpp:224-263): peers validated per lane; shared[j] = x(secrets[j] * peers[j])
inline EcdhResult ecdh_derive_batch(const CurveParams& c, std::span<const Scalar> secrets,
                                    std::span<const AffinePoint> peers, const BatchConfig& = {}) {
    if (secrets.size() != peers.size()) throw std::invalid_argument("ecdh_derive_batch: length mismatch");
    const std::size_t n = secrets.size();
    EcdhResult out;
    out.shared.assign(n, {});
    out.status.assign(n, LaneStatus::ok);
    if (n == 0) return out;
    const auto sec = detail::scalar_records(secrets);
    const auto pr = detail::point_records(c, peers);
    std::vector<std::uint8_t> sh(32 * n);
    std::vector<std::int32_t> st(n);
    const sm2b_status rc = sm2b_ecdh(c.engine->ctx(), n, sec.data(), pr.data(), sh.data(), st.data());
    if (rc == SM2B_ERROR_MALFORMED_INPUT) throw std::invalid_argument("ecdh_derive_batch: secret not below n");
    c.engine->check(rc, "ecdh_derive_batch");
    for (std::size_t i = 0; i < n; ++i) {
        out.status[i] = detail::lane_status_of(st[i]);
        if (st[i] == SM2B_OK) std::copy(sh.begin() + 32 * i, sh.begin() + 32 * i + 32, out.shared[i].begin());
    }
    return out;
}

// Single-lane compositions (protocol.cpp:265-306): the same kernels on a batch of one, with the
// lane's nonce stream passed explicitly.
inline SignResult ecdsa_sign_serial(const CurveParams& c, const Scalar& digest, const KeyPair& key, NonceSource& nonces,
                                    std::uint64_t stream) {
    SignResult out;
    out.sigs.resize(1);
    out.status.assign(1, LaneStatus::nonce_exhausted);
    const auto d = digest.to_bytes_be(), s = key.secret.to_bytes_be();
    for (std::uint32_t attempt = 0; attempt < 8; ++attempt) {
        const auto k = nonces.scalar_for(stream, attempt).to_bytes_be();
        std::uint8_t sg[64];
        std::int32_t ls = 0;
        const sm2b_status rc = gecc_sign_nonces(c.engine->ctx(), 1, d.data(), s.data(), k.data(), sg, &ls);
        if (rc == SM2B_ERROR_MALFORMED_INPUT) throw std::invalid_argument("ecdsa_sign_serial: secret outside (0, n)");
        c.engine->check(rc, "ecdsa_sign_serial");
        if (ls != SM2B_OK) continue;
        out.sigs[0] = Signature::from_bytes(std::span<const std::uint8_t>(sg, 64));
        out.status[0] = LaneStatus::ok;
        break;
    }
    return out;
}
inline bool ecdsa_verify_serial(const CurveParams& c, const Scalar& digest, const AffinePoint& pub, const Signature& sig) {
    const Scalar d[1] = {digest};
    const AffinePoint p[1] = {pub};
    const Signature s[1] = {sig};
    return ecdsa_verify_batch(c, d, p, s)[0];
}

}  // namespace sm2b
