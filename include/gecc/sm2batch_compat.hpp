// C++ mirror of the reference's batch API on top of the C ABI (gecc_b200.h).
//
// Same type and function names, argument meaning and error behaviour as
//   sm2batch/limbs.hpp        Limbs256
//   sm2batch/batch_buffer.hpp BatchColumnBuffer, BitMask           (:15-73)
//   sm2batch/batch_invert.hpp LanePlan, batch_invert               (:29-63)
//   sm2batch/batch_point.hpp  BatchPointBuffer, batch_padd/pdbl/upmul/fpmul (:26-91)
//   sm2batch/curve.hpp        Scalar, CurveParams (as a handle)
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
};

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

struct Scalar {
    Limbs256 v{};
    bool operator==(const Scalar&) const = default;
    bool is_zero() const { return v.is_zero(); }
    unsigned bit(std::size_t i) const { return v.bit(i); }
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

struct FieldParams {  // handle: which field of which engine
    const Engine* engine = nullptr;
    gecc_field which = GECC_FIELD_P;
};

struct CurveParams {
    std::shared_ptr<Engine> engine;
    FieldParams base, order;
    const FieldParams* base_field = nullptr;   // F_q
    const FieldParams* order_field = nullptr;  // F_n

    static const CurveParams& sm2() { return instance(GECC_CURVE_SM2); }
    static const CurveParams& secp256k1() { return instance(GECC_CURVE_SECP256K1); }

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
    field.engine->check(gecc_batch_invert(field.engine->ctx(), field.which, inputs.n, inputs.data(), out.data()),
                        "batch_invert");
    return out;
}

inline BatchPointBuffer batch_padd(const CurveParams& c, const BatchPointBuffer& p, const BatchPointBuffer& t,
                                   const LanePlan& plan, WorkerPool* = nullptr) {
    if (p.n != t.n) throw std::invalid_argument("batch_padd: buffer sizes differ");
    if (plan.total != p.n) throw std::invalid_argument("batch_padd: plan does not match batch");
    BatchPointBuffer out = BatchPointBuffer::make(p.n);
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

struct PrecomputedBase {};  // the table lives on the device, built at context creation
inline const PrecomputedBase& sm2_base_table() {
    static const PrecomputedBase b;
    return b;
}

inline BatchPointBuffer batch_fpmul(const CurveParams& c, std::span<const Scalar> scalars, const PrecomputedBase&,
                                    const LanePlan& plan, WorkerPool* = nullptr) {
    if (plan.total != scalars.size()) throw std::invalid_argument("batch_fpmul: plan does not match batch");
    BatchPointBuffer out = BatchPointBuffer::make(scalars.size());
    auto k = detail::scalar_columns(scalars);
    c.engine->check(gecc_batch_fpmul(c.engine->ctx(), scalars.size(), k.data(), out.x.data(), out.y.data(),
                                     out.infinity_mask.data()),
                    "batch_fpmul");
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

}  // namespace sm2b
