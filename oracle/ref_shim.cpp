// TEST INFRASTRUCTURE ONLY -- never linked into, or called from, the product.
//
// Thin C symbols over the *unmodified* reference C++ batch API so that Python
// (ctypes) tests and bench.py's CPU arm can drive the real reference kernels.
// This file is compiled together with /root/reference/proj/src/*.cpp into
// oracle/_ref/libgecc_ref.so by oracle/Makefile; nothing of the reference is
// copied into this repository.
//
// What it adds on top of the reference:
//   * a curve selector: curve 0 = CurveParams::sm2() (curve.cpp:44-56),
//     curve 1 = a hand-built secp256k1 CurveParams made with
//     FieldParams::make (field.cpp:159-179).  The reference point kernels are
//     generic in q, so they run unmodified on it.
//   * flat column-major ("SoA") array arguments: limb k of element i lives at
//     cols[k*n + i] -- the same layout as BatchColumnBuffer
//     (batch_buffer.hpp:15-35), flattened.
//   * ref_ecdsa_sign / ref_ecdsa_verify: the protocol glue of
//     protocol.cpp:106-222 with n and the G table parameterised (the reference
//     hard-wires SM2 there: curve.cpp:23,30, protocol.cpp:23,43,130,211).  All
//     heavy lifting still goes through the reference's own batch_fpmul,
//     batch_upmul, batch_padd and batch_invert.  For curve 0 the outputs are
//     checked equal to sm2b_sign / sm2b_verify in tests/test_oracle_ref.py.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "sm2batch/batch_invert.hpp"
#include "sm2batch/batch_point.hpp"
#include "sm2batch/curve.hpp"
#include "sm2batch/field.hpp"
#include "sm2batch/protocol.hpp"
#include "sm2batch/worker_pool.hpp"

using namespace sm2b;

namespace {

struct CurveBundle {
    FieldParams fp, fn;
    CurveParams c;
    PrecomputedBase table;
};

Limbs256 L(std::initializer_list<std::uint32_t> msw_first) {
    Limbs256 r;
    std::size_t i = 8;
    for (std::uint32_t w : msw_first) r.w[--i] = w;
    return r;
}

const CurveBundle& secp256k1() {
    static const std::unique_ptr<CurveBundle> b = [] {
        auto p = std::make_unique<CurveBundle>();
        p->fp = FieldParams::make(L({0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu,
                                     0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFEu, 0xFFFFFC2Fu}));
        p->fn = FieldParams::make(L({0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFEu,
                                     0xBAAEDCE6u, 0xAF48A03Bu, 0xBFD25E8Cu, 0xD0364141u}));
        p->c.base_field = &p->fp;
        p->c.order_field = &p->fn;
        p->c.a = to_mont(Limbs256::zero(), p->fp);
        p->c.b = to_mont(L({0, 0, 0, 0, 0, 0, 0, 7}), p->fp);
        p->c.generator = {
            to_mont(L({0x79BE667Eu, 0xF9DCBBACu, 0x55A06295u, 0xCE870B07u,
                       0x029BFCDBu, 0x2DCE28D9u, 0x59F2815Bu, 0x16F81798u}), p->fp),
            to_mont(L({0x483ADA77u, 0x26A3C465u, 0x5DA4FBFCu, 0x0E1108A8u,
                       0xFD17B448u, 0xA6855419u, 0x9C47D08Fu, 0xFB10D4B8u}), p->fp),
            false};
        p->table = precompute_base_table(p->c, p->c.generator);
        return p;
    }();
    return *b;
}

const CurveParams& curve(int id) { return id == 0 ? CurveParams::sm2() : secp256k1().c; }
const PrecomputedBase& gtable(int id) { return id == 0 ? sm2_base_table() : secp256k1().table; }
const FieldParams& field(int id, int which) {
    const CurveParams& c = curve(id);
    return which == 0 ? *c.base_field : *c.order_field;
}

Limbs256 col_get(const std::uint32_t* cols, std::size_t n, std::size_t i) {
    Limbs256 v;
    for (std::size_t k = 0; k < 8; ++k) v.w[k] = cols[k * n + i];
    return v;
}
void col_set(std::uint32_t* cols, std::size_t n, std::size_t i, const Limbs256& v) {
    for (std::size_t k = 0; k < 8; ++k) cols[k * n + i] = v.w[k];
}

BatchColumnBuffer to_buf(const std::uint32_t* cols, std::size_t n) {
    BatchColumnBuffer b = BatchColumnBuffer::make(n);
    for (std::size_t k = 0; k < 8; ++k)
        std::memcpy(b.columns[k].data(), cols + k * n, 4 * n);
    return b;
}
void from_buf(const BatchColumnBuffer& b, std::uint32_t* cols) {
    for (std::size_t k = 0; k < 8; ++k)
        std::memcpy(cols + k * b.n, b.columns[k].data(), 4 * b.n);
}

BatchPointBuffer to_pts(const std::uint32_t* x, const std::uint32_t* y,
                        const std::uint8_t* inf, std::size_t n) {
    BatchPointBuffer b = BatchPointBuffer::make(n);
    b.x = to_buf(x, n);
    b.y = to_buf(y, n);
    for (std::size_t i = 0; i < n; ++i) b.infinity_mask.set(i, inf && inf[i]);
    return b;
}
void from_pts(const BatchPointBuffer& b, std::uint32_t* x, std::uint32_t* y,
              std::uint8_t* inf) {
    from_buf(b.x, x);
    from_buf(b.y, y);
    for (std::size_t i = 0; i < b.n; ++i) inf[i] = b.infinity_mask.get(i) ? 1 : 0;
}

std::vector<Scalar> to_scalars(const std::uint32_t* cols, std::size_t n) {
    std::vector<Scalar> s(n);
    for (std::size_t i = 0; i < n; ++i) s[i].v = col_get(cols, n, i);
    return s;
}

struct Pool {
    std::unique_ptr<WorkerPool> pool;
    explicit Pool(unsigned workers) {
        unsigned w = workers ? workers : std::max(1u, std::thread::hardware_concurrency());
        if (w > 1) pool = std::make_unique<WorkerPool>(w);
    }
    unsigned workers() const { return pool ? pool->workers() : 1; }
    std::size_t lanes(std::size_t n, std::size_t want) const {
        return BatchConfig{want, pool.get()}.effective_lanes(n);
    }
};

bool less_than(const Limbs256& a, const Limbs256& b) {
    return compare(a, b) == std::strong_ordering::less;
}
Limbs256 reduce_once(const Limbs256& v, const Limbs256& n) {
    return less_than(v, n) ? v : sub_with_borrow(v, n).diff;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 2;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (...) {
        return 7;
    }
}

}  // namespace

extern "C" {

// q[8], r[8], r2[8] LSW first; returns q_inv.
std::uint32_t ref_field_params(int curve_id, int which, std::uint32_t* q,
                               std::uint32_t* r, std::uint32_t* r2) {
    const FieldParams& f = field(curve_id, which);
    for (int k = 0; k < 8; ++k) {
        q[k] = f.q.w[k];
        r[k] = f.r.w[k];
        r2[k] = f.r2.w[k];
    }
    return f.q_inv;
}

// a_mont[8], b_mont[8], gx_mont[8], gy_mont[8]
void ref_curve_params(int curve_id, std::uint32_t* a, std::uint32_t* b,
                      std::uint32_t* gx, std::uint32_t* gy) {
    const CurveParams& c = curve(curve_id);
    for (int k = 0; k < 8; ++k) {
        a[k] = c.a.value.w[k];
        b[k] = c.b.value.w[k];
        gx[k] = c.generator.x.value.w[k];
        gy[k] = c.generator.y.value.w[k];
    }
}

// op: 0 mont_mul, 1 mod_add, 2 mod_sub, 3 to_mont (b ignored), 4 from_mont,
//     5 mod_inv_fermat (zero input -> zero output, flagged by return count)
int ref_field_op(int curve_id, int which, int op, std::size_t n,
                 const std::uint32_t* a, const std::uint32_t* b, std::uint32_t* out) {
    const FieldParams& f = field(curve_id, which);
    return guarded([&] {
        for (std::size_t i = 0; i < n; ++i) {
            Limbs256 x = col_get(a, n, i);
            Limbs256 y = b ? col_get(b, n, i) : Limbs256::zero();
            Limbs256 r;
            switch (op) {
                case 0: r = mont_mul({x, &f}, {y, &f}).value; break;
                case 1: r = mod_add({x, &f}, {y, &f}).value; break;
                case 2: r = mod_sub({x, &f}, {y, &f}).value; break;
                case 3: r = to_mont(x, f).value; break;
                case 4: r = from_mont({x, &f}); break;
                case 5: r = x.is_zero() ? x : mod_inv_fermat({x, &f}).value; break;
                default: throw std::invalid_argument("op");
            }
            col_set(out, n, i, r);
        }
    });
}

// c[16 limbs per element, column-major over 16 columns] -> reduce
int ref_mont_reduce(int curve_id, int which, int sm2_route, std::size_t n,
                    const std::uint32_t* c16, std::uint32_t* out) {
    const FieldParams& f = field(curve_id, which);
    return guarded([&] {
        for (std::size_t i = 0; i < n; ++i) {
            Limbs512 c;
            for (std::size_t k = 0; k < 16; ++k) c.w[k] = c16[k * n + i];
            Limbs256 r = sm2_route ? mont_reduce_sm2(c) : mont_reduce_generic(c, f);
            col_set(out, n, i, r);
        }
    });
}

int ref_batch_invert(int curve_id, int which, std::size_t n, const std::uint32_t* in,
                     std::uint32_t* out, std::size_t lanes, unsigned workers) {
    return guarded([&] {
        Pool pool(workers);
        BatchColumnBuffer r = batch_invert(to_buf(in, n), field(curve_id, which),
                                           LanePlan::make(n, pool.lanes(n, lanes)),
                                           pool.pool.get());
        from_buf(r, out);
    });
}

int ref_batch_padd(int curve_id, std::size_t n, const std::uint32_t* px,
                   const std::uint32_t* py, const std::uint8_t* pinf,
                   const std::uint32_t* tx, const std::uint32_t* ty,
                   const std::uint8_t* tinf, std::uint32_t* ox, std::uint32_t* oy,
                   std::uint8_t* oinf, std::size_t lanes, unsigned workers) {
    return guarded([&] {
        Pool pool(workers);
        BatchPointBuffer r = batch_padd(curve(curve_id), to_pts(px, py, pinf, n),
                                        to_pts(tx, ty, tinf, n),
                                        LanePlan::make(n, pool.lanes(n, lanes)),
                                        pool.pool.get());
        from_pts(r, ox, oy, oinf);
    });
}

// Timing entry for the CPU baseline: buffers are converted once outside the
// timed region, then batch_padd runs `repeats` times; *seconds = median run
// (bench.cpp:262-281 protocol, minus its generators).
int ref_batch_padd_timed(int curve_id, std::size_t n, const std::uint32_t* px,
                         const std::uint32_t* py, const std::uint32_t* tx,
                         const std::uint32_t* ty, std::size_t lanes, unsigned workers,
                         unsigned repeats, double* seconds) {
    return guarded([&] {
        Pool pool(workers);
        BatchPointBuffer p = to_pts(px, py, nullptr, n), t = to_pts(tx, ty, nullptr, n);
        LanePlan plan = LanePlan::make(n, pool.lanes(n, lanes));
        std::vector<double> times;
        (void)batch_padd(curve(curve_id), p, t, plan, pool.pool.get());
        for (unsigned r = 0; r < repeats; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            (void)batch_padd(curve(curve_id), p, t, plan, pool.pool.get());
            times.push_back(std::chrono::duration<double>(
                                std::chrono::steady_clock::now() - t0).count());
        }
        std::sort(times.begin(), times.end());
        *seconds = times[times.size() / 2];
    });
}

int ref_batch_pdbl(int curve_id, std::size_t n, const std::uint32_t* px,
                   const std::uint32_t* py, const std::uint8_t* pinf, std::uint32_t* ox,
                   std::uint32_t* oy, std::uint8_t* oinf, std::size_t lanes,
                   unsigned workers) {
    return guarded([&] {
        Pool pool(workers);
        BatchPointBuffer r = batch_pdbl(curve(curve_id), to_pts(px, py, pinf, n),
                                        LanePlan::make(n, pool.lanes(n, lanes)),
                                        pool.pool.get());
        from_pts(r, ox, oy, oinf);
    });
}

// scalars: plain (non-Montgomery) 256-bit values, column-major.
int ref_batch_fpmul(int curve_id, std::size_t n, const std::uint32_t* scalars,
                    std::uint32_t* ox, std::uint32_t* oy, std::uint8_t* oinf,
                    std::size_t lanes, unsigned workers) {
    return guarded([&] {
        Pool pool(workers);
        BatchPointBuffer r = batch_fpmul(curve(curve_id), to_scalars(scalars, n),
                                         gtable(curve_id),
                                         LanePlan::make(n, pool.lanes(n, lanes)),
                                         pool.pool.get());
        from_pts(r, ox, oy, oinf);
    });
}

int ref_batch_upmul(int curve_id, std::size_t n, const std::uint32_t* scalars,
                    const std::uint32_t* px, const std::uint32_t* py,
                    const std::uint8_t* pinf, std::uint32_t* ox, std::uint32_t* oy,
                    std::uint8_t* oinf, std::size_t lanes, unsigned workers) {
    return guarded([&] {
        Pool pool(workers);
        BatchPointBuffer r = batch_upmul(curve(curve_id), to_scalars(scalars, n),
                                         to_pts(px, py, pinf, n),
                                         LanePlan::make(n, pool.lanes(n, lanes)),
                                         pool.pool.get());
        from_pts(r, ox, oy, oinf);
    });
}

// Serial ground truth (curve.cpp:176-185), one lane at a time.
int ref_pmul_serial(int curve_id, std::size_t n, const std::uint32_t* scalars,
                    const std::uint32_t* px, const std::uint32_t* py,
                    const std::uint8_t* pinf, std::uint32_t* ox, std::uint32_t* oy,
                    std::uint8_t* oinf) {
    return guarded([&] {
        const CurveParams& c = curve(curve_id);
        BatchPointBuffer in = to_pts(px, py, pinf, n);
        BatchPointBuffer out = BatchPointBuffer::make(n);
        for (std::size_t i = 0; i < n; ++i) {
            Scalar s{col_get(scalars, n, i)};
            out.set(i, pmul_serial(c, s, in.get(c, i)));
        }
        from_pts(out, ox, oy, oinf);
    });
}

// (seed, stream, attempt) -> 32 big-endian bytes. curve 0 uses the reference
// source directly (protocol.cpp:67-75); other curves restate draw_scalar
// (protocol.cpp:22-34) against their own n.
void ref_nonce(int curve_id, std::uint64_t seed, std::uint64_t stream,
               std::uint32_t attempt, std::uint8_t* out32);

// ECDSA with byte records, semantics of sm2b_sign / sm2b_verify (capi.cpp:171-228)
// for any curve id.  status codes are sm2b_status values.
int ref_ecdsa_sign(int curve_id, std::size_t count, const std::uint8_t* digests,
                   const std::uint8_t* secrets, std::uint64_t nonce_seed,
                   std::uint64_t lane_base, std::uint8_t* signatures,
                   std::int32_t* lane_status, std::size_t lanes, unsigned workers);
int ref_ecdsa_verify(int curve_id, std::size_t count, const std::uint8_t* digests,
                     const std::uint8_t* publics, const std::uint8_t* signatures,
                     std::uint8_t* results, std::size_t lanes, unsigned workers);
int ref_keygen(int curve_id, std::uint64_t seed, std::uint64_t lane_base,
               std::size_t count, std::uint8_t* secrets, std::uint8_t* publics,
               std::size_t lanes, unsigned workers);
int ref_ecdh(int curve_id, std::size_t count, const std::uint8_t* secrets,
             const std::uint8_t* peers, std::uint8_t* shared,
             std::int32_t* lane_status, std::size_t lanes, unsigned workers);

}  // extern "C"

namespace {

std::uint64_t splitmix_step(std::uint64_t& x) {  // protocol.cpp:13-19
    x += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

Scalar nonce_for(int curve_id, std::uint64_t seed, std::uint64_t stream,
                 std::uint32_t attempt) {
    if (curve_id == 0) return DeterministicNonceSource(seed).scalar_for(stream, attempt);
    const Limbs256& n = field(curve_id, 1).q;
    std::uint64_t state = seed;  // protocol.cpp:67-75
    (void)splitmix_step(state);
    state ^= 0xA3EC647659359ACDull * (stream + 1);
    (void)splitmix_step(state);
    state ^= 0xC2B2AE3D27D4EB4Full * (attempt + 1);
    for (;;) {  // protocol.cpp:22-34
        Limbs256 raw;
        for (std::size_t i = 0; i < 8; i += 2) {
            std::uint64_t v = splitmix_step(state);
            raw.w[i] = static_cast<std::uint32_t>(v);
            raw.w[i + 1] = static_cast<std::uint32_t>(v >> 32);
        }
        if (!raw.is_zero() && less_than(raw, n)) return Scalar{raw};
    }
}

AffinePoint decode_or_throw(const CurveParams& c, const std::uint8_t* p65) {
    return decode_point(c, {p65, 65});  // curve.cpp:203-217, generic in c
}

}  // namespace

extern "C" {

void ref_nonce(int curve_id, std::uint64_t seed, std::uint64_t stream,
               std::uint32_t attempt, std::uint8_t* out32) {
    auto b = to_bytes_be(nonce_for(curve_id, seed, stream, attempt).v);
    std::memcpy(out32, b.data(), 32);
}

int ref_keygen(int curve_id, std::uint64_t seed, std::uint64_t lane_base,
               std::size_t count, std::uint8_t* secrets, std::uint8_t* publics,
               std::size_t lanes, unsigned workers) {
    return guarded([&] {  // capi.cpp:145-169
        const CurveParams& c = curve(curve_id);
        Pool pool(workers);
        std::vector<Scalar> ds;
        for (std::size_t i = 0; i < count; ++i)
            ds.push_back(nonce_for(curve_id, seed, lane_base + i, 0));
        auto pubs = transpose_from_columns(
            c, batch_fpmul(c, ds, gtable(curve_id),
                           LanePlan::make(count, pool.lanes(count, lanes)),
                           pool.pool.get()));
        for (std::size_t i = 0; i < count; ++i) {
            auto sb = to_bytes_be(ds[i].v);
            std::memcpy(secrets + 32 * i, sb.data(), 32);
            auto pb = encode_point(pubs[i]);
            std::memcpy(publics + 65 * i, pb.data(), 65);
        }
    });
}

int ref_ecdsa_sign(int curve_id, std::size_t count, const std::uint8_t* digests,
                   const std::uint8_t* secrets, std::uint64_t nonce_seed,
                   std::uint64_t lane_base, std::uint8_t* signatures,
                   std::int32_t* lane_status, std::size_t lanes, unsigned workers) {
    int first_fail = 0;
    int rc = guarded([&] {
        const CurveParams& c = curve(curve_id);
        const FieldParams& nf = *c.order_field;
        Pool pool(workers);
        // capi.cpp:179-186: digests reduced, secrets checked (whole call fails)
        std::vector<Limbs256> es(count), ds(count);
        for (std::size_t i = 0; i < count; ++i) {
            es[i] = reduce_once(from_bytes_be({digests + 32 * i, 32}), nf.q);
            ds[i] = from_bytes_be({secrets + 32 * i, 32});
            if (!less_than(ds[i], nf.q)) throw std::out_of_range("secret >= n");
            if (ds[i].is_zero()) throw std::invalid_argument("zero secret");
        }
        std::vector<int> status(count, 0);
        std::vector<Limbs256> rs(count), ss(count);
        std::vector<std::size_t> pending(count);
        for (std::size_t i = 0; i < count; ++i) pending[i] = i;
        // protocol.cpp:121-164
        for (std::uint32_t attempt = 0; attempt < 8 && !pending.empty(); ++attempt) {
            const std::size_t m = pending.size();
            std::vector<Scalar> ks;
            for (std::size_t idx : pending)
                ks.push_back(nonce_for(curve_id, nonce_seed, lane_base + idx, attempt));
            LanePlan plan = LanePlan::make(m, pool.lanes(m, lanes));
            BatchPointBuffer rpts = batch_fpmul(c, ks, gtable(curve_id), plan, pool.pool.get());
            BatchColumnBuffer kbuf = BatchColumnBuffer::make(m);
            for (std::size_t i = 0; i < m; ++i) kbuf.set(i, to_mont(ks[i].v, nf).value);
            BatchColumnBuffer kinv = batch_invert(kbuf, nf, plan, pool.pool.get());
            std::vector<std::size_t> retry;
            for (std::size_t i = 0; i < m; ++i) {
                const std::size_t lane = pending[i];
                AffinePoint rp = rpts.get(c, i);
                if (rp.infinity) { retry.push_back(lane); continue; }
                Limbs256 r = reduce_once(from_mont(rp.x), nf.q);
                if (r.is_zero()) { retry.push_back(lane); continue; }
                MontElement e_m = to_mont(es[lane], nf);
                MontElement r_m = to_mont(r, nf);
                MontElement d_m = to_mont(ds[lane], nf);
                MontElement kinv_m{kinv.get(i), &nf};
                Limbs256 s = from_mont(mont_mul(kinv_m, mod_add(e_m, mont_mul(r_m, d_m))));
                if (s.is_zero()) { retry.push_back(lane); continue; }
                rs[lane] = r;
                ss[lane] = s;
            }
            pending.swap(retry);
        }
        for (std::size_t lane : pending) status[lane] = 5;  // nonce exhausted
        std::memset(signatures, 0, 64 * count);
        for (std::size_t i = 0; i < count; ++i) {
            if (lane_status) lane_status[i] = status[i];
            if (status[i] != 0) {
                if (!first_fail) first_fail = status[i];
                continue;
            }
            auto rb = to_bytes_be(rs[i]);
            auto sb = to_bytes_be(ss[i]);
            std::memcpy(signatures + 64 * i, rb.data(), 32);
            std::memcpy(signatures + 64 * i + 32, sb.data(), 32);
        }
    });
    if (rc != 0) return rc;
    return lane_status ? 0 : first_fail;
}

int ref_ecdsa_verify(int curve_id, std::size_t count, const std::uint8_t* digests,
                     const std::uint8_t* publics, const std::uint8_t* signatures,
                     std::uint8_t* results, std::size_t lanes, unsigned workers) {
    return guarded([&] {
        const CurveParams& c = curve(curve_id);
        const FieldParams& nf = *c.order_field;
        Pool pool(workers);
        std::memset(results, 0, count);
        // capi.cpp:207-222 + protocol.cpp:184-190
        std::vector<std::size_t> live;
        std::vector<Limbs256> es, rs, sv;
        std::vector<AffinePoint> pubs;
        auto in_range = [&](const Limbs256& v) { return !v.is_zero() && less_than(v, nf.q); };
        for (std::size_t i = 0; i < count; ++i) {
            Limbs256 r = from_bytes_be({signatures + 64 * i, 32});
            Limbs256 s = from_bytes_be({signatures + 64 * i + 32, 32});
            AffinePoint q;
            try {
                q = decode_or_throw(c, publics + 65 * i);
            } catch (const std::invalid_argument&) {
                continue;
            }
            if (!in_range(r) || !in_range(s) || q.infinity) continue;
            live.push_back(i);
            es.push_back(reduce_once(from_bytes_be({digests + 32 * i, 32}), nf.q));
            rs.push_back(r);
            sv.push_back(s);
            pubs.push_back(q);
        }
        if (live.empty()) return;
        const std::size_t m = live.size();
        LanePlan plan = LanePlan::make(m, pool.lanes(m, lanes));
        // protocol.cpp:194-214
        BatchColumnBuffer sbuf = BatchColumnBuffer::make(m);
        for (std::size_t i = 0; i < m; ++i) sbuf.set(i, to_mont(sv[i], nf).value);
        BatchColumnBuffer w = batch_invert(sbuf, nf, plan, pool.pool.get());
        std::vector<Scalar> u1(m), u2(m);
        for (std::size_t i = 0; i < m; ++i) {
            MontElement w_m{w.get(i), &nf};
            u1[i].v = from_mont(mont_mul(to_mont(es[i], nf), w_m));
            u2[i].v = from_mont(mont_mul(to_mont(rs[i], nf), w_m));
        }
        BatchPointBuffer a = batch_fpmul(c, u1, gtable(curve_id), plan, pool.pool.get());
        BatchPointBuffer b = batch_upmul(c, u2, transpose_to_columns(c, pubs), plan, pool.pool.get());
        BatchPointBuffer rp = batch_padd(c, a, b, plan, pool.pool.get());
        for (std::size_t i = 0; i < m; ++i) {  // protocol.cpp:216-220
            AffinePoint p = rp.get(c, i);
            if (p.infinity) continue;
            results[live[i]] = reduce_once(from_mont(p.x), nf.q) == rs[i] ? 1 : 0;
        }
    });
}

int ref_ecdh(int curve_id, std::size_t count, const std::uint8_t* secrets,
             const std::uint8_t* peers, std::uint8_t* shared,
             std::int32_t* lane_status, std::size_t lanes, unsigned workers) {
    int first_fail = 0;
    int rc = guarded([&] {  // capi.cpp:230-261 + protocol.cpp:224-263
        const CurveParams& c = curve(curve_id);
        const FieldParams& nf = *c.order_field;
        Pool pool(workers);
        std::vector<int> status(count, 0);
        std::vector<std::size_t> live;
        std::vector<Scalar> ds;
        std::vector<AffinePoint> ps;
        for (std::size_t i = 0; i < count; ++i) {
            Limbs256 d = from_bytes_be({secrets + 32 * i, 32});
            if (!less_than(d, nf.q)) throw std::out_of_range("secret >= n");
            try {
                AffinePoint p = decode_or_throw(c, peers + 65 * i);
                if (p.infinity) { status[i] = 3; continue; }
                live.push_back(i);
                ds.push_back(Scalar{d});
                ps.push_back(p);
            } catch (const std::invalid_argument&) {
                status[i] = 3;
            }
        }
        std::memset(shared, 0, 32 * count);
        if (!live.empty()) {
            const std::size_t m = live.size();
            BatchPointBuffer prod = batch_upmul(c, ds, transpose_to_columns(c, ps),
                                                LanePlan::make(m, pool.lanes(m, lanes)),
                                                pool.pool.get());
            for (std::size_t i = 0; i < m; ++i) {
                AffinePoint p = prod.get(c, i);
                if (p.infinity) { status[live[i]] = 4; continue; }
                auto xb = to_bytes_be(from_mont(p.x));
                std::memcpy(shared + 32 * live[i], xb.data(), 32);
            }
        }
        for (std::size_t i = 0; i < count; ++i) {
            if (lane_status) lane_status[i] = status[i];
            if (status[i] && !first_fail) first_fail = status[i];
        }
    });
    if (rc != 0) return rc;
    return lane_status ? 0 : first_fail;
}

}  // extern "C"
