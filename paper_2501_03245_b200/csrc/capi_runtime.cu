// Runtime moduli and user curves: the reference's C++ layer is generic in the modulus
// (FieldParams::make(q), field.cpp:159-179; mont_mul / mod_add / mod_sub / inversion on any odd
// 256-bit q, field.cpp:194-246) and in the curve (CurveParams {base_field, a, b}, curve.hpp:51-59;
// batch_invert / batch_padd / batch_pdbl take them as arguments, batch_invert.hpp:61,
// batch_point.hpp:47-60).  The compiled-in curves of this library fold their constants into
// immediates; here the constants travel as a kernel argument (FieldRT, gecc_field.cuh) and the
// same limb code runs on them: word-serial Montgomery reduction (redc_ws_eo), safegcd inversion,
// Montgomery's trick per thread block, the complete pair classification of batch_padd.
//
//   gecc_field_params_make : FieldParams::make -- R, R^2, R^3 mod q, -q^-1 mod 2^32, the 30-bit
//                            limbs of q for the division steps; even q is rejected
//   gecc_field_op_rt       : mont_mul / mod_add / mod_sub / to_mont / from_mont / inversion
//   gecc_batch_invert_rt   : batch_invert (zero -> zero)
//   gecc_batch_padd_rt / gecc_batch_pdbl_rt : batched affine addition / doubling on
//                            y^2 = x^3 + a x + b over F_q (a in Montgomery form; b is not needed)
#include <cstring>

#include "capi_ctx.h"
#include "gecc_batch.cuh"

using namespace gecc;
using namespace gecc_capi;

static_assert(sizeof(FieldRT) <= sizeof(gecc_field_params), "gecc_field_params holds a FieldRT");

namespace {

// ---------------------------------------------------------------- host: FieldParams::make
struct U256 {
    uint32_t w[8];
};
bool u256_geq(const U256& a, const U256& b) {
    for (int i = 7; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] > b.w[i];
    return true;
}
U256 u256_sub_raw(const U256& a, const U256& b) {
    U256 r;
    uint64_t borrow = 0;
    for (int i = 0; i < 8; ++i) {
        const uint64_t d = (uint64_t)a.w[i] - b.w[i] - borrow;
        r.w[i] = (uint32_t)d;
        borrow = (d >> 32) & 1;
    }
    return r;
}
// 2a mod q for a < q (the reference builds R and R^2 by modular doublings, field.cpp:171-176)
U256 dbl_mod(const U256& a, const U256& q) {
    U256 r;
    uint32_t top = 0;
    for (int i = 0; i < 8; ++i) {
        r.w[i] = (a.w[i] << 1) | top;
        top = a.w[i] >> 31;
    }
    if (top || u256_geq(r, q)) r = u256_sub_raw(r, q);
    return r;
}
// low 256 bits of a * b
U256 mul_low(const U256& a, const U256& b) {
    U256 r{};
    for (int i = 0; i < 8; ++i) {
        uint64_t carry = 0;
        for (int j = 0; i + j < 8; ++j) {
            const uint64_t t = (uint64_t)a.w[i] * b.w[j] + r.w[i + j] + carry;
            r.w[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
    }
    return r;
}

bool make_field_rt(const uint32_t q[8], FieldRT* f) {
    if ((q[0] & 1u) == 0) return false;  // "modulus must be odd" (field.cpp:160)
    bool small = true;                   // q >= 3
    for (int i = 1; i < 8; ++i) small = small && q[i] == 0;
    if (small && q[0] < 3) return false;
    U256 Q;
    memcpy(Q.w, q, 32);
    memset(f, 0, sizeof(*f));
    memcpy(f->q_, q, 32);
    // Newton iteration for q^-1 mod 2^32 (field.cpp:164-167), then mod 2^256
    uint32_t x = q[0];
    for (int i = 0; i < 5; ++i) x *= 2u - q[0] * x;
    f->qinv32 = ~x + 1u;
    f->qinv30_ = x & 0x3FFFFFFFu;
    U256 inv{};
    inv.w[0] = x;
    for (int it = 0; it < 3; ++it) {  // 32 -> 64 -> 128 -> 256 bits
        U256 t = mul_low(Q, inv), two{};
        two.w[0] = 2;
        t = u256_sub_raw(two, t);
        inv = mul_low(inv, t);
    }
    const U256 zero{};
    const U256 ninv = u256_sub_raw(zero, inv);
    memcpy(f->ninv_, ninv.w, 32);
    // R = 2^256 mod q by 256 modular doublings of 1, R^2 and R^3 by 256 more each
    U256 t{};
    t.w[0] = 1;
    for (int i = 0; i < 256; ++i) t = dbl_mod(t, Q);
    memcpy(f->r_, t.w, 32);
    for (int i = 0; i < 256; ++i) t = dbl_mod(t, Q);
    memcpy(f->r2_, t.w, 32);
    for (int i = 0; i < 256; ++i) t = dbl_mod(t, Q);
    memcpy(f->r3_, t.w, 32);
    U256 two{};
    two.w[0] = 2;
    const U256 qm2 = u256_sub_raw(Q, two);
    memcpy(f->qm2_, qm2.w, 32);
    for (int i = 0; i < 9; ++i) {  // 30-bit limbs of q
        const int bit = 30 * i, wi = bit >> 5, sh = bit & 31;
        uint32_t v = q[wi] >> sh;
        if (sh > 2 && wi + 1 < 8) v |= q[wi + 1] << (32 - sh);
        f->q30_[i] = v & 0x3FFFFFFFu;
    }
    return true;
}

// ---------------------------------------------------------------- kernels
__global__ void __launch_bounds__(128) k_field_op_rt(FieldRT f, int op, size_t n, const uint32_t* __restrict__ a,
                                                     const uint32_t* __restrict__ b, uint32_t* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const fe x = col_load<8>(a, n, i);
        const fe y = b ? col_load<8>(b, n, i) : fe_zero();
        fe r;
        switch (op) {
            case 0: r = fe_mul(f, x, y); break;
            case 1: r = fe_add(f, x, y); break;
            case 2: r = fe_sub(f, x, y); break;
            case 3: r = fe_to_mont(f, x); break;
            case 4: r = fe_from_mont(f, x); break;
            case 5: r = fe_inv(f, x); break;
            default: r = fe_is_zero(x) ? x : fe_inv_fermat(f, x); break;
        }
        col_store(out, n, i, r);
    }
}

// Montgomery's trick with one inversion per thread block, COOP_K elements per thread (the form of
// k_batch_invert_coop / k_batch_padd_coop / k_batch_pdbl_coop, on runtime constants)
constexpr int RT_THREADS = 128, RT_K = 4;

__global__ void __launch_bounds__(RT_THREADS)
k_batch_invert_rt(FieldRT f, size_t n, const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
    __shared__ uint32_t sm[2 * 8 * (RT_THREADS / 32)];
    const size_t tile = (size_t)blockIdx.x * (RT_THREADS * RT_K) + threadIdx.x;
    fe lp[RT_K];
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 0; k < RT_K; ++k) {
        const size_t i = tile + (size_t)k * RT_THREADS;
        if (i < n) {
            const fe v = col_load<8>(in, n, i);
            if (!fe_is_zero(v)) acc = fe_mul(f, acc, v);
        }
        lp[k] = acc;
    }
    fe inv = coop_block_inverse<FieldRT, RT_THREADS>(f, acc, sm);
#pragma unroll
    for (int k = RT_K - 1; k >= 0; --k) {
        const size_t i = tile + (size_t)k * RT_THREADS;
        if (i < n) {
            const fe v = col_load<8>(in, n, i);
            const bool zero = fe_is_zero(v);
            const fe r = k > 0 ? fe_mul(f, inv, lp[k > 0 ? k - 1 : 0]) : inv;
            if (!zero && k > 0) inv = fe_mul(f, inv, v);
            col_store(out, n, i, zero ? fe_zero() : r);
        }
    }
}

// classification + denominator of one pair (batch_point.cpp:91-111) on runtime constants
__device__ __forceinline__ uint32_t classify_pair_rt(const FieldRT& f, const fe& px, const fe& py, bool pinf,
                                                     const fe& tx, const fe& ty, bool tinf, fe* d) {
    if (pinf && tinf) return K_INFINITY;
    if (pinf) return K_COPY_RIGHT;
    if (tinf) return K_COPY_LEFT;
    if (fe_eq(px, tx)) {
        if (fe_eq(py, ty) && !fe_is_zero(py)) {
            *d = fe_add(f, py, py);
            return K_TANGENT;
        }
        return K_INFINITY;
    }
    *d = fe_sub(f, px, tx);
    return K_GENERIC;
}
__device__ __forceinline__ void finish_rt(const FieldRT& f, const fe& lam, const fe& x1, const fe& x2, const fe& y1,
                                          fe* xr, fe* yr) {
    *xr = fe_sub(f, fe_sub(f, fe_sqr(f, lam), x1), x2);
    *yr = fe_sub(f, fe_mul(f, lam, fe_sub(f, x1, *xr)), y1);
}
__device__ __forceinline__ fe tangent_rt(const FieldRT& f, const fe& a, const fe& x) {  // 3 x^2 + a
    const fe x2 = fe_sqr(f, x);
    return fe_add(f, fe_add(f, fe_add(f, x2, x2), x2), a);
}

// DOUBLE: t == p (batch_pdbl, batch_point.cpp:175-231)
template <bool DOUBLE>
__global__ void __launch_bounds__(RT_THREADS)
k_batch_padd_rt(FieldRT f, fe a, size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                const uint8_t* __restrict__ pinf, const uint32_t* __restrict__ tx, const uint32_t* __restrict__ ty,
                const uint8_t* __restrict__ tinf, uint32_t* __restrict__ ox, uint32_t* __restrict__ oy,
                uint8_t* __restrict__ oinf) {
    __shared__ uint32_t sm[2 * 8 * (RT_THREADS / 32)];
    const size_t tile = (size_t)blockIdx.x * (RT_THREADS * RT_K) + threadIdx.x;
    fe lp[RT_K];
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 0; k < RT_K; ++k) {
        const size_t i = tile + (size_t)k * RT_THREADS;
        if (i < n) {
            const fe ax = col_load<8>(px, n, i), ay = col_load<8>(py, n, i);
            const fe bx = DOUBLE ? ax : col_load<8>(tx, n, i), by = DOUBLE ? ay : col_load<8>(ty, n, i);
            const bool ai = pinf && pinf[i], bi = DOUBLE ? ai : (tinf && tinf[i]);
            fe d = fe_one(f);
            classify_pair_rt(f, ax, ay, ai, bx, by, bi, &d);
            acc = fe_mul(f, acc, d);
        }
        lp[k] = acc;
    }
    fe inv = coop_block_inverse<FieldRT, RT_THREADS>(f, acc, sm);
#pragma unroll
    for (int k = RT_K - 1; k >= 0; --k) {
        const size_t i = tile + (size_t)k * RT_THREADS;
        if (i < n) {
            const fe ax = col_load<8>(px, n, i), ay = col_load<8>(py, n, i);
            const fe bx = DOUBLE ? ax : col_load<8>(tx, n, i), by = DOUBLE ? ay : col_load<8>(ty, n, i);
            const bool ai = pinf && pinf[i], bi = DOUBLE ? ai : (tinf && tinf[i]);
            fe d = fe_one(f);
            const uint32_t kind = classify_pair_rt(f, ax, ay, ai, bx, by, bi, &d);
            const fe dinv = k > 0 ? fe_mul(f, inv, lp[k > 0 ? k - 1 : 0]) : inv;
            if (k > 0) inv = fe_mul(f, inv, d);
            fe xr = fe_zero(), yr = fe_zero();
            uint8_t rinf = 0;
            if (kind == K_GENERIC) {
                finish_rt(f, fe_mul(f, fe_sub(f, ay, by), dinv), ax, bx, ay, &xr, &yr);
            } else if (kind == K_TANGENT) {
                finish_rt(f, fe_mul(f, tangent_rt(f, a, ax), dinv), ax, ax, ay, &xr, &yr);
            } else if (kind == K_COPY_LEFT || (DOUBLE && kind == K_COPY_RIGHT)) {
                xr = ax; yr = ay;
            } else if (kind == K_COPY_RIGHT) {
                xr = bx; yr = by;
            } else {
                rinf = 1;
            }
            col_store(ox, n, i, xr);
            col_store(oy, n, i, yr);
            oinf[i] = rinf;
        }
    }
}

sm2b_status fail_rt(sm2b_ctx* ctx, const char* what, cudaError_t e) {
    ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return SM2B_ERROR_INTERNAL;
}
#define CUR(ctx, call)                                           \
    do {                                                         \
        cudaError_t e__ = (call);                                \
        if (e__ != cudaSuccess) return fail_rt(ctx, #call, e__); \
    } while (0)

size_t pad256(size_t bytes) { return (bytes + 255) & ~(size_t)255; }
unsigned rt_blocks(size_t n) { return (unsigned)((n + (size_t)RT_THREADS * RT_K - 1) / ((size_t)RT_THREADS * RT_K)); }

const FieldRT* as_rt(const gecc_field_params* p) { return reinterpret_cast<const FieldRT*>(p); }
// a usable parameter block was produced by gecc_field_params_make: q odd, limbs of q mirrored
bool params_ok(const gecc_field_params* p) {
    if (!p) return false;
    const FieldRT* f = as_rt(p);
    return (f->q_[0] & 1u) != 0 && f->q30_[0] == (f->q_[0] & 0x3FFFFFFFu) && f->qinv32 * f->q_[0] == 0xFFFFFFFFu;
}

}  // namespace

extern "C" {

sm2b_status gecc_field_params_make(const uint32_t q[8], gecc_field_params* out) {
    if (!q || !out) return SM2B_ERROR_INVALID_ARGUMENT;
    FieldRT f;
    if (!make_field_rt(q, &f)) return SM2B_ERROR_INVALID_ARGUMENT;
    memset(out, 0, sizeof(*out));
    memcpy(out, &f, sizeof(f));
    return SM2B_OK;
}

sm2b_status gecc_field_params_get(const gecc_field_params* params, int which, uint32_t out[8]) {
    if (!params_ok(params) || !out || which < 0 || which > 3) return SM2B_ERROR_INVALID_ARGUMENT;
    const FieldRT* f = as_rt(params);
    const uint32_t* src = which == 0 ? f->q_ : which == 1 ? f->r_ : which == 2 ? f->r2_ : f->r3_;
    memcpy(out, src, 32);
    return SM2B_OK;
}

sm2b_status gecc_field_op_rt(sm2b_ctx* ctx, const gecc_field_params* params, gecc_field_opcode op, size_t n,
                             const uint32_t* a, const uint32_t* b, uint32_t* out) {
    if (!ctx || is_group(ctx) || !params_ok(params) || (unsigned)op > GECC_OP_MOD_INV_FERMAT || (n > 0 && (!a || !out)) ||
        (n > 0 && op <= GECC_OP_MOD_SUB && !b))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t bytes = 32 * n;
    CUR(ctx, ctx->in.ensure(2 * pad256(bytes)));
    CUR(ctx, ctx->out.ensure(pad256(bytes)));
    uint32_t* da = (uint32_t*)ctx->in.p;
    uint32_t* db = (uint32_t*)((uint8_t*)ctx->in.p + pad256(bytes));
    uint32_t* dout = (uint32_t*)ctx->out.p;
    CUR(ctx, cudaMemcpyAsync(da, a, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (b) CUR(ctx, cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, ctx->stream));
    size_t want = (n + 127) / 128;
    k_field_op_rt<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 128, 0, ctx->stream>>>(*as_rt(params), (int)op, n, da,
                                                                                       b ? db : nullptr, dout);
    CUR(ctx, cudaGetLastError());
    ctx->launches += 1;
    CUR(ctx, cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUR(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

sm2b_status gecc_batch_invert_rt(sm2b_ctx* ctx, const gecc_field_params* params, size_t n, const uint32_t* in,
                                 uint32_t* out) {
    if (!ctx || is_group(ctx) || !params_ok(params) || (n > 0 && (!in || !out))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t bytes = 32 * n;
    CUR(ctx, ctx->in.ensure(pad256(bytes)));
    CUR(ctx, ctx->out.ensure(pad256(bytes)));
    CUR(ctx, cudaMemcpyAsync(ctx->in.p, in, bytes, cudaMemcpyHostToDevice, ctx->stream));
    k_batch_invert_rt<<<rt_blocks(n), RT_THREADS, 0, ctx->stream>>>(*as_rt(params), n, (const uint32_t*)ctx->in.p,
                                                                    (uint32_t*)ctx->out.p);
    CUR(ctx, cudaGetLastError());
    ctx->launches += 1;
    account_invert(ctx, n);
    CUR(ctx, cudaMemcpyAsync(out, ctx->out.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUR(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

static sm2b_status padd_rt(sm2b_ctx* ctx, const gecc_field_params* params, const uint32_t a_mont[8], bool dbl, size_t n,
                           const uint32_t* px, const uint32_t* py, const uint8_t* pinf, const uint32_t* tx,
                           const uint32_t* ty, const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || is_group(ctx) || !params_ok(params) || !a_mont ||
        (n > 0 && (!px || !py || !ox || !oy || !oinf || (!dbl && (!tx || !ty)))))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t cb = pad256(32 * n), mb = pad256(n);
    CUR(ctx, ctx->in.ensure(4 * cb + 2 * mb));
    CUR(ctx, ctx->out.ensure(2 * cb + mb));
    uint8_t* base = (uint8_t*)ctx->in.p;
    uint32_t *dpx = (uint32_t*)base, *dpy = (uint32_t*)(base + cb), *dtx = (uint32_t*)(base + 2 * cb),
             *dty = (uint32_t*)(base + 3 * cb);
    uint8_t *dpi = base + 4 * cb, *dti = base + 4 * cb + mb;
    uint8_t* ob = (uint8_t*)ctx->out.p;
    uint32_t *dox = (uint32_t*)ob, *doy = (uint32_t*)(ob + cb);
    uint8_t* doi = ob + 2 * cb;
    cudaStream_t s = ctx->stream;
    CUR(ctx, cudaMemcpyAsync(dpx, px, 32 * n, cudaMemcpyHostToDevice, s));
    CUR(ctx, cudaMemcpyAsync(dpy, py, 32 * n, cudaMemcpyHostToDevice, s));
    if (pinf) CUR(ctx, cudaMemcpyAsync(dpi, pinf, n, cudaMemcpyHostToDevice, s));
    if (!dbl) {
        CUR(ctx, cudaMemcpyAsync(dtx, tx, 32 * n, cudaMemcpyHostToDevice, s));
        CUR(ctx, cudaMemcpyAsync(dty, ty, 32 * n, cudaMemcpyHostToDevice, s));
        if (tinf) CUR(ctx, cudaMemcpyAsync(dti, tinf, n, cudaMemcpyHostToDevice, s));
    }
    fe a;
    memcpy(a.w, a_mont, 32);
    if (dbl)
        k_batch_padd_rt<true><<<rt_blocks(n), RT_THREADS, 0, s>>>(*as_rt(params), a, n, dpx, dpy, pinf ? dpi : nullptr, nullptr,
                                                                  nullptr, nullptr, dox, doy, doi);
    else
        k_batch_padd_rt<false><<<rt_blocks(n), RT_THREADS, 0, s>>>(*as_rt(params), a, n, dpx, dpy, pinf ? dpi : nullptr, dtx, dty,
                                                                   tinf ? dti : nullptr, dox, doy, doi);
    CUR(ctx, cudaGetLastError());
    ctx->launches += 1;
    account_points(ctx, dbl ? OP_PDBL : OP_PADD, n);
    CUR(ctx, cudaMemcpyAsync(ox, dox, 32 * n, cudaMemcpyDeviceToHost, s));
    CUR(ctx, cudaMemcpyAsync(oy, doy, 32 * n, cudaMemcpyDeviceToHost, s));
    CUR(ctx, cudaMemcpyAsync(oinf, doi, n, cudaMemcpyDeviceToHost, s));
    CUR(ctx, cudaStreamSynchronize(s));
    return SM2B_OK;
}

sm2b_status gecc_batch_padd_rt(sm2b_ctx* ctx, const gecc_field_params* params, const uint32_t a_mont[8], size_t n,
                               const uint32_t* px, const uint32_t* py, const uint8_t* pinf, const uint32_t* tx,
                               const uint32_t* ty, const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    return padd_rt(ctx, params, a_mont, false, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf);
}

sm2b_status gecc_batch_pdbl_rt(sm2b_ctx* ctx, const gecc_field_params* params, const uint32_t a_mont[8], size_t n,
                               const uint32_t* px, const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                               uint8_t* oinf) {
    return padd_rt(ctx, params, a_mont, true, n, px, py, pinf, nullptr, nullptr, nullptr, ox, oy, oinf);
}

}  // extern "C"
