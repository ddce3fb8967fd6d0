// C ABI of libgecc_b200.so (include/gecc_b200.h).  Host side of the drop-in
// boundary: mirrors the reference's capi.cpp semantics (argument checks, status
// codes, per-lane reporting, ledger) and hands all arithmetic to CUDA kernels.
// There is no CPU compute path in this file.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/gecc_b200.h"
#include "gecc_host.h"

using namespace gecc;

// grow-only device allocation
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes + bytes / 8 + 256;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct sm2b_ctx {
    int curve = CURVE_SM2;
    int device = 0;
    int sm_count = 148;
    uint32_t workers = 0, lanes = 0;
    std::mutex mu;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    sm2b_op_counts ledger{0, 0, 0, 0};
    uint64_t launches = 0;
    std::string last_error;
    DevBuf in, out, scratch;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

sm2b_status fail(sm2b_ctx* ctx, const char* what, cudaError_t e) {
    ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return SM2B_ERROR_INTERNAL;
}
sm2b_status fail_msg(sm2b_ctx* ctx, const char* what) {
    ctx->last_error = what;
    return SM2B_ERROR_INTERNAL;
}

#define CU(ctx, call)                                        \
    do {                                                     \
        cudaError_t e__ = (call);                            \
        if (e__ != cudaSuccess) return fail(ctx, #call, e__); \
    } while (0)

// carve `count` sub-buffers out of one arena; sizes rounded to 256 B
struct Carver {
    uint8_t* base;
    size_t off = 0;
    explicit Carver(void* p) : base((uint8_t*)p) {}
    template <class T>
    T* take(size_t elems) {
        T* r = (T*)(base + off);
        off += (elems * sizeof(T) + 255) & ~(size_t)255;
        return r;
    }
    static size_t need(size_t bytes) { return (bytes + 255) & ~(size_t)255; }
};

}  // namespace

extern "C" {

sm2b_ctx* gecc_ctx_new(gecc_curve curve, int device) {
    if (curve != GECC_CURVE_SM2 && curve != GECC_CURVE_SECP256K1) return nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        fprintf(stderr, "gecc_b200: no usable CUDA device (this library has no CPU path)\n");
        return nullptr;
    }
    if (device < 0) {
        if (cudaGetDevice(&device) != cudaSuccess) return nullptr;
    }
    if (device >= count) return nullptr;
    sm2b_ctx* ctx = new (std::nothrow) sm2b_ctx();
    if (!ctx) return nullptr;
    ctx->curve = curve == GECC_CURVE_SM2 ? CURVE_SM2 : CURVE_SECP;
    ctx->device = device;
    DeviceGuard g(device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return nullptr;
    }
    ctx->sm_count = prop.multiProcessorCount;
    ctx->stream = ctx->own_stream;
    return ctx;
}

sm2b_ctx* sm2b_ctx_new(uint32_t workers, uint32_t lanes) {
    sm2b_ctx* ctx = gecc_ctx_new(GECC_CURVE_SM2, -1);
    if (ctx) {
        ctx->workers = workers;
        ctx->lanes = lanes;
    }
    return ctx;
}

void sm2b_ctx_free(sm2b_ctx* ctx) {
    if (!ctx) return;
    {
        DeviceGuard g(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        ctx->in.release();
        ctx->out.release();
        ctx->scratch.release();
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    }
    delete ctx;
}

const char* sm2b_version(void) { return "1.0.0"; }

const char* sm2b_status_str(sm2b_status status) {
    static const char* const names[] = {"ok", "invalid argument", "malformed input",
                                        "invalid peer point", "degenerate result",
                                        "nonce retries exhausted",
                                        "cost model has no crossover", "internal error"};
    return (unsigned)status < 8 ? names[status] : "unknown status";
}

sm2b_status sm2b_ledger_read(const sm2b_ctx* ctx, sm2b_op_counts* out) {
    if (!ctx || !out) return SM2B_ERROR_INVALID_ARGUMENT;
    sm2b_ctx* c = const_cast<sm2b_ctx*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    *out = ctx->ledger;
    return SM2B_OK;
}
sm2b_status sm2b_ledger_reset(sm2b_ctx* ctx) {
    if (!ctx) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->ledger = sm2b_op_counts{0, 0, 0, 0};
    return SM2B_OK;
}

// bench.cpp:65-70: c_inv < 5 N c_mul
sm2b_status sm2b_crossover_n(uint64_t cost_add, uint64_t cost_mul, uint64_t cost_inv,
                             uint64_t* out_n) {
    (void)cost_add;
    if (!out_n) return SM2B_ERROR_INVALID_ARGUMENT;
    if (cost_mul == 0) return SM2B_ERROR_NO_CROSSOVER;
    *out_n = cost_inv / (5 * cost_mul) + 1;
    return SM2B_OK;
}

int gecc_ctx_curve(const sm2b_ctx* ctx) {
    return ctx ? (ctx->curve == CURVE_SM2 ? GECC_CURVE_SM2 : GECC_CURVE_SECP256K1) : -1;
}
int gecc_ctx_device(const sm2b_ctx* ctx) { return ctx ? ctx->device : -1; }
const char* gecc_last_error(const sm2b_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }
uint64_t gecc_kernel_launches(const sm2b_ctx* ctx) { return ctx ? ctx->launches : 0; }

sm2b_status gecc_ctx_set_stream(sm2b_ctx* ctx, void* stream) {
    if (!ctx) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
    return SM2B_OK;
}

// ------------------------------------------------------------------ field ops
sm2b_status gecc_field_op_dev(sm2b_ctx* ctx, gecc_field field, gecc_field_opcode op, size_t n,
                              const uint32_t* a, const uint32_t* b, uint32_t* out) {
    if (!ctx || (n > 0 && (!a || !out)) || (unsigned)op > 5 || (unsigned)field > 1)
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n > 0 && op <= GECC_OP_MOD_SUB && !b) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, launch_field_op(ctx->curve, field, op, n, a, b, out, ctx->stream));
    ctx->launches += n ? 1 : 0;
    return SM2B_OK;
}

sm2b_status gecc_field_op(sm2b_ctx* ctx, gecc_field field, gecc_field_opcode op, size_t n,
                          const uint32_t* a, const uint32_t* b, uint32_t* out) {
    if (!ctx || (n > 0 && (!a || !out)) || (unsigned)op > 5 || (unsigned)field > 1)
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n > 0 && op <= GECC_OP_MOD_SUB && !b) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    uint32_t *da, *db, *dout;
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        DeviceGuard g(ctx->device);
        const size_t bytes = 32 * n;
        CU(ctx, ctx->in.ensure(2 * Carver::need(bytes)));
        CU(ctx, ctx->out.ensure(Carver::need(bytes)));
        Carver ci(ctx->in.p);
        da = ci.take<uint32_t>(8 * n);
        db = ci.take<uint32_t>(8 * n);
        dout = (uint32_t*)ctx->out.p;
        CU(ctx, cudaMemcpyAsync(da, a, bytes, cudaMemcpyHostToDevice, ctx->stream));
        if (b) CU(ctx, cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
    sm2b_status st = gecc_field_op_dev(ctx, field, op, n, da, b ? db : nullptr, dout);
    if (st != SM2B_OK) return st;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, cudaMemcpyAsync(out, dout, 32 * n, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

sm2b_status gecc_microbench(sm2b_ctx* ctx, int which, int iters, double* ops_per_clk_per_sm,
                            double* seconds, double* total_ops) {
    if (!ctx || !ops_per_clk_per_sm || !seconds || !total_ops || iters <= 0)
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, run_microbench(which, iters, ctx->sm_count, ops_per_clk_per_sm, seconds, total_ops,
                           ctx->stream));
    ctx->launches += 2;
    return SM2B_OK;
}

// ------------------------------------------------------------------ not yet built
#define GECC_TODO(ctx) ((ctx) ? fail_msg(ctx, "not implemented in this build") : SM2B_ERROR_INVALID_ARGUMENT)

sm2b_status sm2b_keygen(sm2b_ctx* ctx, uint64_t, size_t, uint8_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status sm2b_sign(sm2b_ctx* ctx, size_t, const uint8_t*, const uint8_t*, uint64_t, uint8_t*, int32_t*) { return GECC_TODO(ctx); }
sm2b_status sm2b_verify(sm2b_ctx* ctx, size_t, const uint8_t*, const uint8_t*, const uint8_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status sm2b_ecdh(sm2b_ctx* ctx, size_t, const uint8_t*, const uint8_t*, uint8_t*, int32_t*) { return GECC_TODO(ctx); }
sm2b_status sm2b_bench_run(sm2b_ctx* ctx, const char*, const char*, size_t, size_t, uint32_t, uint64_t, uint32_t, sm2b_bench_report*) { return GECC_TODO(ctx); }
sm2b_status gecc_keygen(sm2b_ctx* ctx, uint64_t, uint64_t, size_t, uint8_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_sign(sm2b_ctx* ctx, size_t, const uint8_t*, const uint8_t*, uint64_t, uint64_t, uint8_t*, int32_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_invert(sm2b_ctx* ctx, gecc_field, size_t, const uint32_t*, uint32_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_padd(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint8_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_pdbl(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_fpmul(sm2b_ctx* ctx, size_t, const uint32_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_upmul(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_msm(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_invert_dev(sm2b_ctx* ctx, gecc_field, size_t, const uint32_t*, uint32_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_padd_dev(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint8_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_pdbl_dev(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_fpmul_dev(sm2b_ctx* ctx, size_t, const uint32_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_batch_upmul_dev(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_verify_dev(sm2b_ctx* ctx, size_t, const uint8_t*, const uint8_t*, const uint8_t*, uint8_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_sign_dev(sm2b_ctx* ctx, size_t, const uint8_t*, const uint8_t*, uint64_t, uint64_t, uint8_t*, int32_t*) { return GECC_TODO(ctx); }
sm2b_status gecc_msm_dev(sm2b_ctx* ctx, size_t, const uint32_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint32_t*, uint32_t*, uint8_t*) { return GECC_TODO(ctx); }

}  // extern "C"
