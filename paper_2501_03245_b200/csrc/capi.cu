// C ABI of libgecc_b200.so (include/gecc_b200.h).  Host side of the drop-in
// boundary: mirrors the reference's capi.cpp semantics (argument checks, status
// codes, per-lane reporting, ledger) and hands all arithmetic to CUDA kernels.
// There is no CPU compute path in this file.
//
// Locking: every entry point holds ctx->mu from its first touch of the context's arenas to
// its last (the reference's contract: calls on one context serialise, sm2batch.h:38-40).  The
// bodies that do the work are the *_locked functions below; they assume the lock is held and
// the device is current, so the host-pointer forms can stage, launch and drain under ONE lock.
#include <cuda_runtime.h>
#include <sys/random.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "capi_ctx.h"

using namespace gecc;
using namespace gecc_capi;

namespace {

sm2b_status fail(sm2b_ctx* ctx, const char* what, cudaError_t e) {
    ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return SM2B_ERROR_INTERNAL;
}
sm2b_status fail_msg(sm2b_ctx* ctx, const char* what) {
    ctx->last_error = what;
    return SM2B_ERROR_INTERNAL;
}

// limbs per element of a column buffer: coordinates follow the curve, scalars are 256-bit
size_t field_limbs(const sm2b_ctx* ctx, int field) { return field == 0 ? (size_t)ctx->limbs : 8; }

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

bool uniform(const sm2b_ctx* ctx) { return ctx->secret_mode == GECC_SECRET_UNIFORM; }

}  // namespace

// ------------------------------------------------------------------ ledger emulation
// The kernels do not count; each call advances the ledger by the reference
// algorithm's closed forms for a batch with no exceptional lanes:
//   batch_invert  (3N-3, 0, 0, 1)            batch_padd (6N-3, 0, 6N, 1)
//   batch_fpmul   256*(6N+3(L-1), 0, 7N, 1)  batch_upmul 256*(14N+3(L-1), 5N, 11N, 1)
namespace {
// lane policy + counters; sm2b_ctx derives its own, sm2b_bench_run builds a scratch one
struct Ledger {
    sm2b_op_counts* ops;
    uint32_t lanes, workers;
};
uint64_t eff_lanes(const Ledger& L, size_t n) {  // BatchConfig::effective_lanes + LanePlan clamp
    uint64_t l = L.lanes;
    if (l == 0) {
        uint64_t w = L.workers ? L.workers : 1;
        l = w * 4;
    }
    if (l > n) l = n ? n : 1;
    return l;
}
void led(const Ledger& L, uint64_t mul, uint64_t add, uint64_t sub, uint64_t inv) {
    L.ops->modmul += mul;
    L.ops->modadd += add;
    L.ops->modsub += sub;
    L.ops->modinv += inv;
}
void led_invert(const Ledger& L, uint64_t n) { if (n) led(L, 3 * n - 3, 0, 0, 1); }
void led_padd(const Ledger& L, uint64_t n) { if (n) led(L, 6 * n - 3, 0, 6 * n, 1); }
void led_pdbl(const Ledger& L, uint64_t n) { if (n) led(L, 7 * n - 3, 4 * n, 4 * n, 1); }
void led_fpmul(const Ledger& L, uint64_t n) {
    if (n) led(L, 256 * (6 * n + 3 * (eff_lanes(L, n) - 1)), 0, 256 * 7 * n, 256);
}
void led_upmul(const Ledger& L, uint64_t n) {
    if (n) led(L, 256 * (14 * n + 3 * (eff_lanes(L, n) - 1)), 256 * 5 * n, 256 * 11 * n, 256);
}
Ledger ledger_of(sm2b_ctx* ctx) { return Ledger{&ctx->ledger, ctx->lanes, ctx->workers}; }
}  // namespace

namespace gecc_capi {
void account_verify(sm2b_ctx* ctx, size_t count) {
    const Ledger L = ledger_of(ctx);
    led_invert(L, count);
    led(L, 2 * count, 0, 0, 0);
    led_fpmul(L, count);
    led_upmul(L, count);
    led_padd(L, count);
}
void account_sign(sm2b_ctx* ctx, size_t count) {
    const Ledger L = ledger_of(ctx);
    led_fpmul(L, count);
    led_invert(L, count);
    led(L, 2 * count, count, 0, 0);
}
void account_keygen(sm2b_ctx* ctx, size_t count) { led_fpmul(ledger_of(ctx), count); }
void account_ecdh(sm2b_ctx* ctx, size_t count) { led_upmul(ledger_of(ctx), count); }
void account_points(sm2b_ctx* ctx, int op, size_t n) {
    const Ledger L = ledger_of(ctx);
    if (op == OP_PADD) led_padd(L, n);
    else if (op == OP_PDBL) led_pdbl(L, n);
    else if (op == OP_FPMUL) led_fpmul(L, n);
    else led_upmul(L, n);
}
void account_invert(sm2b_ctx* ctx, size_t n) { led_invert(ledger_of(ctx), n); }

// seed == 0: system entropy (capi.cpp:75-79), drawn on the host.  No degraded fallback: a
// predictable nonce seed gives away the private key, so a missing entropy source is an error.
bool system_seed(uint64_t* out) {
    uint64_t v = 0;
    for (int tries = 0; tries < 16; ++tries) {
        size_t got = 0;
        while (got < sizeof v) {
            const ssize_t r = getrandom((uint8_t*)&v + got, sizeof v - got, 0);
            if (r <= 0) return false;
            got += (size_t)r;
        }
        if (v) {  // 0 means "system entropy" to the callee, so it is not a usable seed
            *out = v;
            return true;
        }
    }
    return false;
}
}  // namespace gecc_capi

extern "C" {

sm2b_ctx* gecc_ctx_new(gecc_curve curve, int device) {
    if ((unsigned)curve > GECC_CURVE_BLS12_377) return nullptr;
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
    ctx->curve = (int)curve;  // the internal ids equal the public enum
    ctx->limbs = curve_limbs(ctx->curve);
    ctx->device = device;
    DeviceGuard g(device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        sm2b_ctx_free(ctx);
        return nullptr;
    }
    ctx->sm_count = prop.multiProcessorCount;
    ctx->stream = ctx->own_stream;
    if (cudaHostAlloc((void**)&ctx->hflag, 64, cudaHostAllocDefault) != cudaSuccess ||
        ctx->xchg.ensure(16384) != cudaSuccess) {
        sm2b_ctx_free(ctx);
        return nullptr;
    }
    if (curve_is_bls(ctx->curve)) {  // field / batch / MSM layer only: no ECDSA, no fixed-base table
        if (cudaMalloc(&ctx->flags, 256) != cudaSuccess) {
            sm2b_ctx_free(ctx);
            return nullptr;
        }
        return ctx;
    }
    // fixed-base table (sm2b_ctx_new builds sm2_base_table() eagerly too, capi.cpp:101)
    uint32_t* bases = nullptr;
    bool ok = cudaMalloc(&ctx->gtab, gtable_words() * 4) == cudaSuccess &&
              cudaMalloc(&ctx->flags, 256) == cudaSuccess &&
              cudaMalloc(&bases, 64 * 16 * 4 * 8) == cudaSuccess &&
              build_gtable(ctx->curve, false, ctx->gtab, bases, ctx->stream) == cudaSuccess;
    ctx->gtab_rec = ctx->gtab;
    if (ok && ctx->curve == CURVE_SECP)
        ok = cudaMalloc(&ctx->gtab_rec, gtable_words() * 4) == cudaSuccess &&
             build_gtable(ctx->curve, true, ctx->gtab_rec, bases, ctx->stream) == cudaSuccess;
    ok = ok && cudaStreamSynchronize(ctx->stream) == cudaSuccess;
    if (bases) cudaFree(bases);
    if (!ok) {
        fprintf(stderr, "gecc_b200: building the fixed-base table failed: %s\n",
                cudaGetErrorString(cudaGetLastError()));
        sm2b_ctx_free(ctx);
        return nullptr;
    }
    ctx->launches += 2;
    return ctx;
}

sm2b_ctx* gecc_ctx_new_multi(gecc_curve curve, int ndev, const int* devices) {
    if ((unsigned)curve > GECC_CURVE_BLS12_377) return nullptr;
    return group_new(curve, ndev, devices);
}

int gecc_ctx_shards(const sm2b_ctx* ctx) { return !ctx ? 0 : (ctx->shards.empty() ? 1 : (int)ctx->shards.size()); }

// sm2batch.h:44-45.  One visible device: a device context on the current device.  Several: a
// group over all of them ("one ctx owns CUDA streams / device buffers for all
// visible GPUs"), GECC_NDEV=k limits it to the first k.
sm2b_ctx* sm2b_ctx_new(uint32_t workers, uint32_t lanes) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        fprintf(stderr, "gecc_b200: no usable CUDA device (this library has no CPU path)\n");
        return nullptr;
    }
    if (const char* v = getenv("GECC_NDEV")) {
        const int k = atoi(v);
        if (k >= 1 && k < count) count = k;
    }
    sm2b_ctx* ctx = count > 1 ? group_new(GECC_CURVE_SM2, count, nullptr) : gecc_ctx_new(GECC_CURVE_SM2, -1);
    if (ctx) {
        ctx->workers = workers;
        ctx->lanes = lanes;
    }
    return ctx;
}

void sm2b_ctx_free(sm2b_ctx* ctx) {
    if (!ctx) return;
    if (is_group(ctx)) {
        group_free(ctx);
        return;
    }
    {
        DeviceGuard g(ctx->device);
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        comm_release(ctx);
        ctx->in.release();
        ctx->out.release();
        ctx->scratch.release();
        ctx->batch_tmp.release();
        ctx->lane_tabs.release();
        ctx->xchg.release();
        if (ctx->gtab_rec && ctx->gtab_rec != ctx->gtab) cudaFree(ctx->gtab_rec);
        if (ctx->gtab) cudaFree(ctx->gtab);
        if (ctx->flags) cudaFree(ctx->flags);
        if (ctx->hflag) cudaFreeHost(ctx->hflag);
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        if (ctx->h2d_stream) cudaStreamDestroy(ctx->h2d_stream);
        if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
        if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
        if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
        if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
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
    return ctx ? ctx->curve : -1;  // internal ids equal the public enum
}
int gecc_ctx_device(const sm2b_ctx* ctx) { return ctx ? ctx->device : -1; }
const char* gecc_last_error(const sm2b_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }
uint64_t gecc_kernel_launches(const sm2b_ctx* ctx) {
    if (!ctx) return 0;
    uint64_t total = ctx->launches;
    for (const sm2b_ctx* s : ctx->shards) total += s->launches;
    return total;
}

sm2b_status gecc_ctx_set_stream(sm2b_ctx* ctx, void* stream) {
    if (!ctx || is_group(ctx)) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
    return SM2B_OK;
}

sm2b_status gecc_ctx_set_secret_mode(sm2b_ctx* ctx, int mode) {
    if (!ctx || (mode != GECC_SECRET_FAST && mode != GECC_SECRET_UNIFORM)) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->secret_mode = mode;
    for (sm2b_ctx* s : ctx->shards) {
        std::lock_guard<std::mutex> lks(s->mu);
        s->secret_mode = mode;
    }
    return SM2B_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ field ops
namespace {
bool field_args_ok(const sm2b_ctx* ctx, int field, int op, size_t n, const void* a, const void* b, const void* out) {
    if (!ctx || (n > 0 && (!a || !out)) || (unsigned)op > GECC_OP_MOD_INV_WARP || (unsigned)field > 1) return false;
    const bool binary = op <= GECC_OP_MOD_SUB || op == GECC_OP_MONT_REDUCE || op == GECC_OP_LAZY_MUL ||
                        op == GECC_OP_LAZY_ADD || op == GECC_OP_LAZY_SUB;
    if (n > 0 && binary && !b) return false;
    // the weakly reduced representation exists for the secp256k1 base field only
    if (op >= GECC_OP_LAZY_MUL && op <= GECC_OP_LAZY_SUB && !(ctx->curve == CURVE_SECP && field == 0)) return false;
    return true;
}
}  // namespace

extern "C" sm2b_status gecc_field_op_dev(sm2b_ctx* ctx, gecc_field field, gecc_field_opcode op, size_t n,
                                         const uint32_t* a, const uint32_t* b, uint32_t* out) {
    if (!field_args_ok(ctx, field, op, n, a, b, out) || is_group(ctx)) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, launch_field_op(ctx->curve, field, op, n, a, b, out, ctx->stream));
    ctx->launches += n ? 1 : 0;
    return SM2B_OK;
}

namespace gecc_capi {
sm2b_status field_range(sm2b_ctx* ctx, int field, int op, size_t pitch, size_t begin, size_t count,
                        const uint32_t* a, const uint32_t* b, uint32_t* out) {
    if (count == 0) return SM2B_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t L = field_limbs(ctx, field), bytes = 4 * L * count;
    CU(ctx, ctx->in.ensure(2 * Carver::need(bytes)));
    CU(ctx, ctx->out.ensure(Carver::need(bytes)));
    Carver ci(ctx->in.p);
    uint32_t* da = ci.take<uint32_t>(L * count);
    uint32_t* db = ci.take<uint32_t>(L * count);
    uint32_t* dout = (uint32_t*)ctx->out.p;
    CU(ctx, cudaMemcpy2DAsync(da, 4 * count, a + begin, 4 * pitch, 4 * count, L, cudaMemcpyHostToDevice, ctx->stream));
    if (b)
        CU(ctx, cudaMemcpy2DAsync(db, 4 * count, b + begin, 4 * pitch, 4 * count, L, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, launch_field_op(ctx->curve, field, op, count, da, b ? db : nullptr, dout, ctx->stream));
    ctx->launches += 1;
    CU(ctx, cudaMemcpy2DAsync(out + begin, 4 * pitch, dout, 4 * count, 4 * count, L, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}
}  // namespace gecc_capi

extern "C" {

sm2b_status gecc_field_op(sm2b_ctx* ctx, gecc_field field, gecc_field_opcode op, size_t n,
                          const uint32_t* a, const uint32_t* b, uint32_t* out) {
    if (!field_args_ok(ctx, field, op, n, a, b, out)) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    if (is_group(ctx)) return group_field(ctx, field, op, n, a, b, out);
    return field_range(ctx, field, op, n, 0, n, a, b, out);
}

void gecc_set_batch_form(int form) { set_batch_form(form < 0 || form > 9 ? 0 : form); }
void gecc_set_msm_form(int form) { set_msm_form(form < 0 || form > 5 ? 0 : form); }

sm2b_status gecc_microbench(sm2b_ctx* ctx, int which, int iters, double* ops_per_clk_per_sm,
                            double* seconds, double* total_ops) {
    if (!ctx || !ops_per_clk_per_sm || !seconds || !total_ops || iters <= 0 || is_group(ctx))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, run_microbench(which, iters, ctx->sm_count, ops_per_clk_per_sm, seconds, total_ops,
                           ctx->stream));
    ctx->launches += 2;
    return SM2B_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ host-API pipeline
// The byte-record entry points split a large batch into chunks and run three streams:
// H2D of chunk c+1, the kernel of chunk c and D2H of chunk c-1 overlap (events order
// them).  With pinned caller buffers the copies are truly asynchronous; with pageable
// buffers CUDA stages them and the result is the same, only less overlapped.
namespace {
constexpr size_t PIPE_MIN_CHUNK = (size_t)1 << 17;
constexpr size_t PIPE_HEAD_CHUNK = (size_t)1 << 16;
#ifndef GECC_PIPE_MAX_CHUNKS
#define GECC_PIPE_MAX_CHUNKS 4
#endif
constexpr int PIPE_MAX_CHUNKS = GECC_PIPE_MAX_CHUNKS;

// Up to PIPE_MAX_CHUNKS equal chunks of at least PIPE_MIN_CHUNK records, preceded -- when the
// batch is large enough -- by a short head chunk: only the first upload is exposed (nothing
// can run before it), so it should be small; the chunk kernels overlap on two streams, so a
// small head does not cost a wave of its own.
struct Chunks {
    size_t count, size;  // size: the largest chunk
    int n;
    size_t off[PIPE_MAX_CHUNKS + 2];
    explicit Chunks(size_t total, bool with_head = true) : count(total) {
        size_t head = with_head && total >= 4 * PIPE_MIN_CHUNK ? PIPE_HEAD_CHUNK : 0;
        const size_t rest = total - head;
        int k = (int)(rest / PIPE_MIN_CHUNK);
        if (k < 1) k = 1;
        if (k > PIPE_MAX_CHUNKS) k = PIPE_MAX_CHUNKS;
        size = (rest + k - 1) / k;
        n = 0;
        off[0] = 0;
        if (head) off[++n] = head;
        for (size_t at = head; at < total; at += size) off[++n] = at + size < total ? at + size : total;
        if (n == 0) off[++n] = total;  // total == 0 never reaches here; keeps the invariant anyway
    }
    size_t begin(int c) const { return off[c]; }
    size_t len(int c) const { return off[c + 1] - off[c]; }
};

struct EventPool {  // events of one pipelined call; destroyed at scope exit
    std::vector<cudaEvent_t> ev;
    cudaEvent_t get() {
        cudaEvent_t e = nullptr;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        ev.push_back(e);
        return e;
    }
    ~EventPool() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
};

// ------------------------------------------------------------------ protocol layer
constexpr size_t VERIFY_SCRATCH_MAX_LANES = (size_t)1 << 22;  // 2 GiB of lane tables at most
// returns the number of lanes the verify scratch covers (0 on allocation failure)
size_t ensure_lane_tabs(sm2b_ctx* ctx, size_t count) {
    const size_t lanes = count < VERIFY_SCRATCH_MAX_LANES ? count : VERIFY_SCRATCH_MAX_LANES;
    return ctx->lane_tabs.ensure(verify_scratch_bytes(lanes)) == cudaSuccess ? lanes : 0;
}
bool ecdsa_ctx(const sm2b_ctx* ctx) { return ctx && !curve_is_bls(ctx->curve); }  // ECDSA layer: 256-bit curves only

// report_lanes (capi.cpp:64-73)
sm2b_status report_lanes(const int32_t* st, size_t n, int32_t* lane_status) {
    int32_t first = SM2B_OK;
    for (size_t i = 0; i < n; ++i) {
        if (lane_status) lane_status[i] = st[i];
        if (st[i] != SM2B_OK && first == SM2B_OK) first = st[i];
    }
    return lane_status ? SM2B_OK : (sm2b_status)first;
}
}  // namespace

extern "C" {

sm2b_status gecc_verify_dev(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                            const uint8_t* publics, const uint8_t* signatures,
                            uint8_t* results) {
    if (!ecdsa_ctx(ctx) || is_group(ctx) || (count > 0 && (!digests || !publics || !signatures || !results)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t tab_lanes = ensure_lane_tabs(ctx, count);
    CU(ctx, launch_verify(ctx->curve, count, digests, publics, signatures, ctx->gtab_rec, results,
                          (uint32_t*)ctx->lane_tabs.p, tab_lanes, ctx->stream));
    ctx->launches += count ? 1 : 0;
    account_verify(ctx, count);
    return SM2B_OK;
}

sm2b_status sm2b_verify(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                        const uint8_t* publics, const uint8_t* signatures, uint8_t* results) {
    if (!ecdsa_ctx(ctx) || (count > 0 && (!digests || !publics || !signatures || !results)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (is_group(ctx)) return group_verify(ctx, count, digests, publics, signatures, results);
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->in.ensure(Carver::need(32 * count) + Carver::need(65 * count) + Carver::need(64 * count)));
    CU(ctx, ctx->out.ensure(Carver::need(count)));
    Carver ci(ctx->in.p);
    uint8_t* dd = ci.take<uint8_t>(32 * count);
    uint8_t* dp = ci.take<uint8_t>(65 * count);
    uint8_t* ds = ci.take<uint8_t>(64 * count);
    uint8_t* dr = (uint8_t*)ctx->out.p;
    const Chunks ch(count);
    // chunk kernels alternate between two compute streams (the tail of one chunk overlaps the
    // head of the next), each with its own half of the lane-table scratch
    const size_t tab_half = ensure_lane_tabs(ctx, 2 * ch.size) / 2;
    EventPool pool;
    // the arenas may still be in use by earlier work on the compute stream
    cudaEvent_t idle = pool.get();
    CU(ctx, cudaEventRecord(idle, ctx->stream));
    CU(ctx, cudaStreamWaitEvent(ctx->h2d_stream, idle, 0));
    CU(ctx, cudaStreamWaitEvent(ctx->aux_stream, idle, 0));
    for (int c = 0; c < ch.n; ++c) {
        const size_t b = ch.begin(c), m = ch.len(c);
        CU(ctx, cudaMemcpyAsync(dd + 32 * b, digests + 32 * b, 32 * m, cudaMemcpyHostToDevice, ctx->h2d_stream));
        CU(ctx, cudaMemcpyAsync(dp + 65 * b, publics + 65 * b, 65 * m, cudaMemcpyHostToDevice, ctx->h2d_stream));
        CU(ctx, cudaMemcpyAsync(ds + 64 * b, signatures + 64 * b, 64 * m, cudaMemcpyHostToDevice, ctx->h2d_stream));
        cudaEvent_t up = pool.get(), done = pool.get();
        CU(ctx, cudaEventRecord(up, ctx->h2d_stream));
        cudaStream_t ks = (c & 1) ? ctx->aux_stream : ctx->stream;
        uint32_t* tabs = (uint32_t*)ctx->lane_tabs.p + (size_t)(c & 1) * tab_half * 128;  // 512 B per lane
        CU(ctx, cudaStreamWaitEvent(ks, up, 0));
        CU(ctx, launch_verify(ctx->curve, m, dd + 32 * b, dp + 65 * b, ds + 64 * b, ctx->gtab_rec, dr + b, tabs,
                              tab_half, ks));
        CU(ctx, cudaEventRecord(done, ks));
        CU(ctx, cudaStreamWaitEvent(ctx->d2h_stream, done, 0));
        CU(ctx, cudaMemcpyAsync(results + b, dr + b, m, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    }
    ctx->launches += ch.n;
    account_verify(ctx, count);
    CU(ctx, cudaStreamSynchronize(ctx->d2h_stream));
    CU(ctx, cudaStreamSynchronize(ctx->aux_stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

sm2b_status gecc_sign_dev(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                          const uint8_t* secrets, uint64_t nonce_seed, uint64_t lane_base,
                          uint8_t* signatures, int32_t* lane_status) {
    if (!ecdsa_ctx(ctx) || is_group(ctx) || (count > 0 && (!digests || !secrets || !signatures || !lane_status)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nonce_seed == 0) return fail_msg(ctx, "device signing needs a non-zero nonce seed");
    DeviceGuard g(ctx->device);
    CU(ctx, cudaMemsetAsync(ctx->flags, 0, 4, ctx->stream));
    CU(ctx, launch_sign(ctx->curve, count, digests, secrets, nonce_seed, lane_base, ctx->gtab_rec,
                        signatures, lane_status, ctx->flags, ctx->stream, uniform(ctx)));
    ctx->launches += count ? 1 : 0;
    account_sign(ctx, count);
    return SM2B_OK;
}

sm2b_status gecc_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                      uint64_t nonce_seed, uint64_t lane_base, uint8_t* signatures,
                      int32_t* lane_status) {
    if (!ecdsa_ctx(ctx) || (count > 0 && (!digests || !secrets || !signatures)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (nonce_seed == 0 && !system_seed(&nonce_seed)) {
        std::lock_guard<std::mutex> lk(ctx->mu);
        return fail_msg(ctx, "no system entropy for the nonce seed (getrandom failed)");
    }
    if (is_group(ctx)) return group_sign(ctx, count, digests, secrets, nonce_seed, lane_base, signatures, lane_status);
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->in.ensure(2 * Carver::need(32 * count)));
    CU(ctx, ctx->out.ensure(Carver::need(64 * count) + Carver::need(4 * count)));
    Carver ci(ctx->in.p), co(ctx->out.p);
    uint8_t* dd = ci.take<uint8_t>(32 * count);
    uint8_t* dsec = ci.take<uint8_t>(32 * count);
    uint8_t* dsig = co.take<uint8_t>(64 * count);
    int32_t* dst = co.take<int32_t>(count);
    const Chunks ch(count, false);  // all secrets follow chunk 0 anyway: a short head would only idle the GPU
    EventPool pool;
    cudaEvent_t idle = pool.get();
    CU(ctx, cudaEventRecord(idle, ctx->stream));
    CU(ctx, cudaStreamWaitEvent(ctx->h2d_stream, idle, 0));
    CU(ctx, cudaStreamWaitEvent(ctx->d2h_stream, idle, 0));
    CU(ctx, cudaStreamWaitEvent(ctx->aux_stream, idle, 0));
    CU(ctx, cudaMemsetAsync(ctx->flags, 0, 4, ctx->h2d_stream));
    // A zero or oversize secret must fail the whole call before any output is written
    // (capi.cpp:181-184).  Chunk 0 goes up first and starts signing; all remaining secrets follow
    // and are range-checked by a tiny kernel while chunk 0 runs, so the verdict is known about
    // when the first signatures are ready.  From then on it is a three-stream pipeline: H2D of
    // the digests of chunk c+1, the kernel of chunk c, D2H of the signatures of chunk c-1.
    std::vector<cudaEvent_t> done(ch.n);
    cudaEvent_t verdict = pool.get();
    *ctx->hflag = 0;
    for (int c = 0; c < ch.n; ++c) {
        const size_t b = ch.begin(c), m = ch.len(c);
        if (c == 0) CU(ctx, cudaMemcpyAsync(dsec, secrets, 32 * m, cudaMemcpyHostToDevice, ctx->h2d_stream));
        CU(ctx, cudaMemcpyAsync(dd + 32 * b, digests + 32 * b, 32 * m, cudaMemcpyHostToDevice, ctx->h2d_stream));
        cudaEvent_t up = pool.get();
        CU(ctx, cudaEventRecord(up, ctx->h2d_stream));
        // chunk kernels alternate between two streams: a chunk is a fraction of a wave short of
        // filling the chip, and the next chunk's blocks take the free slots
        cudaStream_t ks = (c & 1) ? ctx->aux_stream : ctx->stream;
        CU(ctx, cudaStreamWaitEvent(ks, up, 0));
        CU(ctx, launch_sign(ctx->curve, m, dd + 32 * b, dsec + 32 * b, nonce_seed, lane_base + b, ctx->gtab_rec,
                            dsig + 64 * b, dst + b, ctx->flags, ks, uniform(ctx)));
        done[c] = pool.get();
        CU(ctx, cudaEventRecord(done[c], ks));
        if (c == 0) {  // the rest of the secrets, their check, the verdict
            if (count > m) {
                CU(ctx, cudaMemcpyAsync(dsec + 32 * m, secrets + 32 * m, 32 * (count - m), cudaMemcpyHostToDevice,
                                        ctx->h2d_stream));
                cudaEvent_t sec_up = pool.get();
                CU(ctx, cudaEventRecord(sec_up, ctx->h2d_stream));
                CU(ctx, cudaStreamWaitEvent(ctx->stream, sec_up, 0));
                CU(ctx, launch_secret_range(ctx->curve, count - m, dsec + 32 * m, ctx->flags, ctx->stream));
            }
            CU(ctx, cudaMemcpyAsync(ctx->hflag, ctx->flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
            CU(ctx, cudaEventRecord(verdict, ctx->stream));
        }
    }
    ctx->launches += ch.n + 1;
    account_sign(ctx, count);
    CU(ctx, cudaEventSynchronize(verdict));
    if (*ctx->hflag) {  // nothing has been copied out; let the queued kernels drain
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->aux_stream));
        return SM2B_ERROR_MALFORMED_INPUT;
    }
    // per-lane statuses go straight into the caller's array (no host-side pass over the lanes)
    std::vector<int32_t> hst;
    int32_t* st_dst = lane_status;
    if (!st_dst) {
        hst.resize(count);
        st_dst = hst.data();
    }
    for (int c = 0; c < ch.n; ++c) {
        const size_t b = ch.begin(c), m = ch.len(c);
        CU(ctx, cudaStreamWaitEvent(ctx->d2h_stream, done[c], 0));
        CU(ctx, cudaMemcpyAsync(signatures + 64 * b, dsig + 64 * b, 64 * m, cudaMemcpyDeviceToHost, ctx->d2h_stream));
        CU(ctx, cudaMemcpyAsync(st_dst + b, dst + b, 4 * m, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    }
    CU(ctx, cudaStreamSynchronize(ctx->d2h_stream));
    CU(ctx, cudaStreamSynchronize(ctx->aux_stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    if (lane_status) return SM2B_OK;  // report_lanes (capi.cpp:64-73): statuses delivered, call is OK
    return report_lanes(hst.data(), count, nullptr);
}

sm2b_status sm2b_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                      uint64_t nonce_seed, uint8_t* signatures, int32_t* lane_status) {
    return gecc_sign(ctx, count, digests, secrets, nonce_seed, 0, signatures, lane_status);
}

}  // extern "C"

namespace gecc_capi {
sm2b_status sign_nonces_range(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                              const uint8_t* nonces, uint8_t* signatures, int32_t* lane_status) {
    if (count == 0) return SM2B_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->in.ensure(3 * Carver::need(32 * count)));
    CU(ctx, ctx->out.ensure(Carver::need(64 * count) + Carver::need(4 * count)));
    Carver ci(ctx->in.p), co(ctx->out.p);
    uint8_t* dd = ci.take<uint8_t>(32 * count);
    uint8_t* dsec = ci.take<uint8_t>(32 * count);
    uint8_t* dk = ci.take<uint8_t>(32 * count);
    uint8_t* dsig = co.take<uint8_t>(64 * count);
    int32_t* dst = co.take<int32_t>(count);
    cudaStream_t s = ctx->stream;
    CU(ctx, cudaMemcpyAsync(dd, digests, 32 * count, cudaMemcpyHostToDevice, s));
    CU(ctx, cudaMemcpyAsync(dsec, secrets, 32 * count, cudaMemcpyHostToDevice, s));
    CU(ctx, cudaMemcpyAsync(dk, nonces, 32 * count, cudaMemcpyHostToDevice, s));
    CU(ctx, cudaMemsetAsync(ctx->flags, 0, 4, s));
    CU(ctx, launch_sign_nonces(ctx->curve, count, dd, dsec, dk, ctx->gtab_rec, dsig, dst, ctx->flags, s, uniform(ctx)));
    ctx->launches += 1;
    account_sign(ctx, count);
    *ctx->hflag = 0;
    CU(ctx, cudaMemcpyAsync(ctx->hflag, ctx->flags, 4, cudaMemcpyDeviceToHost, s));
    CU(ctx, cudaStreamSynchronize(s));
    if (*ctx->hflag) return SM2B_ERROR_MALFORMED_INPUT;  // a secret outside (0, n): whole call, nothing written
    std::vector<int32_t> hst;
    int32_t* st_dst = lane_status;
    if (!st_dst) {
        hst.resize(count);
        st_dst = hst.data();
    }
    CU(ctx, cudaMemcpyAsync(signatures, dsig, 64 * count, cudaMemcpyDeviceToHost, s));
    CU(ctx, cudaMemcpyAsync(st_dst, dst, 4 * count, cudaMemcpyDeviceToHost, s));
    CU(ctx, cudaStreamSynchronize(s));
    if (lane_status) return SM2B_OK;
    return report_lanes(hst.data(), count, nullptr);
}
}  // namespace gecc_capi

extern "C" {

sm2b_status gecc_sign_nonces(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                             const uint8_t* nonces, uint8_t* signatures, int32_t* lane_status) {
    if (!ecdsa_ctx(ctx) || (count > 0 && (!digests || !secrets || !nonces || !signatures)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (is_group(ctx)) return group_sign_nonces(ctx, count, digests, secrets, nonces, signatures, lane_status);
    return sign_nonces_range(ctx, count, digests, secrets, nonces, signatures, lane_status);
}

sm2b_status gecc_keygen(sm2b_ctx* ctx, uint64_t seed, uint64_t lane_base, size_t count,
                        uint8_t* secrets, uint8_t* publics) {
    if (!ecdsa_ctx(ctx) || (count > 0 && (!secrets || !publics))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (seed == 0 && !system_seed(&seed)) {
        std::lock_guard<std::mutex> lk(ctx->mu);
        return fail_msg(ctx, "no system entropy for the key seed (getrandom failed)");
    }
    if (is_group(ctx)) return group_keygen(ctx, seed, lane_base, count, secrets, publics);
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->out.ensure(Carver::need(32 * count) + Carver::need(65 * count)));
    Carver co(ctx->out.p);
    uint8_t* dsec = co.take<uint8_t>(32 * count);
    uint8_t* dpub = co.take<uint8_t>(65 * count);
    CU(ctx, launch_keygen(ctx->curve, count, seed, lane_base, ctx->gtab_rec, dsec, dpub, ctx->stream, uniform(ctx)));
    ctx->launches += 1;
    account_keygen(ctx, count);
    CU(ctx, cudaMemcpyAsync(secrets, dsec, 32 * count, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaMemcpyAsync(publics, dpub, 65 * count, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}
sm2b_status sm2b_keygen(sm2b_ctx* ctx, uint64_t seed, size_t count, uint8_t* secrets,
                        uint8_t* publics) {
    return gecc_keygen(ctx, seed, 0, count, secrets, publics);
}

sm2b_status sm2b_ecdh(sm2b_ctx* ctx, size_t count, const uint8_t* secrets, const uint8_t* peers,
                      uint8_t* shared, int32_t* lane_status) {
    if (!ecdsa_ctx(ctx) || (count > 0 && (!secrets || !peers || !shared))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (is_group(ctx)) return group_ecdh(ctx, count, secrets, peers, shared, lane_status);
    std::vector<int32_t> hst(count);
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        DeviceGuard g(ctx->device);
        CU(ctx, ctx->in.ensure(Carver::need(32 * count) + Carver::need(65 * count)));
        CU(ctx, ctx->out.ensure(Carver::need(32 * count) + Carver::need(4 * count)));
        Carver ci(ctx->in.p), co(ctx->out.p);
        uint8_t* dsec = ci.take<uint8_t>(32 * count);
        uint8_t* dpeer = ci.take<uint8_t>(65 * count);
        uint8_t* dsh = co.take<uint8_t>(32 * count);
        int32_t* dst = co.take<int32_t>(count);
        CU(ctx, cudaMemcpyAsync(dsec, secrets, 32 * count, cudaMemcpyHostToDevice, ctx->stream));
        CU(ctx, cudaMemcpyAsync(dpeer, peers, 65 * count, cudaMemcpyHostToDevice, ctx->stream));
        CU(ctx, cudaMemsetAsync(ctx->flags, 0, 4, ctx->stream));
        const size_t tab_lanes = ensure_lane_tabs(ctx, count);
        CU(ctx, launch_ecdh(ctx->curve, count, dsec, dpeer, dsh, dst, ctx->flags, (uint32_t*)ctx->lane_tabs.p,
                            tab_lanes, ctx->stream, uniform(ctx)));
        ctx->launches += 1;
        account_ecdh(ctx, count);
        *ctx->hflag = 0;
        CU(ctx, cudaMemcpyAsync(ctx->hflag, ctx->flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaMemcpyAsync(hst.data(), dst, 4 * count, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        if (*ctx->hflag) return SM2B_ERROR_MALFORMED_INPUT;  // Scalar::checked on a secret (capi.cpp:241)
        CU(ctx, cudaMemcpyAsync(shared, dsh, 32 * count, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return report_lanes(hst.data(), count, lane_status);
}

}  // extern "C"

// ------------------------------------------------------------------ batch layer
namespace {
// bodies of the batch entry points: ctx->mu held, device current, pointers on the device
sm2b_status batch_invert_locked(sm2b_ctx* ctx, int field, size_t n, const uint32_t* in, uint32_t* out, bool account) {
    CU(ctx, launch_batch_invert(ctx->curve, field, n, in, out, ctx->stream));
    ctx->launches += n ? 1 : 0;
    if (account) account_invert(ctx, n);
    return SM2B_OK;
}
sm2b_status points_locked(sm2b_ctx* ctx, int op, size_t n, const uint32_t* k, const uint32_t* px, const uint32_t* py,
                          const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty, const uint8_t* tinf,
                          uint32_t* ox, uint32_t* oy, uint8_t* oinf, const uint32_t* base_tab, bool account) {
    switch (op) {
        case OP_PADD:
            CU(ctx, ctx->batch_tmp.ensure(batch_padd_scratch_bytes(n)));
            CU(ctx, launch_batch_padd(ctx->curve, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, ctx->stream,
                                      ctx->batch_tmp.p, BatchAux{ctx->aux_stream, ctx->ev_fork, ctx->ev_join}));
            break;
        case OP_PDBL:
            CU(ctx, launch_batch_pdbl(ctx->curve, n, px, py, pinf, ox, oy, oinf, ctx->stream));
            break;
        case OP_FPMUL:
            CU(ctx, launch_fpmul(ctx->curve, n, k, base_tab ? base_tab : ctx->gtab, ox, oy, oinf, ctx->stream));
            break;
        default:
            CU(ctx, ctx->lane_tabs.ensure(verify_scratch_bytes(n)));
            CU(ctx, launch_upmul(ctx->curve, n, k, px, py, pinf, ox, oy, oinf, (uint32_t*)ctx->lane_tabs.p,
                                 ctx->stream));
            break;
    }
    ctx->launches += n ? 1 : 0;
    if (account) account_points(ctx, op, n);
    return SM2B_OK;
}
const uint32_t* table_for(const sm2b_ctx* ctx, const gecc_base_table* base) {
    if (!base) return nullptr;
    if (base->owner == ctx) return base->tabs[0];
    const sm2b_ctx* owner = base->owner;  // a shard of the owning group
    for (size_t i = 0; i < owner->shards.size(); ++i)
        if (owner->shards[i] == ctx) return base->tabs[i];
    return nullptr;
}
}  // namespace

extern "C" {

sm2b_status gecc_batch_invert_dev(sm2b_ctx* ctx, gecc_field field, size_t n, const uint32_t* in,
                                  uint32_t* out) {
    if (!ctx || is_group(ctx) || (n > 0 && (!in || !out)) || (unsigned)field > 1) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return batch_invert_locked(ctx, field, n, in, out, true);
}
sm2b_status gecc_batch_padd_dev(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                                const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                                const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || is_group(ctx) || (n > 0 && (!px || !py || !tx || !ty || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return points_locked(ctx, OP_PADD, n, nullptr, px, py, pinf, tx, ty, tinf, ox, oy, oinf, nullptr, true);
}
sm2b_status gecc_batch_pdbl_dev(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                                const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || is_group(ctx) || (n > 0 && (!px || !py || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return points_locked(ctx, OP_PDBL, n, nullptr, px, py, pinf, nullptr, nullptr, nullptr, ox, oy, oinf, nullptr, true);
}
sm2b_status gecc_batch_fpmul_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, uint32_t* ox,
                                 uint32_t* oy, uint8_t* oinf) {
    if (!ecdsa_ctx(ctx) || is_group(ctx) || (n > 0 && (!scalars || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return points_locked(ctx, OP_FPMUL, n, scalars, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ox, oy, oinf,
                         nullptr, true);
}
sm2b_status gecc_batch_fpmul_base_dev(sm2b_ctx* ctx, const gecc_base_table* base, size_t n,
                                      const uint32_t* scalars, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ecdsa_ctx(ctx) || is_group(ctx) || !base || base->owner != ctx || (n > 0 && (!scalars || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return points_locked(ctx, OP_FPMUL, n, scalars, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ox, oy, oinf,
                         base->tabs[0], true);
}
sm2b_status gecc_batch_upmul_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars,
                                 const uint32_t* px, const uint32_t* py, const uint8_t* pinf,
                                 uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ecdsa_ctx(ctx) || is_group(ctx) || (n > 0 && (!scalars || !px || !py || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    return points_locked(ctx, OP_UPMUL, n, scalars, px, py, pinf, nullptr, nullptr, nullptr, ox, oy, oinf, nullptr, true);
}

}  // extern "C"

namespace gecc_capi {
// Host-pointer form shared by the column-buffer entry points, on elements [begin, begin + count)
// of host buffers whose limb rows are `pitch` elements apart: stages up to three column inputs
// (+ up to two infinity masks), runs the kernel, returns one output point buffer.  Large batches
// are cut into chunks: every chunk has its own compact column buffers on the device (count =
// chunk length, so the kernels are unchanged), filled and drained with strided 2-D copies, and
// upload / kernel / download of successive chunks overlap on three streams (PCIe is full duplex).
// The context stays locked from the first staging copy to the last download.
sm2b_status points_range(sm2b_ctx* ctx, int op, size_t pitch, size_t begin, size_t n,
                         const uint32_t* scalars, const HostPoints* p, const HostPoints* t,
                         uint32_t* ox, uint32_t* oy, uint8_t* oinf, const uint32_t* base_tab, bool account) {
    if (n == 0) return SM2B_OK;
    const size_t L = (size_t)ctx->limbs, pb = 4 * L * n;  // bytes per coordinate column buffer
    const size_t cb = Carver::need(pb), mb = Carver::need(n);
    uint32_t *dk = nullptr, *dpx = nullptr, *dpy = nullptr, *dtx = nullptr, *dty = nullptr;
    uint8_t *dpi = nullptr, *dti = nullptr;
    const Chunks ch(n >= ((size_t)1 << 19) ? n : 1, false);  // small batches: one chunk, one copy each
    const int chunks = n >= ((size_t)1 << 19) ? ch.n : 1;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->in.ensure(5 * cb + 2 * mb));
    CU(ctx, ctx->out.ensure(2 * cb + mb));
    Carver ci(ctx->in.p), co(ctx->out.p);
    uint32_t* dox = co.take<uint32_t>(L * n);
    uint32_t* doy = co.take<uint32_t>(L * n);
    uint8_t* doi = co.take<uint8_t>(n);
    if (scalars) dk = ci.take<uint32_t>(8 * n);
    if (p) {
        dpx = ci.take<uint32_t>(L * n); dpy = ci.take<uint32_t>(L * n);
        if (p->inf) dpi = ci.take<uint8_t>(n);
    }
    if (t) {
        dtx = ci.take<uint32_t>(L * n); dty = ci.take<uint32_t>(L * n);
        if (t->inf) dti = ci.take<uint8_t>(n);
    }
    EventPool pool;
    cudaEvent_t idle = pool.get();
    CU(ctx, cudaEventRecord(idle, ctx->stream));
    CU(ctx, cudaStreamWaitEvent(ctx->h2d_stream, idle, 0));
    CU(ctx, cudaStreamWaitEvent(ctx->d2h_stream, idle, 0));
    for (int c = 0; c < chunks; ++c) {
        const size_t b = chunks == 1 ? 0 : ch.begin(c), m = chunks == 1 ? n : ch.len(c);
        const size_t hb = begin + b;  // first element of this chunk in the host buffers
        // rows x m block of a host column buffer (row pitch `pitch`) -> compact device block (row pitch m)
        auto up = [&](const uint32_t* h, uint32_t* d, size_t rows) {
            return cudaMemcpy2DAsync(d + rows * b, 4 * m, h + hb, 4 * pitch, 4 * m, rows, cudaMemcpyHostToDevice,
                                     ctx->h2d_stream);
        };
        auto upm = [&](const uint8_t* h, uint8_t* d) {
            return cudaMemcpyAsync(d + b, h + hb, m, cudaMemcpyHostToDevice, ctx->h2d_stream);
        };
        if (scalars) CU(ctx, up(scalars, dk, 8));
        if (p) CU(ctx, up(p->x, dpx, L));
        if (p) CU(ctx, up(p->y, dpy, L));
        if (p && p->inf) CU(ctx, upm(p->inf, dpi));
        if (t) CU(ctx, up(t->x, dtx, L));
        if (t) CU(ctx, up(t->y, dty, L));
        if (t && t->inf) CU(ctx, upm(t->inf, dti));
        cudaEvent_t upe = pool.get(), done = pool.get();
        CU(ctx, cudaEventRecord(upe, ctx->h2d_stream));
        CU(ctx, cudaStreamWaitEvent(ctx->stream, upe, 0));
        sm2b_status st = points_locked(ctx, op, m, dk ? dk + 8 * b : nullptr, dpx ? dpx + L * b : nullptr,
                                       dpy ? dpy + L * b : nullptr, dpi ? dpi + b : nullptr,
                                       dtx ? dtx + L * b : nullptr, dty ? dty + L * b : nullptr,
                                       dti ? dti + b : nullptr, dox + L * b, doy + L * b, doi + b, base_tab, false);
        if (st != SM2B_OK) {
            cudaStreamSynchronize(ctx->h2d_stream);
            cudaStreamSynchronize(ctx->d2h_stream);
            cudaStreamSynchronize(ctx->stream);
            return st;
        }
        CU(ctx, cudaEventRecord(done, ctx->stream));
        CU(ctx, cudaStreamWaitEvent(ctx->d2h_stream, done, 0));
        CU(ctx, cudaMemcpy2DAsync(ox + hb, 4 * pitch, dox + L * b, 4 * m, 4 * m, L, cudaMemcpyDeviceToHost, ctx->d2h_stream));
        CU(ctx, cudaMemcpy2DAsync(oy + hb, 4 * pitch, doy + L * b, 4 * m, 4 * m, L, cudaMemcpyDeviceToHost, ctx->d2h_stream));
        CU(ctx, cudaMemcpyAsync(oinf + hb, doi + b, m, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    }
    CU(ctx, cudaStreamSynchronize(ctx->d2h_stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    if (account) account_points(ctx, op, n);  // once per call, whatever the chunking
    return SM2B_OK;
}

sm2b_status invert_range(sm2b_ctx* ctx, int field, size_t pitch, size_t begin, size_t count,
                         const uint32_t* in, uint32_t* out, bool account) {
    if (count == 0) return SM2B_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t L = field_limbs(ctx, field), bytes = 4 * L * count;
    CU(ctx, ctx->in.ensure(bytes));
    CU(ctx, ctx->out.ensure(bytes));
    uint32_t* din = (uint32_t*)ctx->in.p;
    uint32_t* dout = (uint32_t*)ctx->out.p;
    CU(ctx, cudaMemcpy2DAsync(din, 4 * count, in + begin, 4 * pitch, 4 * count, L, cudaMemcpyHostToDevice, ctx->stream));
    sm2b_status st = batch_invert_locked(ctx, field, count, din, dout, account);
    if (st != SM2B_OK) return st;
    CU(ctx, cudaMemcpy2DAsync(out + begin, 4 * pitch, dout, 4 * count, 4 * count, L, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}
}  // namespace gecc_capi

extern "C" {

sm2b_status gecc_batch_invert(sm2b_ctx* ctx, gecc_field field, size_t n, const uint32_t* in,
                              uint32_t* out) {
    if (!ctx || (n > 0 && (!in || !out)) || (unsigned)field > 1) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    if (is_group(ctx)) return group_invert(ctx, field, n, in, out);
    return invert_range(ctx, field, n, 0, n, in, out, true);
}

sm2b_status gecc_batch_padd(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                            const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                            const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || (n > 0 && (!px || !py || !tx || !ty || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    HostPoints p{px, py, pinf}, t{tx, ty, tinf};
    if (is_group(ctx)) return group_points(ctx, OP_PADD, n, nullptr, &p, &t, ox, oy, oinf, nullptr);
    return points_range(ctx, OP_PADD, n, 0, n, nullptr, &p, &t, ox, oy, oinf, nullptr, true);
}
sm2b_status gecc_batch_pdbl(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                            const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || (n > 0 && (!px || !py || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    HostPoints p{px, py, pinf};
    if (is_group(ctx)) return group_points(ctx, OP_PDBL, n, nullptr, &p, nullptr, ox, oy, oinf, nullptr);
    return points_range(ctx, OP_PDBL, n, 0, n, nullptr, &p, nullptr, ox, oy, oinf, nullptr, true);
}
sm2b_status gecc_batch_fpmul(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, uint32_t* ox,
                             uint32_t* oy, uint8_t* oinf) {
    if (!ecdsa_ctx(ctx) || (n > 0 && (!scalars || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    if (is_group(ctx)) return group_points(ctx, OP_FPMUL, n, scalars, nullptr, nullptr, ox, oy, oinf, nullptr);
    return points_range(ctx, OP_FPMUL, n, 0, n, scalars, nullptr, nullptr, ox, oy, oinf, nullptr, true);
}
sm2b_status gecc_batch_fpmul_base(sm2b_ctx* ctx, const gecc_base_table* base, size_t n,
                                  const uint32_t* scalars, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ecdsa_ctx(ctx) || !base || base->owner != ctx || (n > 0 && (!scalars || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    if (is_group(ctx)) return group_points(ctx, OP_FPMUL, n, scalars, nullptr, nullptr, ox, oy, oinf, base);
    return points_range(ctx, OP_FPMUL, n, 0, n, scalars, nullptr, nullptr, ox, oy, oinf, table_for(ctx, base), true);
}
sm2b_status gecc_batch_upmul(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                             const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                             uint8_t* oinf) {
    if (!ecdsa_ctx(ctx) || (n > 0 && (!scalars || !px || !py || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    HostPoints p{px, py, pinf};
    if (is_group(ctx)) return group_points(ctx, OP_UPMUL, n, scalars, &p, nullptr, ox, oy, oinf, nullptr);
    return points_range(ctx, OP_UPMUL, n, 0, n, scalars, &p, nullptr, ox, oy, oinf, nullptr, true);
}

// ------------------------------------------------------------------ base tables
// precompute_base_table (batch_point.cpp:341-350) for any on-curve base point: one windowed
// table per device, built on the GPU; an off-curve point is rejected as the reference does.
sm2b_status gecc_base_table_new(sm2b_ctx* ctx, const uint32_t* x, const uint32_t* y, gecc_base_table** out) {
    if (!ecdsa_ctx(ctx) || !x || !y || !out) return SM2B_ERROR_INVALID_ARGUMENT;
    *out = nullptr;
    gecc_base_table* tb = new (std::nothrow) gecc_base_table();
    if (!tb) return SM2B_ERROR_INTERNAL;
    tb->owner = ctx;
    std::lock_guard<std::mutex> glk(ctx->mu);
    std::vector<sm2b_ctx*> devs = ctx->shards.empty() ? std::vector<sm2b_ctx*>{ctx} : ctx->shards;
    sm2b_status st = SM2B_OK;
    for (sm2b_ctx* d : devs) {
        std::unique_lock<std::mutex> lk(d->mu, std::defer_lock);
        if (d != ctx) lk.lock();
        DeviceGuard g(d->device);
        uint32_t *tab = nullptr, *bases = nullptr, *xy = nullptr;
        uint32_t hxy[16];
        memcpy(hxy, x, 32);
        memcpy(hxy + 8, y, 32);
        cudaError_t e = cudaMalloc(&tab, gtable_words() * 4);
        if (e == cudaSuccess) e = cudaMalloc(&bases, 64 * 16 * 4 * 8);
        if (e == cudaSuccess) e = cudaMalloc(&xy, 64);
        if (e == cudaSuccess) e = cudaMemcpyAsync(xy, hxy, 64, cudaMemcpyHostToDevice, d->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(d->flags, 0, 4, d->stream);
        if (e == cudaSuccess) e = build_base_table(d->curve, xy, tab, bases, d->flags, d->stream);
        *d->hflag = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(d->hflag, d->flags, 4, cudaMemcpyDeviceToHost, d->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
        if (bases) cudaFree(bases);
        if (xy) cudaFree(xy);
        d->launches += 2;
        if (e != cudaSuccess) st = fail(ctx, "gecc_base_table_new", e);
        else if (*d->hflag) st = SM2B_ERROR_MALFORMED_INPUT;  // precompute_base_table: point off curve
        if (st != SM2B_OK) {
            if (tab) cudaFree(tab);
            break;
        }
        tb->tabs.push_back(tab);
    }
    if (st != SM2B_OK) {
        for (size_t i = 0; i < tb->tabs.size(); ++i) {
            DeviceGuard g(devs[i]->device);
            cudaFree(tb->tabs[i]);
        }
        delete tb;
        return st;
    }
    *out = tb;
    return SM2B_OK;
}

void gecc_base_table_free(gecc_base_table* tb) {
    if (!tb) return;
    sm2b_ctx* ctx = tb->owner;
    std::vector<sm2b_ctx*> devs = ctx->shards.empty() ? std::vector<sm2b_ctx*>{ctx} : ctx->shards;
    for (size_t i = 0; i < tb->tabs.size() && i < devs.size(); ++i) {
        DeviceGuard g(devs[i]->device);
        cudaStreamSynchronize(devs[i]->stream);
        cudaFree(tb->tabs[i]);
    }
    delete tb;
}

}  // extern "C"

namespace gecc_capi {
const uint32_t* base_table_for(const sm2b_ctx* shard, const gecc_base_table* base) { return table_for(shard, base); }
}

extern "C" {

// ------------------------------------------------------------------ sm2b_bench_run
// bench.cpp:114-282 on the GPU: seeded synthetic inputs with the reference's stream tags,
// both strategies run once and compared before anything is timed, one discarded warm-up,
// a ledger run (closed forms), then the median of `repeats` timed runs (CUDA events).
//   affine-batch     = the production kernels (k_batch_padd / k_fpmul / k_upmul / k_sign / k_verify)
//   jacobian-serial  = independent per-lane kernels (k_padd_jacobian, k_pmul_serial); sign and
//                      verify have a single GPU implementation, their gate is sign -> verify.
} // extern "C"
namespace {
struct BenchBufs {
    uint32_t *k, *k2, *px, *py, *tx, *ty, *ax, *ay, *bx, *by;
    uint8_t *ai, *bi, *dig, *sec, *pub, *sig, *res;
    int32_t* st;
};
}  // namespace
extern "C" {

sm2b_status sm2b_bench_run(sm2b_ctx* ctx, const char* op, const char* strategy, size_t n,
                           size_t lanes, uint32_t workers, uint64_t seed, uint32_t repeats,
                           sm2b_bench_report* out) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || !op || !strategy || !out) return SM2B_ERROR_INVALID_ARGUMENT;
    static const char* const ops[] = {"padd", "fpmul", "upmul", "sign", "verify"};
    int opi = -1;
    for (int i = 0; i < 5; ++i)
        if (!strcmp(op, ops[i])) opi = i;
    const bool batch = !strcmp(strategy, "affine-batch");
    if (opi < 0 || (!batch && strcmp(strategy, "jacobian-serial")) || n == 0 || repeats == 0)
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (seed == 0) seed = 1;
    if (is_group(ctx)) {  // the benchmark protocol times ONE device: the group's first shard
        sm2b_ctx* first = ctx->shards[0];
        first->lanes = ctx->lanes;
        first->workers = ctx->workers;
        sm2b_status st = sm2b_bench_run(first, op, strategy, n, lanes, workers, seed, repeats, out);
        if (st == SM2B_ERROR_INTERNAL) ctx->last_error = first->last_error;
        return st;
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t cb = Carver::need(32 * n), mb = Carver::need(n);
    CU(ctx, ctx->scratch.ensure(10 * cb + 2 * mb + 2 * cb + Carver::need(65 * n) + Carver::need(64 * n) +
                                mb + Carver::need(4 * n)));
    Carver cv(ctx->scratch.p);
    BenchBufs b;
    b.k = cv.take<uint32_t>(8 * n); b.k2 = cv.take<uint32_t>(8 * n);
    b.px = cv.take<uint32_t>(8 * n); b.py = cv.take<uint32_t>(8 * n);
    b.tx = cv.take<uint32_t>(8 * n); b.ty = cv.take<uint32_t>(8 * n);
    b.ax = cv.take<uint32_t>(8 * n); b.ay = cv.take<uint32_t>(8 * n);
    b.bx = cv.take<uint32_t>(8 * n); b.by = cv.take<uint32_t>(8 * n);
    b.ai = cv.take<uint8_t>(n); b.bi = cv.take<uint8_t>(n);
    b.dig = cv.take<uint8_t>(32 * n); b.sec = cv.take<uint8_t>(32 * n);
    b.pub = cv.take<uint8_t>(65 * n); b.sig = cv.take<uint8_t>(64 * n);
    b.res = cv.take<uint8_t>(n); b.st = cv.take<int32_t>(n);
    cudaStream_t s = ctx->stream;
    CU(ctx, ctx->lane_tabs.ensure(verify_scratch_bytes(n)));  // upmul needs all n lanes covered
    const size_t tab_lanes = n;
    const int cv_ = ctx->curve;
    const uint32_t* gt = ctx->gtab;          // column-buffer kernels
    const uint32_t* gr = ctx->gtab_rec;      // byte-record kernels
    uint8_t* scratch_inf = b.res;  // infinity flags of generated points (never set for 0 < k < n)
    // ---- inputs (bench.cpp:139-140,163,167,194-200)
    if (opi == 0) {
        CU(ctx, launch_seeded_scalars(cv_, n, seed, 0x10000, b.k, s));
        CU(ctx, launch_fpmul(cv_, n, b.k, gt, b.px, b.py, scratch_inf, s));
        CU(ctx, launch_seeded_scalars(cv_, n, seed, 0x20000, b.k, s));
        CU(ctx, launch_fpmul(cv_, n, b.k, gt, b.tx, b.ty, scratch_inf, s));
    } else if (opi <= 2) {
        CU(ctx, launch_seeded_scalars(cv_, n, seed, 0x40000, b.k2, s));
        CU(ctx, launch_fpmul(cv_, n, b.k2, gt, b.px, b.py, scratch_inf, s));
        CU(ctx, launch_seeded_scalars(cv_, n, seed, 0x30000, b.k, s));
    } else {
        CU(ctx, launch_keygen(cv_, n, seed, 0x50000, gr, b.dig, b.pub, s));  // digests = seeded scalars
        CU(ctx, launch_keygen(cv_, n, seed, 0x60000, gr, b.sec, b.pub, s));  // key pairs
        CU(ctx, cudaMemsetAsync(ctx->flags, 0, 4, s));
        CU(ctx, launch_sign(cv_, n, b.dig, b.sec, seed, 0, gr, b.sig, b.st, ctx->flags, s));
    }
    auto run = [&](bool use_batch, uint32_t* ox, uint32_t* oy, uint8_t* oi) -> cudaError_t {
        switch (opi) {
            case 0:
                return use_batch ? launch_batch_padd(cv_, n, b.px, b.py, nullptr, b.tx, b.ty, nullptr, ox, oy, oi, s)
                                 : launch_padd_jacobian(cv_, n, b.px, b.py, nullptr, b.tx, b.ty, nullptr, ox, oy, oi, s);
            case 1:
                return use_batch ? launch_fpmul(cv_, n, b.k, gt, ox, oy, oi, s)
                                 : launch_pmul_serial(cv_, n, b.k, nullptr, nullptr, nullptr, ox, oy, oi, s);
            case 2:
                return use_batch ? launch_upmul(cv_, n, b.k, b.px, b.py, nullptr, ox, oy, oi, (uint32_t*)ctx->lane_tabs.p, s)
                                 : launch_pmul_serial(cv_, n, b.k, b.px, b.py, nullptr, ox, oy, oi, s);
            case 3: {
                cudaError_t e = cudaMemsetAsync(ctx->flags, 0, 4, s);
                if (e != cudaSuccess) return e;
                return launch_sign(cv_, n, b.dig, b.sec, seed, 0, gr, b.sig, b.st, ctx->flags, s);
            }
            default:
                return launch_verify(cv_, n, b.dig, b.pub, b.sig, gr, b.res, (uint32_t*)ctx->lane_tabs.p, tab_lanes, s);
        }
    };
    // ---- equivalence gate
    bool agree = true;
    if (opi <= 2) {
        CU(ctx, run(true, b.ax, b.ay, b.ai));
        CU(ctx, run(false, b.bx, b.by, b.bi));
        std::vector<uint32_t> ha(16 * n), hb(16 * n);
        std::vector<uint8_t> ia(n), ib(n);
        CU(ctx, cudaMemcpyAsync(ha.data(), b.ax, 32 * n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaMemcpyAsync(ha.data() + 8 * n, b.ay, 32 * n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaMemcpyAsync(hb.data(), b.bx, 32 * n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaMemcpyAsync(hb.data() + 8 * n, b.by, 32 * n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaMemcpyAsync(ia.data(), b.ai, n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaMemcpyAsync(ib.data(), b.bi, n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaStreamSynchronize(s));
        agree = ha == hb && ia == ib;
    } else {
        CU(ctx, launch_verify(cv_, n, b.dig, b.pub, b.sig, gr, b.res, (uint32_t*)ctx->lane_tabs.p, tab_lanes, s));
        std::vector<uint8_t> hr(n);
        std::vector<int32_t> hs(n);
        CU(ctx, cudaMemcpyAsync(hr.data(), b.res, n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaMemcpyAsync(hs.data(), b.st, 4 * n, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaStreamSynchronize(s));
        for (size_t i = 0; i < n; ++i) agree = agree && hr[i] == 1 && hs[i] == 0;
    }
    if (!agree) return fail_msg(ctx, "run_bench: strategies disagree, aborting");  // bench.cpp:253-256
    // ---- warm-up, timed repeats (median)
    CU(ctx, run(batch, b.ax, b.ay, b.ai));
    cudaEvent_t e0, e1;
    CU(ctx, cudaEventCreate(&e0));
    CU(ctx, cudaEventCreate(&e1));
    std::vector<float> ms(repeats);
    for (uint32_t r = 0; r < repeats; ++r) {
        cudaEventRecord(e0, s);
        cudaError_t e = run(batch, b.ax, b.ay, b.ai);
        cudaEventRecord(e1, s);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) {
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            return fail(ctx, "bench run", e);
        }
        cudaEventElapsedTime(&ms[r], e0, e1);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::sort(ms.begin(), ms.end());
    ctx->launches += 8 + repeats;
    // ---- report: ledger of one run in the reference's closed forms
    sm2b_op_counts run_ops{0, 0, 0, 0};
    const Ledger t{&run_ops, (uint32_t)lanes ? (uint32_t)lanes : ctx->lanes, workers ? workers : ctx->workers};
    if (batch) {
        if (opi == 0) led_padd(t, n);
        else if (opi == 1) led_fpmul(t, n);
        else if (opi == 2) led_upmul(t, n);
        else if (opi == 3) { led_fpmul(t, n); led_invert(t, n); led(t, 2 * n, n, 0, 0); }
        else { led_invert(t, n); led(t, 2 * n, 0, 0, 0); led_fpmul(t, n); led_upmul(t, n); led_padd(t, n); }
    } else {  // Jacobian pipeline: no inversions inside; padd = 11 modmul + 6 modsub per lane
        if (opi == 0) led(t, 11 * n, 0, 6 * n, 0);
        else led(t, (uint64_t)(256 * 10 + 128 * 16) * n, (uint64_t)256 * 7 * n, (uint64_t)(256 * 4 + 128 * 7) * n, n);
    }
    out->lanes_used = eff_lanes(t, n);
    out->wall_seconds = ms[ms.size() / 2] * 1e-3;
    out->throughput = out->wall_seconds > 0 ? (double)n / out->wall_seconds : 0.0;
    out->ops = run_ops;
    out->modeled_cost = (run_ops.modadd + run_ops.modsub) + 5 * run_ops.modmul + 500 * run_ops.modinv;
    out->equivalence_checked = 1;
    return SM2B_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ MSM
namespace {
sm2b_status msm_args(const sm2b_ctx* ctx, size_t n, const void* scalars, const void* px, const void* py,
                     const void* ox, const void* oy, const void* oinf) {
    if (!ctx || !ox || !oy || !oinf || (n > 0 && (!scalars || !px || !py))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n >= ((size_t)1 << 27)) return SM2B_ERROR_INVALID_ARGUMENT;  // 17 n pair positions are 32-bit, the point index 31
    return SM2B_OK;
}
}  // namespace

extern "C" sm2b_status gecc_msm_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                                    const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                                    uint8_t* oinf) {
    if (msm_args(ctx, n, scalars, px, py, ox, oy, oinf) != SM2B_OK || is_group(ctx)) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    if (n == 0) {  // empty sum = point at infinity
        CU(ctx, cudaMemsetAsync(ox, 0, 4 * ctx->limbs, ctx->stream));
        CU(ctx, cudaMemsetAsync(oy, 0, 4 * ctx->limbs, ctx->stream));
        CU(ctx, cudaMemsetAsync(oinf, 1, 1, ctx->stream));
        return SM2B_OK;
    }
    CU(ctx, ctx->scratch.ensure(msm_scratch_bytes(n, ctx->curve)));
    int launches = 0;
    CU(ctx, launch_msm(ctx->curve, n, scalars, px, py, pinf, ox, oy, oinf, ctx->scratch.p, ctx->stream,
                       &launches, nullptr, MsmAux{ctx->aux_stream, ctx->ev_fork, ctx->ev_join}));
    ctx->launches += launches;
    return SM2B_OK;
}

namespace gecc_capi {
// Scalars (and the mask) go up first: digit extraction and the sort run while the points upload.
// The partial sum stays on the device, packed at ctx->xchg.p; nothing is synchronised.
sm2b_status msm_range_enqueue(sm2b_ctx* ctx, size_t pitch, size_t begin, size_t n, const uint32_t* scalars,
                              const uint32_t* px, const uint32_t* py, const uint8_t* pinf) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t L = (size_t)ctx->limbs;
    uint32_t* packed = (uint32_t*)ctx->xchg.p;
    if (n == 0) {  // empty range: the point at infinity
        CU(ctx, cudaMemsetAsync(packed, 0, 4 * (2 * L + 1), ctx->stream));
        CU(ctx, cudaMemsetAsync(packed + 2 * L, 1, 1, ctx->stream));
        return SM2B_OK;
    }
    const size_t cb = Carver::need(4 * L * n), mb = Carver::need(n);
    CU(ctx, ctx->in.ensure(Carver::need(32 * n) + 2 * cb + mb + 256));
    CU(ctx, ctx->out.ensure(1024));
    Carver ci(ctx->in.p), co(ctx->out.p);
    uint32_t* dox = co.take<uint32_t>(L);
    uint32_t* doy = co.take<uint32_t>(L);
    uint8_t* doi = co.take<uint8_t>(1);
    uint32_t* dk = ci.take<uint32_t>(8 * n);
    uint32_t* dpx = ci.take<uint32_t>(L * n);
    uint32_t* dpy = ci.take<uint32_t>(L * n);
    uint8_t* dpi = pinf ? ci.take<uint8_t>(n) : nullptr;
    EventPool pool;
    cudaEvent_t idle = pool.get(), scalars_up = pool.get(), points_up = pool.get();
    CU(ctx, cudaEventRecord(idle, ctx->stream));
    CU(ctx, cudaStreamWaitEvent(ctx->h2d_stream, idle, 0));
    auto up = [&](const uint32_t* h, uint32_t* d, size_t rows) {
        if (pitch == n) return cudaMemcpyAsync(d, h, 4 * rows * n, cudaMemcpyHostToDevice, ctx->h2d_stream);
        return cudaMemcpy2DAsync(d, 4 * n, h + begin, 4 * pitch, 4 * n, rows, cudaMemcpyHostToDevice, ctx->h2d_stream);
    };
    CU(ctx, up(scalars, dk, 8));
    if (pinf) CU(ctx, cudaMemcpyAsync(dpi, pinf + begin, n, cudaMemcpyHostToDevice, ctx->h2d_stream));
    CU(ctx, cudaEventRecord(scalars_up, ctx->h2d_stream));
    CU(ctx, up(px, dpx, L));
    CU(ctx, up(py, dpy, L));
    CU(ctx, cudaEventRecord(points_up, ctx->h2d_stream));
    CU(ctx, cudaStreamWaitEvent(ctx->stream, scalars_up, 0));
    CU(ctx, ctx->scratch.ensure(msm_scratch_bytes(n, ctx->curve)));
    int launches = 0;
    CU(ctx, launch_msm(ctx->curve, n, dk, dpx, dpy, dpi, dox, doy, doi, ctx->scratch.p, ctx->stream, &launches,
                       points_up, MsmAux{ctx->aux_stream, ctx->ev_fork, ctx->ev_join}));
    CU(ctx, launch_point_pack(ctx->curve, dox, doy, doi, packed, ctx->stream));
    ctx->launches += launches + 1;
    // the events of `pool` are destroyed on return; CUDA keeps what the enqueued waits need
    return SM2B_OK;
}
}  // namespace gecc_capi

extern "C" {

sm2b_status gecc_msm(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                     const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                     uint8_t* oinf) {
    if (msm_args(ctx, n, scalars, px, py, ox, oy, oinf) != SM2B_OK) return SM2B_ERROR_INVALID_ARGUMENT;
    const size_t L = (size_t)ctx->limbs;
    if (n == 0) {  // empty sum = point at infinity
        memset(ox, 0, 4 * L);
        memset(oy, 0, 4 * L);
        *oinf = 1;
        return SM2B_OK;
    }
    if (is_group(ctx)) return group_msm(ctx, n, scalars, px, py, pinf, ox, oy, oinf);
    sm2b_status st = msm_range_enqueue(ctx, n, 0, n, scalars, px, py, pinf);
    if (st != SM2B_OK) return st;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    uint32_t host[2 * 12 + 1];
    CU(ctx, cudaMemcpyAsync(host, ctx->xchg.p, 4 * (2 * L + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    memcpy(ox, host, 4 * L);
    memcpy(oy, host + L, 4 * L);
    *oinf = host[2 * L] ? 1 : 0;
    return SM2B_OK;
}

// Every rank's partial sum -> the total on every rank (multi-process MSM).
sm2b_status gecc_msm_combine_dev(sm2b_ctx* ctx, uint32_t* x, uint32_t* y, uint8_t* inf) {
    if (!ctx || is_group(ctx) || !x || !y || !inf) return SM2B_ERROR_INVALID_ARGUMENT;
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (!ctx->nccl_comm) return fail_msg(ctx, "gecc_msm_combine_dev: no communicator (call gecc_comm_init_rank)");
        DeviceGuard g(ctx->device);
        CU(ctx, launch_point_pack(ctx->curve, x, y, inf, (uint32_t*)ctx->xchg.p, ctx->stream));
        ctx->launches += 1;
    }
    sm2b_status st = comm_combine_enqueue(ctx);
    if (st != SM2B_OK) return st;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, launch_point_unpack(ctx->curve, (const uint32_t*)ctx->xchg.p, x, y, inf, ctx->stream));
    ctx->launches += 1;
    return SM2B_OK;
}

}  // extern "C"
