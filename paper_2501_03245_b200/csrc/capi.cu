// C ABI of libgecc_b200.so (include/gecc_b200.h).  Host side of the drop-in
// boundary: mirrors the reference's capi.cpp semantics (argument checks, status
// codes, per-lane reporting, ledger) and hands all arithmetic to CUDA kernels.
// There is no CPU compute path in this file.
#include <cuda_runtime.h>

#include <algorithm>
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
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;  // copy engines of the pipelined host API
    cudaStream_t aux_stream = nullptr;  // second compute stream: consecutive chunk kernels overlap their tails
    sm2b_op_counts ledger{0, 0, 0, 0};
    uint64_t launches = 0;
    std::string last_error;
    DevBuf in, out, scratch;
    DevBuf batch_tmp;  // tile totals of the tiled batch_padd form
    DevBuf lane_tabs;  // per-lane point tables of the verify kernel (512 B per lane, capped)
    uint32_t* gtab = nullptr;   // fixed-base table (Montgomery form), built on the GPU at creation
    uint32_t* gtab_rec = nullptr;  // table of the byte-record kernels (== gtab on SM2, plain form on secp256k1)
    uint32_t* flags = nullptr;  // device word: malformed-call flag of sign / ecdh
    int limbs = 8;              // 32-bit limbs per coordinate (12 on BLS12-381)
    uint32_t* hflag = nullptr;  // pinned host word: the flag comes back without blocking the enqueueing thread
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // fork / join of the two-stream MSM tree levels
    bool ledger_hold = false;   // a pipelined host call runs its chunks with the ledger held and accounts once
    sm2b_op_counts ledger_sink{0, 0, 0, 0};
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

}  // namespace

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
        delete ctx;
        return nullptr;
    }
    ctx->sm_count = prop.multiProcessorCount;
    ctx->stream = ctx->own_stream;
    if (cudaHostAlloc((void**)&ctx->hflag, 64, cudaHostAllocDefault) != cudaSuccess) {
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
        ctx->batch_tmp.release();
        ctx->lane_tabs.release();
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
    if (!ctx || (n > 0 && (!a || !out)) || (unsigned)op > 6 || (unsigned)field > 1)
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
    if (!ctx || (n > 0 && (!a || !out)) || (unsigned)op > 6 || (unsigned)field > 1)
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n > 0 && op <= GECC_OP_MOD_SUB && !b) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    uint32_t *da, *db, *dout;
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        DeviceGuard g(ctx->device);
        const size_t bytes = 4 * field_limbs(ctx, field) * n;
        CU(ctx, ctx->in.ensure(2 * Carver::need(bytes)));
        CU(ctx, ctx->out.ensure(Carver::need(bytes)));
        Carver ci(ctx->in.p);
        da = ci.take<uint32_t>(bytes / 4);
        db = ci.take<uint32_t>(bytes / 4);
        dout = (uint32_t*)ctx->out.p;
        CU(ctx, cudaMemcpyAsync(da, a, bytes, cudaMemcpyHostToDevice, ctx->stream));
        if (b) CU(ctx, cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
    sm2b_status st = gecc_field_op_dev(ctx, field, op, n, da, b ? db : nullptr, dout);
    if (st != SM2B_OK) return st;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, cudaMemcpyAsync(out, dout, 4 * field_limbs(ctx, field) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

void gecc_set_batch_form(int form) { set_batch_form(form < 0 || form > 7 ? 0 : form); }
void gecc_set_msm_form(int form) { set_msm_form(form < 0 || form > 3 ? 0 : form); }

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
void led_fpmul(const Ledger& L, uint64_t n) {
    if (n) led(L, 256 * (6 * n + 3 * (eff_lanes(L, n) - 1)), 0, 256 * 7 * n, 256);
}
void led_upmul(const Ledger& L, uint64_t n) {
    if (n) led(L, 256 * (14 * n + 3 * (eff_lanes(L, n) - 1)), 256 * 5 * n, 256 * 11 * n, 256);
}
Ledger ledger_of(sm2b_ctx* ctx) {
    return Ledger{ctx->ledger_hold ? &ctx->ledger_sink : &ctx->ledger, ctx->lanes, ctx->workers};
}
}  // namespace

// ------------------------------------------------------------------ host-API pipeline
// The byte-record entry points split a large batch into chunks and run three streams:
// H2D of chunk c+1, the kernel of chunk c and D2H of chunk c-1 overlap (events order
// them).  With pinned caller buffers the copies are truly asynchronous; with pageable
// buffers CUDA stages them and the result is the same, only less overlapped.
} // extern "C"
namespace {
constexpr size_t PIPE_MIN_CHUNK = (size_t)1 << 17;
constexpr size_t PIPE_HEAD_CHUNK = (size_t)1 << 16;
constexpr int PIPE_MAX_CHUNKS = 4;

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
}  // namespace
extern "C" {

// ------------------------------------------------------------------ protocol layer
} // extern "C"
namespace {
constexpr size_t VERIFY_SCRATCH_MAX_LANES = (size_t)1 << 22;  // 2 GiB of lane tables at most
// returns the number of lanes the verify scratch covers (0 on allocation failure)
size_t ensure_lane_tabs(sm2b_ctx* ctx, size_t count) {
    const size_t lanes = count < VERIFY_SCRATCH_MAX_LANES ? count : VERIFY_SCRATCH_MAX_LANES;
    return ctx->lane_tabs.ensure(verify_scratch_bytes(lanes)) == cudaSuccess ? lanes : 0;
}
}  // namespace
extern "C" {
sm2b_status gecc_verify_dev(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                            const uint8_t* publics, const uint8_t* signatures,
                            uint8_t* results) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (count > 0 && (!digests || !publics || !signatures || !results)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t tab_lanes = ensure_lane_tabs(ctx, count);
    CU(ctx, launch_verify(ctx->curve, count, digests, publics, signatures, ctx->gtab_rec, results,
                          (uint32_t*)ctx->lane_tabs.p, tab_lanes, ctx->stream));
    ctx->launches += count ? 1 : 0;
    led_invert(ledger_of(ctx), count);
    led(ledger_of(ctx), 2 * count, 0, 0, 0);
    led_fpmul(ledger_of(ctx), count);
    led_upmul(ledger_of(ctx), count);
    led_padd(ledger_of(ctx), count);
    return SM2B_OK;
}

sm2b_status sm2b_verify(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                        const uint8_t* publics, const uint8_t* signatures, uint8_t* results) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (count > 0 && (!digests || !publics || !signatures || !results)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
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
    led_invert(ledger_of(ctx), count);
    led(ledger_of(ctx), 2 * count, 0, 0, 0);
    led_fpmul(ledger_of(ctx), count);
    led_upmul(ledger_of(ctx), count);
    led_padd(ledger_of(ctx), count);
    CU(ctx, cudaStreamSynchronize(ctx->d2h_stream));
    CU(ctx, cudaStreamSynchronize(ctx->aux_stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

sm2b_status gecc_sign_dev(sm2b_ctx* ctx, size_t count, const uint8_t* digests,
                          const uint8_t* secrets, uint64_t nonce_seed, uint64_t lane_base,
                          uint8_t* signatures, int32_t* lane_status) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (count > 0 && (!digests || !secrets || !signatures || !lane_status)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (nonce_seed == 0) return fail_msg(ctx, "device signing needs a non-zero nonce seed");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, cudaMemsetAsync(ctx->flags, 0, 4, ctx->stream));
    CU(ctx, launch_sign(ctx->curve, count, digests, secrets, nonce_seed, lane_base, ctx->gtab_rec,
                        signatures, lane_status, ctx->flags, ctx->stream));
    ctx->launches += count ? 1 : 0;
    led_fpmul(ledger_of(ctx), count);
    led_invert(ledger_of(ctx), count);
    led(ledger_of(ctx), 2 * count, count, 0, 0);
    return SM2B_OK;
}

namespace {
uint64_t system_seed() {  // seed == 0: system entropy (capi.cpp:75-79), drawn on the host
    uint64_t v = 0;
    FILE* f = fopen("/dev/urandom", "rb");
    if (f) {
        if (fread(&v, 1, sizeof v, f) != sizeof v) v = 0;
        fclose(f);
    }
    static uint64_t counter = 0;
    v ^= 0x9E3779B97F4A7C15ull * (++counter) ^ (uint64_t)(uintptr_t)&v;
    return v ? v : 1;
}

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

sm2b_status gecc_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                      uint64_t nonce_seed, uint64_t lane_base, uint8_t* signatures,
                      int32_t* lane_status) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (count > 0 && (!digests || !secrets || !signatures)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (nonce_seed == 0) nonce_seed = system_seed();
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
                            dsig + 64 * b, dst + b, ctx->flags, ks));
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
    led_fpmul(ledger_of(ctx), count);
    led_invert(ledger_of(ctx), count);
    led(ledger_of(ctx), 2 * count, count, 0, 0);
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

sm2b_status gecc_keygen(sm2b_ctx* ctx, uint64_t seed, uint64_t lane_base, size_t count,
                        uint8_t* secrets, uint8_t* publics) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (count > 0 && (!secrets || !publics))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    if (seed == 0) seed = system_seed();
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->out.ensure(Carver::need(32 * count) + Carver::need(65 * count)));
    Carver co(ctx->out.p);
    uint8_t* dsec = co.take<uint8_t>(32 * count);
    uint8_t* dpub = co.take<uint8_t>(65 * count);
    CU(ctx, launch_keygen(ctx->curve, count, seed, lane_base, ctx->gtab_rec, dsec, dpub, ctx->stream));
    ctx->launches += 1;
    led_fpmul(ledger_of(ctx), count);
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
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (count > 0 && (!secrets || !peers || !shared))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (count == 0) return SM2B_OK;
    std::vector<int32_t> hst(count);
    uint32_t flag = 0;
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
                            tab_lanes, ctx->stream));
        ctx->launches += 1;
        led_upmul(ledger_of(ctx), count);
        CU(ctx, cudaMemcpyAsync(&flag, ctx->flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaMemcpyAsync(hst.data(), dst, 4 * count, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        if (flag) return SM2B_ERROR_MALFORMED_INPUT;  // Scalar::checked on a secret (capi.cpp:241)
        CU(ctx, cudaMemcpyAsync(shared, dsh, 32 * count, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return report_lanes(hst.data(), count, lane_status);
}

// ------------------------------------------------------------------ batch layer
sm2b_status gecc_batch_invert_dev(sm2b_ctx* ctx, gecc_field field, size_t n, const uint32_t* in,
                                  uint32_t* out) {
    if (!ctx || (n > 0 && (!in || !out)) || (unsigned)field > 1) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, launch_batch_invert(ctx->curve, field, n, in, out, ctx->stream));
    ctx->launches += n ? 1 : 0;
    led_invert(ledger_of(ctx), n);
    return SM2B_OK;
}
sm2b_status gecc_batch_padd_dev(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                                const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                                const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || (n > 0 && (!px || !py || !tx || !ty || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->batch_tmp.ensure(batch_padd_scratch_bytes(n)));
    CU(ctx, launch_batch_padd(ctx->curve, n, px, py, pinf, tx, ty, tinf, ox, oy, oinf, ctx->stream,
                              ctx->batch_tmp.p));
    ctx->launches += n ? 1 : 0;
    led_padd(ledger_of(ctx), n);
    return SM2B_OK;
}
sm2b_status gecc_batch_pdbl_dev(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                                const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || (n > 0 && (!px || !py || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, launch_batch_pdbl(ctx->curve, n, px, py, pinf, ox, oy, oinf, ctx->stream));
    ctx->launches += n ? 1 : 0;
    if (n) led(ledger_of(ctx), 7 * n - 3, 4 * n, 4 * n, 1);
    return SM2B_OK;
}
sm2b_status gecc_batch_fpmul_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, uint32_t* ox,
                                 uint32_t* oy, uint8_t* oinf) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (n > 0 && (!scalars || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, launch_fpmul(ctx->curve, n, scalars, ctx->gtab, ox, oy, oinf, ctx->stream));
    ctx->launches += n ? 1 : 0;
    led_fpmul(ledger_of(ctx), n);
    return SM2B_OK;
}
sm2b_status gecc_batch_upmul_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars,
                                 const uint32_t* px, const uint32_t* py, const uint8_t* pinf,
                                 uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (n > 0 && (!scalars || !px || !py || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->lane_tabs.ensure(verify_scratch_bytes(n)));
    CU(ctx, launch_upmul(ctx->curve, n, scalars, px, py, pinf, ox, oy, oinf, (uint32_t*)ctx->lane_tabs.p,
                         ctx->stream));
    ctx->launches += n ? 1 : 0;
    led_upmul(ledger_of(ctx), n);
    return SM2B_OK;
}

}  // extern "C"
namespace {
// Host-pointer wrapper shared by the column-buffer entry points: stages up to
// three column inputs (+ up to two infinity masks), runs `body` with the device
// pointers, then returns one output point buffer.
struct HostPoints {
    const uint32_t* x;
    const uint32_t* y;
    const uint8_t* inf;
};
// `body(m, ...)` enqueues the kernel for m elements on ctx->stream; `account()` advances the
// ledger once for the whole call.  Large batches are cut into chunks: every chunk has its own
// compact column buffers on the device (count = chunk length, so the kernels are unchanged),
// filled and drained with strided 2-D copies, and upload / kernel / download of successive
// chunks overlap on three streams (PCIe is full duplex).
template <class Body, class Account>
sm2b_status run_points(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const HostPoints* p,
                       const HostPoints* t, uint32_t* ox, uint32_t* oy, uint8_t* oinf, Body body,
                       Account account) {
    const size_t L = (size_t)ctx->limbs, pb = 4 * L * n;  // bytes per coordinate column buffer
    const size_t cb = Carver::need(pb), mb = Carver::need(n);
    uint32_t *dk = nullptr, *dpx = nullptr, *dpy = nullptr, *dtx = nullptr, *dty = nullptr;
    uint8_t *dpi = nullptr, *dti = nullptr;
    uint32_t *dox, *doy;
    uint8_t* doi;
    const Chunks ch(n >= ((size_t)1 << 19) ? n : 1, false);  // small batches: one chunk, one copy each
    const int chunks = n >= ((size_t)1 << 19) ? ch.n : 1;
    std::unique_lock<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, ctx->in.ensure(5 * cb + 2 * mb));
    CU(ctx, ctx->out.ensure(2 * cb + mb));
    Carver ci(ctx->in.p), co(ctx->out.p);
    dox = co.take<uint32_t>(L * n);
    doy = co.take<uint32_t>(L * n);
    doi = co.take<uint8_t>(n);
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
    ctx->ledger_hold = true;
    sm2b_status st = SM2B_OK;
    for (int c = 0; c < chunks && st == SM2B_OK; ++c) {
        const size_t b = chunks == 1 ? 0 : ch.begin(c), m = chunks == 1 ? n : ch.len(c);
        // rows x m block of a host column buffer (row pitch n) -> compact device block (row pitch m)
        auto up = [&](const uint32_t* h, uint32_t* d, size_t rows) {
            return cudaMemcpy2DAsync(d + rows * b, 4 * m, h + b, 4 * n, 4 * m, rows, cudaMemcpyHostToDevice,
                                     ctx->h2d_stream);
        };
        auto upm = [&](const uint8_t* h, uint8_t* d) {
            return cudaMemcpyAsync(d + b, h + b, m, cudaMemcpyHostToDevice, ctx->h2d_stream);
        };
        cudaError_t e = cudaSuccess;
        if (scalars && e == cudaSuccess) e = up(scalars, dk, 8);
        if (p && e == cudaSuccess) e = up(p->x, dpx, L);
        if (p && e == cudaSuccess) e = up(p->y, dpy, L);
        if (p && p->inf && e == cudaSuccess) e = upm(p->inf, dpi);
        if (t && e == cudaSuccess) e = up(t->x, dtx, L);
        if (t && e == cudaSuccess) e = up(t->y, dty, L);
        if (t && t->inf && e == cudaSuccess) e = upm(t->inf, dti);
        cudaEvent_t upe = pool.get(), done = pool.get();
        if (e == cudaSuccess) e = cudaEventRecord(upe, ctx->h2d_stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->stream, upe, 0);
        if (e != cudaSuccess) { ctx->ledger_hold = false; return fail(ctx, "run_points upload", e); }
        lk.unlock();  // the _dev entry points take the lock themselves
        st = body(m, dk ? dk + 8 * b : nullptr, dpx ? dpx + L * b : nullptr, dpy ? dpy + L * b : nullptr,
                  dpi ? dpi + b : nullptr, dtx ? dtx + L * b : nullptr, dty ? dty + L * b : nullptr,
                  dti ? dti + b : nullptr, dox + L * b, doy + L * b, doi + b);
        lk.lock();
        if (st != SM2B_OK) break;
        e = cudaEventRecord(done, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->d2h_stream, done, 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(ox + b, 4 * n, dox + L * b, 4 * m, 4 * m, L, cudaMemcpyDeviceToHost, ctx->d2h_stream);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(oy + b, 4 * n, doy + L * b, 4 * m, 4 * m, L, cudaMemcpyDeviceToHost, ctx->d2h_stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(oinf + b, doi + b, m, cudaMemcpyDeviceToHost, ctx->d2h_stream);
        if (e != cudaSuccess) { ctx->ledger_hold = false; return fail(ctx, "run_points download", e); }
    }
    ctx->ledger_hold = false;
    cudaError_t e1 = cudaStreamSynchronize(ctx->d2h_stream), e2 = cudaStreamSynchronize(ctx->stream);
    if (st != SM2B_OK) return st;
    if (e1 != cudaSuccess) return fail(ctx, "run_points sync", e1);
    if (e2 != cudaSuccess) return fail(ctx, "run_points sync", e2);
    account();
    return SM2B_OK;
}
}  // namespace
extern "C" {

sm2b_status gecc_batch_invert(sm2b_ctx* ctx, gecc_field field, size_t n, const uint32_t* in,
                              uint32_t* out) {
    if (!ctx || (n > 0 && (!in || !out)) || (unsigned)field > 1) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    uint32_t *din, *dout;
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        DeviceGuard g(ctx->device);
        const size_t bytes = 4 * field_limbs(ctx, field) * n;
        CU(ctx, ctx->in.ensure(bytes));
        CU(ctx, ctx->out.ensure(bytes));
        din = (uint32_t*)ctx->in.p;
        dout = (uint32_t*)ctx->out.p;
        CU(ctx, cudaMemcpyAsync(din, in, bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
    sm2b_status st = gecc_batch_invert_dev(ctx, field, n, din, dout);
    if (st != SM2B_OK) return st;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    CU(ctx, cudaMemcpyAsync(out, dout, 4 * field_limbs(ctx, field) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

sm2b_status gecc_batch_padd(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                            const uint8_t* pinf, const uint32_t* tx, const uint32_t* ty,
                            const uint8_t* tinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || (n > 0 && (!px || !py || !tx || !ty || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    HostPoints p{px, py, pinf}, t{tx, ty, tinf};
    return run_points(ctx, n, nullptr, &p, &t, ox, oy, oinf,
                      [&](size_t m, uint32_t*, uint32_t* dpx, uint32_t* dpy, uint8_t* dpi, uint32_t* dtx,
                          uint32_t* dty, uint8_t* dti, uint32_t* dox, uint32_t* doy, uint8_t* doi) {
                          return gecc_batch_padd_dev(ctx, m, dpx, dpy, dpi, dtx, dty, dti, dox, doy, doi);
                      },
                      [&] { led_padd(ledger_of(ctx), n); });
}
sm2b_status gecc_batch_pdbl(sm2b_ctx* ctx, size_t n, const uint32_t* px, const uint32_t* py,
                            const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    if (!ctx || (n > 0 && (!px || !py || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    HostPoints p{px, py, pinf};
    return run_points(ctx, n, nullptr, &p, nullptr, ox, oy, oinf,
                      [&](size_t m, uint32_t*, uint32_t* dpx, uint32_t* dpy, uint8_t* dpi, uint32_t*, uint32_t*,
                          uint8_t*, uint32_t* dox, uint32_t* doy, uint8_t* doi) {
                          return gecc_batch_pdbl_dev(ctx, m, dpx, dpy, dpi, dox, doy, doi);
                      },
                      [&] { led(ledger_of(ctx), 7 * n - 3, 4 * n, 4 * n, 1); });
}
sm2b_status gecc_batch_fpmul(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, uint32_t* ox,
                             uint32_t* oy, uint8_t* oinf) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (n > 0 && (!scalars || !ox || !oy || !oinf))) return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    return run_points(ctx, n, scalars, nullptr, nullptr, ox, oy, oinf,
                      [&](size_t m, uint32_t* dk, uint32_t*, uint32_t*, uint8_t*, uint32_t*, uint32_t*, uint8_t*,
                          uint32_t* dox, uint32_t* doy, uint8_t* doi) {
                          return gecc_batch_fpmul_dev(ctx, m, dk, dox, doy, doi);
                      },
                      [&] { led_fpmul(ledger_of(ctx), n); });
}
sm2b_status gecc_batch_upmul(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                             const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                             uint8_t* oinf) {
    if (ctx && curve_is_bls(ctx->curve)) return SM2B_ERROR_INVALID_ARGUMENT;  // ECDSA layer: 256-bit curves only
    if (!ctx || (n > 0 && (!scalars || !px || !py || !ox || !oy || !oinf)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n == 0) return SM2B_OK;
    HostPoints p{px, py, pinf};
    return run_points(ctx, n, scalars, &p, nullptr, ox, oy, oinf,
                      [&](size_t m, uint32_t* dk, uint32_t* dpx, uint32_t* dpy, uint8_t* dpi, uint32_t*, uint32_t*,
                          uint8_t*, uint32_t* dox, uint32_t* doy, uint8_t* doi) {
                          return gecc_batch_upmul_dev(ctx, m, dk, dpx, dpy, dpi, dox, doy, doi);
                      },
                      [&] { led_upmul(ledger_of(ctx), n); });
}

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

sm2b_status gecc_msm_dev(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                         const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                         uint8_t* oinf) {
    if (!ctx || !ox || !oy || !oinf || (n > 0 && (!scalars || !px || !py)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n >= ((size_t)1 << 31)) return SM2B_ERROR_INVALID_ARGUMENT;  // point index is 31 bits
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

sm2b_status gecc_msm(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px,
                     const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                     uint8_t* oinf) {
    if (!ctx || !ox || !oy || !oinf || (n > 0 && (!scalars || !px || !py)))
        return SM2B_ERROR_INVALID_ARGUMENT;
    if (n >= ((size_t)1 << 31)) return SM2B_ERROR_INVALID_ARGUMENT;  // point index is 31 bits
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t L = (size_t)ctx->limbs;
    const size_t cb = Carver::need(4 * L * n), mb = Carver::need(n);
    CU(ctx, ctx->in.ensure(Carver::need(32 * n) + 2 * cb + mb + 256));
    CU(ctx, ctx->out.ensure(1024));
    Carver ci(ctx->in.p), co(ctx->out.p);
    uint32_t* dox = co.take<uint32_t>(L);
    uint32_t* doy = co.take<uint32_t>(L);
    uint8_t* doi = co.take<uint8_t>(1);
    if (n == 0) {  // empty sum = point at infinity
        memset(ox, 0, 4 * L);
        memset(oy, 0, 4 * L);
        *oinf = 1;
        return SM2B_OK;
    }
    uint32_t* dk = ci.take<uint32_t>(8 * n);
    uint32_t* dpx = ci.take<uint32_t>(L * n);
    uint32_t* dpy = ci.take<uint32_t>(L * n);
    uint8_t* dpi = pinf ? ci.take<uint8_t>(n) : nullptr;
    // scalars (and the mask) first: digit extraction and the sort run while the points upload
    EventPool pool;
    cudaEvent_t idle = pool.get(), scalars_up = pool.get(), points_up = pool.get();
    CU(ctx, cudaEventRecord(idle, ctx->stream));
    CU(ctx, cudaStreamWaitEvent(ctx->h2d_stream, idle, 0));
    CU(ctx, cudaMemcpyAsync(dk, scalars, 32 * n, cudaMemcpyHostToDevice, ctx->h2d_stream));
    if (pinf) CU(ctx, cudaMemcpyAsync(dpi, pinf, n, cudaMemcpyHostToDevice, ctx->h2d_stream));
    CU(ctx, cudaEventRecord(scalars_up, ctx->h2d_stream));
    CU(ctx, cudaMemcpyAsync(dpx, px, 4 * L * n, cudaMemcpyHostToDevice, ctx->h2d_stream));
    CU(ctx, cudaMemcpyAsync(dpy, py, 4 * L * n, cudaMemcpyHostToDevice, ctx->h2d_stream));
    CU(ctx, cudaEventRecord(points_up, ctx->h2d_stream));
    CU(ctx, cudaStreamWaitEvent(ctx->stream, scalars_up, 0));
    CU(ctx, ctx->scratch.ensure(msm_scratch_bytes(n, ctx->curve)));
    int launches = 0;
    CU(ctx, launch_msm(ctx->curve, n, dk, dpx, dpy, dpi, dox, doy, doi, ctx->scratch.p, ctx->stream, &launches,
                       points_up, MsmAux{ctx->aux_stream, ctx->ev_fork, ctx->ev_join}));
    ctx->launches += launches;
    CU(ctx, cudaMemcpyAsync(ox, dox, 4 * L, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaMemcpyAsync(oy, doy, 4 * L, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaMemcpyAsync(oinf, doi, 1, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return SM2B_OK;
}

}  // extern "C"
