// GROUP contexts: one sm2b_ctx that drives several CUDA devices, and the
// MSM exchange over NCCL.
//
// Every host-pointer entry point splits its batch into contiguous lane ranges, one per device,
// and runs the DEVICE context's own entry point on each range from its own host thread: each
// device uploads, computes and downloads its own slice, there is no data-path collective.  The
// global lane index stays the nonce stream id (protocol.cpp:125-126), so the bytes do not depend
// on the device count.  The reference's context owns its workers the same way (capi.cpp:94-107,
// worker_pool.cpp); here a "worker" is a GPU.
//
// MSM shards by point range.  Each device leaves its partial sum packed in its exchange buffer;
// ONE ncclAllGather of 2L + 1 words per device moves them, then a single-thread kernel adds the
// ndev points (EC addition is not an NCCL reduction operator).  NCCL is loaded with dlopen at the
// first use, so the ECDSA path has no dependency on it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>

#include "capi_ctx.h"

using namespace gecc;

namespace gecc_capi {
const uint32_t* base_table_for(const sm2b_ctx* shard, const gecc_base_table* base);

namespace {

// ---------------------------------------------------------------- NCCL, loaded on demand
struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // libnccl.so.2 matches an already loaded copy (e.g. the one a PyTorch process brought) by soname
        a.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!a.handle) a.handle = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!a.handle) return a;
#define GECC_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.handle, name))
        GECC_SYM(GetUniqueId, "ncclGetUniqueId");
        GECC_SYM(CommInitRank, "ncclCommInitRank");
        GECC_SYM(CommInitAll, "ncclCommInitAll");
        GECC_SYM(CommDestroy, "ncclCommDestroy");
        GECC_SYM(AllGather, "ncclAllGather");
        GECC_SYM(GroupStart, "ncclGroupStart");
        GECC_SYM(GroupEnd, "ncclGroupEnd");
        GECC_SYM(GetErrorString, "ncclGetErrorString");
#undef GECC_SYM
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommInitAll && a.CommDestroy && a.AllGather && a.GroupStart &&
               a.GroupEnd && a.GetErrorString;
        return a;
    }();
    return api;
}

sm2b_status nccl_fail(sm2b_ctx* ctx, const char* what, ncclResult_t r) {
    ctx->last_error = std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
    return SM2B_ERROR_INTERNAL;
}
sm2b_status cuda_fail(sm2b_ctx* ctx, const char* what, cudaError_t e) {
    ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return SM2B_ERROR_INTERNAL;
}

size_t packed_words(const sm2b_ctx* ctx) { return 2 * (size_t)ctx->limbs + 1; }
// exchange buffer: [0, W) this shard's partial sum, [W, W + nranks * W) the gathered partial sums
uint32_t* xchg_mine(sm2b_ctx* ctx) { return (uint32_t*)ctx->xchg.p; }
uint32_t* xchg_all(sm2b_ctx* ctx) { return (uint32_t*)ctx->xchg.p + 64; }

// runs fn(shard index) on one host thread per shard; returns the first non-OK status in shard order
template <class Fn>
sm2b_status for_each_shard(sm2b_ctx* ctx, Fn fn) {
    const size_t k = ctx->shards.size();
    std::vector<sm2b_status> st(k, SM2B_OK);
    std::vector<std::thread> th;
    th.reserve(k);
    for (size_t i = 1; i < k; ++i) th.emplace_back([&, i] { st[i] = fn(i); });
    st[0] = fn(0);  // the calling thread serves the first shard
    for (auto& t : th) t.join();
    for (size_t i = 0; i < k; ++i)
        if (st[i] != SM2B_OK) {
            if (st[i] == SM2B_ERROR_INTERNAL) ctx->last_error = ctx->shards[i]->last_error;
            return st[i];
        }
    return SM2B_OK;
}

bool distinct_devices(const sm2b_ctx* ctx) {
    for (size_t i = 0; i < ctx->shards.size(); ++i)
        for (size_t j = i + 1; j < ctx->shards.size(); ++j)
            if (ctx->shards[i]->device == ctx->shards[j]->device) return false;
    return true;
}

}  // namespace

// ---------------------------------------------------------------- lifetime
sm2b_ctx* group_new(gecc_curve curve, int ndev, const int* devices) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        fprintf(stderr, "gecc_b200: no usable CUDA device (this library has no CPU path)\n");
        return nullptr;
    }
    if (ndev <= 0) {
        ndev = count;
        devices = nullptr;
    }
    if (!devices && ndev > count) return nullptr;
    if (ndev > 64) return nullptr;
    sm2b_ctx* ctx = new (std::nothrow) sm2b_ctx();
    if (!ctx) return nullptr;
    ctx->curve = (int)curve;
    ctx->limbs = curve_limbs(ctx->curve);
    for (int i = 0; i < ndev; ++i) {
        const int dev = devices ? devices[i] : i;
        sm2b_ctx* s = (dev >= 0 && dev < count) ? gecc_ctx_new(curve, dev) : nullptr;
        if (!s) {
            for (sm2b_ctx* made : ctx->shards) sm2b_ctx_free(made);
            delete ctx;
            return nullptr;
        }
        ctx->shards.push_back(s);
    }
    ctx->device = ctx->shards[0]->device;
    ctx->sm_count = ctx->shards[0]->sm_count;
    // the MSM exchange: NCCL communicators for all shards at once (one process, several devices).
    // Created lazily by the first gecc_msm (NCCL start-up is slow and the ECDSA path never needs it).
    return ctx;
}

void comm_release(sm2b_ctx* ctx) {
    if (ctx->nccl_comm && ctx->nccl_owned && nccl().ok) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
    ctx->nccl_owned = false;
}

void group_free(sm2b_ctx* ctx) {
    for (sm2b_ctx* s : ctx->shards) sm2b_ctx_free(s);  // releases each shard's communicator
    ctx->shards.clear();
    delete ctx;
}

// ---------------------------------------------------------------- lane-sharded entry points
sm2b_status group_verify(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* publics,
                         const uint8_t* signatures, uint8_t* results) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    sm2b_status st = for_each_shard(ctx, [&](size_t i) {
        size_t b, e;
        shard_range(count, i, k, &b, &e);
        return sm2b_verify(ctx->shards[i], e - b, digests + 32 * b, publics + 65 * b, signatures + 64 * b, results + b);
    });
    if (st == SM2B_OK) account_verify(ctx, count);
    return st;
}

namespace {
// sign / sign_nonces: a zero or oversize secret anywhere fails the WHOLE call (capi.cpp:181-184).
// A shard that sees one returns MALFORMED_INPUT without writing; the others may already have
// written their slices, so the outputs are cleared before the failure is reported.
template <class Fn>
sm2b_status sign_sharded(sm2b_ctx* ctx, size_t count, uint8_t* signatures, int32_t* lane_status, Fn call) {
    const size_t k = ctx->shards.size();
    std::vector<sm2b_status> st(k, SM2B_OK);
    std::vector<std::thread> th;
    for (size_t i = 1; i < k; ++i) th.emplace_back([&, i] { st[i] = call(i); });
    st[0] = call(0);
    for (auto& t : th) t.join();
    for (size_t i = 0; i < k; ++i)
        if (st[i] == SM2B_ERROR_MALFORMED_INPUT || st[i] == SM2B_ERROR_INTERNAL || st[i] == SM2B_ERROR_INVALID_ARGUMENT) {
            if (st[i] == SM2B_ERROR_INTERNAL) ctx->last_error = ctx->shards[i]->last_error;
            memset(signatures, 0, 64 * count);
            if (lane_status) memset(lane_status, 0, 4 * count);
            return st[i];
        }
    account_sign(ctx, count);
    // lane_status == NULL: every shard returned the code of ITS first failing lane (capi.cpp:64-73);
    // the first non-OK in shard order is the first failing lane of the whole batch
    for (size_t i = 0; i < k; ++i)
        if (st[i] != SM2B_OK) return st[i];
    return SM2B_OK;
}
}  // namespace

sm2b_status group_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                       uint64_t nonce_seed, uint64_t lane_base, uint8_t* signatures, int32_t* lane_status) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    return sign_sharded(ctx, count, signatures, lane_status, [&](size_t i) {
        size_t b, e;
        shard_range(count, i, k, &b, &e);
        return gecc_sign(ctx->shards[i], e - b, digests + 32 * b, secrets + 32 * b, nonce_seed, lane_base + b,
                         signatures + 64 * b, lane_status ? lane_status + b : nullptr);
    });
}

sm2b_status group_sign_nonces(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                              const uint8_t* nonces, uint8_t* signatures, int32_t* lane_status) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    return sign_sharded(ctx, count, signatures, lane_status, [&](size_t i) {
        size_t b, e;
        shard_range(count, i, k, &b, &e);
        return sign_nonces_range(ctx->shards[i], e - b, digests + 32 * b, secrets + 32 * b, nonces + 32 * b,
                                 signatures + 64 * b, lane_status ? lane_status + b : nullptr);
    });
}

sm2b_status group_keygen(sm2b_ctx* ctx, uint64_t seed, uint64_t lane_base, size_t count, uint8_t* secrets,
                         uint8_t* publics) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    sm2b_status st = for_each_shard(ctx, [&](size_t i) {
        size_t b, e;
        shard_range(count, i, k, &b, &e);
        return gecc_keygen(ctx->shards[i], seed, lane_base + b, e - b, secrets + 32 * b, publics + 65 * b);
    });
    if (st == SM2B_OK) account_keygen(ctx, count);
    return st;
}

sm2b_status group_ecdh(sm2b_ctx* ctx, size_t count, const uint8_t* secrets, const uint8_t* peers,
                       uint8_t* shared, int32_t* lane_status) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    std::vector<sm2b_status> st(k, SM2B_OK);
    std::vector<std::thread> th;
    auto call = [&](size_t i) {
        size_t b, e;
        shard_range(count, i, k, &b, &e);
        return sm2b_ecdh(ctx->shards[i], e - b, secrets + 32 * b, peers + 65 * b, shared + 32 * b,
                         lane_status ? lane_status + b : nullptr);
    };
    for (size_t i = 1; i < k; ++i) th.emplace_back([&, i] { st[i] = call(i); });
    st[0] = call(0);
    for (auto& t : th) t.join();
    for (size_t i = 0; i < k; ++i)
        if (st[i] == SM2B_ERROR_MALFORMED_INPUT || st[i] == SM2B_ERROR_INTERNAL || st[i] == SM2B_ERROR_INVALID_ARGUMENT) {
            if (st[i] == SM2B_ERROR_INTERNAL) ctx->last_error = ctx->shards[i]->last_error;
            memset(shared, 0, 32 * count);  // a secret >= n fails the whole call (capi.cpp:241)
            return st[i];
        }
    account_ecdh(ctx, count);
    for (size_t i = 0; i < k; ++i)
        if (st[i] != SM2B_OK) return st[i];  // lane_status == NULL: first failing lane's code
    return SM2B_OK;
}

sm2b_status group_points(sm2b_ctx* ctx, int op, size_t n, const uint32_t* scalars, const HostPoints* p,
                         const HostPoints* t, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                         const gecc_base_table* base) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    sm2b_status st = for_each_shard(ctx, [&](size_t i) {
        size_t b, e;
        shard_range(n, i, k, &b, &e);
        return points_range(ctx->shards[i], op, n, b, e - b, scalars, p, t, ox, oy, oinf,
                            base ? base_table_for(ctx->shards[i], base) : nullptr, false);
    });
    if (st == SM2B_OK) account_points(ctx, op, n);
    return st;
}

sm2b_status group_field(sm2b_ctx* ctx, int field, int op, size_t n, const uint32_t* a, const uint32_t* b,
                        uint32_t* out) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    return for_each_shard(ctx, [&](size_t i) {
        size_t lo, hi;
        shard_range(n, i, k, &lo, &hi);
        return field_range(ctx->shards[i], field, op, n, lo, hi - lo, a, b, out);
    });
}

sm2b_status group_invert(sm2b_ctx* ctx, int field, size_t n, const uint32_t* in, uint32_t* out) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    sm2b_status st = for_each_shard(ctx, [&](size_t i) {
        size_t lo, hi;
        shard_range(n, i, k, &lo, &hi);
        return invert_range(ctx->shards[i], field, n, lo, hi - lo, in, out, false);
    });
    if (st == SM2B_OK) account_invert(ctx, n);
    return st;
}

// ---------------------------------------------------------------- MSM exchange
namespace {
// communicators of a group with distinct devices, created together on first use
sm2b_status group_comm_init(sm2b_ctx* ctx) {
    if (ctx->shards[0]->nccl_comm) return SM2B_OK;
    if (!nccl().ok) {
        ctx->last_error = "libnccl.so.2 could not be loaded (needed for the multi-device MSM exchange)";
        return SM2B_ERROR_INTERNAL;
    }
    const int k = (int)ctx->shards.size();
    std::vector<ncclComm_t> comms(k);
    std::vector<int> devs(k);
    for (int i = 0; i < k; ++i) devs[i] = ctx->shards[i]->device;
    ncclResult_t r = nccl().CommInitAll(comms.data(), k, devs.data());
    if (r != ncclSuccess) return nccl_fail(ctx, "ncclCommInitAll", r);
    for (int i = 0; i < k; ++i) {
        sm2b_ctx* s = ctx->shards[i];
        s->nccl_comm = comms[i];
        s->nccl_rank = i;
        s->nccl_nranks = k;
        s->nccl_owned = true;
    }
    return SM2B_OK;
}
}  // namespace

sm2b_status group_msm(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px, const uint32_t* py,
                      const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t k = ctx->shards.size();
    const size_t W = packed_words(ctx), L = (size_t)ctx->limbs;
    const bool use_nccl = k > 1 && distinct_devices(ctx);
    if (use_nccl) {
        sm2b_status st = group_comm_init(ctx);
        if (st != SM2B_OK) return st;
    }
    // every device sums its own point range; the partial sums stay on the devices
    sm2b_status st = for_each_shard(ctx, [&](size_t i) {
        size_t b, e;
        shard_range(n, i, k, &b, &e);
        return msm_range_enqueue(ctx->shards[i], n, b, e - b, scalars, px, py, pinf);
    });
    if (st != SM2B_OK) return st;
    sm2b_ctx* root = ctx->shards[0];
    if (use_nccl) {  // one all-gather of W words per device, issued for all devices as one group
        ncclResult_t r = nccl().GroupStart();
        for (size_t i = 0; i < k && r == ncclSuccess; ++i) {
            sm2b_ctx* s = ctx->shards[i];
            DeviceGuard g(s->device);
            r = nccl().AllGather(xchg_mine(s), xchg_all(s), W, ncclUint32, (ncclComm_t)s->nccl_comm, s->stream);
        }
        ncclResult_t r2 = nccl().GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess) return nccl_fail(ctx, "ncclAllGather", r != ncclSuccess ? r : r2);
    } else {  // shards that share a device (or a single shard): the gather is peer copies to the root
        for (size_t i = 0; i < k; ++i) {
            sm2b_ctx* s = ctx->shards[i];
            DeviceGuard g(s->device);
            cudaError_t e = cudaStreamSynchronize(s->stream);
            if (e != cudaSuccess) return cuda_fail(ctx, "msm shard", e);
        }
        DeviceGuard g(root->device);
        for (size_t i = 0; i < k; ++i) {
            sm2b_ctx* s = ctx->shards[i];
            cudaError_t e = cudaMemcpyPeerAsync(xchg_all(root) + i * W, root->device, xchg_mine(s), s->device, 4 * W,
                                                root->stream);
            if (e != cudaSuccess) return cuda_fail(ctx, "msm exchange (peer copy)", e);
        }
    }
    // local additions on the first device, then its result comes home
    DeviceGuard g(root->device);
    cudaError_t e = launch_point_fold(ctx->curve, (int)k, xchg_all(root), xchg_mine(root), root->stream);
    root->launches += 1;
    uint32_t host[2 * 12 + 1];
    if (e == cudaSuccess) e = cudaMemcpyAsync(host, xchg_mine(root), 4 * W, cudaMemcpyDeviceToHost, root->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(root->stream);
    if (use_nccl)
        for (size_t i = 1; i < k && e == cudaSuccess; ++i) {  // the other devices' all-gathers have to drain too
            DeviceGuard gi(ctx->shards[i]->device);
            e = cudaStreamSynchronize(ctx->shards[i]->stream);
        }
    if (e != cudaSuccess) return cuda_fail(ctx, "msm exchange", e);
    memcpy(ox, host, 4 * L);
    memcpy(oy, host + L, 4 * L);
    *oinf = host[2 * L] ? 1 : 0;
    return SM2B_OK;
}

// multi-process form: this rank's packed partial sum at xchg_mine -> the total, same place
sm2b_status comm_combine_enqueue(sm2b_ctx* ctx) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx->device);
    const size_t W = packed_words(ctx);
    ncclResult_t r = nccl().AllGather(xchg_mine(ctx), xchg_all(ctx), W, ncclUint32, (ncclComm_t)ctx->nccl_comm, ctx->stream);
    if (r != ncclSuccess) return nccl_fail(ctx, "ncclAllGather", r);
    cudaError_t e = launch_point_fold(ctx->curve, ctx->nccl_nranks, xchg_all(ctx), xchg_mine(ctx), ctx->stream);
    ctx->launches += 1;
    if (e != cudaSuccess) return cuda_fail(ctx, "msm exchange fold", e);
    return SM2B_OK;
}

}  // namespace gecc_capi

using namespace gecc_capi;

extern "C" {

sm2b_status gecc_comm_unique_id(uint8_t id[GECC_COMM_ID_BYTES]) {
    static_assert(sizeof(ncclUniqueId) <= GECC_COMM_ID_BYTES, "id buffer too small");
    if (!id) return SM2B_ERROR_INVALID_ARGUMENT;
    if (!nccl().ok) return SM2B_ERROR_INTERNAL;
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess) return SM2B_ERROR_INTERNAL;
    memset(id, 0, GECC_COMM_ID_BYTES);
    memcpy(id, &u, sizeof u);
    return SM2B_OK;
}

sm2b_status gecc_comm_init_rank(sm2b_ctx* ctx, int nranks, int rank, const uint8_t id[GECC_COMM_ID_BYTES]) {
    if (!ctx || is_group(ctx) || !id || nranks < 1 || rank < 0 || rank >= nranks || nranks > 1024)
        return SM2B_ERROR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!nccl().ok) {
        ctx->last_error = "libnccl.so.2 could not be loaded";
        return SM2B_ERROR_INTERNAL;
    }
    DeviceGuard g(ctx->device);
    comm_release(ctx);
    cudaError_t e = ctx->xchg.ensure(4 * (64 + (size_t)nranks * packed_words(ctx)) + 256);
    if (e != cudaSuccess) return cuda_fail(ctx, "exchange buffer", e);
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    ncclComm_t comm;
    ncclResult_t r = nccl().CommInitRank(&comm, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(ctx, "ncclCommInitRank", r);
    ctx->nccl_comm = comm;
    ctx->nccl_rank = rank;
    ctx->nccl_nranks = nranks;
    ctx->nccl_owned = true;
    return SM2B_OK;
}

}  // extern "C"
