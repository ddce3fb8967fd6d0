// Private to the host side of libgecc_b200.so: the context object behind the opaque
// sm2b_ctx handle and the range-form internals shared by capi.cu (single device) and
// capi_multi.cu (one context driving several devices, the MSM exchange over NCCL).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gecc_b200.h"
#include "gecc_host.h"

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

// A context is either a DEVICE context (one CUDA device: streams, arenas, fixed-base tables)
// or a GROUP context (shards non-empty): it owns one device context per device and splits every
// host-pointer call into contiguous lane ranges, one host thread per device (capi_multi.cu).
struct sm2b_ctx {
    int curve = gecc::CURVE_SM2;
    int device = 0;
    int sm_count = 148;
    uint32_t workers = 0, lanes = 0;
    std::mutex mu;  // held for the WHOLE of every call: calls on one context serialise (sm2batch.h:38-40)
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
    DevBuf xchg;       // MSM exchange: this shard's partial sum + the gathered partial sums
    uint32_t* gtab = nullptr;      // fixed-base table (Montgomery form), built on the GPU at creation
    uint32_t* gtab_rec = nullptr;  // table of the byte-record kernels (== gtab on SM2, plain form on secp256k1)
    uint32_t* flags = nullptr;     // device word: malformed-call flag of sign / ecdh
    int limbs = 8;                 // 32-bit limbs per coordinate (12 on the BLS curves)
    uint32_t* hflag = nullptr;     // pinned host word: the flag comes back without blocking the enqueueing thread
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // fork / join of the two-stream MSM tree levels
    int secret_mode = 0;           // GECC_SECRET_FAST / GECC_SECRET_UNIFORM (gecc_ctx_set_secret_mode)

    // ---- group context
    std::vector<sm2b_ctx*> shards;
    // ---- MSM exchange over NCCL.  In a group context with distinct devices the communicators
    // of all shards are created together (ncclCommInitAll); a device context joins a
    // multi-process communicator through gecc_comm_init_rank.
    void* nccl_comm = nullptr;  // ncclComm_t
    int nccl_rank = 0, nccl_nranks = 1;
    bool nccl_owned = false;
};

// fixed-base table of an arbitrary on-curve point (gecc_base_table_new): one copy per device
struct gecc_base_table {
    sm2b_ctx* owner = nullptr;
    std::vector<uint32_t*> tabs;  // per shard of the owner (one entry on a device context)
};

namespace gecc_capi {

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

inline bool is_group(const sm2b_ctx* ctx) { return !ctx->shards.empty(); }

// Balanced contiguous ranges, sizes differ by at most one (LanePlan::make, batch_invert.cpp:8-29,
// applied to devices instead of lanes).
inline void shard_range(size_t total, size_t rank, size_t world, size_t* begin, size_t* end) {
    const size_t base = total / world, rem = total % world;
    *begin = rank * base + (rank < rem ? rank : rem);
    *end = *begin + base + (rank < rem ? 1 : 0);
}

// ---- closed-form ledger of one call; lanes / workers as the context holds them
void account_verify(sm2b_ctx* ctx, size_t count);
void account_sign(sm2b_ctx* ctx, size_t count);
void account_keygen(sm2b_ctx* ctx, size_t count);
void account_ecdh(sm2b_ctx* ctx, size_t count);
enum PointsOp { OP_PADD = 0, OP_PDBL, OP_FPMUL, OP_UPMUL };
void account_points(sm2b_ctx* ctx, int op, size_t n);
void account_invert(sm2b_ctx* ctx, size_t n);

struct HostPoints {
    const uint32_t* x;
    const uint32_t* y;
    const uint8_t* inf;
};

// ---- range forms on a DEVICE context (take ctx->mu themselves).  Host column buffers have
// `pitch` elements per limb row; elements [begin, begin + count) are processed and written.
sm2b_status points_range(sm2b_ctx* ctx, int op, size_t pitch, size_t begin, size_t count,
                         const uint32_t* scalars, const HostPoints* p, const HostPoints* t,
                         uint32_t* ox, uint32_t* oy, uint8_t* oinf, const uint32_t* base_tab, bool account);
sm2b_status field_range(sm2b_ctx* ctx, int field, int op, size_t pitch, size_t begin, size_t count,
                        const uint32_t* a, const uint32_t* b, uint32_t* out);
sm2b_status invert_range(sm2b_ctx* ctx, int field, size_t pitch, size_t begin, size_t count,
                         const uint32_t* in, uint32_t* out, bool account);
// MSM over elements [begin, begin + count) of host column buffers; the partial sum is left on the
// device, packed as x[L] y[L] inf (2L + 1 words) at ctx->xchg.p, enqueued on ctx->stream, not synchronised
sm2b_status msm_range_enqueue(sm2b_ctx* ctx, size_t pitch, size_t begin, size_t count,
                              const uint32_t* scalars, const uint32_t* px, const uint32_t* py,
                              const uint8_t* pinf);
sm2b_status sign_nonces_range(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                              const uint8_t* nonces, uint8_t* signatures, int32_t* lane_status);
// 64 bits of system entropy (getrandom); false when the system cannot provide them
bool system_seed(uint64_t* out);

// ---- group context (capi_multi.cu)
sm2b_ctx* group_new(gecc_curve curve, int ndev, const int* devices);
void group_free(sm2b_ctx* ctx);
sm2b_status group_verify(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* publics,
                         const uint8_t* signatures, uint8_t* results);
sm2b_status group_sign(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                       uint64_t nonce_seed, uint64_t lane_base, uint8_t* signatures, int32_t* lane_status);
sm2b_status group_sign_nonces(sm2b_ctx* ctx, size_t count, const uint8_t* digests, const uint8_t* secrets,
                              const uint8_t* nonces, uint8_t* signatures, int32_t* lane_status);
sm2b_status group_keygen(sm2b_ctx* ctx, uint64_t seed, uint64_t lane_base, size_t count, uint8_t* secrets,
                         uint8_t* publics);
sm2b_status group_ecdh(sm2b_ctx* ctx, size_t count, const uint8_t* secrets, const uint8_t* peers,
                       uint8_t* shared, int32_t* lane_status);
sm2b_status group_points(sm2b_ctx* ctx, int op, size_t n, const uint32_t* scalars, const HostPoints* p,
                         const HostPoints* t, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                         const gecc_base_table* base);
sm2b_status group_field(sm2b_ctx* ctx, int field, int op, size_t n, const uint32_t* a, const uint32_t* b,
                        uint32_t* out);
sm2b_status group_invert(sm2b_ctx* ctx, int field, size_t n, const uint32_t* in, uint32_t* out);
sm2b_status group_msm(sm2b_ctx* ctx, size_t n, const uint32_t* scalars, const uint32_t* px, const uint32_t* py,
                      const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf);
// all ranks' partial sums (packed at ctx->xchg.p) -> the total, in place, on ctx->stream
sm2b_status comm_combine_enqueue(sm2b_ctx* ctx);
void comm_release(sm2b_ctx* ctx);

}  // namespace gecc_capi
