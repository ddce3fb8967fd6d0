// Multi-scalar multiplication  sum_i k_i * P_i  (Pippenger's bucket method).
//
// The reference has no MSM; the contract here is the
// definition, checked against the oracle's sum of pmul_serial results and against
// the identity  sum_i s_i (t_i G) = (sum_i s_i t_i) G  at full size.
//
//   1. k_msm_digits   : every scalar (folded below 2^255) is recoded into 16 signed 16-bit digits
//                       plus a rarely non-zero carry digit
//                       (same offset recoding as the fixed-base path); one
//                       (bucket id, point index | sign) pair per non-zero digit.
//   2. radix sort of the pairs by bucket id (CUB, plumbing only).
//   3. k_msm_buckets  : one thread per bucket sums its points (mixed Jacobian adds).
//   4. bucket reduction  S_w = sum_b (b+1) B_w[b]  without any long serial chain:
//      b = lo + 32 mid + 1024 top, so S_w = sum B + sum_k 32^k sum_e e * C^k_e with the
//      three marginal sums C^k_e (each over 1024 buckets, done as 32 x 32).
//   5. k_msm_combine  : sum_w 2^(16 w) S_w, one affine point out.
// Bucket ids: window w, magnitude m = 1..2^15  ->  w * 2^15 + (m - 1).
#include <cub/device/device_radix_sort.cuh>

#include "gecc_ecdsa.cuh"
#include "gecc_host.h"

namespace gecc {

constexpr int MSM_C = 16;                          // window bits
constexpr int MSM_WINDOWS = 256 / MSM_C + 1;       // 17: scalars are folded below 2^255 first, so the
                                                   // 17th (recoding-carry) window is hit with probability
                                                   // ~2^-16 only -- it must exist, but stays almost empty
constexpr int MSM_BUCKETS = 1 << (MSM_C - 1);      // 32768 per window
constexpr uint32_t MSM_NB = MSM_WINDOWS * MSM_BUCKETS;
constexpr uint32_t MSM_KEY_NONE = 0xFFFFFu;        // sorts behind every real bucket (20-bit keys)

template <class C>
__global__ void __launch_bounds__(256)
k_msm_digits(size_t n, const uint32_t* __restrict__ scalars, const uint8_t* __restrict__ pinf,
             uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    fe k = scalar_reduce_once<typename C::Fn>(col_load(scalars, n, i));
    const bool skip = pinf && pinf[i];
    // k >= 2^255: use (n - k) * (-P).  A carry window would otherwise collect ~n/2 points in
    // ONE bucket (a single thread adding half a million points).
    const bool flip = (k.w[7] >> 31) != 0;
    if (flip) k = u256_sub(fe_modulus(typename C::Fn{}), k);
    Recoded<MSM_C> rc = recode_signed<MSM_C>(k);  // k < 2^255: rc.carry is 1 only for 0x7FFF8... tops
#pragma unroll
    for (int w = 0; w < MSM_WINDOWS; ++w) {
        int d = w == MSM_WINDOWS - 1 ? (int)rc.carry : recoded_digit<MSM_C>(rc, w);
        uint32_t key = MSM_KEY_NONE, val = 0;
        if (d != 0 && !skip) {
            const uint32_t mag = (uint32_t)(d < 0 ? -d : d);
            key = (uint32_t)w * MSM_BUCKETS + (mag - 1);
            val = (uint32_t)i | (((d < 0) != flip) ? 0x80000000u : 0u);
        }
        keys[(size_t)w * n + i] = key;   // window-major: coalesced writes
        vals[(size_t)w * n + i] = val;
    }
}

// first position whose key is >= bucket (sorted keys)
__device__ __forceinline__ size_t lower_bound_key(const uint32_t* keys, size_t m, uint32_t bucket) {
    size_t lo = 0, hi = m;
    while (lo < hi) {
        size_t mid = (lo + hi) >> 1;
        if (keys[mid] < bucket) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Jacobian point arrays are stored word-major: word k (0..23: X, Y, Z) of element e at
// buf[k * count + e].
__device__ __forceinline__ void jac_store(uint32_t* buf, size_t count, size_t e, const jac& p) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        buf[(size_t)k * count + e] = p.X.w[k];
        buf[(size_t)(8 + k) * count + e] = p.Y.w[k];
        buf[(size_t)(16 + k) * count + e] = p.Z.w[k];
    }
}
__device__ __forceinline__ jac jac_load(const uint32_t* buf, size_t count, size_t e) {
    jac p;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        p.X.w[k] = buf[(size_t)k * count + e];
        p.Y.w[k] = buf[(size_t)(8 + k) * count + e];
        p.Z.w[k] = buf[(size_t)(16 + k) * count + e];
    }
    return p;
}

// Bucket accumulation, load-balanced: thread t owns the fixed-size slice
// [t * MSM_SLICE, (t+1) * MSM_SLICE) of the SORTED pairs, whatever buckets it crosses (a
// thread per bucket makes every warp wait for its largest bucket: sizes are Poisson(32)).
// A run of equal keys that starts and ends strictly inside the slice is a complete bucket
// and is stored directly.  The first and the last run of a slice may continue in the
// neighbouring slices: those sums go to edge[2t] / edge[2t+1] with their bucket ids, and
// k_msm_bucket_edges adds, for every bucket, the edge partials that belong to it.
// Buckets that receive nothing are pre-set to infinity (Z = 0) by a memset.
constexpr int MSM_SLICE = 32;

template <class C>
__global__ void __launch_bounds__(128)
k_msm_buckets(size_t n, size_t m, const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
              const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
              uint32_t* __restrict__ buckets, uint32_t* __restrict__ edge, uint32_t* __restrict__ edge_key,
              size_t slices) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= slices) return;
    const typename C::Fp f{};
    const size_t lo = t * MSM_SLICE, hi = lo + MSM_SLICE < m ? lo + MSM_SLICE : m;
    const uint32_t prev_key = lo > 0 ? keys[lo - 1] : 0xFFFFFFFFu;
    const uint32_t next_key = hi < m ? keys[hi] : 0xFFFFFFFFu;
    edge_key[2 * t] = edge_key[2 * t + 1] = MSM_KEY_NONE;
    jac acc = jac_infinity<C>();
    uint32_t cur = keys[lo];
    bool first_run = true;
#pragma unroll 1
    for (size_t p = lo; p <= hi; ++p) {
        const uint32_t key = p < hi ? keys[p] : 0xFFFFFFFEu;  // sentinel closes the last run
        if (key != cur) {
            if (cur < MSM_NB) {  // close the run of bucket `cur`
                const bool open_left = first_run && cur == prev_key;
                const bool open_right = p == hi && cur == next_key;
                if (open_left) {
                    jac_store(edge, 2 * slices, 2 * t, acc);
                    edge_key[2 * t] = cur;
                    // the whole slice lies inside one bucket: mark "continues to the right"
                    // (no point is stored in the right edge; the high bit says so)
                    if (open_right) edge_key[2 * t + 1] = cur | 0x80000000u;
                } else if (open_right) {
                    jac_store(edge, 2 * slices, 2 * t + 1, acc);
                    edge_key[2 * t + 1] = cur;
                } else {
                    jac_store(buckets, MSM_NB, cur, acc);
                }
            }
            first_run = false;
            acc = jac_infinity<C>();
            cur = key;
        }
        if (p < hi && key < MSM_NB) {
            const uint32_t v = vals[p];
            const size_t idx = v & 0x7FFFFFFFu;
            aff q{col_load(px, n, idx), col_load(py, n, idx)};
            if (v >> 31) q.y = fe_neg(f, q.y);
            acc = jac_madd<C>(acc, q);
        }
    }
}

// one thread per slice edge that opens a bucket from the left side of a chain: a bucket
// spanning slices t0 < ... < t1 has partials right(t0), left(t0+1) [whole slices in between
// are left edges too], ..., left(t1).  The thread holding right(t0) walks to the right and
// adds every following left edge with the same key, then stores the bucket.
template <class C>
__global__ void __launch_bounds__(128)
k_msm_bucket_edges(uint32_t* __restrict__ buckets, const uint32_t* __restrict__ edge,
                   const uint32_t* __restrict__ edge_key, size_t slices) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= slices) return;
    const uint32_t key = edge_key[2 * t + 1];
    if (key >= MSM_NB) return;  // this slice's last run does not continue to the right
    jac acc = jac_load(edge, 2 * slices, 2 * t + 1);
#pragma unroll 1
    for (size_t u = t + 1; u < slices && edge_key[2 * u] == key; ++u) {
        acc = jac_add<C>(acc, jac_load(edge, 2 * slices, 2 * u));
        if (edge_key[2 * u + 1] != (key | 0x80000000u)) break;  // the run ended inside slice u
    }
    jac_store(buckets, MSM_NB, key, acc);
}

// marginal sums, stage 1: thread (w, k, e, part) adds the 32 buckets of window w whose
// k-th base-32 digit is e and whose next digit (cyclically) is `part`.
template <class C>
__global__ void __launch_bounds__(128)
k_msm_marginal_parts(const uint32_t* __restrict__ buckets, uint32_t* __restrict__ parts) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= MSM_WINDOWS * 3 * 32 * 32) return;
    const uint32_t part = t & 31, e = (t >> 5) & 31, k = (t >> 10) % 3, w = t / (3 * 1024);
    jac acc = jac_infinity<C>();
#pragma unroll 1
    for (uint32_t v = 0; v < 32; ++v) {
        uint32_t b;
        if (k == 0) b = e + 32 * part + 1024 * v;        // lo = e
        else if (k == 1) b = part + 32 * e + 1024 * v;   // mid = e
        else b = part + 32 * v + 1024 * e;               // top = e
        acc = jac_add<C>(acc, jac_load(buckets, MSM_NB, (size_t)w * MSM_BUCKETS + b));
    }
    jac_store(parts, (size_t)MSM_WINDOWS * 3 * 1024, t, acc);
}
// stage 2: thread (w, k, e) folds its 32 parts
template <class C>
__global__ void __launch_bounds__(128)
k_msm_marginal_fold(const uint32_t* __restrict__ parts, uint32_t* __restrict__ marg) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= MSM_WINDOWS * 3 * 32) return;
    jac acc = jac_infinity<C>();
#pragma unroll 1
    for (uint32_t p = 0; p < 32; ++p)
        acc = jac_add<C>(acc, jac_load(parts, (size_t)MSM_WINDOWS * 3 * 1024, (size_t)t * 32 + p));
    jac_store(marg, (size_t)MSM_WINDOWS * 3 * 32, t, acc);
}
// stage 3: thread (w, j): j < 3 -> sum_e e * C^j_e (running sums); j == 3 -> sum_e C^0_e
template <class C>
__global__ void __launch_bounds__(128)
k_msm_weighted(const uint32_t* __restrict__ marg, uint32_t* __restrict__ wsum) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= MSM_WINDOWS * 4) return;
    const uint32_t w = t >> 2, j = t & 3;
    const size_t cnt = (size_t)MSM_WINDOWS * 3 * 32;
    jac acc = jac_infinity<C>();
    if (j == 3) {
#pragma unroll 1
        for (uint32_t e = 0; e < 32; ++e) acc = jac_add<C>(acc, jac_load(marg, cnt, (size_t)(w * 3) * 32 + e));
    } else {
        jac run = jac_infinity<C>();
#pragma unroll 1
        for (int e = 31; e >= 1; --e) {
            run = jac_add<C>(run, jac_load(marg, cnt, (size_t)(w * 3 + j) * 32 + e));
            acc = jac_add<C>(acc, run);
        }
    }
    jac_store(wsum, (size_t)MSM_WINDOWS * 4, t, acc);
}
// stage 4 (one block of 32 threads): thread w forms S_w = (sum B) + W0 + 32 W1 + 1024 W2
// (weights b + 1), shifts it by 2^(16 w); thread 0 adds the windows and converts to affine.
template <class C>
__global__ void __launch_bounds__(32)
k_msm_combine(const uint32_t* __restrict__ wsum, uint32_t* __restrict__ ox, uint32_t* __restrict__ oy,
              uint8_t* __restrict__ oinf) {
    __shared__ uint32_t win[24 * MSM_WINDOWS];
    const uint32_t w = threadIdx.x;
    const size_t cnt = (size_t)MSM_WINDOWS * 4;
    if (w < MSM_WINDOWS) {
        jac s = jac_load(wsum, cnt, w * 4 + 2);
#pragma unroll 1
        for (int i = 0; i < 5; ++i) s = jac_dbl<C>(s);
        s = jac_add<C>(s, jac_load(wsum, cnt, w * 4 + 1));
#pragma unroll 1
        for (int i = 0; i < 5; ++i) s = jac_dbl<C>(s);
        s = jac_add<C>(s, jac_load(wsum, cnt, w * 4 + 0));
        s = jac_add<C>(s, jac_load(wsum, cnt, w * 4 + 3));
#pragma unroll 1
        for (uint32_t i = 0; i < MSM_C * w; ++i) s = jac_dbl<C>(s);
        jac_store(win, MSM_WINDOWS, w, s);
    }
    __syncthreads();
    if (w == 0) {
        const typename C::Fp f{};
        jac acc = jac_infinity<C>();
#pragma unroll 1
        for (int i = 0; i < MSM_WINDOWS; ++i) acc = jac_add<C>(acc, jac_load(win, MSM_WINDOWS, i));
        if (jac_is_inf<C>(acc)) {
            col_store(ox, 1, 0, fe_zero());
            col_store(oy, 1, 0, fe_zero());
            oinf[0] = 1;
        } else {
            aff a = jac_to_aff_with<C>(acc, fe_inv(f, acc.Z));
            col_store(ox, 1, 0, a.x);
            col_store(oy, 1, 0, a.y);
            oinf[0] = 0;
        }
    }
}

// ---------------------------------------------------------------- host side
struct MsmPlan {
    size_t pairs, sort_temp, total;
    size_t slices;
    size_t off_keys, off_vals, off_keys2, off_vals2, off_buckets, off_edge, off_edge_key, off_parts, off_marg, off_wsum, off_temp;
};
static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

static MsmPlan msm_plan(size_t n) {
    MsmPlan p{};
    p.pairs = n * MSM_WINDOWS;
    cub::DeviceRadixSort::SortPairs(nullptr, p.sort_temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)p.pairs, 0, 20);
    size_t at = 0;
    auto take = [&](size_t bytes) { size_t o = at; at += align256(bytes); return o; };
    p.off_keys = take(4 * p.pairs);
    p.off_vals = take(4 * p.pairs);
    p.off_keys2 = take(4 * p.pairs);
    p.off_vals2 = take(4 * p.pairs);
    p.slices = (p.pairs + MSM_SLICE - 1) / MSM_SLICE;
    p.off_buckets = take((size_t)96 * MSM_NB);
    p.off_edge = take((size_t)96 * 2 * p.slices);
    p.off_edge_key = take((size_t)4 * 2 * p.slices);
    p.off_parts = take((size_t)96 * MSM_WINDOWS * 3 * 1024);
    p.off_marg = take((size_t)96 * MSM_WINDOWS * 3 * 32);
    p.off_wsum = take((size_t)96 * MSM_WINDOWS * 4);
    p.off_temp = take(p.sort_temp);
    p.total = at;
    return p;
}
size_t msm_scratch_bytes(size_t n) { return n ? msm_plan(n).total : 0; }

template <class C>
static cudaError_t run_msm(size_t n, const uint32_t* scalars, const uint32_t* px, const uint32_t* py,
                           const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                           void* scratch, cudaStream_t s, int* launches) {
    MsmPlan p = msm_plan(n);
    uint8_t* base = (uint8_t*)scratch;
    uint32_t *keys = (uint32_t*)(base + p.off_keys), *vals = (uint32_t*)(base + p.off_vals);
    uint32_t *keys2 = (uint32_t*)(base + p.off_keys2), *vals2 = (uint32_t*)(base + p.off_vals2);
    uint32_t *buckets = (uint32_t*)(base + p.off_buckets), *parts = (uint32_t*)(base + p.off_parts);
    uint32_t *marg = (uint32_t*)(base + p.off_marg), *wsum = (uint32_t*)(base + p.off_wsum);
    k_msm_digits<C><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, scalars, pinf, keys, vals);
    size_t temp = p.sort_temp;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(base + p.off_temp, temp, keys, keys2, vals, vals2,
                                                    (int64_t)p.pairs, 0, 20, s);
    if (e != cudaSuccess) return e;
    uint32_t *edge = (uint32_t*)(base + p.off_edge), *edge_key = (uint32_t*)(base + p.off_edge_key);
    e = cudaMemsetAsync(buckets, 0, (size_t)96 * MSM_NB, s);  // empty buckets = infinity (Z = 0)
    if (e != cudaSuccess) return e;
    const unsigned sb = (unsigned)((p.slices + 127) / 128);
    k_msm_buckets<C><<<sb, 128, 0, s>>>(n, p.pairs, keys2, vals2, px, py, buckets, edge, edge_key, p.slices);
    k_msm_bucket_edges<C><<<sb, 128, 0, s>>>(buckets, edge, edge_key, p.slices);
    k_msm_marginal_parts<C><<<(MSM_WINDOWS * 3 * 1024 + 127) / 128, 128, 0, s>>>(buckets, parts);
    k_msm_marginal_fold<C><<<(MSM_WINDOWS * 3 * 32 + 127) / 128, 128, 0, s>>>(parts, marg);
    k_msm_weighted<C><<<1, 128, 0, s>>>(marg, wsum);
    k_msm_combine<C><<<1, 32, 0, s>>>(wsum, ox, oy, oinf);
    *launches = 7 + 4;  // ours + the sort's passes (approximate; CUB picks the pass count)
    return cudaGetLastError();
}

cudaError_t launch_msm(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                       const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                       uint8_t* oinf, void* scratch, cudaStream_t s, int* launches) {
    if (curve == CURVE_SECP)
        return run_msm<SecpCurve>(n, scalars, px, py, pinf, ox, oy, oinf, scratch, s, launches);
    return run_msm<Sm2Curve>(n, scalars, px, py, pinf, ox, oy, oinf, scratch, s, launches);
}

}  // namespace gecc
