// Multi-scalar multiplication  sum_i k_i * P_i  (Pippenger's bucket method).
//
// The reference has no MSM; the contract here is the
// definition, checked against the oracle's sum of pmul_serial results and against
// the identity  sum_i s_i (t_i G) = (sum_i s_i t_i) G  at full size.
//
//   1. k_msm_digits   : every scalar (reduced mod the group order, folded below 2^255) is recoded
//                       into 16 signed 16-bit digits plus a rarely non-zero carry digit (same
//                       offset recoding as the fixed-base path); one (bucket id, point index |
//                       sign) pair per non-zero digit.
//   2. radix sort of the pairs by bucket id (CUB, plumbing only).
//   3. bucket accumulation, selectable with gecc_set_msm_form:
//        batch-affine (default) : segmented pairwise tree over the sorted pairs, affine additions
//                                 sharing one inversion per thread block -- "batch-affine bucket
//                                 accumulation" below; three launches per level, or one;
//        mixed Jacobian         : k_msm_buckets, fixed slices of the sorted pairs per thread.
//   4. bucket reduction  S_w = sum_b (b+1) B_w[b]  without any long serial chain:
//      b = lo + 32 mid + 1024 top, so S_w = sum B + sum_k 32^k sum_e e * C^k_e with the
//      three marginal sums C^k_e (each over 1024 buckets): k_msm_red_* (warp-shuffle trees,
//      reads the tree's slots directly) after the batch-affine form, k_msm_marginal_* /
//      k_msm_weighted after the Jacobian one.
//   5. window combine : sum_w 2^(16 w) S_w, one affine point out (k_msm_red_combine: the
//      doubling chain is run by groups of four lanes).
// All of it is a template over the curve: 8-limb SM2 / secp256k1 (the latter accumulates on its
// lazy plain field), 12-limb BLS12-381 / BLS12-377 G1.
// Bucket ids: window w, magnitude m = 1..2^15  ->  w * 2^15 + (m - 1).
#include <cstdlib>
#include <type_traits>

#include "gecc_batch.cuh"
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

// The (bucket, point | sign) pair of scalar i in window w; key == MSM_KEY_NONE when the digit is zero.
template <class C>
struct MsmDigits {
    Recoded<MSM_C> rc;
    bool flip, skip;
    uint32_t index;
    __device__ __forceinline__ MsmDigits(size_t n, size_t i, const uint32_t* __restrict__ scalars,
                                         const uint8_t* __restrict__ pinf) {
        // any 256-bit scalar is accepted: below 2n for the 256-bit curves (one subtraction), below
        // 3r for BLS12-381's 255-bit group order (two), below 14r for BLS12-377's 253-bit one (13)
        constexpr uint32_t top = C::Fn::q(7);
        constexpr int subs = top >= 0x80000000u ? 1 : (int)(0xFFFFFFFFu / top);
        fe k = col_load<8>(scalars, n, i);
#pragma unroll 1
        for (int it = 0; it < subs; ++it) k = scalar_reduce_once<typename C::Fn>(k);
        skip = pinf && pinf[i];
        // k >= 2^255: use (n - k) * (-P).  A carry window would otherwise collect ~n/2 points in
        // ONE bucket (a single thread adding half a million points).
        flip = (k.w[7] >> 31) != 0;
        if (flip) k = u256_sub(fe_modulus(typename C::Fn{}), k);
        rc = recode_signed<MSM_C>(k);  // k < 2^255: rc.carry is 1 only for 0x7FFF8... tops
        index = (uint32_t)i;
    }
    __device__ __forceinline__ void pair(int w, uint32_t* key, uint32_t* val) const {
        const int d = w == MSM_WINDOWS - 1 ? (int)rc.carry : recoded_digit<MSM_C>(rc, w);
        *key = MSM_KEY_NONE;
        *val = 0;
        if (d != 0 && !skip) {
            const uint32_t mag = (uint32_t)(d < 0 ? -d : d);
            *key = (uint32_t)w * MSM_BUCKETS + (mag - 1);
            *val = index | (((d < 0) != flip) ? 0x80000000u : 0u);
        }
    }
};

template <class C>
__global__ void __launch_bounds__(256)
k_msm_digits(size_t n, const uint32_t* __restrict__ scalars, const uint8_t* __restrict__ pinf,
             uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const MsmDigits<C> dg(n, i, scalars, pinf);
#pragma unroll
    for (int w = 0; w < MSM_WINDOWS; ++w) {
        uint32_t key, val;
        dg.pair(w, &key, &val);
        keys[(size_t)w * n + i] = key;   // window-major: coalesced writes
        vals[(size_t)w * n + i] = val;
    }
}

// The sorted pairs are ONE array of (bucket id, point index | sign) words: the scatter of the sort
// writes a pair with a single 8-byte store (it is bound by the number of scattered write
// transactions, not by bytes), and level 0 of the tree reads the two pairs of a join with one
// 16-byte load.  PairKeys / PairVals are the two views the kernels index.
struct PairKeys {
    const uint2* p;
    __device__ __forceinline__ uint32_t operator[](size_t i) const { return p[i].x; }
};
struct PairVals {
    const uint2* p;
    __device__ __forceinline__ uint32_t operator[](size_t i) const { return p[i].y; }
};

// ---------------------------------------------------------------- bucket sort (counting sort)
// The pairs have to be grouped by bucket; nothing else about their order matters (a bucket's sum
// does not depend on the order of its points).  Keys are w * 2^15 + m - 1 < 17 * 2^15, so this is
// a counting sort over 557 056 counters -- no general radix sort is needed:
//   k_msm_hist    : recodes every scalar and counts its 17 buckets (atomics on L2-resident words);
//   k_msm_scan_*  : the counts become first positions (`starts`, 0xFFFFFFFF for an empty bucket --
//                   the array the bucket reduction reads) and scatter cursors; the unused tail of
//                   the pair arrays is marked;
//   k_msm_scatter : recodes again (cheaper than parking 142 MB of unsorted pairs) and writes every
//                   pair at cursor[bucket]++.  Threads walk window by window, so at any time the
//                   scattered writes fall into one window's 8 MB of the output and merge in L2.
template <class C>
__global__ void __launch_bounds__(256)
k_msm_hist(size_t n, const uint32_t* __restrict__ scalars, const uint8_t* __restrict__ pinf,
           uint32_t* __restrict__ counts) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const MsmDigits<C> dg(n, i, scalars, pinf);
#pragma unroll
    for (int w = 0; w < MSM_WINDOWS; ++w) {
        uint32_t key, val;
        dg.pair(w, &key, &val);
        if (key != MSM_KEY_NONE) atomicAdd(counts + key, 1u);
    }
}

// exclusive scan of the 557 056 counts in three small launches: per-block scans (coalesced, one
// counter per thread), a scan of the 544 block totals, and the pass that adds the block offsets
constexpr int MSM_SCAN_THREADS = 1024;
constexpr unsigned MSM_SCAN_BLOCKS = (MSM_NB + MSM_SCAN_THREADS - 1) / MSM_SCAN_THREADS;
static_assert(MSM_SCAN_BLOCKS <= MSM_SCAN_THREADS, "the block totals are scanned by one block");

// inclusive scan of v over the block; returns this thread's inclusive value, *total = block sum
__device__ __forceinline__ uint32_t block_scan_inclusive(uint32_t v, uint32_t* sh, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t ws = sh[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, ws, d);
            if (lane >= (uint32_t)d) ws += o;
        }
        sh[lane] = ws;
    }
    __syncthreads();
    *total = sh[31];
    return inc + (warp ? sh[warp - 1] : 0u);
}
__global__ void __launch_bounds__(MSM_SCAN_THREADS)
k_msm_scan_blocks(const uint32_t* __restrict__ counts, uint32_t* __restrict__ local, uint32_t* __restrict__ block_totals) {
    __shared__ uint32_t sh[32];
    const uint32_t b = blockIdx.x * MSM_SCAN_THREADS + threadIdx.x;
    const uint32_t c = b < MSM_NB ? counts[b] : 0u;
    uint32_t total;
    const uint32_t inc = block_scan_inclusive(c, sh, &total);
    if (b < MSM_NB) local[b] = inc - c;  // exclusive, local to the block
    if (threadIdx.x == 0) block_totals[blockIdx.x] = total;
}
// Window w owns the positions [w * region, (w + 1) * region) of the sorted pair arrays (region =
// n rounded up to the tree's largest node): the windows are then independent sub-problems whose
// trees and reductions run as a pipeline on two streams.  block_totals[b] becomes the first
// position of scan block b (32 blocks per window), block_totals[MSM_SCAN_BLOCKS + w] the number
// of pairs of window w.
constexpr unsigned MSM_SCAN_BLOCKS_PER_WINDOW = MSM_BUCKETS / MSM_SCAN_THREADS;
static_assert(MSM_BUCKETS % MSM_SCAN_THREADS == 0, "whole scan blocks per window");
__global__ void __launch_bounds__(MSM_SCAN_THREADS)
k_msm_scan_tops(uint32_t* __restrict__ block_totals, uint32_t region) {
    __shared__ uint32_t sh[32];
    __shared__ uint32_t inc_all[MSM_SCAN_THREADS];
    const uint32_t t = threadIdx.x;
    const uint32_t c = t < MSM_SCAN_BLOCKS ? block_totals[t] : 0u;
    uint32_t total;
    const uint32_t inc = block_scan_inclusive(c, sh, &total);
    inc_all[t] = inc;
    __syncthreads();
    if (t < MSM_SCAN_BLOCKS) {
        const uint32_t w = t / MSM_SCAN_BLOCKS_PER_WINDOW, first = w * MSM_SCAN_BLOCKS_PER_WINDOW;
        const uint32_t before = first ? inc_all[first - 1] : 0u;      // pairs of the windows below
        block_totals[t] = (inc - c) - before + w * region;
        if (t == first) block_totals[MSM_SCAN_BLOCKS + w] = inc_all[first + MSM_SCAN_BLOCKS_PER_WINDOW - 1] - before;
    }
}
__global__ void __launch_bounds__(MSM_SCAN_THREADS)
k_msm_scan_finish(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ block_totals,
                  uint32_t* __restrict__ starts /* in: local prefixes */, uint32_t* __restrict__ cursor,
                  uint2* __restrict__ pairs_sorted, uint32_t region) {
    const uint32_t b = blockIdx.x * MSM_SCAN_THREADS + threadIdx.x;
    // the positions of a window's region behind its last pair hold "no bucket" (zero digits, points
    // at infinity, the rounding of the region; the carry window is almost all of that kind)
    for (uint32_t w = 0; w < MSM_WINDOWS; ++w) {
        const size_t end = (size_t)(w + 1) * region;
        for (size_t p = (size_t)w * region + block_totals[MSM_SCAN_BLOCKS + w] + b; p < end; p += (size_t)gridDim.x * MSM_SCAN_THREADS)
            pairs_sorted[p] = make_uint2(MSM_KEY_NONE, 0u);
    }
    if (b >= MSM_NB) return;
    const uint32_t at = starts[b] + block_totals[blockIdx.x];
    cursor[b] = at;
    starts[b] = counts[b] ? at : 0xFFFFFFFFu;  // first position of the bucket's run; none for an empty bucket
}

template <class C>
__global__ void __launch_bounds__(256)
k_msm_scatter(size_t n, const uint32_t* __restrict__ scalars, const uint8_t* __restrict__ pinf,
              uint32_t* __restrict__ cursor, uint2* __restrict__ pairs_sorted) {
    // block b serves window b / blocks_per_window: the grid runs through the windows in order
    const unsigned bpw = (unsigned)((n + 255) / 256);
    const int w = (int)(blockIdx.x / bpw);
    const size_t i = (size_t)(blockIdx.x % bpw) * 256 + threadIdx.x;
    if (i >= n) return;
    const MsmDigits<C> dg(n, i, scalars, pinf);
    uint32_t key, val;
    dg.pair(w, &key, &val);
    if (key == MSM_KEY_NONE) return;
    const uint32_t pos = atomicAdd(cursor + key, 1u);
    pairs_sorted[pos] = make_uint2(key, val);
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

// Jacobian point arrays are stored word-major: word k (0..3N-1: X, Y, Z) of element e at
// buf[k * count + e].
template <int N>
__device__ __forceinline__ void jac_store(uint32_t* buf, size_t count, size_t e, const jacN<N>& p) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
        buf[(size_t)k * count + e] = p.X.w[k];
        buf[(size_t)(N + k) * count + e] = p.Y.w[k];
        buf[(size_t)(2 * N + k) * count + e] = p.Z.w[k];
    }
}
template <int N>
__device__ __forceinline__ jacN<N> jac_load(const uint32_t* buf, size_t count, size_t e) {
    jacN<N> p;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        p.X.w[k] = buf[(size_t)k * count + e];
        p.Y.w[k] = buf[(size_t)(N + k) * count + e];
        p.Z.w[k] = buf[(size_t)(2 * N + k) * count + e];
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
k_msm_buckets(size_t n, size_t m, const PairKeys keys, const PairVals vals,
              const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
              uint32_t* __restrict__ buckets, uint32_t* __restrict__ edge, uint32_t* __restrict__ edge_key,
              size_t slices) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
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
                    jac_store<NL>(edge, 2 * slices, 2 * t, acc);
                    edge_key[2 * t] = cur;
                    // the whole slice lies inside one bucket: mark "continues to the right"
                    // (no point is stored in the right edge; the high bit says so)
                    if (open_right) edge_key[2 * t + 1] = cur | 0x80000000u;
                } else if (open_right) {
                    jac_store<NL>(edge, 2 * slices, 2 * t + 1, acc);
                    edge_key[2 * t + 1] = cur;
                } else {
                    jac_store<NL>(buckets, MSM_NB, cur, acc);
                }
            }
            first_run = false;
            acc = jac_infinity<C>();
            cur = key;
        }
        if (p < hi && key < MSM_NB) {
            const uint32_t v = vals[p];
            const size_t idx = v & 0x7FFFFFFFu;
            aff q{col_load<NL>(px, n, idx), col_load<NL>(py, n, idx)};
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
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= slices) return;
    const uint32_t key = edge_key[2 * t + 1];
    if (key >= MSM_NB) return;  // this slice's last run does not continue to the right
    jac acc = jac_load<NL>(edge, 2 * slices, 2 * t + 1);
#pragma unroll 1
    for (size_t u = t + 1; u < slices && edge_key[2 * u] == key; ++u) {
        acc = jac_add<C>(acc, jac_load<NL>(edge, 2 * slices, 2 * u));
        if (edge_key[2 * u + 1] != (key | 0x80000000u)) break;  // the run ended inside slice u
    }
    jac_store<NL>(buckets, MSM_NB, key, acc);
}

// ---------------------------------------------------------------- batch-affine bucket accumulation
// The bucket sums are formed with AFFINE additions that share their inversions (Montgomery's
// trick across a thread block), 5M + 1S + the scan share per addition instead of the 8M + 3S
// of a mixed Jacobian addition.  Independent additions come from a segmented pairwise tree
// over the SORTED pair list (positions 0 .. m-1):
//   invariant after level l: inside every aligned node [a, a + 2^l) the partial sum of key k
//   over the node's entries sits in slot max(a, runstart(k));
//   level l joins the two halves of every node of size 2^(l+1): only the key that straddles
//   the middle c needs work,  slot[max(a, runstart)] += slot[c]  -- all joins of one level are
//   independent, and a consumed slot is never read again.
// Level 0 reads the points themselves (64-byte AoS records, gathered by index, sign applied)
// and fills the slots.  After MSM_TREE_LEVELS levels a bucket whose run is [s, e) has its sum
// spread over slot s and the slots at multiples of 2^MSM_TREE_LEVELS inside (s, e): the tail
// kernel (one thread per bucket) adds those few (mean run length is 32) with mixed Jacobian
// additions and writes the bucket in the layout the reduction kernels read.
// All formulas are complete: the point at infinity is a slot whose x is all ones (slot_is_inf); equal points take the tangent,
// opposite points give infinity (classification as batch_padd, batch_point.cpp:91-111).
constexpr int MSM_TREE_LEVELS = 6;
constexpr int MSM_TREE_THREADS = 128;

// A record is x | y, 2N limbs = N/2 16-byte words (64 B for 256-bit, 96 B for 381-bit curves).
enum { LD_PLAIN = 0, LD_STREAM = 1, LD_KEEP = 2 };
template <int N, int MODE>
__device__ __forceinline__ feN<N> fe_load_u4(const uint4* p) {
    feN<N> r;
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
        const uint4 v = MODE == LD_STREAM ? __ldcs(p + q) : MODE == LD_KEEP ? __ldg(p + q) : p[q];
        r.w[4 * q] = v.x; r.w[4 * q + 1] = v.y; r.w[4 * q + 2] = v.z; r.w[4 * q + 3] = v.w;
    }
    return r;
}
template <int N, bool STREAM>
__device__ __forceinline__ void fe_store_u4(uint4* p, const feN<N>& v) {
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
        const uint4 t = make_uint4(v.w[4 * q], v.w[4 * q + 1], v.w[4 * q + 2], v.w[4 * q + 3]);
        if (STREAM) __stcs(p + q, t);
        else p[q] = t;
    }
}
// Cache policy: the input records (64 MiB at 2^20) are gathered at random and re-read by every
// window, so they should stay in L2; slots, prefix products and thread totals are written once
// and read once per level, far apart -- they go through with streaming (evict-first) accesses.
template <int N>
__device__ __forceinline__ void rec_store(uint4* rec, size_t i, const feN<N>& x, const feN<N>& y) {
    fe_store_u4<N, true>(rec + (N / 2) * i, x);
    fe_store_u4<N, true>(rec + (N / 2) * i + N / 4, y);
}
// The point at infinity is the slot whose x is ALL ONES -- never a stored coordinate: the canonical
// fields stay below their modulus, and the weakly reduced field canonicalises the one value that
// collides (2^256 - 1 == c - 1).  No separate flag array: a one-byte flag read at random costs a
// whole DRAM burst, as much as the coordinate it describes (the flags were half of the traffic of
// the forward passes above level 0).
template <int N>
__device__ __forceinline__ bool slot_is_inf(const feN<N>& x) {
    uint32_t a = 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < N; ++i) a &= x.w[i];
    return a == 0xFFFFFFFFu;
}
template <class C>
__device__ __forceinline__ void slot_store(uint4* slots, size_t i, cfe<C> x, const cfe<C>& y, bool inf) {
    constexpr int N = C::Fp::N;
    if (inf) {
#pragma unroll
        for (int k = 0; k < N; ++k) x.w[k] = 0xFFFFFFFFu;
    } else if (slot_is_inf(x)) {
        if constexpr (C::Fp::kind == KIND_SECP_LAZY) x = lazy_canon(typename C::Fp{}, x);
    }
    rec_store<N>(slots, i, x, y);
}
template <int N>
__device__ __forceinline__ feN<N> rec_x(const uint4* rec, size_t i) {  // slots: streaming
    return fe_load_u4<N, LD_STREAM>(rec + (N / 2) * i);
}
template <int N>
__device__ __forceinline__ feN<N> rec_y(const uint4* rec, size_t i) {
    return fe_load_u4<N, LD_STREAM>(rec + (N / 2) * i + N / 4);
}
template <int N>
__device__ __forceinline__ feN<N> pt_x(const uint4* __restrict__ rec, size_t i) {  // input points: keep
    return fe_load_u4<N, LD_KEEP>(rec + (N / 2) * i);
}
template <int N>
__device__ __forceinline__ feN<N> pt_y(const uint4* __restrict__ rec, size_t i) {
    return fe_load_u4<N, LD_KEEP>(rec + (N / 2) * i + N / 4);
}
template <int N>
__device__ __forceinline__ void fe_store_cs(uint4* p, const feN<N>& v) { fe_store_u4<N, true>(p, v); }
template <int N>
__device__ __forceinline__ feN<N> fe_load_cs(const uint4* p) { return fe_load_u4<N, LD_STREAM>(p); }

// column-major coordinates -> 64-byte records (one gather of a point = two 32-byte sectors
// instead of sixteen)
// CE: the curve of the caller's column buffers (Montgomery form); CI: the curve the accumulation
// computes on.  They differ on secp256k1 only, where the tree and the reduction run on the lazy
// plain field of the ECDSA kernels (a product is 145 instead of 204 instructions): coordinates
// are taken out of Montgomery form once here and put back once at the very end.
template <class CE, class CI>
__device__ __forceinline__ cfe<CI> msm_to_internal(const cfe<CE>& v) {
    if constexpr (std::is_same<CE, CI>::value) return v;
    else return fe_from_mont(typename CE::Fp{}, v);   // canonical plain residue: a valid lazy element
}
template <class CE, class CI>
__device__ __forceinline__ cfe<CE> msm_to_external(const cfe<CI>& v) {
    if constexpr (std::is_same<CE, CI>::value) return v;
    else return fe_to_mont(typename CE::Fp{}, fe_from_mont(typename CI::Fp{}, v));  // canonicalise, then x R
}
template <class CE, class CI>
__global__ void __launch_bounds__(256)
k_msm_aos(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
          uint4* __restrict__ rec) {
    constexpr int N = CE::Fp::N;
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    fe_store_u4<N, false>(rec + (N / 2) * i, msm_to_internal<CE, CI>(col_load<N>(px, n, i)));
    fe_store_u4<N, false>(rec + (N / 2) * i + N / 4, msm_to_internal<CE, CI>(col_load<N>(py, n, i)));
}

// One join (see above).  LEVEL0: the operands are input points fetched through vals.
template <class C, bool LEVEL0>
struct TreeJoin {
    size_t dst, src;
    bool active;      // an addition happens
    bool copy2;       // level 0 only: keys differ, both points pass through
    uint32_t v0, v1;  // level 0: vals of the two entries
};

template <class C, bool LEVEL0>
__device__ __forceinline__ TreeJoin<C, LEVEL0> tree_locate(size_t j, int level, size_t m,
                                                           const PairKeys keys, const PairVals vals) {
    TreeJoin<C, LEVEL0> t;
    t.active = t.copy2 = false;
    t.dst = t.src = 0;
    t.v0 = t.v1 = 0;
    if (LEVEL0) {
        const size_t a = 2 * j;
        if (a >= m) return t;
        // the two pairs of the join in one 16-byte load (a is even and the groups start on multiples of 64)
        uint32_t k0, k1 = 0xFFFFFFFFu, va, vb = 0;
        if (a + 1 < m) {
            const uint4 q = *reinterpret_cast<const uint4*>(keys.p + a);
            k0 = q.x; va = q.y; k1 = q.z; vb = q.w;
        } else {
            k0 = keys[a];
            va = vals[a];
        }
        if (k0 >= MSM_NB) return t;  // sorted: k1 is not a bucket either
        t.dst = a;
        t.src = a + 1;
        t.v0 = va;
        if (k1 == k0) {
            t.active = true;
            t.v1 = vb;
        } else {
            t.copy2 = true;          // dst gets entry a; src gets entry a + 1 when it is a bucket
            if (k1 < MSM_NB) t.v1 = vb;
            else t.src = (size_t)-1;
        }
        return t;
    }
    const size_t half = (size_t)1 << level;
    const size_t c = (2 * j + 1) * half;
    if (c >= m) return t;
    const uint32_t k = keys[c];
    if (k >= MSM_NB || keys[c - 1] != k) return t;
    size_t lo = c - half, hi = c - 1;  // first position of key k inside the left half
    while (lo < hi) {
        const size_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    t.dst = lo;
    t.src = c;
    t.active = true;
    return t;
}

template <class C>
__device__ __forceinline__ caff<C> msm_point(const uint4* __restrict__ rec, uint32_t v) {
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    const size_t idx = v & 0x7FFFFFFFu;
    aff q{pt_x<NL>(rec, idx), pt_y<NL>(rec, idx)};
    if (v >> 31) q.y = fe_neg(typename C::Fp{}, q.y);
    return q;
}

// denominator of a join (one when nothing is inverted for it)
template <class C, bool LEVEL0>
__device__ __forceinline__ cfe<C> tree_denominator(const TreeJoin<C, LEVEL0>& t, const uint4* __restrict__ rec,
                                                   const uint4* slots) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    const typename C::Fp f{};
    fe d = fe_one(f);
    if (!t.active) return d;
    fe ax, bx;
    bool ai = false, bi = false;
    if (LEVEL0) {
        ax = pt_x<NL>(rec, t.v0 & 0x7FFFFFFFu);
        bx = pt_x<NL>(rec, t.v1 & 0x7FFFFFFFu);
    } else {
        ax = rec_x<NL>(slots, t.dst);
        bx = rec_x<NL>(slots, t.src);
        ai = slot_is_inf(ax);
        bi = slot_is_inf(bx);
    }
    if (ai || bi) return d;
    if (fe_eq(f, ax, bx)) {  // y is only needed when the x's collide
        fe ay, by;
        if (LEVEL0) {
            ay = msm_point<C>(rec, t.v0).y;
            by = msm_point<C>(rec, t.v1).y;
        } else {
            ay = rec_y<NL>(slots, t.dst);
            by = rec_y<NL>(slots, t.src);
        }
        classify_pair<C>(ax, ay, false, bx, by, false, &d);
        return d;
    }
    return fe_sub(f, ax, bx);
}

// backward step of Montgomery's trick for one join: inv holds the inverse of the product of
// the denominators up to and including this join's; prev the product before it.
template <class C, bool LEVEL0>
__device__ __forceinline__ void tree_apply(const TreeJoin<C, LEVEL0>& t, cfe<C>& inv, const cfe<C>& prev, bool first,
                                           const uint4* __restrict__ rec, uint4* slots) {
    using fe = cfe<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    const typename C::Fp f{};
    if (LEVEL0 && t.copy2) {
        const aff p0 = msm_point<C>(rec, t.v0);
        slot_store<C>(slots, t.dst, p0.x, p0.y, false);
        if (t.src != (size_t)-1) {
            const aff p1 = msm_point<C>(rec, t.v1);
            slot_store<C>(slots, t.src, p1.x, p1.y, false);
        }
        return;
    }
    if (!t.active) return;
    aff A, B;
    bool ai = false, bi = false;
    if (LEVEL0) {
        A = msm_point<C>(rec, t.v0);
        B = msm_point<C>(rec, t.v1);
    } else {
        A.x = rec_x<NL>(slots, t.dst); A.y = rec_y<NL>(slots, t.dst);
        B.x = rec_x<NL>(slots, t.src); B.y = rec_y<NL>(slots, t.src);
        ai = slot_is_inf(A.x);
        bi = slot_is_inf(B.x);
    }
    fe d = fe_one(f);
    const uint32_t kind = classify_pair<C>(A.x, A.y, ai, B.x, B.y, bi, &d);
    fe dinv = inv;
    if (!first) {
        dinv = fe_mul(f, inv, prev);
        inv = fe_mul(f, inv, d);
    }
    fe xr = fe_zero_n<NL>(), yr = fe_zero_n<NL>();
    uint8_t rinf = 0;
    if (kind == K_GENERIC) {
        fe lam = fe_mul(f, fe_sub(f, A.y, B.y), dinv);
        finish_lambda<C>(lam, A.x, B.x, A.y, &xr, &yr);
    } else if (kind == K_TANGENT) {
        fe lam = fe_mul(f, tangent_numerator<C>(A.x), dinv);
        finish_lambda<C>(lam, A.x, A.x, A.y, &xr, &yr);
    } else if (kind == K_COPY_LEFT) {
        xr = A.x; yr = A.y;
    } else if (kind == K_COPY_RIGHT) {
        xr = B.x; yr = B.y;
    } else {
        rinf = 1;
    }
    slot_store<C>(slots, t.dst, xr, yr, rinf != 0);
}

// Single-launch form of one level: the block's one inversion happens inside the kernel
// (prefix products in shared memory; the other warps wait while warp 0 inverts).
template <class C, int K, bool LEVEL0>
__global__ void __launch_bounds__(MSM_TREE_THREADS)
k_msm_tree(size_t m, size_t joins, int level, const PairKeys keys,
           const PairVals vals, const uint4* __restrict__ rec,
           uint4* slots) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    __shared__ uint32_t sm_scan[2 * NL * (MSM_TREE_THREADS / 32)];
    __shared__ uint32_t sm_pref[K * NL * MSM_TREE_THREADS];
    const typename C::Fp f{};
    const size_t j0 = (size_t)blockIdx.x * (MSM_TREE_THREADS * K) + threadIdx.x;
    fe acc = fe_one(f);
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const size_t j = j0 + (size_t)k * MSM_TREE_THREADS;
        if (j < joins) {
            const TreeJoin<C, LEVEL0> t = tree_locate<C, LEVEL0>(j, level, m, keys, vals);
            if (t.active) acc = fe_mul(f, acc, tree_denominator<C, LEVEL0>(t, rec, slots));
        }
#pragma unroll
        for (int w = 0; w < NL; ++w) sm_pref[(k * NL + w) * MSM_TREE_THREADS + threadIdx.x] = acc.w[w];
    }
    fe inv = coop_block_inverse<decltype(f), MSM_TREE_THREADS>(f, acc, sm_scan);
#pragma unroll 1
    for (int k = K - 1; k >= 0; --k) {
        const size_t j = j0 + (size_t)k * MSM_TREE_THREADS;
        if (j >= joins) continue;
        const TreeJoin<C, LEVEL0> t = tree_locate<C, LEVEL0>(j, level, m, keys, vals);
        fe prev = fe_one(f);
        if (k > 0) {
#pragma unroll
            for (int w = 0; w < NL; ++w) prev.w[w] = sm_pref[((k - 1) * NL + w) * MSM_TREE_THREADS + threadIdx.x];
        }
        tree_apply<C, LEVEL0>(t, inv, prev, k == 0, rec, slots);
    }
}

// Three-launch form of one level (no warp ever waits for an inversion):
//   k_msm_tree_fwd : running products of the denominators, parked in `pref` (32 B per join);
//                    every thread keeps the product of ALL OTHER thread totals of its block
//                    (`others`), the block total goes to `totals` (column buffer);
//   batch_invert   : the block totals (a batch MSM_TREE_THREADS * K times smaller);
//   k_msm_tree_bwd : thread total^-1 = block total^-1 * others, unwind, chord / tangent.
// (6K + 8) / K products per addition.
template <class C, int K, bool LEVEL0>
__global__ void __launch_bounds__(MSM_TREE_THREADS, C::Fp::N > 8 ? 4 : 5)
k_msm_tree_fwd(size_t m, size_t joins, int level, const PairKeys keys,
               const PairVals vals, const uint4* __restrict__ rec,
               const uint4* __restrict__ slots,
               uint4* __restrict__ pref, uint4* __restrict__ others, uint32_t* __restrict__ totals,
               size_t tiles, size_t tile0) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    __shared__ uint32_t sm_scan[2 * NL * (MSM_TREE_THREADS / 32)];
    const typename C::Fp f{};
    const size_t tile = tile0 + blockIdx.x;  // tiles [tile0, tile0 + gridDim.x) of the level; totals / tiles are local to this launch
    const size_t j0 = tile * (MSM_TREE_THREADS * K) + threadIdx.x;
    fe acc = fe_one(f);
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const size_t j = j0 + (size_t)k * MSM_TREE_THREADS;
        if (j >= joins) break;
        const TreeJoin<C, LEVEL0> t = tree_locate<C, LEVEL0>(j, level, m, keys, vals);
        if (t.active) acc = fe_mul(f, acc, tree_denominator<C, LEVEL0>(t, rec, slots));
        fe_store_cs<NL>(pref + (NL / 4) * j, acc);
    }
    fe total;
    const fe oth = block_others_product<decltype(f), MSM_TREE_THREADS>(f, acc, sm_scan, &total);
    const size_t tid = tile * MSM_TREE_THREADS + threadIdx.x;
    fe_store_cs<NL>(others + (NL / 4) * tid, oth);
    if (threadIdx.x == 0) col_store(totals, tiles, blockIdx.x, total);
}

template <class C, int K, bool LEVEL0>
__global__ void __launch_bounds__(MSM_TREE_THREADS, C::Fp::N > 8 ? 4 : 5)
k_msm_tree_bwd(size_t m, size_t joins, int level, const PairKeys keys,
               const PairVals vals, const uint4* __restrict__ rec,
               uint4* slots, const uint4* __restrict__ pref,
               const uint4* __restrict__ others, const uint32_t* __restrict__ total_inv, size_t tiles,
               size_t tile0) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const typename C::Fp f{};
    const size_t tile = tile0 + blockIdx.x;
    const size_t j0 = tile * (MSM_TREE_THREADS * K) + threadIdx.x;
    if (j0 >= joins) return;
    const size_t tid = tile * MSM_TREE_THREADS + threadIdx.x;
    fe inv = fe_mul(f, col_load<NL>(total_inv, tiles, blockIdx.x), fe_load_cs<NL>(others + (NL / 4) * tid));
#pragma unroll 1
    for (int k = K - 1; k >= 0; --k) {
        const size_t j = j0 + (size_t)k * MSM_TREE_THREADS;
        if (j >= joins) continue;
        const TreeJoin<C, LEVEL0> t = tree_locate<C, LEVEL0>(j, level, m, keys, vals);
        fe prev = fe_one(f);
        if (k > 0) {
            const size_t jp = j - MSM_TREE_THREADS;
            prev = fe_load_cs<NL>(pref + (NL / 4) * jp);
        }
        tree_apply<C, LEVEL0>(t, inv, prev, k == 0, rec, slots);
    }
}

// Fused form: ALL levels of the tree in one launch.  A block owns the aligned chunk of
// 2 * THREADS * K0 positions: its level-l joins touch only slots of that chunk, so the levels run one
// after the other inside the block (slots go through L2; __syncthreads orders them) and nothing is
// parked in global memory: prefix products live in shared memory, every level does ONE block-level
// (or, on the thin upper levels, warp-level) inversion -- the variable-time one, ~7 us of one warp's
// time while the other resident blocks compute.  Level l has THREADS * K0 / 2^l joins per block:
// K0 / 2^l per thread while that is >= FUSED_KMIN, then warp 0 alone takes them all (K = count / 32),
// so that the scan share (12-14 products per thread and level) stays small against the joins.
// One launch instead of 36, and 8 (keys) + 64 (gather) + ~130 (slots, L2) bytes per addition
// instead of ~320.
constexpr int MSM_FUSED_KMIN = 4;

template <class C, bool LEVEL0, int THREADS_ACTIVE, int NSM>
__device__ __forceinline__ void tree_level_in_block(size_t m, int level, size_t j_first, int K, size_t joins,
                                                    const PairKeys keys, const PairVals vals,
                                                    const uint4* __restrict__ rec, uint4* slots,
                                                    uint32_t* sm_pref, uint32_t* sm_scan) {
    // the THREADS_ACTIVE calling threads (the whole block, or warp 0) take K joins each:
    // j = j_first + k * THREADS_ACTIVE + tid.  sm_pref is word-interleaved over NSM threads.
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    const typename C::Fp f{};
    const int tid = threadIdx.x;
    fe acc = fe_one(f);
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const size_t j = j_first + (size_t)k * THREADS_ACTIVE + tid;
        if (j < joins) {
            const TreeJoin<C, LEVEL0> t = tree_locate<C, LEVEL0>(j, level, m, keys, vals);
            if (t.active) acc = fe_mul(f, acc, tree_denominator<C, LEVEL0>(t, rec, slots));
        }
#pragma unroll
        for (int w = 0; w < NL; ++w) sm_pref[(k * NL + w) * NSM + tid] = acc.w[w];
    }
    fe inv = coop_block_inverse<decltype(f), THREADS_ACTIVE>(f, acc, sm_scan);
#pragma unroll 1
    for (int k = K - 1; k >= 0; --k) {
        const size_t j = j_first + (size_t)k * THREADS_ACTIVE + tid;
        if (j >= joins) continue;
        const TreeJoin<C, LEVEL0> t = tree_locate<C, LEVEL0>(j, level, m, keys, vals);
        fe prev = fe_one(f);
        if (k > 0) {
#pragma unroll
            for (int w = 0; w < NL; ++w) prev.w[w] = sm_pref[((k - 1) * NL + w) * NSM + tid];
        }
        tree_apply<C, LEVEL0>(t, inv, prev, k == 0, rec, slots);
    }
}

template <class C, int K0>
__global__ void __launch_bounds__(MSM_TREE_THREADS, K0 * C::Fp::N > 128 ? 2 : K0 * C::Fp::N > 64 ? 3 : 5)
k_msm_tree_fused(size_t m, const PairKeys keys, const PairVals vals,
                 const uint4* __restrict__ rec, uint4* slots) {
    constexpr int NL = C::Fp::N;
    constexpr int T = MSM_TREE_THREADS;
    static_assert((T * K0) >> (MSM_TREE_LEVELS - 1) >= 32, "the last level still fills a warp");
    static_assert(K0 >= 2 * MSM_FUSED_KMIN, "warp 0 takes at most K0 joins per lane on the thin levels");
    extern __shared__ uint32_t sm_dyn[];
    uint32_t* sm_pref = sm_dyn;                       // K0 * NL * T words
    uint32_t* sm_scan = sm_dyn + K0 * NL * T;         // 2 * NL * (T / 32) words
    {
        const size_t joins = (m + 1) / 2;
        tree_level_in_block<C, true, T, T>(m, 0, (size_t)blockIdx.x * (T * K0), K0, joins, keys, vals, rec, slots,
                                           sm_pref, sm_scan);
    }
#pragma unroll 1
    for (int level = 1; level < MSM_TREE_LEVELS; ++level) {
        __syncthreads();  // the slots of the level below are complete (and sm_pref / sm_scan are free)
        const size_t span = (size_t)2 << level;
        const size_t joins = (m + span - 1) / span;
        const int count = (T * K0) >> level;          // joins of this block on this level
        const size_t j_first = (size_t)blockIdx.x * count;
        if (j_first >= joins) continue;               // uniform over the block
        if (count >= T * MSM_FUSED_KMIN) {
            tree_level_in_block<C, false, T, T>(m, level, j_first, count / T, joins, keys, vals, rec, slots, sm_pref, sm_scan);
        } else if (threadIdx.x < 32) {                // warp 0 alone: K = count / 32 <= 4 * KMIN
            tree_level_in_block<C, false, 32, T>(m, level, j_first, count / 32, joins, keys, vals, rec, slots, sm_pref, sm_scan);
        }
    }
}

// The THIN levels fused: levels [first, MSM_TREE_LEVELS) in one launch.  Level 0 and 1 are wide and
// bound by memory latency (they want every warp the SM can hold: the three-launch kernels); from
// level 2 on a level has so few joins that its three launches mostly wait -- for the inversion of
// the totals and for each other.  Here a block owns 2 * THREADS * K0 << first positions and walks
// the remaining levels by itself (block-level inversion per level while the level still gives every
// thread a join, warp 0 alone below that); 16 KB of shared memory per block, so several blocks per
// SM hide each other's inversions.
template <class C, int K0>
__global__ void __launch_bounds__(MSM_TREE_THREADS, C::Fp::N > 8 ? 4 : 5)
k_msm_tree_upper(size_t m, int first, const PairKeys keys, const PairVals vals,
                 const uint4* __restrict__ rec, uint4* slots) {
    constexpr int NL = C::Fp::N;
    constexpr int T = MSM_TREE_THREADS;
    __shared__ uint32_t sm_pref[K0 * NL * T];
    __shared__ uint32_t sm_scan[2 * NL * (T / 32)];
#pragma unroll 1
    for (int level = first; level < MSM_TREE_LEVELS; ++level) {
        if (level > first) __syncthreads();  // the slots of the level below are complete
        const size_t span = (size_t)2 << level;
        const size_t joins = (m + span - 1) / span;
        const int count = (T * K0) >> (level - first);  // joins of this block on this level
        const size_t j_first = (size_t)blockIdx.x * count;
        if (j_first >= joins) continue;                 // uniform over the block
        if (count >= T) {
            tree_level_in_block<C, false, T, T>(m, level, j_first, count / T, joins, keys, vals, rec, slots, sm_pref, sm_scan);
        } else if (threadIdx.x < 32) {
            tree_level_in_block<C, false, 32, T>(m, level, j_first, count / 32, joins, keys, vals, rec, slots, sm_pref, sm_scan);
        }
    }
}

// marginal sums, stage 1: thread (w, k, e, part) adds the 32 buckets of window w whose
// k-th base-32 digit is e and whose next digit (cyclically) is `part`.
template <class C>
__global__ void __launch_bounds__(128)
k_msm_marginal_parts(const uint32_t* __restrict__ buckets, uint32_t* __restrict__ parts) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
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
        acc = jac_add<C>(acc, jac_load<NL>(buckets, MSM_NB, (size_t)w * MSM_BUCKETS + b));
    }
    jac_store<NL>(parts, (size_t)MSM_WINDOWS * 3 * 1024, t, acc);
}
// stage 2: thread (w, k, e) folds its 32 parts
template <class C>
__global__ void __launch_bounds__(128)
k_msm_marginal_fold(const uint32_t* __restrict__ parts, uint32_t* __restrict__ marg) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= MSM_WINDOWS * 3 * 32) return;
    jac acc = jac_infinity<C>();
#pragma unroll 1
    for (uint32_t p = 0; p < 32; ++p)
        acc = jac_add<C>(acc, jac_load<NL>(parts, (size_t)MSM_WINDOWS * 3 * 1024, (size_t)t * 32 + p));
    jac_store<NL>(marg, (size_t)MSM_WINDOWS * 3 * 32, t, acc);
}
// stage 3: thread (w, j): j < 3 -> sum_e e * C^j_e (running sums); j == 3 -> sum_e C^0_e
template <class C>
__global__ void __launch_bounds__(128)
k_msm_weighted(const uint32_t* __restrict__ marg, uint32_t* __restrict__ wsum) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= MSM_WINDOWS * 4) return;
    const uint32_t w = t >> 2, j = t & 3;
    const size_t cnt = (size_t)MSM_WINDOWS * 3 * 32;
    jac acc = jac_infinity<C>();
    if (j == 3) {
#pragma unroll 1
        for (uint32_t e = 0; e < 32; ++e) acc = jac_add<C>(acc, jac_load<NL>(marg, cnt, (size_t)(w * 3) * 32 + e));
    } else {
        jac run = jac_infinity<C>();
#pragma unroll 1
        for (int e = 31; e >= 1; --e) {
            run = jac_add<C>(run, jac_load<NL>(marg, cnt, (size_t)(w * 3 + j) * 32 + e));
            acc = jac_add<C>(acc, run);
        }
    }
    jac_store<NL>(wsum, (size_t)MSM_WINDOWS * 4, t, acc);
}
// stage 4 (one block of 32 threads): thread w forms S_w = (sum B) + W0 + 32 W1 + 1024 W2
// (weights b + 1), shifts it by 2^(16 w); thread 0 adds the windows and converts to affine.
template <class C>
__global__ void __launch_bounds__(32)
k_msm_combine(const uint32_t* __restrict__ wsum, uint32_t* __restrict__ ox, uint32_t* __restrict__ oy,
              uint8_t* __restrict__ oinf) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    __shared__ uint32_t win[3 * NL * MSM_WINDOWS];
    const uint32_t w = threadIdx.x;
    const size_t cnt = (size_t)MSM_WINDOWS * 4;
    if (w < MSM_WINDOWS) {
        jac s = jac_load<NL>(wsum, cnt, w * 4 + 2);
#pragma unroll 1
        for (int i = 0; i < 5; ++i) s = jac_dbl<C>(s);
        s = jac_add<C>(s, jac_load<NL>(wsum, cnt, w * 4 + 1));
#pragma unroll 1
        for (int i = 0; i < 5; ++i) s = jac_dbl<C>(s);
        s = jac_add<C>(s, jac_load<NL>(wsum, cnt, w * 4 + 0));
        s = jac_add<C>(s, jac_load<NL>(wsum, cnt, w * 4 + 3));
#pragma unroll 1
        for (uint32_t i = 0; i < MSM_C * w; ++i) s = jac_dbl<C>(s);
        jac_store<NL>(win, MSM_WINDOWS, w, s);
    }
    __syncthreads();
    if (w == 0) {
        const typename C::Fp f{};
        jac acc = jac_infinity<C>();
#pragma unroll 1
        for (int i = 0; i < MSM_WINDOWS; ++i) acc = jac_add<C>(acc, jac_load<NL>(win, MSM_WINDOWS, i));
        if (jac_is_inf<C>(acc)) {
            col_store(ox, 1, 0, fe_zero_n<NL>());
            col_store(oy, 1, 0, fe_zero_n<NL>());
            oinf[0] = 1;
        } else {
            aff a = jac_to_aff_with<C>(acc, fe_inv_var(f, acc.Z));
            col_store(ox, 1, 0, a.x);
            col_store(oy, 1, 0, a.y);
            oinf[0] = 0;
        }
    }
}

// ---------------------------------------------------------------- bucket reduction, second form
// Used after the batch-affine tree.  Same decomposition as above (three base-32 marginal sums
// per window), arranged so that no thread runs a long serial chain -- the chip is nearly empty
// at this stage, so depth, not work, is the cost:
//   k_msm_red_parts    : thread (w, k, e, part, sub) adds 8 buckets.  A bucket is read straight
//                        from the tree's slots (slot[start] and the slots at multiples of
//                        2^MSM_TREE_LEVELS inside its run), all AFFINE operands: mixed additions.
//   k_msm_red_fold     : warp (w, k, e): 4 partials per lane, then a 5-step shuffle tree.
//   k_msm_red_weighted : warp (w, k): lane e holds C_e; inclusive suffix scan S_e = sum_{e' >= e} C_e'
//                        (5 steps), then sum_e e C_e = sum_{e >= 1} S_e (5-step tree); S_0 is the
//                        plain total.
//   k_msm_red_combine  : lane w forms S_w, shifts it by 2^(16 w); shuffle tree over the windows.
constexpr uint32_t MSM_RED_PARTS = MSM_WINDOWS * 3 * 32 * 32 * 4;

template <int N>
__device__ __forceinline__ jacN<N> jac_shfl_down(const jacN<N>& p, int d) {
    jacN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        r.X.w[i] = __shfl_down_sync(0xFFFFFFFFu, p.X.w[i], d);
        r.Y.w[i] = __shfl_down_sync(0xFFFFFFFFu, p.Y.w[i], d);
        r.Z.w[i] = __shfl_down_sync(0xFFFFFFFFu, p.Z.w[i], d);
    }
    return r;
}
// lane 0 ends with the sum of all 32 lanes' points
template <class C>
__device__ __forceinline__ cjac<C> warp_sum_points(cjac<C> acc, int lane) {
    using jac = cjac<C>;
#pragma unroll 1
    for (int d = 16; d >= 1; d >>= 1) {
        const jac other = jac_shfl_down(acc, d);
        if (lane < d) acc = jac_add<C>(acc, other);
    }
    return acc;
}

template <class C>
__global__ void __launch_bounds__(128, 4)
k_msm_red_parts(size_t m, const PairKeys keys, const uint32_t* __restrict__ starts,
                const uint4* __restrict__ slots,
                uint32_t* __restrict__ parts, uint32_t w0) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x + w0 * (3 * 4096);  // windows [w0, w0 + gridDim.x / 96)
    if (t >= MSM_RED_PARTS) return;
    const uint32_t sub = t & 3, part = (t >> 2) & 31, e = (t >> 7) & 31, k = (t >> 12) % 3, w = t / (3 * 4096);
    const size_t step = (size_t)1 << MSM_TREE_LEVELS;
    jac acc = jac_infinity<C>();
#pragma unroll 1
    for (uint32_t v = sub * 8; v < sub * 8 + 8; ++v) {
        uint32_t b;
        if (k == 0) b = e + 32 * part + 1024 * v;        // lo = e
        else if (k == 1) b = part + 32 * e + 1024 * v;   // mid = e
        else b = part + 32 * v + 1024 * e;               // top = e
        const uint32_t id = w * MSM_BUCKETS + b;
        const size_t s = starts[id];
        if (s == 0xFFFFFFFFu) continue;
        {
            const fe x = rec_x<NL>(slots, s);
            if (!slot_is_inf(x)) acc = jac_madd<C>(acc, aff{x, rec_y<NL>(slots, s)});
        }
#pragma unroll 1
        for (size_t a = (s / step + 1) * step; a < m && keys[a] == id; a += step)
        {
            const fe x = rec_x<NL>(slots, a);
            if (!slot_is_inf(x)) acc = jac_madd<C>(acc, aff{x, rec_y<NL>(slots, a)});
        }
    }
    jac_store<NL>(parts, MSM_RED_PARTS, t, acc);
}

template <class C>
__global__ void __launch_bounds__(128)
k_msm_red_fold(const uint32_t* __restrict__ parts, uint32_t* __restrict__ marg, uint32_t w0) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const uint32_t gw = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) + w0 * 96, lane = threadIdx.x & 31;
    if (gw >= MSM_WINDOWS * 3 * 32) return;  // whole warps leave together
    const size_t base = ((size_t)gw * 32 + lane) * 4;
    jac acc = jac_load<NL>(parts, MSM_RED_PARTS, base);
#pragma unroll 1
    for (int sub = 1; sub < 4; ++sub) acc = jac_add<C>(acc, jac_load<NL>(parts, MSM_RED_PARTS, base + sub));
    acc = warp_sum_points<C>(acc, lane);
    if (lane == 0) jac_store<NL>(marg, (size_t)MSM_WINDOWS * 3 * 32, gw, acc);
}

template <class C>
__global__ void __launch_bounds__(128)
k_msm_red_weighted(const uint32_t* __restrict__ marg, uint32_t* __restrict__ wsum, uint32_t w0, uint32_t w1) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const uint32_t gw = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) + w0 * 3, lane = threadIdx.x & 31;
    if (gw >= w1 * 3) return;
    const uint32_t w = gw / 3, k = gw % 3;
    jac S = jac_load<NL>(marg, (size_t)MSM_WINDOWS * 3 * 32, (size_t)gw * 32 + lane);
#pragma unroll 1
    for (int d = 1; d < 32; d <<= 1) {  // inclusive suffix sums
        const jac other = jac_shfl_down(S, d);
        if (lane + d < 32) S = jac_add<C>(S, other);
    }
    const size_t cnt = (size_t)MSM_WINDOWS * 4;
    if (lane == 0 && k == 0) jac_store<NL>(wsum, cnt, w * 4 + 3, S);  // S_0 = sum_e C_e
    jac R = lane == 0 ? jac_infinity<C>() : S;
    R = warp_sum_points<C>(R, lane);                              // sum_{e >= 1} S_e = sum_e e C_e
    if (lane == 0) jac_store<NL>(wsum, cnt, w * 4 + k, R);
}

// Doubling of one point by a GROUP of four adjacent lanes: the seven products of dbl-2009-l
// (a = 0) have depth three, the eight of dbl-2001-b (a = -3) depth four, so the lanes run one
// product each per level and exchange the
// results with shuffles; every lane of the group holds the whole point before and after.  A
// chain of dependent doublings run by a single warp is pure latency: three products per
// doubling instead of seven.  All 32 lanes of the warp must call (full-mask shuffles).
template <int N>
__device__ __forceinline__ feN<N> fe_from_lane(const feN<N>& v, int src) {
    feN<N> r;
#pragma unroll
    for (int i = 0; i < N; ++i) r.w[i] = __shfl_sync(0xFFFFFFFFu, v.w[i], src);
    return r;
}
template <class C>
__device__ __forceinline__ cjac<C> jac_dbl_group4(const cjac<C>& p, int lane) {
    static_assert(C::a_kind == A_ZERO || C::a_kind == A_MINUS3, "group doubling: a = 0 or a = -3");
    using fe = cfe<C>;
    const typename C::Fp f{};
    const int r = lane & 3, base = lane & ~3;
    if constexpr (C::a_kind == A_MINUS3) {  // dbl-2001-b: eight products in four levels
        // level 1: Z^2 | Y^2 | (Y + Z)^2
        fe u = fe_select(r == 0, p.Z, fe_select(r == 1, p.Y, fe_add(f, p.Y, p.Z)));
        const fe l1 = fe_mul_inl(f, u, u);
        const fe delta = fe_from_lane(l1, base), gamma = fe_from_lane(l1, base + 1), yz2 = fe_from_lane(l1, base + 2);
        // level 2: X gamma | (X - delta)(X + delta)
        u = fe_select(r == 0, p.X, fe_sub(f, p.X, delta));
        fe v = fe_select(r == 0, gamma, fe_add(f, p.X, delta));
        const fe l2 = fe_mul_inl(f, u, v);
        const fe beta = fe_from_lane(l2, base), t = fe_from_lane(l2, base + 1);
        const fe alpha = fe_add(f, fe_dbl(f, t), t);
        // level 3: alpha^2 | gamma^2
        u = fe_select(r == 0, alpha, gamma);
        const fe l3 = fe_mul_inl(f, u, u);
        const fe alpha2 = fe_from_lane(l3, base), gamma2 = fe_from_lane(l3, base + 1);
        const fe beta4 = fe_dbl(f, fe_dbl(f, beta));
        cjac<C> o;
        o.X = fe_sub(f, alpha2, fe_dbl(f, beta4));
        o.Z = fe_sub(f, fe_sub(f, yz2, gamma), delta);
        // level 4: alpha (4 beta - X3), the same on every lane
        o.Y = fe_sub(f, fe_mul_inl(f, alpha, fe_sub(f, beta4, o.X)), fe_mul8(f, gamma2));
        return o;
    }
    // level 1: X^2 | Y^2 | Y Z
    fe u = fe_select(r == 1 || r == 2, p.Y, p.X);
    fe v = fe_select(r == 2, p.Z, u);
    const fe l1 = fe_mul_inl(f, u, v);
    const fe A = fe_from_lane(l1, base), B = fe_from_lane(l1, base + 1), YZ = fe_from_lane(l1, base + 2);
    // level 2: B^2 | (X + B)^2 | (3A)^2
    const fe E = fe_add(f, fe_dbl(f, A), A);
    u = fe_select(r == 1, fe_add(f, p.X, B), fe_select(r == 2, E, B));
    const fe l2 = fe_mul_inl(f, u, u);
    const fe Cc = fe_from_lane(l2, base), T = fe_from_lane(l2, base + 1), F = fe_from_lane(l2, base + 2);
    fe D = fe_dbl(f, fe_sub(f, fe_sub(f, T, A), Cc));
    cjac<C> o;
    o.X = fe_sub(f, F, fe_dbl(f, D));
    // level 3: E (D - X3), the same on every lane
    o.Y = fe_sub(f, fe_mul_inl(f, E, fe_sub(f, D, o.X)), fe_mul8(f, Cc));
    o.Z = fe_dbl(f, YZ);
    return o;
}

// Window combine, two kernels.  k_msm_red_shift: groups of four lanes own one window each of
// [w0, w1): S_w by Horner over its three weighted marginals, then the shift by 2^(16 w) --
// doublings by the lane group -- and the shifted window sum goes to `win`.  k_msm_red_final: one
// warp tree-sums the windows and converts to affine.  (Split so that the window groups of the
// pipeline shift independently, the long chains of the high windows behind other groups' trees.)
constexpr int MSM_COMBINE_THREADS = 96;
template <class C>
__global__ void __launch_bounds__(MSM_COMBINE_THREADS)
k_msm_red_shift(const uint32_t* __restrict__ wsum, uint32_t* __restrict__ win, uint32_t w0, uint32_t w1) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    static_assert(MSM_WINDOWS * 4 <= MSM_COMBINE_THREADS, "one lane group per window");
    const int lane = threadIdx.x & 31;
    const uint32_t w = w0 + (threadIdx.x >> 2);  // window of this lane group
    const size_t cnt = (size_t)MSM_WINDOWS * 4;
    const bool live = w < w1;
    auto dbl = [&](const jac& p) -> jac {
        if constexpr (C::a_kind == A_ZERO || C::a_kind == A_MINUS3) return jac_dbl_group4<C>(p, lane);
        else return jac_dbl_flat<C>(p);
    };
    jac s = jac_infinity<C>();
    if (live) s = jac_load<NL>(wsum, cnt, w * 4 + 2);
#pragma unroll 1
    for (int i = 0; i < 5; ++i) s = dbl(s);
    if (live) s = jac_add<C>(s, jac_load<NL>(wsum, cnt, w * 4 + 1));
#pragma unroll 1
    for (int i = 0; i < 5; ++i) s = dbl(s);
    if (live) {
        s = jac_add<C>(s, jac_load<NL>(wsum, cnt, w * 4 + 0));
        s = jac_add<C>(s, jac_load<NL>(wsum, cnt, w * 4 + 3));
    }
    // an empty window (the carry window almost always is) has nothing to shift; the loop runs as
    // long as the warp's highest non-empty window needs (uniform trip count: shuffles inside)
    uint32_t reps = live && !jac_is_inf<C>(s) ? MSM_C * w : 0u;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, reps, d);
        reps = other > reps ? other : reps;
    }
    const uint32_t mine = live && !jac_is_inf<C>(s) ? MSM_C * w : 0u;
#pragma unroll 1
    for (uint32_t i = 0; i < reps; ++i) {
        const jac t = dbl(s);
        if (i < mine) s = t;
    }
    if (live && (threadIdx.x & 3) == 0) jac_store<NL>(win, MSM_WINDOWS, w, s);
}
template <class C, class CE>
__global__ void __launch_bounds__(32)
k_msm_red_final(const uint32_t* __restrict__ win, uint32_t* __restrict__ ox, uint32_t* __restrict__ oy,
                uint8_t* __restrict__ oinf) {
    using fe = cfe<C>;
    using jac = cjac<C>;
    using aff = caff<C>;
    constexpr int NL = C::Fp::N;
    (void)sizeof(fe); (void)sizeof(jac); (void)sizeof(aff);
    const int lane = threadIdx.x & 31;
    jac acc = lane < MSM_WINDOWS ? jac_load<NL>(win, MSM_WINDOWS, lane) : jac_infinity<C>();
    acc = warp_sum_points<C>(acc, lane);
    if (lane == 0) {
        const typename C::Fp f{};
        if (jac_is_inf<C>(acc)) {
            col_store(ox, 1, 0, fe_zero_n<NL>());
            col_store(oy, 1, 0, fe_zero_n<NL>());
            oinf[0] = 1;
        } else {
            aff a = jac_to_aff_with<C>(acc, fe_inv_var(f, acc.Z));
            col_store(ox, 1, 0, msm_to_external<CE, C>(a.x));
            col_store(oy, 1, 0, msm_to_external<CE, C>(a.y));
            oinf[0] = 0;
        }
    }
}

// ---------------------------------------------------------------- host side
struct MsmPlan {
    size_t pairs, region, sort_temp, total;
    size_t slices;
    size_t off_keys, off_vals, off_keys2, off_vals2, off_buckets, off_edge, off_edge_key, off_parts, off_marg, off_wsum, off_win, off_temp;
    size_t off_rec, off_slots, off_starts, off_pref, off_others, off_totals;
    size_t max_tiles;
};
static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

// 0 auto (= 2), 1 mixed-Jacobian slices, 2 batch-affine tree with three launches per level,
// 3 batch-affine tree with one launch per level (inversion inside the block),
// 4 / 5 batch-affine tree, all levels fused into one launch (16 / 8 level-0 joins per thread)
static int g_msm_form = 0;
void set_msm_form(int form) { g_msm_form = form; }
static bool msm_affine() { return g_msm_form != 1; }
constexpr int MSM_TREE_KMIN = 2;  // fewest joins per thread any level uses
constexpr int MSM_GROUPS = 4;     // most window groups of the two-stream pipeline (scratch is sized for it)
constexpr uint32_t MSM_GROUP_CUT = 8;  // first window of the high group when there are two
constexpr int MSM_GROUPS_DEFAULT = 2;  // measured: 4.02 / 3.80 / 4.41 ms with 1 / 2 / 4 groups (secp256k1, 2^20)

static MsmPlan msm_plan(size_t n, int limbs) {
    MsmPlan p{};
    const size_t jb = (size_t)12 * limbs, rb = (size_t)8 * limbs, fb = (size_t)4 * limbs;  // bytes: Jacobian point, record, element
    p.region = (n + ((size_t)1 << MSM_TREE_LEVELS) - 1) >> MSM_TREE_LEVELS << MSM_TREE_LEVELS;  // positions per window
    p.pairs = p.region * MSM_WINDOWS;
    p.sort_temp = (size_t)2 * 4 * MSM_NB + 4 * 1024;  // bucket counts | scatter cursors | block totals of the scan
    size_t at = 0;
    auto take = [&](size_t bytes) { size_t o = at; at += align256(bytes); return o; };
    p.off_keys = p.off_vals = 0;  // unsorted pairs are never stored (the counting sort recodes)
    p.off_keys2 = take(8 * p.pairs);  // (key, val) pairs
    p.off_vals2 = p.off_keys2;
    p.slices = (p.pairs + MSM_SLICE - 1) / MSM_SLICE;
    p.off_buckets = take(jb * MSM_NB);
    p.off_parts = take(jb * MSM_RED_PARTS);
    p.off_marg = take(jb * MSM_WINDOWS * 3 * 32);
    p.off_wsum = take(jb * MSM_WINDOWS * 4);
    p.off_win = take(jb * MSM_WINDOWS);
    p.off_temp = take(p.sort_temp);
    p.off_starts = take((size_t)4 * MSM_NB);
    // the two accumulation forms never run in the same call: their scratch overlaps
    const size_t fork = at;
    p.off_edge = take(jb * 2 * p.slices);
    p.off_edge_key = take((size_t)4 * 2 * p.slices);
    const size_t end_jac = at;
    at = fork;
    p.off_rec = take(rb * n);
    p.off_slots = take(rb * p.pairs);
    const size_t joins0 = (p.pairs + 1) / 2;
    p.off_pref = take(fb * joins0);
    // tiles of the thinnest level, one rounding tile per window group; totals | inverses per group
    p.max_tiles = (joins0 + (size_t)MSM_TREE_THREADS * MSM_TREE_KMIN - 1) / ((size_t)MSM_TREE_THREADS * MSM_TREE_KMIN) + 2 * MSM_GROUPS;
    p.off_others = take(fb * MSM_TREE_THREADS * p.max_tiles);
    p.off_totals = take(2 * fb * (p.max_tiles + 64 * (MSM_GROUPS + 1)));
    p.total = at > end_jac ? at : end_jac;
    return p;
}
size_t msm_scratch_bytes(size_t n, int curve) { return n ? msm_plan(n, curve_limbs(curve)).total : 0; }

struct TreeBufs {
    PairKeys keys;
    PairVals vals;
    const uint4* rec;
    uint4* slots;
    uint4 *pref, *others;
    uint32_t* totals;
    size_t max_tiles;
    cudaStream_t aux;           // second stream + fork / join events (may be null: one stream then)
    cudaEvent_t fork, join;
};
template <class C, int K, bool LEVEL0>
static cudaError_t launch_tree(int curve, size_t m, int level, const TreeBufs& b, bool split, cudaStream_t s) {
    const size_t span = (size_t)2 << level;
    const size_t joins = (m + span - 1) / span;  // nodes of size 2^(level+1) that have a left half
    const size_t per_block = (size_t)MSM_TREE_THREADS * K;
    const size_t tiles = (joins + per_block - 1) / per_block;
    const unsigned blocks = (unsigned)tiles;
    if constexpr (K * C::Fp::N <= 64) {  // the single-launch form parks K prefixes per thread in shared memory
        if (!split) {
            k_msm_tree<C, K, LEVEL0><<<blocks, MSM_TREE_THREADS, 0, s>>>(m, joins, level, b.keys, b.vals, b.rec, b.slots);
            return cudaGetLastError();
        }
    }
    // The totals' inversion is ~40 us of pure latency (one warp per 512 totals runs safegcd).  A level
    // is therefore cut into parts that alternate between two streams: while one part inverts, the
    // forward pass or the unwind of another runs.
    constexpr int NL = C::Fp::N;
    const size_t parts = b.aux && tiles >= 64 ? 2 : 1;  // four parts measured slower (two inversions in a row per stream)
    const size_t cap = b.max_tiles + 64;  // totals | inverses: `parts` regions of cap / parts elements each
    if (parts > 1) {
        if (cudaError_t e = cudaEventRecord(b.fork, s)) return e;
        if (cudaError_t e = cudaStreamWaitEvent(b.aux, b.fork, 0)) return e;
    }
    for (size_t h = 0; h < parts; ++h) {
        const size_t t0 = tiles * h / parts, cnt = tiles * (h + 1) / parts - t0;
        cudaStream_t hs = (h & 1) ? b.aux : s;
        uint32_t* tot = b.totals + (size_t)NL * (cap / parts) * h;
        uint32_t* inv = b.totals + (size_t)NL * (cap + (cap / parts) * h);
        k_msm_tree_fwd<C, K, LEVEL0><<<(unsigned)cnt, MSM_TREE_THREADS, 0, hs>>>(m, joins, level, b.keys, b.vals, b.rec, b.slots,
                                                                               b.pref, b.others, tot, cnt, t0);
        if constexpr (C::Fp::kind == KIND_SECP_LAZY) {
            if (cudaError_t e = launch_batch_invert_secp_lazy(cnt, tot, inv, hs)) return e;
        } else {
            if (cudaError_t e = launch_batch_invert(curve, 0, cnt, tot, inv, hs)) return e;
        }
        k_msm_tree_bwd<C, K, LEVEL0><<<(unsigned)cnt, MSM_TREE_THREADS, 0, hs>>>(m, joins, level, b.keys, b.vals, b.rec, b.slots,
                                                                               b.pref, b.others, inv, cnt, t0);
    }
    if (parts > 1) {
        if (cudaError_t e = cudaEventRecord(b.join, b.aux)) return e;
        if (cudaError_t e = cudaStreamWaitEvent(s, b.join, 0)) return e;
    }
    return cudaGetLastError();
}

template <class C, int K0>
static cudaError_t launch_tree_fused(size_t m, const TreeBufs& b, cudaStream_t s) {
    constexpr int NL = C::Fp::N;
    const size_t per_block = (size_t)2 * MSM_TREE_THREADS * K0;  // positions
    const unsigned blocks = (unsigned)((m + per_block - 1) / per_block);
    const size_t smem = ((size_t)K0 * NL * MSM_TREE_THREADS + 2 * NL * (MSM_TREE_THREADS / 32)) * sizeof(uint32_t);
    if (smem > 48 * 1024)
        if (cudaError_t e = cudaFuncSetAttribute(k_msm_tree_fused<C, K0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
            return e;
    k_msm_tree_fused<C, K0><<<blocks, MSM_TREE_THREADS, smem, s>>>(m, b.keys, b.vals, b.rec, b.slots);
    return cudaGetLastError();
}

template <class C, int K0>
static cudaError_t launch_tree_upper(size_t m, int first, const TreeBufs& b, cudaStream_t s) {
    static_assert((MSM_TREE_THREADS * K0) >> (MSM_TREE_LEVELS - 1) >= 8, "warp 0 still has joins on the last level");
    const size_t per_block = ((size_t)2 * MSM_TREE_THREADS * K0) << first;  // positions
    const unsigned blocks = (unsigned)((m + per_block - 1) / per_block);
    k_msm_tree_upper<C, K0><<<blocks, MSM_TREE_THREADS, 0, s>>>(m, first, b.keys, b.vals, b.rec, b.slots);
    return cudaGetLastError();
}

template <class C, class CI = C>
static cudaError_t run_msm(int curve, size_t n, const uint32_t* scalars, const uint32_t* px, const uint32_t* py,
                           const uint8_t* pinf, uint32_t* ox, uint32_t* oy, uint8_t* oinf,
                           void* scratch, cudaStream_t s, int* launches, cudaEvent_t points_ready,
                           const MsmAux& aux) {
    constexpr int NL = C::Fp::N;
    MsmPlan p = msm_plan(n, NL);
    uint8_t* base = (uint8_t*)scratch;
    uint32_t *keys = (uint32_t*)(base + p.off_keys), *vals = (uint32_t*)(base + p.off_vals);
    uint2* pairs2 = (uint2*)(base + p.off_keys2);
    uint32_t *buckets = (uint32_t*)(base + p.off_buckets), *parts = (uint32_t*)(base + p.off_parts);
    uint32_t *marg = (uint32_t*)(base + p.off_marg), *wsum = (uint32_t*)(base + p.off_wsum);
    (void)keys; (void)vals;  // the unsorted pairs are never stored: the scatter pass recodes
    uint32_t* counts = (uint32_t*)(base + p.off_temp);
    uint32_t* cursor = counts + MSM_NB;
    uint32_t* starts = (uint32_t*)(base + p.off_starts);
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)4 * MSM_NB, s);
    if (e != cudaSuccess) return e;
    const unsigned bpw = (unsigned)((n + 255) / 256);
    k_msm_hist<C><<<bpw, 256, 0, s>>>(n, scalars, pinf, counts);
    uint32_t* block_totals = cursor + MSM_NB;
    k_msm_scan_blocks<<<MSM_SCAN_BLOCKS, MSM_SCAN_THREADS, 0, s>>>(counts, starts, block_totals);
    k_msm_scan_tops<<<1, MSM_SCAN_THREADS, 0, s>>>(block_totals, (uint32_t)p.region);
    k_msm_scan_finish<<<MSM_SCAN_BLOCKS, MSM_SCAN_THREADS, 0, s>>>(counts, block_totals, starts, cursor, pairs2, (uint32_t)p.region);
    k_msm_scatter<C><<<bpw * MSM_WINDOWS, 256, 0, s>>>(n, scalars, pinf, cursor, pairs2);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // digits and sort need the scalars (and the infinity mask) only: a host caller uploads the
    // points meanwhile and hands over the event that says they have arrived
    if (points_ready && (e = cudaStreamWaitEvent(s, points_ready, 0)) != cudaSuccess) return e;
    if (msm_affine()) {
        uint4 *rec = (uint4*)(base + p.off_rec), *slots = (uint4*)(base + p.off_slots);
        k_msm_aos<C, CI><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, px, py, rec);
        uint32_t* win = (uint32_t*)(base + p.off_win);
        const bool fused = g_msm_form == 4 || g_msm_form == 5;
        const bool split = g_msm_form != 3;
        // Window groups, highest windows first: a group is an independent sub-problem (its own
        // region of the sorted pairs, its own buckets), so the groups alternate between two streams
        // and the latency-bound tail of one -- thin tree levels, the totals' inversions, the
        // marginal folds, the doubling chain of its shift (longest for the high windows) -- runs
        // behind the wide tree levels of the next.
        static const int groups_knob = [] { const char* v = getenv("GECC_MSM_GROUPS"); return v ? atoi(v) : 0; }();  // A/B timing
        const int want_groups = groups_knob >= 1 && groups_knob <= MSM_GROUPS ? groups_knob : MSM_GROUPS_DEFAULT;
        const int G = (aux.stream && aux.fork && aux.join && !fused && n >= ((size_t)1 << 16)) ? want_groups : 1;
        if (G > 1) {
            if ((e = cudaEventRecord(aux.fork, s)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(aux.stream, aux.fork, 0)) != cudaSuccess) return e;
        }
        size_t tile_base = 0;
        for (int g = 0; g < G; ++g) {
            uint32_t w1 = (uint32_t)(MSM_WINDOWS * (G - g) / G), w0 = (uint32_t)(MSM_WINDOWS * (G - g - 1) / G);
            if (G == 2) {  // the high group carries the long doubling chain of its shift: it gets fewer windows
                static const int cut_knob = [] { const char* v = getenv("GECC_MSM_CUT"); return v ? atoi(v) : 0; }();  // A/B timing
                const uint32_t cut = cut_knob >= 1 && cut_knob < MSM_WINDOWS ? (uint32_t)cut_knob : MSM_GROUP_CUT;
                w1 = g == 0 ? MSM_WINDOWS : cut;
                w0 = g == 0 ? cut : 0;
            }
            const size_t pos0 = (size_t)w0 * p.region, m = (size_t)(w1 - w0) * p.region;
            cudaStream_t hs = (g & 1) ? aux.stream : s;
            const size_t tiles_max = ((m + 1) / 2 + (size_t)MSM_TREE_THREADS * MSM_TREE_KMIN - 1) / ((size_t)MSM_TREE_THREADS * MSM_TREE_KMIN) + 1;
            TreeBufs tb{PairKeys{pairs2 + pos0}, PairVals{pairs2 + pos0}, rec, slots + (NL / 2) * pos0,
                        (uint4*)(base + p.off_pref) + (NL / 4) * (pos0 / 2),
                        (uint4*)(base + p.off_others) + (size_t)(NL / 4) * MSM_TREE_THREADS * tile_base,
                        (uint32_t*)(base + p.off_totals) + (size_t)2 * NL * (tile_base + (size_t)64 * g), tiles_max,
                        G > 1 ? nullptr : aux.stream, aux.fork, aux.join};
            tile_base += tiles_max;
            // K joins per thread: as many as keep >= ~8 blocks per SM in flight (the scan share is
            // 14 / K products per join); thin levels take fewer so that the chip stays filled.  The
            // single-launch form parks prefixes in shared memory: K <= 8.
            const size_t fill = (size_t)148 * (G > 1 ? 4 : 8) * MSM_TREE_THREADS;  // two groups share the chip
            const size_t joins0 = (m + 1) / 2;
            if (fused) {
                e = g_msm_form == 4 ? launch_tree_fused<CI, 16>(m, tb, hs) : launch_tree_fused<CI, 8>(m, tb, hs);
            } else {
                if (split && joins0 >= 16 * fill) e = launch_tree<CI, 16, true>(curve, m, 0, tb, split, hs);
                else e = launch_tree<CI, 8, true>(curve, m, 0, tb, split, hs);
                static const int upper_knob = [] { const char* v = getenv("GECC_MSM_UPPER"); return v ? atoi(v) : 0; }();  // A/B timing
                const int first_fused = upper_knob >= 1 && upper_knob < MSM_TREE_LEVELS ? upper_knob : MSM_TREE_LEVELS;
                for (int l = 1; l < MSM_TREE_LEVELS && e == cudaSuccess; ++l) {
                    if (l == first_fused) {  // the remaining levels in one launch
                        e = launch_tree_upper<CI, 4>(m, l, tb, hs);
                        break;
                    }
                    const size_t joins = (m + ((size_t)2 << l) - 1) / ((size_t)2 << l);
                    if (split && joins >= 16 * fill) e = launch_tree<CI, 16, false>(curve, m, l, tb, split, hs);
                    else if (joins >= 8 * fill) e = launch_tree<CI, 8, false>(curve, m, l, tb, split, hs);
                    else if (joins >= 4 * fill) e = launch_tree<CI, 4, false>(curve, m, l, tb, split, hs);
                    else e = launch_tree<CI, MSM_TREE_KMIN, false>(curve, m, l, tb, split, hs);
                }
            }
            if (e != cudaSuccess) return e;
            const uint32_t nw = w1 - w0;
            k_msm_red_parts<CI><<<nw * 96, 128, 0, hs>>>(p.pairs, PairKeys{pairs2}, starts, slots, parts, w0);
            k_msm_red_fold<CI><<<nw * 24, 128, 0, hs>>>(parts, marg, w0);
            k_msm_red_weighted<CI><<<(nw * 3 + 3) / 4, 128, 0, hs>>>(marg, wsum, w0, w1);
            k_msm_red_shift<CI><<<1, (nw * 4 + 31) / 32 * 32, 0, hs>>>(wsum, win, w0, w1);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        if (G > 1) {
            if ((e = cudaEventRecord(aux.join, aux.stream)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(s, aux.join, 0)) != cudaSuccess) return e;
        }
        k_msm_red_final<CI, C><<<1, 32, 0, s>>>(win, ox, oy, oinf);
        const int per_level = fused ? 0 : (split ? 3 : 1) * (G > 1 || !aux.stream ? 1 : 2);
        *launches = 6 + G * ((fused ? 1 : per_level * MSM_TREE_LEVELS) + 4) + 1;  // sort (5) + records + groups x (tree + reduction) + final
        return cudaGetLastError();
    } else {
        uint32_t *edge = (uint32_t*)(base + p.off_edge), *edge_key = (uint32_t*)(base + p.off_edge_key);
        e = cudaMemsetAsync(buckets, 0, (size_t)12 * NL * MSM_NB, s);  // empty buckets = infinity (Z = 0)
        if (e != cudaSuccess) return e;
        const unsigned sb = (unsigned)((p.slices + 127) / 128);
        k_msm_buckets<C><<<sb, 128, 0, s>>>(n, p.pairs, PairKeys{pairs2}, PairVals{pairs2}, px, py, buckets, edge, edge_key, p.slices);
        k_msm_bucket_edges<C><<<sb, 128, 0, s>>>(buckets, edge, edge_key, p.slices);
        *launches = 5 + 2;
    }
    k_msm_marginal_parts<C><<<(MSM_WINDOWS * 3 * 1024 + 127) / 128, 128, 0, s>>>(buckets, parts);
    k_msm_marginal_fold<C><<<(MSM_WINDOWS * 3 * 32 + 127) / 128, 128, 0, s>>>(parts, marg);
    k_msm_weighted<C><<<1, 128, 0, s>>>(marg, wsum);
    k_msm_combine<C><<<1, 32, 0, s>>>(wsum, ox, oy, oinf);
    *launches += 4;  // reduction
    return cudaGetLastError();
}

cudaError_t launch_msm(int curve, size_t n, const uint32_t* scalars, const uint32_t* px,
                       const uint32_t* py, const uint8_t* pinf, uint32_t* ox, uint32_t* oy,
                       uint8_t* oinf, void* scratch, cudaStream_t s, int* launches, cudaEvent_t points_ready,
                       MsmAux aux) {
    if (curve == CURVE_BLS381)
        return run_msm<Bls381Curve>(curve, n, scalars, px, py, pinf, ox, oy, oinf, scratch, s, launches, points_ready, aux);
    if (curve == CURVE_BLS377)
        return run_msm<Bls377Curve>(curve, n, scalars, px, py, pinf, ox, oy, oinf, scratch, s, launches, points_ready, aux);
    if (curve == CURVE_SECP)
        return run_msm<SecpCurve, SecpLCurve>(curve, n, scalars, px, py, pinf, ox, oy, oinf, scratch, s, launches, points_ready, aux);
    return run_msm<Sm2Curve>(curve, n, scalars, px, py, pinf, ox, oy, oinf, scratch, s, launches, points_ready, aux);
}

}  // namespace gecc
