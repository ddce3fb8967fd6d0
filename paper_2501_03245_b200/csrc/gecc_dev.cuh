// Device-side access helpers shared by the kernels: column-major (SoA) limb
// buffers (batch_buffer.hpp:15-35) and the big-endian wire records
// (limbs.cpp:5-27, sm2batch.h:4-9).
#pragma once
#include "gecc_field.cuh"

namespace gecc {

// limb k of element i at cols[k*n + i]: a warp reads 32 consecutive words per limb.
template <int N = 8>
GECC_HD feN<N> col_load(const uint32_t* __restrict__ cols, size_t n, size_t i) {
    feN<N> v;
#pragma unroll
    for (int k = 0; k < N; ++k) v.w[k] = cols[(size_t)k * n + i];
    return v;
}
template <int N>
GECC_HD void col_store(uint32_t* __restrict__ cols, size_t n, size_t i, const feN<N>& v) {
#pragma unroll
    for (int k = 0; k < N; ++k) cols[(size_t)k * n + i] = v.w[k];
}

// 32 big-endian bytes -> limbs (limbs.cpp:5-14).  p need not be aligned.
GECC_HD fe be32_load(const uint8_t* p) {
    fe v;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint8_t* s = p + 4 * (7 - i);
        v.w[i] = ((uint32_t)s[0] << 24) | ((uint32_t)s[1] << 16) | ((uint32_t)s[2] << 8) | s[3];
    }
    return v;
}
GECC_HD void be32_store(uint8_t* p, const fe& v) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint8_t* d = p + 4 * (7 - i);
        d[0] = (uint8_t)(v.w[i] >> 24);
        d[1] = (uint8_t)(v.w[i] >> 16);
        d[2] = (uint8_t)(v.w[i] >> 8);
        d[3] = (uint8_t)v.w[i];
    }
}

// The same codec for records that sit on a 16-byte boundary (every record of a 32- or 64-byte
// stride array whose base is 16-byte aligned): two 16-byte vector accesses and eight byte
// permutes instead of 32 single-byte accesses -- the byte loads were what throttled the
// load/store unit of the signing kernel (profiles/r01j_sign_metrics.csv: lg_throttle).
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ fe be32_load_v4(const uint8_t* p) {
    const uint4 a = *reinterpret_cast<const uint4*>(p), b = *reinterpret_cast<const uint4*>(p + 16);
    fe v;
    v.w[7] = __byte_perm(a.x, 0, 0x0123); v.w[6] = __byte_perm(a.y, 0, 0x0123);
    v.w[5] = __byte_perm(a.z, 0, 0x0123); v.w[4] = __byte_perm(a.w, 0, 0x0123);
    v.w[3] = __byte_perm(b.x, 0, 0x0123); v.w[2] = __byte_perm(b.y, 0, 0x0123);
    v.w[1] = __byte_perm(b.z, 0, 0x0123); v.w[0] = __byte_perm(b.w, 0, 0x0123);
    return v;
}
__device__ __forceinline__ void be32_store_v4(uint8_t* p, const fe& v) {
    *reinterpret_cast<uint4*>(p) = make_uint4(__byte_perm(v.w[7], 0, 0x0123), __byte_perm(v.w[6], 0, 0x0123),
                                              __byte_perm(v.w[5], 0, 0x0123), __byte_perm(v.w[4], 0, 0x0123));
    *reinterpret_cast<uint4*>(p + 16) = make_uint4(__byte_perm(v.w[3], 0, 0x0123), __byte_perm(v.w[2], 0, 0x0123),
                                                   __byte_perm(v.w[1], 0, 0x0123), __byte_perm(v.w[0], 0, 0x0123));
}
#endif
// aligned: the caller has checked that p is 16-byte aligned (uniform over the launch)
GECC_HD fe be32_load_a(const uint8_t* p, bool aligned) {
#if defined(__CUDA_ARCH__)
    if (aligned) return be32_load_v4(p);
#endif
    (void)aligned;
    return be32_load(p);
}
GECC_HD void be32_store_a(uint8_t* p, const fe& v, bool aligned) {
#if defined(__CUDA_ARCH__)
    if (aligned) {
        be32_store_v4(p, v);
        return;
    }
#endif
    (void)aligned;
    be32_store(p, v);
}
GECC_HD bool ptr_aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace gecc
