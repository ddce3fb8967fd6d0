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

}  // namespace gecc
