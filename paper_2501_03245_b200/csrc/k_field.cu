// Element-wise field kernels over column buffers: the GPU form of the reference's
// field layer (field.cpp:194-246) used for parity tests of the limb arithmetic.
#include "gecc_dev.cuh"
#include "gecc_modinv.cuh"
#include "gecc_host.h"

namespace gecc {

template <class F>
__global__ void __launch_bounds__(256) k_field_op(int op, size_t n, const uint32_t* __restrict__ a,
                                                  const uint32_t* __restrict__ b,
                                                  uint32_t* __restrict__ out) {
    const F f{};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        constexpr int N = F::N;
        feN<N> x = col_load<N>(a, n, i);
        feN<N> y = b ? col_load<N>(b, n, i) : fe_zero_n<N>();
        feN<N> r;
        switch (op) {
            case 0: r = fe_mul(f, x, y); break;
            case 1: r = fe_add(f, x, y); break;
            case 2: r = fe_sub(f, x, y); break;
            case 3: r = fe_to_mont(f, x); break;
            case 4: r = fe_from_mont(f, x); break;
            case 5: r = fe_inv(f, x); break;  // safegcd; zero -> zero
            case 6: r = fe_is_zero(x) ? x : fe_inv_fermat(f, x); break;  // Fermat cross-check
            case 7: {  // mont_reduce of the 2N-limb value y:x through the field's own reduction route
                uint32_t t[2 * N];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    t[k] = x.w[k];
                    t[N + k] = y.w[k];
                }
                r = redc(f, t);
                break;
            }
            default: {  // 8..11: the weakly reduced plain field of the fused secp256k1 kernels
                r = x;
                if constexpr (std::is_same<F, SecpP>::value) {
                    const SecpPL l{};
                    if (op == 8) r = fe_mul(l, x, y);
                    else if (op == 9) r = fe_sqr(l, x);
                    else if (op == 10) r = fe_add(l, x, y);
                    else r = fe_sub(l, x, y);
                    r = lazy_canon(l, r);
                }
                break;
            }
        }
        col_store(out, n, i, r);
    }
}

// op 12: every element inverted by a whole warp (the inversion of coop_block_inverse).  Lane e's
// element is broadcast, inverted by all 32 lanes together, and kept by lane e.
template <class F>
__global__ void __launch_bounds__(128) k_field_inv_warp(size_t n, const uint32_t* __restrict__ a,
                                                        uint32_t* __restrict__ out) {
    const F f{};
    constexpr int N = F::N;
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;  // whole warps stay in the loop
    const int lane = threadIdx.x & 31;
    feN<N> x = i < n ? col_load<N>(a, n, i) : fe_zero_n<N>();
    feN<N> r = x;
#pragma unroll 1
    for (int e = 0; e < 32; ++e) {
        feN<N> xe;
#pragma unroll
        for (int k = 0; k < N; ++k) xe.w[k] = __shfl_sync(0xFFFFFFFFu, x.w[k], e);
        const feN<N> re = fe_inv_warp(f, xe);
        if (lane == e) r = re;
    }
    if (i < n) col_store(out, n, i, r);
}

cudaError_t launch_field_op(int curve, int field, int op, size_t n, const uint32_t* a,
                            const uint32_t* b, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (op == 12) {
        const unsigned wb = (unsigned)((n + 127) / 128);
        if (curve == CURVE_BLS381) {
            if (field == 0) k_field_inv_warp<Bls381P><<<wb, 128, 0, s>>>(n, a, out);
            else k_field_inv_warp<Bls381R><<<wb, 128, 0, s>>>(n, a, out);
        } else if (curve == CURVE_BLS377) {
            if (field == 0) k_field_inv_warp<Bls377P><<<wb, 128, 0, s>>>(n, a, out);
            else k_field_inv_warp<Bls377R><<<wb, 128, 0, s>>>(n, a, out);
        } else if (curve == CURVE_SECP) {
            if (field == 0) k_field_inv_warp<SecpP><<<wb, 128, 0, s>>>(n, a, out);
            else k_field_inv_warp<SecpN><<<wb, 128, 0, s>>>(n, a, out);
        } else {
            if (field == 0) k_field_inv_warp<Sm2P><<<wb, 128, 0, s>>>(n, a, out);
            else k_field_inv_warp<Sm2N><<<wb, 128, 0, s>>>(n, a, out);
        }
        return cudaGetLastError();
    }
    const int threads = 256;
    size_t want = (n + threads - 1) / threads;
    const int blocks = (int)(want < 148 * 16 ? want : 148 * 16);
    if (curve == CURVE_BLS381) {  // base field: 12 limbs per element, scalar field: 8
        if (field == 0) k_field_op<Bls381P><<<blocks, threads, 0, s>>>(op, n, a, b, out);
        else k_field_op<Bls381R><<<blocks, threads, 0, s>>>(op, n, a, b, out);
    } else if (curve == CURVE_BLS377) {
        if (field == 0) k_field_op<Bls377P><<<blocks, threads, 0, s>>>(op, n, a, b, out);
        else k_field_op<Bls377R><<<blocks, threads, 0, s>>>(op, n, a, b, out);
    } else if (curve == CURVE_SECP) {
        if (field == 0) k_field_op<SecpP><<<blocks, threads, 0, s>>>(op, n, a, b, out);
        else k_field_op<SecpN><<<blocks, threads, 0, s>>>(op, n, a, b, out);
    } else {
        if (field == 0) k_field_op<Sm2P><<<blocks, threads, 0, s>>>(op, n, a, b, out);
        else k_field_op<Sm2N><<<blocks, threads, 0, s>>>(op, n, a, b, out);
    }
    return cudaGetLastError();
}

}  // namespace gecc
