// The local side of the MSM exchange: every device / rank holds one partial sum,
// the partial sums are all-gathered (NCCL or peer copies, capi_multi.cu) and added here.  Elliptic
// curve addition is not a reduction operator NCCL knows, so the reduce is "gather + local adds".
// A point travels as 2L + 1 words: x[L] y[L] (Montgomery form) and the infinity flag.
#include "gecc_curve.cuh"
#include "gecc_dev.cuh"
#include "gecc_modinv.cuh"
#include "gecc_host.h"

namespace gecc {

template <class C>
__global__ void k_point_fold(int parts, const uint32_t* __restrict__ packed, uint32_t* __restrict__ out) {
    constexpr int L = C::Fp::N;
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const typename C::Fp f{};
    cjac<C> acc = jac_infinity<C>();
#pragma unroll 1
    for (int r = 0; r < parts; ++r) {
        const uint32_t* p = packed + (size_t)r * (2 * L + 1);
        if (p[2 * L]) continue;  // this rank's partial sum is the point at infinity
        caff<C> q;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            q.x.w[i] = p[i];
            q.y.w[i] = p[L + i];
        }
        acc = jac_madd<C>(acc, q);  // complete: equal points double, opposite points cancel
    }
    if (jac_is_inf<C>(acc)) {
        for (int i = 0; i < 2 * L; ++i) out[i] = 0;
        out[2 * L] = 1;
        return;
    }
    const caff<C> a = jac_to_aff_with<C>(acc, fe_inv_var(f, acc.Z));
#pragma unroll
    for (int i = 0; i < L; ++i) {
        out[i] = a.x.w[i];
        out[L + i] = a.y.w[i];
    }
    out[2 * L] = 0;
}

__global__ void k_point_pack(int L, const uint32_t* __restrict__ x, const uint32_t* __restrict__ y,
                             const uint8_t* __restrict__ inf, uint32_t* __restrict__ packed) {
    const int i = threadIdx.x;
    if (i < L) {
        packed[i] = x[i];
        packed[L + i] = y[i];
    }
    if (i == 0) packed[2 * L] = inf[0] ? 1u : 0u;
}
__global__ void k_point_unpack(int L, const uint32_t* __restrict__ packed, uint32_t* __restrict__ x,
                               uint32_t* __restrict__ y, uint8_t* __restrict__ inf) {
    const int i = threadIdx.x;
    if (i < L) {
        x[i] = packed[i];
        y[i] = packed[L + i];
    }
    if (i == 0) inf[0] = packed[2 * L] ? 1 : 0;
}

cudaError_t launch_point_fold(int curve, int parts, const uint32_t* packed, uint32_t* out, cudaStream_t s) {
    if (curve == CURVE_BLS381) k_point_fold<Bls381Curve><<<1, 32, 0, s>>>(parts, packed, out);
    else if (curve == CURVE_BLS377) k_point_fold<Bls377Curve><<<1, 32, 0, s>>>(parts, packed, out);
    else if (curve == CURVE_SECP) k_point_fold<SecpCurve><<<1, 32, 0, s>>>(parts, packed, out);
    else k_point_fold<Sm2Curve><<<1, 32, 0, s>>>(parts, packed, out);
    return cudaGetLastError();
}
cudaError_t launch_point_pack(int curve, const uint32_t* x, const uint32_t* y, const uint8_t* inf,
                              uint32_t* packed, cudaStream_t s) {
    k_point_pack<<<1, 32, 0, s>>>(curve_limbs(curve), x, y, inf, packed);
    return cudaGetLastError();
}
cudaError_t launch_point_unpack(int curve, const uint32_t* packed, uint32_t* x, uint32_t* y, uint8_t* inf,
                                cudaStream_t s) {
    k_point_unpack<<<1, 32, 0, s>>>(curve_limbs(curve), packed, x, y, inf);
    return cudaGetLastError();
}

}  // namespace gecc
