// Fixed-base table for k*G: entry (j, d) = d * 2^(WG*j) * G, affine, Montgomery
// form, 16 words (x then y).  Replaces the reference's 256-entry doubling ladder
// (precompute_base_table, batch_point.cpp:341-350): with WG = 16 a scalar
// multiplication is 16-17 mixed additions and no doublings.  Built once per
// (device, curve) at context creation, entirely on the GPU.
#include "gecc_ecdsa.cuh"
#include "gecc_host.h"

namespace gecc {

// `base` == nullptr: the curve's generator; otherwise an affine point (x[8] y[8], the field's own
// representation) whose curve membership is checked here: precompute_base_table rejects off-curve
// input (batch_point.cpp:343-344), flags[0] reports it.
template <class C, int WG>
__global__ void k_gtable_bases(uint32_t* __restrict__ bases, const uint32_t* __restrict__ base,
                               uint32_t* __restrict__ flags) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= GTable<WG>::windows) return;
    const typename C::Fp f{};
    aff g = curve_g<C>();
    if (base) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            g.x.w[i] = base[i];
            g.y.w[i] = base[8 + i];
        }
        const bool ok = fe_lt_modulus(f, g.x) && fe_lt_modulus(f, g.y) && aff_on_curve<C>(g);
        if (!ok) {
            if (j == 0) atomicOr(flags, 1u);
            return;
        }
    }
    jac b;
    b.X = g.x; b.Y = g.y; b.Z = fe_one(f);
#pragma unroll 1
    for (int k = 0; k < WG * j; ++k) b = jac_dbl<C>(b);
    aff a = jac_to_aff_with<C>(b, fe_inv(f, b.Z));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        bases[j * 16 + i] = a.x.w[i];
        bases[j * 16 + 8 + i] = a.y.w[i];
    }
}

template <class C, int WG>
__global__ void __launch_bounds__(128) k_gtable_fill(const uint32_t* __restrict__ bases,
                                                      uint32_t* __restrict__ tab) {
    using GT = GTable<WG>;
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)GT::windows * GT::per_window) return;
    const int j = (int)(idx / GT::per_window);
    const uint32_t d = (uint32_t)(idx % GT::per_window) + 1;  // 1 .. 2^(WG-1)
    const typename C::Fp f{};
    aff b;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        b.x.w[i] = bases[j * 16 + i];
        b.y.w[i] = bases[j * 16 + 8 + i];
    }
    jac acc = jac_infinity<C>();
#pragma unroll 1
    for (int bit = WG - 1; bit >= 0; --bit) {
        acc = jac_dbl<C>(acc);
        if ((d >> bit) & 1u) acc = jac_madd<C>(acc, b);
    }
    aff a = jac_to_aff_with<C>(acc, fe_inv(f, acc.Z));
    uint4* out = reinterpret_cast<uint4*>(tab + idx * 16);
    out[0] = make_uint4(a.x.w[0], a.x.w[1], a.x.w[2], a.x.w[3]);
    out[1] = make_uint4(a.x.w[4], a.x.w[5], a.x.w[6], a.x.w[7]);
    out[2] = make_uint4(a.y.w[0], a.y.w[1], a.y.w[2], a.y.w[3]);
    out[3] = make_uint4(a.y.w[4], a.y.w[5], a.y.w[6], a.y.w[7]);
}

size_t gtable_words() { return (size_t)GTable<GECC_WG>::windows * GTable<GECC_WG>::per_window * 16; }

cudaError_t build_gtable(int curve, bool lazy_plain, uint32_t* tab, uint32_t* bases_scratch,
                         cudaStream_t s) {
    using GT = GTable<GECC_WG>;
    const size_t entries = (size_t)GT::windows * GT::per_window;
    const int blocks = (int)((entries + 127) / 128);
    if (curve == CURVE_SECP && lazy_plain) {  // table of the fused ECDSA kernels (plain coordinates)
        k_gtable_bases<SecpLCurve, GECC_WG><<<1, 32, 0, s>>>(bases_scratch, nullptr, nullptr);
        k_gtable_fill<SecpLCurve, GECC_WG><<<blocks, 128, 0, s>>>(bases_scratch, tab);
    } else if (curve == CURVE_SECP) {
        k_gtable_bases<SecpCurve, GECC_WG><<<1, 32, 0, s>>>(bases_scratch, nullptr, nullptr);
        k_gtable_fill<SecpCurve, GECC_WG><<<blocks, 128, 0, s>>>(bases_scratch, tab);
    } else {
        k_gtable_bases<Sm2Curve, GECC_WG><<<1, 32, 0, s>>>(bases_scratch, nullptr, nullptr);
        k_gtable_fill<Sm2Curve, GECC_WG><<<blocks, 128, 0, s>>>(bases_scratch, tab);
    }
    return cudaGetLastError();
}

// precompute_base_table(c, g) for any on-curve g (batch_point.cpp:341-350): the same windowed
// table as the generator's, Montgomery-form coordinates (it feeds the column-buffer kernel k_fpmul).
cudaError_t build_base_table(int curve, const uint32_t* xy_dev, uint32_t* tab, uint32_t* bases_scratch,
                             uint32_t* flags, cudaStream_t s) {
    using GT = GTable<GECC_WG>;
    const size_t entries = (size_t)GT::windows * GT::per_window;
    const int blocks = (int)((entries + 127) / 128);
    if (curve == CURVE_SECP) {
        k_gtable_bases<SecpCurve, GECC_WG><<<1, 32, 0, s>>>(bases_scratch, xy_dev, flags);
        k_gtable_fill<SecpCurve, GECC_WG><<<blocks, 128, 0, s>>>(bases_scratch, tab);
    } else {
        k_gtable_bases<Sm2Curve, GECC_WG><<<1, 32, 0, s>>>(bases_scratch, xy_dev, flags);
        k_gtable_fill<Sm2Curve, GECC_WG><<<blocks, 128, 0, s>>>(bases_scratch, tab);
    }
    return cudaGetLastError();
}

}  // namespace gecc
