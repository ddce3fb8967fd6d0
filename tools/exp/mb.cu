// Experiment harness (not part of the library): issue-rate of field products under different
// shapes -- chains per thread, warps per scheduler, inlined vs called -- on the lazy secp256k1 field.
#include <cstdio>
#include <vector>
#include "../../paper_2501_03245_b200/csrc/gecc_field.cuh"
using namespace gecc;

template <int MODE, int THREADS>
__global__ void __launch_bounds__(THREADS) k(int iters, uint32_t seed, uint64_t* cycles, uint32_t* sink) {
    const SecpPL f{};
    fe x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[c].w[k] = seed * (k + 3 + 11 * c) + threadIdx.x * (c + 1);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // 1 chain, inlined mul
            x[0] = fe_mul_inl(f, x[0], x[1]);
            x[1] = fe_mul_inl(f, x[1], x[0]);
        } else if (MODE == 1) {  // 2 chains, inlined mul
            x[0] = fe_mul_inl(f, x[0], x[1]);
            x[2] = fe_mul_inl(f, x[2], x[3]);
            x[1] = fe_mul_inl(f, x[1], x[0]);
            x[3] = fe_mul_inl(f, x[3], x[2]);
        } else if (MODE == 2) {  // 1 chain, inlined sqr
            x[0] = fe_sqr_inl(f, x[0]);
            x[0] = fe_sqr_inl(f, x[0]);
        } else if (MODE == 3) {  // 2 chains, inlined sqr
            x[0] = fe_sqr_inl(f, x[0]);
            x[1] = fe_sqr_inl(f, x[1]);
            x[0] = fe_sqr_inl(f, x[0]);
            x[1] = fe_sqr_inl(f, x[1]);
        } else if (MODE == 4) {  // 1 chain, called mul
            x[0] = fe_mul(f, x[0], x[1]);
            x[1] = fe_mul(f, x[1], x[0]);
        } else if (MODE == 5) {  // 1 chain, called sqr
            x[0] = fe_sqr(f, x[0]);
            x[0] = fe_sqr(f, x[0]);
        } else if (MODE == 6) {  // mixed: mul + sqr independent (2 chains)
            x[0] = fe_mul_inl(f, x[0], x[1]);
            x[2] = fe_sqr_inl(f, x[2]);
            x[1] = fe_mul_inl(f, x[1], x[0]);
            x[2] = fe_sqr_inl(f, x[2]);
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) s ^= x[c].w[k];
    if (s == 0x12345678u) sink[0] = s;
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (uint64_t)(t1 - t0);
}

template <int MODE, int THREADS>
void run(const char* name, double prods_per_iter, double wide_per_prod) {
    int sms = 148, iters = 2000;
    uint64_t* dc; uint32_t* ds;
    cudaMalloc(&dc, 8 * sms); cudaMalloc(&ds, 4);
    for (int p = 0; p < 2; ++p) k<MODE, THREADS><<<sms, THREADS>>>(iters, 17, dc, ds);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint64_t> c(sms);
    cudaMemcpy(c.data(), dc, 8 * sms, cudaMemcpyDeviceToHost);
    double sum = 0;
    for (int i = 0; i < sms; ++i) sum += prods_per_iter * iters * THREADS / (double)c[i];
    double per = sum / sms;
    printf("%-34s thr/SM %4d  %.4f prod/clk/SM  cycles/warp-prod/SMSP %.1f  IMAD.WIDE util %.3f  %s\n", name, THREADS, per,
           32.0 / per / 4.0, per * wide_per_prod / 32.0, cudaGetErrorString(e));
    cudaFree(dc); cudaFree(ds);
}

int main() {
    run<0, 256>("mul 1 chain inl", 2, 72);
    run<0, 512>("mul 1 chain inl", 2, 72);
    run<0, 1024>("mul 1 chain inl", 2, 72);
    run<1, 256>("mul 2 chains inl", 4, 72);
    run<1, 512>("mul 2 chains inl", 4, 72);
    run<2, 256>("sqr 1 chain inl", 2, 44);
    run<2, 512>("sqr 1 chain inl", 2, 44);
    run<2, 1024>("sqr 1 chain inl", 2, 44);
    run<3, 256>("sqr 2 chains inl", 4, 44);
    run<3, 512>("sqr 2 chains inl", 4, 44);
    run<4, 512>("mul 1 chain call", 2, 72);
    run<5, 512>("sqr 1 chain call", 2, 44);
    run<6, 512>("mul+sqr 2 chains inl", 4, 58);
    return 0;
}
