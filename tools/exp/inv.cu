// Experiment: latency of ONE modular inversion executed by one warp (what bounds small batch_padd).
#include <cstdio>
#include "../../paper_2501_03245_b200/csrc/gecc_modinv.cuh"
using namespace gecc;

#ifndef UNIFORM
#define UNIFORM 1
#endif
template <class F, int MODE>
__global__ void k(uint32_t seed, uint64_t* cycles, uint32_t* out) {
    const F f{};
    fel<F> x;
    for (int k = 0; k < F::N; ++k) x.w[k] = seed * (k + 3) * 2654435761u + (UNIFORM ? 0 : threadIdx.x * 7) + 1;
    x.w[F::N - 1] &= 0x00FFFFFFu;
    fel<F> r;
    long long t0 = clock64();
    if (MODE == 0) r = safegcd_inverse(f, x);
    else if (MODE == 4) r = safegcd_inverse_var(f, x);
    else if (MODE == 5) r = safegcd_inverse_sched<false>(f, x);
    else if (MODE == 6) r = safegcd_inverse_sched<true>(f, x);
    else if (MODE == 7) r = safegcd_inverse_warp<false>(f, x);
    else if (MODE == 8) r = safegcd_inverse_warp<true>(f, x);
    else if (MODE == 1) r = fe_inv_fermat(f, x);
    else if (MODE == 2) r = fe_mul(f, x, x);
    else {
        r = x;
#pragma unroll 1
        for (int i = 0; i < 100; ++i) r = fe_sqr(f, r);
    }
    long long t1 = clock64();
    for (int k = 0; k < 8; ++k) out[threadIdx.x * 8 + k] = r.w[k];
    if (MODE >= 4) {  // cross-check against the plain rounds
        fel<F> w = safegcd_inverse(f, x);
        for (int k = 0; k < F::N; ++k) if (w.w[k] != r.w[k]) out[0] = 0xDEADBEEF, cycles[1] = 1;
    }
    if (threadIdx.x == 0) cycles[0] = (uint64_t)(t1 - t0);
}

template <class F, int MODE>
void run(const char* name, int threads) {
    uint64_t* dc; uint32_t* d;
    cudaMalloc(&dc, 16); cudaMemset(dc, 0, 16); cudaMalloc(&d, 32 * 1024);
    uint64_t c = 0, bad = 0;
    for (int p = 0; p < 3; ++p) {
        k<F, MODE><<<1, threads>>>(17 + p, dc, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&bad, dc + 1, 8, cudaMemcpyDeviceToHost);
    }
    if (bad) printf("   MISMATCH vs plain safegcd\n");
    printf("%-28s threads %3d: %8llu cycles  %.2f us @1.965GHz  %s\n", name, threads, (unsigned long long)c, c / 1965.0,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(dc); cudaFree(d);
}

int main() {
    run<SecpP, 0>("safegcd SecpP", 32);
    run<SecpP, 4>("safegcd var SecpP", 32);
    run<SecpPL, 4>("safegcd var lazy", 32);
    run<SecpP, 7>("safegcd warp-coop SecpP", 32);
    run<SecpP, 8>("safegcd warp-coop var SecpP", 32);
    run<Bls381P, 8>("safegcd warp-coop var BLS381", 32);
    run<SecpPL, 7>("safegcd warp-coop lazy", 32);
    run<Bls381P, 7>("safegcd warp-coop BLS381", 32);
    run<SecpP, 5>("safegcd sched SecpP", 32);
    run<SecpP, 6>("safegcd sched+exit SecpP", 32);
    run<Bls381P, 5>("safegcd sched BLS381", 32);
    run<Bls381P, 6>("safegcd sched+exit BLS381", 32);
    run<Bls381P, 0>("safegcd BLS381", 32);
    run<Bls381P, 4>("safegcd var BLS381", 32);
    run<SecpP, 0>("safegcd SecpP", 1);
    run<SecpN, 0>("safegcd SecpN", 32);
    run<SecpP, 1>("fermat SecpP", 32);
    run<SecpP, 2>("one fe_mul SecpP", 32);
    run<SecpP, 3>("100 dependent fe_sqr SecpP", 32);
    run<SecpPL, 3>("100 dependent fe_sqr lazy", 32);
    return 0;
}
