// Experiment: where the time of the single-launch batch_padd (2^16 pairs, 128 threads, K pairs
// per thread) goes.  The kernel body is k_batch_padd_coop's generic-pair path with globaltimer
// stamps taken by thread 0 of every block; the host prints the median phase boundaries relative
// to the earliest block start.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o _build/padd_timeline padd_timeline.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../../paper_2501_03245_b200/csrc/gecc_batch.cuh"
using namespace gecc;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int NSTAMP = 8;

template <class C, int THREADS, int K>
__global__ void __launch_bounds__(THREADS, THREADS == 128 ? 4 : 1)
k_padd(size_t n, const uint32_t* __restrict__ px, const uint32_t* __restrict__ py, const uint32_t* __restrict__ tx,
       const uint32_t* __restrict__ ty, uint32_t* __restrict__ ox, uint32_t* __restrict__ oy,
       unsigned long long* __restrict__ stamps) {
    using fe = cfe<C>;
    constexpr int NL = C::Fp::N;
    constexpr int NW = THREADS / 32;
    __shared__ uint32_t sm[2 * NL * NW];
    const typename C::Fp f{};
    unsigned long long* st = stamps + (size_t)blockIdx.x * NSTAMP;
    const bool rec = threadIdx.x == 0;
    if (rec) st[0] = gtime();
    const size_t tile = (size_t)blockIdx.x * (THREADS * K) + threadIdx.x;
    fe lp[K];
    fe acc = fe_one(f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const size_t i = tile + (size_t)k * THREADS;
        if (i < n) {
            fe ax = col_load<NL>(px, n, i), bx = col_load<NL>(tx, n, i);
            fe d = fe_sub(f, ax, bx);
            acc = fe_mul(f, acc, d);
        }
        lp[k] = acc;
    }
    if (rec) st[1] = gtime();  // loads + local products
    // ---- coop_block_inverse, opened up
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const fe one = fe_one(f);
    fe P, Q;
    warp_scan_products(f, acc, lane, 32, &P, &Q);
    fe E = fe_select(lane == 0, one, fe_shfl_up(P, 1));
    fe S = fe_select(lane == 31, one, fe_shfl_down(Q, 1));
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < NL; ++i) sm[i * NW + warp] = P.w[i];
    }
    if (rec) st[2] = gtime();  // warp scans
    __syncthreads();
    if (warp == (int)(blockIdx.x % NW)) {
        fe w = one;
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < NL; ++i) w.w[i] = sm[i * NW + lane];
        }
        fe PP, QQ;
        warp_scan_products(f, w, lane, NW, &PP, &QQ);
        fe total;
#pragma unroll
        for (int i = 0; i < NL; ++i) total.w[i] = __shfl_sync(0xFFFFFFFFu, PP.w[i], NW - 1);
        if (lane == 0) st[5] = gtime();  // inverting warp: before the inversion
        const fe inv = fe_inv_warp(f, total);
        if (lane == 0) st[6] = gtime();  // inverting warp: after the inversion
        fe EE = fe_select(lane == 0, one, fe_shfl_up(PP, 1));
        fe SS = fe_select(lane == 31, one, fe_shfl_down(QQ, 1));
        fe wi = fe_mul(f, fe_mul(f, inv, EE), SS);
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < NL; ++i) sm[(NL + i) * NW + lane] = wi.w[i];
        }
    }
    __syncthreads();
    fe wi;
#pragma unroll
    for (int i = 0; i < NL; ++i) wi.w[i] = sm[(NL + i) * NW + warp];
    fe inv = fe_mul(f, fe_mul(f, wi, E), S);
    if (rec) st[3] = gtime();  // inverse of the thread total in hand
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
        const size_t i = tile + (size_t)k * THREADS;
        if (i < n) {
            fe ax = col_load<NL>(px, n, i), ay = col_load<NL>(py, n, i);
            fe bx = col_load<NL>(tx, n, i), by = col_load<NL>(ty, n, i);
            fe d = fe_sub(f, ax, bx);
            fe dinv = k > 0 ? fe_mul(f, inv, lp[k > 0 ? k - 1 : 0]) : inv;
            if (k > 0) inv = fe_mul(f, inv, d);
            fe xr, yr;
            fe lam = fe_mul(f, fe_sub(f, ay, by), dinv);
            finish_lambda<C>(lam, ax, bx, ay, &xr, &yr);
            col_store(ox, n, i, xr);
            col_store(oy, n, i, yr);
        }
    }
    if (rec) st[4] = gtime();  // unwound, stored
}

template <int THREADS, int K>
void run(size_t n) {
    const size_t words = n * 8;
    uint32_t *px, *py, *tx, *ty, *ox, *oy;
    std::vector<uint32_t> h(words);
    uint32_t** bufs[] = {&px, &py, &tx, &ty, &ox, &oy};
    uint32_t seed = 12345;
    for (auto b : bufs) {
        cudaMalloc(b, words * 4);
        for (auto& v : h) { seed = seed * 1664525u + 1013904223u; v = seed; }
        for (size_t i = 0; i < n; ++i) h[7 * n + i] &= 0x7FFFFFFFu;
        cudaMemcpy(*b, h.data(), words * 4, cudaMemcpyHostToDevice);
    }
    const unsigned blocks = (unsigned)((n + THREADS * K - 1) / (THREADS * K));
    unsigned long long* ds;
    cudaMalloc(&ds, (size_t)blocks * NSTAMP * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(ds, 0, (size_t)blocks * NSTAMP * 8);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k_padd<SecpMLCurve, THREADS, K><<<blocks, THREADS>>>(n, px, py, tx, ty, ox, oy, ds);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms, e0, e1);
    }
    std::vector<unsigned long long> s((size_t)blocks * NSTAMP);
    cudaMemcpy(s.data(), ds, s.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tend = 0;
    for (unsigned b = 0; b < blocks; ++b) { t0 = std::min(t0, s[b * NSTAMP]); tend = std::max(tend, s[b * NSTAMP + 4]); }
    printf("n=2^%d threads %d K %d blocks %u: event %.1f us, first start -> last end %.1f us  (%s)\n", (int)__builtin_ctzll(n), THREADS,
           K, blocks, ms * 1e3, (tend - t0) / 1e3, cudaGetErrorString(cudaGetLastError()));
    const char* names[NSTAMP] = {"start", "local products", "warp scans", "thread inverse", "end", "inv begin", "inv end", ""};
    const int order[] = {0, 1, 2, 5, 6, 3, 4};
    for (int j : order) {
        std::vector<double> v;
        for (unsigned b = 0; b < blocks; ++b) v.push_back((s[b * NSTAMP + j] - t0) / 1e3);
        std::sort(v.begin(), v.end());
        printf("   %-16s min %6.2f  median %6.2f  max %6.2f us\n", names[j], v.front(), v[v.size() / 2], v.back());
    }
    for (auto b : bufs) cudaFree(*b);
    cudaFree(ds);
}

int main() {
    run<128, 2>((size_t)1 << 16);
    run<128, 1>((size_t)1 << 16);
    run<128, 4>((size_t)1 << 16);
    run<128, 1>((size_t)1 << 14);
    run<128, 1>((size_t)1 << 12);
    run<32, 4>((size_t)1 << 16);
    run<32, 2>((size_t)1 << 16);
    run<64, 2>((size_t)1 << 16);
    return 0;
}
