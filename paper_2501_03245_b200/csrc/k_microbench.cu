// Integer-pipe issue-rate microbenchmarks: the measured denominator of the IMAD
// roofline (SURVEY.md section 8d asks for it to be measured, not assumed).
// One 1024-thread block per SM (8 warps per scheduler); each block times its own
// span with clock64(), so the figure is independent of the SM clock.
#include <vector>

#include "gecc_dev.cuh"
#include "gecc_host.h"

namespace gecc {

template <int WHICH>
__global__ void __launch_bounds__(1024) k_rate(int iters, uint32_t seed, uint64_t* cycles,
                                               uint32_t* sink) {
    uint32_t a = seed + threadIdx.x, b = seed * 3 + blockIdx.x;
    uint64_t acc[8];
    uint32_t x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        acc[k] = a * (k + 1);
        x[k] = b + k;
    }
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int rep = 0; rep < 8; ++rep) {
            if (WHICH == 0) {  // 4 accumulator pairs: independent IMAD.WIDE.U32 with accumulate
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        // multiplier = a neighbour pair's high word: changes every step
                        uint32_t m = x[(2 * k + 3) & 7];
                        x[2 * k] = mad_lo_cc(a, m, x[2 * k]);
                        x[2 * k + 1] = madc_hi(a, m, x[2 * k + 1]);
                    }
            } else if (WHICH == 1) {  // one accumulator pair: dependent IMAD.WIDE.U32
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    uint32_t m = x[1];
                    x[0] = mad_lo_cc(a, m, x[0]);
                    x[1] = madc_hi(a, m, x[1]);
                }
            } else if (WHICH == 2) {  // IMAD (32-bit)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(a), "r"(b));
            } else if (WHICH == 3) {  // IMAD.HI
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(a), "r"(b));
            } else if (WHICH == 4) {  // 3-input adds
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    uint32_t t;
                    asm volatile("add.u32 %0, %1, %2;" : "=r"(t) : "r"(x[k]), "r"(a));
                    asm volatile("add.u32 %0, %1, %2;" : "=r"(x[k]) : "r"(t), "r"(b));
                }
            } else if (WHICH == 5) {  // one 8-limb carry chain
                x[0] = add_cc(x[0], a);
#pragma unroll
                for (int k = 1; k < 8; ++k) x[k] = addc_cc(x[k], b);
            } else if (WHICH == 6) {  // 4 IMAD.WIDE (2 pairs) + 4-limb carry chain, interleaved
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        uint32_t m = x[(2 * k + 3) & 3];
                        x[2 * k] = mad_lo_cc(a, m, x[2 * k]);
                        x[2 * k + 1] = madc_hi(a, m, x[2 * k + 1]);
                    }
                x[4] = add_cc(x[4], a);
#pragma unroll
                for (int k = 5; k < 8; ++k) x[k] = addc_cc(x[k], b);
            }
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= (uint32_t)acc[k] ^ (uint32_t)(acc[k] >> 32) ^ x[k];
    if (s == 0x12345678u) sink[0] = s;  // keep everything live
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (uint64_t)(t1 - t0);
}

template <class F, int WHICH>
__global__ void __launch_bounds__(1024) k_rate_fe(int iters, uint32_t seed, uint64_t* cycles,
                                                  uint32_t* sink) {
    const F f{};
    fe x, y;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x.w[k] = seed * (k + 3) + threadIdx.x;
        y.w[k] = seed * (k + 7) + blockIdx.x;
    }
    x.w[7] &= 0x7FFFFFFFu;
    y.w[7] &= 0x7FFFFFFFu;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        if (WHICH == 0) {         // inlined product + reduction
            x = fe_mul_inl(f, x, y);
            y = fe_mul_inl(f, y, x);
        } else if (WHICH == 1) {
            x = fe_add(f, x, y);
            y = fe_sub(f, y, x);
        } else if (WHICH == 2) {  // the by-value function the kernels call
            x = fe_mul(f, x, y);
            y = fe_mul(f, y, x);
        } else if (WHICH == 3) {
            x = fe_sqr_inl(f, x);
            y = fe_sqr_inl(f, y);
        } else {
            x = fe_sqr(f, x);
            y = fe_sqr(f, y);
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= x.w[k] ^ y.w[k];
    if (s == 0x12345678u) sink[0] = s;
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (uint64_t)(t1 - t0);
}

cudaError_t run_microbench(int which, int iters, int sm_count, double* ops_per_clk_per_sm,
                           double* seconds, double* total_ops, cudaStream_t s) {
    uint64_t* d_cycles = nullptr;
    uint32_t* d_sink = nullptr;
    cudaError_t e = cudaMalloc(&d_cycles, sizeof(uint64_t) * sm_count);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&d_sink, 4);
    if (e != cudaSuccess) { cudaFree(d_cycles); return e; }
    cudaEvent_t ev0, ev1;
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    double ops_per_thread_iter = 64.0;
    for (int pass = 0; pass < 2; ++pass) {  // pass 0 = warm-up
        cudaEventRecord(ev0, s);
        switch (which) {
            case 0: k_rate<0><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 1: k_rate<1><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 2: k_rate<2><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 3: k_rate<3><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 4: k_rate<4><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 5: k_rate<5><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 6: k_rate<6><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink); break;
            case 7: k_rate_fe<SecpP, 0><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink);
                ops_per_thread_iter = 2.0; break;
            case 8: k_rate_fe<SecpN, 0><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink);
                ops_per_thread_iter = 2.0; break;
            case 9: k_rate_fe<SecpP, 1><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink);
                ops_per_thread_iter = 2.0; break;
            case 10: k_rate_fe<SecpP, 2><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink);
                ops_per_thread_iter = 2.0; break;
            case 11: k_rate_fe<SecpP, 3><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink);
                ops_per_thread_iter = 2.0; break;
            case 12: k_rate_fe<SecpP, 4><<<sm_count, 1024, 0, s>>>(iters, 17, d_cycles, d_sink);
                ops_per_thread_iter = 2.0; break;
            default: cudaFree(d_cycles); cudaFree(d_sink); return cudaErrorInvalidValue;
        }
        cudaEventRecord(ev1, s);
        e = cudaEventSynchronize(ev1);
        if (e != cudaSuccess) break;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        std::vector<uint64_t> cyc(sm_count);
        cudaMemcpy(cyc.data(), d_cycles, sizeof(uint64_t) * sm_count, cudaMemcpyDeviceToHost);
        double per_block_ops = ops_per_thread_iter * iters * 1024.0, sum = 0;
        for (int i = 0; i < sm_count; ++i) sum += per_block_ops / (double)cyc[i];
        *ops_per_clk_per_sm = sum / sm_count;
        *seconds = ms * 1e-3;
        *total_ops = per_block_ops * sm_count;
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    cudaFree(d_cycles);
    cudaFree(d_sink);
    return e;
}

}  // namespace gecc
