// 32-bit carry-chain primitives.
//
// Device build (sm_100a): one PTX instruction each (add.cc / addc / mad.lo.cc /
// madc.hi.cc ...).  ptxas turns the carry flag into explicit predicate operands
// (IADD3.X, IMAD.WIDE.U32.X), so independent chains interleave freely in SASS.
// Every wrapper is `asm volatile` so nvcc keeps the program order of chains.
//
// Host build (tests/hostsim only, never part of libgecc_b200.so's data path):
// the same wrappers emulate the flag with a thread-local, so the *identical*
// limb code can be run on the CPU of the authoring container, which has no GPU.
#pragma once
#include <stdint.h>
#if !defined(__CUDA_ARCH__)
#include <stdio.h>
#include <stdlib.h>
#endif

#if defined(__CUDACC__)
#define GECC_HD __host__ __device__ __forceinline__
#define GECC_D __device__ __forceinline__
// Point-level operations (7-16 field multiplications each) are real functions on
// the device: one copy per kernel instead of one per call site keeps a fused ECDSA
// kernel at a few thousand instructions (compile time, instruction cache).
#define GECC_HD_CALL __host__ __device__ __noinline__
#else
#define GECC_HD inline
#define GECC_D inline
#define GECC_HD_CALL inline
#endif

namespace gecc {

#if defined(__CUDA_ARCH__)

GECC_D uint32_t add_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
GECC_D uint32_t addc_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
GECC_D uint32_t addc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("addc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
GECC_D uint32_t sub_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
GECC_D uint32_t subc_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
GECC_D uint32_t subc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("subc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
GECC_D uint32_t mul_lo(uint32_t a, uint32_t b) { return a * b; }
GECC_D uint32_t mul_hi(uint32_t a, uint32_t b) { return __umulhi(a, b); }
// r = lo(a*b) + c, CF = carry
GECC_D uint32_t mad_lo_cc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("mad.lo.cc.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
GECC_D uint32_t mad_hi_cc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("mad.hi.cc.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
GECC_D uint32_t madc_lo_cc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("madc.lo.cc.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
GECC_D uint32_t madc_hi_cc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("madc.hi.cc.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
GECC_D uint32_t madc_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("madc.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
GECC_D uint32_t madc_hi(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("madc.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

#else  // host emulation ------------------------------------------------------

// The emulation also polices a hardware fact the PTX text hides: after sub.cc the
// machine flag is the INVERTED borrow, so a flag produced by the sub family must
// only be consumed by the sub family (and add by add).  Mixing aborts here, so the
// mistake is caught on the CPU instead of as wrong limbs on the GPU.
inline uint32_t& cf_() {
    static thread_local uint32_t cf = 0;
    return cf;
}
inline int& fam_() {  // 0 none, 1 add family, 2 sub family
    static thread_local int fam = 0;
    return fam;
}
inline void need_(int fam) {
    if (fam_() != fam) {
        fprintf(stderr, "gecc_prims: carry flag of family %d consumed by family %d\n", fam_(), fam);
        abort();
    }
}
inline uint32_t add3_(uint32_t a, uint32_t b, bool use, bool set) {
    if (use) need_(1);
    uint64_t t = (uint64_t)a + b + (use ? cf_() : 0);
    if (set) { cf_() = (uint32_t)(t >> 32); fam_() = 1; }
    return (uint32_t)t;
}
inline uint32_t sub3_(uint32_t a, uint32_t b, bool use, bool set) {
    if (use) need_(2);
    uint64_t t = (uint64_t)a - b - (use ? cf_() : 0);
    if (set) { cf_() = (uint32_t)((t >> 32) & 1); fam_() = 2; }
    return (uint32_t)t;
}
inline uint32_t add_cc(uint32_t a, uint32_t b) { return add3_(a, b, false, true); }
inline uint32_t addc_cc(uint32_t a, uint32_t b) { return add3_(a, b, true, true); }
inline uint32_t addc(uint32_t a, uint32_t b) { return add3_(a, b, true, false); }
inline uint32_t sub_cc(uint32_t a, uint32_t b) { return sub3_(a, b, false, true); }
inline uint32_t subc_cc(uint32_t a, uint32_t b) { return sub3_(a, b, true, true); }
inline uint32_t subc(uint32_t a, uint32_t b) { return sub3_(a, b, true, false); }
inline uint32_t mul_lo(uint32_t a, uint32_t b) { return a * b; }
inline uint32_t mul_hi(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
inline uint32_t mad_lo_cc(uint32_t a, uint32_t b, uint32_t c) { return add3_(a * b, c, false, true); }
inline uint32_t mad_hi_cc(uint32_t a, uint32_t b, uint32_t c) { return add3_(mul_hi(a, b), c, false, true); }
inline uint32_t madc_lo_cc(uint32_t a, uint32_t b, uint32_t c) { return add3_(a * b, c, true, true); }
inline uint32_t madc_hi_cc(uint32_t a, uint32_t b, uint32_t c) { return add3_(mul_hi(a, b), c, true, true); }
inline uint32_t madc_lo(uint32_t a, uint32_t b, uint32_t c) { return add3_(a * b, c, true, false); }
inline uint32_t madc_hi(uint32_t a, uint32_t b, uint32_t c) { return add3_(mul_hi(a, b), c, true, false); }

#endif

}  // namespace gecc
