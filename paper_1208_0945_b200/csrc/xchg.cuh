// xchg.cuh -- device helpers of the order-independent exact all-reduce
// shared by the single-fit sweep (ccd_kernels.cu) and the batched engine
// (batch.cu): relaxed red.add / volatile poll words and the exact split of
// a non-negative double into three 42-bit limbs of a 2^-80 fixed-point
// number (and the correctly rounded reconstruction).  See DESIGN.md §4.2.
#pragma once

#include <cstdint>

namespace bsccs_b200 {

// Exchange words: relaxed at GPU scope (each word validates itself, so no
// fences are needed; peers on other GPUs would use .sys).
__device__ __forceinline__ void red_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// peer exchange areas (other GPUs, mapped through CUDA IPC over NVLink)
__device__ __forceinline__ void red_add_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_poll(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
constexpr unsigned long long kXCnt = 1ull << 50;
constexpr unsigned long long kXData = kXCnt - 1;
constexpr unsigned long long kM42 = (1ull << 42) - 1;

// limb i (0..2) of v in [0, 2^46) at 2^-80 resolution; false if out of range
__device__ __forceinline__ bool limb_of(double v, int i, unsigned long long& out) {
    if (!(v >= 0.0 && v < 0x1p46)) {
        out = 0;
        return false;
    }
    const double t2 = floor(__dmul_rn(v, 0x1p-4));
    if (i == 2) {
        out = static_cast<unsigned long long>(t2);
        return true;
    }
    const double r = __dsub_rn(v, __dmul_rn(t2, 16.0)); // exact, [0, 16)
    const double s1 = __dmul_rn(r, 0x1p38);
    const double t1 = floor(s1);
    if (i == 1) {
        out = static_cast<unsigned long long>(t1);
        return true;
    }
    out = static_cast<unsigned long long>(floor(__dmul_rn(__dsub_rn(s1, t1), 0x1p42))); // exact below 2^-80
    return true;
}

__device__ __forceinline__ double pow2(int e) { // 2^e for normal exponents
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

// correctly rounded double of (L2*2^84 + L1*2^42 + L0) * 2^-80
__device__ __forceinline__ double from_limbs(unsigned long long L0, unsigned long long L1, unsigned long long L2) {
    L1 += L0 >> 42;
    L0 &= kM42;
    L2 += L1 >> 42;
    L1 &= kM42;
    // 128-bit V = hi:lo
    const unsigned long long lo = L0 | (L1 << 42);
    const unsigned long long hi = (L1 >> 22) | (L2 << 20);
    if ((hi | lo) == 0) return 0.0;
    int lz;
    unsigned long long m, rest;
    if (hi) {
        lz = __clzll(static_cast<long long>(hi));
        m = lz ? (hi << lz) | (lo >> (64 - lz)) : hi;
        rest = lz ? lo << lz : lo;
    } else {
        lz = 64 + __clzll(static_cast<long long>(lo));
        m = lo << (lz - 64);
        rest = 0;
    }
    m |= rest != 0 ? 1ull : 0ull; // sticky bit for correct rounding
    return __dmul_rn(__ull2double_rn(m), pow2(64 - lz - 80));
}


// l * exp(x'beta), the reference's l_exp_xbeta expression (engine.hpp:77-78,224-225)
#ifndef EXPFN
#define EXPFN exp // profiling variants may substitute a cheaper function
#endif
__device__ __forceinline__ double lexp(int len, double xb) { return __dmul_rn(static_cast<double>(len), EXPFN(xb)); }

} // namespace bsccs_b200
