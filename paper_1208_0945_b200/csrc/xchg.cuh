// xchg.cuh -- device helpers of the order-independent exact all-reduce
// shared by the single-fit sweep (ccd_kernels.cu) and the batched engine
// (batch.cu): relaxed red.add / volatile poll words and the exact split of
// a non-negative double into three 41-bit limbs of a 2^-80 fixed-point
// number (and the reconstruction of their integer sums).  See DESIGN.md §4.2.
//
// Word layout: bits 0..51 carry the sum of the participants' limbs, bits
// 52..63 count arrivals.  A limb is < 2^41, so up to kMaxParticipants =
// 2^11 arrivals can never carry into the count (2^11 * (2^41 - 1) < 2^52),
// and the 12-bit count holds 2^11 arrivals per use of a buffer.
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
constexpr int kXCntShift = 52;
constexpr unsigned long long kXCnt = 1ull << kXCntShift;
constexpr unsigned long long kXData = kXCnt - 1;
constexpr int kLimbBits = 41;
constexpr unsigned long long kMLimb = (1ull << kLimbBits) - 1;
constexpr int kMaxParticipants = 1 << 11;
constexpr double kXMaxValue = 0x1p43; // partials must lie in [0, 2^43): 3 x 41 bits from 2^-80
static_assert(static_cast<unsigned long long>(kMaxParticipants) * kMLimb < kXCnt, "limb sums must not reach the count");
static_assert(kMaxParticipants < (1 << (64 - kXCntShift)), "the count field must hold kMaxParticipants arrivals");

// limb i (0..2) of v in [0, 2^43) at 2^-80 resolution: v = L2*2^2 + L1*2^-39
// + L0*2^-80 (bits below 2^-80 dropped: *inexact, limb 0 only); false if out
// of range
__device__ __forceinline__ bool limb_of(double v, int i, unsigned long long& out, bool* inexact = nullptr) {
    if (!(v >= 0.0 && v < kXMaxValue)) {
        out = 0;
        return false;
    }
    const double t2 = floor(__dmul_rn(v, 0x1p-2));
    if (i == 2) {
        out = static_cast<unsigned long long>(t2);
        return true;
    }
    const double r = __dsub_rn(v, __dmul_rn(t2, 4.0)); // exact, [0, 4)
    const double s1 = __dmul_rn(r, 0x1p39);
    const double t1 = floor(s1);
    if (i == 1) {
        out = static_cast<unsigned long long>(t1);
        return true;
    }
    const double s0 = __dmul_rn(__dsub_rn(s1, t1), 0x1p41); // exact
    const double t0 = floor(s0);
    if (inexact) *inexact = s0 != t0; // nonzero bits below 2^-80
    out = static_cast<unsigned long long>(t0);
    return true;
}

// Error-word layout (data bits): participants reporting an error in bits
// 0..11, participants whose first / second partial lost bits below 2^-80 in
// bits 12..23 / 24..35 (each count <= 2^11).
constexpr int kXInexA = 12, kXInexB = 24;
constexpr unsigned long long kXCountMask = 0xfffull;
// Refinement of small totals.  A partial below 2^-28 can carry bits below
// the 2^-80 resolution; the total then has fewer than 53 significant bits
// when it is below (inexact partials) * 2^-80 * 2^53.  Every participant sees
// the same totals and counts, so all of them decide alike to exchange the
// same partials again scaled by 2^s, with s chosen from an upper bound U of
// every partial (U = total + loss bound; partials are >= 0) so that the
// scaled partials stay below 2^42.  Each round gains >= 57 bits of
// resolution; at s = kXMaxScale the resolution is 2^-1074 (every double is
// representable) and the sum is exact.
constexpr int kXMaxScale = 994;
__device__ __forceinline__ bool needs_refine(double total, unsigned inexact, int s) {
    return inexact != 0 && s < kXMaxScale && total < ldexp(static_cast<double>(inexact), 53 - 80 - s);
}
__device__ __forceinline__ int next_scale(double total, unsigned inexact, int s) {
    const double U = total + ldexp(static_cast<double>(inexact), -80 - s);
    return min(kXMaxScale, max(s + 1, 41 - ilogb(U)));
}

__device__ __forceinline__ double pow2(int e) { // 2^e for normal exponents
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

// (L2*2^82 + L1*2^41 + L0) * 2^-80 for the limb sums L0..L2 (< 2^52 each,
// no carries needed): each limb sum converts to double exactly, and the
// value is (L2*2^2 + L1*2^-39) + L0*2^-80 in that order -- within one ulp
// of the exact sum, and a pure function of the integer sums, so every
// participant (and every partition of the data) gets the same bits.  Lanes
// can convert their own limb and combine with two shuffles (poll()).
__device__ __forceinline__ double limb_part(unsigned long long L, int i) { // i = limb index 0..2
    return __dmul_rn(__ull2double_rn(L), pow2(kLimbBits * i - 80));
}
__device__ __forceinline__ double limbs_combine(double p0, double p1, double p2) {
    return __dadd_rn(__dadd_rn(p2, p1), p0);
}
constexpr double kXMaxTotal = 0x1p48; // totals beyond are reported (DERR_SUM_RANGE)
__device__ __forceinline__ double from_limbs(unsigned long long L0, unsigned long long L1, unsigned long long L2,
                                             bool& ovf) {
    const double v = limbs_combine(limb_part(L0, 0), limb_part(L1, 1), limb_part(L2, 2));
    ovf = !(v < kXMaxTotal);
    return ovf ? 0.0 : v;
}

// l * exp(x'beta), the reference's l_exp_xbeta expression (engine.hpp:77-78,224-225)
#ifndef EXPFN
#define EXPFN exp // profiling variants may substitute a cheaper function
#endif
__device__ __forceinline__ double lexp(int len, double xb) { return __dmul_rn(static_cast<double>(len), EXPFN(xb)); }

} // namespace bsccs_b200
