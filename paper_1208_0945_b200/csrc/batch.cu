// batch.cu -- batched weighted multi-fit CCD engine.
//
// The many-fit callers of fit() -- the prior-variance CV grid
// (cross_validation.hpp:146-173) and the bootstrap replicates
// (bootstrap.hpp:103-114) -- refit the model on subject selections of one
// parent dataset.  A selection in which subject i appears m_i times is the
// parent dataset with every per-subject term weighted by m_i: the copies of a
// subject share x'beta, the denominator and w, so
//   gradient sum   sum_runs m_i n_i w_i,   hessian sum  sum_runs m_i n_i w_i (1 - w_i)
//   y_dot_x        sum_pairs m_i y_k,      criterion    sum_eras m_i |x'b - snap|
//   log likelihood sum_eras m_i y_k x'b_k - sum_i m_i n_i log den_i
// which equal the materialised subset's (subset_dataset, dataset.hpp:157-217)
// up to summation order.  The skip rule (solver.hpp:119-121) uses the
// weighted column count.  Held-out folds use the complementary weights.
//
// R <= RB fits run in one persistent cooperative launch per cycle over the
// parent's CSC: pairs stream once per coordinate for all fits, and one exact
// all-reduce carries every fit's (gradient, hessian) partials.  Per-fit state
// is fit-minor ([era][RB], [subject][RB]), so a scattered era touches one
// contiguous RB*8-byte run instead of RB separate sectors.  Every fit takes
// its own step (lane r of warp 0), trust radius, convergence and errors; a
// converged or failed fit is masked out of later cycles.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "devutil.h"
#include "engine.h"
#include "prior.h"
#include "rng.h"
#include "xchg.cuh"

#ifndef BSCCS_DIAG_NOLOAD
#define BSCCS_DIAG_NOLOAD 0
#endif
#ifndef BSCCS_DIAG_NOCOMPUTE
#define BSCCS_DIAG_NOCOMPUTE 0
#endif

namespace bsccs_b200 {

namespace {

constexpr int kBT = 512;              // threads per CTA
constexpr int kBWarps = kBT / 32;
constexpr int kBXStride = 32;         // u64 between exchange words (256 B)
constexpr int kBMaxRB = 16;
constexpr int kBSmemBudget = 200 * 1024;
constexpr double kBXbBound = 700.0;   // xbeta_bound<double> engine.hpp:20-23

template <int RB>
struct BCfg {
    static constexpr int kErrWords = (RB + 5) / 6;       // 8-bit error counters, 6 fits per word
    static constexpr int kNW = 6 * RB + kErrWords;       // exchange words per round
    static constexpr int kPollThreads = (kNW + 31) / 32 * 32; // exchanging threads
    static constexpr int kQStep = kBT / RB;              // pairs per block-wide pass
    // staged l*exp per slot + two pair buffers
    static constexpr int kCapP = (kBSmemBudget - 4096) / (RB * 8 + 16) / kQStep * kQStep;
#ifndef BSCCS_BSLOTS
#define BSCCS_BSLOTS 8
#endif
    static constexpr int kU = BSCCS_BSLOTS; // slots per thread whose gathers are in flight together
};

struct BatchArgs {
    const int2* pairs;
    const longlong2* vsplit; // [ctas][nvisit]
    const int32_t* visit;
    int nvisit;
    const int32_t* cta_subj;
    const int32_t* subject_offsets;
    const int32_t* era_len;
    const int32_t* eps;      // events_per_subject
    const int32_t* era_subj; // subject of every era
    double* xb;              // [K][RB]
    double* snap;            // [K][RB]
    double* den;             // subject blocks: [N][2*RB] doubles = den[RB] | m*n[RB] (int32) | pad
    const int32_t* m;        // [N][RB] multiplicities
    const int32_t* wn;       // m * n_i inside the subject blocks: int index s*4*RB + f from (int*)den + 2*RB
    double* beta;            // [J][RB]
    double* trust;           // [J][RB]
    const double* ydx;       // [J][RB]
    const uint8_t* colnz;    // [J][RB]
    PriorParams prior[kBMaxRB];
    unsigned live;           // fits taking part in this cycle
    int normalized;
    int ctas;
    unsigned long long* xarea; // exchange area
    unsigned long long* xcounter;
    int* fit_err;            // [RB] first error code per fit (0 = none)
    double* fit_errv;        // [RB]
    double* crit;            // [RB] criterion, [RB..2RB) change, magnitude
    long long* visited;      // [RB]
    long long* moved;        // [RB]
    const int64_t* col_ptr;  // byte accounting
    const int32_t* col_runs;
    int64_t K;
    double* bytes;           // algorithmic bytes of this launch (CTA 0)
    unsigned long long* trace; // profiling only: [ntrace][ctas][6] globaltimer stamps
    int ntrace;
};

#ifndef BSCCS_BPREFETCH
#define BSCCS_BPREFETCH 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ unsigned long long bgtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define BTRACE(slot)                                                                                     \
    do {                                                                                                 \
        if (A.trace && threadIdx.x == 0 && idx < A.ntrace)                                               \
            A.trace[(static_cast<size_t>(idx) * gridDim.x + blockIdx.x) * 6 + (slot)] = bgtimer();        \
    } while (0)

// Per-fit CTA reduction of (a, b, e): result in smem ra/rb/re[RB] (fixed order).
template <int RB>
__device__ __forceinline__ void breduce(double a, double b, int e, double* wa, double* wb, int* we, double* ra,
                                        double* rb, int* re) {
    // lanes l and l + RB*k hold the same fit
#pragma unroll
    for (int o = 16; o >= RB; o >>= 1) {
        a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
        e |= __shfl_xor_sync(0xffffffffu, e, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane < RB) {
        wa[warp * RB + lane] = a;
        wb[warp * RB + lane] = b;
        we[warp * RB + lane] = e;
    }
    __syncthreads();
    if (threadIdx.x < RB) {
        double x = 0.0, y = 0.0;
        int z = 0;
        for (int w = 0; w < kBWarps; ++w) {
            x = __dadd_rn(x, wa[w * RB + threadIdx.x]);
            y = __dadd_rn(y, wb[w * RB + threadIdx.x]);
            z |= we[w * RB + threadIdx.x];
        }
        ra[threadIdx.x] = x;
        rb[threadIdx.x] = y;
        re[threadIdx.x] = z;
    }
    __syncthreads();
}

template <int RB>
struct BSmem {
    double wa[kBWarps * RB], wb[kBWarps * RB];
    int we[kBWarps * RB];
    double ra[RB], rb[RB];
    int re[RB];
    unsigned long long xd[BCfg<RB>::kNW];
    unsigned long long pv[2][BCfg<RB>::kNW]; // running totals of both buffers (warp 0)
    double delta[RB];
    double em1[RB];   // expm1(delta): the update scales l*exp by exp(delta)
    int status[RB];   // 0 ok, else error code of the fit (it stops)
    unsigned live;
    // warp 0 lane r: fit r's coordinate scalars and counters (kept out of
    // the registers of every thread)
    double bj[2][RB], rj[2][RB], yj[2][RB], bv[2][RB], abytes[RB]; // [coordinate parity][fit]
    int nz[2][RB];
    double nzj[2], uj[2]; // column nnz and subject runs (byte accounting)
    long long nvis[RB], nmov[RB];
    int2 pst[2][BCfg<RB>::kCapP];         // pairs of this / the next coordinate's slice
    double le[BCfg<RB>::kCapP * RB];      // l*exp per slot (then the update's differences)
};

// Exchange round over the first kPollThreads threads, one word per thread:
// publish the CTA's per-fit (ra, rb, re) word as a limb or error counter,
// poll it until every participant has added, leave the total's word in
// sm.xd, then a named barrier joins the exchanging warps.  (One word per
// lane across several warps halves the exchange against one warp looping
// over 4 words each: scripts/xbench2.cu.)
template <int RB>
__device__ __forceinline__ void bexchange(const BatchArgs& A, BSmem<RB>& sm, unsigned long long seq) {
    using Cf = BCfg<RB>;
    const int w = threadIdx.x;
    const unsigned buf = static_cast<unsigned>(seq & 1ull);
    if (w < Cf::kNW) {
        unsigned long long* p = A.xarea + (static_cast<size_t>(buf) * Cf::kNW + w) * kBXStride;
        unsigned long long v = 0;
        if (w < 6 * RB) {
            const int f = w / 6, part = w % 6;
            const double x = part < 3 ? sm.ra[f] : sm.rb[f];
            if (!limb_of(x, part % 3, v)) v = 0; // out-of-range partials flagged below
        } else {
            const int e0 = (w - 6 * RB) * 6;
            for (int f = e0; f < e0 + 6 && f < RB; ++f) {
                const bool bad = sm.re[f] != 0 || !(sm.ra[f] >= 0.0 && sm.ra[f] < kXMaxValue) ||
                                 !(sm.rb[f] >= 0.0 && sm.rb[f] < kXMaxValue);
                if (bad) v += 1ull << (8 * (f - e0));
            }
        }
        red_add(p, v + kXCnt);
        const unsigned long long prev = sm.pv[buf][w];
        unsigned long long x, diff;
        do {
            x = ld_poll(p);
            diff = x - prev;
        } while ((diff >> kXCntShift) < static_cast<unsigned long long>(A.ctas));
        sm.pv[buf][w] = x;
        sm.xd[w] = diff & kXData;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(Cf::kPollThreads) : "memory");
}

template <int RB>
__device__ __forceinline__ int berr_count(const BSmem<RB>& sm, int f) {
    const int w = 6 * RB + f / 6;
    return static_cast<int>((sm.xd[w] >> (8 * (f % 6))) & 0xffull);
}

// per-slot run bookkeeping: subject of pair q of the slice
__device__ __forceinline__ int pair_subj(const int2* pairs, int64_t p0, int q) { return __ldg(&pairs[p0 + q].y); }

// Run sums of slots beyond the staging capacity: the run head walks its run
// from global memory (rare: only slices longer than kCapP pairs).
template <int RB>
__device__ __forceinline__ void gh_tail_head(const BatchArgs& A, int64_t p0, int q, int np, int fit, double& gs,
                                             double& hs, int& ferr) {
    const int2 pr = __ldg(&A.pairs[p0 + q]);
    if (q > 0 && __ldg(&A.pairs[p0 + q - 1].y) == pr.y) return; // not a head
    const int m = A.m[static_cast<size_t>(pr.y) * RB + fit];
    if (m == 0) return;
    double num = 0.0;
    for (int q2 = q; q2 < np; ++q2) {
        const int2 p2 = __ldg(&A.pairs[p0 + q2]);
        if (p2.y != pr.y) break;
        num = __dadd_rn(num, lexp(A.era_len[p2.x], A.xb[static_cast<size_t>(p2.x) * RB + fit]));
    }
    const double den = A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit];
    if (!(den > 0.0)) ferr = ferr ? ferr : DERR_DEN_NONPOSITIVE;
    double w = num / den;
    if (w > 1.0) w = 1.0;
    const double nw = __dmul_rn(static_cast<double>(m) * static_cast<double>(A.eps[pr.y]), w);
    gs = __dadd_rn(gs, nw);
    hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
}

template <int RB>
__device__ __forceinline__ void upd_tail_head(const BatchArgs& A, int64_t p0, int q, int np, int fit, double d,
                                              int& ferr, double& ferrv) {
    const int2 pr = __ldg(&A.pairs[p0 + q]);
    if (q > 0 && __ldg(&A.pairs[p0 + q - 1].y) == pr.y) return;
    if (A.m[static_cast<size_t>(pr.y) * RB + fit] == 0) return;
    double den = A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit];
    for (int q2 = q; q2 < np; ++q2) {
        const int2 p2 = __ldg(&A.pairs[p0 + q2]);
        if (p2.y != pr.y) break;
        double* xp = A.xb + static_cast<size_t>(p2.x) * RB + fit;
        const double old = *xp;
        const int len = A.era_len[p2.x];
        const double upd = __dadd_rn(old, d);
        if (!(fabs(upd) <= kBXbBound)) {
            ferr = ferr ? ferr : DERR_OVERFLOW;
            ferrv = fabs(upd);
            break;
        }
        den = __dadd_rn(den, __dsub_rn(lexp(len, upd), lexp(len, old)));
        *xp = upd;
    }
    A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit] = den;
}

// kChunk: the chunked path for slices beyond the register slots is compiled
// in; the host launches the instantiation without it when every slice fits
// (its register pressure slows the common single-chunk path).
template <int RB, bool kChunk>
__global__ void __launch_bounds__(kBT, 1) k_bccd(const __grid_constant__ BatchArgs A) {
    using Cf = BCfg<RB>;
    constexpr int U = Cf::kU;
    constexpr int QS = Cf::kQStep;
    constexpr int CAP = Cf::kCapP;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BSmem<RB>& sm = *reinterpret_cast<BSmem<RB>*>(smem_raw);
    const int c = blockIdx.x;
    const int fit = static_cast<int>(threadIdx.x) % RB;
    const int qfirst = static_cast<int>(threadIdx.x) / RB;
    const bool w0 = threadIdx.x < 32;
    unsigned long long seq = *A.xcounter;
    {
        const unsigned long long* tot = A.xarea + static_cast<size_t>(2) * Cf::kNW * kBXStride;
        for (int w = threadIdx.x; w < Cf::kNW; w += kBT) {
            sm.pv[0][w] = tot[w];
            sm.pv[1][w] = tot[Cf::kNW + w];
        }
    }
    if (threadIdx.x == 0) sm.live = A.live;
    if (threadIdx.x < RB) sm.status[threadIdx.x] = 0;
    const longlong2* vs = A.vsplit + static_cast<size_t>(c) * A.nvisit;
    if (A.nvisit > 0) { // first slice's pairs and per-fit scalars
        const longlong2 s0 = vs[0];
        const int n0 = min(static_cast<int>(s0.y - s0.x), CAP);
        for (int q = threadIdx.x; q < n0; q += kBT) sm.pst[0][q] = __ldg(&A.pairs[s0.x + q]);
        if (threadIdx.x < RB) {
            const size_t o = static_cast<size_t>(A.visit[0]) * RB + threadIdx.x;
            sm.bj[0][threadIdx.x] = A.beta[o];
            sm.bv[0][threadIdx.x] = beta_over_v(A.prior[threadIdx.x], sm.bj[0][threadIdx.x]);
            sm.rj[0][threadIdx.x] = A.trust[o];
            sm.yj[0][threadIdx.x] = A.ydx[o];
            sm.nz[0][threadIdx.x] = A.colnz[o];
        } else if (threadIdx.x == RB) {
            const int j0 = A.visit[0];
            sm.nzj[0] = static_cast<double>(A.col_ptr[j0 + 1] - A.col_ptr[j0]);
            sm.uj[0] = static_cast<double>(A.col_runs[j0]);
        }
    }
    __syncthreads();
    if (threadIdx.x < RB) {
        sm.nvis[threadIdx.x] = 0;
        sm.nmov[threadIdx.x] = 0;
        sm.abytes[threadIdx.x] = 0.0;
    }
    int ferr = 0;                 // this thread's fit: error seen (code)
    double ferrv = 0.0;
    for (int idx = 0; idx < A.nvisit; ++idx) {
        const int cur = idx & 1;
        const int2* P = sm.pst[cur];
        const int j = A.visit[idx];
        const longlong2 sl = vs[idx];
        const int64_t p0 = sl.x;
        const int np = static_cast<int>(sl.y - sl.x);
        const int lim = np < CAP ? np : CAP;
        BTRACE(0);
        const unsigned live = sm.live;
        const bool flive = (live >> fit) & 1u;
        // Single-chunk slices (every slot of this thread fits its U
        // registers) keep each slot's gathered values in registers from the
        // gradient pass through the update: one gather round trip per
        // coordinate.  Larger slices take the chunked path with reloads.
        const bool fast = !kChunk || np <= U * QS;
        double xbv[U], dn[U];
        int len[U], mm[U], fl[U]; // mm: m * n_i of the slot's subject; fl: bit0 valid, bit1 head, bit2 single run
        double gs = 0.0, hs = 0.0;
        // ---- gradient / hessian partials (engine.hpp:97-132, weighted) ----
        if (flive && fast) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = qfirst + u * QS;
                fl[u] = 0;
                mm[u] = 0;
                if (q < np) {
                    const int2 pr = P[q];
                    const int sp = q > 0 ? P[q - 1].y : -1;
                    const int sn = q + 1 < np ? P[q + 1].y : -1;
                    const bool hd = pr.y != sp;
                    fl[u] = 1 | (hd ? 2 : 0) | (hd && sn != pr.y ? 4 : 0);
#if BSCCS_DIAG_NOLOAD // profiling variant: no gathers (compute on stand-in values)
                    xbv[u] = -1e-3 * q;
                    len[u] = 10;
                    mm[u] = 1;
                    dn[u] = 50.0;
#else
                    xbv[u] = A.xb[static_cast<size_t>(pr.x) * RB + fit];
                    len[u] = __ldg(&A.era_len[pr.x]);
                    mm[u] = __ldg(&A.wn[static_cast<size_t>(pr.y) * (4 * RB) + fit]);
                    if (hd) dn[u] = A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit];
#endif
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = qfirst + u * QS;
                if (fl[u] & 1) {
#if BSCCS_DIAG_NOCOMPUTE // profiling variant: gathers consumed without exp / divide
                    {
                        const double lz = xbv[u] + len[u];
                        if ((fl[u] & 4) && mm[u] != 0) {
                            gs = __dadd_rn(gs, lz + dn[u]);
                            hs = __dadd_rn(hs, lz);
                        }
                        sm.le[q * RB + fit] = lz;
                        continue;
                    }
#endif
                    if (mm[u] == 0) continue; // a left-out subject: no term, no update (engine work skipped)
                    const double le = lexp(len[u], xbv[u]);
                    sm.le[q * RB + fit] = le;
                    if (fl[u] & 4) { // single-pair run: its term now
                        if (!(dn[u] > 0.0)) ferr = ferr ? ferr : DERR_DEN_NONPOSITIVE;
                        double w = le / dn[u];
                        if (w > 1.0) w = 1.0;
                        const double nw = __dmul_rn(static_cast<double>(mm[u]), w);
                        gs = __dadd_rn(gs, nw);
                        hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
                    }
                }
            }
        } else if (kChunk && flive) {
            for (int base = qfirst; base < lim; base += U * QS) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = base + u * QS;
                    fl[u] = 0;
                    mm[u] = 0;
                    if (q < lim) {
                        const int2 pr = P[q];
                        const int sp = q > 0 ? P[q - 1].y : -1;
                        const int sn = q + 1 < lim ? P[q + 1].y : (q + 1 < np ? pair_subj(A.pairs, p0, q + 1) : -1);
                        const bool sg = pr.y != sp && sn != pr.y;
                        fl[u] = 1 | (sg ? 4 : 0);
                        xbv[u] = A.xb[static_cast<size_t>(pr.x) * RB + fit];
                        len[u] = __ldg(&A.era_len[pr.x]);
                        if (sg) {
                            mm[u] = __ldg(&A.wn[static_cast<size_t>(pr.y) * (4 * RB) + fit]);
                            dn[u] = A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit];
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = base + u * QS;
                    if (fl[u] & 1) {
                        const double le = lexp(len[u], xbv[u]);
                        sm.le[q * RB + fit] = le;
                        if ((fl[u] & 4) && mm[u] != 0) {
                            if (!(dn[u] > 0.0)) ferr = ferr ? ferr : DERR_DEN_NONPOSITIVE;
                            double w = le / dn[u];
                            if (w > 1.0) w = 1.0;
                            const double nw = __dmul_rn(static_cast<double>(mm[u]), w);
                            gs = __dadd_rn(gs, nw);
                            hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
                        }
                    }
                }
            }
            for (int q = CAP + qfirst; q < np; q += QS) gh_tail_head<RB>(A, p0, q, np, fit, gs, hs, ferr);
        }
        BTRACE(1);
        __syncthreads();
        // heads of runs longer than one pair: numerator in ascending row order
        if (flive && fast) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if ((fl[u] & 6) != 2 || mm[u] == 0) continue; // head of a multi-pair run
                const int q = qfirst + u * QS;
                const int s = P[q].y;
                double num = 0.0;
                for (int q2 = q; q2 < np && P[q2].y == s; ++q2) num = __dadd_rn(num, sm.le[q2 * RB + fit]);
                if (!(dn[u] > 0.0)) ferr = ferr ? ferr : DERR_DEN_NONPOSITIVE;
                double w = num / dn[u];
                if (w > 1.0) w = 1.0;
                const double nw = __dmul_rn(static_cast<double>(mm[u]), w);
                gs = __dadd_rn(gs, nw);
                hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
            }
        } else if (kChunk && flive) {
            for (int q = qfirst; q < lim; q += QS) {
                const int s = P[q].y;
                if (q > 0 && P[q - 1].y == s) continue;
                const bool multi = q + 1 < np && (q + 1 < lim ? P[q + 1].y : pair_subj(A.pairs, p0, q + 1)) == s;
                if (!multi) continue;
                const int m = A.m[static_cast<size_t>(s) * RB + fit];
                if (m == 0) continue;
                double num = 0.0;
                int q2 = q;
                for (; q2 < lim && P[q2].y == s; ++q2) num = __dadd_rn(num, sm.le[q2 * RB + fit]);
                for (; q2 < np; ++q2) {
                    const int2 p2 = __ldg(&A.pairs[p0 + q2]);
                    if (p2.y != s) break;
                    num = __dadd_rn(num, lexp(A.era_len[p2.x], A.xb[static_cast<size_t>(p2.x) * RB + fit]));
                }
                const double den = A.den[static_cast<size_t>(s) * (2 * RB) + fit];
                if (!(den > 0.0)) ferr = ferr ? ferr : DERR_DEN_NONPOSITIVE;
                double w = num / den;
                if (w > 1.0) w = 1.0;
                const double nw = __dmul_rn(static_cast<double>(m) * static_cast<double>(A.eps[s]), w);
                gs = __dadd_rn(gs, nw);
                hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
            }
        }
        // warp 0's beta/trust loads were consumed into shared memory before
        // the barriers of this reduction, so the publish cannot overtake them
        // (CTA 0 overwrites them after the exchange)
        breduce<RB>(gs, hs, ferr, sm.wa, sm.wb, sm.we, sm.ra, sm.rb, sm.re);
        BTRACE(2);
        if (threadIdx.x < Cf::kPollThreads) bexchange<RB>(A, sm, seq);
        if (w0) {
            const int r = threadIdx.x;
            if (r < RB) {
                // this coordinate's beta / trust / y_dot_x, prefetched during
                // the previous exchange (CTA 0 writes column j only after
                // this coordinate's exchange, which needs this CTA's publish)
                const double bj = sm.bj[cur][r], rj = sm.rj[cur][r];
                double delta = 0.0;
                int st = sm.status[r];
                const bool lr = ((live >> r) & 1u) && st == 0;
                const bool skip = !sm.nz[cur][r] && bj == 0.0; // solver.hpp:119-121 (weighted column)
                if (lr && !skip) {
                    if (berr_count<RB>(sm, r) != 0) {
                        st = -1; // an error seen by some CTA (recorded there)
                    } else {
                        bool o1, o2;
                        const double tg = from_limbs(sm.xd[6 * r], sm.xd[6 * r + 1], sm.xd[6 * r + 2], o1);
                        const double th = from_limbs(sm.xd[6 * r + 3], sm.xd[6 * r + 4], sm.xd[6 * r + 5], o2);
                        const double g = __dsub_rn(sm.yj[cur][r], tg);
                        const double h = th == 0.0 ? 0.0 : -th;
                        double step = 0.0;
                        const int serr = (o1 || o2) ? DERR_SUM_RANGE
                                                    : penalized_step_pre(A.prior[r], bj, sm.bv[cur][r], g, h, &step);
                        if (serr) {
                            st = serr;
                            if (c == 0) {
                                A.fit_err[r] = serr;
                                A.fit_errv[r] = h;
                            }
                        } else {
                            delta = clamp_step(step, rj);
                            if (delta != 0.0 && !isfinite(delta)) {
                                st = DERR_STEP_NONFINITE;
                                delta = 0.0;
                                if (c == 0) {
                                    A.fit_err[r] = DERR_STEP_NONFINITE;
                                    A.fit_errv[r] = step;
                                }
                            } else {
                                ++sm.nvis[r];
                                const double nzj = sm.nzj[cur], uj = sm.uj[cur];
                                double ab = 8.0 * nzj + 12.0 * uj; // x'beta gathers; den, m per run
                                if (delta != 0.0) {
                                    ++sm.nmov[r];
                                    ab += 8.0 * nzj + 8.0 * uj; // x'beta, den writes
                                }
                                if (r == 0) // pairs + era lengths + event counts, once for all fits
                                    ab += 12.0 * nzj + 4.0 * uj;
                                sm.abytes[r] += ab;
                                if (c == 0) {
                                    A.beta[static_cast<size_t>(j) * RB + r] = __dadd_rn(bj, delta);
                                    A.trust[static_cast<size_t>(j) * RB + r] = next_trust(delta, rj);
                                }
                            }
                        }
                    }
                }
                sm.delta[r] = st == 0 ? delta : 0.0;
                sm.em1[r] = st == 0 ? expm1(delta) : 0.0;
                sm.status[r] = st;
            }
        } else if (threadIdx.x >= Cf::kPollThreads && idx + 1 < A.nvisit) {
            // while the partials travel: the next coordinate's per-fit scalars ...
            const int tt = static_cast<int>(threadIdx.x) - Cf::kPollThreads;
            if (tt < RB) {
                const size_t o = static_cast<size_t>(A.visit[idx + 1]) * RB + tt;
                const double b1 = A.beta[o];
                sm.bj[cur ^ 1][tt] = b1;
                sm.bv[cur ^ 1][tt] = beta_over_v(A.prior[tt], b1);
                sm.rj[cur ^ 1][tt] = A.trust[o];
                sm.yj[cur ^ 1][tt] = A.ydx[o];
                sm.nz[cur ^ 1][tt] = A.colnz[o];
            } else if (tt == RB) {
                const int j1 = A.visit[idx + 1];
                sm.nzj[cur ^ 1] = static_cast<double>(A.col_ptr[j1 + 1] - A.col_ptr[j1]);
                sm.uj[cur ^ 1] = static_cast<double>(A.col_runs[j1]);
            }
            // ... and the next slice's pairs
            const longlong2 nsl = vs[idx + 1];
            const int nn = min(static_cast<int>(nsl.y - nsl.x), CAP);
            int2* Q = sm.pst[cur ^ 1];
            // single-chunk slices only: measured -14% sweep time at config 2
            // (1M), +10% at config 3 (10M, chunked slices) where the extra
            // line fetches compete with the gathers
            const bool pf = BSCCS_BPREFETCH && nsl.y - nsl.x <= U * QS;
            for (int q = threadIdx.x - Cf::kPollThreads; q < nn; q += kBT - Cf::kPollThreads) {
                const int2 pr = __ldg(&A.pairs[nsl.x + q]);
                Q[q] = pr;
#if BSCCS_BPREFETCH
                // ... and their gathers, into L2: the next gradient pass then
                // hits L2 instead of HBM (the update below writes through L2,
                // so nothing prefetched can go stale)
                if (!pf) continue;
                prefetch_l2(A.xb + static_cast<size_t>(pr.x) * RB);
                prefetch_l2(A.era_len + pr.x);
                prefetch_l2(A.den + static_cast<size_t>(pr.y) * (2 * RB));
                if (RB * 8 >= 128) prefetch_l2(A.den + static_cast<size_t>(pr.y) * (2 * RB) + RB);
#endif
            }
        }
        ++seq;
        __syncthreads();
        BTRACE(3);
        if (threadIdx.x == 0) {
            unsigned lv = live;
            for (int r = 0; r < RB; ++r)
                if (sm.status[r] != 0) lv &= ~(1u << r);
            sm.live = lv;
        }
        // ---- sparse update (engine.hpp:205-231), weighted subjects only ----
        const double d = sm.delta[fit];
        // l*exp(x'b + d) - l*exp(x'b) = l*exp(x'b) * expm1(d): the reference's
        // difference (engine.hpp:224-226) up to rounding, with no per-era exp
        const double em1 = sm.em1[fit];
        if (flive && d != 0.0 && fast) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!(fl[u] & 1) || mm[u] == 0) continue;
                const int q = qfirst + u * QS;
                const int2 pr = P[q];
                const double upd = __dadd_rn(xbv[u], d);
                double diff = 0.0;
                if (!(fabs(upd) <= kBXbBound)) {
                    ferr = ferr ? ferr : DERR_OVERFLOW;
                    ferrv = fabs(upd);
                } else {
                    diff = __dmul_rn(sm.le[q * RB + fit], em1);
                    A.xb[static_cast<size_t>(pr.x) * RB + fit] = upd;
                }
                if (fl[u] & 4) A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit] = __dadd_rn(dn[u], diff);
                else sm.le[q * RB + fit] = diff; // this slot's l*exp is no longer needed
            }
        } else if (kChunk && flive && d != 0.0) {
            for (int base = qfirst; base < lim; base += U * QS) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = base + u * QS;
                    mm[u] = 0;
                    fl[u] = 0;
                    if (q < lim) {
                        const int2 pr = P[q];
                        const int sp = q > 0 ? P[q - 1].y : -1;
                        const int sn = q + 1 < lim ? P[q + 1].y : (q + 1 < np ? pair_subj(A.pairs, p0, q + 1) : -1);
                        const bool sg = pr.y != sp && sn != pr.y;
                        fl[u] = 1 | (sg ? 4 : 0);
                        mm[u] = __ldg(&A.wn[static_cast<size_t>(pr.y) * (4 * RB) + fit]);
                        xbv[u] = A.xb[static_cast<size_t>(pr.x) * RB + fit];
                        if (sg) dn[u] = A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = base + u * QS;
                    if ((fl[u] & 1) && mm[u] != 0) {
                        const int2 pr = P[q];
                        const double upd = __dadd_rn(xbv[u], d);
                        double diff = 0.0;
                        if (!(fabs(upd) <= kBXbBound)) {
                            ferr = ferr ? ferr : DERR_OVERFLOW;
                            ferrv = fabs(upd);
                        } else {
                            diff = __dmul_rn(sm.le[q * RB + fit], em1);
                            A.xb[static_cast<size_t>(pr.x) * RB + fit] = upd;
                        }
                        if (fl[u] & 4) A.den[static_cast<size_t>(pr.y) * (2 * RB) + fit] = __dadd_rn(dn[u], diff);
                        else sm.le[q * RB + fit] = diff;
                    }
                }
            }
            for (int q = CAP + qfirst; q < np; q += QS) upd_tail_head<RB>(A, p0, q, np, fit, d, ferr, ferrv);
        }
        BTRACE(4);
        __syncthreads();
        if (flive && d != 0.0 && fast) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if ((fl[u] & 6) != 2 || mm[u] == 0) continue;
                const int q = qfirst + u * QS;
                const int s = P[q].y;
                double den = dn[u];
                for (int q2 = q; q2 < np && P[q2].y == s; ++q2) den = __dadd_rn(den, sm.le[q2 * RB + fit]);
                A.den[static_cast<size_t>(s) * (2 * RB) + fit] = den;
            }
        } else if (kChunk && flive && d != 0.0) {
            for (int q = qfirst; q < lim; q += QS) {
                const int s = P[q].y;
                if (q > 0 && P[q - 1].y == s) continue;
                const bool multi = q + 1 < np && (q + 1 < lim ? P[q + 1].y : pair_subj(A.pairs, p0, q + 1)) == s;
                if (!multi) continue;
                if (A.m[static_cast<size_t>(s) * RB + fit] == 0) continue;
                double* dp = A.den + static_cast<size_t>(s) * (2 * RB) + fit;
                double den = *dp;
                int q2 = q;
                for (; q2 < lim && P[q2].y == s; ++q2) den = __dadd_rn(den, sm.le[q2 * RB + fit]);
                for (; q2 < np; ++q2) { // tail beyond the staging capacity
                    const int2 p2 = __ldg(&A.pairs[p0 + q2]);
                    if (p2.y != s) break;
                    double* xp = A.xb + static_cast<size_t>(p2.x) * RB + fit;
                    const double old = *xp;
                    const int len1 = A.era_len[p2.x];
                    const double upd = __dadd_rn(old, d);
                    if (!(fabs(upd) <= kBXbBound)) {
                        ferr = ferr ? ferr : DERR_OVERFLOW;
                        ferrv = fabs(upd);
                        break;
                    }
                    den = __dadd_rn(den, __dsub_rn(lexp(len1, upd), lexp(len1, old)));
                    *xp = upd;
                }
                *dp = den;
            }
        }
        __syncthreads(); // slice writes of this coordinate before the next reads
        BTRACE(5);
    }

    // ---- criterion (solver.hpp:154-165) per fit, snapshot in the same pass ----
    // (era, fit) slots of the CTA's era range, fit-minor: fully coalesced
    {
        const unsigned live = sm.live;
        const bool flive = (live >> fit) & 1u;
        double ch = 0.0, mg = 0.0;
        if (flive) {
            const int e0 = A.subject_offsets[A.cta_subj[c]], e1 = A.subject_offsets[A.cta_subj[c + 1]];
            // software-pipelined: the next block's era -> subject map loads
            // while this block's multiplicities (which depend on it) load
            int es[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = e0 + qfirst + u * QS;
                es[u] = k < e1 ? __ldg(&A.era_subj[k]) : 0;
            }
            for (int base = e0 + qfirst; base < e1; base += U * QS) {
                double x[U], sn[U];
                int mm[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = base + u * QS;
                    if (k < e1) {
                        const size_t o = static_cast<size_t>(k) * RB + fit;
                        x[u] = A.xb[o];
                        sn[u] = A.snap[o];
                        mm[u] = A.m[static_cast<size_t>(es[u]) * RB + fit];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = base + U * QS + u * QS;
                    es[u] = k < e1 ? __ldg(&A.era_subj[k]) : 0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = base + u * QS;
                    if (k < e1 && mm[u] != 0) {
                        const double mw = static_cast<double>(mm[u]);
                        ch = __dadd_rn(ch, __dmul_rn(mw, fabs(__dsub_rn(x[u], sn[u]))));
                        if (A.normalized) mg = __dadd_rn(mg, __dmul_rn(mw, fabs(x[u])));
                        A.snap[static_cast<size_t>(k) * RB + fit] = x[u];
                    }
                }
            }
        }
        breduce<RB>(ch, mg, ferr, sm.wa, sm.wb, sm.we, sm.ra, sm.rb, sm.re);
        if (threadIdx.x < Cf::kPollThreads) bexchange<RB>(A, sm, seq);
        if (w0) {
            const int r = threadIdx.x;
            if (r < RB && c == 0) {
                bool o1, o2;
                const double tch = from_limbs(sm.xd[6 * r], sm.xd[6 * r + 1], sm.xd[6 * r + 2], o1);
                const double tmg = from_limbs(sm.xd[6 * r + 3], sm.xd[6 * r + 4], sm.xd[6 * r + 5], o2);
                if ((o1 || o2) && ((live >> r) & 1u)) atomicCAS(&A.fit_err[r], 0, DERR_SUM_RANGE);
                A.crit[r] = A.normalized ? tch / (1.0 + tmg) : tch;
                A.crit[RB + r] = tch;
                A.crit[2 * RB + r] = tmg;
                if (berr_count<RB>(sm, r) != 0 && ((live >> r) & 1u)) atomicCAS(&A.fit_err[r], 0, -1);
                A.visited[r] += sm.nvis[r];
                A.moved[r] += sm.nmov[r];
                // criterion pass: x'beta, snapshot read + write per era, m per era
                double cb = 0.0;
                if ((live >> r) & 1u) cb = 24.0 * static_cast<double>(A.K) + 4.0 * static_cast<double>(A.K);
                A.bytes[r] = sm.abytes[r] + cb;
            }
            if (c == 0 && threadIdx.x == 0) *A.xcounter = seq + 1;
            if (c == 0) {
                unsigned long long* tot = A.xarea + static_cast<size_t>(2) * Cf::kNW * kBXStride;
                for (int w = threadIdx.x; w < Cf::kNW; w += 32) {
                    tot[w] = sm.pv[0][w];
                    tot[Cf::kNW + w] = sm.pv[1][w];
                }
            }
        }
    }
    // errors detected by this thread are recorded with their first value
    if (ferr > 0) {
        const int old = atomicCAS(&A.fit_err[fit], 0, ferr);
        if (old == 0 || (old == -1 && atomicCAS(&A.fit_err[fit], -1, ferr) == -1)) A.fit_errv[fit] = ferrv;
    }
}

__global__ void k_era_subj(const int32_t* __restrict__ off, int32_t N, int32_t* era_subj) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        for (int32_t k = off[i]; k < off[i + 1]; ++k) era_subj[k] = static_cast<int32_t>(i);
}

// ---- dense rebuild, log likelihood, weights ---------------------------------

// x'beta per era and fit from the row-major copy, ascending drugs, zeros
// skipped (engine.hpp:173-181); snapshot := x'beta; overflow per fit.
template <int RB>
__global__ void k_bdense_xb(const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_col,
                            const double* __restrict__ beta, int32_t K, unsigned mask, double* xb, double* snap,
                            int* fit_err, double* fit_errv) {
    const int fit = threadIdx.x % RB;
    const int64_t step = static_cast<int64_t>(gridDim.x) * (blockDim.x / RB);
    if (!((mask >> fit) & 1u)) return;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x / RB) + threadIdx.x / RB; k < K; k += step) {
        double x = 0.0;
        for (int64_t q = csr_ptr[k]; q < csr_ptr[k + 1]; ++q) {
            const double b = beta[static_cast<size_t>(csr_col[q]) * RB + fit];
            if (b != 0.0) x = __dadd_rn(x, b);
        }
        if (!(fabs(x) <= kBXbBound)) {
            if (atomicCAS(&fit_err[fit], 0, DERR_OVERFLOW) == 0) fit_errv[fit] = fabs(x);
        }
        xb[static_cast<size_t>(k) * RB + fit] = x;
        snap[static_cast<size_t>(k) * RB + fit] = x;
    }
}

template <int RB>
__global__ void k_bdense_den(const int32_t* __restrict__ off, const int32_t* __restrict__ len,
                             const double* __restrict__ xb, int32_t N, unsigned mask, double* den) {
    const int fit = threadIdx.x % RB;
    const int64_t step = static_cast<int64_t>(gridDim.x) * (blockDim.x / RB);
    if (!((mask >> fit) & 1u)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x / RB) + threadIdx.x / RB; i < N; i += step) {
        double t = 0.0;
        for (int32_t k = off[i]; k < off[i + 1]; ++k) t = __dadd_rn(t, lexp(len[k], xb[static_cast<size_t>(k) * RB + fit]));
        den[static_cast<size_t>(i) * (2 * RB) + fit] = t; // subject block layout
    }
}

constexpr int kBLLBlocks = 296;
constexpr int kBLLThreads = 256;

// weighted log_likelihood (engine.hpp:404-425) per fit: fixed two-level sum
template <int RB>
__global__ void k_bll_partial(const int32_t* __restrict__ off, const int32_t* __restrict__ y,
                              const int32_t* __restrict__ eps, const double* __restrict__ xb,
                              const double* __restrict__ den, const int32_t* __restrict__ w, int32_t N, unsigned mask,
                              double* partial, int* fit_err, double* fit_errv) {
    const int fit = threadIdx.x % RB;
    const int64_t step = static_cast<int64_t>(gridDim.x) * (blockDim.x / RB);
    double lin = 0.0, lg = 0.0;
    if ((mask >> fit) & 1u) {
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x / RB) + threadIdx.x / RB; i < N; i += step) {
            const int m = w[static_cast<size_t>(i) * RB + fit];
            if (m == 0) continue;
            double a = 0.0;
            for (int32_t k = off[i]; k < off[i + 1]; ++k) {
                const int yk = y[k];
                if (yk != 0) a = __dadd_rn(a, __dmul_rn(static_cast<double>(yk), xb[static_cast<size_t>(k) * RB + fit]));
            }
            const double d = den[static_cast<size_t>(i) * (2 * RB) + fit];
            if (!(d > 0.0)) {
                if (atomicCAS(&fit_err[fit], 0, DERR_LL_DEN_NONPOSITIVE) == 0) fit_errv[fit] = d;
            }
            const double mm = static_cast<double>(m);
            lin = __dadd_rn(lin, __dmul_rn(mm, a));
            lg = __dadd_rn(lg, __dmul_rn(mm * static_cast<double>(eps[i]), log(d)));
        }
    }
    __shared__ double sa[kBLLThreads], sb[kBLLThreads];
    sa[threadIdx.x] = lin;
    sb[threadIdx.x] = lg;
    __syncthreads();
    if (threadIdx.x < RB) {
        double x = 0.0, z = 0.0;
        for (int t = threadIdx.x; t < kBLLThreads; t += RB) {
            x = __dadd_rn(x, sa[t]);
            z = __dadd_rn(z, sb[t]);
        }
        partial[(static_cast<size_t>(blockIdx.x) * RB + threadIdx.x) * 2] = x;
        partial[(static_cast<size_t>(blockIdx.x) * RB + threadIdx.x) * 2 + 1] = z;
    }
}

template <int RB>
__global__ void k_bll_final(const double* partial, int nb, double* out) {
    const int r = threadIdx.x;
    if (r >= RB) return;
    double x = 0.0, z = 0.0;
    for (int b = 0; b < nb; ++b) {
        x = __dadd_rn(x, partial[(static_cast<size_t>(b) * RB + r) * 2]);
        z = __dadd_rn(z, partial[(static_cast<size_t>(b) * RB + r) * 2 + 1]);
    }
    out[r] = __dsub_rn(x, z);
}

// weighted y_dot_x and column occupancy per fit (dataset.hpp:140-150 over
// the selection): one block per column, exact integer sums
template <int RB>
__global__ void k_bwn(const int32_t* __restrict__ m, const int32_t* __restrict__ eps, int32_t N, int32_t* wn) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < static_cast<int64_t>(N) * RB;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        wn[(t / RB) * (4 * RB) + 2 * RB + t % RB] = m[t] * eps[t / RB]; // into the subject block
}

template <int RB>
__global__ void k_bydx(const int2* __restrict__ pairs, const int64_t* __restrict__ col_ptr,
                       const int32_t* __restrict__ y, const int32_t* __restrict__ m, int J, double* ydx,
                       uint8_t* colnz) {
    const int j = blockIdx.x;
    const int fit = threadIdx.x % RB;
    long long sy = 0, sm = 0;
    for (int64_t p = col_ptr[j] + threadIdx.x / RB; p < col_ptr[j + 1]; p += blockDim.x / RB) {
        const int2 pr = pairs[p];
        const long long mm = m[static_cast<size_t>(pr.y) * RB + fit];
        sy += mm * y[pr.x];
        sm += mm;
    }
    __shared__ long long a[256], b[256];
    a[threadIdx.x] = sy;
    b[threadIdx.x] = sm;
    __syncthreads();
    if (threadIdx.x < RB) {
        long long x = 0, z = 0;
        for (int t = threadIdx.x; t < static_cast<int>(blockDim.x); t += RB) {
            x += a[t];
            z += b[t];
        }
        ydx[static_cast<size_t>(j) * RB + threadIdx.x] = static_cast<double>(x);
        colnz[static_cast<size_t>(j) * RB + threadIdx.x] = z > 0 ? 1 : 0;
    }
}

// per-fit weight rows [R][N] -> fit-minor [N][RB] (zero beyond R)
template <int RB>
__global__ void k_btranspose(const int32_t* __restrict__ w, int64_t n, int R, int32_t* m, int* bad) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * RB;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = t / RB;
        const int r = static_cast<int>(t % RB);
        const int32_t v = r < R ? w[static_cast<int64_t>(r) * n + s] : 0;
        if (v < 0) atomicOr(bad, 1);
        m[t] = v;
    }
}

// multiplicities of R resamples: idx[r][N] -> m[s][RB] (+1 per draw)
template <int RB>
__global__ void k_bcount(const int32_t* __restrict__ idx, int64_t n, int R, int32_t* m) {
    const int64_t total = n * R;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(t / n);
        atomicAdd(&m[static_cast<size_t>(idx[t]) * RB + r], 1);
    }
}

// k-fold weights: train m = (fold != f_r), held-out = (fold == f_r)
template <int RB>
__global__ void k_bfold(const int32_t* __restrict__ fold_of, int32_t N, const int32_t* __restrict__ fold_r, int R,
                        int32_t* mtrain, int32_t* mheld) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < static_cast<int64_t>(N) * RB;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = t / RB;
        const int r = static_cast<int>(t % RB);
        const int in = r < R ? (fold_of[s] == fold_r[r]) : 0;
        mtrain[t] = r < R ? 1 - in : 0;
        mheld[t] = in;
    }
}

} // namespace

// ---------------------------------------------------------------------------
// Host side

struct Batch {
    const bsccs_dataset* ds = nullptr;
    int RB = 16;
    cudaStream_t stream = nullptr;
    double *xb = nullptr, *snap = nullptr, *den = nullptr;
    int32_t *m = nullptr, *mheld = nullptr;
    int32_t* era_subj = nullptr;
    double *beta = nullptr, *trust = nullptr, *ydx = nullptr;
    uint8_t* colnz = nullptr;
    int32_t* visit = nullptr;
    longlong2* vsplit = nullptr;
    unsigned long long *xarea = nullptr, *xcounter = nullptr;
    int* fit_err = nullptr;
    double* fit_errv = nullptr;
    double* crit = nullptr;
    long long *visited = nullptr, *moved = nullptr;
    double* ll_partial = nullptr;
    double* ll_out = nullptr;
    double* bytes_d = nullptr;
    int32_t* scratch_i = nullptr;
    int64_t scratch_n = 0;
    std::vector<int32_t> visit_h;
    int64_t bytes = 0;
    double sweep_ms = 0.0, alg_bytes = 0.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

size_t xarea_words(int RB) {
    const int nw = RB == 8 ? BCfg<8>::kNW : BCfg<16>::kNW;
    return static_cast<size_t>(2) * nw * kBXStride + 2 * static_cast<size_t>(nw) + 64;
}

template <int RB>
size_t smem_bytes() {
    return sizeof(BSmem<RB>);
}

} // namespace

Batch* batch_create(const bsccs_dataset* ds, int RB) {
    if (RB != 8 && RB != 16) internal_error("batch: block size must be 8 or 16");
    DeviceGuard g(ds->device);
    auto* b = new Batch();
    b->ds = ds;
    b->RB = RB;
    try {
        CUDA_TRY(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
        cudaStream_t s = b->stream;
        const int64_t K = ds->K, N = ds->N, J = ds->J;
        b->xb = dalloc<double>(K * RB, b->bytes, s);
        b->snap = dalloc<double>(K * RB, b->bytes, s);
        // per subject one 2*RB-double block: the denominators and, right
        // after them, the m*n weights -- one DRAM page per subject gather
        b->den = dalloc<double>(N * 2 * RB, b->bytes, s);
        b->m = dalloc<int32_t>(N * RB, b->bytes, s);
        b->mheld = dalloc<int32_t>(N * RB, b->bytes, s);
        b->era_subj = dalloc<int32_t>(K, b->bytes, s);
        k_era_subj<<<build_grid(ds->device), 256, 0, s>>>(ds->subject_offsets, ds->N, b->era_subj);
        count_launches(1);
        b->beta = dalloc<double>(J * RB, b->bytes, s);
        b->trust = dalloc<double>(J * RB, b->bytes, s);
        b->ydx = dalloc<double>(J * RB, b->bytes, s);
        b->colnz = dalloc<uint8_t>(J * RB, b->bytes, s);
        b->visit = dalloc<int32_t>(J, b->bytes, s);
        b->vsplit = dalloc<longlong2>(J * ds->ctas, b->bytes, s);
        b->xarea = dalloc<unsigned long long>(static_cast<int64_t>(xarea_words(RB)), b->bytes, s);
        b->xcounter = dalloc<unsigned long long>(1, b->bytes, s);
        b->fit_err = dalloc<int>(RB, b->bytes, s);
        b->fit_errv = dalloc<double>(RB, b->bytes, s);
        b->crit = dalloc<double>(3 * RB, b->bytes, s);
        b->visited = dalloc<long long>(RB, b->bytes, s);
        b->moved = dalloc<long long>(RB, b->bytes, s);
        b->ll_partial = dalloc<double>(static_cast<int64_t>(kBLLBlocks) * RB * 2, b->bytes, s);
        b->ll_out = dalloc<double>(RB, b->bytes, s);
        b->bytes_d = dalloc<double>(RB, b->bytes, s);
        CUDA_TRY(cudaMemsetAsync(b->xarea, 0, sizeof(unsigned long long) * xarea_words(RB), s));
        CUDA_TRY(cudaMemsetAsync(b->xcounter, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaEventCreate(&b->ev0));
        CUDA_TRY(cudaEventCreate(&b->ev1));
        if (RB == 8) {
            CUDA_TRY(cudaFuncSetAttribute(k_bccd<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem_bytes<8>())));
            CUDA_TRY(cudaFuncSetAttribute(k_bccd<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem_bytes<8>())));
        } else {
            CUDA_TRY(cudaFuncSetAttribute(k_bccd<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem_bytes<16>())));
            CUDA_TRY(cudaFuncSetAttribute(k_bccd<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem_bytes<16>())));
        }
        CUDA_TRY(cudaStreamSynchronize(s));
    } catch (...) {
        batch_destroy(b);
        throw;
    }
    return b;
}

void batch_destroy(Batch* b) {
    if (!b) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(b->ds->device);
    cudaStream_t s = b->stream;
    if (s) {
        for (void** p : {(void**)&b->xb, (void**)&b->snap, (void**)&b->den, (void**)&b->m, (void**)&b->mheld, (void**)&b->era_subj,
                         (void**)&b->beta, (void**)&b->trust, (void**)&b->ydx, (void**)&b->colnz, (void**)&b->visit,
                         (void**)&b->vsplit, (void**)&b->xarea, (void**)&b->xcounter, (void**)&b->fit_err,
                         (void**)&b->fit_errv, (void**)&b->crit, (void**)&b->visited, (void**)&b->moved,
                         (void**)&b->ll_partial, (void**)&b->ll_out, (void**)&b->bytes_d, (void**)&b->scratch_i}) {
            if (*p) cudaFreeAsync(*p, s);
            *p = nullptr;
        }
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
    if (b->ev0) cudaEventDestroy(b->ev0);
    if (b->ev1) cudaEventDestroy(b->ev1);
    if (prev >= 0) cudaSetDevice(prev);
    delete b;
}

int32_t* batch_scratch(Batch* b, int64_t n) {
    if (b->scratch_n < n) {
        if (b->scratch_i) cudaFreeAsync(b->scratch_i, b->stream);
        int64_t dummy = 0;
        b->scratch_i = dalloc<int32_t>(n, dummy, b->stream);
        b->scratch_n = n;
    }
    return b->scratch_i;
}

namespace {

template <int RB>
void launch_weights_ydx(Batch* b) {
    const bsccs_dataset* ds = b->ds;
    k_bydx<RB><<<ds->J, 256, 0, b->stream>>>(ds->pairs, ds->col_ptr, ds->event_counts, b->m, ds->J, b->ydx,
                                             b->colnz);
    k_bwn<RB><<<grid_for(static_cast<int64_t>(ds->N) * RB, 256, sm_count(ds->device)), 256, 0, b->stream>>>(
        b->m, ds->events_per_subject, ds->N, reinterpret_cast<int32_t*>(b->den));
    count_launches(2);
}

template <int RB>
void launch_dense(Batch* b, unsigned mask) {
    const bsccs_dataset* ds = b->ds;
    const int g = build_grid(ds->device);
    k_bdense_xb<RB><<<g, 256, 0, b->stream>>>(ds->csr_ptr, ds->csr_col, b->beta, ds->K, mask, b->xb, b->snap,
                                              b->fit_err, b->fit_errv);
    k_bdense_den<RB><<<g, 256, 0, b->stream>>>(ds->subject_offsets, ds->era_lengths, b->xb, ds->N, mask, b->den);
    count_launches(2);
}

template <int RB>
void launch_ll(Batch* b, const int32_t* w, unsigned mask) {
    const bsccs_dataset* ds = b->ds;
    k_bll_partial<RB><<<kBLLBlocks, kBLLThreads, 0, b->stream>>>(ds->subject_offsets, ds->event_counts,
                                                                ds->events_per_subject, b->xb, b->den, w, ds->N, mask,
                                                                b->ll_partial, b->fit_err, b->fit_errv);
    k_bll_final<RB><<<1, 32, 0, b->stream>>>(b->ll_partial, kBLLBlocks, b->ll_out);
    count_launches(2);
}

template <int RB>
void launch_cycle(Batch* b, BatchArgs& a) {
    void* params[] = {&a};
    // the single-chunk instantiation when every slice fits the register slots
    const bool chunk = b->ds->max_slice > BCfg<RB>::kU * BCfg<RB>::kQStep;
    void* fn = chunk ? reinterpret_cast<void*>(k_bccd<RB, true>) : reinterpret_cast<void*>(k_bccd<RB, false>);
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(b->ds->ctas), dim3(kBT), params, smem_bytes<RB>(), b->stream));
    count_launches(1);
}

} // namespace

// Multiplicities: host array [N][RB] (fit-minor) already laid out.
void batch_set_weights(Batch* b, const int32_t* m_host, const int32_t* mheld_host) {
    const bsccs_dataset* ds = b->ds;
    DeviceGuard g(ds->device);
    const size_t n = static_cast<size_t>(ds->N) * b->RB;
    CUDA_TRY(cudaMemcpyAsync(b->m, m_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice, b->stream));
    if (mheld_host) CUDA_TRY(cudaMemcpyAsync(b->mheld, mheld_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice, b->stream));
    if (b->RB == 8) launch_weights_ydx<8>(b);
    else launch_weights_ydx<16>(b);
    CUDA_TRY(cudaStreamSynchronize(b->stream));
}

// Weights as R host rows of N (bsccs_fit_batch layout), transposed on the device.
void batch_set_weight_rows(Batch* b, const int32_t* rows_host, int R) {
    const bsccs_dataset* ds = b->ds;
    DeviceGuard g(ds->device);
    const int64_t n = ds->N;
    int32_t* d = batch_scratch(b, n * R + 1);
    int* bad = reinterpret_cast<int*>(d + n * R);
    CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), b->stream));
    if (rows_host) {
        h2d(d, rows_host, sizeof(int32_t) * static_cast<size_t>(n * R), b->stream, ds->device);
    } else {
        std::vector<int32_t> ones(static_cast<size_t>(n), 1);
        for (int r = 0; r < R; ++r)
            CUDA_TRY(cudaMemcpyAsync(d + r * n, ones.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, b->stream));
        CUDA_TRY(cudaStreamSynchronize(b->stream));
    }
    const int grid = grid_for(n * b->RB, 256, sm_count(ds->device));
    if (b->RB == 8) k_btranspose<8><<<grid, 256, 0, b->stream>>>(d, n, R, b->m, bad);
    else k_btranspose<16><<<grid, 256, 0, b->stream>>>(d, n, R, b->m, bad);
    count_launches(1);
    int hb = 0;
    CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, b->stream));
    CUDA_TRY(cudaStreamSynchronize(b->stream));
    if (hb) input_error("fit_batch: negative subject weight");
    if (b->RB == 8) launch_weights_ydx<8>(b);
    else launch_weights_ydx<16>(b);
    CUDA_TRY(cudaStreamSynchronize(b->stream));
}

// Bootstrap multiplicities from R resample index lists (host, [R][N]).
void batch_set_resamples(Batch* b, const int32_t* idx_host, int R) {
    const bsccs_dataset* ds = b->ds;
    DeviceGuard g(ds->device);
    const int64_t n = ds->N;
    int32_t* d_idx = batch_scratch(b, n * R);
    h2d(d_idx, idx_host, sizeof(int32_t) * static_cast<size_t>(n * R), b->stream, ds->device);
    CUDA_TRY(cudaMemsetAsync(b->m, 0, sizeof(int32_t) * static_cast<size_t>(n) * b->RB, b->stream));
    const int grid = grid_for(n * R, 256, sm_count(ds->device));
    if (b->RB == 8) k_bcount<8><<<grid, 256, 0, b->stream>>>(d_idx, n, R, b->m);
    else k_bcount<16><<<grid, 256, 0, b->stream>>>(d_idx, n, R, b->m);
    count_launches(1);
    if (b->RB == 8) launch_weights_ydx<8>(b);
    else launch_weights_ydx<16>(b);
    CUDA_TRY(cudaStreamSynchronize(b->stream));
}

// CV fold weights from the fold of every subject and the fold of every fit.
void batch_set_folds(Batch* b, const int32_t* fold_of_host, const int32_t* fold_r, int R) {
    const bsccs_dataset* ds = b->ds;
    DeviceGuard g(ds->device);
    const int64_t n = ds->N;
    int32_t* d = batch_scratch(b, n + kBMaxRB);
    h2d(d, fold_of_host, sizeof(int32_t) * static_cast<size_t>(n), b->stream, ds->device);
    std::vector<int32_t> fr(kBMaxRB, -1);
    std::copy(fold_r, fold_r + R, fr.begin());
    CUDA_TRY(cudaMemcpyAsync(d + n, fr.data(), sizeof(int32_t) * kBMaxRB, cudaMemcpyHostToDevice, b->stream));
    const int grid = grid_for(n * b->RB, 256, sm_count(ds->device));
    if (b->RB == 8) k_bfold<8><<<grid, 256, 0, b->stream>>>(d, ds->N, d + n, R, b->m, b->mheld);
    else k_bfold<16><<<grid, 256, 0, b->stream>>>(d, ds->N, d + n, R, b->m, b->mheld);
    count_launches(1);
    if (b->RB == 8) launch_weights_ydx<8>(b);
    else launch_weights_ydx<16>(b);
    CUDA_TRY(cudaStreamSynchronize(b->stream));
}

// fit_impl (solver.hpp:170-199) for R fits at once.  init: [R][J] or null
// rows (per fit, null = zeros).  Outputs per fit: beta [R][J], results.
// held: also evaluate the held-out weights' log likelihood (predictive LL).
void batch_fit(Batch* b, int R, const PriorParams* priors, const double* const* init, const bsccs_solver_config* cfg,
               double* beta_out, bsccs_fit_result* res, int* err_code, double* pred_ll) {
    NvtxRange nvtx_("fit_batch");
    const bsccs_dataset* ds = b->ds;
    const int RB = b->RB;
    if (R < 1 || R > RB) internal_error("batch: fit count out of range");
    DeviceGuard g(ds->device);
    cudaStream_t s = b->stream;
    const int32_t J = ds->J;
    const unsigned all = R == 32 ? 0xffffffffu : ((1u << R) - 1u);
    // beta / trust [J][RB]
    std::vector<double> bh(static_cast<size_t>(J) * RB, 0.0), th(static_cast<size_t>(J) * RB, cfg->trust_init);
    for (int r = 0; r < R; ++r)
        if (init && init[r])
            for (int32_t j = 0; j < J; ++j) {
                if (!std::isfinite(init[r][j])) input_error("init_state: non-finite coefficient");
                bh[static_cast<size_t>(j) * RB + r] = init[r][j];
            }
    CUDA_TRY(cudaMemcpyAsync(b->beta, bh.data(), sizeof(double) * bh.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(b->trust, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(b->fit_err, 0, sizeof(int) * RB, s));
    CUDA_TRY(cudaMemsetAsync(b->visited, 0, sizeof(long long) * RB, s));
    CUDA_TRY(cudaMemsetAsync(b->moved, 0, sizeof(long long) * RB, s));
    auto dense = [&](unsigned mask) {
        if (RB == 8) launch_dense<8>(b, mask);
        else launch_dense<16>(b, mask);
    };
    dense(all);
    for (int r = 0; r < R; ++r) {
        std::memset(&res[r], 0, sizeof(bsccs_fit_result));
        res[r].final_criterion = INFINITY;
        res[r].log_posterior = -INFINITY;
        err_code[r] = 0;
    }
    std::vector<int> ferr(RB);
    std::vector<double> ferrv(RB), crit(3 * RB);
    std::vector<long long> vis(RB), mov(RB);
    unsigned live = all;
    int cycles = 0;
    auto read_errors = [&]() {
        CUDA_TRY(cudaMemcpyAsync(ferr.data(), b->fit_err, sizeof(int) * RB, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(ferrv.data(), b->fit_errv, sizeof(double) * RB, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        CUDA_TRY(cudaGetLastError());
        for (int r = 0; r < R; ++r)
            if (ferr[r] != 0 && err_code[r] == 0) {
                err_code[r] = ferr[r] < 0 ? 99 : ferr[r]; // 99: reported through the exchange only
                live &= ~(1u << r);
            }
    };
    read_errors(); // init_state overflow
    // visit list: every column non-empty in the parent (an empty parent column
    // is empty for every selection; its beta stays at its start value and the
    // skip rule holds unless a warm start made it non-zero -- then visit it);
    // the per-fit skip rule (solver.hpp:119-121) runs in the kernel
    std::vector<uint8_t> keep(static_cast<size_t>(J), 0);
    for (int32_t j = 0; j < J; ++j) {
        bool any_nz = false;
        for (int r = 0; r < R && !any_nz; ++r) any_nz = bh[static_cast<size_t>(j) * RB + r] != 0.0;
        keep[static_cast<size_t>(j)] = ds->col_nonempty_h[static_cast<size_t>(j)] || any_nz;
    }
    // visit order: ascending, or reshuffled every cycle (solver.hpp:109-114)
    // by the generator every fit of the batch shares (same seed, same cycle)
    std::vector<int32_t> order(static_cast<size_t>(J));
    for (int32_t j = 0; j < J; ++j) order[static_cast<size_t>(j)] = j;
    Xoshiro order_rng(cfg->cycle_seed);
    std::vector<int32_t> visit;
    auto upload_visit = [&]() {
        visit.clear();
        for (int32_t j : order)
            if (keep[static_cast<size_t>(j)]) visit.push_back(j);
        if (visit != b->visit_h) {
            b->visit_h = visit;
            if (!visit.empty()) {
                CUDA_TRY(
                    cudaMemcpyAsync(b->visit, visit.data(), sizeof(int32_t) * visit.size(), cudaMemcpyHostToDevice, s));
                build_vsplit(ds, b->visit, static_cast<int>(visit.size()), b->vsplit, s);
                CUDA_TRY(cudaStreamSynchronize(s)); // `visit` is reused by the next cycle
            }
        }
    };
    if (!cfg->random_cycle) upload_visit();
    BatchArgs a;
    std::memset(&a, 0, sizeof a);
    a.pairs = ds->pairs;
    a.vsplit = b->vsplit;
    a.visit = b->visit;
    a.nvisit = static_cast<int>(std::count(keep.begin(), keep.end(), static_cast<uint8_t>(1)));
    a.cta_subj = ds->cta_subj;
    a.subject_offsets = ds->subject_offsets;
    a.era_len = ds->era_lengths;
    a.eps = ds->events_per_subject;
    a.era_subj = b->era_subj;
    a.xb = b->xb;
    a.snap = b->snap;
    a.den = b->den;
    a.m = b->m;
    a.wn = reinterpret_cast<const int32_t*>(b->den) + 2 * RB;
    a.beta = b->beta;
    a.trust = b->trust;
    a.ydx = b->ydx;
    a.colnz = b->colnz;
    for (int r = 0; r < R; ++r) a.prior[r] = priors[r];
    a.normalized = cfg->convergence != 0;
    a.ctas = ds->ctas;
    a.xarea = b->xarea;
    a.xcounter = b->xcounter;
    a.fit_err = b->fit_err;
    a.fit_errv = b->fit_errv;
    a.crit = b->crit;
    a.visited = b->visited;
    a.moved = b->moved;
    a.col_ptr = ds->col_ptr;
    a.col_runs = ds->col_runs;
    a.K = ds->K;
    a.bytes = b->bytes_d;
    a.trace = debug_trace_buffer(&a.ntrace);
    std::vector<double> lb(RB);
    b->sweep_ms = 0.0;
    b->alg_bytes = 0.0;
    while (live && cycles < cfg->max_cycles) {
        if (cfg->random_cycle) {
            for (size_t jj = order.size(); jj > 1; --jj) {
                const size_t rr = static_cast<size_t>(order_rng.below(jj));
                std::swap(order[jj - 1], order[rr]);
            }
            upload_visit();
        }
        a.live = live;
        CUDA_TRY(cudaEventRecord(b->ev0, s));
        if (RB == 8) launch_cycle<8>(b, a);
        else launch_cycle<16>(b, a);
        CUDA_TRY(cudaEventRecord(b->ev1, s));
        CUDA_TRY(cudaMemcpyAsync(crit.data(), b->crit, sizeof(double) * 3 * RB, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(lb.data(), b->bytes_d, sizeof(double) * RB, cudaMemcpyDeviceToHost, s));
        read_errors();
        for (int r = 0; r < RB; ++r) b->alg_bytes += lb[r];
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, b->ev0, b->ev1));
        b->sweep_ms += ms;
        ++cycles;
        for (int r = 0; r < R; ++r) {
            if (!((a.live >> r) & 1u)) continue;
            res[r].cycles_run = cycles;
            if (err_code[r]) continue;
            res[r].final_criterion = crit[r];
            if (crit[r] <= cfg->epsilon) { // solver.hpp:183-185
                res[r].converged = 1;
                live &= ~(1u << r);
            }
        }
        if (live && cycles % cfg->dense_refresh_interval == 0) { // solver.hpp:187-189
            dense(live);
            for (int r = 0; r < R; ++r)
                if ((live >> r) & 1u) ++res[r].dense_refreshes;
            read_errors();
        }
    }
    // final rebuild of every fit that did not fail (solver.hpp:192)
    unsigned ok = 0;
    for (int r = 0; r < R; ++r)
        if (!err_code[r]) ok |= 1u << r;
    if (ok) {
        dense(ok);
        read_errors();
    }
    ok = 0;
    for (int r = 0; r < R; ++r)
        if (!err_code[r]) ok |= 1u << r;
    std::vector<double> ll(RB, 0.0), pll(RB, 0.0);
    if (ok) {
        if (RB == 8) launch_ll<8>(b, b->m, ok);
        else launch_ll<16>(b, b->m, ok);
        CUDA_TRY(cudaMemcpyAsync(ll.data(), b->ll_out, sizeof(double) * RB, cudaMemcpyDeviceToHost, s));
        if (pred_ll) {
            CUDA_TRY(cudaStreamSynchronize(s));
            if (RB == 8) launch_ll<8>(b, b->mheld, ok);
            else launch_ll<16>(b, b->mheld, ok);
            CUDA_TRY(cudaMemcpyAsync(pll.data(), b->ll_out, sizeof(double) * RB, cudaMemcpyDeviceToHost, s));
        }
        read_errors();
    }
    CUDA_TRY(cudaMemcpyAsync(bh.data(), b->beta, sizeof(double) * bh.size(), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(vis.data(), b->visited, sizeof(long long) * RB, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(mov.data(), b->moved, sizeof(long long) * RB, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int r = 0; r < R; ++r) {
        double* out = beta_out + static_cast<size_t>(r) * J;
        for (int32_t j = 0; j < J; ++j) out[j] = bh[static_cast<size_t>(j) * RB + r];
        res[r].coordinates_visited = vis[r];
        res[r].coordinates_moved = mov[r];
        res[r].dense_refreshes += 1;
        res[r].sweep_seconds = b->sweep_ms * 1e-3;
        res[r].algorithmic_bytes = b->alg_bytes; // the whole batch's (shared stream included)
        if (!err_code[r]) {
            res[r].log_posterior = ll[r] + log_density(priors[r], out, J);
            if (pred_ll) pred_ll[r] = pll[r];
        }
    }
}

double batch_sweep_ms(const Batch* b) { return b->sweep_ms; }
double batch_alg_bytes(const Batch* b) { return b->alg_bytes; }

// ---- drivers over the batched engine ----------------------------------------

namespace {

int pick_rb(int wanted, int R) {
    if (wanted == 8 || (wanted <= 0 && R <= 8)) return 8;
    return 16;
}

// every device error of a fit maps to numeric_error / internal_error in the
// reference (engine.hpp, prior.hpp): an invalid CV cell, never an input error
bool cell_error_is_numeric(int code) { return code != 0; }

} // namespace

void cv_folds_batched(const bsccs_dataset* ds, const bsccs_cv_config* cfg, const std::vector<double>& grid,
                      const std::vector<int32_t>& fold_subjects, const std::vector<int32_t>& fold_sizes, int32_t f0,
                      int32_t f1, bsccs_cv_cell* cells, bsccs_cv_result* res) {
    const int32_t folds = cfg->folds, N = ds->N, J = ds->J;
    const int points = static_cast<int>(grid.size());
    std::vector<int32_t> fold_of(static_cast<size_t>(N));
    {
        int64_t p = 0;
        for (int32_t f = 0; f < folds; ++f)
            for (int32_t i = 0; i < fold_sizes[static_cast<size_t>(f)]; ++i) fold_of[fold_subjects[p++]] = f;
    }
    const int RB = pick_rb(cfg->batch, f1 - f0);
    Batch* b = batch_create(ds, RB);
    try {
        for (int32_t fb = f0; fb < f1; fb += RB) {
            const int R = std::min<int32_t>(RB, f1 - fb);
            std::vector<int32_t> fr(static_cast<size_t>(R));
            for (int r = 0; r < R; ++r) fr[r] = fb + r;
            batch_set_folds(b, fold_of.data(), fr.data(), R);
            std::vector<std::vector<double>> carried(static_cast<size_t>(R));
            std::vector<double> beta(static_cast<size_t>(R) * J), pll(static_cast<size_t>(R));
            std::vector<bsccs_fit_result> fr_res(static_cast<size_t>(R));
            std::vector<int> err(static_cast<size_t>(R));
            for (int g = 0; g < points; ++g) {
                bsccs_prior pr{cfg->prior_kind, cfg->variance_is_laplace_scale, grid[static_cast<size_t>(g)]};
                const PriorParams p = to_params(&pr);
                std::vector<PriorParams> priors(static_cast<size_t>(R), p);
                std::vector<const double*> init(static_cast<size_t>(R), nullptr);
                for (int r = 0; r < R; ++r)
                    if (cfg->warm_start && !carried[r].empty()) init[r] = carried[r].data();
                batch_fit(b, R, priors.data(), init.data(), &cfg->solver, beta.data(), fr_res.data(), err.data(),
                          pll.data());
                for (int r = 0; r < R; ++r) {
                    bsccs_cv_cell& cell = cells[static_cast<size_t>(g) * folds + fb + r];
                    cell = bsccs_cv_cell{-std::numeric_limits<double>::infinity(), 0, 0, 0, 0};
                    if (cell_error_is_numeric(err[r])) continue; // the fit threw: invalid cell
                    cell.cycles = fr_res[r].cycles_run;
                    cell.converged = fr_res[r].converged;
                    cell.predictive_ll = pll[r];
                    cell.valid = 1;
                    res->fits += 1;
                    res->coordinates_visited += fr_res[r].coordinates_visited;
                    if (cfg->warm_start)
                        carried[r].assign(beta.begin() + static_cast<size_t>(r) * J,
                                          beta.begin() + static_cast<size_t>(r + 1) * J);
                }
                res->device_seconds += batch_sweep_ms(b) * 1e-3;
            }
        }
    } catch (...) {
        batch_destroy(b);
        throw;
    }
    batch_destroy(b);
}

void boot_replicates_batched(const bsccs_dataset* ds, const bsccs_bootstrap_config* cfg, const double* beta_full,
                             int32_t r0, int32_t r1, double* est, int32_t* conv, bsccs_bootstrap_result* res) {
    const int32_t N = ds->N, J = ds->J;
    const PriorParams p = to_params(&cfg->prior);
    const int RB = pick_rb(cfg->batch, r1 - r0);
    Batch* b = batch_create(ds, RB);
    try {
        std::vector<int32_t> idx;
        for (int32_t rb = r0; rb < r1; rb += RB) {
            const int R = std::min<int32_t>(RB, r1 - rb);
            idx.resize(static_cast<size_t>(R) * N);
            { // replicate r's draws are a pure function of (seed, r): one host thread each
                std::vector<std::thread> th;
                for (int r = 0; r < R; ++r)
                    th.emplace_back([&, r] {
                        resample(N, cfg->seed, static_cast<uint64_t>(rb + r) + 1,
                                 idx.data() + static_cast<size_t>(r) * N);
                    });
                for (auto& t : th) t.join();
            }
            batch_set_resamples(b, idx.data(), R);
            std::vector<PriorParams> priors(static_cast<size_t>(R), p);
            std::vector<const double*> init(static_cast<size_t>(R), cfg->warm_start ? beta_full : nullptr);
            std::vector<bsccs_fit_result> fr(static_cast<size_t>(R));
            std::vector<int> err(static_cast<size_t>(R));
            batch_fit(b, R, priors.data(), init.data(), &cfg->solver, est + static_cast<size_t>(rb - r0) * J, fr.data(),
                      err.data(), nullptr);
            for (int r = 0; r < R; ++r) {
                if (err[r]) { // the reference propagates a replicate's exception
                    double v = 0.0;
                    throw_device_error(err[r], v);
                }
                conv[rb - r0 + r] = fr[r].converged;
                res->total_cycles += fr[r].cycles_run;
                res->coordinates_visited += fr[r].coordinates_visited;
            }
            res->device_seconds += batch_sweep_ms(b) * 1e-3;
        }
    } catch (...) {
        batch_destroy(b);
        throw;
    }
    batch_destroy(b);
}

} // namespace bsccs_b200
