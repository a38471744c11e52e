// ccd_kernels.cu -- sm_100a kernels of the CCD hot path and their launchers.
//
// Kernels (DESIGN.md §4 gives the roofline of each):
//   k_ccd            persistent cooperative kernel, one CTA per SM.  A launch
//                    runs one full cycle (run_cycle, solver.hpp:101-166) or a
//                    single tier-1 op.  Per coordinate: fused grad/hess over
//                    the CTA's subject-aligned slice of the column
//                    (engine.hpp:97-132), an exact order-independent
//                    all-reduce of the per-CTA partials (fixed-point limbs
//                    added with red.add into self-validating words, §4.2),
//                    the penalized step evaluated redundantly by every CTA
//                    (prior.hpp:72-122), and the sparse update of the
//                    slice's runs (engine.hpp:205-231) -- no grid barrier,
//                    one exchange per coordinate.  The next coordinate's
//                    records are gathered speculatively while the partials
//                    travel and repaired from the update's record.  Four
//                    instantiations: subject tile in shared memory or not,
//                    streamed path for large slices compiled in or not.
//   k_dense_xb       dense_recompute xbeta / l*exp rebuild (engine.hpp:68-90,
//                    170-183) from the row-major copy, reference add order
//   k_dense_den      per-subject ascending sum of l*exp (engine.hpp:81-89)
//   k_ll_partial/    log_likelihood (engine.hpp:404-425), fixed-order
//   k_ll_final       two-level reduction
//   k_ccd_dense      the reference's dense update route (UpdatePath::dense)
//   dataset build    interleave + validation, stable radix sort (CUB) to
//                    build the CSR, nnz-balanced CTA subject ranges, split.
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <chrono>
#include <atomic>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "engine.h"
#include "devutil.h"
#include "xchg.cuh"

namespace bsccs_b200 {

namespace {
std::atomic<long long> g_launches{0};
}
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fail(BSCCS_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
    }
}

namespace {

constexpr int kModeSweep = 0;
constexpr int kModeGradHess = 1;
constexpr int kModeUpdate = 2;
constexpr int kModeReduce = 3; // exact all-reduce of two host scalars over every participant
constexpr int kT = kSweepThreads;   // threads per CTA; warp 0 is the control warp
constexpr int kD = kT - 32;         // data threads (warps 1..): tile v holds pairs p0 + v*kD + (tid - 32)
#ifndef BSCCS_CACHED_TILES
#define BSCCS_CACHED_TILES 3
#endif
constexpr int kWarps = kT / 32;
constexpr int kLLBlocks = 592;      // fixed => deterministic LL reduction
constexpr int kLLThreads = 256;
constexpr int kFLBlocks = 2 * kLLBlocks; // k_final_xb / k_final_den (a fit's closing log-likelihood)
constexpr double kXbBound = 700.0;  // xbeta_bound<double> engine.hpp:20-23
// the same bound on exp(x'beta) (k_rcd): exp(+-700) as doubles
constexpr double kExpXbMax = 0x1.d945df4f8ec8ep+1009; // exp(700)
constexpr double kExpXbMin = 0x1.14f2b0fb9307fp-1010; // exp(-700)
constexpr int kHtBits = 11;         // subject hash table of the speculation repair
constexpr int kHt = 1 << kHtBits;

struct ShardArgs {
    const unsigned long long* xslots; // exchange area this shard polls (its rank's)
    unsigned long long* lslots;       // hierarchical exchange: its rank's local area (else null)
    int p_local;                      // hierarchical exchange: participants of the local area
    unsigned long long* xcounter;     // exchange sequence word of that area
    int xowner;                       // this shard's CTA 0 stores the area's baseline / counter
    const int4* pq;                   // {era slot, block slot, era length, subject - cta_subj[c]} per pair
    double* snap;
    const longlong2* vsplit; // [ctas][nvisit] (p0, p1) of each CTA's slice in visit order
    uint8_t* moved;          // [nvisit] delta != 0 per visited coordinate (CTA 0 writes)
    const int64_t* col_ptr;
    const int32_t* col_runs;
    const int64_t* split;
    const int32_t* cta_era;
    const int32_t* cta_subj;  // [ctas+1] first subject of each CTA (dense path)
    const int32_t* subject_offsets;
    double* num;              // [N] run numerators of the dense path (zero between uses)
    double* X;                // subject blocks {den, n, x'beta of each era}
    const int32_t* row_slot;  // [K] slot of each era
    const int32_t* bstart;    // [N] block of each subject
    const int32_t* era_len;   // [K] era lengths (dense path)
    // resident-beta sweep (rsweep.cuh)
    const RRec* rq;           // [nnz] pair records, CSC order
    const uint16_t* rovf;     // overflow drug lists (eras with more than 8 other drugs)
    double* denc;             // [N] denominators
    const double* beta_prev;  // [J] beta at the start of the cycle (criterion)
    const int64_t* csr_ptr;   // [K+1] row -> drugs (criterion)
    const int32_t* csr_col;
    const uint8_t* edeg;      // [K] drugs per era (criterion chunks)
    const uint16_t* ecol;     // [nnz] csr_col as u16 (criterion chunks)
    double* beta;
    double* trust;
    DevErr* err;
    DevResult* res;
    int ctas;
    int cta_begin;
    int pid_base;
    int K;
};

struct SweepArgs {
    ShardArgs sh[kMaxLocalShards];
    int nsh;
    const int32_t* visit; // coordinates of this cycle in visit order (skip rule applied)
    int nvisit;
    const double* y_dot_x;
    const uint8_t* col_nonempty;
    int J;
    PriorParams prior;
    int mode;
    int visit_begin; // kModeSweep: first visit-list entry of this launch
    int single_j;
    double single_delta;
    int normalized;
    unsigned long long* dst[kMaxRanks];
    int ndst;
    const unsigned long long* slots;
    int P;      // arrivals per polled word: every participant (flat) or every rank (hier)
    int hier;   // hierarchical exchange (multi-rank groups): see forward_local
    unsigned long long* counter;
    double red_a, red_b; // kModeReduce inputs (this rank's values)
    int prefetch; // L2 prefetch of the records two coordinates ahead (small slices only)
    int stream_off, stream_cap; // streamed-slice staging buffer in dynamic shared memory (bytes offset, pairs)
    int bm_words; // touched-subject bitmaps (words each) instead of the hash table (no subject tile)
    int ss_cap; // capacity of the shared-memory subject tile (0: subjects stay in HBM)
    int beta_cap; // k_rcd: doubles of shared memory reserved for beta (>= J, multiple of 16)
    int crit_E, crit_cap; // k_rcd criterion: eras per chunk (multiple of the CTA size), drugs per chunk buffer
    double beta_limit;    // k_rcd: |beta_j| above this stops the sweep (products of exp(beta) stay in range)
    int dbg; // profiling only: bit0 skip grad/hess, bit1 skip update, bit2 skip exchange, bit4 no speculation
    unsigned long long* trace; // profiling only: [ntrace][gridDim][kTr] globaltimer stamps
    int ntrace;
    unsigned long long poll_timeout_ns; // bounded exchange spin (DERR_XCHG_TIMEOUT)
};

constexpr int kTr = 16; // stamps: top, pre-publish, gather done, update done, post-issue, poll done,
                        // data warp at the step barrier, step computed (warp 0); k_rcd data warp 1:
                        // 8 update diffs, 9 update staged, 10 heads done, 11 repaired, 12 gh staged,
                        // 13 run terms done, 14 window issued, 15 records of idx+1 landed
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- memory helpers ----------------------------------------------------------

// one 16-byte load of the sweep's pair record (read-only for the launch)
__device__ __forceinline__ int4 ld_pq(const int4* p) { return __ldg(p); }
// the subject index field alone (run-edge tests of neighbouring pairs)
__device__ __forceinline__ int ld_pq_sub(const int4* p) { return __ldg(&p->w); }

// x'beta of an era / the header {den, n} of a subject block (read-write
// data: no read-only path; the header is 16-B aligned, bstart is even)
__device__ __forceinline__ double ld_x(const double* X, int slot) { return X[slot]; }
struct Subj {
    double den;
    int n;
};
__device__ __forceinline__ Subj ld_hdr(const double* X, int slot) {
    const double2 h = *reinterpret_cast<const double2*>(X + slot);
    Subj r;
    r.den = h.x;
    r.n = static_cast<int>(h.y);
    return r;
}

__device__ __forceinline__ void record_error(DevErr* e, int code, double value) {
    if (atomicCAS(&e->code, 0, code) == 0) e->value = value;
}

__device__ __forceinline__ int warp_id() { return static_cast<int>(threadIdx.x) >> 5; }
__device__ __forceinline__ int lane_id() { return static_cast<int>(threadIdx.x) & 31; }

// ---- order-independent exchange -------------------------------------------------
//
// Each participant splits its partial exactly into three 41-bit limbs of a
// 2^-80 fixed-point number and issues seven relaxed red.add.u64 (six limbs
// plus an error word) into the exchange area of every destination; each word
// also gains 2^52 per arrival.  A poller knows a word is complete when its
// growth since the previous use of that buffer carries P arrivals in the
// bits above 2^52 -- every word validates itself, no fences or flags.  The
// integer sum is associative, so every CTA reconstructs bit-identical totals
// whatever the arrival order: the exact sum of the partials truncated to
// 2^-80, converted within one ulp (xchg.cuh from_limbs).
// Words sit 256 B apart so the adds land on distinct L2 slices; two buffers
// alternate by sequence parity.
constexpr int kXStride = 32; // u64 words between exchange words (256 B)
constexpr int kXWords = 7;
constexpr int kXBase = 2 * kXWords * kXStride; // running totals at launch end
// Running totals of the two buffers (lanes 0..6 of warp 0): of the polled
// area (b0, b1) and, for the forwarding CTA of a hierarchical exchange, of
// its rank's local area (l0, l1).
struct XPrev {
    unsigned long long b0, b1, l0, l1;
};

__device__ __forceinline__ void xprev_load(const ShardArgs& S, XPrev& pv) {
    const int l = lane_id();
    if (threadIdx.x < 32 && l < kXWords) {
        pv.b0 = S.xslots[kXBase + l];
        pv.b1 = S.xslots[kXBase + kXWords + l];
        pv.l0 = S.lslots ? S.lslots[kXBase + l] : 0ull;
        pv.l1 = S.lslots ? S.lslots[kXBase + kXWords + l] : 0ull;
    }
}

__device__ __forceinline__ void xprev_store(const ShardArgs& S, const XPrev& pv) {
    const int l = lane_id();
    if (threadIdx.x < 32 && l < kXWords) {
        const_cast<unsigned long long*>(S.xslots)[kXBase + l] = pv.b0;
        const_cast<unsigned long long*>(S.xslots)[kXBase + kXWords + l] = pv.b1;
        if (S.lslots) {
            S.lslots[kXBase + l] = pv.l0;
            S.lslots[kXBase + kXWords + l] = pv.l1;
        }
    }
}

// Hierarchical exchange (multi-rank groups): a rank's CTAs add into its LOCAL
// area; its CTA 0 waits for all of them and adds the local integer sums,
// unconverted, into every rank's polled area as ONE arrival -- so a polled
// word takes `world` remote arrivals per exchange instead of world x CTAs,
// and integer addition keeps the totals bit-identical to the flat exchange.
// A local wait that times out forwards an error so that no peer hangs.
struct LPrev {
    unsigned long long l0, l1;
};
__device__ __noinline__ LPrev forward_local(const SweepArgs& A, const unsigned long long* lslots, int p_local,
                                            unsigned long long seq, LPrev pv) {
    const int l = lane_id();
    const unsigned buf = static_cast<unsigned>(seq & 1ull);
    const size_t off = static_cast<size_t>(buf) * kXWords * kXStride + static_cast<size_t>(l) * kXStride;
    unsigned long long diff = 0;
    bool timed_out = false;
    if (l < kXWords) {
        const unsigned long long prev = buf ? pv.l1 : pv.l0;
        unsigned long long v, t_first = 0;
        unsigned spins = 0;
        do {
            v = ld_poll(lslots + off);
            diff = v - prev;
            if ((++spins & 4095u) == 0u) {
                const unsigned long long now = gtimer();
                if (t_first == 0) t_first = now;
                else if (now - t_first > A.poll_timeout_ns) {
                    timed_out = true;
                    break;
                }
            }
        } while ((diff >> kXCntShift) < static_cast<unsigned long long>(p_local));
        if (buf) pv.l1 = v;
        else pv.l0 = v;
    }
    const bool to = __any_sync(0x7fu, timed_out);
    if (l < kXWords) {
        unsigned long long w = to ? (l == 6 ? 1ull : 0ull) : (diff & kXData);
        w += kXCnt;
        for (int d = 0; d < A.ndst; ++d) red_add_sys(A.dst[d] + off, w);
    }
    return pv;
}

// lanes 0..6 of warp 0 (all holding the same (a, b, e)) each add one word;
// the error word also counts the partials that lost bits below 2^-80
__device__ __forceinline__ void publish(const SweepArgs& A, const ShardArgs& S, int c, unsigned long long seq,
                                        double a, double b, int e, XPrev& pv) {
    const int l = lane_id();
    if (threadIdx.x >= 32 || l >= kXWords) return;
    unsigned long long w;
    bool ok = true, inex = false;
    if (l < 3) ok = limb_of(a, l, w, &inex);
    else if (l < 6) ok = limb_of(b, l - 3, w, &inex);
    else w = 0;
    const unsigned lost = __ballot_sync(0x7fu, inex);
    const bool okab = __all_sync(0x7fu, ok) && (0.0 <= a && a < kXMaxValue && 0.0 <= b && b < kXMaxValue);
    if (l == 6)
        w = ((e || !okab) ? 1ull : 0ull) | ((lost & 1u) ? 1ull << kXInexA : 0ull) |
            ((lost & 8u) ? 1ull << kXInexB : 0ull);
    w += kXCnt;
    const size_t off = static_cast<size_t>(seq & 1ull) * kXWords * kXStride + static_cast<size_t>(l) * kXStride;
    if (A.hier) {
        red_add(S.lslots + off, w);
        if (c == 0) { // out of line, by value: single fits never take this path
            const LPrev lp = forward_local(A, S.lslots, S.p_local, seq, LPrev{pv.l0, pv.l1});
            pv.l0 = lp.l0;
            pv.l1 = lp.l1;
        }
    } else if (A.ndst == 1) {
        red_add(A.dst[0] + off, w);
    } else {
        for (int d = 0; d < A.ndst; ++d) red_add_sys(A.dst[d] + off, w);
    }
}

// warp 0 only: wait for the exchange `seq`, return the totals in every lane.
// The spin is bounded (A.poll_timeout_ns of globaltimer): a participant that
// never publishes -- a peer rank that failed on the host or died -- turns
// into DERR_XCHG_TIMEOUT instead of a hang.
struct PollOut {
    double ta, tb;
    int te;
    unsigned ia, ib; // participants whose partial a / b lost bits below 2^-80
    XPrev pv;
};
__device__ __forceinline__ PollOut poll_body(const SweepArgs& A, const unsigned long long* slots, unsigned long long seq, XPrev pv,
                  unsigned long long* stamp) {
    double ta, tb;
    int te;
    const int l = lane_id();
    const unsigned buf = static_cast<unsigned>(seq & 1ull);
    unsigned long long diff = 0;
    bool timed_out = false;
    if (l < kXWords) {
        const unsigned long long* p =
            slots + static_cast<size_t>(buf) * kXWords * kXStride + static_cast<size_t>(l) * kXStride;
        const unsigned long long prev = buf ? pv.b1 : pv.b0;
        unsigned long long v, t_first = 0;
        unsigned spins = 0;
        do {
            v = ld_poll(p);
            diff = v - prev;
            if ((++spins & 4095u) == 0u) {
                const unsigned long long now = gtimer();
                if (t_first == 0) t_first = now;
                else if (now - t_first > A.poll_timeout_ns) {
                    timed_out = true;
                    break;
                }
            }
        } while ((diff >> kXCntShift) < static_cast<unsigned long long>(A.P));
        if (buf) pv.b1 = v;
        else pv.b0 = v;
    }
    __syncwarp();
    if (stamp && l == 0) *stamp = gtimer();
    const unsigned long long d = diff & kXData;
    // lane 0 rebuilds a from lanes 0..2, lane 3 rebuilds b from lanes 3..5
    const unsigned long long d1 = __shfl_down_sync(0xffffffffu, d, 1);
    const unsigned long long d2 = __shfl_down_sync(0xffffffffu, d, 2);
    bool ovf;
    const double v = from_limbs(d, d1, d2, ovf);
    ta = __shfl_sync(0xffffffffu, v, 0);
    tb = __shfl_sync(0xffffffffu, v, 3);
    const unsigned bad = __ballot_sync(0xffffffffu, ovf) & 0x9u; // lanes 0 (a) and 3 (b)
    const bool to = __any_sync(0xffffffffu, timed_out);
    const unsigned long long ew = __shfl_sync(0xffffffffu, d, 6);
    te = ((ew & kXCountMask) != 0 || bad || to) ? 1 : 0;
    if (l == 0) {
        if (to) record_error(A.sh[0].err, DERR_XCHG_TIMEOUT, 0.0);
        else if (bad) record_error(A.sh[0].err, DERR_SUM_RANGE, 0.0);
    }
    return PollOut{ta, tb, te, static_cast<unsigned>((ew >> kXInexA) & kXCountMask),
                   static_cast<unsigned>((ew >> kXInexB) & kXCountMask), pv};
}

// The same, out of line.  Which one a kernel instantiation uses is a
// measured code-generation choice: inline in the sweep with
// the shared-memory subject tile (config 2: 3% faster), out of line without
// it (config 3: 4% faster).
__device__ __noinline__ PollOut poll_ool(const SweepArgs& A, const unsigned long long* slots, unsigned long long seq,
                                         XPrev pv, unsigned long long* stamp) {
    return poll_body(A, slots, seq, pv, stamp);
}

template <bool kOOL = false>
__device__ __forceinline__ void poll(const SweepArgs& A, const unsigned long long* slots, unsigned long long seq,
                                     XPrev& pv, double& ta, double& tb, int& te, unsigned long long* stamp,
                                     unsigned* inexact = nullptr) {
    PollOut o;
    if constexpr (kOOL) o = poll_ool(A, slots, seq, pv, stamp);
    else o = poll_body(A, slots, seq, pv, stamp);
    ta = o.ta;
    tb = o.tb;
    te = o.te;
    pv = o.pv;
    if (inexact) {
        inexact[0] = o.ia;
        inexact[1] = o.ib;
    }
}

// Warp 0, after the first poll of a (gs, hs) exchange: when a total came out
// with fewer than 53 significant bits (partials that lost bits below 2^-80;
// xchg.cuh needs_refine), exchange the same partials again scaled by powers
// of two until it does -- the reference forms gs and hs in full double
// precision however small (engine.hpp:108-129), so tiny gradients and
// curvatures must not read as 0.  Degenerate fits only (a coordinate driven
// to w ~ 0); every participant takes the same rounds, `seq` advances by one
// per extra round.  Used by the single-coordinate grad/hess launch and the
// dense route; the sweep loop only detects the need and stops (ST_REFINE),
// and the host finishes that coordinate through the single-coordinate
// launches (run_sweep): compiled into the loop, even never taken, these
// rounds slowed the config-2 fit by half (code size and register pressure).
struct Refined {
    double sum_a, sum_b;
    int err;
    unsigned long long next_seq;
    XPrev prev;
};
__device__ __forceinline__ Refined refine_sums(const SweepArgs& A, const ShardArgs& S, int c,
                                              const unsigned long long* slots, unsigned long long seq, XPrev pv,
                                              double a, double b, int e, double ta, double tb, unsigned ia,
                                              unsigned ib) {
    int sa = 0, sb = 0;
    double va = ta, vb = tb;
    for (;;) {
        const bool na = needs_refine(va, ia, sa), nb = needs_refine(vb, ib, sb);
        if (!na && !nb) break;
        if (na) sa = next_scale(va, ia, sa);
        if (nb) sb = next_scale(vb, ib, sb);
        ++seq;
        publish(A, S, c, seq, ldexp(a, sa), ldexp(b, sb), e, pv);
        const PollOut o = poll_body(A, slots, seq, pv, nullptr);
        pv = o.pv;
        if (o.te) return Refined{va, vb, 1, seq, pv};
        va = ldexp(o.ta, -sa); // exact power-of-two rescale
        vb = ldexp(o.tb, -sb);
        ia = o.ia;
        ib = o.ib;
    }
    return Refined{va, vb, 0, seq, pv};
}

// the call site: the common path only tests the two counts
#define BSCCS_REFINE(A, slots, seq, pv, a, b, e, ta, tb, te, inexact)                                \
    do {                                                                                              \
        if (!(te) && ((inexact)[0] | (inexact)[1])) {                                                 \
            const Refined r_ = refine_sums(A, S, c, slots, seq, pv, a, b, e, ta, tb, (inexact)[0], (inexact)[1]); \
            ta = r_.sum_a;                                                                            \
            tb = r_.sum_b;                                                                            \
            te = r_.err;                                                                              \
            seq = r_.next_seq;                                                                        \
            pv = r_.prev;                                                                             \
        }                                                                                             \
    } while (0)

// ---- shared-memory subject tile -----------------------------------------------------
//
// When a CTA's subject range fits in shared memory, a sweep launch keeps the
// range's (den, n) there for the whole cycle: loaded once at the start,
// written back once at the end.  Heads then read and write denominators
// in shared memory -- no subject gathers in the speculative window, and the
// denominator a head reads is always current (no repair).  Subjects are
// CTA-owned (nnz-balanced subject ranges), so no other CTA touches them.
struct SubjTile {
    double* den;
    int2* touch; // per subject: {stamp of the coordinate whose update touched it, run pos | len << 16}
    int* n;
    int base;
};
// bytes per subject of the tile: den, n, and (instantiations without the
// streamed path) the touch entry that replaces the repair hash table
constexpr size_t subj_tile_bytes(bool touch) { return sizeof(double) + sizeof(int) + (touch ? sizeof(int2) : 0); }

// ---- pair slots -------------------------------------------------------------------

// Index data of one pair slot: the pair record, whether it starts a subject
// run (head) and whether the run continues past it.
struct PairSlot {
    int xs;  // era slot (-1: no pair)
    int ds;  // subject block slot
    int len; // era length
    int ls;  // subject index within the CTA's range (run identity, tile index)
    bool head;
    bool cont;
};

// Loads of one pair slot, issued ahead of use: the pair record plus (lane 0
// / lane 31 only) the subjects just outside the warp.  finalize_slot() turns
// them into head / continuation flags with warp shuffles (all lanes of a warp).
struct RawSlot {
    int4 q;
    int edge; // lane 0: subject of pair p-1 ; lane 31: subject of pair p+1
    bool first, last_valid;
};

__device__ __forceinline__ RawSlot issue_slot(const int4* __restrict__ pq, int64_t p, int64_t p0, int64_t p1) {
    RawSlot r;
    const bool valid = p < p1;
    const int l = lane_id();
    r.q = valid ? ld_pq(pq + p) : make_int4(-1, -1, 0, -1);
    r.first = valid && p == p0;
    r.last_valid = p + 1 < p1;
    // one load instruction for both edge lanes (two would serialise the
    // warp on the shared destination register)
    r.edge = -1;
    const bool lo = l == 0 && valid && p > p0, hi = l == 31 && p + 1 < p1;
    if (lo || hi) r.edge = ld_pq_sub(pq + (lo ? p - 1 : p + 1));
    return r;
}

__device__ __forceinline__ PairSlot finalize_slot(const RawSlot& r) {
    PairSlot s;
    const int l = lane_id();
    int prev = __shfl_up_sync(0xffffffffu, r.q.w, 1);
    int next = __shfl_down_sync(0xffffffffu, r.q.w, 1);
    if (l == 0) prev = r.edge;
    if (l == 31) next = r.edge;
    const bool valid = r.q.x >= 0;
    s.xs = r.q.x;
    s.ds = r.q.y;
    s.len = r.q.z;
    s.ls = r.q.w;
    s.head = valid && (r.first || prev != r.q.w);
    s.cont = valid && r.last_valid && next == r.q.w;
    return s;
}

__device__ __forceinline__ PairSlot invalid_slot() {
    PairSlot s;
    s.xs = -1;
    s.ds = -1;
    s.len = 0;
    s.ls = -1;
    s.head = false;
    s.cont = false;
    return s;
}

__device__ __forceinline__ PairSlot load_slot(const int4* __restrict__ pq, int64_t p, int64_t p0, int64_t p1) {
    return finalize_slot(issue_slot(pq, p, p0, p1));
}

__device__ __forceinline__ bool slot_valid(const PairSlot& s) { return s.xs >= 0; }

// Data-warp order: warps share schedulers by (warp % 4), so the control warp's
// scheduler-mates (warps 4, 8, ...) take the highest data ranks -- on small
// slices they hold no pairs and warp 0 issues without competition.
__device__ __forceinline__ int data_warp() {
    const int w = static_cast<int>(threadIdx.x) >> 5;
    constexpr int kMates = (kWarps - 1) / 4; // warps 4, 8, ... below kWarps
    if ((w & 3) == 0) return (kWarps - 1 - kMates) + (w >> 2) - 1;
    return w - (w >> 2) - 1;
}
__device__ __forceinline__ int data_tid() { return data_warp() * 32 + (static_cast<int>(threadIdx.x) & 31); }
__device__ __forceinline__ int slot_pos(int v) { return v * kD + data_tid(); }

// warp-uniform: does this (data) warp hold any pair of tile v of [p0, p1)?
__device__ __forceinline__ bool warp_active(int v, int64_t p0, int64_t p1) {
    return threadIdx.x >= 32 && p0 + static_cast<int64_t>(v) * kD + data_warp() * 32 < p1;
}

// ---- fused grad/hess and sparse update ------------------------------------------

// Fused per-run reduction term (engine.hpp:108-129): numerator summed in
// ascending row order, w = min(num/den, 1), nw = n*w, (nw, nw*(1-w)).
__device__ __forceinline__ void run_terms(double num, double den, int n, double& gs, double& hs, int& err) {
    if (!(den > 0.0)) err = DERR_DEN_NONPOSITIVE;
    double w = num / den;
    if (w > 1.0) w = 1.0;
    const double nw = __dmul_rn(static_cast<double>(n), w);
    gs = __dadd_rn(gs, nw);
    hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ int ht_hash(int s) {
    return static_cast<int>((static_cast<unsigned>(s) * 2654435761u) >> (32 - kHtBits));
}

// ---- slices beyond the register tiles (skewed columns) ----------------------
//
// Pairs [b0, p1) are processed in chunks of up to `cap` pairs staged in a
// dynamic shared-memory buffer (l*exp or the update's differences, and the
// subject of every pair).  Every thread stages its pairs in groups of kSU
// with all their loads in flight together (no per-pair state survives the
// staging, so the path adds little register pressure); run sums are then
// taken in ascending pair order from shared memory, and a run crossing a
// chunk edge is carried to the next chunk in shared memory (thread 0
// finishes it there).  A run that starts in the register tiles and
// continues is carried in the same way.
#ifndef BSCCS_STREAM_UNROLL
#define BSCCS_STREAM_UNROLL 2
#endif
constexpr int kSU = BSCCS_STREAM_UNROLL;
#ifndef BSCCS_STREAM_NOINLINE
#define BSCCS_STREAM_NOINLINE 0
#endif
#if BSCCS_STREAM_NOINLINE
#define STREAM_FN __noinline__
#else
#define STREAM_FN __forceinline__
#endif

struct StreamBuf {
    double* x; // [cap] l*exp (grad/hess) or fresh - old (update)
    int* sub;  // [cap] subject of each staged pair
    int cap;   // a multiple of kT
};

// (the accumulators travel by value, so the fast path's allocation is not
// disturbed by references into it)
struct GhAcc {
    double gs, hs;
    int err;
};
struct UpdErr {
    int err;
    double errv;
};

enum StepStatus { ST_OK = 0, ST_REMOTE_ERR = 1, ST_STEP_ERR = 2, ST_NONFINITE = 3, ST_REFINE = 4 };

// ---- resident-beta sweep helpers (rsweep.cuh) ---------------------------------

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// generic-proxy accesses of a buffer before the async proxy (bulk copy) rewrites it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = smem_u32(bar);
    unsigned done;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(a), "r"(parity)
                     : "memory");
    } while (!done);
}
// one bulk copy global -> shared (TMA), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                         uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
                 : "memory");
}
// L2 eviction policies: the streamed pair records go first, the denominators stay
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
#ifndef RCD_DEN_CG
#define RCD_DEN_CG 0 // experiment hook: the heads' denominator loads bypass L1
#endif
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
    double v;
    // volatile (issued where written, in the speculative window, not sunk to
    // the first use) but no memory clobber: the other loads stay free to move
#if RCD_DEN_CG
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#else
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#endif
    return v;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// ---- the sweep kernel, per register-tile count -------------------------------
namespace t3 {
#define SWEEP_TILES BSCCS_CACHED_TILES
#include "sweep_impl.cuh"
#undef SWEEP_TILES
} // namespace t3
namespace t1 {
#define SWEEP_TILES 1
#include "sweep_impl.cuh"
#undef SWEEP_TILES
} // namespace t1
// resident-beta sweep shapes: 1 slot x 384 threads (slices <= 352 pairs),
// 2 x 512 (<= 960), 3 x 384 (<= 1,056)
#ifndef RS_WIDE_THREADS
#define RS_WIDE_THREADS 512
#endif
#ifndef RS_WIDE_TILES
#define RS_WIDE_TILES 2
#endif

namespace r1 {
#define RS_TILES 1
#define RS_THREADS 384
#include "rsweep.cuh"
#undef RS_THREADS
#undef RS_TILES
} // namespace r1
namespace r2 {
#define RS_TILES RS_WIDE_TILES
#define RS_THREADS RS_WIDE_THREADS
#include "rsweep.cuh"
#undef RS_THREADS
#undef RS_TILES
} // namespace r2
namespace r3 {
#define RS_TILES 3
#define RS_THREADS 384
#include "rsweep.cuh"
#undef RS_THREADS
#undef RS_TILES
} // namespace r3

// ---- the dense update path (UpdatePath::dense) ---------------------------------
//
// The reference's benchmark route (engine.hpp:368-401, solver.hpp:124-146):
// per coordinate, the column's run numerators are scattered into a
// per-subject array, a full sweep over every subject forms (g, h), and an
// accepted step is applied to the column's rows followed by a full rebuild
// of every denominator from x'beta (refresh_from_xbeta, engine.hpp:68-90).
// Subjects and their eras are CTA-owned, so each CTA does all of that for
// its own subject range; only the (g, h) sum crosses CTAs (the exact
// exchange of §4.2).  Results equal the sparse path up to addition order.
constexpr int kDT = 256;
struct DSmem {
    double ra[kDT / 32], rb[kDT / 32];
    int re[kDT / 32];
    double delta;
    int status;
};

__device__ __forceinline__ void dblock_reduce(double& a, double& b, int& e, DSmem& sm) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    e = __reduce_or_sync(0xffffffffu, e);
    if (lane_id() == 0) {
        sm.ra[warp_id()] = a;
        sm.rb[warp_id()] = b;
        sm.re[warp_id()] = e;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = 0.0, y = 0.0;
        int z = 0;
        for (int i = 0; i < kDT / 32; ++i) {
            x = __dadd_rn(x, sm.ra[i]);
            y = __dadd_rn(y, sm.rb[i]);
            z |= sm.re[i];
        }
        a = x;
        b = y;
        e = z;
    }
}

__global__ void __launch_bounds__(kDT) k_ccd_dense(const __grid_constant__ SweepArgs A) {
    __shared__ DSmem sm;
    const ShardArgs& S = A.sh[0];
    const int c = static_cast<int>(blockIdx.x);
    const bool w0 = threadIdx.x < 32;
    unsigned long long seq = *S.xcounter;
    XPrev pv{0ull, 0ull};
    xprev_load(S, pv);
    int err = 0;
    double errv = 0.0;
    long long nvisit = 0, nmoved = 0;
    const int V = A.nvisit;
    const longlong2* vs = S.vsplit + static_cast<size_t>(c) * static_cast<size_t>(V);
    const int s0 = S.cta_subj[c], s1 = S.cta_subj[c + 1];
    bool aborted = false;
    for (int idx = 0; idx < V; ++idx) {
        const int j = A.visit[idx];
        const longlong2 sl = vs[idx];
        double bj = 0.0, rj = 1.0;
        if (w0) {
            bj = S.beta[j];
            rj = S.trust[j];
        }
        // run numerators of the column into num[subject] (engine.hpp:376-380)
        for (int64_t p = sl.x + threadIdx.x; p < sl.y; p += kDT) {
            const int4 pr = ld_pq(S.pq + p);
            if (p > sl.x && ld_pq_sub(S.pq + p - 1) == pr.w) continue;
            double numv = 0.0;
            for (int64_t q = p; q < sl.y; ++q) {
                const int4 p2 = ld_pq(S.pq + q);
                if (p2.w != pr.w) break;
                numv = __dadd_rn(numv, lexp(p2.z, ld_x(S.X, p2.x)));
            }
            S.num[s0 + pr.w] = numv;
        }
        __syncthreads();
        // full sweep over the CTA's subjects (engine.hpp:381-395)
        double gs = 0.0, hs = 0.0;
        for (int s = s0 + static_cast<int>(threadIdx.x); s < s1; s += kDT) {
            const Subj sr = ld_hdr(S.X, S.bstart[s]);
            if (!(sr.den > 0.0)) err = DERR_DEN_NONPOSITIVE;
            double w = S.num[s] / sr.den;
            if (w > 1.0) w = 1.0;
            const double nw = __dmul_rn(static_cast<double>(sr.n), w);
            gs = __dadd_rn(gs, nw);
            hs = __dadd_rn(hs, __dmul_rn(nw, __dsub_rn(1.0, w)));
        }
        int e = err | ((bj != bj) || (rj != rj) ? 1 : 0);
        dblock_reduce(gs, hs, e, sm);
        publish(A, S, c, seq, gs, hs, e, pv);
        if (w0) {
            double tg, th;
            int te = 0;
            unsigned inexact[2];
            poll(A, S.xslots, seq, pv, tg, th, te, nullptr, inexact);
            BSCCS_REFINE(A, S.xslots, seq, pv, gs, hs, e, tg, th, te, inexact);
            int status = ST_OK;
            double delta = 0.0;
            if (te) {
                status = ST_REMOTE_ERR;
            } else {
                const double g = __dsub_rn(A.y_dot_x[j], tg);
                const double h = th == 0.0 ? 0.0 : -th;
                double step = 0.0;
                const int serr = penalized_step(A.prior, bj, g, h, &step);
                if (serr) {
                    status = ST_STEP_ERR;
                    if (c == 0 && threadIdx.x == 0) record_error(S.err, serr, h);
                } else {
                    delta = clamp_step(step, rj);
                    if (delta != 0.0 && !isfinite(delta)) {
                        status = ST_NONFINITE;
                        if (c == 0 && threadIdx.x == 0) record_error(S.err, DERR_STEP_NONFINITE, delta);
                    }
                }
            }
            if (threadIdx.x == 0) {
                sm.delta = delta;
                sm.status = status;
                if (c == 0 && status == ST_OK) {
                    S.moved[idx] = delta != 0.0 ? 1 : 0;
                    S.beta[j] = __dadd_rn(bj, delta);
                    S.trust[j] = next_trust(delta, rj);
                }
            }
        }
        ++seq;
        __syncthreads();
        const int status = sm.status;
        const double delta = sm.delta;
        // the numerators are consumed: back to zero for the next column
        for (int64_t p = sl.x + threadIdx.x; p < sl.y; p += kDT) S.num[s0 + ld_pq_sub(S.pq + p)] = 0.0;
        if (status != ST_OK) {
            aborted = true;
            if (status == ST_REMOTE_ERR && c == 0 && threadIdx.x == 0) S.res->err_remote = 1;
            break;
        }
        ++nvisit;
        if (delta != 0.0) {
            ++nmoved;
            // x'beta of the column's rows (solver.hpp:138-143) ...
            for (int64_t p = sl.x + threadIdx.x; p < sl.y; p += kDT) {
                const int xs = ld_pq(S.pq + p).x;
                S.X[xs] = __dadd_rn(S.X[xs], delta);
            }
            __syncthreads();
            // ... then every denominator rebuilt from x'beta (engine.hpp:68-90)
            for (int s = s0 + static_cast<int>(threadIdx.x); s < s1; s += kDT) {
                double total = 0.0;
                const int b = S.bstart[s] + kBlockHeader, k0 = S.subject_offsets[s];
                for (int k = k0; k < S.subject_offsets[s + 1]; ++k) {
                    const double xb = S.X[b + (k - k0)];
                    if (!(fabs(xb) <= kXbBound)) {
                        err = DERR_OVERFLOW;
                        errv = fabs(xb);
                    }
                    total = __dadd_rn(total, lexp(S.era_len[k], xb));
                }
                S.X[S.bstart[s]] = total;
            }
        }
        __syncthreads();
    }
    if (!aborted) {
        // criterion (solver.hpp:154-165), snapshot for the next cycle
        const int e0 = S.cta_era[c], e1 = S.cta_era[c + 1];
        double ch = 0.0, mg = 0.0;
        for (int k = e0 + static_cast<int>(threadIdx.x); k < e1; k += kDT) {
            const double xb = S.X[S.row_slot[k]];
            ch = __dadd_rn(ch, fabs(__dsub_rn(xb, S.snap[k])));
            if (A.normalized) mg = __dadd_rn(mg, fabs(xb));
            S.snap[k] = xb;
        }
        int e = err;
        dblock_reduce(ch, mg, e, sm);
        publish(A, S, c, seq, ch, mg, e, pv);
        if (w0) {
            double tch, tmg;
            int te;
            poll(A, S.xslots, seq, pv, tch, tmg, te, nullptr);
            if (c == 0 && threadIdx.x == 0) {
                S.res->change = tch;
                S.res->magnitude = tmg;
                S.res->criterion = A.normalized ? tch / (1.0 + tmg) : tch;
                S.res->err_remote = te;
            }
        }
        ++seq;
    }
    if (err) record_error(S.err, err, errv);
    if (c == 0 && threadIdx.x == 0) {
        S.res->visited = nvisit;
        S.res->moved = nmoved;
        S.res->counter = seq;
        S.res->refine_at = -1; // refines in place
        if (S.xowner) *S.xcounter = seq;
    }
    if (c == 0 && S.xowner) xprev_store(S, pv);
}

// ---- dense kernels ---------------------------------------------------------

// zero state: every block's header {den 0, n_i} and x'beta 0 for its eras
__global__ void k_init_blocks(double* X, const int32_t* __restrict__ bstart, const int32_t* __restrict__ off,
                              const int32_t* __restrict__ n, int32_t N) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = bstart[i];
        X[b] = 0.0;
        X[b + 1] = static_cast<double>(n[i]);
        const int E = off[i + 1] - off[i];
        for (int q = 0; q < E; ++q) X[b + kBlockHeader + q] = 0.0;
    }
}

// xbeta_k = sum over drugs of row k in ascending j of beta_j, skipping
// zeros (engine.hpp:173-181), with the overflow guard (engine.hpp:70-74).
// snapshot := xbeta.
__global__ void k_dense_xb(double* X, double* snap, const int64_t* __restrict__ csr_ptr,
                           const int32_t* __restrict__ csr_col, const double* __restrict__ beta,
                           const int32_t* __restrict__ row_slot, int32_t K, DevErr* err) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double xb = 0.0;
        for (int64_t q = csr_ptr[k]; q < csr_ptr[k + 1]; ++q) {
            const double b = beta[csr_col[q]];
            if (b != 0.0) xb = __dadd_rn(xb, b);
        }
        if (!(fabs(xb) <= kXbBound)) record_error(err, DERR_OVERFLOW, fabs(xb));
        X[row_slot[k]] = xb;
        snap[k] = xb;
    }
}

// denominators: per subject, ascending sum of l*exp(x'beta) (engine.hpp:76-89)
__global__ void k_dense_den(double* X, const int32_t* __restrict__ len, const int32_t* __restrict__ off,
                            const int32_t* __restrict__ bstart, int32_t N, double* denc) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = bstart[i], k0 = off[i], k1 = off[i + 1];
        double total = 0.0;
        for (int k = k0; k < k1; ++k) total = __dadd_rn(total, lexp(len[k], X[b + kBlockHeader + (k - k0)]));
        X[b] = total;
        if (denc) denc[i] = total;
    }
}

// criterion snapshot of the cycle start rebuilt from beta at that point (a
// cycle the resident-beta sweep began and k_ccd finishes): k_dense_xb's sum
__global__ void k_snap_from_beta(double* snap, const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_col,
                                 const double* __restrict__ beta, int32_t K) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double xb = 0.0;
        for (int64_t q = csr_ptr[k]; q < csr_ptr[k + 1]; ++q) {
            const double b = beta[csr_col[q]];
            if (b != 0.0) xb = __dadd_rn(xb, b);
        }
        snap[k] = xb;
    }
}

// resident-beta sweep state <-> subject-block headers
__global__ void k_hdr_to_denc(const double* X, const int32_t* __restrict__ bstart, double* denc, int32_t N) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        denc[i] = X[bstart[i]];
}
__global__ void k_denc_to_hdr(double* X, const int32_t* __restrict__ bstart, const double* denc, int32_t N) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        X[bstart[i]] = denc[i];
}

__global__ void k_snapshot(const double* X, const int32_t* __restrict__ row_slot, double* snap, int32_t K) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        snap[k] = X[row_slot[k]];
}

// out[i] = X[idx[i]] (+ l*exp when len != nullptr): state_get's gathers
__global__ void k_gather_slots(const double* X, const int32_t* __restrict__ idx, const int32_t* __restrict__ len,
                               double* out, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = X[idx[i]];
        out[i] = len ? lexp(len[i], x) : x;
    }
}

__global__ void k_ll_partial(const double* X, const int32_t* __restrict__ row_slot, const int32_t* __restrict__ y,
                             const int32_t* __restrict__ bstart, int32_t K, int32_t N, double* partial, DevErr* err) {
    double lin = 0.0, lg = 0.0;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int yk = y[k];
        if (yk != 0) lin = __dadd_rn(lin, __dmul_rn(static_cast<double>(yk), X[row_slot[k]]));
    }
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const Subj sr = ld_hdr(X, bstart[i]);
        if (!(sr.den > 0.0)) record_error(err, DERR_LL_DEN_NONPOSITIVE, sr.den);
        lg = __dadd_rn(lg, __dmul_rn(static_cast<double>(sr.n), log(sr.den)));
    }
    __shared__ double sa[kLLThreads / 32], sb[kLLThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lin = __dadd_rn(lin, __shfl_xor_sync(0xffffffffu, lin, o));
        lg = __dadd_rn(lg, __shfl_xor_sync(0xffffffffu, lg, o));
    }
    if ((threadIdx.x & 31) == 0) {
        sa[threadIdx.x >> 5] = lin;
        sb[threadIdx.x >> 5] = lg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y2 = 0.0;
        for (int w = 0; w < kLLThreads / 32; ++w) {
            x = __dadd_rn(x, sa[w]);
            y2 = __dadd_rn(y2, sb[w]);
        }
        partial[2 * blockIdx.x] = x;
        partial[2 * blockIdx.x + 1] = y2;
    }
}

// block sum of (a, b) in a fixed order into partial[2 * block + slot] (slot
// 0: a, 1: b; the k_ll_final layout)
__device__ __forceinline__ void ll_block_sum(double v, double* partial, int slot) {
    __shared__ double sv[kLLThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0;
        for (int w = 0; w < kLLThreads / 32; ++w) x = __dadd_rn(x, sv[w]);
        partial[2 * blockIdx.x + slot] = x;
    }
}

// The fit's closing refresh and log-likelihood (solver.hpp:192-196:
// dense_recompute, then log_likelihood, engine.hpp:68-90,404-425) without
// rebuilding the subject blocks.  Pass 1, one thread per era: x'beta from the
// row-major copy (k_dense_xb's sum and overflow check) into the criterion
// snapshot (what the refresh leaves there) and the linear term.  Pass 2, one
// thread per subject: the denominator from the snapshot (k_dense_den's sum)
// and the log term.  The blocks are rebuilt from beta on the state's next
// use (bsccs_state::dense_pending).
__global__ void k_final_xb(const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_col,
                           const double* __restrict__ beta, const int32_t* __restrict__ y, int32_t K, double* snap,
                           double* partial, DevErr* err) {
    double lin = 0.0;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double xb = 0.0;
        for (int64_t q = csr_ptr[k]; q < csr_ptr[k + 1]; ++q) {
            const double b = beta[csr_col[q]];
            if (b != 0.0) xb = __dadd_rn(xb, b);
        }
        if (!(fabs(xb) <= kXbBound)) record_error(err, DERR_OVERFLOW, fabs(xb));
        snap[k] = xb;
        const int yk = y[k];
        if (yk != 0) lin = __dadd_rn(lin, __dmul_rn(static_cast<double>(yk), xb));
    }
    ll_block_sum(lin, partial, 0);
}
__global__ void k_final_den(const double* __restrict__ snap, const int32_t* __restrict__ len,
                            const int32_t* __restrict__ off, const int32_t* __restrict__ eps, int32_t N,
                            double* partial, DevErr* err) {
    double lg = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double total = 0.0;
        for (int k = off[i]; k < off[i + 1]; ++k) total = __dadd_rn(total, lexp(len[k], snap[k]));
        if (!(total > 0.0)) record_error(err, DERR_LL_DEN_NONPOSITIVE, total);
        lg = __dadd_rn(lg, __dmul_rn(static_cast<double>(eps[i]), log(total)));
    }
    ll_block_sum(lg, partial, 1);
}

// cold start (beta = 0) for the resident-beta sweep: the compact
// denominators sum l * exp(0) (k_dense_den's value); x'beta and the subject
// blocks are rebuilt from beta when an op reads them (x_stale)
__global__ void k_den_zero(const int32_t* __restrict__ len, const int32_t* __restrict__ off, int32_t N, double* denc) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double total = 0.0;
        for (int k = off[i]; k < off[i + 1]; ++k) total = __dadd_rn(total, lexp(len[k], 0.0));
        denc[i] = total;
    }
}

// cold start (beta = 0): x'beta = 0 in every era without reading the CSR
// (k_dense_den then sums l * exp(0))
__global__ void k_zero_xb(double* X, double* snap, const int32_t* __restrict__ row_slot, int32_t K) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        X[row_slot[k]] = 0.0;
        snap[k] = 0.0;
    }
}

// one warp, fixed order: lane l sums the partials b = l mod 32 ascending,
// then a butterfly
__global__ void k_ll_final(const double* partial, int n, DevResult* res) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    double x = 0.0, y = 0.0;
    for (int b = static_cast<int>(threadIdx.x); b < n; b += 32) {
        x = __dadd_rn(x, partial[2 * b]);
        y = __dadd_rn(y, partial[2 * b + 1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
        y = __dadd_rn(y, __shfl_xor_sync(0xffffffffu, y, o));
    }
    if (threadIdx.x == 0) {
        res->ll_linear = x;
        res->ll_logden = y;
    }
}

// ---- dataset build kernels -------------------------------------------------

// bsccs_dataset_create with subjects == NULL: each pair's subject derived
// from its row (build_dataset pushes the era's owner with the era,
// dataset.hpp:134-136): the era -> subject table, then one gather per pair.
// Offsets that are not monotone or out of range are clamped here and
// rejected by k_validate_small; a row out of range gets subject -1 (k_pair_meta).
__global__ void k_era_owner(const int32_t* __restrict__ off, int32_t N, int32_t K, int32_t* esub) {
    for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < N;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int k1 = min(K, off[s + 1]);
        for (int k = max(0, off[s]); k < k1; ++k) esub[k] = static_cast<int32_t>(s);
    }
}
__global__ void k_subject_of_row(const int32_t* __restrict__ rows, const int32_t* __restrict__ esub, int32_t K,
                                 int64_t nnz, int32_t* subj) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = rows[p];
        subj[p] = (r >= 0 && r < K) ? esub[r] : -1;
    }
}

__global__ void k_interleave(const int32_t* rows, const int32_t* subjects, int2* pairs, int64_t nnz) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        pairs[p] = make_int2(rows[p], subjects[p]);
}

// column of every pair (upper_bound on col_ptr), row histogram, and the
// structural checks of build_dataset (dataset.hpp:135-175): row in range,
// subject in range and owning the row, rows strictly ascending in a column.
// Per pair: its column (for the row-major copy), and the build_dataset
// checks (dataset.hpp:135-175): row / subject in range, the subject owns
// the row, rows strictly ascending within the column.  Each block walks a
// contiguous pair range and finds the column of its first pair once; the
// threads then advance their column monotonically (no per-pair search, no
// atomics -- the CSR row pointers come from the sorted keys afterwards).
__global__ void k_pair_meta(const int2* pairs, const int64_t* __restrict__ col_ptr, int32_t J,
                            const int32_t* __restrict__ off, int32_t N, int32_t K, int64_t nnz, int32_t* col_of,
                            int* bad) {
    const int64_t per = (nnz + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = static_cast<int64_t>(blockIdx.x) * per, b1 = min(nnz, b0 + per);
    if (b0 >= b1) return;
    __shared__ int jc0;
    if (threadIdx.x == 0) {
        int lo = 0, hi = J; // first j with col_ptr[j+1] > b0
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (col_ptr[mid + 1] > b0) hi = mid;
            else lo = mid + 1;
        }
        jc0 = lo;
    }
    __syncthreads();
    int jc = jc0;
    int nbad = 0;
    for (int64_t p = b0 + threadIdx.x; p < b1; p += blockDim.x) {
        while (col_ptr[jc + 1] <= p) ++jc;
        col_of[p] = jc;
        const int2 pr = pairs[p];
        bool ok = pr.x >= 0 && pr.x < K && pr.y >= 0 && pr.y < N;
        if (ok) ok = off[pr.y] <= pr.x && pr.x < off[pr.y + 1];
        if (ok && p > col_ptr[jc]) ok = pairs[p - 1].x < pr.x;
        nbad |= ok ? 0 : 1;
    }
    if (__syncthreads_or(nbad) && threadIdx.x == 0) atomicOr(bad, 1);
}

// CSR row pointers from the row-sorted keys: csr_ptr[k] = first sorted
// position with row >= k (= the exclusive scan of the row counts).
__global__ void k_csr_ptr(const int32_t* __restrict__ sorted_rows, int64_t nnz, int32_t K, int64_t* csr_ptr) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p <= nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = p < nnz ? sorted_rows[p] : K;
        const int rp = p > 0 ? sorted_rows[p - 1] : -1;
        for (int k = rp + 1; k <= r; ++k) csr_ptr[k] = p;
    }
}

__global__ void k_validate_small(const int32_t* off, int32_t N, const int32_t* len, int32_t K, int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N || i < K;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < N && off[i + 1] <= off[i]) atomicOr(bad, 2);
        if (i < K && len[i] <= 0) atomicOr(bad, 4);
    }
}

__global__ void k_subject_weight(const int32_t* off, const int64_t* csr_ptr, int32_t N, long long* w) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t a = off[i], b = off[i + 1];
        w[i] = static_cast<long long>(b - a) + (csr_ptr[b] - csr_ptr[a]);
    }
}

// cta_subj[c] = first subject whose exclusive weight prefix >= ceil(total*c/C)
__global__ void k_cta_bounds(const long long* excl, int32_t N, int C, const int32_t* off, int32_t* cta_subj,
                             int32_t* cta_era) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > C) return;
    const long long total = excl[N];
    int s;
    if (c == C) {
        s = N;
    } else {
        const long long target = (total * c + C - 1) / C;
        int lo = 0, hi = N;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (excl[mid] >= target) hi = mid;
            else lo = mid + 1;
        }
        s = lo;
    }
    cta_subj[c] = s;
    cta_era[c] = off[s];
}

__global__ void k_split(const int2* pairs, const int64_t* col_ptr, int32_t J, const int32_t* cta_subj, int C,
                        int64_t* split) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(J) * (C + 1)) return;
    const int j = static_cast<int>(t / (C + 1));
    const int c = static_cast<int>(t % (C + 1));
    int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
    const int target = cta_subj[c];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pairs[mid].y >= target) hi = mid;
        else lo = mid + 1;
    }
    split[t] = lo;
}

// (p0, p1) of every CTA's slice, laid out per CTA in visit order
__global__ void k_build_vsplit(const int64_t* __restrict__ split, const int32_t* __restrict__ visit, int V, int C,
                               longlong2* vsplit) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(V) * C) return;
    const int c = static_cast<int>(t / V), idx = static_cast<int>(t % V);
    const int64_t* row = split + static_cast<int64_t>(visit[idx]) * (C + 1) + c;
    vsplit[t] = make_longlong2(row[0], row[1]);
}

// subject runs per column (heads of the CSC pair list)
// largest per-CTA slice of any column (decides whether sweeps need the
// streamed path)
__global__ void k_max_slice(const int64_t* __restrict__ split, int32_t J, int C, int* out) {
    const int64_t n = static_cast<int64_t>(J) * C;
    int m = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = i / C, c = i % C;
        const int64_t a = split[j * (C + 1) + c], b = split[j * (C + 1) + c + 1];
        m = max(m, static_cast<int>(min(b - a, static_cast<int64_t>(1 << 30))));
    }
    atomicMax(out, m);
}

__global__ void k_col_runs(const int2* pairs, const int64_t* col_ptr, int32_t* runs, int J) {
    const int j = blockIdx.x;
    if (j >= J) return;
    __shared__ int part[256];
    int acc = 0;
    for (int64_t p = col_ptr[j] + threadIdx.x; p < col_ptr[j + 1]; p += blockDim.x)
        acc += (p == col_ptr[j] || pairs[p - 1].y != pairs[p].y) ? 1 : 0;
    part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < static_cast<int>(blockDim.x); ++i) t += part[i];
        runs[j] = t;
    }
}

__global__ void k_ydotx(const int2* pairs, const int64_t* col_ptr, const int32_t* y, double* out, int J) {
    const int j = blockIdx.x;
    if (j >= J) return;
    __shared__ long long part[256];
    long long acc = 0;
    for (int64_t p = col_ptr[j] + threadIdx.x; p < col_ptr[j + 1]; p += blockDim.x) acc += y[pairs[p].x];
    part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < static_cast<int>(blockDim.x); ++i) t += part[i];
        out[j] = static_cast<double>(t);
    }
}

// ---- subject blocks (engine.h) --------------------------------------------
// Blocks are packed per chunk of kBlockChunk subjects, each chunk from a line
// boundary (chunks pack in parallel; the gaps cost < 2%).  A block of
// z = 2 + E slots starts on an even slot (its 16-B header load); if z <= 16
// it never straddles a 16-slot (128-B) line, a longer one starts on a line.
__device__ __forceinline__ long long pack_at(long long c, int z) {
    c = (c + 1) & ~1ll;
    const long long in_line = c & (kLineSlots - 1);
    if (z > kLineSlots ? in_line != 0 : in_line + z > kLineSlots) c = (c + kLineSlots - 1) & ~(kLineSlots - 1ll);
    return c;
}

__global__ void k_block_chunks(const int32_t* __restrict__ off, int32_t N, long long* chunk_slots, int64_t nchunks) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nchunks;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s1 = min(static_cast<int64_t>(N), (t + 1) * kBlockChunk);
        long long c = 0;
        for (int64_t i = t * kBlockChunk; i < s1; ++i) {
            const int z = kBlockHeader + (off[i + 1] - off[i]);
            c = pack_at(c, z) + z;
        }
        chunk_slots[t] = (c + kLineSlots - 1) & ~(kLineSlots - 1ll);
    }
}

__global__ void k_block_place(const int32_t* __restrict__ off, int32_t N, const long long* __restrict__ chunk_base,
                              int64_t nchunks, int32_t* bstart, int32_t* row_slot) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nchunks;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s1 = min(static_cast<int64_t>(N), (t + 1) * kBlockChunk);
        const long long base = chunk_base[t];
        long long c = 0;
        for (int64_t i = t * kBlockChunk; i < s1; ++i) {
            const int k0 = off[i], E = off[i + 1] - k0, z = kBlockHeader + E;
            c = pack_at(c, z);
            bstart[i] = static_cast<int32_t>(base + c);
            for (int q = 0; q < E; ++q) row_slot[k0 + q] = static_cast<int32_t>(base + c + kBlockHeader + q);
            c += z;
        }
    }
}

// The sweep's pair records: {era slot, block slot, era length, subject index
// within the owning CTA's range} (the CTA that owns the subject owns the
// pair's slice: splits are subject-aligned).
__global__ void k_build_pq(const int2* __restrict__ pairs, int64_t nnz, const int32_t* __restrict__ row_slot,
                           const int32_t* __restrict__ bstart, const int32_t* __restrict__ len,
                           const int32_t* __restrict__ cta_subj, int C, int4* pq) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int2 pr = pairs[p];
        int lo = 0, hi = C + 1; // first c with cta_subj[c] > subject
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cta_subj[mid] > pr.y) hi = mid;
            else lo = mid + 1;
        }
        pq[p] = make_int4(row_slot[pr.x], bstart[pr.y], len[pr.x], pr.y - cta_subj[lo - 1]);
    }
}

// ---- pair records of the resident-beta sweep (engine.h RRec) ---------------
// The CSR sort carries each pair's CSC position with its column, so the
// records are written per era from its (contiguous) drug list: one 32-B
// store per pair, no per-pair search.
// Each CSC position with its run flags in bits 30 / 31 (the sort carries
// them to the CSR order, where k_build_rq puts them into the record): the
// pair heads a run of its subject in its column (the previous pair is in
// another column or another subject's), the next pair continues the run.
// CTA slices are subject-aligned, so these are the per-slice run flags.
constexpr uint32_t kPosMask = (1u << 30) - 1;
__global__ void k_iota_flags(const int2* __restrict__ pairs, const int32_t* __restrict__ col_of, int64_t nnz,
                             uint32_t* out) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int s = pairs[p].y, j = col_of[p];
        const bool head = p == 0 || col_of[p - 1] != j || pairs[p - 1].y != s;
        const bool cont = p + 1 < nnz && col_of[p + 1] == j && pairs[p + 1].y == s;
        out[p] = static_cast<uint32_t>(p) | (head ? 1u << 30 : 0u) | (cont ? 1u << 31 : 0u);
    }
}
// csr_col holds each CSR entry's CSC position (and run flags) after the sort: keep it in pos,
// and the entry's column in csr_col -- found by binary search in col_ptr
// (L1-resident) rather than a random gather of the per-pair column array
// (the search starts from a bucket table: the column holding position
// b << kPosBucketBits, so a column of typical size takes one or two steps)
constexpr int kPosBucketBits = 14;
__global__ void k_pos_buckets(const int64_t* __restrict__ col_ptr, int32_t J, int64_t nnz, int32_t* bucket) {
    const int64_t nb = ((nnz - 1) >> kPosBucketBits) + 2;
    for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t p = min(b << kPosBucketBits, nnz - 1);
        int lo = 0, hi = J; // last column j with col_ptr[j] <= p
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (col_ptr[mid] <= p) lo = mid;
            else hi = mid;
        }
        bucket[b] = lo;
    }
}
__global__ void k_pos_col(int32_t* csr_col, const int64_t* __restrict__ col_ptr, const int32_t* __restrict__ bucket,
                          int64_t nnz, uint32_t* pos) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nnz;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t raw = static_cast<uint32_t>(csr_col[q]);
        const uint32_t p = raw & kPosMask;
        pos[q] = raw; // (with the run flags)
        const int b = static_cast<int>(p >> kPosBucketBits);
        int lo = __ldg(bucket + b), hi = __ldg(bucket + b + 1) + 1; // last column j in [lo, hi) with col_ptr[j] <= p
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(col_ptr + mid) <= static_cast<int64_t>(p)) lo = mid;
            else hi = mid;
        }
        csr_col[q] = lo;
    }
}
// the criterion's compact CSR: drugs per era (u8) and the drugs (u16)
__global__ void k_compact_csr(const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_col, int32_t K,
                              int64_t nnz, uint8_t* edeg, uint16_t* ecol) {
    const int64_t n = max(static_cast<int64_t>(K), nnz);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < K) edeg[i] = static_cast<uint8_t>(csr_ptr[i + 1] - csr_ptr[i]);
        if (i < nnz) ecol[i] = static_cast<uint16_t>(csr_col[i]);
    }
}
// overflow entries of one era's pairs (each pair's list padded to 8)
__device__ __forceinline__ long long era_overflow(int deg) {
    return deg - 1 > kRInline ? static_cast<long long>(deg) * ((deg - 1 - kRInline + 7) & ~7) : 0;
}

// per subject: overflow drug entries of its pairs; bad |= 1 when an era has
// more than kRMaxOthers + 1 drugs or n_i exceeds the record's field
__global__ void k_rq_count(const int32_t* __restrict__ off, const int32_t* __restrict__ events,
                           const int64_t* __restrict__ csr_ptr, int32_t N, long long* cnt, int* bad, int* max_deg) {
    for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < N;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        long long o = 0, md = 0;
        int b = events[s] > kRMaxEvents || events[s] < 0;
        for (int k = off[s]; k < off[s + 1]; ++k) {
            const long long deg = csr_ptr[k + 1] - csr_ptr[k];
            if (deg - 1 > kRMaxOthers) b = 1;
            o += era_overflow(static_cast<int>(deg)); // lists padded to 16 B
            md = deg > md ? deg : md;
        }
        cnt[s] = o;
        if (b) atomicOr(bad, 1);
        atomicMax(max_deg, static_cast<int>(md < (1 << 30) ? md : (1 << 30)));
    }
}
// subject of every era (one thread per subject writes its eras)
__global__ void k_era_subject(const int32_t* __restrict__ off, int32_t N, int32_t* esub) {
    for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < N;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x)
        for (int k = off[s]; k < off[s + 1]; ++k) esub[k] = static_cast<int32_t>(s);
}

// one 32-B record in a single 256-bit store (sm_100: STG.256 -- one L2
// request per record instead of two for the scattered writes)
__device__ __forceinline__ void st_global_256(void* p, int4 a, int4 b) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
                 "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
}

// The pair records, one thread per era: the era's drug list (contiguous in
// the CSR) gives every pair's other drugs; each record is one 32-B store at
// the pair's CSC position.  Overflow lists: the subject's offset (scan over
// subjects) plus its earlier eras' (only subjects that have any).
__global__ void k_build_rq(const int32_t* __restrict__ off, const int32_t* __restrict__ esub,
                           const int32_t* __restrict__ events, const int32_t* __restrict__ len,
                           const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_col,
                           const uint32_t* __restrict__ pos, const int32_t* __restrict__ cta_subj, int C,
                           const long long* __restrict__ ovb, int32_t K, int32_t J, RRec* rq, uint16_t* rovf) {
    extern __shared__ int cs[]; // [C + 1] the CTA subject ranges (searched per era)
    for (int i = threadIdx.x; i <= C; i += blockDim.x) cs[i] = cta_subj[i];
    __syncthreads();
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t q0 = csr_ptr[k];
        const int deg = static_cast<int>(csr_ptr[k + 1] - q0);
        if (deg == 0) continue;
        const int s = esub[k];
        int lo = 0, hi = C + 1; // first c with cta_subj[c] > s
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cs[mid] > s) hi = mid;
            else lo = mid + 1;
        }
        const int ls = s - cs[lo - 1];
        const int n = events[s];
        const int lk = len[k];
        if (deg - 1 <= kRInline) { // no overflow list: the record is built in registers
            // the era's drugs, the unit drug J past the end
            // (every load issued before the first store: one round trip per era)
            unsigned c[kRInline + 1], pp[kRInline + 1];
#pragma unroll
            for (int b = 0; b <= kRInline; ++b) {
                c[b] = b < deg ? static_cast<unsigned>(csr_col[q0 + b]) : static_cast<unsigned>(J);
                pp[b] = b < deg ? pos[q0 + b] : 0u; // CSC position | run flags << 30
            }
#pragma unroll
            for (int a = 0; a <= kRInline; ++a) {
                if (a >= deg) break;
                unsigned o[kRInline]; // the era's drugs without drug a, in order
#pragma unroll
                for (int i = 0; i < kRInline; ++i) o[i] = i < a ? c[i] : c[i + 1];
                const int4 head = make_int4(ls, lk, (deg - 1) | static_cast<int>((pp[a] >> 30) << 8) | (n << 16), 0);
                const int4 tail = make_int4(static_cast<int>(o[0] | (o[1] << 16)), static_cast<int>(o[2] | (o[3] << 16)),
                                            static_cast<int>(o[4] | (o[5] << 16)), static_cast<int>(o[6] | (o[7] << 16)));
                st_global_256(rq + (pp[a] & kPosMask), head, tail);
            }
            continue;
        }
        long long ov = ovb[s];
        if (ovb[s + 1] != ov)
            for (int k2 = off[s]; k2 < k; ++k2) ov += era_overflow(static_cast<int>(csr_ptr[k2 + 1] - csr_ptr[k2]));
        for (int a = 0; a < deg; ++a) {
            RRec r;
            r.ls = ls;
            r.len = lk;
            const uint32_t pa = pos[q0 + a];
            r.meta = (deg - 1) | static_cast<int>((pa >> 30) << 8) | (n << 16); // run flags: head bit 8, cont bit 9
            r.ovf = deg - 1 > kRInline ? static_cast<int32_t>(ov) : 0;
            int i = 0;
            for (int b = 0; b < deg; ++b) {
                if (b == a) continue;
                const uint16_t d = static_cast<uint16_t>(csr_col[q0 + b]);
                if (i < kRInline) r.o[i] = d;
                else rovf[ov + (i - kRInline)] = d;
                ++i;
            }
            for (; i < kRInline; ++i) r.o[i] = static_cast<uint16_t>(J); // the unit drug: exp(beta) = 1
            if (deg - 1 > kRInline) { // pad the overflow list to a multiple of 8 (one 16-B load per 8)
                const int ext = (deg - 1 - kRInline + 7) & ~7;
                for (int t = deg - 1 - kRInline; t < ext; ++t) rovf[ov + t] = static_cast<uint16_t>(J);
                ov += ext;
            }
            rq[pa & kPosMask] = r;
        }
    }
}

// resident-beta sweep enabled (BSCCS_SWEEP=classic keeps every sweep on k_ccd)
bool rcd_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("BSCCS_SWEEP");
        return !(e && std::string(e) == "classic");
    }();
    return on;
}

std::atomic<int> g_sweep_kind{0};       // tests: 1 forces k_ccd
std::atomic<double> g_beta_limit{0.0};  // tests: lower k_rcd's |beta| bound
std::atomic<int> g_last_sweep{0};
std::atomic<int> g_last_rcd_shape{0};

// Small pinned result blocks for the per-state D2H of kernel scalars.
struct PinnedResults {
    std::mutex m;
    std::vector<DevResult*> free_list;
};
PinnedResults g_pinned;

DevResult* pinned_result() {
    std::lock_guard<std::mutex> lk(g_pinned.m);
    if (g_pinned.free_list.empty()) {
        DevResult* block = nullptr;
        CUDA_TRY(cudaMallocHost(&block, sizeof(DevResult) * 64));
        for (int i = 0; i < 64; ++i) g_pinned.free_list.push_back(block + i);
    }
    DevResult* r = g_pinned.free_list.back();
    g_pinned.free_list.pop_back();
    return r;
}

void release_pinned_result(DevResult* r) {
    if (!r) return;
    std::lock_guard<std::mutex> lk(g_pinned.m);
    g_pinned.free_list.push_back(r);
}

void sync_and_check(bsccs_state* st) {
    CUDA_TRY(cudaStreamSynchronize(st->stream));
    CUDA_TRY(cudaGetLastError());
}

void check_err_block(bsccs_state* st) {
    DevErr e;
    CUDA_TRY(cudaMemcpyAsync(&e, st->err, sizeof e, cudaMemcpyDeviceToHost, st->stream));
    CUDA_TRY(cudaStreamSynchronize(st->stream));
    if (e.code != 0) {
        CUDA_TRY(cudaMemsetAsync(st->err, 0, sizeof(DevErr), st->stream));
        CUDA_TRY(cudaStreamSynchronize(st->stream));
        throw_device_error(e.code, e.value);
    }
}


} // namespace

void throw_device_error(int code, double value) {
    char buf[256];
    switch (code) {
    case DERR_OVERFLOW:
        std::snprintf(buf, sizeof buf,
                      "linear predictor overflow: |x'beta| reached %f (bound 700.000000); the fit has diverged",
                      value);
        numeric_error(buf);
    case DERR_DEN_NONPOSITIVE:
        internal_error("fused reduction: nonpositive subject denominator");
    case DERR_STEP_NONFINITE:
        numeric_error("sparse_delta_update: non-finite step");
    case DERR_FLAT_NO_PRIOR:
        numeric_error("undefined Newton step: flat likelihood direction with no prior");
    case DERR_POS_CURVATURE:
        internal_error("penalized_step: positive likelihood curvature");
    case DERR_LL_DEN_NONPOSITIVE:
        internal_error("log_likelihood: nonpositive subject denominator");
    case DERR_SUM_RANGE:
        numeric_error("exact all-reduce: a partial sum outside [0, 2^43) or a total at or above 2^48");
    case DERR_XCHG_TIMEOUT:
        internal_error("exact all-reduce: a participant stopped publishing (a peer rank failed or exited); "
                       "the group must be recreated");

    default:
        std::snprintf(buf, sizeof buf, "device error code %d", code);
        internal_error(buf);
    }
}

constexpr int kMaxSweepSmem = 225 * 1024; // opt-in dynamic shared memory per CTA (227 KB less static use)

void ensure_kernel_attrs(int device) {
    static std::atomic<unsigned> done{0};
    if (device < 32 && (done.load() & (1u << device))) return;
    for (void* fn : {reinterpret_cast<void*>(t3::k_ccd<false, false>), reinterpret_cast<void*>(t3::k_ccd<false, true>),
                     reinterpret_cast<void*>(t3::k_ccd<true, false>), reinterpret_cast<void*>(t3::k_ccd<true, true>),
                     reinterpret_cast<void*>(t1::k_ccd<false, false>), reinterpret_cast<void*>(t1::k_ccd<true, false>),
                     reinterpret_cast<void*>(t1::k_ccd<false, true>), reinterpret_cast<void*>(t1::k_ccd<true, true>),
                     reinterpret_cast<void*>(r3::k_rcd<false>), reinterpret_cast<void*>(r3::k_rcd<true>),
                     reinterpret_cast<void*>(r2::k_rcd<false>), reinterpret_cast<void*>(r2::k_rcd<true>),
                     reinterpret_cast<void*>(r1::k_rcd<false>), reinterpret_cast<void*>(r1::k_rcd<true>)})
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSweepSmem));
    if (device < 32) done.fetch_or(1u << device);
}

int default_ctas(int device) {
    // one persistent CTA per SM (launch bounds force 1 resident CTA of 512)
    ensure_kernel_attrs(device);
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, t3::k_ccd<false, true>, kSweepThreads,
                                                           sizeof(t3::Smem)));
    if (per_sm < 1) internal_error("sweep kernel cannot be resident");
    return sm_count(device);
}

// ---------------------------------------------------------------------------
namespace {

// Allocates the dataset's device arrays (sizes and CTA count already set).
void alloc_dataset(bsccs_dataset* ds) {
    const int C = ds->ctas;
    const int32_t N = ds->N, K = ds->K, J = ds->J;
    const int64_t nnz = ds->nnz;
    int64_t& B = ds->device_bytes;
    CUDA_TRY(cudaStreamCreateWithFlags(&ds->stream, cudaStreamNonBlocking));
    cudaStream_t s = ds->stream;
    ds->pairs = dalloc<int2>(nnz, B, s);
    // pair records of the resident-beta sweep, allocated before the build's
    // temporaries (a stable allocation order lets the pool reuse blocks
    // across dataset rebuilds); freed again if the dataset does not qualify
    if (rcd_enabled() && nnz > 0 && nnz < (1ll << 30) && J < 65535) { // u16 drugs, index J the unit drug; 30-bit positions
        ds->rq = dalloc<RRec>(nnz, B, s);
        if (reinterpret_cast<uintptr_t>(ds->rq) % 32 != 0) internal_error("pair records not 32-B aligned (STG.256)");
        ds->edeg = dalloc<uint8_t>(static_cast<int64_t>(K) + 32, B, s);
        ds->ecol = dalloc<uint16_t>(nnz + 16, B, s);
    }
    ds->row_slot = dalloc<int32_t>(K, B, s);
    ds->bstart = dalloc<int32_t>(N, B, s);
    ds->col_ptr = dalloc<int64_t>(J + 1, B, s);
    ds->split = dalloc<int64_t>(static_cast<int64_t>(J) * (C + 1), B, s);
    ds->cta_era = dalloc<int32_t>(C + 1, B, s);
    ds->cta_subj = dalloc<int32_t>(C + 1, B, s);
    ds->subject_offsets = dalloc<int32_t>(N + 1, B, s);
    ds->events_per_subject = dalloc<int32_t>(N, B, s);
    ds->era_lengths = dalloc<int32_t>(K, B, s);
    ds->event_counts = dalloc<int32_t>(K, B, s);
    ds->csr_ptr = dalloc<int64_t>(static_cast<int64_t>(K) + 1, B, s);
    ds->csr_col = dalloc<int32_t>(nnz, B, s);
    ds->y_dot_x = dalloc<double>(J, B, s);
    ds->col_nonempty = dalloc<uint8_t>(J, B, s);
    ds->col_runs = dalloc<int32_t>(J, B, s);
}

} // namespace

// Device half of the dataset build.  On entry the small arrays (col_ptr,
// subject_offsets, events_per_subject, era_lengths, event_counts) are on the
// device, ds->col_ptr_h holds the column pointers, and d_rows / d_subj (owned
// here, freed on return) hold the CSC pair arrays.  Validates the
// build_dataset invariants (dataset.hpp:135-175), builds the interleaved
// pairs, the row-major copy, the CTA ranges and the per-column splits.
// BSCCS_BUILD_TIMING=1: host-side phase times of the dataset build on stderr
// (each phase synchronised; profiling only)
struct BuildTimer {
    bool on;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t;
    explicit BuildTimer(cudaStream_t st) : on([] {
        const char* e = std::getenv("BSCCS_BUILD_TIMING");
        return e && e[0] == '1';
    }()), s(st), t(std::chrono::steady_clock::now()) {}
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[build] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

void finish_dataset(bsccs_dataset* ds, int32_t* d_rows, int32_t* d_subj, const int64_t* y_dot_x_global,
                    const int64_t* col_nnz_global, cudaEvent_t era_ready) {
    BuildTimer bt(ds->stream);
    bt.mark("enter");
    const int C = ds->ctas;
    const int32_t N = ds->N, K = ds->K, J = ds->J;
    const int64_t nnz = ds->nnz;
    const int sms = sm_count(ds->device);
    cudaStream_t s = ds->stream;
    int64_t scratch_bytes = 0;
    int32_t* d_col = dalloc<int32_t>(nnz, scratch_bytes, s);
    long long* d_w = dalloc<long long>(static_cast<int64_t>(N) + 1, scratch_bytes, s);
    long long* d_excl = dalloc<long long>(static_cast<int64_t>(N) + 1, scratch_bytes, s);
    int* d_bad = dalloc<int>(1, scratch_bytes, s);
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
    // resident-beta sweep records (allocated with the dataset, alloc_dataset)
    bool want_rq = ds->rq != nullptr;
    uint32_t* d_iota = nullptr; // CSC positions, sorted by row with the keys
    if (nnz > 0) {
        k_interleave<<<grid_for(nnz, 256, sms), 256, 0, s>>>(d_rows, d_subj, ds->pairs, nnz);
        k_pair_meta<<<grid_for(nnz, 256, sms), 256, 0, s>>>(ds->pairs, ds->col_ptr, J, ds->subject_offsets, N, K,
                                                           nnz, d_col, d_bad);
    }
    // CSR: stable sort by row, row pointers from the sorted keys
    {
        size_t tmp_bytes = 0;
        size_t sort_bytes = 0;
        int end_bit = 1;
        while ((1ll << end_bit) < static_cast<long long>(K)) ++end_bit;
        // resident-beta sweep records need each CSR entry's CSC position:
        // the sort then carries positions, the columns are gathered after
        if (want_rq) {
            d_iota = dalloc<uint32_t>(nnz, scratch_bytes, s);
            k_iota_flags<<<grid_for(nnz, 256, sms), 256, 0, s>>>(ds->pairs, d_col, nnz, d_iota);
            count_launches(1);
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, d_rows, d_subj, d_iota,
                                                     reinterpret_cast<uint32_t*>(ds->csr_col), nnz, 0, end_bit, s));
        } else if (nnz > 0)
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, d_rows, d_subj, d_col, ds->csr_col, nnz, 0,
                                                     end_bit, s));
        size_t scan2 = 0;
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan2, d_w, d_excl, N + 1, s));
        const size_t tb = std::max(std::max(tmp_bytes, sort_bytes), scan2);
        unsigned char* tmp = dalloc<unsigned char>(static_cast<int64_t>(std::max<size_t>(tb, 16)), scratch_bytes, s);
        if (want_rq) {
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, d_rows, d_subj, d_iota,
                                                     reinterpret_cast<uint32_t*>(ds->csr_col), nnz, 0, end_bit, s));
            // d_rows (the consumed keys) receives the CSC positions
            const int64_t nbk = ((nnz - 1) >> kPosBucketBits) + 2;
            int32_t* d_bk = dalloc<int32_t>(nbk, scratch_bytes, s);
            k_pos_buckets<<<grid_for(nbk, 256, sms), 256, 0, s>>>(ds->col_ptr, J, nnz, d_bk);
            k_pos_col<<<grid_for(nnz, 256, sms), 256, 0, s>>>(ds->csr_col, ds->col_ptr, d_bk, nnz,
                                                               reinterpret_cast<uint32_t*>(d_rows));
            count_launches(2);
            dfree(d_bk, s);
            dfree(d_iota, s);
        } else if (nnz > 0) {
            // keys: rows (consumed); d_subj is free after interleave and
            // receives the sorted keys
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, d_rows, d_subj, d_col, ds->csr_col, nnz, 0,
                                                     end_bit, s));
        }
        bt.mark("sort");
        k_csr_ptr<<<grid_for(nnz + 1, 256, sms), 256, 0, s>>>(d_subj, nnz, K, ds->csr_ptr);
        // the era arrays may still be arriving on a side stream: the pair-side
        // build above overlapped their upload
        if (era_ready) CUDA_TRY(cudaStreamWaitEvent(s, era_ready, 0));
        k_validate_small<<<grid_for(std::max<int64_t>(N, K), 256, sms), 256, 0, s>>>(ds->subject_offsets, N,
                                                                                 ds->era_lengths, K, d_bad);
        // nnz-balanced CTA subject ranges
        k_subject_weight<<<grid_for(N, 256, sms), 256, 0, s>>>(ds->subject_offsets, ds->csr_ptr, N, d_w);
        CUDA_TRY(cudaMemsetAsync(d_w + N, 0, sizeof(long long), s));
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, scan2, d_w, d_excl, N + 1, s));
        k_cta_bounds<<<(C + 1 + 127) / 128, 128, 0, s>>>(d_excl, N, C, ds->subject_offsets, ds->cta_subj,
                                                         ds->cta_era);
        k_col_runs<<<J, 256, 0, s>>>(ds->pairs, ds->col_ptr, ds->col_runs, J);
        const int64_t nsplit = static_cast<int64_t>(J) * (C + 1);
        k_split<<<static_cast<int>((nsplit + 255) / 256), 256, 0, s>>>(ds->pairs, ds->col_ptr, J, ds->cta_subj, C,
                                                                        ds->split);
        bt.mark("csr, cta ranges, split");
        // subject blocks and the sweep's pair records (engine.h)
        {
            const int64_t nch = (static_cast<int64_t>(N) + kBlockChunk - 1) / kBlockChunk;
            int64_t b3 = 0;
            long long* d_cs = dalloc<long long>(nch + 1, b3, s);
            long long* d_cb = dalloc<long long>(nch + 1, b3, s);
            CUDA_TRY(cudaMemsetAsync(d_cs + nch, 0, sizeof(long long), s));
            k_block_chunks<<<grid_for(nch, 128, sms), 128, 0, s>>>(ds->subject_offsets, N, d_cs, nch);
            size_t sb = 0;
            CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, sb, d_cs, d_cb, nch + 1, s));
            unsigned char* tmp2 = dalloc<unsigned char>(static_cast<int64_t>(std::max<size_t>(sb, 16)), b3, s);
            CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp2, sb, d_cs, d_cb, nch + 1, s));
            long long total = 0;
            CUDA_TRY(cudaMemcpyAsync(&total, d_cb + nch, sizeof(long long), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (total >= (1ll << 31) - kLineSlots)
                input_error("dataset: eras plus subject headers exceed the 32-bit slot range");
            ds->nslots = total;
            k_block_place<<<grid_for(nch, 128, sms), 128, 0, s>>>(ds->subject_offsets, N, d_cb, nch, ds->bstart,
                                                                  ds->row_slot);
            count_launches(3);
            dfree(tmp2, s);
            dfree(d_cs, s);
            dfree(d_cb, s);
        }
        bt.mark("subject blocks, pq");
        if (want_rq) { // resident-beta sweep pair records (engine.h RRec)
            int64_t b4 = 0;
            long long* d_oc = dalloc<long long>(static_cast<int64_t>(N) + 1, b4, s);
            long long* d_ob = dalloc<long long>(static_cast<int64_t>(N) + 1, b4, s);
            int* d_rbad = dalloc<int>(2, b4, s); // [0] bad, [1] largest era
            CUDA_TRY(cudaMemsetAsync(d_rbad, 0, 2 * sizeof(int), s));
            CUDA_TRY(cudaMemsetAsync(d_oc + N, 0, sizeof(long long), s));
            k_rq_count<<<grid_for(N, 256, sms), 256, 0, s>>>(ds->subject_offsets, ds->events_per_subject, ds->csr_ptr,
                                                             N, d_oc, d_rbad, d_rbad + 1);
            size_t sb = 0;
            CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, sb, d_oc, d_ob, N + 1, s));
            unsigned char* tmp3 = dalloc<unsigned char>(static_cast<int64_t>(std::max<size_t>(sb, 16)), b4, s);
            CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp3, sb, d_oc, d_ob, N + 1, s));
            long long novf = 0;
            int rbad[2] = {0, 0};
            CUDA_TRY(cudaMemcpyAsync(&novf, d_ob + N, sizeof(long long), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(rbad, d_rbad, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            bt.mark("rq: count, scan");
            if (!rbad[0] && novf < (1ll << 31)) {
                ds->novf = novf;
                ds->max_deg = std::max(1, rbad[1]);
                ds->rovf = dalloc<uint16_t>(std::max<long long>(novf, 8), ds->device_bytes, s);
                int64_t b5 = 0;
                int32_t* d_esub = nnz >= K ? d_col : dalloc<int32_t>(K, b5, s); // d_col is free by now
                k_era_subject<<<grid_for(N, 256, sms), 256, 0, s>>>(ds->subject_offsets, N, d_esub);
                const int g_rq = static_cast<int>(std::min<int64_t>((static_cast<int64_t>(K) + 255) / 256, 1 << 20));
                k_build_rq<<<g_rq, 256, sizeof(int) * (C + 1), s>>>(ds->subject_offsets, d_esub, ds->events_per_subject,
                                                ds->era_lengths, ds->csr_ptr, ds->csr_col,
                                                reinterpret_cast<const uint32_t*>(d_rows), ds->cta_subj, C, d_ob, K, J,
                                                ds->rq, ds->rovf);
                if (d_esub != d_col) dfree(d_esub, s);
                count_launches(1);
                bt.mark("rq: records");
                CUDA_TRY(cudaMemsetAsync(ds->edeg, 0, static_cast<size_t>(K) + 32, s));
                CUDA_TRY(cudaMemsetAsync(ds->ecol, 0, sizeof(uint16_t) * (nnz + 16), s));
                k_compact_csr<<<grid_for(std::max<int64_t>(K, nnz), 256, sms), 256, 0, s>>>(ds->csr_ptr, ds->csr_col,
                                                                                            K, nnz, ds->edeg, ds->ecol);
                count_launches(2);
            } else { // outside the record format: every sweep runs k_ccd
                ds->device_bytes -= static_cast<int64_t>(sizeof(RRec) * nnz + K + 32 + 2 * (nnz + 16));
                dfree(ds->rq, s);
                dfree(ds->edeg, s);
                dfree(ds->ecol, s);
            }
            count_launches(1);
            dfree(tmp3, s);
            dfree(d_oc, s);
            dfree(d_ob, s);
            dfree(d_rbad, s);
        }
        bt.mark("rq");
        if (y_dot_x_global) {
            std::vector<double> yd(static_cast<size_t>(J));
            for (int32_t j = 0; j < J; ++j) yd[static_cast<size_t>(j)] = static_cast<double>(y_dot_x_global[j]);
            CUDA_TRY(cudaMemcpyAsync(ds->y_dot_x, yd.data(), sizeof(double) * J, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaStreamSynchronize(s)); // yd is stack-owned
        } else {
            k_ydotx<<<J, 256, 0, s>>>(ds->pairs, ds->col_ptr, ds->event_counts, ds->y_dot_x, J);
        }
        count_launches(6 + (nnz > 0 ? 2 : 0) + (y_dot_x_global ? 0 : 1));
        dfree(tmp, s);
    }
    int bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    dfree(d_rows, s);
    dfree(d_subj, s);
    dfree(d_col, s);
    dfree(d_w, s);
    dfree(d_excl, s);
    dfree(d_bad, s);
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    if (bad & 2) input_error("dataset: every subject needs at least one era");
    if (bad & 4) input_error("dataset: era length must be positive");
    if (bad & 1) input_error("dataset: invalid pair (row/subject out of range, subject not owning its row, "
                             "or rows not strictly ascending within a column)");

    bt.mark("frees, validation");
    ds->col_runs_h.resize(static_cast<size_t>(J));
    CUDA_TRY(cudaMemcpy(ds->col_runs_h.data(), ds->col_runs, sizeof(int32_t) * J, cudaMemcpyDeviceToHost));
    {
        int* d_mx = nullptr;
        int64_t b2 = 0;
        d_mx = dalloc<int>(1, b2, s);
        CUDA_TRY(cudaMemsetAsync(d_mx, 0, sizeof(int), s));
        const int64_t nsl = static_cast<int64_t>(J) * C;
        if (nsl > 0) k_max_slice<<<grid_for(nsl, 256, sms), 256, 0, s>>>(ds->split, J, C, d_mx);
        CUDA_TRY(cudaMemcpyAsync(&ds->max_slice, d_mx, sizeof(int), cudaMemcpyDeviceToHost, s));
        dfree(d_mx, s);
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    {
        std::vector<int32_t> cs(static_cast<size_t>(C) + 1);
        CUDA_TRY(cudaMemcpy(cs.data(), ds->cta_subj, sizeof(int32_t) * (C + 1), cudaMemcpyDeviceToHost));
        ds->max_cta_subjects = 0;
        for (int c = 0; c < C; ++c) ds->max_cta_subjects = std::max(ds->max_cta_subjects, cs[c + 1] - cs[c]);
        CUDA_TRY(cudaMemcpy(cs.data(), ds->cta_era, sizeof(int32_t) * (C + 1), cudaMemcpyDeviceToHost));
        ds->max_cta_eras = 0;
        for (int c = 0; c < C; ++c) ds->max_cta_eras = std::max(ds->max_cta_eras, cs[c + 1] - cs[c]);
    }
    ds->col_nonempty_h.resize(static_cast<size_t>(J));
    for (int32_t j = 0; j < J; ++j) {
        const int64_t cnt =
            col_nnz_global ? col_nnz_global[j] : (ds->col_ptr_h[static_cast<size_t>(j) + 1] - ds->col_ptr_h[j]);
        ds->col_nonempty_h[static_cast<size_t>(j)] = cnt > 0 ? 1 : 0;
    }
    CUDA_TRY(cudaMemcpy(ds->col_nonempty, ds->col_nonempty_h.data(), J, cudaMemcpyHostToDevice));
    bt.mark("metadata");
}

bsccs_dataset* dataset_new(int32_t N, int32_t K, int32_t J, int64_t nnz, int device, int ctas_override) {
    ensure_pool(device);
    auto* ds = new bsccs_dataset();
    try {
        ds->device = device;
        ds->N = N;
        ds->K = K;
        ds->J = J;
        ds->nnz = nnz;
        ds->ctas = ctas_override > 0 ? ctas_override : default_ctas(device);
        alloc_dataset(ds);
    } catch (...) {
        dataset_destroy(ds);
        throw;
    }
    return ds;
}

bsccs_dataset* dataset_create(int32_t N, int32_t K, int32_t J, int64_t nnz, const int32_t* subject_offsets,
                              const int32_t* events_per_subject, const int32_t* era_lengths,
                              const int32_t* event_counts, const int64_t* col_ptr, const int32_t* rows,
                              const int32_t* subjects, const int64_t* y_dot_x_global,
                              const int64_t* col_nnz_global, int device, int ctas_override) {
    NvtxRange nvtx_("bsccs_dataset_create");
    if (N < 1) input_error("dataset: no subjects");
    if (K < 1 || J < 1 || nnz < 0) input_error("dataset: invalid sizes");
    if (!subject_offsets || !events_per_subject || !era_lengths || !event_counts || !col_ptr)
        input_error("dataset: null array");
    if (nnz > 0 && !rows) input_error("dataset: null pair arrays"); // subjects may be NULL: derived from rows
    // small-array invariants on the host (dataset.hpp:45-60)
    if (subject_offsets[0] != 0 || subject_offsets[N] != K) input_error("dataset: subject offsets must span [0, num_eras]");
    if (col_ptr[0] != 0 || col_ptr[J] != nnz) input_error("dataset: column pointers must span [0, nnz]");
    for (int32_t j = 0; j < J; ++j)
        if (col_ptr[j + 1] < col_ptr[j]) input_error("dataset: column pointers must be non-decreasing");
    // per-subject and per-era checks run on the device after the upload

    DeviceGuard g(device);
    bsccs_dataset* ds = dataset_new(N, K, J, nnz, device, ctas_override);
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_alloc = nullptr, ev_era = nullptr;
    std::exception_ptr failure;
    try {
        cudaStream_t s = ds->stream;
        h2d(ds->col_ptr, col_ptr, sizeof(int64_t) * (J + 1), s, device);
        h2d(ds->subject_offsets, subject_offsets, sizeof(int32_t) * (N + 1), s, device);
        h2d(ds->events_per_subject, events_per_subject, sizeof(int32_t) * N, s, device);
        int64_t scratch_bytes = 0;
        int32_t* d_rows = dalloc<int32_t>(nnz, scratch_bytes, s);
        int32_t* d_subj = dalloc<int32_t>(nnz, scratch_bytes, s);
        CUDA_TRY(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ev_alloc, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ev_era, cudaEventDisableTiming));
        // the pair arrays first: the build starts on them while the era
        // arrays upload on a side stream (copy and compute overlap)
        if (nnz > 0 && subjects) {
            h2d(d_rows, rows, sizeof(int32_t) * nnz, s, device);
            h2d(d_subj, subjects, sizeof(int32_t) * nnz, s, device);
        } else if (nnz > 0) { // subjects derived on the device: no upload of the redundant array
            // rows in chunks on the side stream; each chunk's owners are looked
            // up (a gather per pair) while the next chunk is on the link
            const int sms = sm_count(device);
            int64_t eb = 0;
            int32_t* d_esub = dalloc<int32_t>(K, eb, s);
            k_era_owner<<<grid_for(N, 256, sms), 256, 0, s>>>(ds->subject_offsets, N, K, d_esub);
            CUDA_TRY(cudaEventRecord(ev_alloc, s));
            CUDA_TRY(cudaStreamWaitEvent(s2, ev_alloc, 0));
            constexpr int kRowChunks = 4;
            cudaEvent_t evc[kRowChunks] = {};
            try {
                for (int c = 0; c < kRowChunks; ++c) {
                    const int64_t a = nnz * c / kRowChunks, b = nnz * (c + 1) / kRowChunks;
                    CUDA_TRY(cudaEventCreateWithFlags(&evc[c], cudaEventDisableTiming));
                    if (b > a) h2d(d_rows + a, rows + a, sizeof(int32_t) * (b - a), s2, device);
                    CUDA_TRY(cudaEventRecord(evc[c], s2));
                    CUDA_TRY(cudaStreamWaitEvent(s, evc[c], 0));
                    if (b > a)
                        k_subject_of_row<<<grid_for(b - a, 256, sms), 256, 0, s>>>(d_rows + a, d_esub, K, b - a,
                                                                                    d_subj + a);
                }
            } catch (...) {
                for (auto e : evc)
                    if (e) cudaEventDestroy(e);
                throw;
            }
            for (auto e : evc) cudaEventDestroy(e);
            CUDA_TRY(cudaGetLastError());
            count_launches(1 + kRowChunks);
            dfree(d_esub, s);
        }
        CUDA_TRY(cudaEventRecord(ev_alloc, s)); // the era arrays were allocated on s
        CUDA_TRY(cudaStreamWaitEvent(s2, ev_alloc, 0));
        h2d(ds->era_lengths, era_lengths, sizeof(int32_t) * K, s2, device);
        h2d(ds->event_counts, event_counts, sizeof(int32_t) * K, s2, device);
        CUDA_TRY(cudaEventRecord(ev_era, s2));
        ds->col_ptr_h.assign(col_ptr, col_ptr + J + 1);
        finish_dataset(ds, d_rows, d_subj, y_dot_x_global, col_nnz_global, ev_era);
    } catch (...) {
        failure = std::current_exception();
    }
    if (s2) {
        cudaStreamSynchronize(s2);
        cudaStreamDestroy(s2);
    }
    if (ev_alloc) cudaEventDestroy(ev_alloc);
    if (ev_era) cudaEventDestroy(ev_era);
    if (failure) {
        dataset_destroy(ds);
        std::rethrow_exception(failure);
    }
    return ds;
}

void dataset_destroy(bsccs_dataset* ds) {
    if (!ds) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(ds->device);
    cudaStream_t s = ds->stream;
    dfree(ds->pairs, s);
    dfree(ds->pq, s);
    dfree(ds->row_slot, s);
    dfree(ds->bstart, s);
    dfree(ds->col_ptr, s);
    dfree(ds->split, s);
    dfree(ds->cta_era, s);
    dfree(ds->cta_subj, s);
    dfree(ds->subject_offsets, s);
    dfree(ds->events_per_subject, s);
    dfree(ds->era_lengths, s);
    dfree(ds->event_counts, s);
    dfree(ds->csr_ptr, s);
    dfree(ds->csr_col, s);
    dfree(ds->y_dot_x, s);
    dfree(ds->col_nonempty, s);
    dfree(ds->col_runs, s);
    dfree(ds->rq, s);
    dfree(ds->rovf, s);
    dfree(ds->edeg, s);
    dfree(ds->ecol, s);
    if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
    if (prev >= 0) cudaSetDevice(prev);
    delete ds;
}

namespace {

void launch_dense(bsccs_state* st, bool beta_zero = false) {
    const bsccs_dataset* ds = st->ds;
    const int g = build_grid(ds->device);
    if (beta_zero)
        k_zero_xb<<<g, 256, 0, st->stream>>>(st->X, st->snap, ds->row_slot, ds->K);
    else
        k_dense_xb<<<g, 256, 0, st->stream>>>(st->X, st->snap, ds->csr_ptr, ds->csr_col, st->beta, ds->row_slot,
                                              ds->K, st->err);
    k_dense_den<<<g, 256, 0, st->stream>>>(st->X, ds->era_lengths, ds->subject_offsets, ds->bstart, ds->N, st->denc);
    count_launches(2);
    CUDA_TRY(cudaGetLastError());
    st->dense_pending = false;
    st->snap_valid = true;
    st->x_stale = false;
    st->denc_valid = st->denc != nullptr;
}

void alloc_state(bsccs_state* st, const bsccs_dataset* ds) {
    int64_t b = 0;
    st->ds = ds;
    ensure_pool(ds->device);
    CUDA_TRY(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
    cudaStream_t s = st->stream;
    st->X = dalloc<double>(ds->nslots, b, s);
    st->snap = dalloc<double>(ds->K, b, s);
    st->beta = dalloc<double>(ds->J, b, s);
    st->trust = dalloc<double>(ds->J, b, s);
    st->visit = dalloc<int32_t>(ds->J, b, s);
    st->vsplit = dalloc<longlong2>(static_cast<int64_t>(ds->J) * ds->ctas, b, s);
    st->slots = dalloc<unsigned long long>(kXchgAreaWords, b, s);
    st->moved = dalloc<uint8_t>(ds->J, b, s);
    st->counter = dalloc<unsigned long long>(1, b, s);
    st->err = dalloc<DevErr>(1, b, s);
    st->res = dalloc<DevResult>(1, b, s);
    st->scratch = dalloc<double>(2 * kFLBlocks, b, s);
    if (ds->rq) {
        st->denc = dalloc<double>(ds->N, b, s);
        st->beta_prev = dalloc<double>(ds->J, b, s);
    }
    st->res_h = pinned_result();
    CUDA_TRY(cudaEventCreate(&st->ev0));
    CUDA_TRY(cudaEventCreate(&st->ev1));
    CUDA_TRY(cudaMemsetAsync(st->slots, 0, sizeof(unsigned long long) * kXchgAreaWords, s));
    CUDA_TRY(cudaMemsetAsync(st->counter, 0, sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(st->err, 0, sizeof(DevErr), s));
    CUDA_TRY(cudaMemsetAsync(st->res, 0, sizeof(DevResult), s));
}

} // namespace

bsccs_state* state_create(const bsccs_dataset* ds, const double* beta_host) {
    if (!ds) input_error("null dataset");
    if (beta_host)
        for (int32_t j = 0; j < ds->J; ++j)
            if (!std::isfinite(beta_host[j])) input_error("init_state: non-finite coefficient");
    DeviceGuard g(ds->device);
    auto* st = new bsccs_state();
    try {
        alloc_state(st, ds);
        const int grid = build_grid(ds->device);
        k_init_blocks<<<grid, 256, 0, st->stream>>>(st->X, ds->bstart, ds->subject_offsets, ds->events_per_subject,
                                                    ds->N);
        count_launches(1);
        if (beta_host)
            CUDA_TRY(cudaMemcpyAsync(st->beta, beta_host, sizeof(double) * ds->J, cudaMemcpyHostToDevice, st->stream));
        else
            CUDA_TRY(cudaMemsetAsync(st->beta, 0, sizeof(double) * ds->J, st->stream));
        if (!beta_host && st->denc) { // cold start for the resident-beta sweep (dense_recompute_zero)
            k_den_zero<<<grid, 256, 0, st->stream>>>(ds->era_lengths, ds->subject_offsets, ds->N, st->denc);
            count_launches(1);
            st->denc_valid = true;
            st->x_stale = true;
            st->snap_valid = false;
        } else {
            launch_dense(st, beta_host == nullptr);
        }
        sync_and_check(st);
        check_err_block(st);
    } catch (...) {
        state_destroy(st);
        throw;
    }
    return st;
}

bsccs_state* state_clone(const bsccs_state* src) {
    const bsccs_dataset* ds = src->ds;
    DeviceGuard g(ds->device);
    auto* st = new bsccs_state();
    try {
        alloc_state(st, ds);
        CUDA_TRY(cudaStreamSynchronize(src->stream));
        CUDA_TRY(cudaMemcpyAsync(st->X, src->X, sizeof(double) * ds->nslots, cudaMemcpyDeviceToDevice, st->stream));
        CUDA_TRY(cudaMemcpyAsync(st->snap, src->snap, sizeof(double) * ds->K, cudaMemcpyDeviceToDevice, st->stream));
        CUDA_TRY(cudaMemcpyAsync(st->beta, src->beta, sizeof(double) * ds->J, cudaMemcpyDeviceToDevice, st->stream));
        if (st->denc && src->denc)
            CUDA_TRY(cudaMemcpyAsync(st->denc, src->denc, sizeof(double) * ds->N, cudaMemcpyDeviceToDevice, st->stream));
        st->snap_valid = src->snap_valid;
        st->x_stale = src->x_stale;
        st->denc_valid = src->denc_valid;
        sync_and_check(st);
    } catch (...) {
        state_destroy(st);
        throw;
    }
    return st;
}

void state_destroy(bsccs_state* st) {
    if (!st) return;
    int prev = -1;
    cudaGetDevice(&prev);
    if (st->ds) cudaSetDevice(st->ds->device);
    cudaStream_t s = st->stream;
    if (s) {
        dfree(st->X, s);
        dfree(st->snap, s);
        dfree(st->le_tmp, s);
        dfree(st->num, s);
        dfree(st->beta, s);
        dfree(st->trust, s);
        dfree(st->visit, s);
        dfree(st->moved, s);
        dfree(st->vsplit, s);
        dfree(st->slots, s);
        dfree(st->counter, s);
        dfree(st->err, s);
        dfree(st->res, s);
        dfree(st->scratch, s);
        dfree(st->denc, s);
        dfree(st->beta_prev, s);
        cudaStreamSynchronize(s);
    }
    release_pinned_result(st->res_h);
    if (st->ev0) cudaEventDestroy(st->ev0);
    if (st->ev1) cudaEventDestroy(st->ev1);
    if (s) cudaStreamDestroy(s);
    if (prev >= 0) cudaSetDevice(prev);
    delete st;
}

// X (subject blocks) brought up to date after resident-beta sweeps: x'beta
// rebuilt from beta (the value those sweeps use) with its snapshot, the
// headers from the compact denominators.
// the closing refresh a fit skipped (k_final_xb / k_final_den), done before the state's
// next use
void settle_dense(bsccs_state* st) {
    if (!st->dense_pending) return;
    launch_dense(st);
    sync_and_check(st);
    check_err_block(st);
}

void sync_x(bsccs_state* st) {
    settle_dense(st);
    if (!st->x_stale) return;
    const bsccs_dataset* ds = st->ds;
    const int g = build_grid(ds->device);
    k_dense_xb<<<g, 256, 0, st->stream>>>(st->X, st->snap, ds->csr_ptr, ds->csr_col, st->beta, ds->row_slot, ds->K,
                                          st->err);
    k_denc_to_hdr<<<g, 256, 0, st->stream>>>(st->X, ds->bstart, st->denc, ds->N);
    CUDA_TRY(cudaGetLastError());
    count_launches(2);
    st->x_stale = false;
    st->snap_valid = true;
}

// compact denominators from the headers (after an op that wrote X)
void sync_denc(bsccs_state* st) {
    settle_dense(st);
    if (st->denc_valid || !st->denc) return;
    const bsccs_dataset* ds = st->ds;
    k_hdr_to_denc<<<build_grid(ds->device), 256, 0, st->stream>>>(st->X, ds->bstart, st->denc, ds->N);
    CUDA_TRY(cudaGetLastError());
    count_launches(1);
    st->denc_valid = true;
}

void dense_recompute_zero(bsccs_state* st) {
    NvtxRange nvtx_("dense_recompute (beta = 0)");
    const bsccs_dataset* ds = st->ds;
    DeviceGuard g(ds->device);
    CUDA_TRY(cudaMemsetAsync(st->beta, 0, sizeof(double) * ds->J, st->stream));
    if (st->denc) { // the resident-beta sweep needs only the denominators
        k_den_zero<<<build_grid(ds->device), 256, 0, st->stream>>>(ds->era_lengths, ds->subject_offsets, ds->N,
                                                                    st->denc);
        CUDA_TRY(cudaGetLastError());
        count_launches(1);
        st->denc_valid = true;
        st->x_stale = true; // x'beta (0) and the headers on first use (sync_x)
        st->snap_valid = false;
        st->dense_pending = false;
    } else {
        launch_dense(st, true);
    }
    sync_and_check(st);
    check_err_block(st);
}

double final_log_likelihood(bsccs_state* st) {
    NvtxRange nvtx_("final refresh + log_likelihood");
    const bsccs_dataset* ds = st->ds;
    DeviceGuard dg(ds->device);
    k_final_xb<<<kFLBlocks, kLLThreads, 0, st->stream>>>(ds->csr_ptr, ds->csr_col, st->beta, ds->event_counts, ds->K,
                                                         st->snap, st->scratch, st->err);
    k_final_den<<<kFLBlocks, kLLThreads, 0, st->stream>>>(st->snap, ds->era_lengths, ds->subject_offsets,
                                                          ds->events_per_subject, ds->N, st->scratch, st->err);
    k_ll_final<<<1, 32, 0, st->stream>>>(st->scratch, kFLBlocks, st->res);
    count_launches(3);
    CUDA_TRY(cudaMemcpyAsync(st->res_h, st->res, sizeof(DevResult), cudaMemcpyDeviceToHost, st->stream));
    sync_and_check(st);
    check_err_block(st);
    st->dense_pending = true; // the blocks are rebuilt on their next use
    st->snap_valid = true;
    return st->res_h->ll_linear - st->res_h->ll_logden;
}

void dense_recompute(bsccs_state* st, const double* beta_host) {
    NvtxRange nvtx_("dense_recompute");
    const bsccs_dataset* ds = st->ds;
    if (beta_host)
        for (int32_t j = 0; j < ds->J; ++j)
            if (!std::isfinite(beta_host[j])) input_error("dense_recompute: non-finite coefficient");
    DeviceGuard g(ds->device);
    if (beta_host)
        CUDA_TRY(cudaMemcpyAsync(st->beta, beta_host, sizeof(double) * ds->J, cudaMemcpyHostToDevice, st->stream));
    launch_dense(st);
    sync_and_check(st);
    check_err_block(st);
}

namespace {

SweepArgs base_args(const ExchangePlan& plan) {
    SweepArgs a;
    std::memset(&a, 0, sizeof a);
    if (plan.shards.empty() || plan.shards.size() > static_cast<size_t>(kMaxLocalShards))
        internal_error("exchange plan: bad shard count");
    int begin = 0;
    for (size_t i = 0; i < plan.shards.size(); ++i) {
        bsccs_state* st = plan.shards[i];
        ShardArgs& s = a.sh[i];
        s.xslots = plan.shard_slots.empty() ? plan.local_slots : plan.shard_slots[i];
        s.xcounter = plan.shard_counters.empty() ? plan.counter : plan.shard_counters[i];
        s.xowner = plan.shard_slots.empty() ? (i == 0) : 1;
        s.lslots = plan.hier ? plan.shard_local[i] : nullptr;
        s.p_local = st->ds->ctas;
        s.pq = st->ds->pq;
        s.snap = st->snap;
        s.vsplit = st->vsplit;
        s.moved = st->moved;
        s.col_ptr = st->ds->col_ptr;
        s.col_runs = st->ds->col_runs;
        s.K = st->ds->K;
        s.split = st->ds->split;
        s.cta_era = st->ds->cta_era;
        s.cta_subj = st->ds->cta_subj;
        s.subject_offsets = st->ds->subject_offsets;
        s.num = st->num;
        s.X = st->X;
        s.row_slot = st->ds->row_slot;
        s.bstart = st->ds->bstart;
        s.era_len = st->ds->era_lengths;
        s.rq = st->ds->rq;
        s.rovf = st->ds->rovf;
        s.denc = st->denc;
        s.beta_prev = st->beta_prev;
        s.csr_ptr = st->ds->csr_ptr;
        s.csr_col = st->ds->csr_col;
        s.edeg = st->ds->edeg;
        s.ecol = st->ds->ecol;
        s.beta = st->beta;
        s.trust = st->trust;
        s.err = st->err;
        s.res = st->res;
        s.ctas = st->ds->ctas;
        s.cta_begin = begin;
        s.pid_base = plan.participant_base + begin;
        begin += s.ctas;
    }
    a.nsh = static_cast<int>(plan.shards.size());
    const bsccs_state* s0 = plan.shards[0];
    a.visit = s0->visit;
    a.nvisit = static_cast<int>(s0->visit_h.size());
    a.y_dot_x = s0->ds->y_dot_x;
    a.col_nonempty = s0->ds->col_nonempty;
    a.J = s0->ds->J;
    if (plan.dst.empty() || plan.dst.size() > static_cast<size_t>(kMaxRanks)) internal_error("exchange plan: bad peers");
    for (size_t d = 0; d < plan.dst.size(); ++d) a.dst[d] = plan.dst[d];
    a.ndst = static_cast<int>(plan.dst.size());
    a.slots = plan.local_slots;
    a.P = plan.hier ? static_cast<int>(plan.dst.size()) : plan.total_participants;
    a.hier = plan.hier ? 1 : 0;
    if (plan.hier && plan.shard_local.size() != plan.shards.size()) internal_error("exchange plan: local areas");
    a.counter = plan.counter;
    static const unsigned long long timeout_ns = [] {
        const char* e = std::getenv("BSCCS_XCHG_TIMEOUT_S");
        const double sec = e ? std::atof(e) : 120.0;
        return static_cast<unsigned long long>((sec > 0.0 ? sec : 120.0) * 1e9);
    }();
    a.poll_timeout_ns = timeout_ns;
    if (a.P > kMaxParticipants) internal_error("exchange plan: too many participants (limit 2048 CTAs over all ranks)");
    return a;
}

int plan_ctas(const ExchangePlan& plan) {
    int n = 0;
    for (auto* st : plan.shards) n += st->ds->ctas;
    return n;
}

// Sweeps keep each CTA's subject records in shared memory when every
// shard's largest CTA subject range fits (BSCCS_SUBJ_SMEM=0 disables it).
int subject_tile_cap(const ExchangePlan& plan, bool streamed, size_t tile_offset) {
    static const bool enabled = [] {
        const char* e = std::getenv("BSCCS_SUBJ_SMEM");
        return !(e && e[0] == '0');
    }();
    if (!enabled) return 0;
    int m = 0;
    for (auto* st : plan.shards) m = std::max(m, st->ds->max_cta_subjects);
    const int cap = (m + 1) / 2 * 2; // keeps the arrays 8-byte aligned
    const size_t bytes = tile_offset + static_cast<size_t>(cap) * subj_tile_bytes(!streamed);
    return bytes <= static_cast<size_t>(kMaxSweepSmem) ? std::max(cap, 2) : 0;
}

// The L2 prefetch of the records two coordinates ahead pays while the
// slices are small: measured -3% fit time at ~200 pairs per CTA per
// coordinate (config 2), +4% at ~740 (config 3), where the extra line
// fetches compete with the gathers.  BSCCS_PREFETCH=0/1 forces it.
// mean pairs per CTA per (non-empty) coordinate
double mean_slice(const ExchangePlan& plan) {
    int64_t nnz = 0, ctas = 0;
    for (auto* st : plan.shards) {
        nnz += st->ds->nnz;
        ctas += st->ds->ctas;
    }
    const bsccs_dataset* ds = plan.shards[0]->ds;
    int64_t cols = 0;
    for (uint8_t nz : ds->col_nonempty_h) cols += nz ? 1 : 0;
    if (cols == 0 || ctas == 0) return 0.0;
    return static_cast<double>(nnz) / static_cast<double>(cols) / static_cast<double>(ctas);
}

int prefetch_enabled(const ExchangePlan& plan) {
    static const int forced = [] {
        const char* e = std::getenv("BSCCS_PREFETCH");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    if (forced >= 0) return forced;
    const double per_cta = mean_slice(plan);
    return per_cta > 0.0 && per_cta <= 384.0 ? 1 : 0;
}

// k_ccd's pair records, built on first use (datasets the resident-beta sweep
// runs need them only for the single-coordinate ops and hand-overs)
std::mutex g_pq_mutex;
void ensure_pq(const bsccs_dataset* cds) {
    std::lock_guard<std::mutex> lk(g_pq_mutex);
    auto* ds = const_cast<bsccs_dataset*>(cds);
    if (ds->pq || ds->nnz == 0) return;
    DeviceGuard g(ds->device);
    ds->pq = dalloc<int4>(ds->nnz, ds->device_bytes, ds->stream);
    k_build_pq<<<grid_for(ds->nnz, 256, sm_count(ds->device)), 256, 0, ds->stream>>>(
        ds->pairs, ds->nnz, ds->row_slot, ds->bstart, ds->era_lengths, ds->cta_subj, ds->ctas, ds->pq);
    CUDA_TRY(cudaGetLastError());
    count_launches(1);
    CUDA_TRY(cudaStreamSynchronize(ds->stream));
}

void launch_ccd(const ExchangePlan& plan, SweepArgs& a) {
    bsccs_state* s0 = plan.shards[0];
    for (size_t i = 0; i < plan.shards.size(); ++i) {
        ensure_pq(plan.shards[i]->ds);
        a.sh[i].pq = plan.shards[i]->ds->pq;
    }
    ensure_kernel_attrs(s0->ds->device);
    // the streamed path only when some slice exceeds the register tiles
    // (and always for the single-coordinate ops, whose update streams); its
    // staging buffer takes the shared memory left beside the subject tile
    // (up to kStreamMax pairs; the tile is dropped if that leaves too little)
    // one register tile when every slice fits it (1 tile = 352 pairs per
    // CTA and coordinate; config 2's slices are ~200): fewer registers and
    // less shared memory, measured 10% faster than 3 tiles at config 2.
    // Also when the typical slice is well inside it and only some columns
    // exceed it (skewed prevalence): those stream, the rest run lighter --
    // Zipf 1M 54.7 -> 47.5 ms; config 3 (mean ~740) stays on 3 tiles.
    static const int tiles_forced = [] {
        const char* e = std::getenv("BSCCS_TILES"); // experiment hook: 1 or 3
        return e ? std::atoi(e) : 0;
    }();
    bool one_tile = a.mode == kModeSweep && tiles_forced != 3;
    for (auto* st : plan.shards) one_tile = one_tile && st->ds->max_slice <= t1::kCap;
    if (a.mode == kModeSweep && tiles_forced != 3 && mean_slice(plan) <= 0.75 * t1::kCap) one_tile = true;
    if (a.mode == kModeSweep && tiles_forced == 1) one_tile = true;
    bool streamed = a.mode != kModeSweep;
    for (auto* st : plan.shards) streamed = streamed || st->ds->max_slice > (one_tile ? t1::kCap : t3::kCap);
    const size_t smem_size = one_tile ? sizeof(t1::Smem) : sizeof(t3::Smem);
    const size_t tile_off = one_tile ? t1::kSmemSubjOffset : t3::kSmemSubjOffset;
    a.ss_cap = a.mode == kModeSweep ? subject_tile_cap(plan, streamed, tile_off) : 0;
    a.bm_words = 0;
    if (a.mode == kModeSweep && a.ss_cap == 0) { // touched-subject bitmaps instead of the hash table
        int m = 0;
        for (auto* st : plan.shards) m = std::max(m, st->ds->max_cta_subjects);
        const int words = (m + 31) / 32 + 1;
        static const bool bm_on = [] {
            const char* e = std::getenv("BSCCS_TOUCH_BITS"); // experiment hook
            return !(e && e[0] == '0');
        }();
        if (bm_on && 2 * static_cast<size_t>(words) * sizeof(unsigned) <= 64 * 1024) a.bm_words = words;
    }
    a.prefetch = a.mode == kModeSweep ? prefetch_enabled(plan) : 0;
    constexpr size_t kPairBytes = sizeof(double) + sizeof(int);
    static const int kStreamMax = [] {
        const char* e = std::getenv("BSCCS_STREAM_MAX"); // experiment hook
        return e ? std::atoi(e) : 1536;
    }();
    auto base_bytes = [&] {
        return a.ss_cap > 0 ? tile_off + static_cast<size_t>(a.ss_cap) * subj_tile_bytes(!streamed)
               : a.bm_words > 0 ? tile_off + 2 * static_cast<size_t>(a.bm_words) * sizeof(unsigned)
                                : smem_size;
    };
    size_t bytes = base_bytes();
    a.stream_off = 0;
    a.stream_cap = 0;
    if (streamed) {
        auto room = [&] { return (static_cast<size_t>(kMaxSweepSmem) - (base_bytes() + 15) / 16 * 16) / kPairBytes; };
        if (a.ss_cap > 0 && room() < static_cast<size_t>(2 * kT)) a.ss_cap = 0;
        const size_t off = (base_bytes() + 15) / 16 * 16;
        const int cap = static_cast<int>(std::min<size_t>(room(), kStreamMax)) / kT * kT;
        if (cap < kT) internal_error("sweep: no shared memory for the streamed-slice buffer");
        a.stream_off = static_cast<int>(off);
        a.stream_cap = cap;
        bytes = off + static_cast<size_t>(cap) * kPairBytes;
    }
    void* params[] = {&a};
    void* fn;
    if (one_tile && streamed)
        fn = a.ss_cap > 0 ? reinterpret_cast<void*>(t1::k_ccd<true, true>) : reinterpret_cast<void*>(t1::k_ccd<false, true>);
    else if (one_tile)
        fn = a.ss_cap > 0 ? reinterpret_cast<void*>(t1::k_ccd<true, false>) : reinterpret_cast<void*>(t1::k_ccd<false, false>);
    else if (a.ss_cap > 0)
        fn = streamed ? reinterpret_cast<void*>(t3::k_ccd<true, true>) : reinterpret_cast<void*>(t3::k_ccd<true, false>);
    else
        fn = streamed ? reinterpret_cast<void*>(t3::k_ccd<false, true>) : reinterpret_cast<void*>(t3::k_ccd<false, false>);
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(plan_ctas(plan)), dim3(kSweepThreads), params, bytes, s0->stream));
    count_launches(1);
}

// Launch shape of the resident-beta sweep, or ok = false when a shard does
// not qualify (no pair records, a slice beyond three register tiles, or
// beta plus the staging buffers and the touched-subject bitmaps beyond the
// shared memory): those sweeps run k_ccd.
struct RcdShape {
    bool ok = false, kss = false;
    int tiles = 0, threads = 0;
    int ss_cap = 0, bm_words = 0, beta_cap = 0, crit_E = 0, crit_cap = 0;
    double beta_limit = 0.0; // |beta_j| beyond this: partial products of exp(beta) could leave range
    size_t bytes = 0;
};
RcdShape rcd_shape(const ExchangePlan& plan) {
    RcdShape r;
    if (!rcd_enabled() || g_sweep_kind.load() == 1) return r;
    int maxslice = 0, maxsub = 0, maxdeg = 1;
    for (auto* st : plan.shards) {
        if (!st->ds->rq || !st->ds->edeg || !st->denc) return r;
        maxslice = std::max(maxslice, st->ds->max_slice);
        maxsub = std::max(maxsub, st->ds->max_cta_subjects);
        maxdeg = std::max(maxdeg, st->ds->max_deg);
    }
    r.beta_limit = 700.0 / maxdeg;
    if (g_beta_limit.load() > 0.0) r.beta_limit = std::min(r.beta_limit, g_beta_limit.load());
    static const int tiles_forced = [] {
        const char* e = std::getenv("BSCCS_RTILES"); // experiment hook: 1, 2 or 3
        return e ? std::atoi(e) : 0;
    }();
    // the smallest shape whose slots hold every slice
    size_t smem_fixed = 0, bufs = 0;
    if ((tiles_forced == 0 || tiles_forced == 1) && maxslice <= r1::kRC) {
        r.tiles = 1, r.threads = r1::kT, smem_fixed = r1::kRSmemBytes, bufs = r1::kRBufs * r1::kRBufBytes;
    } else if ((tiles_forced == 0 || tiles_forced == 2) && maxslice <= r2::kRC) {
        r.tiles = 2, r.threads = r2::kT, smem_fixed = r2::kRSmemBytes, bufs = r2::kRBufs * r2::kRBufBytes;
    } else if (maxslice <= r3::kRC) {
        r.tiles = 3, r.threads = r3::kT, smem_fixed = r3::kRSmemBytes, bufs = r3::kRBufs * r3::kRBufBytes;
    } else {
        return r;
    }
    r.beta_cap = (plan.shards[0]->ds->J + 1 + 15) / 16 * 16; // + the unit drug J
    const size_t head = smem_fixed + 2 * static_cast<size_t>(r.beta_cap) * sizeof(double);
    const size_t base = head + bufs;
    static const bool tile_on = [] {
        const char* e = std::getenv("BSCCS_SUBJ_SMEM");
        return !(e && e[0] == '0');
    }();
    const int cap = std::max(2, (maxsub + 1) / 2 * 2);
    if (tile_on && base + static_cast<size_t>(cap) * sizeof(double) <= static_cast<size_t>(kMaxSweepSmem)) {
        r.kss = true;
        r.ss_cap = cap;
        r.bytes = base + static_cast<size_t>(cap) * sizeof(double);
    } else {
        r.bm_words = (maxsub / 32 + 2) & ~1; // even: the lookup table after the bitmaps stays 8-B aligned
        r.bytes = base + 2 * static_cast<size_t>(r.bm_words) * sizeof(unsigned) + r3::kHTab * sizeof(int2);
        if (r.bytes > static_cast<size_t>(kMaxSweepSmem)) return r;
    }
    // criterion chunks in the union region: beta at cycle start plus two
    // buffers of crit_E eras' degrees and ~1.25x their expected drugs, and
    // the chunks' first-drug offsets
    double deg = 0.0;
    for (auto* st : plan.shards) deg = std::max(deg, static_cast<double>(st->ds->nnz) / std::max(1, st->ds->K));
    constexpr int kCB = r1::kCBufs; // the same in every shape
    int maxera = 0;
    for (auto* st : plan.shards) maxera = std::max(maxera, st->ds->max_cta_eras);
    for (int eper = 8; eper >= 1; eper /= 2) {
        const int E = eper * r.threads;
        const int ccap = (static_cast<int>(E * deg * 1.25) + 256 + 7) / 8 * 8;
        const size_t nchunk = static_cast<size_t>(maxera) / E + 2; // chunk offsets kept in shared memory
        const size_t crit = head + static_cast<size_t>(r.beta_cap) * sizeof(double) + kCB * static_cast<size_t>(E + 32) +
                            kCB * sizeof(uint16_t) * static_cast<size_t>(ccap + 16) + 8 + nchunk * sizeof(int64_t);
        if (crit <= static_cast<size_t>(kMaxSweepSmem) || eper == 1) {
            r.crit_E = E;
            r.crit_cap = ccap;
            r.bytes = std::max(r.bytes, (crit + 15) / 16 * 16);
            break;
        }
    }
    if (r.bytes > static_cast<size_t>(kMaxSweepSmem)) return r;
    r.ok = true;
    return r;
}

void launch_rcd(const ExchangePlan& plan, SweepArgs& a, const RcdShape& sh) {
    bsccs_state* s0 = plan.shards[0];
    ensure_kernel_attrs(s0->ds->device);
    a.beta_cap = sh.beta_cap;
    a.ss_cap = sh.kss ? sh.ss_cap : 0;
    a.bm_words = sh.kss ? 0 : sh.bm_words;
    a.crit_E = sh.crit_E;
    a.crit_cap = sh.crit_cap;
    a.beta_limit = sh.beta_limit;
    g_last_rcd_shape = sh.tiles | (sh.kss ? 16 : 0);
    void* params[] = {&a};
    void* fn = sh.tiles == 1   ? (sh.kss ? reinterpret_cast<void*>(r1::k_rcd<true>) : reinterpret_cast<void*>(r1::k_rcd<false>))
               : sh.tiles == 2 ? (sh.kss ? reinterpret_cast<void*>(r2::k_rcd<true>) : reinterpret_cast<void*>(r2::k_rcd<false>))
                               : (sh.kss ? reinterpret_cast<void*>(r3::k_rcd<true>) : reinterpret_cast<void*>(r3::k_rcd<false>));
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(plan_ctas(plan)), dim3(sh.threads), params, sh.bytes, s0->stream));
    count_launches(1);
}

ExchangePlan single_plan(bsccs_state* st) {
    ExchangePlan p;
    p.shards = {st};
    p.dst = {st->slots};
    p.local_slots = st->slots;
    p.counter = st->counter;
    p.total_participants = st->ds->ctas;
    p.participant_base = 0;
    return p;
}

} // namespace

void grad_hess(bsccs_state* st, int32_t j, double* g, double* h) {
    const bsccs_dataset* ds = st->ds;
    if (j < 0 || j >= ds->J) input_error("fused_grad_hess: coordinate out of range");
    DeviceGuard dg(ds->device);
    sync_x(st);
    ExchangePlan plan = single_plan(st);
    SweepArgs a = base_args(plan);
    a.mode = kModeGradHess;
    a.single_j = j;
    launch_ccd(plan, a);
    CUDA_TRY(cudaMemcpyAsync(st->res_h, st->res, sizeof(DevResult), cudaMemcpyDeviceToHost, st->stream));
    sync_and_check(st);
    check_err_block(st);
    *g = st->res_h->g;
    *h = st->res_h->h;
}

void sparse_update(bsccs_state* st, int32_t j, double delta) {
    const bsccs_dataset* ds = st->ds;
    if (j < 0 || j >= ds->J) input_error("sparse_delta_update: coordinate out of range");
    if (!std::isfinite(delta)) numeric_error("sparse_delta_update: non-finite step");
    if (delta == 0.0) return;
    DeviceGuard dg(ds->device);
    sync_x(st);
    ExchangePlan plan = single_plan(st);
    SweepArgs a = base_args(plan);
    a.mode = kModeUpdate;
    a.single_j = j;
    a.single_delta = delta;
    launch_ccd(plan, a);
    st->snap_valid = false;
    st->denc_valid = false;
    sync_and_check(st);
    check_err_block(st);
}

double log_likelihood(bsccs_state* st) {
    NvtxRange nvtx_("log_likelihood");
    const bsccs_dataset* ds = st->ds;
    DeviceGuard dg(ds->device);
    sync_x(st);
    k_ll_partial<<<kLLBlocks, kLLThreads, 0, st->stream>>>(st->X, ds->row_slot, ds->event_counts, ds->bstart, ds->K,
                                                           ds->N, st->scratch, st->err);
    k_ll_final<<<1, 32, 0, st->stream>>>(st->scratch, kLLBlocks, st->res);
    count_launches(2);
    CUDA_TRY(cudaMemcpyAsync(st->res_h, st->res, sizeof(DevResult), cudaMemcpyDeviceToHost, st->stream));
    sync_and_check(st);
    check_err_block(st);
    return st->res_h->ll_linear - st->res_h->ll_logden;
}

void state_get(bsccs_state* st, double* beta, double* xbeta, double* le, double* den) {
    const bsccs_dataset* ds = st->ds;
    DeviceGuard dg(ds->device);
    sync_x(st);
    CUDA_TRY(cudaStreamSynchronize(st->stream));
    if (beta) CUDA_TRY(cudaMemcpy(beta, st->beta, sizeof(double) * ds->J, cudaMemcpyDeviceToHost));
    if (!st->le_tmp) {
        int64_t b = 0;
        st->le_tmp = dalloc<double>(std::max(ds->K, ds->N), b, st->stream);
    }
    // gathered out of the subject blocks on the device (l*exp with the
    // kernels' own expression)
    auto gather = [&](const int32_t* idx, const int32_t* len, int64_t n, double* out) {
        k_gather_slots<<<build_grid(ds->device), 256, 0, st->stream>>>(st->X, idx, len, st->le_tmp, n);
        count_launches(1);
        CUDA_TRY(cudaMemcpyAsync(out, st->le_tmp, sizeof(double) * n, cudaMemcpyDeviceToHost, st->stream));
        CUDA_TRY(cudaStreamSynchronize(st->stream));
    };
    if (xbeta) gather(ds->row_slot, nullptr, ds->K, xbeta);
    if (le) gather(ds->row_slot, ds->era_lengths, ds->K, le);
    if (den) gather(ds->bstart, nullptr, ds->N, den);
}

void prepare_snapshot(bsccs_state* st) {
    if (st->snap_valid) return;
    const bsccs_dataset* ds = st->ds;
    DeviceGuard dg(ds->device);
    k_snapshot<<<build_grid(ds->device), 256, 0, st->stream>>>(st->X, ds->row_slot, st->snap, ds->K);
    CUDA_TRY(cudaGetLastError());
    count_launches(1);
    st->snap_valid = true;
}

namespace {
int g_debug_flags = 0;
unsigned long long* g_trace = nullptr;
int g_ntrace = 0;
size_t g_trace_words = 0;
}
namespace {
// n participants, one per thread: limbs + one arrival each into three words
// (the publish of §4.2), then thread 0 checks the count and reconstructs
__global__ void k_xsum_test(const double* v, int n, unsigned long long* words, double* out, int* status) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bool ok = true;
        for (int l = 0; l < 3; ++l) {
            unsigned long long w;
            ok = limb_of(v[i], l, w) && ok;
            red_add(words + l, w + kXCnt);
        }
        if (!ok) atomicOr(status, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long w0 = ld_poll(words), w1 = ld_poll(words + 1), w2 = ld_poll(words + 2);
        if ((w0 >> kXCntShift) != static_cast<unsigned long long>(n) || (w1 >> kXCntShift) != (w0 >> kXCntShift) ||
            (w2 >> kXCntShift) != (w0 >> kXCntShift))
            atomicOr(status, 4);
        bool ovf;
        *out = from_limbs(w0 & kXData, w1 & kXData, w2 & kXData, ovf);
        if (ovf) atomicOr(status, 2);
    }
}
} // namespace

void debug_exchange_sum(int device, const double* partials, int n, double* sum, int* status) {
    DeviceGuard g(device);
    cudaStream_t s = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double* dv = nullptr;
    unsigned long long* dw = nullptr;
    double* dout = nullptr;
    int* dst = nullptr;
    CUDA_TRY(cudaMalloc(&dv, sizeof(double) * n));
    CUDA_TRY(cudaMalloc(&dw, sizeof(unsigned long long) * 3));
    CUDA_TRY(cudaMalloc(&dout, sizeof(double)));
    CUDA_TRY(cudaMalloc(&dst, sizeof(int)));
    CUDA_TRY(cudaMemcpyAsync(dv, partials, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(dw, 0, sizeof(unsigned long long) * 3, s));
    CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(int), s));
    k_xsum_test<<<1, 1024, 0, s>>>(dv, n, dw, dout, dst);
    count_launches(1);
    int st = 0;
    CUDA_TRY(cudaMemcpyAsync(sum, dout, sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&st, dst, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    cudaFree(dv);
    cudaFree(dw);
    cudaFree(dout);
    cudaFree(dst);
    cudaStreamDestroy(s);
    *status = (st & 1) ? 1 : (st & 2) ? 2 : (st & 4) ? 3 : 0;
}

void set_debug_flags(int f) { g_debug_flags = f; }
void set_debug_sweep(int kind, double beta_limit) {
    g_sweep_kind = kind;
    g_beta_limit = beta_limit;
}
int debug_last_sweep() { return g_last_sweep; }
int debug_last_rcd_shape() { return g_last_rcd_shape; }
void set_debug_trace(int ncoords, int ctas) {
    if (g_trace) cudaFree(g_trace);
    g_trace = nullptr;
    g_ntrace = ncoords;
    g_trace_words = static_cast<size_t>(ncoords) * ctas * kTr;
    if (ncoords > 0) {
        CUDA_TRY(cudaMalloc(&g_trace, g_trace_words * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(g_trace, 0, g_trace_words * sizeof(unsigned long long)));
    }
}
unsigned long long* debug_trace_buffer(int* ncoords) {
    *ncoords = g_ntrace;
    return g_trace;
}
void read_debug_trace(unsigned long long* host, size_t words) {
    if (!g_trace) return;
    CUDA_TRY(cudaMemcpy(host, g_trace, std::min(words, g_trace_words) * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost));
}

// Exact, deterministic sum over every participant of the plan of two
// non-negative host scalars (this rank contributes (a, b)).
void plan_allreduce(const ExchangePlan& plan, double a, double b, double* ta, double* tb) {
    bsccs_state* s0 = plan.shards[0];
    DeviceGuard dg(s0->ds->device);
    for (auto* st : plan.shards)
        if (st->stream != s0->stream) CUDA_TRY(cudaStreamSynchronize(st->stream));
    SweepArgs args = base_args(plan);
    args.mode = kModeReduce;
    args.red_a = a;
    args.red_b = b;
    launch_ccd(plan, args);
    CUDA_TRY(cudaMemcpyAsync(s0->res_h, s0->res, sizeof(DevResult), cudaMemcpyDeviceToHost, s0->stream));
    CUDA_TRY(cudaStreamSynchronize(s0->stream));
    CUDA_TRY(cudaGetLastError());
    if (s0->res_h->err_remote) numeric_error("all-reduce: invalid contribution");
    *ta = s0->res_h->change;
    *tb = s0->res_h->magnitude;
}

void build_vsplit(const bsccs_dataset* ds, const int32_t* d_visit, int V, longlong2* out, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(V) * ds->ctas;
    if (n == 0) return;
    k_build_vsplit<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(ds->split, d_visit, V, ds->ctas, out);
    CUDA_TRY(cudaGetLastError());
    count_launches(1);
}

namespace {

void check_plan_errors(const ExchangePlan& plan) {
    for (auto* st : plan.shards) check_err_block(st);
    for (auto* st : plan.shards)
        if (st->res_h->err_remote) numeric_error("sweep aborted: a device error was raised on another shard");
}

// One coordinate finished on the host's side of the C ABI after the sweep
// stopped before it (ST_REFINE): the single-coordinate grad/hess launch
// (exact exchange with refinement rounds), the reference step on the host
// (the same prior.h code the kernel runs, solver.hpp:131-150), and the
// single-coordinate update launch.  Every rank of a group takes the same
// path (the stop is decided from identical exchange results).  Returns
// whether the coordinate moved.
bool refine_coordinate(const ExchangePlan& plan, const PriorParams& prior, int32_t j) {
    bsccs_state* s0 = plan.shards[0];
    SweepArgs g = base_args(plan);
    g.mode = kModeGradHess;
    g.single_j = j;
    launch_ccd(plan, g);
    for (auto* st : plan.shards)
        CUDA_TRY(cudaMemcpyAsync(st->res_h, st->res, sizeof(DevResult), cudaMemcpyDeviceToHost, s0->stream));
    double bj = 0.0, rj = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&bj, s0->beta + j, sizeof(double), cudaMemcpyDeviceToHost, s0->stream));
    CUDA_TRY(cudaMemcpyAsync(&rj, s0->trust + j, sizeof(double), cudaMemcpyDeviceToHost, s0->stream));
    CUDA_TRY(cudaStreamSynchronize(s0->stream));
    CUDA_TRY(cudaGetLastError());
    check_plan_errors(plan);
    const double gv = s0->res_h->g, hv = s0->res_h->h;
    double step = 0.0;
    const int serr = penalized_step_pre(prior, bj, beta_over_v(prior, bj), gv, hv, &step);
    if (serr) throw_device_error(serr, hv);
    const double delta = clamp_step(step, rj);
    if (delta != 0.0 && !std::isfinite(delta)) throw_device_error(DERR_STEP_NONFINITE, delta);
    if (delta != 0.0) {
        SweepArgs u = base_args(plan);
        u.mode = kModeUpdate;
        u.single_j = j;
        u.single_delta = delta;
        launch_ccd(plan, u);
        CUDA_TRY(cudaStreamSynchronize(s0->stream));
        CUDA_TRY(cudaGetLastError());
        for (auto* st : plan.shards) check_err_block(st);
    }
    const double rn = next_trust(delta, rj);
    for (auto* st : plan.shards)
        CUDA_TRY(cudaMemcpyAsync(st->trust + j, &rn, sizeof(double), cudaMemcpyHostToDevice, s0->stream));
    CUDA_TRY(cudaStreamSynchronize(s0->stream));
    return delta != 0.0;
}

} // namespace

SweepOutcome run_sweep(const ExchangePlan& plan, const PriorParams& prior, bool normalized, bool dense) {
    NvtxRange nvtx_("ccd_cycle");
    bsccs_state* s0 = plan.shards[0];
    if (dense && (plan.shards.size() != 1 || plan.dst.size() != 1))
        input_error("solver: the dense update path runs on an unsharded dataset");
    if (dense && !s0->num) {
        int64_t b = 0;
        s0->num = dalloc<double>(s0->ds->N, b, s0->stream);
        CUDA_TRY(cudaMemsetAsync(s0->num, 0, sizeof(double) * s0->ds->N, s0->stream));
    }
    DeviceGuard dg(s0->ds->device);
    // visit list of this cycle: order filtered by the skip rule
    // (solver.hpp:119-121: empty column and beta_j == 0)
    const bsccs_dataset* ds0 = s0->ds;
    const int32_t J = ds0->J;
    bool any_empty = false;
    for (int32_t j = 0; j < J; ++j) any_empty = any_empty || !ds0->col_nonempty_h[static_cast<size_t>(j)];
    std::vector<double> beta_h;
    if (any_empty) {
        beta_h.resize(static_cast<size_t>(J));
        CUDA_TRY(cudaMemcpyAsync(beta_h.data(), s0->beta, sizeof(double) * J, cudaMemcpyDeviceToHost, s0->stream));
        CUDA_TRY(cudaStreamSynchronize(s0->stream));
    }
    std::vector<int32_t> visit;
    visit.reserve(static_cast<size_t>(J));
    for (int32_t i = 0; i < J; ++i) {
        const int32_t j = s0->order_h.empty() ? i : s0->order_h[static_cast<size_t>(i)];
        if (ds0->col_nonempty_h[static_cast<size_t>(j)] || (any_empty && beta_h[static_cast<size_t>(j)] != 0.0))
            visit.push_back(j);
    }
    const RcdShape rcd = dense ? RcdShape{} : rcd_shape(plan);
    // the products of exp(beta) stay in range while max|beta| <= beta_limit
    auto beta_in_range = [&] {
        std::vector<double> b(static_cast<size_t>(J));
        CUDA_TRY(cudaMemcpyAsync(b.data(), s0->beta, sizeof(double) * J, cudaMemcpyDeviceToHost, s0->stream));
        CUDA_TRY(cudaStreamSynchronize(s0->stream));
        for (double x : b)
            if (!(std::fabs(x) <= rcd.beta_limit)) return false;
        return true;
    };
    bool use_rcd = rcd.ok && beta_in_range();
    int kinds = 0; // 1: k_ccd launched, 2: k_rcd launched
    for (auto* st : plan.shards) {
        if (use_rcd) { // compact denominators current; beta at the start of the cycle for the criterion
            sync_denc(st);
            CUDA_TRY(cudaMemcpyAsync(st->beta_prev, st->beta, sizeof(double) * J, cudaMemcpyDeviceToDevice,
                                     st->stream));
        } else {
            sync_x(st);
            prepare_snapshot(st);
        }
        if (!st->visit_valid || st->visit_h != visit) {
            st->visit_h = visit;
            st->visit_valid = true;
            if (!visit.empty()) {
                CUDA_TRY(cudaMemcpyAsync(st->visit, visit.data(), sizeof(int32_t) * visit.size(),
                                         cudaMemcpyHostToDevice, st->stream));
                const int64_t n = static_cast<int64_t>(visit.size()) * st->ds->ctas;
                k_build_vsplit<<<static_cast<int>((n + 255) / 256), 256, 0, st->stream>>>(
                    st->ds->split, st->visit, static_cast<int>(visit.size()), st->ds->ctas, st->vsplit);
                CUDA_TRY(cudaGetLastError());
                count_launches(1);
            }
        }
        if (st->stream != s0->stream) CUDA_TRY(cudaStreamSynchronize(st->stream));
    }
    if (s0->visit_h.size() != visit.size()) internal_error("visit list mismatch across shards");
    CUDA_TRY(cudaEventRecord(s0->ev0, s0->stream));
    // Launch from `begin`; a launch that stops before a coordinate whose sums
    // need refinement (res->refine_at) is followed by that coordinate on the
    // single-coordinate path and a relaunch after it.
    long long visited = 0, nmoved = 0;
    std::vector<std::pair<int, uint8_t>> refined; // (visit index, moved)
    int begin = 0;
    for (;;) {
        SweepArgs a = base_args(plan);
        a.mode = kModeSweep;
        a.visit_begin = begin;
        a.dbg = g_debug_flags;
        a.trace = g_trace;
        a.ntrace = g_ntrace;
        a.prior = prior;
        a.normalized = normalized ? 1 : 0;
        if (dense) {
            ensure_pq(s0->ds);
            a.sh[0].pq = s0->ds->pq;
            void* params[] = {&a};
            CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_ccd_dense), dim3(s0->ds->ctas), dim3(kDT),
                                                 params, 0, s0->stream));
            count_launches(1);
        } else if (use_rcd) {
            kinds |= 2;
            launch_rcd(plan, a, rcd);
            for (auto* st : plan.shards) st->x_stale = true;
        } else {
            kinds |= 1;
            launch_ccd(plan, a);
        }
        for (size_t i = 0; i < plan.shards.size(); ++i) {
            bsccs_state* st = plan.shards[i];
            CUDA_TRY(cudaMemcpyAsync(st->res_h, st->res, sizeof(DevResult), cudaMemcpyDeviceToHost, s0->stream));
        }
        CUDA_TRY(cudaStreamSynchronize(s0->stream));
        CUDA_TRY(cudaGetLastError());
        check_plan_errors(plan);
        visited += s0->res_h->visited;
        nmoved += s0->res_h->moved;
        const int ra = s0->res_h->refine_at;
        if (ra < 0) break;
        if (use_rcd) // the single-coordinate launches run on the subject blocks
            for (auto* st : plan.shards) sync_x(st);
        const bool mv = refine_coordinate(plan, prior, visit[static_cast<size_t>(ra)]);
        if (use_rcd) {
            for (auto* st : plan.shards) st->denc_valid = false;
            if (beta_in_range()) {
                for (auto* st : plan.shards) sync_denc(st);
            } else { // the rest of the cycle on k_ccd, its criterion against the cycle start
                use_rcd = false;
                const bsccs_dataset* d0 = s0->ds;
                for (auto* st : plan.shards) {
                    k_snap_from_beta<<<build_grid(d0->device), 256, 0, st->stream>>>(
                        st->snap, st->ds->csr_ptr, st->ds->csr_col, st->beta_prev, st->ds->K);
                    CUDA_TRY(cudaGetLastError());
                    count_launches(1);
                    st->snap_valid = true;
                }
            }
        }
        refined.emplace_back(ra, mv ? 1 : 0);
        ++visited;
        nmoved += mv ? 1 : 0;
        begin = ra + 1;
    }
    CUDA_TRY(cudaEventRecord(s0->ev1, s0->stream));
    g_last_sweep = kinds;
    std::vector<uint8_t> moved(visit.size());
    if (!visit.empty())
        CUDA_TRY(cudaMemcpyAsync(moved.data(), s0->moved, visit.size(), cudaMemcpyDeviceToHost, s0->stream));
    CUDA_TRY(cudaStreamSynchronize(s0->stream));
    for (const auto& r : refined) moved[static_cast<size_t>(r.first)] = r.second;
    for (auto* st : plan.shards) {
        if (use_rcd) { // X stays stale until an op reads it (sync_x)
            st->x_stale = true;
            st->snap_valid = false;
        } else {
            st->snap_valid = true;
            st->denc_valid = false;
        }
    }
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, s0->ev0, s0->ev1));
    s0->sweep_ms += ms;
    // SURVEY §8(d) algorithmic bytes of this sweep, every shard: per visited
    // coordinate 16*nnz_j + 12*u_j, per moved one + 28*nnz_j + 8*u_j, plus
    // 32*K for the criterion / snapshot pass
    const long long nv = visited;
    for (auto* st : plan.shards) {
        const bsccs_dataset* d = st->ds;
        double bytes = 32.0 * static_cast<double>(d->K);
        for (long long i = 0; i < nv && i < static_cast<long long>(visit.size()); ++i) {
            const size_t j = static_cast<size_t>(visit[static_cast<size_t>(i)]);
            const double nnz = static_cast<double>(d->col_ptr_h[j + 1] - d->col_ptr_h[j]);
            const double runs = static_cast<double>(d->col_runs_h[j]);
            bytes += 16.0 * nnz + 12.0 * runs;
            if (dense) { // the subject sweep; on a step the full rebuild (engine.hpp:68-90)
                bytes += 24.0 * static_cast<double>(d->N);
                if (moved[static_cast<size_t>(i)]) bytes += 16.0 * nnz + 16.0 * d->K + 8.0 * d->N;
            } else if (moved[static_cast<size_t>(i)]) {
                bytes += 28.0 * nnz + 8.0 * runs;
            }
        }
        s0->alg_bytes += bytes;
    }
    SweepOutcome out{0.0, 0, 0};
    out.criterion = s0->res_h->criterion;
    out.visited = visited;
    out.moved = nmoved;
    return out;
}

} // namespace bsccs_b200
