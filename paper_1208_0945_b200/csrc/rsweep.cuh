// rsweep.cuh -- k_rcd, the resident-beta sweep (one persistent cooperative
// launch per CCD cycle, run_cycle solver.hpp:101-166).  ccd_kernels.cu
// includes it once per register-tile count (namespaces r3 / r1, RS_TILES).
// No include guard, by design.
//
// What changes against k_ccd (sweep_impl.cuh): the state has no per-era
// x'beta.  Every CTA holds beta and E_j = exp(beta_j) in shared memory (all
// CTAs of all ranks compute the identical step, so every copy stays
// identical), and a pair's l*exp(x'beta) is rebuilt when it is needed as
// l * (prod of E over the era's other drugs) * E_j -- the reference's
// l*exp(sum of beta) (engine.hpp:77-78,173-181) as a product of per-drug
// exponentials -- from the era's drug list, which travels with the pair
// record.  The only random-access state left is the per-subject
// denominator (8 B per subject: 77 MB at 10M, L2-resident), so a pair visit
// costs a streamed 32-B record instead of a random DRAM line, and no exp.
//
// Pair records (dataset rq, CSC order, 32 B): {subject index within the
// CTA's range, era length, other-drug count | n_i << 8, overflow offset,
// up to 8 other drugs of the era (u16, ascending)}; a CTA's slice of a
// column is contiguous, so one bulk copy (TMA, cp.async.bulk) per
// coordinate stages it in shared memory, two coordinates ahead.
//
// Numerics: the reference carries x'beta incrementally (x'beta += delta,
// engine.hpp:219-229) and l*exp(x'beta) from it; here l*exp(x'beta) is the
// product above.  The two agree to a few ulps (exp of a sum with rounded
// increments against a product of rounded exponentials).  The update is
// the reference's: fresh = l*exp(x'beta + delta) (the product with
// E_j' = exp(beta_j + delta)), den += fresh - old in pair order, the x'beta
// bound (engine.hpp:17-28) checked on exp(x'beta + delta).  Partial products
// stay in range while max|beta| * (largest era) <= 700 (ds->max_deg): the
// host runs the sweep only then, and a step that leaves that range stops
// the sweep (ST_REFINE) so the host finishes the cycle on k_ccd.

// experiment hooks (build_native(variant=...))
#ifndef RCD_DEN_EARLY
#define RCD_DEN_EARLY 0 // heads' denominator loads before (1) or after (0) the products
#endif
#ifndef RCD_TRACE
#define RCD_TRACE 0 // globaltimer phase stamps (scripts/trace_sweep.py builds the variant with 1)
#endif
#ifndef RCD_DIAG_NOCRIT
#define RCD_DIAG_NOCRIT 0
#endif
#ifndef RCD_DIAG_NODEN
#define RCD_DIAG_NODEN 0
#endif
#ifndef RCD_TREE_REDUCE
#define RCD_TREE_REDUCE 0 // 1: butterfly sum of the warps' partials in every shape (default: 16-warp shape only)
#endif
#ifndef RCD_OVF_PREFETCH
#define RCD_OVF_PREFETCH 1 // 16-B loads of drugs 9..16 issued before the inline products
#endif

// CTA shape of this instantiation: RS_THREADS threads (warp 0 the control
// warp), RS_TILES pair slots per data thread.  These shadow the k_ccd shape
// (kT, kD, kWarps and the slot mapping) inside this namespace.
constexpr int kT = RS_THREADS;
constexpr int kD = kT - 32;
constexpr int kWarps = kT / 32;
static_assert(kT % 32 == 0 && kT >= 64, "CTA shape");
__device__ __forceinline__ int data_warp() {
    const int w = static_cast<int>(threadIdx.x) >> 5;
    constexpr int kMates = (kWarps - 1) / 4; // warps 4, 8, ...: warp 0's scheduler mates take the last data ranks
    if ((w & 3) == 0) return (kWarps - 1 - kMates) + (w >> 2) - 1;
    return w - (w >> 2) - 1;
}
__device__ __forceinline__ int data_tid() { return data_warp() * 32 + (static_cast<int>(threadIdx.x) & 31); }
__device__ __forceinline__ int slot_pos(int v) { return v * kD + data_tid(); }

constexpr int kRT = RS_TILES;
constexpr int kRC = kRT * kD; // pairs a CTA stages per coordinate (largest slice this instantiation runs)
constexpr int kRBufs = 3;     // record buffers: coordinate idx, idx+1 (speculated), idx+2 (in flight)
constexpr int kHTab = 2048;   // touched-subject lookup entries (no subject tile)
#ifndef RCD_CBUFS
#define RCD_CBUFS 2
#endif
constexpr int kCBufs = RCD_CBUFS; // criterion chunk buffers (kCBufs - 1 chunks in flight)

struct RSmem {
    double stage[kRC];  // l*exp (grad/hess) or fresh - old (update), per pair slot
    double stageD[kRC]; // the update's fresh - old per pair slot (its own array: no barrier between the
                        // update's heads and the next coordinate's staging)
    int ssub[2][kRC];   // subject per slot, by coordinate parity (the repair searches the previous slice)
    double jden[kRC];   // no subject tile: the denominator each head of the previous update wrote
    double ra[kWarps], rb[kWarps];
    int re[kWarps];
    double delta, bnew, enew;
    int status;
    unsigned long long bar[kRBufs]; // mbarriers of the record buffers
    unsigned long long cbar[kCBufs]; // mbarriers of the criterion chunk buffers
    XPrev xpv[32];                  // warp 0: the exchange's running totals per lane between uses
};
constexpr size_t kRSmemBytes = (sizeof(RSmem) + 127) / 128 * 128;
constexpr size_t kRBufBytes = static_cast<size_t>(kRC) * sizeof(RRec);

// CTA reduction of (a, b, e); result in every lane of warp 0 (fixed order)
__device__ __forceinline__ void block_reduce_r(double& a, double& b, int& e, bool idle, RSmem& sm) {
    if (!idle) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
    } else {
        a = 0.0;
        b = 0.0;
    }
    e = __reduce_or_sync(0xffffffffu, e);
    if (lane_id() == 0) {
        sm.ra[warp_id()] = a;
        sm.rb[warp_id()] = b;
        sm.re[warp_id()] = e;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // warp 0 sums the warps' partials: a butterfly in the 16-warp shape
        // (config 3: 0.8% faster fit than the 16 serial adds; the 12-warp
        // shapes measured 1% slower with it)
        if constexpr (RCD_TREE_REDUCE || kWarps == 16) {
            static_assert(kWarps <= 16, "tree reduce over at most 16 warps");
            const int l = static_cast<int>(threadIdx.x & 15); // both half-warps alike
            double x = l < kWarps ? sm.ra[l] : 0.0, y = l < kWarps ? sm.rb[l] : 0.0;
            const int z = l < kWarps ? sm.re[l] : 0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {
                x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
                y = __dadd_rn(y, __shfl_xor_sync(0xffffffffu, y, o));
            }
            a = x;
            b = y;
            e = __reduce_or_sync(0xffffffffu, z);
        } else {
            double x = 0.0, y = 0.0;
            int z = 0;
#pragma unroll
            for (int i = 0; i < kWarps; ++i) {
                x = __dadd_rn(x, sm.ra[i]);
                y = __dadd_rn(y, sm.rb[i]);
                z |= sm.re[i];
            }
            a = x;
            b = y;
            e = z;
        }
    }
}

__device__ __forceinline__ bool r_slot_valid(int v, int n) { return slot_pos(v) < n && threadIdx.x >= 32; }

// Per-thread state of one coordinate's slots: the rebuilt x'beta and its
// l*exp, the head's denominator (no subject tile), and the record fields
// the later phases need.
struct RSpec {
    double pre[kRT], le[kRT], den[kRT]; // pre: product of E over the era's other drugs
    int ls[kRT], len[kRT]; // (n_i is read from the record where a head needs it)
    unsigned head; // bit v: slot v starts a subject run
    unsigned cont; // bit v: the next pair belongs to the same subject (multi-pair run)
    unsigned dep;  // bit v: the era also holds the coordinate visited just before (its x'beta waits for that step)
};

// exp(x'beta) of a pair without its own drug: the product of E over the
// era's other drugs in ascending order (the inline ones, then the overflow
// list); dep: one of them is `jdep`
__device__ __forceinline__ double r_pre(const RRec& r, const double* se, const uint16_t* __restrict__ rovf, int jdep,
                                        bool& dep) {
    const int cnt = r.meta & 0xff;
    double p = 1.0;
    dep = false;
    for (int i = 0; i < cnt; ++i) {
        const int d = i < kRInline ? r.o[i] : __ldg(rovf + r.ovf + (i - kRInline));
        p = __dmul_rn(p, se[d]);
        dep = dep || d == jdep;
    }
    return p;
}

// The coordinate `jn` (records in `rb`, n pairs) speculated while the
// previous coordinate's partials travel: every slot's product of E over the
// era's other drugs (the slots' chains interleaved; the drugs past the 8
// inline ones through the scalar r_pre), l*exp(x'beta) = l * (pre * E_jn),
// run heads, and (no subject tile) the heads' denominators.  dep marks the
// eras that also hold `jprev`, whose step is still in flight.
template <bool kSS>
__device__ __forceinline__ void r_speculate(const RRec* rb, int n, int jn, int jprev, int junit, const double* se,
                                            const uint16_t* __restrict__ rovf, const double* __restrict__ denc,
                                            int subj_base, uint64_t pol_keep, RSpec& P) {
    uint32_t w[kRT][4];
    int cnt[kRT], ovo[kRT];
    P.dep = 0u;
    P.head = 0u;
    P.cont = 0u;
    bool any_ovf = false;
    const uint32_t unit2 = static_cast<uint32_t>(junit) * 0x10001u; // two unit drugs (padding)
#pragma unroll
    for (int v = 0; v < kRT; ++v) {
        const bool ok = r_slot_valid(v, n);
        const uint4* q = reinterpret_cast<const uint4*>(rb + slot_pos(v));
        const uint4 a = ok ? q[0] : make_uint4(0xffffffffu, 0, 0, 0);
        const uint4 o = ok ? q[1] : make_uint4(unit2, unit2, unit2, unit2);
        P.ls[v] = static_cast<int>(a.x);
        P.len[v] = static_cast<int>(a.y);
        cnt[v] = static_cast<int>(a.z & 0xffu);
        // run head / continuation: static per slice, carried in the record
        // (meta bits 8 and 9, k_iota_flags); an empty slot reads 0
        P.head |= ((a.z >> 8) & 1u) << v;
        P.cont |= ((a.z >> 9) & 1u) << v;
        w[v][0] = o.x;
        w[v][1] = o.y;
        w[v][2] = o.z;
        w[v][3] = o.w;
        P.pre[v] = 1.0;
        any_ovf = any_ovf || cnt[v] > kRInline;
        ovo[v] = static_cast<int>(a.w);
    }
#if RCD_DEN_EARLY
    if constexpr (!kSS) {
#pragma unroll
        for (int v = 0; v < kRT; ++v)
            if ((P.head >> v) & 1u) P.den[v] = ld_keep(denc + subj_base + P.ls[v], pol_keep);
    }
#endif
    // drugs 9..16 of eras with more than 8 others: one 16-B load each, in
    // flight while the inline products run
    uint4 ov[kRT];
    if (RCD_OVF_PREFETCH && any_ovf) {
#pragma unroll
        for (int v = 0; v < kRT; ++v)
            if (cnt[v] > kRInline) ov[v] = __ldg(reinterpret_cast<const uint4*>(rovf + ovo[v]));
    }
    // the inline drugs (predicated: padding lanes issue no shared-memory
    // load -- measured faster than multiplying the unit drug's E = 1)
#pragma unroll
    for (int i = 0; i < kRInline; ++i) {
#pragma unroll
        for (int v = 0; v < kRT; ++v) {
            if (i < cnt[v]) {
                const int d = static_cast<int>((w[v][i >> 1] >> (16 * (i & 1))) & 0xffffu);
                P.pre[v] = __dmul_rn(P.pre[v], se[d]);
            }
        }
    }
    // eras holding jprev: a zero 16-bit lane of (drugs ^ jprev), two per word
    if (jprev >= 0) {
        const uint32_t jj = static_cast<uint32_t>(jprev) * 0x10001u;
#pragma unroll
        for (int v = 0; v < kRT; ++v) {
            uint32_t z = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t x = w[v][k] ^ jj;
                z |= (x - 0x00010001u) & ~x & 0x80008000u;
            }
            if (z) P.dep |= 1u << v;
        }
    }
    if (any_ovf) { // rare
#pragma unroll
        for (int v = 0; v < kRT; ++v) {
            if (cnt[v] <= kRInline) continue;
            if (!RCD_OVF_PREFETCH) ov[v] = __ldg(reinterpret_cast<const uint4*>(rovf + ovo[v]));
            const uint32_t x[4] = {ov[v].x, ov[v].y, ov[v].z, ov[v].w};
#pragma unroll
            for (int i = 0; i < 8; ++i) { // padded with the unit drug as well
                const int d = static_cast<int>((x[i >> 1] >> (16 * (i & 1))) & 0xffffu);
                P.pre[v] = __dmul_rn(P.pre[v], se[d]);
                if (d == jprev) P.dep |= 1u << v;
            }
            for (int i = kRInline + 8; i < cnt[v]; ++i) { // more than 16 other drugs
                const int d = __ldg(rovf + ovo[v] + (i - kRInline));
                P.pre[v] = __dmul_rn(P.pre[v], se[d]);
                if (d == jprev) P.dep |= 1u << v;
            }
        }
    }
    const double ej = se[jn];
#pragma unroll
    for (int v = 0; v < kRT; ++v) P.le[v] = __dmul_rn(__dmul_rn(P.pre[v], ej), static_cast<double>(P.len[v]));
#if !RCD_DEN_EARLY
    if constexpr (!kSS) {
#pragma unroll
        for (int v = 0; v < kRT; ++v)
#if RCD_DIAG_NODEN // diagnostic only (wrong results): no denominator gathers
            if ((P.head >> v) & 1u) P.den[v] = 20.0 * P.le[v];
#else
            if ((P.head >> v) & 1u) P.den[v] = ld_keep(denc + subj_base + P.ls[v], pol_keep);
#endif
    }
#endif
}

template <bool kSS>
__global__ void __launch_bounds__(kT, 1) k_rcd(const __grid_constant__ SweepArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    RSmem& sm = *reinterpret_cast<RSmem*>(smem_raw);
    // dynamic shared memory: RSmem | beta | exp(beta) | union { the sweep:
    // record buffers, subject tile or bitmaps ; the criterion: beta at
    // cycle start, two chunk buffers }
    double* sb = reinterpret_cast<double*>(smem_raw + kRSmemBytes);
    double* se = sb + A.beta_cap;
    unsigned char* uni = smem_raw + kRSmemBytes + 2 * static_cast<size_t>(A.beta_cap) * sizeof(double);
    RRec* rbuf = reinterpret_cast<RRec*>(uni);
    double* tile = reinterpret_cast<double*>(uni + kRBufs * kRBufBytes); // subject tile (kSS) or bitmaps (!kSS)
    int si = 0;
    while (si + 1 < A.nsh && static_cast<int>(blockIdx.x) >= A.sh[si + 1].cta_begin) ++si;
    const ShardArgs& S = A.sh[si];
    const int c = static_cast<int>(blockIdx.x) - S.cta_begin;
    const int tid = static_cast<int>(threadIdx.x);
    const bool w0 = tid < 32;
    const bool issuer = tid == 32; // stages the record buffers (a data thread: warp 0 polls)
    unsigned long long seq = *S.xcounter;
    int err = 0;
    double errv = 0.0;
    // the exchange's running totals live in shared memory between uses (warp
    // 0 only): registers held through the data warps' phases cost a spill
    if (w0) {
        XPrev pv{0ull, 0ull, 0ull, 0ull};
        xprev_load(S, pv);
        sm.xpv[tid] = pv;
    }
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const int subj_base = S.cta_subj[c];
    const int nsubj = S.cta_subj[c + 1] - subj_base;
    unsigned* bm0 = reinterpret_cast<unsigned*>(tile);
    unsigned* bm1 = bm0 + A.bm_words;
    // no subject tile: direct-mapped (subject, head position) of the last update's heads
    int2* htab = reinterpret_cast<int2*>(bm1 + A.bm_words);

    // beta into shared memory; the CTA's denominators into the tile
    for (int j = tid; j < A.J; j += kT) {
        const double b = S.beta[j];
        sb[j] = b;
        se[j] = exp(b);
    }
    if (tid == 0) se[A.J] = 1.0; // the unit drug (record padding)
    if constexpr (kSS) {
        for (int t = tid; t < nsubj; t += kT) tile[t] = S.denc[subj_base + t];
    } else {
        for (int i = tid; i < 2 * A.bm_words; i += kT) bm0[i] = 0u;
    }
    if (tid == 0) {
        for (int b = 0; b < kRBufs; ++b) mbar_init(&sm.bar[b], 1);
        for (int b = 0; b < kCBufs; ++b) mbar_init(&sm.cbar[b], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const int B0 = A.visit_begin;
    const int V = A.nvisit - B0;
    const longlong2* vs = S.vsplit + static_cast<size_t>(c) * static_cast<size_t>(A.nvisit) + B0;
    const int32_t* visit = A.visit + B0;
    long long nvisit = 0, nmoved = 0;
    int refine_at = -1;
    bool aborted = false;

    // stage coordinate i's records into buffer i % 3 (one bulk copy; every
    // use of a buffer completes exactly one phase of its mbarrier)
    auto stage = [&](int i) {
        const longlong2 sl = vs[i];
        const unsigned bytes = static_cast<unsigned>((sl.y - sl.x) * static_cast<long long>(sizeof(RRec)));
        unsigned long long* bar = &sm.bar[i % kRBufs];
        fence_proxy_async();
        mbar_arrive_tx(bar, bytes);
        if (bytes) bulk_g2s(rbuf + static_cast<size_t>(i % kRBufs) * kRC, S.rq + sl.x, bytes, bar, pol_stream);
    };
    auto wait_records = [&](int i) { mbar_wait(&sm.bar[i % kRBufs], static_cast<unsigned>((i / kRBufs) & 1)); };

    if (V > 0) {
        if (issuer) {
            stage(0);
            if (V > 1) stage(1);
        }
        int j = visit[0];
        double bj = 0.0, rj = 1.0, ydx = 0.0;
        if (w0) {
            bj = sb[j];
            rj = S.trust[j];
            ydx = A.y_dot_x[j];
        }
        RSpec P; // coordinate idx
        RSpec Q; // coordinate idx+1, speculated during idx's window
        int ncur = static_cast<int>(vs[0].y - vs[0].x);
        int nn1 = V > 1 ? static_cast<int>(vs[1].y - vs[1].x) : 0; // slice length of idx+1 (loaded a window ahead)
        if (!w0) {
            wait_records(0);
            r_speculate<kSS>(rbuf, ncur, j, -1, A.J, se, S.rovf, S.denc, subj_base, pol_keep, P);
        }
        bool moved_prev = false; // did coordinate idx-1 move (its x'beta / den repairs apply)
        int nprev = 0;
        // subjects whose touched bit the last update set (cleared one window later)
        int clr_sub[kRT];
        unsigned clr = 0u;
        // profiling only: globaltimer stamps per coordinate (scripts/trace_sweep.py)
        const size_t trs = static_cast<size_t>(gridDim.x) * kTr;
        unsigned long long* trb = (RCD_TRACE && A.trace != nullptr && (tid == 0 || tid == 32))
                                      ? A.trace + static_cast<size_t>(blockIdx.x) * kTr
                                      : nullptr;
#pragma unroll 1
        for (int idx = 0; idx < A.nvisit - A.visit_begin; ++idx) { // (bound from the parameters: no register held)
            const RRec* rc = rbuf + static_cast<size_t>(idx % kRBufs) * kRC;
            int* ssub = sm.ssub[idx & 1];
            const bool tr = RCD_TRACE && trb && idx < A.ntrace;
            if (tr && tid == 0) trb[idx * trs + 0] = gtimer();
            double gs = 0.0, hs = 0.0;
            // ---- repair the speculated values, stage, run sums -------------
            if (!w0) {
                if (moved_prev) { // eras that also hold the previous coordinate's drug
#pragma unroll
                    for (int v = 0; v < kRT; ++v) {
                        if ((P.dep >> v) & 1u) {
                            bool d;
                            P.pre[v] = r_pre(rc[slot_pos(v)], se, S.rovf, -1, d);
                            P.le[v] = __dmul_rn(__dmul_rn(P.pre[v], se[j]), static_cast<double>(P.len[v]));
                        }
                    }
                }
                if (tr && tid == 32) trb[idx * trs + 11] = gtimer();
#pragma unroll
                for (int v = 0; v < kRT; ++v) {
                    if (r_slot_valid(v, ncur)) {
                        sm.stage[slot_pos(v)] = P.le[v];
                        ssub[slot_pos(v)] = P.ls[v];
                    }
                }
            }
            // this barrier also orders the previous update's denominators,
            // marks and records before the reads below (no end-of-coordinate
            // barrier: the update stages its differences in its own array)
            __syncthreads();
            if (tr && tid == 32) trb[idx * trs + 12] = gtimer();
            if (!w0) {
                if (!kSS && moved_prev) { // heads whose subject the previous update touched
                    const int* sprev = sm.ssub[(idx + 1) & 1];
                    const unsigned* bmprev = (idx & 1) ? bm0 : bm1; // marks of coordinate idx-1
#pragma unroll
                    for (int v = 0; v < kRT; ++v) {
                        if (!((P.head >> v) & 1u)) continue;
                        const int s = P.ls[v];
                        if (!((bmprev[s >> 5] >> (s & 31)) & 1u)) continue;
                        int lo;
                        const int2 e = htab[s & (kHTab - 1)]; // direct-mapped (subject, head position)
                        if (e.x == s) {
                            lo = e.y;
                        } else { // evicted by a colliding subject: search the previous slice
                            int hi = nprev;
                            lo = 0;
                            while (lo < hi) {
                                const int mid = (lo + hi) >> 1;
                                if (sprev[mid] < s) lo = mid + 1;
                                else hi = mid;
                            }
                        }
                        P.den[v] = sm.jden[lo];
                    }
                }
#pragma unroll
                for (int v = 0; v < kRT; ++v) {
                    if (!((P.head >> v) & 1u)) continue;
                    const int pos = slot_pos(v);
                    const int s = P.ls[v];
                    double num = P.le[v];
                    if ((P.cont >> v) & 1u) { // a multi-pair run: the other pairs' l*exp in order
                        int q = pos + 1;
                        while (q < ncur && ssub[q] == s) num = __dadd_rn(num, sm.stage[q++]);
                    }
                    run_terms(num, kSS ? tile[s] : P.den[v], static_cast<int>(static_cast<unsigned>(rc[pos].meta) >> 16), gs,
                              hs, err);
                }
            }
            if (tr && tid == 32) trb[idx * trs + 13] = gtimer() + (gs == 1.2345 ? 1 : 0);
            if (err) record_error(S.err, err, errv);
            int e = err | ((bj != bj) || (rj != rj) ? 1 : 0);
            const bool idle = w0 || !__any_sync(0xffffffffu, slot_pos(0) < ncur);
            block_reduce_r(gs, hs, e, idle, sm);
            if (tr && tid == 0) trb[idx * trs + 1] = gtimer();
            if (w0) {
                XPrev pv = sm.xpv[tid];
                publish(A, S, c, seq, gs, hs, e, pv);
                sm.xpv[tid] = pv;
            }
            // ---- while the partials travel ------------------------------------
            const bool more = idx + 1 < V;
            const int jn = more ? visit[idx + 1] : 0;
            const int nnext = nn1;
            nn1 = idx + 2 < V ? static_cast<int>(vs[idx + 2].y - vs[idx + 2].x) : 0;
            if (!w0) {
                if (issuer && idx + 2 < V) stage(idx + 2);
                if constexpr (!kSS) { // the marks of idx-1 were read above: clear them for this update
                    unsigned* b = (idx & 1) ? bm0 : bm1;
#pragma unroll
                    for (int v = 0; v < kRT; ++v)
                        if ((clr >> v) & 1u) b[clr_sub[v] >> 5] = 0u;
                    clr = 0u;
                }
                if (tr && tid == 32) trb[idx * trs + 14] = gtimer();
                if (more) {
                    wait_records(idx + 1);
                    if (tr && tid == 32) trb[idx * trs + 15] = gtimer();
                    r_speculate<kSS>(rbuf + static_cast<size_t>((idx + 1) % kRBufs) * kRC, nnext, jn, j, A.J, se, S.rovf,
                                     S.denc, subj_base, pol_keep, Q);
                }
                if (tr && tid == 32) { // the stamp waits for the speculated values
                    double dep = 0.0;
#pragma unroll
                    for (int v = 0; v < kRT; ++v) dep += r_slot_valid(v, nnext) ? Q.le[v] : 0.0;
                    trb[idx * trs + 6] = gtimer() + (dep == 1.2345 ? 1 : 0);
                }
            } else {
                double bn = 0.0, rn = 1.0, yn = 0.0;
                if (more) {
                    bn = sb[jn];
                    rn = S.trust[jn];
                    yn = A.y_dot_x[jn];
                }
                const double bv = beta_over_v(A.prior, bj);
                double tg, th;
                int te = 0;
                unsigned inexact[2] = {0u, 0u};
                if (tr && tid == 0) trb[idx * trs + 4] = gtimer();
                XPrev pv = sm.xpv[tid];
                poll<false>(A, S.xslots, seq, pv, tg, th, te, tr ? trb + idx * trs + 5 : nullptr, inexact);
                sm.xpv[tid] = pv;
                int status = ST_OK;
                double delta = 0.0;
                if (te) {
                    status = ST_REMOTE_ERR;
                } else if ((inexact[0] | inexact[1]) &&
                           (needs_refine(tg, inexact[0], 0) || needs_refine(th, inexact[1], 0))) {
                    status = ST_REFINE; // the host finishes this coordinate (run_sweep)
                } else {
                    const double g = __dsub_rn(ydx, tg);
                    const double h = th == 0.0 ? 0.0 : -th;
                    double step = 0.0;
                    const int serr = penalized_step_pre(A.prior, bj, bv, g, h, &step);
                    if (serr) {
                        status = ST_STEP_ERR;
                        if (c == 0 && tid == 0) record_error(S.err, serr, h);
                    } else {
                        delta = clamp_step(step, rj);
                        if (delta != 0.0 && !isfinite(delta)) {
                            status = ST_NONFINITE;
                            if (c == 0 && tid == 0) record_error(S.err, DERR_STEP_NONFINITE, delta);
                        } else if (fabs(__dadd_rn(bj, delta)) > A.beta_limit) {
                            status = ST_REFINE; // partial products could leave range: the host takes over
                        }
                    }
                }
                if (tid == 0) {
                    const double bnew = __dadd_rn(bj, delta);
                    sm.delta = delta;
                    sm.bnew = bnew;
                    sm.enew = exp(bnew);
                    sm.status = status;
                    if (c == 0 && status == ST_OK) {
                        S.moved[B0 + idx] = delta != 0.0 ? 1 : 0;
                        S.beta[j] = __dadd_rn(bj, delta);
                        S.trust[j] = next_trust(delta, rj);
                    }
                }
                bj = bn;
                rj = rn;
                ydx = yn;
                if (tr && tid == 0) trb[idx * trs + 7] = gtimer();
            }
            ++seq;
            __syncthreads();
            if (tr && tid == 0) trb[idx * trs + 2] = gtimer();
            const int status = sm.status;
            const double delta = sm.delta;
            if (status != ST_OK) {
                aborted = true;
                // a bulk copy still in flight must land before the CTA exits
                if (issuer && idx + 2 < V) wait_records(idx + 2);
                if (status == ST_REMOTE_ERR && c == 0 && tid == 0) S.res->err_remote = 1;
                if (status == ST_REFINE) refine_at = B0 + idx;
                break;
            }
            ++nvisit;
            moved_prev = delta != 0.0;
            if (moved_prev) {
                ++nmoved;
                // beta_j in shared memory (the window's readers are past the
                // barrier; the update below does not read beta)
                const double enew = sm.enew;
                if (tid == 0) {
                    sb[j] = sm.bnew;
                    se[j] = enew;
                }
                // ---- sparse update (engine.hpp:205-231): updated = x'beta + delta,
                // fresh = l*exp(updated), den += fresh - old in pair order
                if (!w0) {
                    double diff[kRT];
#pragma unroll
                    for (int v = 0; v < kRT; ++v) {
                        const double x = __dmul_rn(P.pre[v], enew); // exp(x'beta + delta)
                        diff[v] = 0.0;
                        if (!r_slot_valid(v, ncur)) continue;
                        if (!(x >= kExpXbMin && x <= kExpXbMax)) { // |x'beta + delta| > 700
                            err = DERR_OVERFLOW;
                            errv = fabs(log(x));
                        } else {
                            diff[v] = __dsub_rn(__dmul_rn(x, static_cast<double>(P.len[v])), P.le[v]);
                        }
                    }
                    if (tr && tid == 32) trb[idx * trs + 8] = gtimer() + (diff[0] == 1.2345 ? 1 : 0);
#pragma unroll
                    for (int v = 0; v < kRT; ++v)
                        if (r_slot_valid(v, ncur)) sm.stageD[slot_pos(v)] = diff[v];
                }
                __syncthreads();
                if (tr && tid == 32) trb[idx * trs + 9] = gtimer();
                if (!w0) {
                    unsigned* bmcur = (idx & 1) ? bm1 : bm0;
                    double den[kRT];
#pragma unroll
                    for (int v = 0; v < kRT; ++v) { // run sums for every head first ...
                        if (!((P.head >> v) & 1u)) continue;
                        const int pos = slot_pos(v);
                        const int s = P.ls[v];
                        double dv = __dadd_rn(kSS ? tile[s] : P.den[v], sm.stageD[pos]);
                        if ((P.cont >> v) & 1u) {
                            int q = pos + 1;
                            while (q < ncur && ssub[q] == s) dv = __dadd_rn(dv, sm.stageD[q++]);
                        }
                        den[v] = dv;
                    }
#pragma unroll
                    for (int v = 0; v < kRT; ++v) { // ... then the stores
                        if (!((P.head >> v) & 1u)) continue;
                        const int s = P.ls[v];
                        if constexpr (kSS) {
                            tile[s] = den[v];
                        } else {
                            st_keep(S.denc + subj_base + s, den[v], pol_keep);
                            sm.jden[slot_pos(v)] = den[v];
                            // colliding subjects may race for an entry: either
                            // (subject, position) pair is valid, the reader checks the
                            // subject (an atomic exchange: one 8-B write, no torn pair)
                            atomicExch(reinterpret_cast<unsigned long long*>(&htab[s & (kHTab - 1)]),
                                       static_cast<unsigned long long>(static_cast<unsigned>(s)) |
                                           (static_cast<unsigned long long>(static_cast<unsigned>(slot_pos(v))) << 32));
                            atomicOr(&bmcur[s >> 5], 1u << (s & 31));
                            clr_sub[v] = s;
                        }
                    }
                    if constexpr (!kSS) clr = P.head;
                    if (tr && tid == 32) trb[idx * trs + 10] = gtimer();
                }
            }
            if (tr && tid == 0) trb[idx * trs + 3] = gtimer();
            P = Q;
            nprev = ncur;
            ncur = nnext;
            j = jn;
        }
        __syncthreads(); // the last update's writes
        if constexpr (kSS) { // the cycle's denominators back to HBM
            for (int t = tid; t < nsubj; t += kT) S.denc[subj_base + t] = tile[t];
        }
    }

    if (!aborted) {
        // criterion (solver.hpp:154-165): |x'beta - snapshot| over the CTA's
        // eras -- x'beta at the end minus x'beta at the start of the cycle,
        // taken as the sum of the era's coefficient changes (sbp).
        // The eras' drug lists stream through two chunk buffers (bulk
        // copies of the degrees and drugs of A.crit_E eras, one chunk ahead);
        // each thread sums crit_E / kT consecutive eras from its first era's
        // CSR offset.
        double ch = 0.0, mg = 0.0;
        const int e0 = S.cta_era[c], e1 = S.cta_era[c + 1];
        const int E = A.crit_E, cap = A.crit_cap, eper = E / kT;
        double* sbp = reinterpret_cast<double*>(uni);
        uint8_t* dbuf = reinterpret_cast<uint8_t*>(sbp + A.beta_cap);           // [kCBufs][E + 32]
        uint16_t* cbuf = reinterpret_cast<uint16_t*>(dbuf + kCBufs * (E + 32));  // [kCBufs][cap + 16]
        int64_t* cpt = reinterpret_cast<int64_t*>(cbuf + kCBufs * (cap + 16));   // [nch + 1] chunk drug offsets
        __syncthreads(); // the sweep's last readers of the union region are done
        // the cycle's change of each coefficient: an era's x'beta change is
        // their sum over its drugs (ascending, like x'beta itself)
        for (int jj = tid; jj < A.J; jj += kT) sbp[jj] = __dsub_rn(sb[jj], S.beta_prev[jj]);
        const int nch = RCD_DIAG_NOCRIT ? 0 : (e1 - e0 + E - 1) / E; // (diagnostic: no criterion)
        // every chunk's first drug, loaded once (not on each chunk's path)
        for (int i = tid; i <= nch; i += kT) cpt[i] = S.csr_ptr[min(e1, e0 + i * E)];
        __syncthreads();
        // chunk i: eras [a, b), drugs [ca, cb); staged when they fit the buffer
        auto crit_stage = [&](int i) {
            const int a = e0 + i * E, b = min(e1, a + E);
            const int64_t ca = cpt[i], cb = cpt[i + 1];
            const int a16 = a & ~15, b16 = (b + 15) & ~15;
            const int64_t ca8 = ca & ~7ll, cb8 = (cb + 7) & ~7ll;
            unsigned long long* bar = &sm.cbar[i % kCBufs];
            fence_proxy_async();
            const bool fits = cb8 - ca8 <= cap;
            const unsigned bytes = static_cast<unsigned>(b16 - a16) + (fits ? static_cast<unsigned>(2 * (cb8 - ca8)) : 0u);
            mbar_arrive_tx(bar, bytes);
            bulk_g2s(dbuf + (i % kCBufs) * (E + 32), S.edeg + a16, static_cast<unsigned>(b16 - a16), bar, pol_stream);
            if (fits) bulk_g2s(cbuf + (i % kCBufs) * (cap + 16), S.ecol + ca8, static_cast<unsigned>(2 * (cb8 - ca8)), bar,
                               pol_stream);
        };
        if (tid == 0) {
            for (int i = 0; i < kCBufs && i < nch; ++i) crit_stage(i);
        }
        __syncthreads(); // sbp
        // this thread's first drug in each chunk (its first era's CSR offset),
        // loaded one chunk ahead: no block scan of the degrees
        int64_t first = nch > 0 ? S.csr_ptr[min(e1, e0 + tid * eper)] : 0;
        for (int i = 0; i < nch; ++i) {
            const int a = e0 + i * E, b = min(e1, a + E);
            const int64_t ca = cpt[i];
            const int64_t cb = cpt[i + 1];
            const bool fits = ((cb + 7) & ~7ll) - (ca & ~7ll) <= cap;
            const int64_t mine = first;
            if (i + 1 < nch) first = S.csr_ptr[min(e1, a + E + tid * eper)];
            mbar_wait(&sm.cbar[i % kCBufs], static_cast<unsigned>((i / kCBufs) & 1));
            const uint8_t* dg = dbuf + (i % kCBufs) * (E + 32) + (a - (a & ~15));
            const uint16_t* cl = cbuf + (i % kCBufs) * (cap + 16) + (ca - (ca & ~7ll));
            // this thread's eras [k0, k1) of the chunk and their first drug
            const int k0 = min(b - a, tid * eper), k1 = min(b - a, k0 + eper);
            int off = static_cast<int>(mine - ca);
            if (!A.normalized) {
                for (int k = k0; k < k1; ++k) {
                    const int deg = dg[k];
                    double dx = 0.0;
                    if (fits && deg <= 8) {
                        // the era's gathers issued together, summed in order
                        double v[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) v[q] = q < deg ? sbp[cl[off + q]] : 0.0;
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (q < deg) dx = __dadd_rn(dx, v[q]);
                    } else {
                        for (int q = 0; q < deg; ++q) {
                            const int d = fits ? cl[off + q] : __ldg(S.ecol + ca + off + q);
                            dx = __dadd_rn(dx, sbp[d]);
                        }
                    }
                    off += deg;
                    ch = __dadd_rn(ch, fabs(dx));
                }
            } else { // normalized: also |x'beta| (solver.hpp:159-161)
                for (int k = k0; k < k1; ++k) {
                    const int deg = dg[k];
                    double dx = 0.0, xn = 0.0;
                    for (int q = 0; q < deg; ++q) {
                        const int d = fits ? cl[off + q] : __ldg(S.ecol + ca + off + q);
                        dx = __dadd_rn(dx, sbp[d]);
                        xn = __dadd_rn(xn, sb[d]);
                    }
                    off += deg;
                    ch = __dadd_rn(ch, fabs(dx));
                    mg = __dadd_rn(mg, fabs(xn));
                }
            }
            __syncthreads(); // the chunk buffer is free again
            if (tid == 0 && i + kCBufs < nch) crit_stage(i + kCBufs);
        }
        if (err) record_error(S.err, err, errv);
        int e = err;
        block_reduce_r(ch, mg, e, false, sm);
        XPrev pv = w0 ? sm.xpv[tid & 31] : XPrev{0ull, 0ull, 0ull, 0ull};
        publish(A, S, c, seq, ch, mg, e, pv);
        if (w0) {
            double tch, tmg;
            int te;
            poll(A, S.xslots, seq, pv, tch, tmg, te, nullptr);
            sm.xpv[tid] = pv;
            if (c == 0 && tid == 0) {
                S.res->change = tch;
                S.res->magnitude = tmg;
                S.res->criterion = A.normalized ? tch / (1.0 + tmg) : tch;
                S.res->err_remote = te;
            }
        }
        ++seq;
    }
    if (err) record_error(S.err, err, errv);
    if (c == 0 && tid == 0) {
        S.res->visited = nvisit;
        S.res->moved = nmoved;
        S.res->counter = seq;
        S.res->refine_at = refine_at;
        if (S.xowner) *S.xcounter = seq;
    }
    if (c == 0 && S.xowner && w0) xprev_store(S, sm.xpv[tid]);
}
