// sweep_impl.cuh -- the persistent sweep kernel k_ccd and the machinery
// whose shapes depend on the number of register tiles per data thread:
// shared memory, the cached slots, speculative records and their repair,
// the grad/hess and update phases.  ccd_kernels.cu includes it once per
// tile count, each into its own namespace (SWEEP_TILES): 3 tiles (1,056
// pairs per CTA and coordinate) in general, 1 tile (352 pairs) when every
// slice of the dataset fits -- fewer registers and less shared memory made
// the config-2 fit 10% faster.  No include guard, by design.

constexpr int kCached = SWEEP_TILES; // register tiles per data thread
constexpr int kCap = kCached * kD;   // pairs a CTA keeps in registers per coordinate
// the repair hash table holds every run head of a cached slice (at most kCap);
// a full table would make the insert probe spin forever
static_assert(kCap <= kHt, "repair hash table smaller than the register tiles (raise kHtBits)");

struct Smem {
    double stage[kCap]; // per-pair l*exp (grad/hess) or l*exp delta (update)
    int ssub[kCap];     // per-pair subject of the cached tiles
    // what the previous coordinate's update changed, for repairing the
    // speculatively gathered records of the next coordinate
    double jxb[kCap], jle[kCap], jden[kCap];
    int jrow[kCap], jsub[kCap];
    int htk[kHt], htv[kHt];
    double ra[kWarps], rb[kWarps];
    int re[kWarps];
    // broadcast of the exchange result / step decision by warp 0
    double ta, tb, delta;
    int te, status;
    // a subject run crossing a chunk edge of a streamed slice: its partial
    // numerator (grad/hess) or denominator (update), carried to the next chunk
    double cr_num, cr_den;
    int cr_on, cr_subj, cr_n, cr_ds;
};

// ---- CTA reduction -------------------------------------------------------------

// Reduce (a, b, e) over the CTA; result valid in every lane of warp 0 (each
// lane sums the warp partials in the same order, so the values agree).
// Warps with nothing to add (warp-uniform `idle`) skip the shuffle tree.
__device__ __forceinline__ void block_reduce(double& a, double& b, int& e, bool idle, Smem& sm) {
    if (!idle) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        e = __reduce_or_sync(0xffffffffu, e);
    } else {
        a = 0.0;
        b = 0.0;
        e = __reduce_or_sync(0xffffffffu, e);
    }
    if (lane_id() == 0) {
        sm.ra[warp_id()] = a;
        sm.rb[warp_id()] = b;
        sm.re[warp_id()] = e;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
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

struct Cached {
    PairSlot slot[kCached];
};

struct RawCached {
    RawSlot slot[kCached];
};

__device__ __forceinline__ void load_cached(const ShardArgs& S, int64_t p0, int64_t p1, Cached& C) {
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (warp_active(v, p0, p1)) C.slot[v] = load_slot(S.pq, p0 + slot_pos(v), p0, p1);
        else C.slot[v] = invalid_slot();
    }
}

__device__ __forceinline__ void issue_cached(const ShardArgs& S, int64_t p0, int64_t p1, RawCached& R) {
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (warp_active(v, p0, p1)) {
            R.slot[v] = issue_slot(S.pq, p0 + slot_pos(v), p0, p1);
        } else {
            R.slot[v].q = make_int4(-1, -1, 0, -1);
            R.slot[v].edge = -1;
            R.slot[v].first = false;
            R.slot[v].last_valid = false;
        }
    }
}

__device__ __forceinline__ void finalize_cached(const RawCached& R, Cached& C) {
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        // warp-uniform: a warp whose tile is empty has every lane invalid
        if (__any_sync(0xffffffffu, R.slot[v].q.x >= 0)) C.slot[v] = finalize_slot(R.slot[v]);
        else C.slot[v] = invalid_slot();
    }
}

// Per-lane records of the register tiles.  Every lane gathers its era's
// x'beta; run heads also gather their subject block's header {den, n} --
// in the same 128-B line as the era for nearly every pair (engine.h).  Runs
// are combined from shared memory in ascending pair order, so a head never
// issues a dependent global load unless its run spills past the register
// tiles.
struct HeadRegs {
    double xb[kCached], le[kCached], den[kCached];
    int n[kCached];
};

// loads only (the registers are consumed later): lets the speculative
// gathers ride through the exchange without holding up the step broadcast
template <bool kSS>
__device__ __forceinline__ void issue_records(const ShardArgs& S, const Cached& C, HeadRegs& H) {
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (slot_valid(C.slot[v])) {
            H.xb[v] = ld_x(S.X, C.slot[v].xs);
            if (!kSS && C.slot[v].head) {
                const Subj sr = ld_hdr(S.X, C.slot[v].ds);
                H.den[v] = sr.den;
                H.n[v] = sr.n;
            }
        }
    }
}

__device__ __forceinline__ void finish_records(const Cached& C, HeadRegs& H) {
#pragma unroll
    for (int v = 0; v < kCached; ++v)
        if (slot_valid(C.slot[v])) H.le[v] = lexp(C.slot[v].len, H.xb[v]);
}

template <bool kSS>
__device__ __forceinline__ void gather_records(const ShardArgs& S, const Cached& C, HeadRegs& H) {
    issue_records<kSS>(S, C, H);
    finish_records(C, H);
}

template <bool kSS>
__device__ __forceinline__ void prefetch_records(const ShardArgs& S, const RawCached& R) {
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (R.slot[v].q.x >= 0) {
            prefetch_l2(S.X + R.slot[v].q.x);
            if (!kSS && (R.slot[v].q.x ^ R.slot[v].q.y) >= kLineSlots) prefetch_l2(S.X + R.slot[v].q.y);
        }
    }
}

// Patch speculatively gathered records with what the previous coordinate's
// update wrote: a subject found in the table was touched, so its head takes
// the new denominator and any of its eras among the updated rows takes the
// new (x'beta, l*exp).  Shared-memory only.
// Touched-subject bitmaps (one bit per subject of the CTA's range, two
// alternating by coordinate parity): the update sets its heads' bits with one
// atomicOr each; the repair tests a bit and, for the few touched subjects,
// finds the run by binary search in the previous slice's subjects (a slice
// is in ascending subject order).  Used when the subject tile does not fit.
struct TouchBits {
    unsigned* b0; // even coordinates' marks
    unsigned* b1; // odd
    int base;
    __device__ __forceinline__ unsigned* of(int parity) const { return parity ? b1 : b0; }
};

template <bool kSS, bool kTouch>
__device__ __forceinline__ void repair(const Cached& C, HeadRegs& H, const Smem& sm, const SubjTile& T,
                                       int stamp_prev, const unsigned* bmprev = nullptr,
                                       int nprev = 0) {
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (!slot_valid(C.slot[v])) continue;
        const int s = C.slot[v].ls; // subject index within the CTA's range
        int val;
        if constexpr (kTouch) { // direct-mapped: the subject's entry carries the stamp of its last update
            const int2 tc = T.touch[s];
            if (tc.x != stamp_prev) continue;
            val = tc.y;
        } else if (bmprev) {
            const int t = s;
            if (!((bmprev[t >> 5] >> (t & 31)) & 1u)) continue;
            int lo = 0, hi = nprev; // first position of subject s in the previous slice
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sm.jsub[mid] < s) lo = mid + 1;
                else hi = mid;
            }
            int e = lo;
            while (e < nprev && sm.jsub[e] == s) ++e;
            val = lo | ((e - lo) << 16);
        } else {
            int h = ht_hash(s);
            int k;
            for (;;) {
                k = sm.htk[h];
                if (k == s || k == -1) break;
                h = (h + 1) & (kHt - 1);
            }
            if (k != s) continue;
            val = sm.htv[h];
        }
        const int posj = val & 0xffff, runj = val >> 16;
        if (!kSS && C.slot[v].head) H.den[v] = sm.jden[posj];
        const int row = C.slot[v].xs; // era identity: its slot
        for (int q = posj; q < posj + runj; ++q) {
            if (sm.jrow[q] == row) {
                H.xb[v] = sm.jxb[q];
                H.le[v] = sm.jle[q];
                break;
            }
        }
    }
}

template <bool kSS>
__device__ STREAM_FN GhAcc gh_streamed(const ShardArgs& S, int64_t p0, int64_t b0, int64_t p1, GhAcc acc,
                                             Smem& sm, const SubjTile T, const StreamBuf X) {
    const int4* __restrict__ pq = S.pq;
    double gs = acc.gs, hs = acc.hs;
    int err = acc.err;
    const int tid = static_cast<int>(threadIdx.x);
    for (int64_t b = b0; b < p1; b += X.cap) {
        const int ne = static_cast<int>(min(p1 - b, static_cast<int64_t>(X.cap)));
        __syncthreads(); // the previous chunk's readers of the buffer / carry are done
        int cr_on = 0, cr_subj = -1, cr_n = 0;
        double cr_num = 0.0, cr_den = 0.0;
        if (tid == 0) {
            cr_on = sm.cr_on;
            cr_subj = sm.cr_subj;
            cr_num = sm.cr_num;
            cr_den = sm.cr_den;
            cr_n = sm.cr_n;
            sm.cr_on = 0;
        }
        for (int q0 = tid; q0 < ne; q0 += kSU * kT) {
            int4 pr[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                if (q0 + u * kT < ne) pr[u] = ld_pq(pq + b + q0 + u * kT);
            double xb[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                if (q0 + u * kT < ne) xb[u] = ld_x(S.X, pr[u].x);
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const int q = q0 + u * kT;
                if (q < ne) {
                    X.x[q] = lexp(pr[u].z, xb[u]);
                    X.sub[q] = pr[u].w;
                }
            }
        }
        __syncthreads();
        const int before = b > p0 ? ld_pq_sub(pq + b - 1) : -1; // subject just before the chunk
        const int after = b + ne < p1 ? ld_pq_sub(pq + b + ne) : -1; // ... and just past it
        for (int q = tid; q < ne; q += kT) {
            const int s = X.sub[q];
            if ((q > 0 ? X.sub[q - 1] : before) == s) continue; // not a run head
            double num = 0.0;
            int e = q;
            while (e < ne && X.sub[e] == s) num = __dadd_rn(num, X.x[e++]);
            double den;
            int n;
            if constexpr (kSS) {
                den = T.den[s];
                n = T.n[s];
            } else {
                const Subj sr = ld_hdr(S.X, ld_pq(pq + b + q).y);
                den = sr.den;
                n = sr.n;
            }
            if (e == ne && after == s) {
                sm.cr_num = num;
                sm.cr_den = den;
                sm.cr_n = n;
                sm.cr_subj = s;
                sm.cr_on = 1;
            } else {
                run_terms(num, den, n, gs, hs, err);
            }
        }
        if (cr_on) { // thread 0: the run carried into this chunk
            double num = cr_num;
            int e = 0;
            while (e < ne && X.sub[e] == cr_subj) num = __dadd_rn(num, X.x[e++]);
            if (e == ne && after == cr_subj) {
                sm.cr_num = num;
                sm.cr_den = cr_den;
                sm.cr_n = cr_n;
                sm.cr_subj = cr_subj;
                sm.cr_on = 1;
            } else {
                run_terms(num, cr_den, cr_n, gs, hs, err);
            }
        }
    }
    return GhAcc{gs, hs, err};
}

// The sparse update of a streamed slice, same chunking: every lane updates
// its own era (engine.hpp:219-229) and stages fresh - old; heads (and the
// carried run) apply the differences to the denominator in pair order.
template <bool kSS>
__device__ STREAM_FN UpdErr update_streamed(const ShardArgs& S, int64_t p0, int64_t b0, int64_t p1, double d,
                                                  UpdErr ue, Smem& sm, const SubjTile T, const StreamBuf X) {
    const int4* __restrict__ pq = S.pq;
    int err = ue.err;
    double errv = ue.errv;
    const int tid = static_cast<int>(threadIdx.x);
    for (int64_t b = b0; b < p1; b += X.cap) {
        const int ne = static_cast<int>(min(p1 - b, static_cast<int64_t>(X.cap)));
        __syncthreads();
        int cr_on = 0, cr_subj = -1, cr_ds = 0;
        double cr_den = 0.0;
        if (tid == 0) {
            cr_on = sm.cr_on;
            cr_subj = sm.cr_subj;
            cr_den = sm.cr_den;
            cr_ds = sm.cr_ds;
            sm.cr_on = 0;
        }
        for (int q0 = tid; q0 < ne; q0 += kSU * kT) {
            int4 pr[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                if (q0 + u * kT < ne) pr[u] = ld_pq(pq + b + q0 + u * kT);
            double xb[kSU];
#pragma unroll
            for (int u = 0; u < kSU; ++u)
                if (q0 + u * kT < ne) xb[u] = ld_x(S.X, pr[u].x);
#pragma unroll
            for (int u = 0; u < kSU; ++u) {
                const int q = q0 + u * kT;
                if (q < ne) {
                    const double updated = __dadd_rn(xb[u], d);
                    double diff = 0.0;
                    if (!(fabs(updated) <= kXbBound)) {
                        err = DERR_OVERFLOW;
                        errv = fabs(updated);
                    } else {
                        diff = __dsub_rn(lexp(pr[u].z, updated), lexp(pr[u].z, xb[u]));
                        S.X[pr[u].x] = updated;
                    }
                    X.x[q] = diff;
                    X.sub[q] = pr[u].w;
                }
            }
        }
        __syncthreads();
        const int before = b > p0 ? ld_pq_sub(pq + b - 1) : -1;
        const int after = b + ne < p1 ? ld_pq_sub(pq + b + ne) : -1;
        for (int q = tid; q < ne; q += kT) {
            const int s = X.sub[q];
            if ((q > 0 ? X.sub[q - 1] : before) == s) continue;
            const int ds = kSS ? 0 : ld_pq(pq + b + q).y;
            double den = kSS ? T.den[s] : S.X[ds];
            int e = q;
            while (e < ne && X.sub[e] == s) den = __dadd_rn(den, X.x[e++]);
            if (e == ne && after == s) {
                sm.cr_den = den;
                sm.cr_subj = s;
                sm.cr_ds = ds;
                sm.cr_on = 1;
            } else if constexpr (kSS) {
                T.den[s] = den;
            } else {
                S.X[ds] = den;
            }
        }
        if (cr_on) {
            double den = cr_den;
            int e = 0;
            while (e < ne && X.sub[e] == cr_subj) den = __dadd_rn(den, X.x[e++]);
            if (e == ne && after == cr_subj) {
                sm.cr_den = den;
                sm.cr_subj = cr_subj;
                sm.cr_ds = cr_ds;
                sm.cr_on = 1;
            } else if constexpr (kSS) {
                T.den[cr_subj] = den;
            } else {
                S.X[cr_ds] = den;
            }
        }
    }
    return UpdErr{err, errv};
}

template <bool kSS, bool kST>
__device__ __forceinline__ void gh_compute(const ShardArgs& S, const Cached& C, int64_t p0, int64_t p1,
                                           const HeadRegs& H, double& gs, double& hs, int& err, Smem& sm,
                                           const SubjTile& T, const StreamBuf X) {
    const int4* __restrict__ pq = S.pq;
    const int ncached = static_cast<int>(min(p1 - p0, static_cast<int64_t>(kCap)));
    if (threadIdx.x == 0) sm.cr_on = 0;
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (slot_valid(C.slot[v])) {
            const int pos = slot_pos(v);
            sm.stage[pos] = H.le[v];
            sm.ssub[pos] = C.slot[v].ls;
        }
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < kCached; ++v) {
        if (C.slot[v].head) {
            double num = H.le[v];
            const int s = C.slot[v].ls;
            double den;
            int n;
            if constexpr (kSS) {
                den = T.den[s];
                n = T.n[s];
            } else {
                den = H.den[v];
                n = H.n[v];
            }
            if (C.slot[v].cont) {
                int q = slot_pos(v) + 1;
                while (q < ncached && sm.ssub[q] == s) num = __dadd_rn(num, sm.stage[q++]);
                if constexpr (kST) {
                    if (q == ncached && p0 + q < p1 && ld_pq_sub(pq + p0 + q) == s) {
                        // the run continues into the streamed part: carried there
                        sm.cr_num = num;
                        sm.cr_den = den;
                        sm.cr_n = n;
                        sm.cr_subj = s;
                        sm.cr_on = 1;
                        continue;
                    }
                }
            }
            run_terms(num, den, n, gs, hs, err);
        }
    }
    if constexpr (kST) {
        if (p1 - p0 > kCap) {
            const GhAcc a = gh_streamed<kSS>(S, p0, p0 + kCap, p1, GhAcc{gs, hs, err}, sm, T, X);
            gs = a.gs;
            hs = a.hs;
            err = a.err;
        }
    }
}

template <bool kSS, bool kST>
__device__ __forceinline__ void update_slice(const ShardArgs& S, const Cached& C, const HeadRegs& H, bool cached,
                                             int64_t p0, int64_t p1, double d, int& err, double& errv, Smem& sm,
                                             const SubjTile& T, const StreamBuf X, bool record = false,
                                             int* myht = nullptr, int stamp = 0, unsigned* bmcur = nullptr) {
    const int4* __restrict__ pq = S.pq;
    if (threadIdx.x == 0) sm.cr_on = 0;
    if (cached) {
        const int ncached = static_cast<int>(min(p1 - p0, static_cast<int64_t>(kCap)));
        // every lane updates its own era (engine.hpp:219-229) and stages
        // fresh - old for its run head
#pragma unroll
        for (int v = 0; v < kCached; ++v) {
            if (slot_valid(C.slot[v])) {
                const int pos = slot_pos(v);
                const double updated = __dadd_rn(H.xb[v], d);
                double diff = 0.0;
                if (!(fabs(updated) <= kXbBound)) {
                    err = DERR_OVERFLOW;
                    errv = fabs(updated);
                } else {
                    const double fresh = lexp(C.slot[v].len, updated);
                    diff = __dsub_rn(fresh, H.le[v]);
                    S.X[C.slot[v].xs] = updated;
                    if (record) {
                        sm.jxb[pos] = updated;
                        sm.jle[pos] = fresh;
                    }
                }
                if (record) {
                    sm.jrow[pos] = C.slot[v].xs;
                    if constexpr (!kSS) sm.jsub[pos] = C.slot[v].ls;
                }
                sm.stage[pos] = diff;
            }
        }
        __syncthreads();
        // heads apply the run's differences to the denominator in order
#pragma unroll
        for (int v = 0; v < kCached; ++v) {
            if (C.slot[v].head) {
                const int pos = slot_pos(v);
                const int s = C.slot[v].ls;
                int q = pos;
                double den = __dadd_rn(kSS ? T.den[s] : H.den[v], sm.stage[q++]);
                if (C.slot[v].cont) {
                    while (q < ncached && sm.ssub[q] == s) den = __dadd_rn(den, sm.stage[q++]);
                    if constexpr (kST) {
                        if (q == ncached && p0 + q < p1 && ld_pq_sub(pq + p0 + q) == s) {
                            // continues into the streamed part: carried there
                            sm.cr_den = den;
                            sm.cr_subj = s;
                            sm.cr_ds = C.slot[v].ds;
                            sm.cr_on = 1;
                            continue;
                        }
                    }
                }
                if constexpr (kSS) T.den[s] = den;
                else S.X[C.slot[v].ds] = den;
                if (record) { // publish (subject -> run) for the next coordinate's repair
                    if constexpr (kSS && !kST) {
                        T.touch[s] = make_int2(stamp, pos | ((q - pos) << 16));
                    } else {
                        if constexpr (!kSS) sm.jden[pos] = den;
                        if (!kSS && bmcur) {
                            atomicOr(&bmcur[s >> 5], 1u << (s & 31));
                        } else {
                            int h = ht_hash(s);
                            while (atomicCAS(&sm.htk[h], -1, s) != -1) h = (h + 1) & (kHt - 1);
                            sm.htv[h] = pos | ((q - pos) << 16);
                            myht[v] = h;
                        }
                    }
                }
            }
        }
    }
    if constexpr (kST) {
        const int64_t start = cached ? p0 + static_cast<int64_t>(kCap) : p0;
        if (start < p1) {
            const UpdErr u = update_streamed<kSS>(S, p0, start, p1, d, UpdErr{err, errv}, sm, T, X);
            err = u.err;
            errv = u.errv;
        }
    }
}

__device__ __forceinline__ bool any_slot(const Cached& C) {
    bool a = false;
#pragma unroll
    for (int v = 0; v < kCached; ++v) a = a || slot_valid(C.slot[v]);
    return a;
}

// ---- the persistent kernel ------------------------------------------------------


constexpr size_t kSmemSubjOffset = (sizeof(Smem) + 15) / 16 * 16;

// kSS: subject records in shared memory for the cycle.  kST: slices may
// exceed the register tiles (the streamed path is compiled in); the host
// picks kST = false when no slice of the dataset does, so the common case
// carries none of the streamed path's register pressure.
template <bool kSS, bool kST>
__global__ void __launch_bounds__(kSweepThreads, 1) k_ccd(const __grid_constant__ SweepArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    SubjTile T{nullptr, nullptr, 0};
    const StreamBuf X{reinterpret_cast<double*>(smem_raw + A.stream_off),
                      reinterpret_cast<int*>(smem_raw + A.stream_off + sizeof(double) * A.stream_cap), A.stream_cap};
    int si = 0;
    while (si + 1 < A.nsh && static_cast<int>(blockIdx.x) >= A.sh[si + 1].cta_begin) ++si;
    const ShardArgs& S = A.sh[si];
    const int c = static_cast<int>(blockIdx.x) - S.cta_begin;
    const int64_t* split_c = S.split + c;
    const int stride = S.ctas + 1;
    unsigned long long seq = *S.xcounter;
    int err = 0;
    double errv = 0.0;
    Cached C;
    HeadRegs H;
    XPrev pv{0ull, 0ull};
    if (A.mode != kModeUpdate) xprev_load(S, pv);

    if (A.mode == kModeUpdate) {
        const int j = A.single_j;
        const int64_t p0 = split_c[static_cast<int64_t>(j) * stride], p1 = split_c[static_cast<int64_t>(j) * stride + 1];
        if constexpr (kST) update_slice<false, true>(S, C, H, false, p0, p1, A.single_delta, err, errv, sm, T, X);
        if (err) record_error(S.err, err, errv);
        if (c == 0 && threadIdx.x == 0) S.beta[j] = __dadd_rn(S.beta[j], A.single_delta);
        return;
    }

    if (A.mode == kModeReduce) {
        // CTA 0 of the first local shard contributes this rank's values
        const bool src = (c == 0 && si == 0);
        const double a = src ? A.red_a : 0.0, b = src ? A.red_b : 0.0;
        publish(A, S, c, seq, a, b, 0, pv);
        if (threadIdx.x < 32) {
            double ta, tb;
            int te;
            poll(A, S.xslots, seq, pv, ta, tb, te, nullptr);
            if (c == 0 && threadIdx.x == 0) {
                S.res->change = ta;
                S.res->magnitude = tb;
                S.res->err_remote = te;
                if (S.xowner) *S.xcounter = seq + 1;
            }
            if (c == 0 && S.xowner) xprev_store(S, pv);
        }
        return;
    }

    if (A.mode == kModeGradHess) {
        const int j = A.single_j;
        const int64_t p0 = split_c[static_cast<int64_t>(j) * stride], p1 = split_c[static_cast<int64_t>(j) * stride + 1];
        load_cached(S, p0, p1, C);
        double gs = 0.0, hs = 0.0;
        gather_records<false>(S, C, H);
        gh_compute<false, kST>(S, C, p0, p1, H, gs, hs, err, sm, T, X);
        if (err) record_error(S.err, err, 0.0);
        block_reduce(gs, hs, err, false, sm);
        publish(A, S, c, seq, gs, hs, err, pv);
        if (threadIdx.x < 32) {
            double tg, th;
            int te;
            unsigned inexact[2];
            poll(A, S.xslots, seq, pv, tg, th, te, nullptr, inexact);
            BSCCS_REFINE(A, S.xslots, seq, pv, gs, hs, err, tg, th, te, inexact);
            if (c == 0 && threadIdx.x == 0) {
                S.res->g = __dsub_rn(A.y_dot_x[j], tg);
                S.res->h = th == 0.0 ? 0.0 : -th;
                S.res->err_remote = te;
                if (S.xowner) *S.xcounter = seq + 1;
            }
            if (c == 0 && S.xowner) xprev_store(S, pv);
        }
        return;
    }

    // ---- one full cycle -------------------------------------------------
    // Software pipeline over the visit list.  While coordinate idx's
    // partials travel: the pair slots of idx+2 load, and -- when both slices
    // fit the register tiles -- the era / subject records of idx+1 are
    // gathered speculatively.  The update of idx then records what it wrote
    // (shared memory + subject hash table) and idx+1 repairs the few records
    // it touched, so no HBM gather sits on the per-coordinate critical path.
    // Scalar work (exchange, penalized step, clamp) runs on warp 0 only and
    // is broadcast through shared memory at the one barrier that follows.
    long long nvisit = 0, nmoved = 0;
    // this launch runs the visit list from A.visit_begin (a restart after a
    // coordinate whose sums needed refinement, run_sweep) to its end
    const int B0 = A.visit_begin;
    const int V = A.nvisit - B0;
    const longlong2* vs = S.vsplit + static_cast<size_t>(c) * static_cast<size_t>(A.nvisit) + B0;
    const int32_t* visit = A.visit + B0;
    int refine_at = -1;
    bool aborted = false;
    const bool w0 = threadIdx.x < 32;
    if (V > 0) {
        for (int i = threadIdx.x; i < kHt; i += kT) sm.htk[i] = -1;
        TouchBits TB{nullptr, nullptr, 0};
        if (!kSS && A.bm_words > 0) {
            TB.base = S.cta_subj[c];
            TB.b0 = reinterpret_cast<unsigned*>(smem_raw + kSmemSubjOffset);
            TB.b1 = TB.b0 + A.bm_words;
            for (int i = threadIdx.x; i < 2 * A.bm_words; i += kT) TB.b0[i] = 0u;
        }
        int nprev = 0; // slice length of the previous coordinate (its record's extent)
        if constexpr (kSS) {
            T.base = S.cta_subj[c];
            const int ns = S.cta_subj[c + 1] - T.base;
            T.den = reinterpret_cast<double*>(smem_raw + kSmemSubjOffset);
            T.touch = kST ? nullptr : reinterpret_cast<int2*>(T.den + A.ss_cap);
            T.n = kST ? reinterpret_cast<int*>(T.den + A.ss_cap) : reinterpret_cast<int*>(T.touch + A.ss_cap);
            for (int t = threadIdx.x; t < ns; t += kT) {
                const Subj sr = ld_hdr(S.X, S.bstart[T.base + t]);
                T.den[t] = sr.den;
                T.n[t] = sr.n;
                if constexpr (!kST) T.touch[t] = make_int2(0, 0);
            }
        }
        const longlong2 z2 = make_longlong2(0, 0);
        longlong2 cur = vs[0];
        int j = visit[0];
        double bj = 0.0, rj = 1.0, ydx = 0.0;
        if (w0) {
            bj = S.beta[j];
            rj = S.trust[j];
            ydx = A.y_dot_x[j];
        }
        load_cached(S, cur.x, cur.y, C);
        longlong2 nxt = V > 1 ? vs[1] : z2;
        int jn = V > 1 ? visit[1] : 0;
        Cached N;
        load_cached(S, nxt.x, nxt.y, N);
        longlong2 nxt2 = V > 2 ? vs[2] : z2;
        HeadRegs SH;
        bool spec = false;
        int myht[kCached];
#pragma unroll
        for (int v = 0; v < kCached; ++v) myht[v] = -1;
        __syncthreads(); // hash table initialised
        const bool tr = A.trace != nullptr && threadIdx.x == 0;
        const bool trd = A.trace != nullptr && threadIdx.x == 32;
        unsigned long long* trbd = trd ? A.trace + static_cast<size_t>(blockIdx.x) * kTr : nullptr;
        unsigned long long* trb = tr ? A.trace + static_cast<size_t>(blockIdx.x) * kTr : nullptr;
        const size_t trs = static_cast<size_t>(gridDim.x) * kTr;
        for (int idx = 0; idx < V; ++idx) {
            const int64_t p0 = cur.x, p1 = cur.y;
            if (tr && idx < A.ntrace) trb[idx * trs + 0] = gtimer();
            double gs = 0.0, hs = 0.0;
            const bool active = any_slot(C) || (p1 - p0 > kCap);
            const bool idle = !__any_sync(0xffffffffu, active);
            if (!(A.dbg & 1)) {
                if (!idle) {
                    if (spec) {
                        if (A.dbg & 64) finish_records(C, H);
                        repair<kSS, kSS && !kST>(C, H, sm, T, idx, // stamps: coordinate idx-1 wrote idx
                                                 TB.b0 ? TB.of((idx + 1) & 1) : nullptr, nprev);
                    } else {
                        gather_records<kSS>(S, C, H);
                    }
                }
                gh_compute<kSS, kST>(S, C, p0, p1, H, gs, hs, err, sm, T, X);
            }
            if (err) record_error(S.err, err, errv);
            // The publish below must not be observable before this
            // coordinate's beta/trust loads complete (CTA 0 overwrites them
            // after the exchange): folding them into the published error
            // word makes the adds data-dependent on the loads.
            int e = err | ((bj != bj) || (rj != rj) ? 1 : 0);
            block_reduce(gs, hs, e, idle && !(A.dbg & 1) ? true : idle, sm);
            // every lookup of the previous coordinate's entries is done
#pragma unroll
            for (int v = 0; v < kCached; ++v) {
                if (myht[v] >= 0) {
                    sm.htk[myht[v]] = -1;
                    myht[v] = -1;
                }
            }
            if (tr && idx < A.ntrace) trb[idx * trs + 1] = gtimer();
            if (!(A.dbg & 4)) publish(A, S, c, seq, gs, hs, e, pv);
            if (TB.b0) { // the previous coordinate's marks were read above: clear them for the next update
                unsigned* b = TB.of((idx + 1) & 1);
                for (int i = threadIdx.x; i < A.bm_words; i += kT) b[i] = 0u;
            }
            // while the partials travel
            RawCached NR;
            // the speculative gathers go out first (they are on the critical
            // path), then idx+2's pairs, then the gathers are consumed
            const bool more = idx + 1 < V;
            const bool spec_next = more && !(A.dbg & 16) && (p1 - p0) <= kCap && (nxt.y - nxt.x) <= kCap;
            if (spec_next) issue_records<kSS>(S, N, SH);
            issue_cached(S, nxt2.x, nxt2.y, NR);
            if (spec_next && !(A.dbg & 64)) finish_records(N, SH);
            // ... and, once idx+2's pairs have landed, its records into L2, so
            // the speculative gathers of the next window hit L2, not HBM
            if (A.prefetch && more && (nxt.y - nxt.x) <= kCap && (nxt2.y - nxt2.x) <= kCap)
                prefetch_records<kSS>(S, NR);
            const longlong2 nxt3 = idx + 3 < V ? vs[idx + 3] : z2;
            int jn2 = 0;
            double bn = 0.0, rn = 1.0, yn = 0.0;
            if (w0) {
                if (more) {
                    bn = S.beta[jn];
                    rn = S.trust[jn];
                    yn = A.y_dot_x[jn];
                }
                jn2 = idx + 2 < V ? visit[idx + 2] : 0;
                if (tr && idx < A.ntrace) trb[idx * trs + 4] = gtimer();
                // exchange, then the scalar step (prior.hpp:72-122,
                // solver.hpp:131-150), broadcast with the next barrier
                const double bv = beta_over_v(A.prior, bj); // while the partials travel
                double tg, th;
                int te = 0;
                unsigned inexact[2] = {0u, 0u};
                if (A.dbg & 4) {
                    tg = gs;
                    th = hs;
                } else {
                    poll<!kSS>(A, S.xslots, seq, pv, tg, th, te, (tr && idx < A.ntrace) ? trb + idx * trs + 5 : nullptr,
                               inexact);
                }
                int status = ST_OK;
                double delta = 0.0;
                if (te) {
                    status = ST_REMOTE_ERR;
                } else if ((inexact[0] | inexact[1]) &&
                           (needs_refine(tg, inexact[0], 0) || needs_refine(th, inexact[1], 0))) {
                    // a sum below the exchange's resolution (degenerate fits only):
                    // stop here; the host refines this coordinate and restarts the
                    // sweep after it (run_sweep), keeping the refinement rounds out
                    // of this loop's code
                    status = ST_REFINE;
                } else {
                    const double g = __dsub_rn(ydx, tg);
                    const double h = th == 0.0 ? 0.0 : -th;
                    double step = 0.0;
                    const int serr = penalized_step_pre(A.prior, bj, bv, g, h, &step);
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
                        S.moved[B0 + idx] = delta != 0.0 ? 1 : 0;
                        S.beta[j] = __dadd_rn(bj, delta);
                        S.trust[j] = next_trust(delta, rj);
                    }
                }
            }
            if (!(A.dbg & 4)) ++seq;
            if (tr && idx < A.ntrace) trb[idx * trs + 7] = gtimer();
            if (trd && idx < A.ntrace) {
                // the stamp waits for the window's speculative gathers
                double dep = 0.0;
#pragma unroll
                for (int v = 0; v < kCached; ++v) dep += slot_valid(N.slot[v]) ? SH.le[v] : 0.0;
                trbd[idx * trs + 6] = gtimer() + (dep == 1.2345 ? 1 : 0);
            }
            __syncthreads();
            if (tr && idx < A.ntrace) trb[idx * trs + 2] = gtimer();
            const int status = sm.status;
            const double delta = sm.delta;
            if (status != ST_OK) {
                aborted = true;
                if (status == ST_REMOTE_ERR && c == 0 && threadIdx.x == 0) S.res->err_remote = 1;
                if (status == ST_REFINE) refine_at = B0 + idx;
                break;
            }
            ++nvisit;
            if (delta != 0.0) {
                ++nmoved;
                if (!(A.dbg & 2))
                    update_slice<kSS, kST>(S, C, H, true, p0, p1, delta, err, errv, sm, T, X, spec_next, myht,
                                           idx + 1, TB.b0 ? TB.of(idx & 1) : nullptr);
            }
            __syncthreads(); // slice writes of this coordinate before the next reads
            if (tr && idx < A.ntrace) trb[idx * trs + 3] = gtimer();
            C = N;
            finalize_cached(NR, N);
            H = SH;
            spec = spec_next;
            nprev = static_cast<int>(p1 - p0);
            cur = nxt;
            nxt = nxt2;
            nxt2 = nxt3;
            j = jn;
            jn = jn2;
            bj = bn;
            rj = rn;
            ydx = yn;
        }
        if constexpr (kSS) { // the cycle's denominators back to HBM (ordered by the loop's last barrier)
            const int ns = S.cta_subj[c + 1] - T.base;
            for (int t = threadIdx.x; t < ns; t += kT) S.X[S.bstart[T.base + t]] = T.den[t];
        }
    }

    if (!aborted) {
        // criterion (solver.hpp:154-165) over the CTA's eras, snapshot for
        // the next cycle taken in the same pass
        const int e0 = S.cta_era[c], e1 = S.cta_era[c + 1];
        double ch = 0.0, mg = 0.0;
        for (int k = e0 + static_cast<int>(threadIdx.x); k < e1; k += kT) {
            const double xb = S.X[S.row_slot[k]];
            ch = __dadd_rn(ch, fabs(__dsub_rn(xb, S.snap[k])));
            if (A.normalized) mg = __dadd_rn(mg, fabs(xb));
            S.snap[k] = xb;
        }
        if (err) record_error(S.err, err, errv);
        int e = err;
        block_reduce(ch, mg, e, false, sm);
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
    } else if (err) {
        record_error(S.err, err, errv);
    }
    if (err) record_error(S.err, err, errv);
    if (c == 0 && threadIdx.x == 0) {
        S.res->visited = nvisit;
        S.res->moved = nmoved;
        S.res->counter = seq;
        S.res->refine_at = refine_at;
        if (S.xowner) *S.xcounter = seq;
    }
    if (c == 0 && S.xowner) xprev_store(S, pv);
}

