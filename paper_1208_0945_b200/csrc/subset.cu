// subset.cu -- device-side subset_dataset (dataset.hpp:157-217) and the
// host-side subject selections that feed it: kfold_split
// (cross_validation.hpp:58-80) and resample (bootstrap.hpp:43-52).
//
// The reference rebuilds a subset by walking every column for every selected
// subject with a lower_bound (O(J * n * log nnz); 243 s for one 1M-patient
// bootstrap replicate).  Here the subset is produced from the
// parent's device-resident row-major copy (csr_ptr / csr_col):
//   1. k_sub_counts   per selected subject: era and pair counts
//   2. two scans      new subject offsets and each subject's first pair
//   3. k_sub_emit     per selected subject s, its eras in order and, per era,
//                     its drugs in ascending order: (j, new_row, s)
//   4. stable radix   sort by drug j -> CSC order.  The emission order is
//                     (s ascending, row ascending), so within a column the
//                     rows come out ascending exactly as the reference lays
//                     them out (dataset.hpp:197-216)
//   5. k_sub_colptr   column fences by binary search on the sorted keys
// and then the common device build (finish_dataset).  Layout and every
// integer of the result equal the reference's subset_dataset bit for bit.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>
#include <vector>

#include "devutil.h"
#include "engine.h"
#include "rng.h"

namespace bsccs_b200 {

namespace {

__global__ void k_sub_counts(const int32_t* __restrict__ sel, int64_t n, const int32_t* __restrict__ off,
                             const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ eps, int32_t N,
                             long long* ecnt, long long* pcnt, int32_t* out_eps, int* bad) {
    for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t i = sel[s];
        if (i < 0 || i >= N) {
            atomicOr(bad, 1);
            ecnt[s] = 0;
            pcnt[s] = 0;
            out_eps[s] = 0;
            continue;
        }
        const int32_t lo = off[i], hi = off[i + 1];
        ecnt[s] = hi - lo;
        pcnt[s] = csr_ptr[hi] - csr_ptr[lo];
        out_eps[s] = eps[i];
    }
}

// one thread per selected subject: its eras (lengths, counts) and its pairs
// in (row, drug) order -- keys are the drugs, values (new row, new subject)
__global__ void k_sub_emit(const int32_t* __restrict__ sel, int64_t n, const int32_t* __restrict__ off,
                           const int64_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_col,
                           const int32_t* __restrict__ len, const int32_t* __restrict__ y,
                           const long long* __restrict__ era_start, const long long* __restrict__ pair_start,
                           int32_t* out_off, int32_t* out_len, int32_t* out_y, uint32_t* keys, int2* vals) {
    for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t i = sel[s];
        const int32_t lo = off[i], hi = off[i + 1];
        const int32_t r0 = static_cast<int32_t>(era_start[s]);
        out_off[s] = r0;
        long long q = pair_start[s];
        for (int32_t k = lo; k < hi; ++k) {
            const int32_t row = r0 + (k - lo);
            out_len[row] = len[k];
            out_y[row] = y[k];
            for (int64_t c = csr_ptr[k]; c < csr_ptr[k + 1]; ++c, ++q) {
                keys[q] = static_cast<uint32_t>(csr_col[c]);
                vals[q] = make_int2(row, static_cast<int>(s));
            }
        }
    }
}

// col_ptr[j] = first sorted pair with drug >= j
__global__ void k_sub_colptr(const uint32_t* __restrict__ keys, int64_t nnz, int32_t J, int64_t* col_ptr) {
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (j > J) return;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] >= static_cast<uint32_t>(j)) hi = mid;
        else lo = mid + 1;
    }
    col_ptr[j] = lo;
}

__global__ void k_sub_split(const int2* __restrict__ vals, int64_t nnz, int32_t* rows, int32_t* subj) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int2 v = vals[p];
        rows[p] = v.x;
        subj[p] = v.y;
    }
}

__global__ void k_export_pairs(const int2* __restrict__ pairs, int64_t nnz, int32_t* rows, int32_t* subj) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int2 v = pairs[p];
        rows[p] = v.x;
        subj[p] = v.y;
    }
}

} // namespace

bsccs_dataset* dataset_subset(const bsccs_dataset* parent, const int32_t* subject_indices, int64_t n,
                              int ctas_override) {
    NvtxRange nvtx_("subset_dataset");
    if (!parent) input_error("subset_dataset: null dataset");
    if (n <= 0 || !subject_indices) input_error("subset_dataset: empty subject selection");
    if (n > 0x7fffffffll) input_error("subset_dataset: selection too large for int32 subject indices");
    DeviceGuard g(parent->device);
    const int device = parent->device;
    const int sms = sm_count(device);
    cudaStream_t ps = parent->stream;
    CUDA_TRY(cudaStreamSynchronize(ps));
    ensure_pool(device);
    // selection and counts on the parent's stream (its arrays are read there)
    int64_t tmpb = 0;
    int32_t* d_sel = dalloc<int32_t>(n, tmpb, ps);
    long long* d_ecnt = dalloc<long long>(n + 1, tmpb, ps);
    long long* d_pcnt = dalloc<long long>(n + 1, tmpb, ps);
    long long* d_estart = dalloc<long long>(n + 1, tmpb, ps);
    long long* d_pstart = dalloc<long long>(n + 1, tmpb, ps);
    int32_t* d_eps = dalloc<int32_t>(n, tmpb, ps);
    int* d_bad = dalloc<int>(1, tmpb, ps);
    auto free_tmp = [&]() {
        dfree(d_sel, ps);
        dfree(d_ecnt, ps);
        dfree(d_pcnt, ps);
        dfree(d_estart, ps);
        dfree(d_pstart, ps);
        dfree(d_eps, ps);
        dfree(d_bad, ps);
    };
    h2d(d_sel, subject_indices, sizeof(int32_t) * static_cast<size_t>(n), ps, device);
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), ps));
    CUDA_TRY(cudaMemsetAsync(d_ecnt + n, 0, sizeof(long long), ps));
    CUDA_TRY(cudaMemsetAsync(d_pcnt + n, 0, sizeof(long long), ps));
    k_sub_counts<<<grid_for(n, 256, sms), 256, 0, ps>>>(d_sel, n, parent->subject_offsets, parent->csr_ptr,
                                                         parent->events_per_subject, parent->N, d_ecnt, d_pcnt, d_eps,
                                                         d_bad);
    {
        size_t tb = 0;
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_ecnt, d_estart, n + 1, ps));
        unsigned char* tmp = dalloc<unsigned char>(static_cast<int64_t>(std::max<size_t>(tb, 16)), tmpb, ps);
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, d_ecnt, d_estart, n + 1, ps));
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, d_pcnt, d_pstart, n + 1, ps));
        dfree(tmp, ps);
    }
    count_launches(1);
    long long totals[2] = {0, 0};
    int bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&totals[0], d_estart + n, sizeof(long long), cudaMemcpyDeviceToHost, ps));
    CUDA_TRY(cudaMemcpyAsync(&totals[1], d_pstart + n, sizeof(long long), cudaMemcpyDeviceToHost, ps));
    CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ps));
    CUDA_TRY(cudaStreamSynchronize(ps));
    if (bad) {
        free_tmp();
        CUDA_TRY(cudaStreamSynchronize(ps));
        input_error("subset_dataset: subject index out of range");
    }
    const long long K2 = totals[0], nnz2 = totals[1];
    if (K2 > 0x7fffffffll) {
        free_tmp();
        CUDA_TRY(cudaStreamSynchronize(ps));
        input_error("subset_dataset: too many eras for int32 row indices");
    }
    const int32_t N2 = static_cast<int32_t>(n), J = parent->J;
    bsccs_dataset* ds = nullptr;
    try {
        ds = dataset_new(N2, static_cast<int32_t>(K2), J, nnz2, device, ctas_override);
        cudaStream_t s = ds->stream;
        // the new dataset's stream waits for the counts
        CUDA_TRY(cudaStreamSynchronize(ps));
        int64_t sb = 0;
        uint32_t* keys[2] = {dalloc<uint32_t>(nnz2, sb, s), dalloc<uint32_t>(nnz2, sb, s)};
        int2* vals[2] = {dalloc<int2>(nnz2, sb, s), dalloc<int2>(nnz2, sb, s)};
        k_sub_emit<<<grid_for(n, 128, sms), 128, 0, s>>>(
            d_sel, n, parent->subject_offsets, parent->csr_ptr, parent->csr_col, parent->era_lengths,
            parent->event_counts, d_estart, d_pstart, ds->subject_offsets, ds->era_lengths, ds->event_counts, keys[0],
            vals[0]);
        CUDA_TRY(cudaMemcpyAsync(ds->subject_offsets + N2, &d_estart[n], sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(ds->events_per_subject, d_eps, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
        count_launches(1);
        int sel_buf = 0;
        if (nnz2 > 0) {
            int end_bit = 1;
            while ((1ll << end_bit) < static_cast<long long>(J)) ++end_bit;
            cub::DoubleBuffer<uint32_t> dk(keys[0], keys[1]);
            cub::DoubleBuffer<int2> dv(vals[0], vals[1]);
            size_t tb = 0;
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, nnz2, 0, end_bit, s));
            unsigned char* tmp = dalloc<unsigned char>(static_cast<int64_t>(std::max<size_t>(tb, 16)), sb, s);
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, nnz2, 0, end_bit, s));
            dfree(tmp, s);
            sel_buf = dk.selector;
            if (dv.selector != sel_buf) internal_error("subset_dataset: sort buffers out of step");
        }
        k_sub_colptr<<<(J + 1 + 255) / 256, 256, 0, s>>>(keys[sel_buf], nnz2, J, ds->col_ptr);
        int32_t* d_rows = dalloc<int32_t>(nnz2, sb, s);
        int32_t* d_subj = dalloc<int32_t>(nnz2, sb, s);
        k_sub_split<<<grid_for(nnz2, 256, sms), 256, 0, s>>>(vals[sel_buf], nnz2, d_rows, d_subj);
        count_launches(2);
        ds->col_ptr_h.resize(static_cast<size_t>(J) + 1);
        CUDA_TRY(cudaMemcpyAsync(ds->col_ptr_h.data(), ds->col_ptr, sizeof(int64_t) * (J + 1), cudaMemcpyDeviceToHost,
                                 s));
        for (int b = 0; b < 2; ++b) {
            dfree(keys[b], s);
            dfree(vals[b], s);
        }
        CUDA_TRY(cudaStreamSynchronize(s));
        free_tmp();
        CUDA_TRY(cudaStreamSynchronize(ps));
        finish_dataset(ds, d_rows, d_subj, nullptr, nullptr, nullptr);
        ds->drug_ids = parent->drug_ids; // labels carried over unchanged (dataset.hpp:160-162)
    } catch (...) {
        if (ds) dataset_destroy(ds);
        throw;
    }
    return ds;
}

bsccs_dataset* dataset_from_row_pairs(int32_t N, int32_t K, int32_t J, int64_t nnz, const int32_t* subject_offsets,
                                      const int32_t* events_per_subject, const int32_t* era_lengths,
                                      const int32_t* event_counts, const uint32_t* drug, const int2* row_subj,
                                      int device, int ctas_override) {
    DeviceGuard g(device);
    const int sms = sm_count(device);
    bsccs_dataset* ds = dataset_new(N, K, J, nnz, device, ctas_override);
    try {
        cudaStream_t s = ds->stream;
        h2d(ds->subject_offsets, subject_offsets, sizeof(int32_t) * (static_cast<size_t>(N) + 1), s, device);
        h2d(ds->events_per_subject, events_per_subject, sizeof(int32_t) * N, s, device);
        h2d(ds->era_lengths, era_lengths, sizeof(int32_t) * K, s, device);
        h2d(ds->event_counts, event_counts, sizeof(int32_t) * K, s, device);
        int64_t sb = 0;
        uint32_t* keys[2] = {dalloc<uint32_t>(nnz, sb, s), dalloc<uint32_t>(nnz, sb, s)};
        int2* vals[2] = {dalloc<int2>(nnz, sb, s), dalloc<int2>(nnz, sb, s)};
        int sel = 0;
        if (nnz > 0) {
            h2d(keys[0], drug, sizeof(uint32_t) * static_cast<size_t>(nnz), s, device);
            h2d(vals[0], row_subj, sizeof(int2) * static_cast<size_t>(nnz), s, device);
            int end_bit = 1;
            while ((1ll << end_bit) < static_cast<long long>(J)) ++end_bit;
            cub::DoubleBuffer<uint32_t> dk(keys[0], keys[1]);
            cub::DoubleBuffer<int2> dv(vals[0], vals[1]);
            size_t tb = 0;
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, nnz, 0, end_bit, s));
            unsigned char* tmp = dalloc<unsigned char>(static_cast<int64_t>(std::max<size_t>(tb, 16)), sb, s);
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, nnz, 0, end_bit, s));
            dfree(tmp, s);
            sel = dk.selector;
        }
        k_sub_colptr<<<(J + 1 + 255) / 256, 256, 0, s>>>(keys[sel], nnz, J, ds->col_ptr);
        int32_t* d_rows = dalloc<int32_t>(nnz, sb, s);
        int32_t* d_subj = dalloc<int32_t>(nnz, sb, s);
        k_sub_split<<<grid_for(nnz, 256, sms), 256, 0, s>>>(vals[sel], nnz, d_rows, d_subj);
        count_launches(2);
        ds->col_ptr_h.resize(static_cast<size_t>(J) + 1);
        CUDA_TRY(cudaMemcpyAsync(ds->col_ptr_h.data(), ds->col_ptr, sizeof(int64_t) * (J + 1), cudaMemcpyDeviceToHost,
                                 s));
        for (int b = 0; b < 2; ++b) {
            dfree(keys[b], s);
            dfree(vals[b], s);
        }
        CUDA_TRY(cudaStreamSynchronize(s));
        finish_dataset(ds, d_rows, d_subj, nullptr, nullptr, nullptr);
    } catch (...) {
        dataset_destroy(ds);
        throw;
    }
    return ds;
}

void dataset_export(const bsccs_dataset* ds, int32_t* subject_offsets, int32_t* events_per_subject,
                    int32_t* era_lengths, int32_t* event_counts, int64_t* col_ptr, int32_t* rows, int32_t* subjects,
                    int64_t* y_dot_x) {
    if (!ds) input_error("null dataset");
    DeviceGuard g(ds->device);
    cudaStream_t s = ds->stream;
    CUDA_TRY(cudaStreamSynchronize(s));
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    d2h(subject_offsets, ds->subject_offsets, sizeof(int32_t) * (static_cast<size_t>(ds->N) + 1));
    d2h(events_per_subject, ds->events_per_subject, sizeof(int32_t) * static_cast<size_t>(ds->N));
    d2h(era_lengths, ds->era_lengths, sizeof(int32_t) * static_cast<size_t>(ds->K));
    d2h(event_counts, ds->event_counts, sizeof(int32_t) * static_cast<size_t>(ds->K));
    if (col_ptr) std::copy(ds->col_ptr_h.begin(), ds->col_ptr_h.end(), col_ptr);
    if ((rows || subjects) && ds->nnz > 0) {
        int64_t b = 0;
        int32_t* r = dalloc<int32_t>(ds->nnz, b, s);
        int32_t* q = dalloc<int32_t>(ds->nnz, b, s);
        k_export_pairs<<<grid_for(ds->nnz, 256, sm_count(ds->device)), 256, 0, s>>>(ds->pairs, ds->nnz, r, q);
        count_launches(1);
        d2h(rows, r, sizeof(int32_t) * static_cast<size_t>(ds->nnz));
        d2h(subjects, q, sizeof(int32_t) * static_cast<size_t>(ds->nnz));
        dfree(r, s);
        dfree(q, s);
    }
    std::vector<double> yd;
    if (y_dot_x) {
        yd.resize(static_cast<size_t>(ds->J));
        d2h(yd.data(), ds->y_dot_x, sizeof(double) * yd.size());
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    if (y_dot_x)
        for (int32_t j = 0; j < ds->J; ++j) y_dot_x[j] = static_cast<int64_t>(yd[static_cast<size_t>(j)]);
}

// kfold_split (cross_validation.hpp:58-80): Fisher-Yates over subject ids
// with Rng(seed).below(i), dealt round-robin.  subjects_out holds the fold
// lists back to back (fold f's list in the reference's order).
void kfold_split(int32_t N, int32_t folds, uint64_t seed, int32_t* subjects_out, int32_t* fold_sizes) {
    if (folds < 2) input_error("cross-validation needs at least 2 folds");
    if (folds > N) input_error("more folds than subjects");
    std::vector<int32_t> order(static_cast<size_t>(N));
    std::iota(order.begin(), order.end(), 0);
    Xoshiro rng(seed);
    for (size_t i = order.size(); i > 1; --i) {
        const size_t r = static_cast<size_t>(rng.below(i));
        std::swap(order[i - 1], order[r]);
    }
    std::vector<int32_t> start(static_cast<size_t>(folds) + 1, 0);
    for (int32_t f = 0; f < folds; ++f) {
        const int32_t sz = N / folds + (f < N % folds ? 1 : 0);
        if (fold_sizes) fold_sizes[f] = sz;
        start[static_cast<size_t>(f) + 1] = start[static_cast<size_t>(f)] + sz;
    }
    if (subjects_out) {
        std::vector<int32_t> fill(start.begin(), start.end() - 1);
        for (size_t i = 0; i < order.size(); ++i) {
            const size_t f = i % static_cast<size_t>(folds);
            subjects_out[fill[f]++] = order[i];
        }
    }
}

// resample (bootstrap.hpp:43-52) with the replicate's generator
// Rng(seed, stream) (bootstrap.hpp:104: stream = r + 1).
void resample(int32_t N, uint64_t seed, uint64_t stream, int32_t* out) {
    if (N < 1) input_error("resample: empty dataset");
    Xoshiro rng(seed, stream);
    for (int32_t s = 0; s < N; ++s) out[s] = static_cast<int32_t>(rng.below(static_cast<uint64_t>(N)));
}

} // namespace bsccs_b200
