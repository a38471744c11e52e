// datagen.cpp -- synthetic SCCS case series for parity tests and the bench.
//
// Two generators, both host-side and bit-reproducible from (seed, sizes):
//
//  * bsccs_synth_simulate restates the reference generative model
//    simulate() (simulate.hpp:50-137): attempted subject s draws from
//    Rng(seed, s+1) its frailty phi ~ N(mean, sd), an era count, and per era
//    a length, one Bernoulli(prevalence_j) exposure draw per drug, and
//    y ~ Poisson(length * exp(phi + x'beta)).  Zero-event subjects are
//    discarded; the survivors are laid out exactly as build_dataset does
//    (dataset.hpp:74-152).  O(K*J) draws: used for the config-1 oracle case.
//
//  * bsccs_synth_fast is the fast generator of SURVEY §8(d) for the 1M / 10M
//    configs: per era m = min(Poisson(lambda_x), J) distinct drugs drawn by
//    below(J) with rejection (uniform variant) or by a 1/(j+1) inverse-CDF
//    draw (Zipf variant), then sorted.  Subjects are generated in parallel
//    chunks, each subject from its own substream, and assembled in attempt
//    order, so the output does not depend on the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "rng.h"
#include "status.h"

struct bsccs_host_dataset {
    int32_t N = 0, K = 0, J = 0;
    int64_t nnz = 0;
    std::vector<int32_t> subject_offsets, events_per_subject, era_lengths, event_counts;
    std::vector<int32_t> rows, subjects;
    std::vector<int64_t> col_ptr, y_dot_x;
};

namespace bsccs_b200 {
namespace {

// Eras of a block of kept subjects in attempt order.
struct SubjectBlock {
    std::vector<int32_t> eras_per_subject;
    std::vector<int32_t> events_per_subject;
    std::vector<int32_t> era_len, era_y, era_ndrug;
    std::vector<int32_t> drugs; // concatenated, ascending within an era
};

// Assembles blocks (in order) into the CSC layout of build_dataset
// (dataset.hpp:162-189): rows numbered in subject order, each column's
// pairs in ascending row order, y_dot_x the event total over the column.
bsccs_host_dataset* assemble(std::vector<SubjectBlock>& blocks, int32_t J, int threads) {
    auto* out = new bsccs_host_dataset();
    out->J = J;
    const size_t B = blocks.size();
    std::vector<int64_t> subj_base(B + 1, 0), era_base(B + 1, 0);
    for (size_t b = 0; b < B; ++b) {
        subj_base[b + 1] = subj_base[b] + static_cast<int64_t>(blocks[b].eras_per_subject.size());
        era_base[b + 1] = era_base[b] + static_cast<int64_t>(blocks[b].era_len.size());
    }
    if (subj_base[B] == 0) {
        delete out;
        input_error("build_dataset: no subjects with events remain after exclusion");
    }
    if (era_base[B] >= std::numeric_limits<int32_t>::max()) {
        delete out;
        input_error("build_dataset: era count overflows the row index type");
    }
    out->N = static_cast<int32_t>(subj_base[B]);
    out->K = static_cast<int32_t>(era_base[B]);
    out->subject_offsets.resize(static_cast<size_t>(out->N) + 1);
    out->events_per_subject.resize(static_cast<size_t>(out->N));
    out->era_lengths.resize(static_cast<size_t>(out->K));
    out->event_counts.resize(static_cast<size_t>(out->K));

    // per-block column histograms and event sums
    std::vector<std::vector<int64_t>> ccount(B, std::vector<int64_t>(static_cast<size_t>(J), 0));
    std::vector<std::vector<int64_t>> cy(B, std::vector<int64_t>(static_cast<size_t>(J), 0));
    auto par = [&](auto&& fn) {
        std::vector<std::thread> pool;
        const int T = std::max(1, std::min<int>(threads, static_cast<int>(B)));
        for (int t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                for (size_t b = static_cast<size_t>(t); b < B; b += static_cast<size_t>(T)) fn(b);
            });
        }
        for (auto& th : pool) th.join();
    };
    par([&](size_t b) {
        const SubjectBlock& blk = blocks[b];
        size_t d = 0;
        for (size_t e = 0; e < blk.era_len.size(); ++e) {
            for (int32_t q = 0; q < blk.era_ndrug[e]; ++q, ++d) {
                ccount[b][static_cast<size_t>(blk.drugs[d])] += 1;
                cy[b][static_cast<size_t>(blk.drugs[d])] += blk.era_y[e];
            }
        }
    });
    out->col_ptr.assign(static_cast<size_t>(J) + 1, 0);
    out->y_dot_x.assign(static_cast<size_t>(J), 0);
    std::vector<std::vector<int64_t>> cpos(B, std::vector<int64_t>(static_cast<size_t>(J), 0));
    for (int32_t j = 0; j < J; ++j) {
        int64_t total = 0;
        for (size_t b = 0; b < B; ++b) {
            cpos[b][static_cast<size_t>(j)] = total;
            total += ccount[b][static_cast<size_t>(j)];
            out->y_dot_x[static_cast<size_t>(j)] += cy[b][static_cast<size_t>(j)];
        }
        out->col_ptr[static_cast<size_t>(j) + 1] = out->col_ptr[static_cast<size_t>(j)] + total;
    }
    out->nnz = out->col_ptr[static_cast<size_t>(J)];
    for (size_t b = 0; b < B; ++b)
        for (int32_t j = 0; j < J; ++j) cpos[b][static_cast<size_t>(j)] += out->col_ptr[static_cast<size_t>(j)];
    out->rows.resize(static_cast<size_t>(out->nnz));
    out->subjects.resize(static_cast<size_t>(out->nnz));
    out->subject_offsets[0] = 0;

    par([&](size_t b) {
        const SubjectBlock& blk = blocks[b];
        int64_t row = era_base[b];
        int64_t subj = subj_base[b];
        size_t e = 0, d = 0;
        auto& pos = cpos[b];
        for (size_t s = 0; s < blk.eras_per_subject.size(); ++s, ++subj) {
            for (int32_t q = 0; q < blk.eras_per_subject[s]; ++q, ++e, ++row) {
                out->era_lengths[static_cast<size_t>(row)] = blk.era_len[e];
                out->event_counts[static_cast<size_t>(row)] = blk.era_y[e];
                for (int32_t r = 0; r < blk.era_ndrug[e]; ++r, ++d) {
                    const int64_t p = pos[static_cast<size_t>(blk.drugs[d])]++;
                    out->rows[static_cast<size_t>(p)] = static_cast<int32_t>(row);
                    out->subjects[static_cast<size_t>(p)] = static_cast<int32_t>(subj);
                }
            }
            out->subject_offsets[static_cast<size_t>(subj) + 1] = static_cast<int32_t>(row);
            out->events_per_subject[static_cast<size_t>(subj)] = blk.events_per_subject[s];
        }
    });
    return out;
}

int hw_threads(int requested) {
    if (requested > 0) return requested;
    const unsigned h = std::thread::hardware_concurrency();
    return h == 0 ? 1 : static_cast<int>(h);
}

} // namespace
} // namespace bsccs_b200

using namespace bsccs_b200;

extern "C" bsccs_status bsccs_synth_simulate(
    int32_t subjects, int32_t drugs, int32_t min_eras, int32_t max_eras,
    int32_t min_era_length, int32_t max_era_length, const double* prevalence,
    const double* true_beta, double baseline_log_rate_mean, double baseline_log_rate_sd,
    uint64_t seed, bsccs_host_dataset** out) {
    return guard([&] {
        // argument checks in the order of simulate.hpp:51-77
        if (subjects < 1) input_error("simulate: need at least one subject");
        if (drugs < 1) input_error("simulate: need at least one drug");
        if (min_eras < 1 || max_eras < min_eras) input_error("simulate: era count bounds are invalid");
        if (min_era_length < 1 || max_era_length < min_era_length)
            input_error("simulate: era length bounds are invalid");
        if (prevalence == nullptr) input_error("simulate: prevalence must list one value per drug");
        for (int32_t j = 0; j < drugs; ++j)
            if (!(prevalence[j] > 0.0 && prevalence[j] < 1.0))
                input_error("simulate: prevalence values must lie in (0, 1)");
        if (true_beta == nullptr) input_error("simulate: true_beta must list one value per drug");
        if (!(baseline_log_rate_sd >= 0.0)) input_error("simulate: baseline rate spread must be non-negative");

        std::vector<SubjectBlock> blocks(1);
        SubjectBlock& blk = blocks[0];
        for (int s = 0; s < subjects; ++s) {
            Xoshiro rng(seed, static_cast<std::uint64_t>(s) + 1);
            const double phi = rng.normal(baseline_log_rate_mean, baseline_log_rate_sd);
            const int eras = rng.uniform_int(min_eras, max_eras);
            const size_t era0 = blk.era_len.size(), drug0 = blk.drugs.size();
            int32_t total = 0;
            for (int e = 0; e < eras; ++e) {
                const int32_t len = rng.uniform_int(min_era_length, max_era_length);
                double xb = 0.0;
                int32_t nd = 0;
                for (int32_t j = 0; j < drugs; ++j) {
                    if (rng.uniform() < prevalence[j]) {
                        blk.drugs.push_back(j);
                        xb += true_beta[j];
                        ++nd;
                    }
                }
                const double mean = static_cast<double>(len) * std::exp(phi + xb);
                const int32_t y = rng.poisson(mean);
                total += y;
                blk.era_len.push_back(len);
                blk.era_y.push_back(y);
                blk.era_ndrug.push_back(nd);
            }
            if (total == 0) { // discarded: roll back this subject's eras
                blk.era_len.resize(era0);
                blk.era_y.resize(era0);
                blk.era_ndrug.resize(era0);
                blk.drugs.resize(drug0);
                continue;
            }
            blk.eras_per_subject.push_back(eras);
            blk.events_per_subject.push_back(total);
        }
        if (blk.eras_per_subject.empty())
            input_error("simulate: every subject drew zero events; raise "
                        "baseline_log_rate_mean or lengthen the eras");
        *out = assemble(blocks, drugs, 1);
    });
}

extern "C" bsccs_status bsccs_synth_fast(int64_t attempts, int32_t drugs, double lambda_x,
                                         int32_t zipf, uint64_t seed, int32_t threads,
                                         bsccs_host_dataset** out) {
    return guard([&] {
        if (attempts < 1) input_error("synth_fast: need at least one subject");
        if (drugs < 1) input_error("synth_fast: need at least one drug");
        if (!(lambda_x >= 0.0)) input_error("synth_fast: lambda_x must be non-negative");
        const int T = hw_threads(threads);
        // planted signal: beta[p*(J/10)] = +0.7 (p even) / -0.5 (p odd), p=0..9
        std::vector<double> beta(static_cast<size_t>(drugs), 0.0);
        const int32_t stride = drugs >= 10 ? drugs / 10 : 1;
        for (int p = 0; p < 10; ++p) {
            const int64_t j = static_cast<int64_t>(p) * stride;
            if (j < drugs) beta[static_cast<size_t>(j)] = (p % 2 == 0) ? 0.7 : -0.5;
        }
        std::vector<double> cdf;
        if (zipf) {
            cdf.resize(static_cast<size_t>(drugs));
            double acc = 0.0;
            for (int32_t j = 0; j < drugs; ++j) {
                acc += 1.0 / static_cast<double>(j + 1);
                cdf[static_cast<size_t>(j)] = acc;
            }
        }
        const int64_t nblocks = std::min<int64_t>(attempts, static_cast<int64_t>(T) * 8);
        std::vector<SubjectBlock> blocks(static_cast<size_t>(nblocks));
        auto gen_block = [&](int64_t b) {
            const int64_t a0 = attempts * b / nblocks, a1 = attempts * (b + 1) / nblocks;
            SubjectBlock& blk = blocks[static_cast<size_t>(b)];
            std::vector<int32_t> era_drugs;
            for (int64_t s = a0; s < a1; ++s) {
                Xoshiro rng(seed, static_cast<std::uint64_t>(s) + 1);
                const double phi = rng.normal(-5.0, 0.5);
                const int eras = rng.uniform_int(10, 20);
                const size_t era0 = blk.era_len.size(), drug0 = blk.drugs.size();
                int32_t total = 0;
                for (int e = 0; e < eras; ++e) {
                    const int32_t len = rng.uniform_int(10, 60);
                    const int32_t m = std::min<int32_t>(rng.poisson(lambda_x), drugs);
                    era_drugs.clear();
                    while (static_cast<int32_t>(era_drugs.size()) < m) {
                        int32_t d;
                        if (zipf) {
                            const double u = rng.uniform() * cdf.back();
                            d = static_cast<int32_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
                            if (d >= drugs) d = drugs - 1;
                        } else {
                            d = static_cast<int32_t>(rng.below(static_cast<std::uint64_t>(drugs)));
                        }
                        if (std::find(era_drugs.begin(), era_drugs.end(), d) == era_drugs.end())
                            era_drugs.push_back(d);
                    }
                    std::sort(era_drugs.begin(), era_drugs.end());
                    double xb = 0.0;
                    for (int32_t d : era_drugs) xb += beta[static_cast<size_t>(d)];
                    const int32_t y = rng.poisson(static_cast<double>(len) * std::exp(phi + xb));
                    total += y;
                    blk.era_len.push_back(len);
                    blk.era_y.push_back(y);
                    blk.era_ndrug.push_back(m);
                    blk.drugs.insert(blk.drugs.end(), era_drugs.begin(), era_drugs.end());
                }
                if (total == 0) {
                    blk.era_len.resize(era0);
                    blk.era_y.resize(era0);
                    blk.era_ndrug.resize(era0);
                    blk.drugs.resize(drug0);
                    continue;
                }
                blk.eras_per_subject.push_back(eras);
                blk.events_per_subject.push_back(total);
            }
        };
        {
            std::vector<std::thread> pool;
            for (int t = 0; t < T; ++t)
                pool.emplace_back([&, t] {
                    for (int64_t b = t; b < nblocks; b += T) gen_block(b);
                });
            for (auto& th : pool) th.join();
        }
        *out = assemble(blocks, drugs, T);
    });
}

extern "C" bsccs_status bsccs_host_dataset_sizes(const bsccs_host_dataset* h, int64_t out[4]) {
    return guard([&] {
        if (!h) input_error("null host dataset");
        out[0] = h->N;
        out[1] = h->K;
        out[2] = h->J;
        out[3] = h->nnz;
    });
}

extern "C" bsccs_status bsccs_host_dataset_arrays(const bsccs_host_dataset* h,
                                                  const int32_t** subject_offsets,
                                                  const int32_t** events_per_subject,
                                                  const int32_t** era_lengths,
                                                  const int32_t** event_counts,
                                                  const int64_t** col_ptr, const int32_t** rows,
                                                  const int32_t** subjects,
                                                  const int64_t** y_dot_x) {
    return guard([&] {
        if (!h) input_error("null host dataset");
        *subject_offsets = h->subject_offsets.data();
        *events_per_subject = h->events_per_subject.data();
        *era_lengths = h->era_lengths.data();
        *event_counts = h->event_counts.data();
        *col_ptr = h->col_ptr.data();
        *rows = h->rows.data();
        *subjects = h->subjects.data();
        *y_dot_x = h->y_dot_x.data();
    });
}

extern "C" bsccs_status bsccs_host_dataset_destroy(bsccs_host_dataset* h) {
    return guard([&] { delete h; });
}
