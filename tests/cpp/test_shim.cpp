// Drop-in check of include/bsccs_b200_solver.hpp: the same call site with the
// namespace switched (bsccs::fit -> bsccs_b200::fit) on the reference's own
// Dataset / PriorSpec / SolverConfig types.  Built against the untouched
// reference headers (test infrastructure); run on the GPU box.
#include <bsccs/bsccs.hpp>
#include <bsccs_b200_solver.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>

int main() {
    bsccs::SimConfig sc;
    sc.subjects = 400;
    sc.drugs = 6;
    sc.min_eras = 2;
    sc.max_eras = 8;
    sc.prevalence = bsccs::uniform_prevalence(6, 0.3);
    sc.true_beta = {0.5, -0.3, 0.0, 0.2, 0.0, -0.6};
    sc.baseline_log_rate_mean = -3.0;
    sc.seed = 7;
    const bsccs::Dataset ds = bsccs::simulate(sc).dataset;
    bsccs::PriorSpec prior;
    prior.kind = bsccs::PriorKind::laplace;
    prior.variance = 0.5;
    bsccs::SolverConfig cfg;
    const bsccs::FitResult ref = bsccs::fit(ds, prior, cfg);
    const bsccs::FitResult dev = bsccs_b200::fit(ds, prior, cfg);
    int bad = dev.cycles_run != ref.cycles_run;
    for (std::size_t j = 0; j < ref.beta_map.size(); ++j) {
        const double r = ref.beta_map[j], d = dev.beta_map[j];
        if (r == 0.0 ? std::abs(d) > 1e-9 : std::abs(d - r) > 1e-6 * std::abs(r)) bad = 1;
    }
    if (std::abs(dev.log_posterior - ref.log_posterior) > 1e-8 * std::abs(ref.log_posterior)) bad = 1;
    // error mapping: a bad config raises the reference exception type
    bool threw = false;
    try {
        bsccs::SolverConfig badc;
        badc.epsilon = 0.0;
        bsccs_b200::fit(ds, prior, badc);
    } catch (const bsccs::input_error&) {
        threw = true;
    }
    // the many-fit callers: same call with the namespace switched, both engines
    bsccs::CVConfig cv;
    cv.folds = 4;
    cv.variance_grid = {0.01, 0.1, 1.0};
    cv.seed = 5;
    const bsccs::CVResult rcv = bsccs::grid_search_cv(ds, cv);
    bsccs::BootstrapConfig bc;
    bc.replicates = 5;
    bc.seed = 9;
    bc.prior.kind = bsccs::PriorKind::normal;
    bc.prior.variance = 0.1;
    const bsccs::BootstrapResult rbt = bsccs::run_bootstrap(ds, bc);
    const bsccs_b200::DeviceDataset dds(ds);
    for (int engine : {BSCCS_ENGINE_SUBSET, BSCCS_ENGINE_BATCHED}) {
        const bsccs::CVResult dcv = bsccs_b200::grid_search_cv(dds, cv, engine);
        if (dcv.selected_index != rcv.selected_index || dcv.total_cycles != rcv.total_cycles) bad = 1;
        for (std::size_t g = 0; g < rcv.cells.size(); ++g)
            for (std::size_t f = 0; f < rcv.cells[g].size(); ++f) {
                const double a = dcv.cells[g][f].predictive_ll, b = rcv.cells[g][f].predictive_ll;
                if (dcv.cells[g][f].cycles != rcv.cells[g][f].cycles || std::abs(a - b) > 1e-8 * std::abs(b)) bad = 1;
            }
        const bsccs::BootstrapResult dbt = bsccs_b200::run_bootstrap(dds, bc, engine);
        if (dbt.used != rbt.used || dbt.p_hat != rbt.p_hat) bad = 1;
        for (std::size_t j = 0; j < rbt.lower.size(); ++j) {
            const double lo = rbt.lower[j], up = rbt.upper[j];
            if (std::abs(dbt.lower[j] - lo) > std::max(1e-6 * std::abs(lo), 1e-9)) bad = 1;
            if (std::abs(dbt.upper[j] - up) > std::max(1e-6 * std::abs(up), 1e-9)) bad = 1;
        }
        std::printf("shim engine %d: cv selected %d/%d, bootstrap used %d/%d\n", engine, dcv.selected_index,
                    rcv.selected_index, dbt.used, rbt.used);
    }
    std::printf("shim: cycles %d/%d lp %.17g/%.17g threw=%d -> %s\n", dev.cycles_run, ref.cycles_run,
                dev.log_posterior, ref.log_posterior, threw, (!bad && threw) ? "OK" : "FAIL");
    return (!bad && threw) ? 0 : 1;
}
