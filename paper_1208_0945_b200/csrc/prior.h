// prior.h -- penalized Newton step and trust clamp, shared verbatim by the
// host (C ABI bsccs_penalized_step) and the persistent sweep kernel, so the
// step every CTA computes from the all-gathered (g, h) is the host's step.
//
// Restates prior.hpp:72-122 (penalized_step) and solver.hpp:131-150 (clamp,
// trust update).  Branch structure and expression forms are kept exactly so
// that fp64 results are bit-identical to the reference: -(g - beta/v)/(h - 1/v)
// for Normal; the BBR two-sided rule with an exact -beta on a zero crossing
// for Laplace; 0/0 -> 0 and g != 0, h == 0 -> numeric error for no prior.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define BSCCS_HD __host__ __device__ __forceinline__
#else
#define BSCCS_HD inline
#endif

namespace bsccs_b200 {

enum PriorCode { PRIOR_NONE = 0, PRIOR_NORMAL = 1, PRIOR_LAPLACE = 2 };

// Device error codes; the host maps them to bsccs_status.
enum DevError {
    DERR_NONE = 0,
    DERR_OVERFLOW = 1,          // numeric_error  engine.hpp:56-65
    DERR_DEN_NONPOSITIVE = 2,   // internal_error engine.hpp:116-118
    DERR_STEP_NONFINITE = 3,    // numeric_error  engine.hpp:210-212
    DERR_FLAT_NO_PRIOR = 4,     // numeric_error  prior.hpp:77-86
    DERR_POS_CURVATURE = 5,     // internal_error prior.hpp:73-75
    DERR_LL_DEN_NONPOSITIVE = 6, // internal_error engine.hpp:418-420
    DERR_SUM_RANGE = 7,          // exact exchange: a partial >= 2^43 or a total >= 2^48 (xchg.cuh)
    DERR_XCHG_TIMEOUT = 8        // exact exchange: a participant stopped publishing (peer rank gone)
};

struct PriorParams {
    int kind;
    double variance;
    double laplace_b; // prior.hpp:22-24, computed once on the host
    double inv_v;     // 1.0 / variance  (the reference's `1.0 / v`, prior.hpp:91)
    double inv_b;     // 1.0 / b         (`1.0 / b`, prior.hpp:110-116; sign / b == +-inv_b exactly)
};

// Host-side construction of the constants (identical IEEE results to the
// expressions they replace).
inline PriorParams make_prior_params(int kind, double variance, bool variance_is_scale) {
    PriorParams p;
    p.kind = kind;
    p.variance = variance;
    p.laplace_b = variance_is_scale ? variance : std::sqrt(variance / 2.0);
    p.inv_v = 1.0 / variance;
    p.inv_b = 1.0 / p.laplace_b;
    return p;
}

// beta_j / v, the only other division of the Normal step; it depends on
// beta_j alone, so the sweep computes it while the exchange is in flight.
BSCCS_HD double beta_over_v(const PriorParams& p, double beta_j) { return beta_j / p.variance; }

// penalized_step with the beta/prior-only divisions precomputed: bitwise
// the same branches and values as penalized_step (each replaced expression
// is the identical IEEE operation; (-1)/b == -(1/b) exactly).
BSCCS_HD int penalized_step_pre(const PriorParams& p, double beta_j, double bv, double g, double h, double* out) {
    if (h > 0.0) return DERR_POS_CURVATURE;
    if (p.kind == PRIOR_NONE) {
        if (h == 0.0) {
            if (g == 0.0) {
                *out = 0.0;
                return DERR_NONE;
            }
            return DERR_FLAT_NO_PRIOR;
        }
        *out = -g / h;
        return DERR_NONE;
    }
    if (p.kind == PRIOR_NORMAL) {
        *out = -(g - bv) / (h - p.inv_v);
        return DERR_NONE;
    }
    if (beta_j != 0.0) {
        if (h == 0.0) {
            *out = -beta_j;
            return DERR_NONE;
        }
        const double sb = beta_j > 0.0 ? p.inv_b : -p.inv_b;
        const double step = -(g - sb) / h;
        const double landed = beta_j + step;
        if ((beta_j > 0.0 && landed < 0.0) || (beta_j < 0.0 && landed > 0.0)) {
            *out = -beta_j;
            return DERR_NONE;
        }
        *out = step;
        return DERR_NONE;
    }
    if (h == 0.0) {
        *out = 0.0;
        return DERR_NONE;
    }
    const double up = -(g - p.inv_b) / h; // both one-sided trials, independent
    const double dn = -(g + p.inv_b) / h;
    if (up > 0.0) {
        *out = up;
        return DERR_NONE;
    }
    if (dn < 0.0) {
        *out = dn;
        return DERR_NONE;
    }
    *out = 0.0;
    return DERR_NONE;
}

// Returns DERR_NONE or the error code; *out receives the unbounded step.
BSCCS_HD int penalized_step(const PriorParams& p, double beta_j, double g, double h, double* out) {
    if (h > 0.0) return DERR_POS_CURVATURE;
    if (p.kind == PRIOR_NONE) {
        if (h == 0.0) {
            if (g == 0.0) {
                *out = 0.0;
                return DERR_NONE;
            }
            return DERR_FLAT_NO_PRIOR;
        }
        *out = -g / h;
        return DERR_NONE;
    }
    if (p.kind == PRIOR_NORMAL) {
        const double v = p.variance;
        *out = -(g - beta_j / v) / (h - 1.0 / v);
        return DERR_NONE;
    }
    const double b = p.laplace_b;
    if (beta_j != 0.0) {
        if (h == 0.0) {
            *out = -beta_j;
            return DERR_NONE;
        }
        const double sign = beta_j > 0.0 ? 1.0 : -1.0;
        const double step = -(g - sign / b) / h;
        const double landed = beta_j + step;
        if ((beta_j > 0.0 && landed < 0.0) || (beta_j < 0.0 && landed > 0.0)) {
            *out = -beta_j;
            return DERR_NONE;
        }
        *out = step;
        return DERR_NONE;
    }
    if (h == 0.0) {
        *out = 0.0;
        return DERR_NONE;
    }
    double step = -(g - 1.0 / b) / h;
    if (step > 0.0) {
        *out = step;
        return DERR_NONE;
    }
    step = -(g + 1.0 / b) / h;
    if (step < 0.0) {
        *out = step;
        return DERR_NONE;
    }
    *out = 0.0;
    return DERR_NONE;
}

// std::clamp(v, -r, r) (solver.hpp:135): v < lo ? lo : (hi < v ? hi : v).
BSCCS_HD double clamp_step(double v, double r) {
    const double lo = -r;
    return v < lo ? lo : (r < v ? r : v);
}

// std::max(2|delta|, r/2) (solver.hpp:150): (a < b) ? b : a.
BSCCS_HD double next_trust(double delta, double r) {
    const double a = 2.0 * (delta < 0.0 ? -delta : delta);
    const double b = r / 2.0;
    return a < b ? b : a;
}

} // namespace bsccs_b200
