// batch.cu -- batched weighted multi-fit engine (placeholder)
#include "engine.h"
namespace bsccs_b200 {
void cv_folds_batched(const bsccs_dataset*, const bsccs_cv_config*, const std::vector<double>&,
                      const std::vector<int32_t>&, const std::vector<int32_t>&, int32_t, int32_t, bsccs_cv_cell*,
                      bsccs_cv_result*) {
    input_error("batched engine: not available");
}
void boot_replicates_batched(const bsccs_dataset*, const bsccs_bootstrap_config*, const double*, int32_t, int32_t,
                             double*, int32_t*, bsccs_bootstrap_result*) {
    input_error("batched engine: not available");
}
} // namespace bsccs_b200
