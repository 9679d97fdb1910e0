// minikv_reference_adapter_harness.cpp -- routes the reference's H2O comparison baseline
// (proj/core/include/minikv/harness.hpp:33-52, unchanged) to the B200 library: the step-wise
// greedy H2O policy runs on the device (csrc/h2o.cu, bit-identical kept sets) and
// persistence_analysis on its output.  Linked, like minikv_reference_adapter.cpp, in place
// of the reference's own definitions (harness.cpp:108-169); see dropin/Makefile.
#include "minikv/harness.hpp"
#include "minikv_b200.hpp"

namespace minikv {

H2OBaselineTrace h2o_dynamic_baseline(const Matrix& prompt_k, const Vector& prompt_scores,
                                      const std::vector<Vector>& decode_qs, const std::vector<Vector>& decode_ks,
                                      std::size_t hh_budget, std::size_t rw_budget, float scale) {
    minikv_b200::Matrix k(prompt_k.rows, prompt_k.cols);
    k.data = prompt_k.data;
    const auto t = minikv_b200::h2o_dynamic_baseline(k, prompt_scores, decode_qs, decode_ks, hh_budget, rw_budget,
                                                     scale);
    H2OBaselineTrace out;
    out.kept_per_step = t.kept_per_step;
    return out;
}

PersistenceReport persistence_analysis(const H2OBaselineTrace& trace, const std::vector<std::size_t>& prefill_hh) {
    minikv_b200::H2OBaselineTrace t;
    t.kept_per_step = trace.kept_per_step;
    const auto r = minikv_b200::persistence_analysis(t, prefill_hh);
    PersistenceReport out;
    out.fractions = r.fractions;
    out.final_fraction = r.final_fraction;
    return out;
}

}  // namespace minikv
