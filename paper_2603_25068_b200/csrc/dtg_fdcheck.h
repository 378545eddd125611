// Internal hooks of the FD-validation host layer (dtg_fdcheck.cpp) used by
// simulate_forward / simulate_gradient (dtg_host.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/dtg_engine.hpp"

namespace dtg {
namespace detail {

/// trace_branches, soft_choices or a surrogate: the run goes through the
/// instrumented device forward (dtg_probe.cu).
bool instrumented(const Scenario& s, const ForwardOptions& opt);
Trajectory forward_instrumented(const Scenario& s, const LinkParams& params, const RngStream& rng,
                                const ForwardOptions& opt);
/// Instrumented forward beside a gradient run: records the surrogate, checks
/// the soft-choice contract and returns the branch hash.  cum_final: the
/// gradient forward's result (must agree bit for bit).
std::uint64_t gradient_instrumentation(const Scenario& s, const LinkParams& params,
                                       const RngStream& rng, const ForwardOptions& opt,
                                       const std::vector<double>& cum_final);

}  // namespace detail
}  // namespace dtg
