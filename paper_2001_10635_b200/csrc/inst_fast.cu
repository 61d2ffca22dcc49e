// Fast-mode instantiations: FMA contraction on (default nvcc), restructured
// stencils; held to relative <= 1e-12 of the reference.
#include "chain.cuh"
#include "heat2x2.cuh"
#include "small.cuh"

namespace pirk {

bool heat_strip_step_ok(const HeatModel& m, double hk) {
    return !PIRK_STRIP_SFORM || heat_sform_coeffs(hk * m.kk, nullptr);
}

template cudaError_t launch_chain_step<false>(const ChainModel&, const WindowArgs&,
                                              const StepConsts&, unsigned long long,
                                              unsigned long long*, cudaStream_t);
template cudaError_t launch_chain_steps<false>(const ChainModel&, const WindowArgs&, const StepConstsN&, int,
                                                unsigned long long, unsigned long long*, cudaStream_t);
template cudaError_t launch_heat_step<false>(const HeatModel&, const WindowArgs&,
                                             const StepConsts&, unsigned long long,
                                             unsigned long long*, cudaStream_t, int);
template cudaError_t launch_small_integrate<false>(const SmallModel&, int, const double*,
                                                   const double*, double, double, double,
                                                   unsigned long long, unsigned long long,
                                                   double*, unsigned long long*, cudaStream_t);
template cudaError_t launch_monte_carlo<false>(const SmallModel&, const McArgs&, cudaStream_t);

}  // namespace pirk
