"""paper_2001_10635_b200 -- B200-native PIRK reachability hot path.

Drop-in for the CTMM (mixed monotonicity), growth-bound and Monte Carlo entry
points of the reference ``ivreach`` library (/root/reference/proj), executed
by hand-written sm_100a kernels in lib/libpirk_b200.so through the C ABI of
include/pirk_c.h.  See DESIGN.md.
"""
from .models import (ARCH_QUAD, CHAIN, DECOMP_JACOBIAN, DECOMP_NATIVE, DECOMP_NONE, HEAT3D,
                     LAUB_LOOMIS, SCALAR_DECAY, SCALAR_LINEAR, TRAFFIC, USER, VDP, ZERO, Program,
                     SystemModel, make_arch_quadrotor, make_chain, make_heat3d, make_laub_loomis,
                     make_scalar_decay, make_scalar_linear, make_traffic, make_user_model,
                     make_vdp, make_zero, with_jacobian_decomposition)
from .reach import (Context, Engine, IntervalVector, MonteCarloSpec, PhaseTimes, ReachProblem,
                    ReachTube, RunReport, StepPlan, TubeEntry, center, contains, coverage_estimate,
                    from_center_radius, get_context, get_worker_context, growth_bound, half_width,
                    mixed_monotonicity, monte_carlo, monte_carlo_range, plan_steps,
                    record_schedule, sample_count, set_default_mode, step_window, subset_of,
                    tube_to_csv, validate)
from .driver import bench, bench_csv, dispatch, report_to_json, tube_to_json

__all__ = [n for n in dir() if not n.startswith("_")]
