"""B200-native Kino-PAX planner (arXiv 2409.06807) -- drop-in for the reference ``kinopax`` API.

The planner loop (frontier propagation, region update, frontier/tree update) runs as
hand-written sm_100a CUDA behind a C ABI (``include/kpx.h`` -> ``libkpx.so``); this
package is the host-side mirror of the reference's planner interface.
"""
from .backend import (Batch, CudaBackend, CudaF32Backend, PlanContext, available_backends, cuda_available,
                      get_backend)
from .batch import (BatchPlanner, BatchResult, RaceFlags, gather_records, goal_for_query, goals_for_queries, plan_batch,
                    race, shard_queries)
from .core import (ConfigError, DeviceError, Environment, EnvironmentFormatError, EnvironmentIOError, GoalBall,
                   KinopaxError, PlannerConfig, PlanResult, PlanStats, PlanStatus, TrajectorySegment,
                   environment_from_dict, environment_to_dict, load_environment, save_environment,
                   suggest_cells_per_dim, validate_config)
from .decomposition import GridGeometry, RegionRecord, RegionState
from .dynamics import (DOUBLE_INTEGRATOR_6D, DUBINS_AIRPLANE_6D, QUADCOPTER_12D, DynamicsModel, derivative,
                       get_model, model_names, propagate_ode, sample_control, sample_duration,
                       stacked_double_integrator)
from .envgen import GenerationError, gen_environment
from .planner import (IterationTrace, KinoPax, TreeArena, compute_branching_factor, extract_trajectory, plan)
from .problem import Problem, build_problem
from .rng import RngStream
from .runner import StatsTable, TrialRecord, dump_regions, export_trajectory, run_trials, summarize, sweep_te
from .validity import ValidityChecker, in_goal

__version__ = "0.1.0"
