"""Host-side HexGen planner, restated from the reference (``heteroplan``).

The north star keeps the genetic-algorithm plan search and its cost model on
the host and requires the same plan as the reference for the same seed. The
modules restate, in the reference's floating-point order and RNG streams:

==================  ==========================================  =====================
module              what                                        reference
==================  ==========================================  =====================
``pool``            devices, links, (machine, type) buckets     ``cluster.py``, ``presets.py``
``cost_model``      stage / pipeline latency and memory         ``costs.py``
``layout_dp``       optimal stage layout of one group           ``dp.py``
``grouping``        k-means + elbow seed groups                 ``kmeans.py``
``evolution``       GA: mutations, evaluation, search, replan   ``genetic.py``
``slo_sim``         Poisson traces, SLO simulation, sweeps      ``simulate.py``
``cmdline``         plan/replan/simulate/dp/costs/ablate CLI    ``cli.py``
==================  ==========================================  =====================

Plans, model and task documents and the error classes are shared with the
data path (``paper_2311_11514_b200.plan``).
"""

from ..plan import (GlobalAssignment, InfeasibleError, InputError, InternalError, ModelSpec, Request,
                    StageAssignment, TaskSpec, load_model, load_plan, load_task, plan_notation)
from .cost_model import (MemoryVerdict, StageCostBreakdown, assert_valid_assignment, check_memory, comp_cost,
                         mem_footprint, pipeline_cost, pp_comm_cost, prefill_decode_estimate, stage_breakdowns,
                         tp_comm_cost)
from .evolution import (EvalOutcome, Genome, InfeasiblePoolError, SearchConfig, SearchResult, evolve,
                        init_population, make_genome, mutate_merge, mutate_split, mutate_swap,
                        random_mutation_baseline, refine_partition, replan)
from .grouping import cluster_groups, device_features, kmeans_fit
from .layout_dp import DEFAULT_TP_CANDIDATES, DpResult, DpTable, dp_transition, solve_pipeline, visited_state_count
from .pool import (B200, Bucket, ClusterSpec, Device, GpuType, TypeVector, a100_like_cluster, b200_node,
                   build_cluster, cluster_from_dict, cluster_to_dict, llama70b, load_cluster, remove_devices,
                   three_tier_cluster, toy_model, two_region_cluster)
from .slo_sim import (MeasuredServiceModel, SloConfig, SloReport, WorkloadSpec, generate_workload, load_slo,
                      load_workload, pipeline_shape, place_shape, service_times, simulate, sweep_rate, sweep_slo_scale)

__all__ = [n for n in dir() if not n.startswith("_")]
