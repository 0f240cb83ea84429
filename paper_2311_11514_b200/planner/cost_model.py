"""Closed-form stage cost and memory model (the planner's latency oracle).

Restatement of the reference ``pkg/src/heteroplan/costs.py``. Every
expression keeps the reference's floating-point evaluation order, because the
search compares and writes these numbers (``plan.json``'s ``mean_latency_s``
must be byte-identical):

* compute (``costs.py:106-120``): per layer, the slowest device's weight scan
  ``12 H^2 B s_out / (n bw)`` plus its FLOP term ``24 b (s_in+s_out) H^2 / (n c)``;
* TP all-reduce (``costs.py:123-147``): per device, the sum over its stage
  peers of ``alpha + bytes / (n beta)``; the worst device, x4 supersteps per
  layer, prefill message ``b s_in H B`` once and decode message ``b H B`` per
  output token;
* PP hand-off (``costs.py:150-165``): best cross link for each message;
* memory (``costs.py:168-192``): weight shard + 2 activations per layer
  (``/n``) + 4 activation buffers per device.

These formulas are the reference's *model* of the data path this repo runs
on the B200; ``serve.measured_service_times`` replaces their output with
measured seconds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

from ..plan import (GlobalAssignment, InfeasibleError, InternalError, ModelSpec, StageAssignment,
                    TaskSpec, validate_pipeline)
from .pool import ClusterSpec


@dataclass(frozen=True)
class StageCostBreakdown:
    comp: float
    comm_tp: float
    comm_pp_to_next: float
    mem_per_device: float

    def total(self) -> float:
        return self.comp + self.comm_tp + self.comm_pp_to_next


@dataclass(frozen=True)
class MemoryVerdict:
    feasible: bool
    margins: dict
    violations: tuple[int, ...]


def _one_bucket(stage: StageAssignment, cluster: ClusterSpec) -> None:
    ks = sorted({cluster.bucket_of(d) for d in stage.devices})
    if len(ks) != 1:
        raise ValueError(f"stage devices {stage.devices} span buckets {ks}")


def _slowest(stage: StageAssignment, cluster: ClusterSpec, numer, attr: str) -> float:
    """max over the stage's devices of numer / (n * rate_d)."""
    n = stage.tp_degree
    return max(numer / (n * getattr(cluster.devices[d].gpu_type, attr)) for d in stage.devices)


def _allreduce_superstep(stage: StageAssignment, cluster: ClusterSpec, nbytes) -> float:
    """Worst device's sum over its peers of alpha + nbytes / (n beta)."""
    n, alpha, beta = stage.tp_degree, cluster.alpha, cluster.beta
    worst = 0.0
    for d in stage.devices:
        acc = 0.0
        for p in stage.devices:
            if p != d:
                acc += alpha[d, p] + nbytes / (n * beta[d, p])
        worst = max(worst, acc)
    return worst


def _best_link(src: StageAssignment, dst: StageAssignment, cluster: ClusterSpec, nbytes) -> float:
    alpha, beta = cluster.alpha, cluster.beta
    best = math.inf
    for d in src.devices:
        for p in dst.devices:
            best = min(best, alpha[d, p] + nbytes / beta[d, p])
    return best


def comp_cost(stage: StageAssignment, model: ModelSpec, task: TaskSpec, cluster: ClusterSpec) -> float:
    _one_bucket(stage, cluster)
    hsq = model.hidden_dim * model.hidden_dim
    scan = _slowest(stage, cluster, 12 * hsq * model.bytes_per_param * task.output_len, "mem_bandwidth")
    flop = _slowest(stage, cluster, 24 * task.batch_size * (task.input_len + task.output_len) * hsq, "compute")
    return scan * stage.num_layers + flop * stage.num_layers


def tp_comm_cost(stage: StageAssignment, model: ModelSpec, task: TaskSpec, cluster: ClusterSpec) -> float:
    _one_bucket(stage, cluster)
    if stage.tp_degree == 1:
        return 0.0
    row = task.batch_size * model.hidden_dim * model.bytes_per_param
    pre = _allreduce_superstep(stage, cluster, row * task.input_len)
    dec = _allreduce_superstep(stage, cluster, row)
    l = stage.num_layers
    return pre * 4 * l + dec * 4 * task.output_len * l


def pp_comm_cost(stage: StageAssignment, next_stage: StageAssignment, model: ModelSpec, task: TaskSpec,
                 cluster: ClusterSpec) -> float:
    _one_bucket(stage, cluster)
    _one_bucket(next_stage, cluster)
    row = task.batch_size * model.hidden_dim * model.bytes_per_param
    pre = _best_link(stage, next_stage, cluster, row * task.input_len)
    dec = _best_link(stage, next_stage, cluster, row)
    return pre + dec * task.output_len


def _act_bytes(model: ModelSpec, task: TaskSpec) -> int:
    return task.batch_size * (task.input_len + task.output_len) * model.hidden_dim * model.bytes_per_param


def mem_footprint(stage: StageAssignment, model: ModelSpec, task: TaskSpec) -> float:
    act = _act_bytes(model, task)
    per_layer = (12 * model.hidden_dim * model.hidden_dim * model.bytes_per_param + 2 * act) / stage.tp_degree
    return per_layer * stage.num_layers + 4 * act


def check_memory(pipeline: Sequence[StageAssignment], model: ModelSpec, task: TaskSpec,
                 cluster: ClusterSpec) -> MemoryVerdict:
    margins: dict[int, float] = {}
    over: list[int] = []
    for stage in pipeline:
        need = mem_footprint(stage, model, task)
        for d in stage.devices:
            margins[d] = cluster.devices[d].gpu_type.mem_limit - need
            if margins[d] < 0:
                over.append(d)
    return MemoryVerdict(not over, margins, tuple(sorted(over)))


def stage_breakdowns(pipeline: Sequence[StageAssignment], model: ModelSpec, task: TaskSpec,
                     cluster: ClusterSpec) -> list[StageCostBreakdown]:
    rows = []
    for j, stage in enumerate(pipeline):
        pp = pp_comm_cost(stage, pipeline[j + 1], model, task, cluster) if j + 1 < len(pipeline) else 0.0
        rows.append(StageCostBreakdown(comp_cost(stage, model, task, cluster),
                                       tp_comm_cost(stage, model, task, cluster), pp,
                                       mem_footprint(stage, model, task)))
    return rows


def pipeline_cost(pipeline: Sequence[StageAssignment], model: ModelSpec, task: TaskSpec,
                  cluster: ClusterSpec) -> tuple[float, list[StageCostBreakdown]]:
    """Seconds per request for one pipeline (costs.py:213-237): structural
    errors are ``ValueError``, a memory violation is ``InfeasibleError``."""
    validate_pipeline(pipeline, model.num_layers)
    verdict = check_memory(pipeline, model, task, cluster)
    if not verdict.feasible:
        raise InfeasibleError(f"memory limit exceeded on devices {verdict.violations}")
    rows = stage_breakdowns(pipeline, model, task, cluster)
    return sum(r.total() for r in rows), rows


def prefill_decode_estimate(pipeline: Sequence[StageAssignment], model: ModelSpec, task: TaskSpec,
                            cluster: ClusterSpec) -> tuple[float, float]:
    """The same terms regrouped into (prefill s, decode s) (costs.py:240-284)."""
    hsq = model.hidden_dim * model.hidden_dim
    row = task.batch_size * model.hidden_dim * model.bytes_per_param
    prefill = decode = 0.0
    for j, stage in enumerate(pipeline):
        _one_bucket(stage, cluster)
        l = stage.num_layers
        prefill += l * _slowest(stage, cluster, 24 * task.batch_size * task.input_len * hsq, "compute")
        decode += l * _slowest(stage, cluster, 12 * hsq * model.bytes_per_param * task.output_len,
                               "mem_bandwidth")
        decode += l * _slowest(stage, cluster, 24 * task.batch_size * task.output_len * hsq, "compute")
        if stage.tp_degree > 1:
            prefill += _allreduce_superstep(stage, cluster, row * task.input_len) * 4 * l
            decode += _allreduce_superstep(stage, cluster, row) * 4 * task.output_len * l
        if j + 1 < len(pipeline):
            prefill += _best_link(stage, pipeline[j + 1], cluster, row * task.input_len)
            decode += _best_link(stage, pipeline[j + 1], cluster, row) * task.output_len
    return prefill, decode


def assert_valid_assignment(assignment: GlobalAssignment, model: ModelSpec, task: TaskSpec,
                            cluster: ClusterSpec) -> None:
    """Emit-side invariant check (costs.py:287-302); violations are ``InternalError``."""
    used: set[int] = set()
    for pipe in assignment.pipelines:
        total = sum(s.num_layers for s in pipe)
        if total != model.num_layers:
            raise InternalError(f"pipeline layers sum to {total} != {model.num_layers}")
        for stage in pipe:
            for d in stage.devices:
                if d in used:
                    raise InternalError(f"device {d} assigned twice across pipelines")
                used.add(d)
        if not check_memory(pipe, model, task, cluster).feasible:
            raise InternalError("emitted pipeline violates memory limits")
