"""Optimal stage layout of one pipeline group (the planner's DP).

Restates ``pkg/src/heteroplan/dp.py:137-242``. Given the group's device
counts per bucket and a fixed layer split l_1..l_S, choose for every stage a
(bucket k, TP size n) so that the sum of stage costs (compute + TP
all-reduce, ``cost_model``) plus hand-off edges between consecutive stages is
minimal; a stage whose per-device footprint exceeds the device memory is
excluded. Devices are handed out in id order within a bucket (a stage taking
n devices of bucket k gets the next n unassigned ids), so the DP state is the
count already taken per bucket plus the move that formed the last stage (the
edge cost depends on which devices the previous stage holds,
``dp.py:12-18``).

Determinism rules that make the emitted plan identical to the reference's:
states of a level are expanded in sorted (tau, move) order (the empty move
sorts first), moves in (size ascending, bucket ascending) order, a state is
only replaced by a strictly cheaper path, and the final winner is the least
(cost, size, bucket, tau).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

from ..plan import ModelSpec, StageAssignment, TaskSpec
from .cost_model import comp_cost, mem_footprint, pp_comm_cost, tp_comm_cost
from .pool import ClusterSpec, TypeVector, check_type_vector

DEFAULT_TP_CANDIDATES = (1, 2, 4, 8)

_NO_MOVE = (-1, -1)


class DpTable:
    """The DP memo as the reference exposes it (dp.py:42-95): best cost per
    (stage index, assigned counts tau, entering move) with a parent link;
    DP[0; 0] = 0, every other key +inf until relaxed, costs only decrease."""

    def __init__(self, n_buckets: int):
        self.n_buckets = n_buckets
        self.entries: dict = {(0, (0,) * n_buckets, None): (0.0, None, ())}

    def cost(self, key) -> float:
        got = self.entries.get(key)
        return got[0] if got else math.inf

    def best_cost(self, stage_index: int, assigned) -> float:
        """Minimum over the moves entering (j, tau)."""
        assigned = tuple(assigned)
        return min((c for (j, tau, _), (c, _, _) in self.entries.items() if j == stage_index and tau == assigned),
                   default=math.inf)

    def update(self, key, cost: float, parent, stage_devices=()) -> bool:
        if cost < self.cost(key):
            self.entries[key] = (cost, parent, tuple(stage_devices))
            return True
        return False


def dp_transition(table: DpTable, stage_index: int, assigned, move, stage_cost: float) -> DpTable:
    """One relaxation DP[j; tau] <- min(old, DP[j-1; tau - move] + stage_cost)
    (dp.py:98-122); an infinite (memory-violating) stage cost changes nothing."""
    k, n = move
    assigned = tuple(assigned)
    if n < 1 or not 0 <= k < len(assigned) or assigned[k] < n:
        raise ValueError(f"move {move} exceeds assigned counts {assigned}")
    prev = assigned[:k] + (assigned[k] - n,) + assigned[k + 1:]
    base = table.best_cost(stage_index - 1, prev)
    total = base + stage_cost if math.isfinite(base) and math.isfinite(stage_cost) else math.inf
    if math.isfinite(total):
        parent, pcost = None, math.inf
        for key, (c, _, _) in table.entries.items():
            if key[0] == stage_index - 1 and key[1] == prev and c < pcost:
                parent, pcost = key, c
        table.update((stage_index, assigned, tuple(move)), total, parent)
    return table


@dataclass
class DpResult:
    cost: float
    stages: list[StageAssignment] | None
    visited_states: int

    @property
    def feasible(self) -> bool:
        return self.stages is not None and math.isfinite(self.cost)


class _Costs:
    """Memoised stage and edge costs for one solve."""

    def __init__(self, pools, model, task, cluster):
        self.pools, self.model, self.task, self.cluster = pools, model, task, cluster
        self.stage_memo: dict = {}
        self.edge_memo: dict = {}

    def devices(self, k: int, offset: int, n: int) -> tuple[int, ...]:
        return tuple(self.pools[k][offset:offset + n])

    def stage(self, k: int, n: int, offset: int, layers: int) -> float:
        key = (k, n, offset, layers)
        if key not in self.stage_memo:
            st = StageAssignment(self.devices(k, offset, n), layers)
            cap = self.cluster.devices[st.devices[0]].gpu_type.mem_limit
            if mem_footprint(st, self.model, self.task) > cap:
                self.stage_memo[key] = math.inf
            else:
                self.stage_memo[key] = (comp_cost(st, self.model, self.task, self.cluster)
                                        + tp_comm_cost(st, self.model, self.task, self.cluster))
        return self.stage_memo[key]

    def edge(self, src: tuple[int, ...], dst: tuple[int, ...], src_layers: int) -> float:
        key = (src, dst)
        if key not in self.edge_memo:
            self.edge_memo[key] = pp_comm_cost(StageAssignment(src, src_layers), StageAssignment(dst, 0),
                                               self.model, self.task, self.cluster)
        return self.edge_memo[key]


def _partition(partition: Sequence[int], model: ModelSpec) -> tuple[int, ...]:
    part = tuple(int(x) for x in partition)
    if not part or min(part) < 1:
        raise ValueError(f"every stage needs >= 1 layer, got {part}")
    if sum(part) != model.num_layers:
        raise ValueError(f"partition sums to {sum(part)}, model has {model.num_layers} layers")
    return part


def solve_pipeline(group: TypeVector, partition: Sequence[int], model: ModelSpec, task: TaskSpec,
                   cluster: ClusterSpec, tp_candidates: Sequence[int] = DEFAULT_TP_CANDIDATES,
                   device_pools: Sequence[Sequence[int]] | None = None) -> DpResult:
    """Cheapest bucket-homogeneous stage layout for ``group`` under ``partition``
    (reference dp.py:137-233). ``device_pools[k]`` are the ids backing bucket
    k's count (default: the bucket's first ``group[k]`` ids)."""
    check_type_vector(cluster, group)
    part = _partition(partition, model)
    sizes = sorted({int(c) for c in tp_candidates})
    if not sizes or sizes[0] < 1:
        raise ValueError(f"tp_candidates must be positive, got {tp_candidates}")
    if device_pools is None:
        pools = [b.device_ids[:c] for b, c in zip(cluster.buckets, group)]
    else:
        pools = [tuple(p) for p in device_pools]
        for k, (p, c) in enumerate(zip(pools, group)):
            if len(p) != c:
                raise ValueError(f"bucket {k}: pool of {len(p)} ids for count {c}")
    costs = _Costs(pools, model, task, cluster)
    nb = len(group)

    # levels[j]: {(tau, move): (cost, parent state, devices of stage j)}
    start = ((0,) * nb, None)
    levels = [{start: (0.0, None, ())}]
    seen: set = set()
    for j, layers in enumerate(part, start=1):
        cur = levels[-1]
        nxt: dict = {}
        for state in sorted(cur, key=lambda s: (s[0], s[1] or _NO_MOVE)):
            base, _, prev_devs = cur[state]
            tau = state[0]
            for n in sizes:
                for k in range(nb):
                    if tau[k] + n > group[k]:
                        continue
                    sc = costs.stage(k, n, tau[k], layers)
                    if sc == math.inf:
                        continue
                    devs = costs.devices(k, tau[k], n)
                    total = base + sc
                    if j > 1:
                        total += costs.edge(prev_devs, devs, part[j - 2])
                    key = (tau[:k] + (tau[k] + n,) + tau[k + 1:], (k, n))
                    if total < nxt.get(key, (math.inf,))[0]:
                        nxt[key] = (total, state, devs)
        seen.update((j, t) for t, _ in nxt)
        levels.append(nxt)
        if not nxt:
            break
    if len(levels) <= len(part) or not levels[len(part)]:
        return DpResult(math.inf, None, len(seen))
    final = levels[len(part)]
    win = min(final, key=lambda s: (final[s][0], s[1][1], s[1][0], s[0]))
    chain, state = [], win
    for j in range(len(part), 0, -1):
        _, parent, devs = levels[j][state]
        chain.append(devs)
        state = parent
    chain.reverse()
    return DpResult(final[win][0], [StageAssignment(d, l) for d, l in zip(chain, part)], len(seen))


def visited_state_count(group: TypeVector, partition: Sequence[int], model: ModelSpec, task: TaskSpec,
                        cluster: ClusterSpec, tp_candidates: Sequence[int] = DEFAULT_TP_CANDIDATES) -> int:
    """Distinct (stage index, tau) states expanded (dp.py:236-242)."""
    return solve_pipeline(group, partition, model, task, cluster, tp_candidates).visited_states
