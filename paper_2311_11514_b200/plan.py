"""Plan boundary: the reference planner's plan / model / task types, restated.

The reference (`heteroplan`, a pure-Python planner) hands the runtime a
``plan.json`` plus a model document and request shapes. This module mirrors
exactly those interfaces so that a plan emitted by the reference loads here
unchanged and a plan written here loads in the reference:

* ``StageAssignment`` / ``GlobalAssignment`` / ``plan_notation``
  -- reference ``pkg/src/heteroplan/costs.py:43-97``
* ``plan_to_dict`` / ``plan_from_dict`` / ``load_plan``
  -- reference ``pkg/src/heteroplan/cli.py:75-115`` (reader uses only
  ``devices`` and ``layers``; writer is sorted-keys, indent 2, ``cli.py:50-51``)
* ``ModelSpec`` / ``TaskSpec`` / ``load_model`` / ``load_task``
  -- reference ``pkg/src/heteroplan/cluster.py:223-268``
* ``Request`` -- reference ``pkg/src/heteroplan/simulate.py:56-60``
* error classes and their CLI exit codes -- ``cluster.py:29-30``,
  ``costs.py:35-40``, ``cli.py:454-475``
* ``validate_pipeline`` -- the structural checks of ``pipeline_cost``
  (``costs.py:222-232``): layer sum equals model depth, stages disjoint.

Nothing here touches a GPU; it is the host-side contract of the data path.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Mapping, Sequence

SCHEMA_VERSION = 1
PLAN_SCHEMA_VERSION = 1


class InputError(ValueError):
    """Malformed or inconsistent input (reference cluster.py:29-30; exit 2)."""


class InfeasibleError(RuntimeError):
    """A plan violates a hard constraint such as memory (costs.py:35-36; exit 3)."""


class InternalError(RuntimeError):
    """An internal invariant was violated (costs.py:39-40; exit 4)."""


EXIT_CODES = {InputError: 2, InfeasibleError: 3, InternalError: 4}


@dataclass(frozen=True)
class StageAssignment:
    """One pipeline stage: TP rank r is ``devices[r]``; owns ``num_layers``
    contiguous layers (reference costs.py:43-56)."""

    devices: tuple[int, ...]
    num_layers: int

    def __post_init__(self):
        if not self.devices:
            raise ValueError("stage needs at least one device")
        if self.num_layers < 0:
            raise ValueError("num_layers must be >= 0")

    @property
    def tp_degree(self) -> int:
        return len(self.devices)


Pipeline = tuple[StageAssignment, ...]


@dataclass(frozen=True)
class GlobalAssignment:
    """Disjoint pipelines, each an ordered stage list (reference costs.py:80-92)."""

    pipelines: tuple[Pipeline, ...]
    provenance: object = None

    def all_devices(self) -> list[int]:
        out: list[int] = []
        for pipe in self.pipelines:
            for stage in pipe:
                out.extend(stage.devices)
        return out


def plan_notation(pipeline: Sequence[StageAssignment]) -> str:
    """TP degrees by stage, e.g. ``"[4,2,2]"`` (reference costs.py:95-97)."""
    return "[" + ",".join(str(s.tp_degree) for s in pipeline) + "]"


def plan_to_dict(assignment: GlobalAssignment, extra: dict | None = None) -> dict:
    """Plan document, schema_version 1 (reference cli.py:75-92)."""
    doc = {
        "schema_version": PLAN_SCHEMA_VERSION,
        "pipelines": [
            {
                "notation": plan_notation(pipe),
                "stages": [
                    {"devices": list(s.devices), "tp_degree": s.tp_degree,
                     "layers": s.num_layers}
                    for s in pipe
                ],
            }
            for pipe in assignment.pipelines
        ],
    }
    if extra:
        doc.update(extra)
    return doc


def plan_from_dict(doc) -> GlobalAssignment:
    """Parse a plan document; reads only ``devices`` and ``layers``
    (reference cli.py:95-106). Malformed input raises ``InputError``."""
    try:
        pipelines = []
        for pipe in doc["pipelines"]:
            stages = tuple(
                StageAssignment(tuple(int(d) for d in st["devices"]), int(st["layers"]))
                for st in pipe["stages"]
            )
            pipelines.append(stages)
        return GlobalAssignment(tuple(pipelines))
    except (KeyError, TypeError, ValueError) as exc:
        raise InputError(f"bad plan document: {exc}") from exc


def write_plan(path, assignment: GlobalAssignment, extra: dict | None = None) -> None:
    """Write like the reference's ``_write_json`` (cli.py:50-51)."""
    Path(path).write_text(json.dumps(plan_to_dict(assignment, extra), indent=2,
                                     sort_keys=True) + "\n")


def _load_json(path):
    with open(path) as fh:
        try:
            return json.load(fh)
        except json.JSONDecodeError as exc:
            raise InputError(f"{path}: {exc}") from exc


def load_plan(path) -> GlobalAssignment:
    """reference cli.py:109-115"""
    return plan_from_dict(_load_json(path))


@dataclass(frozen=True)
class ModelSpec:
    """The reference's model triple (cluster.py:223-237)."""

    num_layers: int
    hidden_dim: int
    bytes_per_param: int

    def __post_init__(self):
        if self.num_layers < 1 or self.hidden_dim < 1:
            raise InputError("model dimensions must be >= 1")
        if self.bytes_per_param not in (1, 2, 4):
            raise InputError("bytes_per_param must be 1, 2 or 4")

    def param_bytes(self) -> int:
        return 12 * self.hidden_dim * self.hidden_dim * self.bytes_per_param * self.num_layers


@dataclass(frozen=True)
class TaskSpec:
    """Request shape (cluster.py:240-248)."""

    batch_size: int
    input_len: int
    output_len: int

    def __post_init__(self):
        if min(self.batch_size, self.input_len, self.output_len) < 1:
            raise InputError("task shape fields must be >= 1")


@dataclass(frozen=True)
class Request:
    """One arrival of the serving trace (simulate.py:56-60)."""

    index: int
    arrival: float
    task: TaskSpec


def model_from_dict(doc: Mapping) -> ModelSpec:
    try:
        return ModelSpec(int(doc["num_layers"]), int(doc["hidden_dim"]), int(doc["bytes_per_param"]))
    except (KeyError, TypeError, ValueError) as exc:
        raise InputError(f"bad model document: {exc}") from exc


def load_model(path) -> ModelSpec:
    """reference cluster.py:251-260 (extra keys ignored)."""
    return model_from_dict(_load_json(path))


def task_from_dict(doc: Mapping) -> TaskSpec:
    try:
        return TaskSpec(int(doc["batch_size"]), int(doc["input_len"]), int(doc["output_len"]))
    except (KeyError, TypeError, ValueError) as exc:
        raise InputError(f"bad task document: {exc}") from exc


def load_task(path) -> TaskSpec:
    return task_from_dict(_load_json(path))


def validate_pipeline(pipeline: Sequence[StageAssignment], num_layers: int) -> None:
    """Structural checks of reference ``pipeline_cost`` (costs.py:222-232):
    non-empty, layer sum equals model depth, no device in two stages.
    Raises ``ValueError`` exactly like the reference."""
    if not pipeline:
        raise ValueError("pipeline has no stages")
    total_layers = sum(s.num_layers for s in pipeline)
    if total_layers != num_layers:
        raise ValueError(f"stage layers sum to {total_layers}, model has {num_layers}")
    seen: set[int] = set()
    for stage in pipeline:
        for d in stage.devices:
            if d in seen:
                raise ValueError(f"device {d} appears in more than one stage")
            seen.add(d)


def stage_layer_ranges(pipeline: Sequence[StageAssignment]) -> list[tuple[int, int]]:
    """Stage j owns layers [sum_{<j} l, sum_{<=j} l) (contiguous, in order)."""
    out, start = [], 0
    for s in pipeline:
        out.append((start, start + s.num_layers))
        start += s.num_layers
    return out


def simple_plan(tp_degrees: Sequence[int], layers: Sequence[int], first_device: int = 0) -> GlobalAssignment:
    """One pipeline with consecutive device ids, e.g. ``simple_plan([4,2,2], [40,20,20])``."""
    if len(tp_degrees) != len(layers):
        raise InputError("tp_degrees and layers differ in length")
    stages, d = [], first_device
    for tp, l in zip(tp_degrees, layers):
        stages.append(StageAssignment(tuple(range(d, d + tp)), int(l)))
        d += tp
    return GlobalAssignment((tuple(stages),))
