"""Who does what for one pipeline of a plan: stages, TP ranks, hand-off routes.

The plan (reference ``costs.py:43-92``) lists, per pipeline, ordered stages
whose ``devices`` tuple gives the TP group (TP rank r = ``devices[r]``) and
whose ``num_layers`` are contiguous layers. The paper's runtime sends each
stage's activation from a leader GPU that then broadcasts inside the next TP
group (``PAPER.md:197``); after the row-parallel all-reduce every rank of a
stage holds the identical hidden state, so here receiver r' of stage j+1
simply pulls from sender ``r' mod TP_j`` of stage j -- no broadcast, every
receiver gets exactly one message, and with uniform NVSwitch links no leader
election is needed. The generated token ids return
from the last stage to stage 0 the same way.

Pure Python; unit-tested on CPU and exercised under gloo.
"""

from __future__ import annotations

from dataclasses import dataclass

from .config import LlamaConfig
from .plan import GlobalAssignment, InputError, StageAssignment, stage_layer_ranges, validate_pipeline


@dataclass(frozen=True)
class Role:
    """One (stage, TP rank) slot of a pipeline, bound to a device id."""

    device: int
    stage: int
    tp_rank: int
    tp: int
    layers: tuple[int, int]          # [l0, l1)
    tp_group: tuple[int, ...]        # device ids of the stage, TP order
    num_stages: int
    send_to: tuple[int, ...]         # devices of stage+1 that receive my hidden state
    recv_from: int | None            # device of stage-1 I receive from
    ids_send_to: tuple[int, ...]     # (last stage) stage-0 devices I return token ids to
    ids_recv_from: int | None        # (stage 0) last-stage device I receive ids from

    @property
    def is_first(self) -> bool:
        return self.stage == 0

    @property
    def is_last(self) -> bool:
        return self.stage == self.num_stages - 1

    @property
    def output_device(self) -> int:
        return self.tp_group[0]


def _routes(src: StageAssignment, dst: StageAssignment):
    """receiver r' <- sender r' mod |src|; returns {sender dev: (receiver devs)}, {receiver: sender}."""
    sends: dict[int, list[int]] = {d: [] for d in src.devices}
    recv: dict[int, int] = {}
    for rp, d in enumerate(dst.devices):
        s = src.devices[rp % src.tp_degree]
        sends[s].append(d)
        recv[d] = s
    return {k: tuple(v) for k, v in sends.items()}, recv


def pipeline_roles(assignment: GlobalAssignment, pipeline: int, cfg: LlamaConfig) -> list[Role]:
    """All roles of one pipeline, validated like the reference's pipeline_cost
    (costs.py:222-232) plus the TP divisibility the Megatron split needs."""
    if not 0 <= pipeline < len(assignment.pipelines):
        raise InputError(f"plan has no pipeline {pipeline}")
    pipe = assignment.pipelines[pipeline]
    validate_pipeline(pipe, cfg.num_layers)
    for st in pipe:
        cfg.check_tp(st.tp_degree)
        if st.num_layers == 0:
            raise InputError("stages with 0 layers are not executable")
    ranges = stage_layer_ranges(pipe)
    n = len(pipe)
    fwd = [_routes(pipe[j], pipe[j + 1]) for j in range(n - 1)]
    back = _routes(pipe[-1], pipe[0]) if n > 1 else None
    roles = []
    for j, st in enumerate(pipe):
        for r, d in enumerate(st.devices):
            roles.append(Role(
                device=d, stage=j, tp_rank=r, tp=st.tp_degree, layers=ranges[j],
                tp_group=tuple(st.devices), num_stages=n,
                send_to=fwd[j][0][d] if j + 1 < n else (),
                recv_from=fwd[j - 1][1][d] if j > 0 else None,
                ids_send_to=back[0][d] if (back and j == n - 1) else (),
                ids_recv_from=back[1][d] if (back and j == 0) else None,
            ))
    return roles


def role_of(assignment: GlobalAssignment, device: int, cfg: LlamaConfig):
    """(pipeline index, Role) for a device, or (None, None) if the plan leaves it idle."""
    for p, pipe in enumerate(assignment.pipelines):
        for st in pipe:
            if device in st.devices:
                return p, next(r for r in pipeline_roles(assignment, p, cfg) if r.device == device)
    return None, None
