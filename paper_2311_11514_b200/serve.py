"""Measured service times in the reference's table shape.

The reference simulator asks ``service_times(assignment, model, tasks,
cluster)`` for ``{(replica, TaskSpec): seconds}`` and fills it with the
closed-form ``pipeline_cost`` (reference ``simulate.py:135-142``,
``costs.py:213-237``). ``measured_service_times`` returns the same dict
with seconds measured by running each replica's pipeline through the engine
on the B200 -- the seam through which the reference's ``simulate`` /
``sweep_*`` (``simulate.py:145-212``) run unchanged on real latencies
(INTEGRATION.md shows the one-line hook).
"""

from __future__ import annotations

from typing import Iterable

import numpy as np

from .config import LlamaConfig
from .engine import Engine
from .plan import GlobalAssignment, InputError, TaskSpec


def measured_service_times(assignment: GlobalAssignment, cfg: LlamaConfig, tasks: Iterable[TaskSpec],
                           cluster=None, *, comm: str = "local", device=None, dtype: str = "bf16",
                           weights: str = "device", repeats: int = 1, seed: int = 1,
                           kernels=None, emulated: bool = False) -> dict:
    """{(replica index, TaskSpec): seconds} for every pipeline and distinct shape.

    ``comm='local'`` measures single-GPU replicas in this process on
    ``device`` (multi-GPU replicas only with ``emulated=True``: their ranks
    then run one after another, so the seconds are not a service time);
    ``comm='dist'`` runs under torchrun where this process's rank is a device
    of the (single) pipeline. Each engine is closed (peer mappings, IPC
    buffers) before the next is built. ``cluster`` is accepted for
    signature parity with the reference and unused: the hardware is measured.
    """
    shapes = sorted(set(tasks), key=lambda t: (t.batch_size, t.input_len, t.output_len))
    if comm == "local" and not emulated:
        wide = [r for r, pipe in enumerate(assignment.pipelines) if sum(len(st.devices) for st in pipe) > 1]
        if wide:
            raise InputError(f"replicas {wide} span several GPUs: comm='local' would run their ranks one after "
                             "another on one device, which is not their service time -- measure them under "
                             "torchrun (comm='dist', tools/measure_service.py) or pass emulated=True for a "
                             "functional (untimed-semantics) run")
    table = {}
    for r in range(len(assignment.pipelines)):
        for task in shapes:
            eng = Engine(assignment, cfg, dtype=dtype, batch=task.batch_size, max_prompt=task.input_len,
                         max_out=task.output_len, pipeline=r, comm=comm, device=device, weights=weights,
                         kernels=kernels)
            rng = np.random.default_rng(seed)
            prompt = rng.integers(0, cfg.vocab, size=(task.batch_size, task.input_len), dtype=np.int32)
            eng.generate(prompt, task.output_len)  # warm-up + graph capture
            ts = [eng.service_time(task, prompt) for _ in range(max(1, repeats))]
            table[(r, task)] = float(np.median(ts))
            eng.close()
            del eng
    return table
