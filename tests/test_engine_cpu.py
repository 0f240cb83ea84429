"""Engine host logic on CPU (test kernels in tests/cpu_kernels.py, LocalComm):
asymmetric plans reproduce the HF-pinned greedy ids of the tiny config."""

from pathlib import Path

import numpy as np
import pytest

import cpu_kernels
from paper_2311_11514_b200.config import TINY
from paper_2311_11514_b200.engine import Engine, PagedKVCache
from paper_2311_11514_b200.plan import InputError, TaskSpec, simple_plan

G = np.load(Path(__file__).parent / "golden" / "tiny_hf.npz")


@pytest.mark.parametrize("tps,layers", [([2, 1], [3, 1]), ([1], [4]), ([1, 2, 4], [1, 1, 2])])
def test_asymmetric_plans_match_golden(tps, layers):
    eng = Engine(simple_plan(tps, layers), TINY, dtype="fp32", batch=2, max_prompt=64, max_out=16,
                 device="cpu", kernels=cpu_kernels, page_size=16)
    r = eng.generate(G["prompt"], 16, return_logits=True)
    assert np.array_equal(r.ids, G["ids"])
    assert np.abs(r.logits[..., G["cols"]] - G["col_val"]).max() / G["max_abs"] < 1e-3


def test_request_shape_checks():
    eng = Engine(simple_plan([1], [4]), TINY, dtype="fp32", batch=2, max_prompt=8, max_out=4,
                 device="cpu", kernels=cpu_kernels, page_size=16)
    with pytest.raises(InputError):
        eng.generate(np.zeros((2, 9), np.int32), 4)
    with pytest.raises(InputError):
        eng.generate(np.zeros((3, 8), np.int32), 4)     # more sequences than the engine holds
    with pytest.raises(InputError):
        eng.generate(np.zeros((2, 8), np.int32), 5)     # more outputs than the KV cache holds
    t = eng.service_time(TaskSpec(2, 8, 3))
    assert t > 0


def test_kv_pages_are_interleaved_and_recycled():
    kv = PagedKVCache(1, 3, 40, 2, 8, 16, __import__("torch").float32, "cpu")
    kv.assign(3, 40)
    bt = kv.block_table.numpy()
    assert bt[:, 0].tolist() == [0, 1, 2] and bt[:, 1].tolist() == [3, 4, 5]
    with pytest.raises(InputError):
        kv.assign(3, 100)
    kv.assign(2, 16)
    assert len(kv.owned) == 2 and len(kv.free) == kv.num_blocks - 2


def test_measured_service_times_has_reference_table_shape():
    """Same keys as the reference's service_times (simulate.py:135-142)."""
    from paper_2311_11514_b200.plan import GlobalAssignment, StageAssignment
    from paper_2311_11514_b200.serve import measured_service_times
    ga = GlobalAssignment(((StageAssignment((0, 1), 3), StageAssignment((2,), 1)),
                           (StageAssignment((3,), 4),)))
    tasks = [TaskSpec(2, 8, 3), TaskSpec(2, 8, 3), TaskSpec(2, 16, 2)]
    with pytest.raises(InputError):   # a multi-GPU replica is not timed by emulation
        measured_service_times(ga, TINY, tasks, comm="local", device="cpu", dtype="fp32",
                               weights="host", kernels=cpu_kernels)
    tab = measured_service_times(ga, TINY, tasks, comm="local", device="cpu", dtype="fp32",
                                 weights="host", kernels=cpu_kernels, emulated=True)
    assert set(tab) == {(r, t) for r in range(2) for t in set(tasks)}
    assert all(v > 0 for v in tab.values())


@pytest.mark.parametrize("tps,layers", [([2, 1], [3, 1]), ([1, 1, 1], [2, 1, 1])])
def test_microbatched_prefill_matches_golden(tps, layers, monkeypatch):
    """Pipelined prefill in 2 micro-batches (one sequence each): KV tables,
    residual rows and hand-offs are windowed per micro-batch; ids unchanged."""
    monkeypatch.setenv("HX_PREFILL_MB", "2")
    eng = Engine(simple_plan(tps, layers), TINY, dtype="fp32", batch=2, max_prompt=64, max_out=16,
                 device="cpu", kernels=cpu_kernels, page_size=16)
    assert eng.prefill_microbatches(2, 64) == 2
    r = eng.generate(G["prompt"], 16, return_logits=True)
    assert np.array_equal(r.ids, G["ids"])
    assert np.abs(r.logits[..., G["cols"]] - G["col_val"]).max() / G["max_abs"] < 1e-3


def test_smaller_batch_than_engine_matches_golden():
    """Requests of any batch up to the engine's: b=1 and b=2 on a b=3 engine give
    the golden ids of their sequences (the kernels run on the first b rows)."""
    eng = Engine(simple_plan([2, 1], [3, 1]), TINY, dtype="fp32", batch=3, max_prompt=64, max_out=16,
                 device="cpu", kernels=cpu_kernels, page_size=16)
    r2 = eng.generate(G["prompt"], 16)
    assert np.array_equal(r2.ids, G["ids"])
    r1 = eng.generate(G["prompt"][1:2], 16)
    assert np.array_equal(r1.ids, G["ids"][1:2])
