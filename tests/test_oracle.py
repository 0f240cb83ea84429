"""Pin the CPU oracle before trusting it: against HF transformers'
LlamaForCausalLM on the C1 tiny config (golden vectors in
tests/golden/tiny_hf.npz), and its sharded restatement against itself."""

from pathlib import Path

import numpy as np
import pytest

from oracle.llama_oracle import Oracle, ShardedOracle, bf16_round, bf16_weights
from paper_2311_11514_b200.config import TINY
from paper_2311_11514_b200.weights import init_host_weights, init_tensor, synthetic_prompts

G = np.load(Path(__file__).parent / "golden" / "tiny_hf.npz")


@pytest.fixture(scope="module")
def tiny_w():
    return init_host_weights(TINY, seed=0)


@pytest.fixture(scope="module")
def tiny_run(tiny_w):
    return Oracle(TINY, tiny_w).generate(G["prompt"], 16)


def test_prompts_are_the_golden_prompts():
    assert np.array_equal(synthetic_prompts(TINY, 2, 64, seed=1), G["prompt"])


def test_oracle_greedy_ids_match_hf(tiny_run):
    ids, _ = tiny_run
    assert np.array_equal(ids, G["ids"])


def test_oracle_logits_match_hf(tiny_run):
    _, lg = tiny_run
    scale = float(G["max_abs"])
    cols = lg[..., G["cols"]]
    assert np.abs(cols - G["col_val"]).max() / scale < 1e-5
    top = np.take_along_axis(lg, G["top_idx"].astype(np.int64), axis=-1)
    assert np.abs(top - G["top_val"]).max() / scale < 1e-5


@pytest.mark.parametrize("stages", [[(2, (0, 3)), (1, (3, 4))], [(1, (0, 1)), (4, (1, 3)), (2, (3, 4))],
                                    [(8, (0, 4))]])
def test_sharded_oracle_equals_unsharded(tiny_w, tiny_run, stages):
    ids, lg = tiny_run
    ids2, lg2 = ShardedOracle(TINY, tiny_w, stages).generate(G["prompt"], 16)
    assert np.array_equal(ids, ids2)
    assert np.abs(lg - lg2).max() / np.abs(lg).max() < 1e-5


def test_weight_streams_are_deterministic_and_independent():
    a = init_tensor(TINY, 0, "q", 2)
    b = init_tensor(TINY, 0, "q", 2)
    c = init_tensor(TINY, 0, "q", 3)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    g = init_tensor(TINY, 0, "ln_attn", 0)
    assert abs(float(g.mean()) - 1.0) < 0.01


def test_bf16_round_is_rne():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5e-3, 3.0e38], dtype=np.float32)
    r = bf16_round(x)
    import torch
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(r, ref)


def test_teacher_forcing_reproduces_free_run(tiny_w, tiny_run):
    ids, lg = tiny_run
    ids2, lg2 = Oracle(TINY, tiny_w).generate(G["prompt"], 16, forced=ids)
    assert np.array_equal(ids, ids2) and np.allclose(lg, lg2)


def test_bf16_weights_keep_gains_fp32(tiny_w):
    w = bf16_weights(tiny_w)
    assert np.array_equal(w["layers"][0]["ln_attn"], tiny_w["layers"][0]["ln_attn"])
    assert not np.array_equal(w["layers"][0]["q"], tiny_w["layers"][0]["q"])
