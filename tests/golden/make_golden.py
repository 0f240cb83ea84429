"""Generate the committed golden fixtures (run in the build container only).

1. ``tiny_hf.npz`` -- HF transformers ``LlamaForCausalLM`` (third-party,
   v5.5, present in the container; NOT the reference) greedy generation on the
   C1 tiny config with this repo's seeded weights: the greedy ids and, per
   step, the top-8 logits plus 512 fixed-column logits. Pins the CPU oracle's
   Llama math (RMSNorm, RoPE, SwiGLU, scaling, argmax ties).
2. ``reference_plans.json`` -- outputs of the importable reference planner
   (``/root/reference/pkg/src/heteroplan``): plan_to_dict / plan_from_dict
   round trips, ``plan_notation``, ``pipeline_cost`` structural errors and
   ``check_memory`` verdicts, plus the reference ``three_tier`` golden plan
   (``heteroplan plan ... --pop 16 --gens 30 --seed 0``).
   Pins the plan boundary (``paper_2311_11514_b200/plan.py``).

Usage:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from paper_2311_11514_b200.config import TINY  # noqa: E402
from paper_2311_11514_b200.weights import init_host_weights, synthetic_prompts, to_hf_state_dict  # noqa: E402

S_OUT = 16
LOGIT_COLS = np.random.default_rng(7).choice(TINY.vocab, size=512, replace=False).astype(np.int64)


def make_hf():
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    torch.set_num_threads(os.cpu_count())
    cfg = TINY
    hf_cfg = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden_dim,
                         intermediate_size=cfg.intermediate, num_hidden_layers=cfg.num_layers,
                         num_attention_heads=cfg.num_heads, num_key_value_heads=cfg.num_kv_heads,
                         rms_norm_eps=cfg.rms_eps, rope_theta=cfg.rope_theta,
                         max_position_embeddings=4096, tie_word_embeddings=False,
                         attention_bias=False, mlp_bias=False, hidden_act="silu",
                         torch_dtype=torch.float32)
    hf_cfg._attn_implementation = "eager"
    model = LlamaForCausalLM(hf_cfg).float().eval()
    w = init_host_weights(cfg, seed=0)
    sd = {k: torch.from_numpy(v.copy()) for k, v in to_hf_state_dict(cfg, w).items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("rotary" in m for m in missing), missing
    prompt = synthetic_prompts(cfg, 2, 64, seed=1)
    with torch.no_grad():
        out = model.generate(torch.from_numpy(prompt.astype(np.int64)), max_new_tokens=S_OUT,
                             do_sample=False, output_logits=True, return_dict_in_generate=True,
                             pad_token_id=0, eos_token_id=None)
    ids = out.sequences[:, 64:].numpy().astype(np.int32)
    logits = torch.stack(out.logits, 0).float().numpy()           # [s_out, b, V]
    top_idx = np.argsort(-logits, axis=-1, kind="stable")[..., :8]
    top_val = np.take_along_axis(logits, top_idx, axis=-1)
    srt = np.sort(logits, axis=-1)
    margin = (srt[..., -1] - srt[..., -2]).min()
    np.savez_compressed(HERE / "tiny_hf.npz", prompt=prompt, ids=ids,
                        top_idx=top_idx.astype(np.int32), top_val=top_val.astype(np.float32),
                        cols=LOGIT_COLS, col_val=logits[..., LOGIT_COLS].astype(np.float32),
                        max_abs=np.float32(np.abs(logits).max()), margin=np.float32(margin))
    print("hf ids", ids.tolist(), "min top-2 margin", margin)


def make_reference_plans():
    sys.path.insert(0, "/root/reference/pkg/src")
    from heteroplan import cli, costs
    from heteroplan.cluster import (ClusterSpec, Device, GpuType, ModelSpec, TaskSpec,
                                    build_cluster)

    b200 = GpuType("b200", 180e9, 6.551e12, 1.6669e15)

    def cluster(machines):
        devs, d = [], 0
        for m, n in enumerate(machines):
            for _ in range(n):
                devs.append(Device(d, f"m{m}", "r0", b200))
                d += 1
        n = d
        alpha = np.full((n, n), 3e-6)
        np.fill_diagonal(alpha, 0.0)
        beta = np.full((n, n), 9e11)
        return build_cluster(devs, alpha, beta)

    cases = []
    specs = [
        ("tiny_21", [2, 1], [[0, 1], [2]], [3, 1], (4, 256, 4), (2, 64, 16)),
        ("13b_21", [2, 1], [[0, 1], [2]], [28, 12], (40, 5120, 2), (8, 512, 128)),
        ("13b_22", [2, 2], [[0, 1], [2, 3]], [20, 20], (40, 5120, 2), (8, 512, 128)),
        ("13b_11", [1, 1], [[0], [1]], [24, 16], (40, 5120, 2), (8, 512, 128)),
        ("70b_422", [4, 2, 2], [[0, 1, 2, 3], [4, 5], [6, 7]], [40, 20, 20], (80, 8192, 2), (32, 1024, 256)),
        ("70b_422_uneven", [4, 2, 2], [[0, 1, 2, 3], [4, 5], [6, 7]], [48, 16, 16], (80, 8192, 2), (32, 1024, 256)),
        ("70b_211", [2, 1, 1], [[0, 1], [2], [3]], [40, 20, 20], (80, 8192, 2), (32, 1024, 256)),
        ("70b_11", [1, 1], [[0], [1]], [40, 40], (80, 8192, 2), (32, 1024, 256)),
        ("70b_8", [8], [list(range(8))], [80], (80, 8192, 2), (32, 1024, 256)),
        ("70b_1", [1], [[0]], [80], (80, 8192, 2), (32, 1024, 256)),
        ("7b_1", [1], [[0]], [32], (32, 4096, 2), (8, 512, 128)),
    ]
    for name, machines, devs, layers, mspec, tspec in specs:
        cl = cluster(machines)
        model = ModelSpec(*mspec)
        task = TaskSpec(*tspec)
        pipe = tuple(costs.StageAssignment(tuple(d), l) for d, l in zip(devs, layers))
        ga = costs.GlobalAssignment((pipe,))
        doc = cli.plan_to_dict(ga)
        back = cli.plan_from_dict(json.loads(json.dumps(doc)))
        verdict = costs.check_memory(pipe, model, task, cl)
        try:
            total, _ = costs.pipeline_cost(pipe, model, task, cl)
            err = None
        except Exception as exc:  # noqa: BLE001
            total, err = None, f"{type(exc).__name__}: {exc}"
        pre, dec = costs.prefill_decode_estimate(pipe, model, task, cl)
        cases.append({
            "name": name, "doc": doc,
            "text": json.dumps(doc, indent=2, sort_keys=True) + "\n",
            "parsed": [[list(s.devices), s.num_layers] for s in back.pipelines[0]],
            "notation": costs.plan_notation(pipe),
            "mem_per_device": [costs.mem_footprint(s, model, task) for s in pipe],
            "feasible": verdict.feasible, "pipeline_cost": total, "error": err,
            "prefill_s": pre, "decode_s": dec,
            "model": list(mspec), "task": list(tspec),
        })
    # structural errors pipeline_cost raises (costs.py:222-232)
    cl = cluster([2, 1])
    model = ModelSpec(4, 256, 4)
    task = TaskSpec(2, 64, 16)
    errors = []
    for devs, layers in (([[0, 1], [2]], [3, 2]), ([[0, 1], [1]], [3, 1])):
        pipe = tuple(costs.StageAssignment(tuple(d), l) for d, l in zip(devs, layers))
        try:
            costs.pipeline_cost(pipe, model, task, cl)
            errors.append({"devices": devs, "layers": layers, "error": None})
        except ValueError as exc:
            errors.append({"devices": devs, "layers": layers, "error": str(exc)})
    bad_docs = []
    for bad in ({"pipelines": [{"stages": [{"devices": "xyz"}]}]}, {"nope": 1},
                {"pipelines": [{"stages": [{"devices": [0], "layers": "x"}]}]}):
        try:
            cli.plan_from_dict(bad)
            bad_docs.append({"doc": bad, "raises": None})
        except Exception as exc:  # noqa: BLE001
            bad_docs.append({"doc": bad, "raises": type(exc).__name__})
    # the reference golden plan: its own CLI on its own three_tier bundle
    # ([4,2,2] layers [57,14,9], sha256 2fcfd0a3...)
    import subprocess
    import tempfile
    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src")
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([sys.executable, "-B", "/root/reference/pkg/scripts/make_inputs.py",
                        "--out-dir", f"{tmp}/inputs"], check=True, env=env, capture_output=True)
        inp = f"{tmp}/inputs/three_tier"
        subprocess.run([sys.executable, "-B", "-m", "heteroplan.cli", "plan",
                        "--cluster", f"{inp}/cluster.json", "--model", f"{inp}/model.json",
                        "--workload", f"{inp}/workload.json", "--slo", f"{inp}/slo.json",
                        "--out-dir", f"{tmp}/plan", "--pop", "16", "--gens", "30", "--seed", "0"],
                       check=True, env=env, capture_output=True)
        text = Path(f"{tmp}/plan/plan.json").read_text()
        doc = json.loads(text)
        back = cli.plan_from_dict(doc)
    golden = {"text": text, "parsed": [[[list(s.devices), s.num_layers] for s in p] for p in back.pipelines],
              "notation": [costs.plan_notation(p) for p in back.pipelines]}
    out = {"cases": cases, "errors": errors, "bad_docs": bad_docs, "golden_plan": golden}
    (HERE / "reference_plans.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", len(cases), "plan cases")


if __name__ == "__main__":
    which = sys.argv[1:] or ["hf", "plans"]
    if "hf" in which:
        make_hf()
    if "plans" in which:
        make_reference_plans()
