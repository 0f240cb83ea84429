"""The plan boundary against the reference planner's own outputs
(tests/golden/reference_plans.json, made by make_golden.py from
/root/reference/pkg/src/heteroplan). Mirrors the reference tests
test_cli.py:286-300 (round trip, bad document -> InputError)."""

import json
from pathlib import Path

import pytest

from paper_2311_11514_b200 import plan as P
from paper_2311_11514_b200.config import LLAMA2_13B, LLAMA2_70B, TINY, config_from_dict, preset

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_plans.json").read_text())


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_plan_round_trip_matches_reference(case, tmp_path):
    ga = P.plan_from_dict(case["doc"])
    assert [[list(s.devices), s.num_layers] for s in ga.pipelines[0]] == case["parsed"]
    assert P.plan_notation(ga.pipelines[0]) == case["notation"]
    # writer is byte-identical to the reference's _write_json(plan_to_dict(...))
    out = tmp_path / "plan.json"
    P.write_plan(out, ga)
    assert out.read_text() == case["text"]
    assert P.load_plan(out) == ga


def test_reference_golden_plan_loads():
    g = GOLD["golden_plan"]
    doc = json.loads(g["text"])
    ga = P.plan_from_dict(doc)
    assert [[[list(s.devices), s.num_layers] for s in p] for p in ga.pipelines] == g["parsed"]
    assert [P.plan_notation(p) for p in ga.pipelines] == g["notation"] == ["[4,2,2]"]
    assert [s.num_layers for s in ga.pipelines[0]] == [57, 14, 9]
    # the extra keys the reference writes (fitness, generations_run, ...) are ignored
    assert "fitness" in doc


@pytest.mark.parametrize("bad", GOLD["bad_docs"], ids=lambda b: json.dumps(b["doc"])[:30])
def test_bad_documents_raise_like_reference(bad):
    assert bad["raises"] == "InputError"
    with pytest.raises(P.InputError):
        P.plan_from_dict(bad["doc"])


@pytest.mark.parametrize("err", GOLD["errors"], ids=lambda e: str(e["layers"]))
def test_structural_errors_match_pipeline_cost(err):
    pipe = tuple(P.StageAssignment(tuple(d), l) for d, l in zip(err["devices"], err["layers"]))
    with pytest.raises(ValueError) as ei:
        P.validate_pipeline(pipe, 4)
    assert str(ei.value) == err["error"]


def test_model_document_superset_stays_reference_loadable(tmp_path):
    doc = LLAMA2_70B.to_model_dict()
    spec = P.model_from_dict(doc)
    assert spec == P.ModelSpec(80, 8192, 2)
    assert config_from_dict(doc) == LLAMA2_70B
    # a reference-only (3-key) document completes from the matching preset
    assert config_from_dict({"num_layers": 40, "hidden_dim": 5120, "bytes_per_param": 2}) == LLAMA2_13B
    assert config_from_dict(TINY.to_model_dict()) == TINY
    with pytest.raises(P.InputError):
        config_from_dict({"num_layers": 3, "hidden_dim": 7, "bytes_per_param": 2})


def test_task_and_errors():
    assert P.task_from_dict({"batch_size": 8, "input_len": 512, "output_len": 128}) == P.TaskSpec(8, 512, 128)
    with pytest.raises(P.InputError):
        P.TaskSpec(0, 1, 1)
    with pytest.raises(P.InputError):
        P.task_from_dict({"batch_size": "x"})
    assert P.EXIT_CODES[P.InputError] == 2 and P.EXIT_CODES[P.InfeasibleError] == 3


def test_simple_plan_and_ranges():
    ga = P.simple_plan([4, 2, 2], [40, 20, 20])
    assert [s.devices for s in ga.pipelines[0]] == [(0, 1, 2, 3), (4, 5), (6, 7)]
    assert P.stage_layer_ranges(ga.pipelines[0]) == [(0, 40), (40, 60), (60, 80)]
    assert preset("llama2-7b").params_per_layer() == 202_383_360
    assert preset("llama2-70b").params_per_layer() == 855_654_400
