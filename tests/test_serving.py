"""The measured service-time seam on CPU: the planner's
simulator driven by a ``{(replica, TaskSpec): seconds}`` table -- the shape the
engine's ``serve.measured_service_times`` returns -- reproduces the closed-form
run exactly when the table holds the closed-form values, and the CLI's
``simulate --service`` reads the JSON form of the same table."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2311_11514_b200 import planner as P
from paper_2311_11514_b200.planner import cmdline

ROOT = Path(__file__).resolve().parents[1]
B = ROOT / "tests" / "golden" / "planner" / "b200_homog" / "inputs"


def test_service_table_equals_cost_model_when_fed_its_values():
    cluster, model = P.load_cluster(B / "cluster.json"), P.load_model(B / "model.json")
    wl, slo = P.load_workload(B / "workload.json"), P.load_slo(B / "slo.json")
    plan = P.load_plan(B / "plan.json")
    reqs = P.generate_workload(wl)
    table = P.service_times(plan, model, [r.task for r in reqs], cluster)
    a = P.simulate(plan, reqs, slo, model, cluster)
    b = P.simulate(plan, reqs, slo, model, cluster, service=dict(table))
    assert a == b
    # a slower measured replica shifts routing toward the others
    slow = {k: (v * 3 if k[0] == 0 else v) for k, v in table.items()}
    c = P.simulate(plan, reqs, slo, model, cluster, service=slow)
    assert sum(o.replica == 0 for o in c.per_request) < sum(o.replica == 0 for o in a.per_request)


def test_cli_simulate_with_service_file(tmp_path):
    cluster, model = P.load_cluster(B / "cluster.json"), P.load_model(B / "model.json")
    wl = P.load_workload(B / "workload.json")
    plan = P.load_plan(B / "plan.json")
    task = wl.dominant_task()
    table = P.service_times(plan, model, [task], cluster)
    doc = {"entries": [{"replica": r, "batch_size": t.batch_size, "input_len": t.input_len,
                        "output_len": t.output_len, "seconds": s} for (r, t), s in table.items()]}
    svc = tmp_path / "svc.json"
    svc.write_text(json.dumps(doc))
    common = ["simulate", "--cluster", str(B / "cluster.json"), "--model", str(B / "model.json"),
              "--workload", str(B / "workload.json"), "--slo", str(B / "slo.json"), "--plan", str(B / "plan.json")]
    assert cmdline.main(common + ["--out-dir", str(tmp_path / "a")]) == 0
    assert cmdline.main(common + ["--out-dir", str(tmp_path / "b"), "--service", str(svc)]) == 0
    for f in ("report.json", "requests.csv", "attainment_vs_scale.csv", "attainment_vs_rate.csv"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes(), f
    # an incomplete table is an input error (exit 2), not a crash
    doc["entries"] = doc["entries"][:1]
    svc.write_text(json.dumps(doc))
    assert cmdline.main(common + ["--out-dir", str(tmp_path / "c"), "--service", str(svc)]) == 2


def test_c5_report_from_measured_entries(tmp_path):
    svc = tmp_path / "svc"
    svc.mkdir()
    for i, (p, l, s) in enumerate([("[2,2]", [40, 40], 5.4), ("[2]", [80], 6.5), ("[4]", [80], 4.4)]):
        (svc / f"p{i}.json").write_text(json.dumps({"plan": p, "layers": l, "seconds": s}))
    out = tmp_path / "c5.json"
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "c5_report.py"), "--plan",
                        str(ROOT / "tests/golden/planner/b200_422/plan_s0/plan.json"), "--svc", str(svc),
                        "--out", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    d = json.loads(out.read_text())
    ga = d["layouts"]["GA plan (b200 {4,2,2} buckets)"]
    assert ga["pipelines"] == ["[2,2]", "[2]", "[2]"] and ga["service_s"] == [5.4, 6.5, 6.5]
    assert all(0.0 <= a <= 1.0 for a in ga["attainment"])
    assert "missing_measurement" in d["layouts"]["asymmetric 1 x [4,2,2] 40/20/20"]


def test_plan_with_measured_service_model(tmp_path):
    """plan --service: measurements equal to the closed form (scale 1) give the
    byte-identical reference plan; the B200 measurements of profiles/r01/c5
    drive the GA to a valid plan."""
    B4 = ROOT / "tests" / "golden" / "planner" / "b200_422" / "inputs"
    cluster, model = P.load_cluster(B4 / "cluster.json"), P.load_model(B4 / "model.json")
    task = P.load_workload(B4 / "workload.json").dominant_task()
    meas = tmp_path / "meas"
    meas.mkdir()
    for i, (tps, layers) in enumerate((((2, 2), (40, 40)), ((2,), (80,)), ((4,), (80,)))):
        pipe = P.place_shape(tuple(("b200", tp, l) for tp, l in zip(tps, layers)), cluster)
        secs = P.pipeline_cost(pipe, model, task, cluster)[0]
        (meas / f"p{i}.json").write_text(json.dumps({
            "plan": "[" + ",".join(map(str, tps)) + "]", "layers": list(layers), "seconds": secs,
            "batch_size": task.batch_size, "input_len": task.input_len, "output_len": task.output_len}))
    common = ["plan", "--cluster", str(B4 / "cluster.json"), "--model", str(B4 / "model.json"),
              "--workload", str(B4 / "workload.json"), "--slo", str(B4 / "slo.json"),
              "--pop", "16", "--gens", "30", "--seed", "0"]
    assert cmdline.main(common + ["--out-dir", str(tmp_path / "a"), "--service", str(meas)]) == 0
    gold = ROOT / "tests" / "golden" / "planner" / "b200_422" / "plan_s0" / "plan.json"
    assert (tmp_path / "a" / "plan.json").read_bytes() == gold.read_bytes()
    real = ROOT / "profiles" / "r01" / "c5"
    svc_dir = tmp_path / "real"
    svc_dir.mkdir()
    for f in real.glob("p[0-9]*.json"):
        (svc_dir / f.name).write_text(f.read_text())
    assert cmdline.main(common + ["--out-dir", str(tmp_path / "b"), "--service", str(svc_dir)]) == 0
    plan = P.load_plan(tmp_path / "b" / "plan.json")
    assert sorted(d for pipe in plan.pipelines for st in pipe for d in st.devices) == sorted(
        set(d for pipe in plan.pipelines for st in pipe for d in st.devices))
    # the measurements are what the search optimised: measured shapes answer with
    # their measured seconds, and the fitness differs from the closed-form run
    svc = cmdline.load_service(svc_dir, model, cluster, per_replica_ok=False)
    for (shape, t), secs in svc.measured.items():
        assert svc(P.place_shape(shape, cluster), t) == secs
    fit_meas = json.loads((tmp_path / "b" / "plan.json").read_text())["fitness"]
    fit_closed = json.loads(gold.read_text())["fitness"]
    assert fit_meas != fit_closed
    # a replica-indexed table is accepted by simulate only
    table = tmp_path / "table.json"
    table.write_text(json.dumps({"entries": [{"replica": 0, "batch_size": task.batch_size, "input_len": task.input_len,
                                              "output_len": task.output_len, "seconds": 1.0}]}))
    with pytest.raises(P.InputError):
        cmdline.load_service(table, model, cluster, per_replica_ok=False)
    assert cmdline.load_service(table, model, cluster, per_replica_ok=True) == {(0, task): 1.0}


def test_measured_service_model_keys_by_gpu_type():
    """a measurement on one GPU type must not answer for the same
    (TP, layers) shape on another type; unmeasured types use their own scale."""
    cluster = P.three_tier_cluster()
    model = P.toy_model()
    task = P.TaskSpec(4, 64, 16)
    types = sorted({d.gpu_type.type_id for d in cluster.devices})
    t0 = types[0]
    shape = ((t0, 1, model.num_layers),)
    pipe0 = P.place_shape(shape, cluster)
    closed0 = P.pipeline_cost(pipe0, model, task, cluster)[0]
    svc = P.MeasuredServiceModel({(shape, task): 2.0 * closed0}, model, cluster)
    assert svc(pipe0, task) == 2.0 * closed0
    for t in types[1:]:
        other = P.place_shape(((t, 1, model.num_layers),), cluster)
        if other is None:
            continue
        closed = P.pipeline_cost(other, model, task, cluster)[0]
        assert svc(other, task) == pytest.approx(2.0 * closed)   # calibrated closed form, not t0's seconds
        assert svc(other, task) != 2.0 * closed0 or closed == closed0
