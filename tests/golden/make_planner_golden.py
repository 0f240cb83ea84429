"""Generate the planner golden fixtures from the REFERENCE planner (build
container only: needs /root/reference; the outputs are committed).

For every input bundle -- the reference's own three (``scripts/make_inputs.py``:
three_tier, two_region, a100_node) plus B200 bundles for this repo's configs
(8xB200 as one bucket, as pseudo-machines {4,2,2}, and the
tiny C1 bundle) -- run the reference CLI (``heteroplan.cli.main``) for
``plan`` (several seeds), ``simulate``, ``costs``, ``dp``, ``replan`` and
``ablate`` and store every output file except ``manifest.json`` under
``tests/golden/planner/<bundle>/<run>/``. ``runs.json`` lists the argv of each
run; ``tests/test_planner.py`` replays them through this repo's restated CLI
and requires byte-identical files.

Usage:  python tests/golden/make_planner_golden.py
"""

from __future__ import annotations

import contextlib
import io
import json
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "planner"
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/scripts")

from heteroplan import cli  # noqa: E402
from heteroplan.cluster import cluster_to_dict  # noqa: E402
from heteroplan.costs import pipeline_cost, StageAssignment  # noqa: E402
from heteroplan.cluster import Device, GpuType, ModelSpec, TaskSpec, build_cluster  # noqa: E402
import numpy as np  # noqa: E402
import make_inputs  # noqa: E402


def b200_cluster(machines):
    g = GpuType("b200", 180e9, 6.551e12, 1.6669e15)
    devs, d = [], 0
    for m, size in enumerate(machines):
        for _ in range(size):
            devs.append(Device(d, f"node0.{m}", "dc0", g))
            d += 1
    n = d
    alpha = np.full((n, n), 3e-6)
    np.fill_diagonal(alpha, 0.0)
    return build_cluster(devs, alpha, np.full((n, n), 9e11))


def b200_bundles():
    m70 = {"schema_version": 1, "num_layers": 80, "hidden_dim": 8192, "bytes_per_param": 2}
    task = make_inputs.task_doc(32, 1024, 256)
    homog = b200_cluster([8])
    tp8 = StageAssignment(tuple(range(8)), 80)
    base = pipeline_cost([tp8], ModelSpec(80, 8192, 2), TaskSpec(32, 1024, 256), homog)[0]
    for name, machines in (("b200_homog", [8]), ("b200_422", [4, 2, 2])):
        yield name, {
            "cluster.json": cluster_to_dict(b200_cluster(machines)),
            "model.json": m70,
            "task.json": task,
            "workload.json": make_inputs.workload_doc(0.5, 11, 200, task),
            "slo.json": make_inputs.slo_doc(2.0, 0.9, task, base),
        }
    tiny_task = make_inputs.task_doc(2, 64, 16)
    yield "tiny_c1", {
        "cluster.json": cluster_to_dict(b200_cluster([2, 1])),
        "model.json": {"schema_version": 1, "num_layers": 4, "hidden_dim": 256, "bytes_per_param": 4,
                       "num_heads": 8},
        "task.json": tiny_task,
        "workload.json": make_inputs.workload_doc(50.0, 3, 100, tiny_task),
        "slo.json": make_inputs.slo_doc(2.0, 0.9, tiny_task, 1e-3),
    }


PLANS = {  # bundle -> list of (run name, extra argv)
    "three_tier": [("plan_s0", ["--pop", "16", "--gens", "30", "--seed", "0"]),
                   ("plan_s1", ["--pop", "16", "--gens", "30", "--seed", "1"]),
                   ("plan_s5", ["--pop", "24", "--gens", "40", "--seed", "5"])],
    "two_region": [("plan_s0", ["--pop", "16", "--gens", "30", "--seed", "0"]),
                   ("plan_s3", ["--pop", "12", "--gens", "20", "--seed", "3", "--tp-candidates", "1,2,4"])],
    "a100_node": [("plan_s0", ["--pop", "16", "--gens", "20", "--seed", "0"])],
    "b200_homog": [("plan_s0", ["--pop", "16", "--gens", "30", "--seed", "0"])],
    "b200_422": [("plan_s0", ["--pop", "16", "--gens", "30", "--seed", "0"]),
                 ("plan_s2", ["--pop", "16", "--gens", "30", "--seed", "2"])],
    "tiny_c1": [("plan_s0", ["--pop", "8", "--gens", "10", "--seed", "0"])],
}

DPS = {
    "three_tier": [("dp_422", ["--group", "4,2,2", "--partition", "57,14,9"]),
                   ("dp_even", ["--group", "4,2,2", "--partition", "27,27,26"]),
                   ("dp_40", ["--group", "4,0,0", "--partition", "80"])],
    "two_region": [("dp_4", ["--group", "4,0", "--partition", "8"]),
                   ("dp_22", ["--group", "2,2", "--partition", "4,4"])],
    "b200_422": [("dp_422", ["--group", "4,2,2", "--partition", "40,20,20"])],
    "tiny_c1": [("dp_21", ["--group", "2,1", "--partition", "3,1"])],
}

# hand-specified plans for simulate / costs (the configs of BASELINE.json)
FIXED_PLANS = {
    "b200_422": {"schema_version": 1, "pipelines": [{"stages": [
        {"devices": [0, 1, 2, 3], "layers": 40}, {"devices": [4, 5], "layers": 20}, {"devices": [6, 7], "layers": 20}]}]},
    "b200_homog": {"schema_version": 1, "pipelines": [
        {"stages": [{"devices": [0, 1], "layers": 80}]}, {"stages": [{"devices": [2, 3], "layers": 80}]},
        {"stages": [{"devices": [4, 5], "layers": 80}]}, {"stages": [{"devices": [6, 7], "layers": 80}]}]},
    "tiny_c1": {"schema_version": 1, "pipelines": [{"stages": [
        {"devices": [0, 1], "layers": 3}, {"devices": [2], "layers": 1}]}]},
}


def run(argv, out_dir: Path):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    bundles = list(make_inputs.bundles()) + list(b200_bundles())
    index = []
    for name, files in bundles:
        bdir = OUT / name
        (bdir / "inputs").mkdir(parents=True)
        for fname, doc in files.items():
            (bdir / "inputs" / fname).write_text(json.dumps(doc, indent=2) + "\n")
        if name in FIXED_PLANS:
            (bdir / "inputs" / "plan.json").write_text(json.dumps(FIXED_PLANS[name], indent=2) + "\n")
        inp = {k: f"inputs/{k}.json" for k in ("cluster", "model", "workload", "slo", "task")}

        def add(run_name, cmd, extra, uses, stdout_file=None):
            argv = [cmd] + sum([[f"--{u}", inp[u] if u in inp else u] for u in uses], []) + extra
            rdir = bdir / run_name
            rdir.mkdir()
            real = [str(bdir / a) if "/" in a and (bdir / a).is_file() else a for a in argv] + ["--out-dir", str(rdir)]
            rc, out = run(real, rdir)
            (rdir / "manifest.json").unlink(missing_ok=True)
            if stdout_file:
                (rdir / stdout_file).write_text(out)
            index.append({"bundle": name, "run": run_name, "argv": argv, "rc": rc, "stdout_file": stdout_file})
            print(name, run_name, rc)

        for run_name, extra in PLANS.get(name, []):
            add(run_name, "plan", extra, ["cluster", "model", "workload", "slo"])
        for run_name, extra in DPS.get(name, []):
            add(run_name, "dp", extra, ["cluster", "model", "task"], stdout_file="stdout.txt")
        plan_arg = ["--plan", "inputs/plan.json" if name in FIXED_PLANS else "plan_s0/plan.json"]
        add("simulate", "simulate", plan_arg, ["cluster", "model", "workload", "slo"])
        add("costs", "costs", plan_arg, ["cluster", "model", "task"], stdout_file="stdout.txt")
        if name in ("three_tier", "two_region"):
            rm = "0" if name == "three_tier" else "5"
            add("replan", "replan", plan_arg + ["--remove", rm, "--pop", "16", "--gens", "20", "--seed", "0"],
                ["cluster", "model", "workload", "slo"])
        if name == "three_tier":
            add("replan_d7", "replan", plan_arg + ["--remove", "7", "--pop", "16", "--gens", "20", "--seed", "0"],
                ["cluster", "model", "workload", "slo"])
        if name == "two_region":
            add("ablate", "ablate", ["--pop", "8", "--gens", "10", "--seeds", "0,1"],
                ["cluster", "model", "workload", "slo"])
    (OUT / "runs.json").write_text(json.dumps(index, indent=1) + "\n")


if __name__ == "__main__":
    main()
