#!/usr/bin/env python3
"""Benchmark: decode tokens/s of the asymmetric TP/PP data path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step is one request batch through ``Engine.generate`` (prefill, then
s_out - 1 greedy decode steps, CUDA graphs per stage). Workloads (BASELINE.json
configs; synthetic prompts, random-init weights of the named architecture):

  N=1  c2       Llama-2-7B bf16, plan [1] (32 layers), b=8, 512/128      (configs[1])
  N=2  70b-pp2  Llama-2-70B bf16, plan [1,1] layers 42/38, b=32, 1024/256
  N=3  c3-asym  Llama-2-13B bf16, plan [2,1] layers 28/12, b=8, 512/128 (configs[2])
  N=4  70b-pp3  Llama-2-70B bf16, plan [2,1,1] layers 40/20/20, b=32, 1024/256
       c3-sym   Llama-2-13B bf16, plan [2,2] layers 20/20, b=8, 512/128 (--workload c3-sym; configs[2])
  N=8  c4       Llama-2-70B bf16, plan [4,2,2] layers 40/20/20, b=32, 1024/256 (configs[3])

``value`` = decode tokens/s = b * (s_out - 1) * K / (sum of decode-phase device
time, CUDA events, on the last stage -- first to last generated token -- max
over its ranks), inputs resident. ``e2e`` = generated
tokens/s through the public API with host prompts in and host ids out
(b * s_out per request / wall time of generate, prefill included) -- the
same unit and definition in both arms.
Weights (13.5-140 GB) are far larger than the 126 MB L2, so every decode step
streams them from HBM; no L2 flush is needed.

``--impl reference`` times the CPU oracle port (oracle/llama_oracle.py, the
only CPU implementation of the path; the reference repo has none) on the
host cores for the same workload: per step, one transformer layer decode step
at the config shape (batch b, mid-generation context) + lm_head, and one layer
prefill of one prompt + lm_head row, extrapolated to all layers and prompts
(value = decode tok/s, e2e = b * s_out / (prefill + (s_out - 1) decode steps)).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/s (greedy, b x (s_out-1) / decode time)"
UNIT = "tok/s"

WORKLOADS = {
    "c2": dict(model="llama2-7b", tps=[1], layers=[32], batch=8, s_in=512, s_out=128),
    "70b-pp2": dict(model="llama2-70b", tps=[1, 1], layers=[42, 38], batch=32, s_in=1024, s_out=256),
    "70b-pp3": dict(model="llama2-70b", tps=[2, 1, 1], layers=[40, 20, 20], batch=32, s_in=1024, s_out=256),
    "c4": dict(model="llama2-70b", tps=[4, 2, 2], layers=[40, 20, 20], batch=32, s_in=1024, s_out=256),
    "c3-asym": dict(model="llama2-13b", tps=[2, 1], layers=[28, 12], batch=8, s_in=512, s_out=128),
    "c3-sym": dict(model="llama2-13b", tps=[2, 2], layers=[20, 20], batch=8, s_in=512, s_out=128),
}
BY_GPUS = {1: "c2", 2: "70b-pp2", 3: "c3-asym", 4: "70b-pp3", 8: "c4"}


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


def workload(n, args):
    w = dict(WORKLOADS[args.workload or BY_GPUS.get(n, "c2")])
    if args.model:
        w["model"] = args.model
    if args.plan:
        w["tps"] = [int(x) for x in args.plan.split(",")]
    if args.layers:
        w["layers"] = [int(x) for x in args.layers.split(",")]
    for k in ("batch", "s_in", "s_out"):
        if getattr(args, k):
            w[k] = getattr(args, k)
    return w


def wl_name(w):
    return (f"{w['model']} bf16 plan [{','.join(map(str, w['tps']))}] layers "
            f"{'/'.join(map(str, w['layers']))} b={w['batch']} {w['s_in']}/{w['s_out']}")


def config_dict(w, cfg):
    """The workload, identical in both arms' JSON lines."""
    return {"workload": wl_name(w), "model": cfg.name, "plan": w["tps"], "layers": w["layers"],
            "global_batch": w["batch"], "seq_len": w["s_in"], "decode_tokens": w["s_out"],
            "parallelism": "pp%d-tp[%s]" % (len(w["tps"]), ",".join(map(str, w["tps"]))),
            "l2": "weights stream from HBM each step (>> 126 MB L2); no flush"}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


E2E_UNIT = "tok/s"
E2E_DEF = "b x s_out generated tokens per request / request wall time, host prompt in -> host ids out (prefill included)"


# ----------------------------------------------------------------- accounting
def decode_bytes_per_step(cfg, w):
    """Algorithmic HBM bytes of one decode step summed over all GPUs
    (SURVEY §8d): weight shards + lm_head + KV read at the mean context."""
    B = 2
    ctx = w["s_in"] + (w["s_out"] - 1) / 2.0
    per_layer = cfg.params_per_layer() * B
    kv = w["batch"] * ctx * 2 * cfg.num_kv_heads * cfg.head_dim * B
    return cfg.num_layers * (per_layer + kv) + cfg.vocab * cfg.hidden_dim * B


def decode_roofline_step_s(cfg, w, bw):
    """T* = sum over stages of max-per-GPU bytes / BW."""
    B = 2
    ctx = w["s_in"] + (w["s_out"] - 1) / 2.0
    t = 0.0
    for j, (tp, l) in enumerate(zip(w["tps"], w["layers"])):
        b = l * (cfg.params_per_layer() * B / tp + w["batch"] * ctx * 2 * (cfg.num_kv_heads / tp) * cfg.head_dim * B)
        if j == len(w["tps"]) - 1:
            b += cfg.vocab * cfg.hidden_dim * B / tp
        t += b / (bw * 1e9)
    return t


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        power = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------- CPU oracle
_CPU_WEIGHTS: dict = {}


def _cpu_weights(cfg, seed):
    """Layer 0 + final norm + lm_head (weight generation is setup, not timed)."""
    from paper_2311_11514_b200.weights import init_globals, layer_stream
    key = (cfg, seed)
    if key not in _CPU_WEIGHTS:
        _, lw = next(layer_stream(cfg, seed, [0], lookahead=0))
        _CPU_WEIGHTS[key] = {"layers": {0: lw}, **init_globals(cfg, seed, ("norm", "lm_head"))}
    return _CPU_WEIGHTS[key]


def cpu_decode_sample(cfg, w, steps=2, seed=0):
    """Time the CPU oracle on one layer's decode step at the config shape
    (batch b, context = mean generation context) + final norm + lm_head;
    return extrapolated decode tok/s for the full model (all host threads)."""
    from oracle.llama_oracle import Cache, Oracle
    b = w["batch"]
    ctx = int(w["s_in"] + (w["s_out"] - 1) / 2)
    orc = Oracle(cfg, _cpu_weights(cfg, seed))
    rng = np.random.default_rng(0)
    times = []
    for _ in range(steps):
        cache = Cache()
        cache.k[0] = rng.standard_normal((b, cfg.num_kv_heads, ctx, cfg.head_dim), dtype=np.float32)
        cache.v[0] = rng.standard_normal((b, cfg.num_kv_heads, ctx, cfg.head_dim), dtype=np.float32)
        x = rng.standard_normal((b, 1, cfg.hidden_dim), dtype=np.float32)
        t0 = time.perf_counter()
        y = orc.layer(0, x, ctx, cache)
        t1 = time.perf_counter()
        orc.logits(y[:, -1])
        t2 = time.perf_counter()
        times.append((t1 - t0) * cfg.num_layers + (t2 - t1))
    step_s = min(times)
    return b / step_s, step_s


def cpu_prefill_sample(cfg, w, seed=0):
    """Time the CPU oracle on one layer's prefill of ONE prompt (s_in tokens)
    + the lm_head row; return the extrapolated prefill seconds of the whole
    request: x b sequences (independent, same cost) x L layers."""
    from oracle.llama_oracle import Cache, Oracle
    orc = Oracle(cfg, _cpu_weights(cfg, seed))
    x = np.random.default_rng(0).standard_normal((1, w["s_in"], cfg.hidden_dim), dtype=np.float32)
    t0 = time.perf_counter()
    y = orc.layer(0, x, 0, Cache())
    t1 = time.perf_counter()
    orc.logits(y[:, -1])
    t2 = time.perf_counter()
    return w["batch"] * (t1 - t0) * cfg.num_layers + w["batch"] * (t2 - t1)


def run_reference(args, w, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    cores = os.cpu_count()
    torch.set_num_threads(cores)
    for _ in range(max(0, args.warmup)):
        cpu_decode_sample(cfg, w, steps=1)
        cpu_prefill_sample(cfg, w)
    vals, e2es, t0 = [], [], time.perf_counter()
    b, s_out = w["batch"], w["s_out"]
    for _ in range(args.steps):
        v, step_s = cpu_decode_sample(cfg, w, steps=1)
        pre_s = cpu_prefill_sample(cfg, w)
        vals.append(v)
        e2es.append(b * s_out / (pre_s + (s_out - 1) * step_s))
    wall = time.perf_counter() - t0
    value = float(np.mean(vals))
    e2e = float(np.mean(e2es))
    sample = (f"CPU oracle port (numpy fp32, {cores} threads, {cpu_model()}): per step one {cfg.name} layer "
              f"decode step at b={b}, ctx={int(w['s_in'] + (s_out - 1) / 2)} + lm_head (x{cfg.num_layers} layers) "
              f"and one layer prefill of one {w['s_in']}-token prompt + lm_head row (x{b} prompts x"
              f"{cfg.num_layers} layers); e2e = b*s_out / (prefill + (s_out-1) decode steps), extrapolated")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / max(1, args.steps) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_dict(w, cfg),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": e2e, "unit": E2E_UNIT, "definition": E2E_DEF, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- GPU
def gemm_roofline(eng, cfg, w, hbm, reps=5):
    """Live CUDA-event timing of the dominant kernel, hx_linear in its decode
    (weight-streaming) form: one decode step's GEMM sequence of this rank
    (QKV, O, gate/up, down per layer + lm_head) captured in a graph and
    replayed; algorithmic bytes = weights + activations in + outputs."""
    import torch
    from paper_2311_11514_b200 import ops
    e = eng.execs[0]
    b = w["batch"]
    seq, nbytes = [], 0
    for lw in e.w["layers"]:
        for wt, xin, y in ((lw["wqkv"], e.h, e.qkv), (lw["wo"], e.attn, e.proj), (lw["wgu"], e.h, e.gu),
                           (lw["wdown"], e.a, e.proj)):
            seq.append((wt, xin, y))
    if e.role.is_last:
        seq.append((e.w["lm_head"], e.hl, e.logits))
    for wt, xin, y in seq:
        n_out, k = wt.shape
        nbytes += n_out * k * 2 + b * k * 2 + b * n_out * y.element_size()

    def run():
        for wt, xin, y in seq:
            ops.linear(wt, xin, y, b, e.lin_ws)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    st = torch.cuda.current_stream()
    g.replay()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(st)
    for _ in range(reps):
        g.replay()
    s1.record(st)
    torch.cuda.synchronize()
    t = s0.elapsed_time(s1) / 1e3 / reps
    achieved = nbytes / t / 1e9
    # per projection shape: the same GEMM over every layer's weights, back to back
    per_shape = {}
    names = ["qkv", "o", "gate_up", "down"]
    for i, name in enumerate(names):
        sub = seq[i:4 * len(e.w["layers"]):4]
        if not sub:
            continue
        gb = sum(wt.shape[0] * wt.shape[1] * 2 + b * wt.shape[1] * 2 + b * wt.shape[0] * y.element_size()
                 for wt, xin, y in sub)
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            for wt, xin, y in sub:
                ops.linear(wt, xin, y, b, e.lin_ws)
        g2.replay()
        torch.cuda.synchronize()
        s0.record(st)
        for _ in range(reps):
            g2.replay()
        s1.record(st)
        torch.cuda.synchronize()
        ts = s0.elapsed_time(s1) / 1e3 / reps
        per_shape[name] = {"shape": list(sub[0][0].shape), "us_per_launch": round(ts / len(sub) * 1e6, 2),
                           "GBps": round(gb / ts / 1e9, 1)}
    traffic = None
    tfile = ROOT / "profiles" / "r02" / "gemm_traffic.json"
    if cfg.name == "llama2-7b" and w["batch"] == 8 and tfile.exists():
        # dram read+write per launch from ncu --set full captures of the same
        # kernel at this workload's four layer shapes (one launch per shape, each
        # in its own process: tools/gemm_traffic.py), against the algorithmic
        # bytes per launch
        tj = json.loads(tfile.read_text())
        tr, al = tj["traffic_bytes_per_launch_avg_7b_layer"], tj["algorithmic_bytes_per_launch_avg_7b_layer"]
        traffic = {"bytes_per_launch": round(tr), "algorithmic_bytes_per_launch": round(al),
                   "ratio": round(tr / al, 4), "source": "profiles/r02/gemm_traffic.json"}
    return {"bound": "hbm", "kernel": "hx_linear (tcgen05 stream-K decode GEMM)", "achieved": round(achieved, 1),
            "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
            "launches_per_step": len(seq), "avg_launch_us": round(t / len(seq) * 1e6, 2),
            "bytes_per_step": nbytes, "gemm_ms_per_step": round(t * 1e3, 4), "per_shape": per_shape}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hexgen", choices=["hexgen", "reference"])
    ap.add_argument("--workload", choices=sorted(WORKLOADS), help="default by --gpus: " + str(BY_GPUS))
    ap.add_argument("--model")
    ap.add_argument("--plan")
    ap.add_argument("--layers")
    ap.add_argument("--batch", type=int)
    ap.add_argument("--s-in", dest="s_in", type=int)
    ap.add_argument("--s-out", dest="s_out", type=int)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2311_11514_b200.config import preset
    w = workload(args.gpus, args)
    cfg = preset(w["model"])
    if args.impl == "reference":
        return run_reference(args, w, cfg)

    import torch
    import torch.distributed as dist
    from paper_2311_11514_b200 import ops
    from paper_2311_11514_b200.engine import Engine
    from paper_2311_11514_b200.plan import simple_plan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ops.load()
    plan = simple_plan(w["tps"], w["layers"])
    if sum(w["tps"]) != world and world > 1:
        raise SystemExit(f"plan {w['tps']} needs {sum(w['tps'])} ranks, have {world}")
    eng = Engine(plan, cfg, dtype="bf16", batch=w["batch"], max_prompt=w["s_in"], max_out=w["s_out"],
                 comm="dist" if world > 1 else "local", device=dev, weights="device", seed=0)
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(w["batch"], w["s_in"]), dtype=np.int32)
    for _ in range(args.warmup):
        eng.generate(prompt, w["s_out"])
    hbm, tflops, peak_kind = peaks()
    clocks = ClockSampler(local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    clocks.start()
    t_wall0 = time.perf_counter()
    dec_s, pre_s, steps_ms, walls, launches = 0.0, 0.0, [], [], 0
    for _ in range(args.steps):
        a = time.perf_counter()
        r = eng.generate(prompt, w["s_out"])   # host prompt in, host ids out
        walls.append(time.perf_counter() - a)
        dec_s += r.decode_s
        pre_s += r.prefill_s
        steps_ms += r.step_ms
        launches += r.launches
    barrier()
    wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    # The decode phase runs from the first generated token (the last stage's
    # prefill head) to the last one, so its duration is taken on the last
    # stage (max over its ranks). Earlier stages' decode clocks start when their
    # own prefill micro-batches end and also absorb the later stages' prefill
    # tail; that max-over-all-ranks figure is reported as decode_s_all_ranks.
    is_last = any(e.role.is_last for e in eng.execs)
    t = torch.tensor([dec_s, pre_s, wall, sum(walls), dec_s if is_last else 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dec_all, pre_s, wall, wall_gen, dec_s = t.tolist()
    b, s_in, s_out = w["batch"], w["s_in"], w["s_out"]
    value = b * (s_out - 1) * args.steps / dec_s
    e2e = b * s_out * args.steps / wall_gen
    roof = gemm_roofline(eng, cfg, w, hbm)
    if world > 1:
        rt = torch.tensor([roof["frac"]], device=dev, dtype=torch.float64)
        dist.all_reduce(rt, op=dist.ReduceOp.MIN)
    step_rf = decode_roofline_step_s(cfg, w, hbm)
    p50 = statistics.median(steps_ms) if steps_ms else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import torch as _t
        _t.set_num_threads(os.cpu_count())
        v, st = cpu_decode_sample(cfg, w, steps=2)
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "cpu_model": cpu_model(),
               "sample": f"CPU oracle (numpy fp32): 1 {cfg.name} layer decode step b={b} ctx={int(s_in + (s_out - 1) / 2)}"
                         f" + lm_head, x{cfg.num_layers} layers ({st * 1e3:.0f} ms/step extrapolated)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, uniform prompts seed 1)",
            "config": config_dict(w, cfg),
            "p50_decode_step_ms": round(p50, 4) if p50 else None,
            "p90_decode_step_ms": round(float(np.percentile(steps_ms, 90)), 4) if steps_ms else None,
            "prefill_ms": round(pre_s / args.steps * 1e3, 3),
            "decode_ms_per_request": round(dec_s / args.steps * 1e3, 3),
            "decode_s_all_ranks": round(dec_all / args.steps, 4),
            "step_roofline": {"bytes_per_step_all_gpus": decode_bytes_per_step(cfg, w),
                              "t_star_ms": round(step_rf * 1e3, 4),
                              "frac": round(step_rf * 1e3 / p50, 4) if p50 else None,
                              "peak_gbs": hbm, "peak_kind": peak_kind},
            "roofline": roof,
            "e2e": {"value": round(e2e, 2), "unit": E2E_UNIT, "definition": E2E_DEF,
                    "h2d_bytes_per_step": b * s_in * 4, "d2h_bytes_per_step": b * s_out * 4},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        sys.stdout.flush()
        sys.stderr.flush()
        # NCCL communicators captured in CUDA graphs can hang destroy_process_group;
        # the measurement is complete, so every rank exits directly.
        os._exit(0)
    return 0


if __name__ == "__main__":
    sys.exit(main())
