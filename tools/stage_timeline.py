"""Per-stage attribution of the multi-GPU decode step (torchrun, one rank per GPU).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/stage_timeline.py \
        --model llama2-70b --plan 2,1,1 --layers 40,20,20

After a warm generate, every rank:
  1. replays its own stage's decode graph back to back (stage-mates start
     together after a barrier; other stages idle) -> pure stage compute time;
  2. runs real decode steps with CUDA events around its phases
     (ids return, hidden recv, graph replay, hidden send) -> where a step waits.
Prints one line per rank.
"""
import argparse
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import torch.distributed as dist

from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import simple_plan


def main():
    os.environ.setdefault("HX_P2P", "0")  # solo stage replays cannot wait on P2P hand-offs
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-70b")
    ap.add_argument("--plan", default="2,1,1")
    ap.add_argument("--layers", default="40,20,20")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--s-in", type=int, default=1024)
    ap.add_argument("--s-out", type=int, default=64)
    a = ap.parse_args()
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = preset(a.model)
    plan = simple_plan([int(x) for x in a.plan.split(",")], [int(x) for x in a.layers.split(",")])
    eng = Engine(plan, cfg, dtype="bf16", batch=a.batch, max_prompt=a.s_in, max_out=a.s_out, comm="dist",
                 device=dev, weights="device")
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(a.batch, a.s_in), dtype=np.int32)
    r = eng.generate(prompt, a.s_out)
    r = eng.generate(prompt, a.s_out)
    step_p50 = statistics.median(r.step_ms)
    d = eng.drivers[0]
    g = eng._graphs[0]
    # 1. solo replays, stage by stage (the other stages wait at the barrier)
    solo = {}
    for j in range(eng.num_stages):
        dist.barrier()
        torch.cuda.synchronize()
        if d.stage == j:
            if d.tp > 1:
                dist.barrier(group=eng.comm.groups[d.role.tp_group])
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g.replay()
            s0.record()
            for _ in range(10):
                g.replay()
            s1.record()
            torch.cuda.synchronize()
            solo[j] = s0.elapsed_time(s1) / 10
    dist.barrier()
    torch.cuda.synchronize()
    # 2. real steps with phase events (prefill first so the KV state is valid)
    eng._reset(a.batch, a.s_in, a.s_out)
    for e in eng.execs:
        if e.role.is_first:
            e.prompt[:a.batch * a.s_in].copy_(torch.from_numpy(prompt.reshape(-1)))
    eng._prefill(a.batch, a.s_in)
    ph = {"ids": [], "recv": [], "graph": [], "send": []}
    for _ in range(1, a.s_out):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        evs[0].record()
        eng._return_ids()
        evs[1].record()
        if d.stage > 0:
            d.recv_hidden(a.batch)
        evs[2].record()
        g.replay()
        evs[3].record()
        if d.stage < eng.num_stages - 1:
            d.send_hidden(a.batch)
        evs[4].record()
        torch.cuda.synchronize()
        for k, (x, y) in zip(ph, zip(evs, evs[1:])):
            ph[k].append(x.elapsed_time(y))
    med = {k: round(statistics.median(v), 3) for k, v in ph.items()}
    print(f"rank {rank} stage {d.stage} tp {d.tp}: generate p50 step {step_p50:.3f} ms | solo graph "
          f"{solo.get(d.stage, float('nan')):.3f} ms | in-step phases (ms) {med}", flush=True)
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
