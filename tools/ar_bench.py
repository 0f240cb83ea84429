"""Micro-benchmark of the decode-step TP all-reduce (torchrun, 2-8 ranks):
hx fused peer all-reduce + residual + RMSNorm vs NCCL all_reduce, on the
decode message (n_tok x hidden fp32), captured in a CUDA graph of 80 calls.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ar_bench.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.distributed as dist

from paper_2311_11514_b200 import ops


def timed(fn, reps=80, iters=5):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(reps)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            fn(reps)
        g.replay()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(iters):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / iters / reps * 1e3  # us per call


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, tp = dist.get_rank(), dist.get_world_size()
    ops.load()
    H = 8192
    if "--check" in sys.argv:  # push and pull must give identical bits (several calls, both sites)
        res = {}
        for mode in ("pull", "push"):
            par = ops.PeerAllReduce(rank, tp, 32, H, 4, dist.group.WORLD, dist, mode=mode)
            g = torch.Generator(device=dev).manual_seed(1234 + rank)
            x = torch.randn(32, H, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
            gain = torch.rand(H, device=dev, generator=torch.Generator(device=dev).manual_seed(8))
            out = torch.empty(32, H, device=dev, dtype=torch.bfloat16)
            outs = []
            for i in range(7):
                par.slot(i % 4)[:32].copy_(torch.randn(32, H, device=dev, generator=g))
                par.slot(i % 4)[0, :5] = -0.0
                par.allreduce_residual_rmsnorm(x, i % 4, gain, out, 32, 1e-5)
                outs.append(out.clone())
            torch.cuda.synchronize()
            res[mode] = (x.clone(), torch.stack(outs))
        # the all-reduced residual must be bitwise identical; the normalised bf16
        # output may differ by 1 ulp (the push kernel reduces the RMS over a
        # 4-CTA cluster, the pull kernel over one 1024-thread CTA)
        d = (res["pull"][1].float() - res["push"][1].float()).abs()
        ulp = res["pull"][1].float().abs().clamp_min(1e-30) * 2.0 ** -7
        same = torch.equal(res["pull"][0], res["push"][0]) and bool((d <= ulp).all())
        xs = [torch.empty_like(res["push"][0]) for _ in range(tp)]
        dist.all_gather(xs, res["push"][0])
        os_ = [torch.empty_like(res["push"][1]) for _ in range(tp)]
        dist.all_gather(os_, res["push"][1])
        repl = all(torch.equal(xs[0], t) for t in xs) and all(torch.equal(os_[0], t) for t in os_)
        print(f"rank {rank} check push==pull: {same}, replicated: {repl}", flush=True)
        dist.barrier()
        os._exit(0 if same and repl else 1)
    if "--probe-nvls" in sys.argv:   # what torch's symmetric memory offers on this box (NVLS multicast?)
        try:
            import torch.distributed._symmetric_memory as symm
            t = symm.empty(32 * H, device=dev, dtype=torch.float32)
            hdl = symm.rendezvous(t, dist.group.WORLD.group_name)
            mc = getattr(hdl, "multicast_ptr", 0)
            print(f"rank {rank} symm mem: multicast_ptr={mc:#x} has_multicast={bool(mc)}", flush=True)
            for name in ("one_shot_all_reduce", "two_shot_all_reduce_", "multimem_all_reduce_"):
                op = getattr(torch.ops.symm_mem, name, None)
                if op is None:
                    continue
                try:
                    def run(reps, op=op, name=name):
                        for _ in range(reps):
                            if name == "one_shot_all_reduce":
                                op(t, "sum", dist.group.WORLD.group_name)
                            else:
                                op(t, "sum", dist.group.WORLD.group_name)
                    us = timed(run, reps=20, iters=3)
                    if rank == 0:
                        print(f"tp={tp} torch symm_mem.{name} 32x{H} fp32: {us:.2f} us/call", flush=True)
                except Exception as exc:  # noqa: BLE001
                    if rank == 0:
                        print(f"symm_mem.{name}: {type(exc).__name__}: {str(exc)[:160]}", flush=True)
        except Exception as exc:  # noqa: BLE001
            print(f"rank {rank} symm mem unavailable: {type(exc).__name__}: {str(exc)[:200]}", flush=True)
    sweep = ([(m, n) for m in ("push", "push-bf16") for n in (1, 8, 16, 32)] if "--sweep" in sys.argv
             else [("pull", 32), ("push", 8), ("push", 32), ("push-bf16", 32)])
    for mode, n_tok in sweep:
        par = ops.PeerAllReduce(rank, tp, n_tok, H, 80, dist.group.WORLD, dist, mode=mode.split("-")[0],
                                payload="bf16" if mode.endswith("bf16") else "fp32")
        x = torch.randn(n_tok, H, device=dev)
        gain = torch.ones(H, device=dev)
        out = torch.empty(n_tok, H, device=dev, dtype=torch.bfloat16)
        for s in (0, 1):
            par.slot(s)[:n_tok].normal_()

        def peer(reps):
            for i in range(reps):
                par.allreduce_residual_rmsnorm(x, i % 80, gain, out, n_tok, 1e-5)

        buf = torch.randn(n_tok, H, device=dev)

        def nccl(reps):
            for _ in range(reps):
                dist.all_reduce(buf)

        tp_us, nc_us = timed(peer), timed(nccl)
        if rank == 0:
            print(f"tp={tp} n_tok={n_tok} {mode}: hx peer AR+norm {tp_us:.2f} us/call | NCCL all_reduce {nc_us:.2f} us/call",
                  flush=True)
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
