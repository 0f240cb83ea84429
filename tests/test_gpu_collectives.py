"""The multi-GPU decode collectives on ONE GPU: every TP rank (or hand-off end)
is emulated by its own CUDA stream and the peer pointers are same-device
pointers, so the real kernels run with real concurrency -- each rank's
all-reduce kernel genuinely waits for the other ranks' pushes.

* ``hx_tp_allreduce_push_residual_rmsnorm`` (a6/a8; the
  reference's ``tp_comm_cost``, costs.py:123-147) at TP=2 and TP=4, several
  consecutive calls over both call sites (inbox buffer parity, in-place
  re-arm): the residual must be BITWISE the rank-order fp32 sum
  x + (((p0 + p1) + p2) + p3) on every rank, identical to the flag/pull
  variant, and the normalised output within fp32 rounding of torch.
* ``hx_handoff_push`` / ``hx_handoff_pull`` (a9; ``pp_comm_cost``,
  costs.py:150-165): the fan-out 1->2, fan-in 2->1 and 2->2 reshard routes and
  the token-id return, with the receiver's pull launched BEFORE the sender's
  push (it must spin until the data lands), variable sizes, and enough
  consecutive hand-offs to cycle the 3 inbox buffers twice.
"""

import pytest
import torch

from paper_2311_11514_b200 import ops
from paper_2311_11514_b200.config import LlamaConfig
from paper_2311_11514_b200.plan import simple_plan
from paper_2311_11514_b200.topology import pipeline_roles

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(autouse=True, scope="module")
def _lib():
    ops.load()


def _ref_allreduce(x, parts, gain, eps):
    s = parts[0].clone()
    for p in parts[1:]:
        s = s + p
    xn = x + s
    inv = torch.rsqrt(xn.double().pow(2).mean(-1, keepdim=True) + eps)
    return xn, (xn.double() * inv * gain.double()).float()


def _run_group(group, xs, parts_per_call, gain, out_dtype, n_tok, eps=1e-5):
    """Launch every rank's all-reduce of each call on its own stream, all
    ranks' launches of a call queued before anything synchronises."""
    tp = len(group)
    streams = [torch.cuda.Stream() for _ in range(tp)]
    outs_per_call = []
    for call, parts in enumerate(parts_per_call):
        site = call % 4
        for r in range(tp):
            group[r].slot(site)[:n_tok].copy_(parts[r])
        torch.cuda.synchronize()
        outs = [torch.full((n_tok, gain.numel()), float("nan"), device=DEV, dtype=out_dtype) for _ in range(tp)]
        for r in range(tp):
            with torch.cuda.stream(streams[r]):
                group[r].allreduce_residual_rmsnorm(xs[r], site, gain, outs[r], n_tok, eps)
        torch.cuda.synchronize()
        outs_per_call.append([o.clone() for o in outs])
    return outs_per_call


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("n_tok,hidden", [(1, 4096), (8, 4096), (32, 8192), (5, 5120)])
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_peer_allreduce_bf16_payload_single_gpu_streams(tp, n_tok, hidden, out_dtype):
    """bf16 payload: every partial rounded to bf16 once (own included), summed in
    fp32 in rank order -- residual bitwise x + sum_r float(bf16(p_r)), replicated."""
    n_tok = min(n_tok, ops.PEER_AR_CORESIDENT // (4 * tp))   # all emulated ranks' CTAs co-resident
    calls, eps = 4, 1e-5
    g = torch.Generator(device=DEV).manual_seed(tp * 31 + n_tok + hidden)
    x0 = torch.randn(n_tok, hidden, device=DEV, generator=g)
    gain = 1 + 0.02 * torch.randn(hidden, device=DEV, generator=g)
    parts_per_call = []
    for c in range(calls):
        parts = [torch.randn(n_tok, hidden, device=DEV, generator=g) for _ in range(tp)]
        parts[0][0, :9] = -0.0
        parts[-1][-1, -5:] = -1e-42          # rounds to bf16 -0.0: must not read as the sentinel
        parts_per_call.append(parts)
    group = ops.PeerAllReduce.local_group(tp, 32, hidden, 4, mode="push", payload="bf16")
    xs = [x0.clone() for _ in range(tp)]
    outs = _run_group(group, xs, parts_per_call, gain, out_dtype, n_tok, eps)
    for o in group:
        o.close()
    x_ref = x0.clone()
    for c in range(calls):
        x_ref, y_ref = _ref_allreduce(x_ref, [p.bfloat16().float() for p in parts_per_call[c]], gain, eps)
        for r in range(tp):
            tol = 1e-5 if out_dtype == torch.float32 else 8e-3
            assert (outs[c][r].float() - y_ref).abs().max() <= tol * y_ref.abs().max()
            assert torch.equal(outs[c][r], outs[c][0])
    for r in range(tp):
        assert torch.equal(xs[r], x_ref)


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("n_tok,hidden", [(1, 4096), (8, 4096), (32, 8192), (5, 5120)])
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_peer_allreduce_single_gpu_streams(tp, n_tok, hidden, out_dtype):
    n_tok = min(n_tok, ops.PEER_AR_CORESIDENT // (4 * tp))   # all emulated ranks' CTAs co-resident
    calls, eps = 5, 1e-5
    g = torch.Generator(device=DEV).manual_seed(tp * 100 + n_tok + hidden)
    x0 = torch.randn(n_tok, hidden, device=DEV, generator=g)
    gain = 1 + 0.02 * torch.randn(hidden, device=DEV, generator=g)
    parts_per_call = []
    for c in range(calls):
        parts = [torch.randn(n_tok, hidden, device=DEV, generator=g) for _ in range(tp)]
        parts[0][0, :7] = -0.0            # -0.0 partials must not look like the inbox sentinel
        parts[-1][-1, -3:] = -0.0
        parts_per_call.append(parts)
    results = {}
    for mode in ("push", "pull"):
        group = ops.PeerAllReduce.local_group(tp, 32, hidden, 4, mode=mode)
        xs = [x0.clone() for _ in range(tp)]
        outs = _run_group(group, xs, parts_per_call, gain, out_dtype, n_tok, eps)
        results[mode] = (xs, outs)
        for o in group:
            o.close()
    x_ref = x0.clone()
    for c in range(calls):
        x_ref, y_ref = _ref_allreduce(x_ref, parts_per_call[c], gain, eps)
        for mode in ("push", "pull"):
            out = results[mode][1][c]
            for r in range(tp):
                assert not torch.isnan(out[r].float()).any()
                tol = 1e-5 if out_dtype == torch.float32 else 8e-3
                assert (out[r].float() - y_ref).abs().max() <= tol * y_ref.abs().max(), (mode, c, r)
                assert torch.equal(out[r], out[0]), "normalised output not replicated across ranks"
    for mode in ("push", "pull"):
        for r in range(tp):
            assert torch.equal(results[mode][0][r], x_ref), f"{mode}: residual != rank-order fp32 sum (rank {r})"


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("n_tok,hidden,k_dim", [(8, 8192, 2048), (16, 8192, 7168), (5, 4096, 11008)])
def test_peer_allreduce_deferred_gemm_single_gpu(tp, n_tok, hidden, k_dim):
    """TP>1 decode with the row-parallel GEMM deferred (HX_LINEAR_DEFER_REDUCE):
    each rank's all-reduce sums the GEMM's split tiles from its partial slots
    while reading the row (hx_tp_allreduce_push_residual_rmsnorm_sk). Residual
    and output must be BITWISE those of the GEMM with its in-kernel fix-up
    followed by the plain push all-reduce, over consecutive calls."""
    n_tok = min(n_tok, ops.PEER_AR_CORESIDENT // (4 * tp))
    eps, calls = 1e-5, 3
    g = torch.Generator(device=DEV).manual_seed(tp * 7 + n_tok + k_dim)
    x0 = torch.randn(n_tok, hidden, device=DEV, generator=g)
    gain = 1 + 0.02 * torch.randn(hidden, device=DEV, generator=g)
    ws_words = ops.linear_workspace(torch.bfloat16, n_tok, hidden, k_dim) // 4 + 64
    ws = [torch.zeros(ws_words, dtype=torch.int32, device=DEV) for _ in range(tp)]
    calls_in = []
    for c in range(calls):
        w = [ops.PackedWeight((torch.randn(hidden, k_dim, device=DEV, generator=g) * 0.02).bfloat16())
             for _ in range(tp)]
        a = [torch.randn(n_tok, k_dim, device=DEV, generator=g).bfloat16() for _ in range(tp)]
        calls_in.append((w, a))
    results = {}
    for deferred in (False, True):
        group = ops.PeerAllReduce.local_group(tp, 32, hidden, 4, mode="push", payload="bf16")
        xs = [x0.clone() for _ in range(tp)]
        streams = [torch.cuda.Stream() for _ in range(tp)]
        outs = []
        for c, (w, a) in enumerate(calls_in):
            site = c % 4
            for r in range(tp):   # every rank's GEMM first (own workspace), then the all-reduces together
                ops.linear(w[r], a[r], group[r].slot(site), n_tok, ws[r], defer_reduce=deferred)
            torch.cuda.synchronize()
            o = [torch.empty(n_tok, hidden, device=DEV, dtype=torch.bfloat16) for _ in range(tp)]
            for r in range(tp):
                with torch.cuda.stream(streams[r]):
                    kw = {"gemm_ws": ws[r], "k_dim": k_dim} if deferred else {}
                    group[r].allreduce_residual_rmsnorm(xs[r], site, gain, o[r], n_tok, eps, **kw)
            torch.cuda.synchronize()
            outs.append(o)
        for q in group:
            q.close()
        results[deferred] = (xs, outs)
    for r in range(tp):
        assert torch.equal(results[True][0][r], results[False][0][r]), f"residual differs (rank {r})"
        assert torch.equal(results[True][0][r], results[True][0][0])
        for c in range(calls):
            assert torch.equal(results[True][1][c][r], results[False][1][c][r]), f"output differs (call {c})"


def test_peer_allreduce_graph_replay_single_gpu():
    """The emulated ranks' all-reduces captured in one CUDA graph (fork/join
    over per-rank streams) and replayed: the call counters and re-armed
    inboxes carry over between replays."""
    tp, n_tok, hidden = 4, 8, 8192
    group = ops.PeerAllReduce.local_group(tp, n_tok, hidden, 2)
    g = torch.Generator(device=DEV).manual_seed(5)
    gain = torch.ones(hidden, device=DEV)
    parts = [torch.randn(n_tok, hidden, device=DEV, generator=g) for _ in range(tp)]
    for r in range(tp):
        for site in range(2):
            group[r].slot(site)[:n_tok].copy_(parts[r])
    xs = [torch.zeros(n_tok, hidden, device=DEV) for _ in range(tp)]
    outs = [torch.empty(n_tok, hidden, device=DEV, dtype=torch.bfloat16) for _ in range(tp)]
    streams = [torch.cuda.Stream() for _ in range(tp)]

    def step():
        main = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(main)
        done = []
        for site in range(2):
            for r in range(tp):
                streams[r].wait_event(ev)
            evs = []
            for r in range(tp):
                with torch.cuda.stream(streams[r]):
                    group[r].allreduce_residual_rmsnorm(xs[r], site, gain, outs[r], n_tok, 1e-5)
                e = torch.cuda.Event()
                e.record(streams[r])
                evs.append(e)
            ev = evs[-1]
            for r in range(tp):          # next site starts after every rank's call
                for e in evs:
                    streams[r].wait_event(e)
            done = evs
        for e in done:
            main.wait_event(e)

    step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="thread_local"):
        step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    s = parts[0].clone()
    for p in parts[1:]:
        s = s + p
    want = torch.zeros(n_tok, hidden, device=DEV)
    for _ in range(2 * 4):               # eager step + 3 replays, 2 sites each
        want = want + s
    for r in range(tp):
        assert torch.equal(xs[r], want)
    for o in group:
        o.close()


# ------------------------------------------------------------------ P2P hand-off
def _links_for(plan_tps, plan_layers):
    """Every decode hand-off link of a pipeline (hidden j -> j+1, ids last -> 0)."""
    cfg = LlamaConfig("route-probe", sum(plan_layers), 256, 8, 8, 768, 32000)
    roles = pipeline_roles(simple_plan(plan_tps, plan_layers), 0, cfg)
    hidden = [(r.device, d) for r in roles for d in r.send_to]
    ids = [(r.device, d) for r in roles for d in r.ids_send_to]
    return hidden, ids


@pytest.mark.parametrize("tps,layers,route", [
    ([1, 2], [1, 1], "fan-out 1->2"),
    ([2, 1], [1, 1], "fan-in 2->1"),
    ([2, 2], [1, 1], "2->2"),
    ([4, 2, 2], [2, 1, 1], "[4,2,2] incl. token return 2->4"),
])
def test_handoff_routes_single_gpu_streams(tps, layers, route):
    hidden_links, id_links = _links_for(tps, layers)
    H, b = 4096, 8
    for kind, links, words in (("hidden", hidden_links, b * H), ("ids", id_links, b)):
        if not links:
            continue
        objs = {lk: ops.P2PLink.local(lk[0], lk[1], words) for lk in links}
        s_send = {lk: torch.cuda.Stream() for lk in links}
        s_recv = {lk: torch.cuda.Stream() for lk in links}
        g = torch.Generator(device=DEV).manual_seed(len(links))
        for call in range(7):                   # cycles the 3 inbox buffers twice
            n = words if call % 3 else max(4, words // 2 - 4 * call)   # variable sizes
            srcs, dsts = {}, {}
            for lk in links:
                if kind == "hidden":
                    t = torch.randn(n, device=DEV, generator=g)
                    t[:3] = -0.0                # sent as +0.0 (sentinel-safe)
                else:
                    t = torch.randint(0, 32000, (n,), device=DEV, dtype=torch.int32, generator=g)
                srcs[lk] = t
                dsts[lk] = torch.full_like(t, -7 if kind == "ids" else float("nan"))
            torch.cuda.synchronize()
            for lk in links:                    # receivers first: they spin until the data lands
                with torch.cuda.stream(s_recv[lk]):
                    objs[lk].pull(dsts[lk])
            for lk in links:
                with torch.cuda.stream(s_send[lk]):
                    objs[lk].push(srcs[lk])
            torch.cuda.synchronize()
            for lk in links:
                want = srcs[lk] + 0.0 if kind == "hidden" else srcs[lk]   # -0.0 arrives as +0.0
                assert torch.equal(dsts[lk], want), (route, kind, lk, call)
        for o in objs.values():
            o.close()


def test_handoff_push_multi_destination():
    """One push kernel storing into two receivers' inboxes (C-ABI n_dst = 2)."""
    import ctypes
    words = 8 * 1024
    a, b = ops.P2PLink.local(0, 1, words), ops.P2PLink.local(0, 2, words)
    lib = ops.load()
    state = torch.zeros(2, dtype=torch.int32, device=DEV)
    src = torch.randn(words, device=DEV)
    arr = (ctypes.c_void_p * 2)(a._peer, b._peer)
    for _ in range(4):
        da, db = torch.empty_like(src), torch.empty_like(src)
        rc = lib.hx_handoff_push(src.data_ptr(), arr, 2, words, a.max_words, state.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        a.pull(da)
        b.pull(db)
        torch.cuda.synchronize()
        assert torch.equal(da, src) and torch.equal(db, src)
    a.close()
    b.close()


@pytest.mark.parametrize("words", [4096 * 64, 1000 * 8 + 3])
def test_credit_handoff_sender_runs_ahead(words):
    """The prefill stream of hand-offs (hx_handoff_push/pull_credit): the sender
    queues 7 micro-batches before the receiver drains any -- its 4th push must
    wait (over the credit word) until buffer 0 was drained, re-armed and handed
    back; every micro-batch arrives intact and in order."""
    link = ops.P2PLink.local(0, 1, words)
    g = torch.Generator(device=DEV).manual_seed(words % 97)
    n = 7
    srcs = [torch.randn(words - 4 * (k % 2), device=DEV, generator=g) for k in range(n)]
    for s_ in srcs:
        s_[:2] = -0.0
    dsts = [torch.full_like(s_, float("nan")) for s_ in srcs]
    torch.cuda.synchronize()
    send, recv = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(send):
        for s_ in srcs:
            link.push_credit(s_)
    with torch.cuda.stream(recv):
        for d in dsts:
            link.pull_credit(d)
    torch.cuda.synchronize()
    for s_, d in zip(srcs, dsts):
        assert torch.equal(d, s_ + 0.0)
    link.close()
