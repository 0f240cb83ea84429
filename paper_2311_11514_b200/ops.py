"""ctypes bindings to ``libhexgen.so`` (the C-ABI in ``include/hx_api.h``).

Torch tensors are used only as device memory: each wrapper passes raw data
pointers, sizes and the current CUDA stream across the C boundary. There is
no fallback -- if the library is missing or a call fails, these functions
raise (``HxError``); the data path has no CPU or eager-PyTorch substitute.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "libhexgen.so"
HX_F32, HX_BF16 = 0, 1

_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_SZ = ctypes.c_size_t

_SIGS = {
    "hx_version": ([], _I),
    "hx_error_string": ([_I], ctypes.c_char_p),
    "hx_launch_count": ([], ctypes.c_uint64),
    "hx_embed": ([_P, _P, _I, _P, _I, _I, _I, _P], _I),
    "hx_rmsnorm": ([_P, _I, _P, _P, _I, _I, _I, _F, _P], _I),
    "hx_residual_add_rmsnorm": ([_P, _P, _P, _P, _I, _I, _I, _F, _P], _I),
    "hx_linear": ([_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _SZ, _P], _I),
    "hx_linear_workspace": ([_I, _I, _I, _I], _SZ),
    "hx_pack_weight": ([_P, _P, _I, _I, _P], _I),
    "hx_packed_weight_elems": ([_I, _I], _SZ),
    "hx_set_pdl": ([_I], None),
    "hx_debug_trace": ([_P, _SZ], _SZ),
    "hx_splitk_residual_rmsnorm": ([_P, _P, _I, _P, _I, _I, _I, _P, _P, _I, _F, _P], _I),
    "hx_ipc_alloc": ([ctypes.POINTER(ctypes.c_void_p), _SZ], _I),
    "hx_ipc_free": ([_P], _I),
    "hx_ipc_handle": ([_P, ctypes.c_char_p], _I),
    "hx_ipc_open": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)], _I),
    "hx_ipc_close": ([_P], _I),
    "hx_tp_allreduce_residual_rmsnorm": ([_P, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                          _I, _I, _I, _I, _P, _P, _P, _I, _I, _I, _F, _P], _I),
    "hx_tp_inbox_bytes": ([_I, _I, _I], _SZ),
    "hx_tp_inbox_init": ([_P, _I, _I, _I, _P], _I),
    "hx_tp_allreduce_push_residual_rmsnorm": ([_P, _P, ctypes.POINTER(ctypes.c_void_p), _I, _I, _I, _P, _P, _P, _I,
                                               _I, _I, _F, _P], _I),
    "hx_tp_inbox_bytes_ex": ([_I, _I, _I, _I], _SZ),
    "hx_tp_inbox_init_ex": ([_P, _I, _I, _I, _I, _P], _I),
    "hx_tp_allreduce_push_residual_rmsnorm_ex": ([_P, _P, ctypes.POINTER(ctypes.c_void_p), _I, _I, _I, _P, _P, _P,
                                                  _I, _I, _I, _F, _I, _P], _I),
    "hx_tp_allreduce_push_residual_rmsnorm_sk": ([_P, _P, _P, _I, ctypes.POINTER(ctypes.c_void_p), _I, _I, _I, _P,
                                                  _P, _P, _I, _I, _I, _F, _I, _P], _I),
    "hx_handoff_inbox_bytes": ([_SZ], _SZ),
    "hx_handoff_inbox_init": ([_P, _SZ, _P], _I),
    "hx_handoff_push": ([_P, ctypes.POINTER(ctypes.c_void_p), _I, _SZ, _SZ, _P, _P], _I),
    "hx_handoff_pull": ([_P, _P, _SZ, _SZ, _P, _P], _I),
    "hx_handoff_push_credit": ([_P, _P, _SZ, _SZ, _P, _P], _I),
    "hx_handoff_pull_credit": ([_P, _P, _SZ, _SZ, _P, _P], _I),
    "hx_prefill_vt": ([_P, _P, _I, _I, _I, _I, _I, _P], _I),
    "hx_attn_prefill_tc": ([_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P], _I),
    "hx_splitk_swiglu": ([_P, _I, _P, _I, _I, _I, _P, _I, _P], _I),
    "hx_swiglu": ([_P, _P, _I, _I, _I, _P], _I),
    "hx_rope_kv_append": ([_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _F, _P], _I),
    "hx_attn_decode_paged": ([_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _SZ, _P], _I),
    "hx_attn_decode_workspace": ([_I, _I, _I, _I, _I], _SZ),
    "hx_attn_decode_rope_append": ([_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _F, _P, _SZ, _P], _I),
    "hx_attn_prefill": ([_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P], _I),
    "hx_attn_decode_rope_append_sk": ([_P, _I, _P, _I, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _P, _SZ,
                                       _P], _I),
    "hx_advance": ([_P, _I, _I, _P], _I),
    "hx_argmax_partial": ([_P, _P, _I, _I, _I, _I, _P], _I),
    "hx_argmax_finalize": ([_P, _P, _P, _P, _I, _I, _I, _P], _I),
    "hx_kv_bytes": ([_I, _I, _I, _I, _I, _I], _SZ),
}

EXPORTED = tuple(_SIGS)


class HxError(RuntimeError):
    pass


def load(path: Path | str | None = None):
    """Load the C-ABI library; raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("HX_LIB", LIB_PATH))
    if not p.exists():
        raise HxError(f"{p} not built -- run `python -m paper_2311_11514_b200.build` "
                      "(there is no CPU fallback for the data path)")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = load().hx_error_string(rc).decode()
        raise HxError(f"{what} failed: {msg} (code {rc})")


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return HX_F32
    if dt == torch.bfloat16:
        return HX_BF16
    raise HxError(f"unsupported dtype {dt}")


def _p(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(load().hx_launch_count())


def embed(ids, table, x, n_tok):
    _check(load().hx_embed(_p(ids), _p(table), dtype_code(table.dtype), _p(x), n_tok,
                           table.shape[1], table.shape[0], _stream()), "hx_embed")


def rmsnorm(x, gain, out, n_tok, eps, ldx=None):
    H = gain.shape[0]
    _check(load().hx_rmsnorm(_p(x), ldx or H, _p(gain), _p(out), dtype_code(out.dtype), n_tok, H,
                             eps, _stream()), "hx_rmsnorm")


def residual_add_rmsnorm(x, delta, gain, out, n_tok, eps):
    H = x.shape[-1]
    _check(load().hx_residual_add_rmsnorm(_p(x), _p(delta), _p(gain), _p(out),
                                          dtype_code(out.dtype) if out is not None else HX_F32,
                                          n_tok, H, eps, _stream()), "hx_residual_add_rmsnorm")


def linear_workspace(dtype, n_tok, n_out, k_dim) -> int:
    return int(load().hx_linear_workspace(dtype_code(dtype), n_tok, n_out, k_dim))


HX_LINEAR_ACCUMULATE, HX_LINEAR_PACKED = 1, 2


class PackedWeight:
    """A bf16 [n_out, k] weight held in the hx_pack_weight tile layout
    ([n/128][k/64][128][64], zero padded): each 16 KB tile the decode GEMM
    streams is one contiguous HBM range."""

    def __init__(self, w: torch.Tensor):
        if w.dtype != torch.bfloat16 or w.dim() != 2:
            raise HxError("PackedWeight needs a 2-D bf16 tensor")
        self.shape = tuple(w.shape)
        self.dtype = w.dtype
        n, k = self.shape
        self.data = torch.empty(int(load().hx_packed_weight_elems(n, k)), dtype=w.dtype, device=w.device)
        _check(load().hx_pack_weight(_p(w.contiguous()), _p(self.data), n, k, _stream()), "hx_pack_weight")

    def numel(self):
        return self.shape[0] * self.shape[1]

    def element_size(self):
        return 2


def set_pdl(enabled: bool):
    load().hx_set_pdl(1 if enabled else 0)


HX_LINEAR_DEFER_REDUCE = 4


def splitk_residual_rmsnorm(x, y, workspace, n_tok, k_dim, gain, out, eps):
    """Consumer of a deferred decode GEMM (linear(..., defer_reduce=True)) into y:
    x += y (split tiles summed from the workspace slots); out = rmsnorm(x)*gain."""
    n_out = x.shape[-1]
    _check(load().hx_splitk_residual_rmsnorm(_p(x), _p(y), y.shape[-1], _p(workspace), n_tok, n_out, k_dim,
                                             _p(gain), _p(out), dtype_code(out.dtype) if out is not None else HX_F32,
                                             eps, _stream()), "hx_splitk_residual_rmsnorm")


HX_LINEAR_L2_PREFETCH = 8


def linear(w, x, y, n_tok, workspace=None, accumulate=False, defer_reduce=False, l2_prefetch=False):
    """y[:n_tok, :n_out] (+)= x[:n_tok] @ w.T ; w [n_out, K] row-major tensor
    or a PackedWeight. defer_reduce: see splitk_residual_rmsnorm. l2_prefetch:
    stream more weight tiles into L2 before the PDL wait (after an all-reduce)."""
    n_out, k = w.shape
    flags = (HX_LINEAR_ACCUMULATE if accumulate else 0) | (HX_LINEAR_DEFER_REDUCE if defer_reduce else 0) | \
        (HX_LINEAR_L2_PREFETCH if l2_prefetch else 0)
    if isinstance(w, PackedWeight):
        flags |= HX_LINEAR_PACKED
        wp = w.data
    else:
        wp = w
    ws = workspace
    _check(load().hx_linear(_p(wp), _p(x), _p(y), dtype_code(w.dtype), dtype_code(y.dtype), n_tok,
                            n_out, k, y.shape[-1], flags, _p(ws),
                            0 if ws is None else ws.numel() * ws.element_size(), _stream()),
           "hx_linear")


def splitk_swiglu(y, workspace, n_tok, k_dim, out):
    """SwiGLU consuming a deferred gate/up GEMM (linear(..., defer_reduce=True) into fp32 y)."""
    inter = out.shape[-1]
    _check(load().hx_splitk_swiglu(_p(y), y.shape[-1], _p(workspace), n_tok, inter, k_dim, _p(out), out.shape[-1],
                                   _stream()), "hx_splitk_swiglu")


def swiglu(gu, out, n_tok):
    _check(load().hx_swiglu(_p(gu), _p(out), dtype_code(gu.dtype), n_tok, out.shape[-1], _stream()),
           "hx_swiglu")


def rope_kv_append(qkv, q_out, k_cache, v_cache, block_table, seq_lens, n_tok, prefill_len,
                   hq, hkv, hd, theta):
    page = k_cache.shape[2]
    _check(load().hx_rope_kv_append(_p(qkv), _p(q_out), _p(k_cache), _p(v_cache), _p(block_table),
                                    _p(seq_lens), dtype_code(qkv.dtype), n_tok, prefill_len, hq, hkv,
                                    hd, page, block_table.shape[1], theta, _stream()),
           "hx_rope_kv_append")


def attn_decode_workspace(batch, hq, hkv, hd, max_ctx) -> int:
    return int(load().hx_attn_decode_workspace(batch, hq, hkv, hd, max_ctx))


def attn_decode(q, k_cache, v_cache, block_table, seq_lens, o, batch, hq, hkv, hd, max_ctx,
                workspace=None):
    ws = workspace
    _check(load().hx_attn_decode_paged(_p(q), _p(k_cache), _p(v_cache), _p(block_table), _p(seq_lens),
                                       _p(o), dtype_code(q.dtype), batch, hq, hkv, hd, k_cache.shape[2],
                                       block_table.shape[1], max_ctx, _p(ws),
                                       0 if ws is None else ws.numel() * ws.element_size(), _stream()),
           "hx_attn_decode_paged")


def decode_rope_fusable(dtype, hd, page, hq, hkv) -> bool:
    """Whether hx_attn_decode_rope_append takes this shape (bf16, hd 128,
    page 64, GQA group in {1, 2, 4, 8, 16}; HX_ATTN_TMA not 0)."""
    import os
    return (dtype == torch.bfloat16 and hd == 128 and page == 64 and hq % hkv == 0
            and hq // hkv in (1, 2, 4, 8, 16) and os.environ.get("HX_ATTN_TMA", "1") != "0")


def attn_decode_rope_append(qkv, k_cache, v_cache, block_table, seq_lens, o, batch, hq, hkv, hd, max_ctx,
                            theta, workspace=None):
    """RoPE + KV append of the new token fused into decode attention
    (hx_attn_decode_rope_append); q is read un-rotated from the qkv rows."""
    ws = workspace
    _check(load().hx_attn_decode_rope_append(_p(qkv), _p(k_cache), _p(v_cache), _p(block_table), _p(seq_lens),
                                             _p(o), dtype_code(qkv.dtype), batch, hq, hkv, hd, k_cache.shape[2],
                                             block_table.shape[1], max_ctx, theta, _p(ws),
                                             0 if ws is None else ws.numel() * ws.element_size(), _stream()),
           "hx_attn_decode_rope_append")


def attn_decode_rope_append_sk(qkv32, gemm_ws, k_dim, k_cache, v_cache, block_table, seq_lens, o, batch, hq, hkv,
                               hd, max_ctx, theta, workspace=None):
    """hx_attn_decode_rope_append after a deferred QKV GEMM (linear(..., defer_reduce=True)
    into fp32 qkv32 with workspace gemm_ws): the split tiles are reduced in the prologue."""
    ws = workspace
    _check(load().hx_attn_decode_rope_append_sk(_p(qkv32), qkv32.shape[-1], _p(gemm_ws), k_dim, _p(k_cache),
                                                _p(v_cache), _p(block_table), _p(seq_lens), _p(o), batch, hq, hkv,
                                                hd, k_cache.shape[2], block_table.shape[1], max_ctx, theta, _p(ws),
                                                0 if ws is None else ws.numel() * ws.element_size(), _stream()),
           "hx_attn_decode_rope_append_sk")


def attn_prefill(q, k_cache, v_cache, block_table, seq_lens, o, batch, s, hq, hkv, hd):
    _check(load().hx_attn_prefill(_p(q), _p(k_cache), _p(v_cache), _p(block_table), _p(seq_lens), _p(o),
                                  dtype_code(q.dtype), batch, s, hq, hkv, hd, k_cache.shape[2],
                                  block_table.shape[1], _stream()), "hx_attn_prefill")


def prefill_vt(qkv, vt, batch, s, hq, hkv, hd):
    """V of the prompt, transposed per (sequence, kv head), for attn_prefill_tc."""
    _check(load().hx_prefill_vt(_p(qkv), _p(vt), batch, s, hq, hkv, hd, _stream()), "hx_prefill_vt")


def attn_prefill_tc(q, k_cache, vt, block_table, o, batch, s, hq, hkv, hd):
    """Causal prefill attention on tcgen05 (hd 128, s % 128 == 0, page 64, no earlier context)."""
    _check(load().hx_attn_prefill_tc(_p(q), _p(k_cache), _p(vt), _p(block_table), _p(o), batch, s, hq, hkv, hd,
                                     k_cache.shape[2], block_table.shape[1], _stream()), "hx_attn_prefill_tc")


def advance(seq_lens, batch, n):
    _check(load().hx_advance(_p(seq_lens), batch, n, _stream()), "hx_advance")


def argmax_partial(logits, keys, n_tok, n_cols, vocab_offset):
    _check(load().hx_argmax_partial(_p(logits), _p(keys), n_tok, n_cols, logits.shape[-1], vocab_offset,
                                    _stream()), "hx_argmax_partial")


def argmax_finalize(keys, ids, history, step, n_tok, bump=True):
    s_out = history.shape[1] if history is not None else 0
    _check(load().hx_argmax_finalize(_p(keys), _p(ids), _p(history), _p(step), s_out, n_tok,
                                     1 if bump else 0, _stream()), "hx_argmax_finalize")


def kv_bytes(dtype, layers, num_blocks, hkv_rank, page, hd) -> int:
    return int(load().hx_kv_bytes(dtype_code(dtype), layers, num_blocks, hkv_rank, page, hd))


# ---------------------------------------------------------------- NVLink TP all-reduce
def _alloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    _check(load().hx_ipc_alloc(ctypes.byref(p), nbytes), "hx_ipc_alloc")
    return p.value


#: CTAs of the push all-reduce that fit on one B200 at once (4 per token row,
#: __launch_bounds__(256, 2): 2 per SM x 148 SMs). A single-GPU emulation runs
#: every rank's kernel concurrently, so tp * n_tok * 4 must not exceed it.
PEER_AR_CORESIDENT = 2 * 148


class PeerAllReduce:
    """Per-rank state of the fused NVLink all-reduce + residual + RMSNorm of a
    TP>1 decode step. Buffers are cudaIpc-exportable allocations mapped on every
    rank of the TP group (handles exchanged once over ``group``):

    * ``mode='push'`` (default, hx_tp_allreduce_push_residual_rmsnorm): each
      rank stores its partial into every peer's sentinel-armed inbox and polls
      its own -- one one-way NVLink trip per call;
    * ``mode='pull'`` (hx_tp_allreduce_residual_rmsnorm): epoch flags, then
      peer loads of every rank's partial slot.
    Both sum in rank order and give identical bits.

    ``PeerAllReduce.local_group`` builds all TP ranks of a group inside one
    process on one device (peer pointers are plain same-device pointers): the
    same kernels, each emulated rank launching on its own stream, so the
    protocol runs with real concurrency on a single GPU."""

    def __init__(self, rank: int, tp: int, max_tok: int, hidden: int, sites: int, group, dist, mode: str | None = None,
                 payload: str = "fp32"):
        self._setup(rank, tp, max_tok, hidden, sites, mode, payload)
        ptrs = self._alloc_own()
        handles = {}
        lib = load()
        for name, p in ptrs.items():
            h = ctypes.create_string_buffer(64)
            _check(lib.hx_ipc_handle(p, h), "hx_ipc_handle")
            handles[name] = h.raw
        gathered = [None] * tp
        dist.all_gather_object(gathered, handles, group=group)
        peer = {name: [0] * tp for name in ptrs}
        for r in range(tp):
            for name in ptrs:
                if r == rank:
                    peer[name][r] = ptrs[name]
                elif name in ("flags", "inbox") or self.mode == "pull":
                    q = ctypes.c_void_p()
                    _check(lib.hx_ipc_open(gathered[r][name], ctypes.byref(q)), "hx_ipc_open")
                    peer[name][r] = q.value
                    self._opened.append(q.value)
        self._finish(peer)
        self._group, self._dist = group, dist
        dist.barrier(group=group)

    @classmethod
    def local_group(cls, tp: int, max_tok: int, hidden: int, sites: int, mode: str | None = None,
                    payload: str = "fp32"):
        """All ``tp`` ranks of one group in this process (single-GPU emulation)."""
        objs = [cls.__new__(cls) for _ in range(tp)]
        own = []
        for r, o in enumerate(objs):
            o._setup(r, tp, max_tok, hidden, sites, mode, payload)
            o._group = o._dist = None
            own.append(o._alloc_own())
        for r, o in enumerate(objs):
            o._finish({name: [own[q][name] for q in range(tp)] for name in own[r]})
        torch.cuda.synchronize()
        return objs

    def _setup(self, rank, tp, max_tok, hidden, sites, mode, payload="fp32"):
        self.mode = mode or os.environ.get("HX_AR_MODE", "push")
        if self.mode not in ("push", "pull"):
            raise HxError(f"unknown all-reduce mode {self.mode!r}")
        if payload not in ("fp32", "bf16") or (payload == "bf16" and self.mode != "push"):
            raise HxError(f"all-reduce payload {payload!r} (mode {self.mode}) not supported")
        self.payload = payload
        self._pl = HX_BF16 if payload == "bf16" else HX_F32
        self.rank, self.tp, self.max_tok, self.hidden, self.sites = rank, tp, max_tok, hidden, sites
        self._own, self._opened = [], []

    def _alloc_own(self) -> dict:
        lib = load()
        slot_bytes = self.max_tok * self.hidden * 4
        bufs = [("slot0", slot_bytes), ("slot1", slot_bytes)]
        if self.mode == "pull":
            bufs.append(("flags", self.sites * self.max_tok * 8 * 4))
        else:
            bufs.append(("inbox", int(lib.hx_tp_inbox_bytes_ex(self.tp, self.max_tok, self.hidden, self._pl))))
        ptrs = {}
        for name, nbytes in bufs:
            ptrs[name] = _alloc(nbytes)
            self._own.append(ptrs[name])
        if self.mode == "push":
            _check(lib.hx_tp_inbox_init_ex(ptrs["inbox"], self.tp, self.max_tok, self.hidden, self._pl, None),
                   "hx_tp_inbox_init_ex")
            torch.cuda.synchronize()
        return ptrs

    def _finish(self, peer: dict):
        self.peer = peer
        # pull mode: [epoch, done] per call site; push mode: one call counter per CTA (4 per token row)
        self.site_state = torch.zeros(max(2 * self.sites, 4 * self.max_tok), dtype=torch.int32, device="cuda")
        self._arr = {name: (ctypes.c_void_p * self.tp)(*peer[name]) for name in peer}

    def slot(self, site: int) -> torch.Tensor:
        """This rank's partial slot for a call site, as a [max_tok, hidden] fp32 view."""
        ptr = self.peer[f"slot{site % 2}"][self.rank]
        return _tensor_at(ptr, (self.max_tok, self.hidden))

    def allreduce_residual_rmsnorm(self, x, site, gain, out, n_tok, eps, gemm_ws=None, k_dim=0):
        """gemm_ws / k_dim: the slot was written by a deferred GEMM
        (linear(..., defer_reduce=True) with that workspace); push mode only."""
        lib = load()
        if gemm_ws is not None:
            if self.mode != "push":
                raise ValueError("deferred split-K all-reduce needs mode='push'")
            _check(lib.hx_tp_allreduce_push_residual_rmsnorm_sk(
                _p(x), self.peer[f"slot{site % 2}"][self.rank], _p(gemm_ws), k_dim, self._arr["inbox"], self.rank,
                self.tp, self.max_tok, _p(self.site_state), _p(gain), _p(out),
                dtype_code(out.dtype) if out is not None else HX_F32, n_tok, self.hidden, eps, self._pl, _stream()),
                "hx_tp_allreduce_push_residual_rmsnorm_sk")
            return
        if self.mode == "push":
            _check(lib.hx_tp_allreduce_push_residual_rmsnorm_ex(
                _p(x), self.peer[f"slot{site % 2}"][self.rank], self._arr["inbox"], self.rank, self.tp, self.max_tok,
                _p(self.site_state), _p(gain), _p(out), dtype_code(out.dtype) if out is not None else HX_F32,
                n_tok, self.hidden, eps, self._pl, _stream()), "hx_tp_allreduce_push_residual_rmsnorm_ex")
            return
        _check(lib.hx_tp_allreduce_residual_rmsnorm(
            _p(x), self._arr[f"slot{site % 2}"], self._arr["flags"], self.rank, self.tp, site, self.max_tok,
            _p(self.site_state), _p(gain), _p(out), dtype_code(out.dtype) if out is not None else HX_F32,
            n_tok, self.hidden, eps, _stream()), "hx_tp_allreduce_residual_rmsnorm")

    def close(self):
        """Unmap the peers' buffers and free this rank's own (after a group
        barrier, so no peer still maps them). Idempotent."""
        if not getattr(self, "_own", None) and not getattr(self, "_opened", None):
            return
        lib = load()
        torch.cuda.synchronize()
        for q in self._opened:
            lib.hx_ipc_close(q)
        self._opened = []
        if self._dist is not None:
            self._dist.barrier(group=self._group)
        for p in self._own:
            lib.hx_ipc_free(p)
        self._own = []


# ---------------------------------------------------------------- NVLink P2P stage hand-off
class P2PLink:
    """One directed decode hand-off link (sender device -> receiver device) of
    the inter-stage reshard (hx_handoff_push / hx_handoff_pull): the receiver
    owns a sentinel-armed inbox in cudaIpc memory, the sender maps it. Built
    collectively by the two ranks over their 2-rank ``group``.
    ``P2PLink.local`` builds both ends in one process (single-GPU emulation)."""

    def __init__(self, src: int, dst: int, me: int, max_words: int, group, dist):
        lib = load()
        self._init_state(src, dst, me, max_words)
        handle = None
        if me == dst:
            self._alloc_inbox()
            h = ctypes.create_string_buffer(64)
            _check(lib.hx_ipc_handle(self._own, h), "hx_ipc_handle")
            handle = h.raw
        got = [None, None]
        dist.all_gather_object(got, handle, group=group)
        if me == src:
            q = ctypes.c_void_p()
            _check(lib.hx_ipc_open(next(h for h in got if h is not None), ctypes.byref(q)), "hx_ipc_open")
            self._peer = q.value
            self._opened = True
        self._group, self._dist = group, dist
        dist.barrier(group=group)

    @classmethod
    def local(cls, src: int, dst: int, max_words: int):
        o = cls.__new__(cls)
        o._init_state(src, dst, None, max_words)
        o._alloc_inbox()
        o._peer = o._own
        o.recv_state = torch.zeros(2, dtype=torch.int32, device="cuda")   # each end keeps its own counter
        o._group = o._dist = None
        return o

    def _init_state(self, src, dst, me, max_words):
        self.src, self.dst, self.me = src, dst, me
        self.max_words = (max_words + 3) // 4 * 4
        self.state = torch.zeros(2, dtype=torch.int32, device="cuda")
        self.recv_state = self.state
        self._own = self._peer = None
        self._opened = False

    def _alloc_inbox(self):
        lib = load()
        self._own = _alloc(int(lib.hx_handoff_inbox_bytes(self.max_words)))
        _check(lib.hx_handoff_inbox_init(self._own, self.max_words, None), "hx_handoff_inbox_init")
        torch.cuda.synchronize()

    def push(self, t: torch.Tensor):
        """Sender: store ``t`` (contiguous, 32-bit words) into the receiver's inbox."""
        arr = (ctypes.c_void_p * 1)(self._peer)
        _check(load().hx_handoff_push(_p(t), arr, 1, t.numel() * t.element_size() // 4, self.max_words,
                                      _p(self.state), _stream()), "hx_handoff_push")

    def pull(self, t: torch.Tensor):
        """Receiver: wait for this hand-off's data and copy it into ``t``."""
        _check(load().hx_handoff_pull(_p(t), self._own, t.numel() * t.element_size() // 4, self.max_words,
                                      _p(self.recv_state), _stream()), "hx_handoff_pull")

    def push_credit(self, t: torch.Tensor):
        """Sender, flow-controlled stream (prefill micro-batches): wait until the
        target buffer was drained, then store ``t`` into it."""
        _check(load().hx_handoff_push_credit(_p(t), self._peer, t.numel() * t.element_size() // 4, self.max_words,
                                             _p(self.state), _stream()), "hx_handoff_push_credit")

    def pull_credit(self, t: torch.Tensor):
        """Receiver, flow-controlled stream: copy the next hand-off into ``t``,
        re-arm its buffer and hand the buffer back to the sender."""
        _check(load().hx_handoff_pull_credit(_p(t), self._own, t.numel() * t.element_size() // 4, self.max_words,
                                             _p(self.recv_state), _stream()), "hx_handoff_pull_credit")

    def close(self):
        lib = load()
        torch.cuda.synchronize()
        if self._opened:
            lib.hx_ipc_close(self._peer)
            self._opened = False
        if self._dist is not None:
            self._dist.barrier(group=self._group)
        if self._own is not None:
            lib.hx_ipc_free(self._own)
            self._own = None


def _tensor_at(ptr: int, shape) -> torch.Tensor:
    """A torch view of raw device memory (owned elsewhere) via __cuda_array_interface__."""
    class _Holder:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Holder(), device="cuda")
