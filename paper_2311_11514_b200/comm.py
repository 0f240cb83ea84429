"""Collectives and stage hand-off for the executor.

* ``DistComm`` -- production: one process per GPU, ``torch.distributed``
  (NCCL over NVLink on the B200 box, gloo for CPU tests). One process group
  per TP stage carries the two per-layer all-reduces (PAPER.md:158-160,
  modelled by ``tp_comm_cost``, costs.py:123-147) and the vocab-parallel
  argmax; point-to-point send/recv carries the stage hand-off (the
  ``pp_comm_cost`` term, costs.py:150-165) and the token-id return.
* ``LocalComm`` -- all ranks of a pipeline emulated in one process (one GPU,
  or CPU): the all-reduce sums the emulated ranks' partials in rank order and
  writes the sum back to each; send/recv is a copy. Used by parity tests so
  asymmetric plans run on a single device with identical kernel sequences.
"""

from __future__ import annotations

import numpy as np
import torch


class LocalComm:
    kind = "local"
    rank = 0

    def __init__(self):
        self.mail = {}

    def setup(self, roles, local):
        pass

    def all_reduce_sum(self, tensors, group):
        acc = tensors[0]
        for t in tensors[1:]:
            acc.add_(t)
        for t in tensors[1:]:
            t.copy_(acc)

    def all_reduce_max(self, tensors, group):
        acc = tensors[0]
        for t in tensors[1:]:
            torch.maximum(acc, t, out=acc)
        for t in tensors[1:]:
            t.copy_(acc)

    def send(self, t, src, dst):
        self.mail[(src, dst)] = t

    def recv(self, t, src, dst):
        t.copy_(self.mail.pop((src, dst)))

    def broadcast_ids(self, hist, b, s_out, src, device):
        return hist.cpu().numpy().astype(np.int32)

    def gather_logits(self, e):
        raise RuntimeError("local comm holds every rank")


class DistComm:
    kind = "dist"

    def __init__(self):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("comm='dist' needs torch.distributed initialised (torchrun)")
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.groups = {}

    def setup(self, roles, local):
        # every process creates every stage group, in stage order (new_group is collective)
        for r in roles:
            key = r.tp_group
            if key in self.groups or len(key) == 1:
                continue
            self.groups[key] = self.dist.new_group(ranks=sorted(key))
        # one 2-rank communicator per hand-off link (stage j -> j+1, last -> first),
        # so point-to-point traffic never serialises behind other collectives
        self.pairs = {}
        for r in roles:
            for dst in tuple(r.send_to) + tuple(r.ids_send_to):
                key = (min(r.device, dst), max(r.device, dst))
                if key not in self.pairs and key[0] != key[1]:
                    self.pairs[key] = self.dist.new_group(ranks=list(key))

    def all_reduce_sum(self, tensors, group):
        for t in tensors:
            self.dist.all_reduce(t, group=self.groups[group])

    def all_reduce_max(self, tensors, group):
        for t in tensors:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.groups[group])

    def send(self, t, src, dst):
        self.dist.send(t.contiguous(), dst, group=self.pairs.get((min(src, dst), max(src, dst))))

    def recv(self, t, src, dst):
        self.dist.recv(t, src, group=self.pairs.get((min(src, dst), max(src, dst))))

    def broadcast_ids(self, hist, b, s_out, src, device):
        buf = hist.contiguous() if hist is not None and self.rank == src else \
            torch.zeros(b, s_out, dtype=torch.int32, device=device)
        self.dist.broadcast(buf, src=src)
        return buf.cpu().numpy().astype(np.int32)

    def gather_logits(self, e):
        g = self.groups.get(e.role.tp_group)
        if g is None:
            return e.logits.float().cpu().numpy()
        parts = [torch.zeros_like(e.logits) for _ in range(e.role.tp)]
        self.dist.all_gather(parts, e.logits, group=g)
        return torch.cat(parts, -1).cpu().numpy()


def make_comm(kind: str):
    if kind == "local":
        return LocalComm()
    if kind == "dist":
        return DistComm()
    if kind == "auto":
        import torch.distributed as dist
        return DistComm() if dist.is_initialized() and dist.get_world_size() > 1 else LocalComm()
    raise ValueError(f"unknown comm {kind!r}")
