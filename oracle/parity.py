"""bf16-mode parity criteria -- TEST INFRASTRUCTURE ONLY
(imported by ``tests/`` and ``__graft_entry__.smoke()``, never by the product).

* Teacher-forced logits within ``TOL_EMULATED`` of max|logit| (per position)
  of the oracle that rounds activations to bf16 where the engine stores bf16,
  and within ``TOL_FP32ACT`` of the fp32-activation oracle on the same
  bf16-rounded weights.
* Top-1 agreement >= 99 % on the positions whose fp32-oracle top-2 margin
  exceeds ``MARGIN`` (relative to max|logit|, the error's normalisation) --
  a FIXED threshold, independent of the engine's observed error.
* Free-running greedy ids: identical up to each sequence's first divergence,
  which is reported; at that step the oracle's own top-2 margin must be a
  near-tie (below 2 x the engine's observed teacher-forced error), i.e. the
  flip is explained by bf16 rounding, not by a wrong token.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TOL_EMULATED = 2e-2
TOL_FP32ACT = 3e-2
MARGIN = 1e-2
MIN_AGREE = 0.99


def rel_err(lg, ref):
    """|lg - ref| / max|ref| per (step, sequence) row; lg, ref [s_out, b, V]."""
    return np.abs(lg - ref) / np.abs(ref).max(axis=-1, keepdims=True)


def top2_margin(lg):
    srt = np.sort(lg, axis=-1)
    return (srt[..., -1] - srt[..., -2]) / np.abs(lg).max(axis=-1)


def first_divergence(ids_a, ids_b):
    """Per sequence: the first step where the greedy ids differ (-1 = never). ids [b, s_out]."""
    out = []
    for a, b in zip(ids_a, ids_b):
        d = np.nonzero(a != b)[0]
        out.append(int(d[0]) if d.size else -1)
    return out


@dataclass
class Bf16Verdict:
    err_emulated: float
    err_fp32act: float
    agree: float
    checked_positions: int
    divergence: list           # per sequence first divergent free-running step (-1 = none)
    divergence_margins: list   # oracle margin at each divergence
    ok: bool
    why: str

    def line(self) -> str:
        return (f"bf16 teacher-forced max rel logit err {self.err_emulated:.2e} (emulated oracle), "
                f"{self.err_fp32act:.2e} (fp32-act oracle); top-1 agreement {self.agree:.3f} on "
                f"{self.checked_positions} positions with fp32 margin > {MARGIN}; free-running first "
                f"divergence per sequence {self.divergence}")


def bf16_verdict(forced_logits, forced_ids, emu_logits, fp32_logits, free_ids=None, oracle_ids=None,
                 tol_emulated=TOL_EMULATED, tol_fp32act=TOL_FP32ACT) -> Bf16Verdict:
    """forced_logits / emu_logits / fp32_logits [s_out, b, V] (the engine run
    teacher-forced on the oracle's tokens); forced_ids [b, s_out] (engine argmax);
    free_ids / oracle_ids [b, s_out] free-running greedy ids of engine / oracle."""
    e = rel_err(forced_logits, emu_logits)
    ef = rel_err(forced_logits, fp32_logits)
    margin_f = top2_margin(fp32_logits)                     # [s_out, b]
    ok_pos = margin_f > MARGIN
    oracle_top = np.argmax(emu_logits, axis=-1)             # [s_out, b]
    agree_mask = (np.asarray(forced_ids).T == oracle_top)[ok_pos]
    agree = float(agree_mask.mean()) if agree_mask.size else 1.0
    why = []
    if e.max() >= tol_emulated:
        why.append(f"emulated err {e.max():.2e} >= {tol_emulated}")
    if ef.max() >= tol_fp32act:
        why.append(f"fp32-act err {ef.max():.2e} >= {tol_fp32act}")
    if agree < MIN_AGREE:
        why.append(f"top-1 agreement {agree:.3f} < {MIN_AGREE}")
    div, div_m = [], []
    if free_ids is not None and oracle_ids is not None:
        div = first_divergence(np.asarray(free_ids), np.asarray(oracle_ids))
        margin_e = top2_margin(emu_logits)
        for i, t in enumerate(div):
            if t < 0:
                div_m.append(None)
                continue
            m = float(margin_e[t, i])
            div_m.append(m)
            if m > 2 * e.max():
                why.append(f"sequence {i} diverges at step {t} with oracle margin {m:.2e} "
                           f"> 2 x err {e.max():.2e} (not a near-tie)")
    return Bf16Verdict(float(e.max()), float(ef.max()), agree, int(ok_pos.sum()), div, div_m, not why,
                       "; ".join(why))
