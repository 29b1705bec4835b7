"""Synthetic token batches for the engine (SURVEY.md section 8(d) "Synthetic inputs").

int64 ids ``randint(0, vocab, (steps, D, B, b, s+1))`` from one CPU generator seeded
with the reference's DEFAULT_FUZZ_SEED (`pkg/src/zeroppsim/cli.py:26`); input =
``[..., :-1]``, labels = ``[..., 1:]``; ZeRO rank z takes ``[:, z]``.  The test oracle
draws the same tensor independently (tests compare the two).
"""

from __future__ import annotations

import torch

SEED = 20240817


def synthetic_tokens(steps: int, D: int, B: int, b: int, s: int, vocab: int, seed: int = SEED) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (steps, D, B, b, s + 1), generator=g)


def rank_batch(tokens_step: torch.Tensor, z: int) -> tuple[torch.Tensor, torch.Tensor]:
    """tokens_step [D, B, b, s+1] -> (ids, labels) int64 [B, b*s] of ZeRO rank z (CPU)."""
    t = tokens_step[z]
    B = t.shape[0]
    return t[:, :, :-1].reshape(B, -1).contiguous(), t[:, :, 1:].reshape(B, -1).contiguous()
