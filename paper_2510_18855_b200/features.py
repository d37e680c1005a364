"""Hashed feature rows of the reference's toy policy, restated for packing.

The reference's "lm_head" is a 4-hot x W contraction: the logits of a position are
W[f0] + W[f1] + W[f2] + W[f3] (policy.py:279-289) over four hashed feature rows of
the recent token window (policy.py:249-260). That is exactly H.W with H the
multi-hot count vector of those rows, so the drop-in packs H densely and runs the
same dense kernels as the Ling-shaped lm_head (SURVEY.md load-bearing fact 2).

The hash is restated (not imported) so the drop-in needs only the reference's data
objects, not its code: splitmix64 / _mix follow policy.py:67-81, the row functions
policy.py:229-260, and the per-rollout window walk objective.py:162-169.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _splitmix64(x: int) -> int:  # policy.py:67-73
    x = (x + _GOLDEN) & _MASK64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _MASK64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def _mix(*values: int) -> int:  # policy.py:76-81
    h = 0x8A5CD789635D2DFF
    for v in values:
        h = _splitmix64(h ^ (v & _MASK64))
    return h


@lru_cache(maxsize=262144)
def feature_rows(prompt_id: int, prev: int, last: int, n_features: int) -> tuple[int, int, int, int]:
    """(bias, unigram, bigram, bigram_b) rows, policy.py:229-260."""
    return (
        _mix(1) % n_features,
        _mix(3, prompt_id, last) % n_features,
        _mix(4, prompt_id, prev, last) % n_features,
        _mix(5, prompt_id, prev, last) % n_features,
    )


def rollout_feats(prompt_id: int, token_ids, n_features: int) -> np.ndarray:
    """(T, 4) feature rows for every position of a rollout (objective.py:162-169)."""
    feats = np.empty((len(token_ids), 4), dtype=np.int64)
    prev, last = -1, -1
    for t, tok in enumerate(token_ids):
        feats[t] = feature_rows(prompt_id, prev, last, n_features)
        prev, last = last, int(tok)
    return feats


def multihot_device(feats, n_features: int, dtype):
    """`multihot` built on the GPU from the [N, 4] feature ids (a device int64 tensor): the
    counts are small integers, so the float scatter-add is exact in any order."""
    import torch

    h = torch.zeros((feats.shape[0], n_features), dtype=torch.float32, device=feats.device)
    h.scatter_add_(1, feats, torch.ones(feats.shape, dtype=torch.float32, device=feats.device))
    return h.to(dtype)


def multihot(feats: np.ndarray, n_features: int, dtype=np.float64) -> np.ndarray:
    """Dense H[t, f] = multiplicity of row f among the 4 feature rows of position t."""
    h = np.zeros((feats.shape[0], n_features), dtype=dtype)
    rows = np.repeat(np.arange(feats.shape[0]), feats.shape[1])
    np.add.at(h, (rows, feats.reshape(-1)), 1)
    return h
