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


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    """_splitmix64 over a uint64 array (numpy's uint64 arithmetic wraps mod 2^64, as the
    reference's `& _MASK64` does)."""
    x = x + np.uint64(_GOLDEN)
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _mix_np(prefix: tuple, *arrays: np.ndarray) -> np.ndarray:
    """_mix(*prefix, *arrays) per position: the scalar prefix is mixed once in Python, then each
    int64 array (two's complement = the reference's `v & _MASK64`) over all positions."""
    h0 = 0x8A5CD789635D2DFF
    for v in prefix:
        h0 = _splitmix64(h0 ^ (v & _MASK64))
    h = np.full(arrays[0].shape, h0, dtype=np.uint64)
    for v in arrays:
        h = _splitmix64_np(h ^ v.astype(np.uint64))
    return h


def rollout_feats(prompt_id: int, token_ids, n_features: int) -> np.ndarray:
    """(T, 4) feature rows for every position of a rollout (objective.py:162-169): position t
    hashes the window (prev, last) = (token t-2, token t-1), -1 before the start. Vectorised
    over the positions (feature_rows is the scalar form, policy.py:229-260)."""
    tok = np.asarray(token_ids, dtype=np.int64).reshape(-1)
    T = tok.size
    last = np.full(T, -1, dtype=np.int64)
    prev = np.full(T, -1, dtype=np.int64)
    last[1:] = tok[:-1]
    prev[2:] = tok[:-2]
    nf = np.uint64(n_features)
    feats = np.empty((T, 4), dtype=np.int64)
    with np.errstate(over="ignore"):
        feats[:, 0] = int(_mix(1) % n_features)
        feats[:, 1] = (_mix_np((3, prompt_id), last) % nf).astype(np.int64)
        feats[:, 2] = (_mix_np((4, prompt_id), prev, last) % nf).astype(np.int64)
        feats[:, 3] = (_mix_np((5, prompt_id), prev, last) % nf).astype(np.int64)
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
