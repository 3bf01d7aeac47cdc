"""Seeded randomness shared with the reference so synthetic inputs are byte-identical
(pkg/src/pmpd/util.py:12-20)."""
from __future__ import annotations

import hashlib

import numpy as np


def named_rng(seed: int, label: str) -> np.random.Generator:
    """One labelled stream: ``default_rng([seed mod 2^64, sha256(label)[:8] little-endian])``."""
    tag = int.from_bytes(hashlib.sha256(label.encode("utf-8")).digest()[:8], "little")
    return np.random.default_rng([int(seed) & 0xFFFFFFFFFFFFFFFF, tag])
