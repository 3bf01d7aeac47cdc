"""Seeded sub-streams restated from reference ``pkg/src/pmpd/util.py:12-20`` (oracle side)."""
from __future__ import annotations

import hashlib

import numpy as np


def named_rng(seed: int, label: str) -> np.random.Generator:
    """``default_rng([seed mod 2^64, first 8 sha256 bytes of label, little-endian])``."""
    digest = hashlib.sha256(label.encode("utf-8")).digest()
    return np.random.default_rng([int(seed) % (1 << 64), int.from_bytes(digest[:8], "little")])
