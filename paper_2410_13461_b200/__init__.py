"""B200-native PMPD hot path (arXiv 2410.13461): nested bit-plane weights in HBM, a decode GEMV
that reads only the active planes, device-side precision schedulers.

Mirrors the reference package ``pmpd`` (pkg/src/pmpd/__init__.py:9-25) for the names on the
hot path.  Compute runs in the CUDA library ``lib/libpmpd_b200.so``; there is no CPU fallback.
"""
from .errors import ConfigError, ContractViolation, FormatError, InputError, PmpdError  # noqa: F401

__version__ = "0.1.0"
