"""CPU-side checks of the C-ABI boundary: the library loads and exports every header symbol,
and the descriptor/validation logic (no kernel launches) behaves like the reference."""
import ctypes
import os
import re

import pytest

from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.errors import ConfigError, ContractViolation, FormatError, InputError, PmpdError

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pmpd_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(pmpd_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _capi.SIGNATURES, f"{s} has no ctypes signature"


def test_error_hierarchy_matches_reference():
    assert issubclass(FormatError, InputError) and issubclass(InputError, PmpdError)
    assert issubclass(ContractViolation, PmpdError) and issubclass(ConfigError, PmpdError)


def test_describe_geometry_and_errors():
    d = _capi.describe(4096, 11008, 64, 4, _capi.LAYOUT_KN)
    assert (d.n, d.k, d.n_tiles, d.k_tiles, d.groups) == (11008, 4096, 172, 64, 172)
    assert d.plane_bytes == 172 * 64 * 512 and d.scale_bytes == d.plane_bytes
    # 1 bit/weight of f32 scales at g=64 and p/8 bytes per plane: perf.py:101 accounting
    assert d.plane_bytes * 8 == 4096 * 11008 and d.scale_bytes == 8 * 4096 * 11008 // 64
    d = _capi.describe(257, 64, 64, 4, _capi.LAYOUT_NK)
    assert (d.n, d.k, d.n_tiles, d.k_tiles) == (257, 64, 5, 1)
    d = _capi.describe(13, 21, 8, 3, _capi.LAYOUT_REF)
    assert d.plane_bytes >= (13 * 21 + 7) // 8 and d.scale_bytes == 2 * 13 * 3 * 4
    with pytest.raises(ConfigError):
        _capi.describe(4, 4, 64, 9, _capi.LAYOUT_REF)
    with pytest.raises(ConfigError):
        _capi.describe(4, 4, 0, 4, _capi.LAYOUT_REF)
    with pytest.raises(ConfigError):
        _capi.describe(64, 64, 32, 4, _capi.LAYOUT_KN)  # tiled layouts need g % 64 == 0
    with pytest.raises(ConfigError):
        _capi.describe(64, 64, 64, 5, _capi.LAYOUT_KN)  # and p_max <= 4
    with pytest.raises(InputError):
        _capi.describe(0, 4, 4, 4, _capi.LAYOUT_REF)


def test_gemv_validation_without_launch():
    d = _capi.describe(128, 128, 64, 4, _capi.LAYOUT_KN)
    out = ctypes.c_int64()
    with pytest.raises(InputError):
        _capi.call("pmpd_gemv_workspace_bytes", ctypes.byref(d), 9, ctypes.byref(out))
    _capi.call("pmpd_gemv_workspace_bytes", ctypes.byref(d), 1, ctypes.byref(out))
    assert out.value > 0
    r = _capi.describe(128, 128, 64, 4, _capi.LAYOUT_REF)
    with pytest.raises(ConfigError):
        _capi.call("pmpd_gemv_workspace_bytes", ctypes.byref(r), 1, ctypes.byref(out))


def _partition(nt, kt, G, delta=None):
    lib = _capi.lib()
    d = _capi.QTensorDesc()
    d.n_tiles, d.k_tiles = nt, kt
    b = (ctypes.c_int32 * (G + 1))()
    if delta is None:
        assert lib.pmpd_engine_partition_g(ctypes.byref(d), G, b) == 0
    else:
        dl = (ctypes.c_int32 * G)(*delta)
        assert lib.pmpd_engine_partition_w(ctypes.byref(d), G, dl, b) == 0
    return list(b)


@pytest.mark.parametrize("nt,kt", [(344, 64), (192, 64), (64, 172), (500, 64), (3, 7)])
def test_engine_partition_covers_every_tile(nt, kt):
    """Cost-balanced CTA ranges (host code): monotone, start at 0, end at the last tile; a
    zero budget reduction is the plain partition; slower CTAs get no more tiles than before."""
    G = 148
    b = _partition(nt, kt, G)
    assert b[0] == 0 and b[-1] == nt * kt and all(x <= y for x, y in zip(b, b[1:]))
    assert _partition(nt, kt, G, [0] * G) == b
    delta = [2 if c % 6 == 0 else 0 for c in range(G)]
    w = _partition(nt, kt, G, delta)
    assert w[0] == 0 and w[-1] == nt * kt and all(x <= y for x, y in zip(w, w[1:]))
    if nt * kt >= 4 * G:
        slow = [w[c + 1] - w[c] for c in range(G) if delta[c]]
        base = [b[c + 1] - b[c] for c in range(G) if delta[c]]
        assert sum(slow) < sum(base)
