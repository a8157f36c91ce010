"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/tnrd.h declares, and rejects bad arguments without a device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tnrd.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"TNRD_API[^;(]*?\b(tnrd_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ("tnrd_create", "tnrd_set_stage_params", "tnrd_denoise", "tnrd_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_1510_02930_b200 as P
    lib = P.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tnrd_\w+)", out))
    assert set(_declared()) <= exported
    # binding names match the ABI
    for name in _declared():
        assert hasattr(P, name), name


def test_abi_version_and_status_strings():
    import paper_1510_02930_b200 as P
    assert P.tnrd_abi_version() == 1
    assert P.lib().tnrd_status_string(1) == b"TNRD_EINVAL"


def test_create_rejects_bad_shapes_before_touching_the_device():
    import paper_1510_02930_b200 as P
    # ksize: even or < 3 is invalid (S l.31-32); odd sizes up to 11 are built (P l.458-469
    # studies 3..9), larger odd sizes are EUNSUPPORTED
    for args, status in [((0, 8, 3, 63), 1), ((2, 8, 4, 63), 1), ((2, 8, 10, 63), 1), ((2, 8, 1, 63), 1),
                         ((2, 0, 3, 63), 1), ((2, 8, 13, 63), 6), ((2, 8, 3, 0), 1)]:
        with pytest.raises(P.TNRDError) as ei:
            P.tnrd_create(*args)
        assert ei.value.status == status, (args, str(ei.value))
    with pytest.raises(P.TNRDError) as ei:
        P.tnrd_create(2, 8, 3, 63, phi_mode=7)  # unknown phi mode (0 exact, 1 table)
    assert ei.value.status == 1


def test_null_handle_calls_fail_cleanly():
    import paper_1510_02930_b200 as P
    lib = P.lib()
    assert lib.tnrd_denoise(None, None, None, 1, 8, 8, 8, None, None) == 1
    assert lib.tnrd_destroy(None) == 0
    assert lib.tnrd_launch_count(None) == 0
