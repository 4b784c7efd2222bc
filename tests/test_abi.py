"""CPU checks of the drop-in boundary: librwb.so builds for sm_100a, loads,
and exports exactly the symbols include/rwb.h declares, with matching struct
layouts.  No compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

import __graft_entry__ as entry
from paper_2509_26213_b200 import _native

HEADER = os.path.join(ROOT, "include", "rwb.h")


@pytest.fixture(scope="module")
def lib():
    entry.build()
    return _native.load_library()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(rwb_\w+)\(", text, re.M)))


def test_header_declares_the_bound_symbols():
    assert declared_functions() == sorted(_native.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.rwb_abi_version() == _native.ABI_VERSION


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_native.Geometry) == 8 + 3 * 8 * 3
    assert ctypes.sizeof(_native.SolveParams) == 24
    assert ctypes.sizeof(_native.SolveStats) == 7 * 8 + 16 + 8  # ..., int32 sweeps, float cg_ms, ..., int64


def test_workspace_size_query_needs_no_device(lib):
    from paper_2509_26213_b200 import device

    from paper_2509_26213_b200.config import RWConfig

    streaming = RWConfig(resident=False)
    n = device.workspace_bytes((64, 64, 64), (32, 32, 32), cfg=streaming)
    # 9 f32 brick-local arrays (36 B/voxel) plus small per-brick scalars
    assert 36 * 64**3 <= n < 36 * 64**3 + 64 * 1024
    # the brick-resident path iterates on the same brick-local system the streaming setup builds
    assert device.workspace_bytes((64, 64, 64), (32, 32, 32)) == n
    n2 = device.workspace_bytes((128, 128), (64, 64))
    assert 32 * 128**2 <= n2 < 32 * 128**2 + 64 * 1024
    assert device.workspace_bytes((64, 64, 64), (32, 32, 32), n_bricks=2, cfg=streaming) < n


def test_invalid_geometry_reports_error(lib):
    g = _native.Geometry()
    g.ndim = 4
    assert lib.rwb_solve_workspace_bytes(ctypes.byref(g), -1, 0) == 0
    assert lib.rwb_labels_u8(-1, None, None, None) == -1
    assert b"negative" in lib.rwb_last_error()


def test_sass_is_sm100(lib):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_device_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_26213_b200 import device

    with pytest.raises((_native.NativeUnavailable, ValueError)):
        device.lod_down(torch.zeros(4, 4))


def test_solve_flags_match_header():
    """Every RWB_SOLVE_* flag of the header has the same value in the Python binding."""
    text = open(HEADER).read()
    flags = dict(re.findall(r"#define RWB_SOLVE_(\w+)\s+(\d+)", text))
    assert {"NO_GRAPH", "STREAMING", "NO_COOP", "CLUSTER16", "SPLIT_Z", "SETUP2", "SETUP_ONLY", "NO_SETUP",
            "STATS_DEVICE"} <= set(flags)
    for name, value in flags.items():
        assert getattr(_native, f"SOLVE_{name}") == int(value), name
    values = [int(v) for v in flags.values()]
    assert len(set(values)) == len(values) and all(v & (v - 1) == 0 for v in values)  # distinct bits
