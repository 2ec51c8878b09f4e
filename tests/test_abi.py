"""C ABI surface: libmfgpu.so loads on a CPU-only host and exports every
function include/mfgpu.h declares; without a device the context creation
fails loudly (no CPU fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "mfgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(mf_[a-z_0-9]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("mf_decimate", "mf_pool", "mf_unpool", "mf_decimation_copy", "mf_context_create"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2103_15076_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_has_sm100a_code():
    import subprocess

    from paper_2103_15076_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_round_targets_via_abi():
    from oracle import oracle as O

    import paper_2103_15076_b200 as mfg

    for n, t, r in [(115114, 41449, "auto"), (1000, 130, "auto"), (400, 100, 2), (10242, 3585, "auto"),
                    (5, 5, "auto"), (999, 3, 5), (7, 2, 1), (10004569, 5002285, "auto")]:
        assert mfg.round_targets(n, t, r) == O.round_targets(n, t, r)


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import numpy as np

    import paper_2103_15076_b200 as mfg

    mesh = mfg.TriMesh(np.eye(3), [[0, 1, 2]])
    with pytest.raises(mfg.NativeError):
        mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=2))
