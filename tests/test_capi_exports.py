"""CPU-only: the C-ABI library loads and exports every symbol include/exflow_c.h
declares (no compute calls without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "exflow_c.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(exf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2401_08383_b200 import _capi
    lib = _capi.load()
    declared = _declared_symbols()
    assert len(declared) >= 9
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding covers the whole header
    assert set(declared) <= set(_capi.SIGNATURES), set(declared) - set(_capi.SIGNATURES)


def test_version_and_device_probe_do_not_need_a_gpu():
    from paper_2401_08383_b200 import _capi
    lib = _capi.load()
    assert lib.exf_version() >= 100
    assert lib.exf_device_ok() in (0, 1)


def test_invalid_arguments_raise_reference_errors_without_gpu():
    # validation happens before any device work (trace.cpp:193-196 messages)
    import numpy as np
    from paper_2401_08383_b200 import affinity, _capi
    with pytest.raises(_capi.ExflowInvalidArgument, match="gap 2 out of range"):
        affinity.count_transitions(np.array([[0, 1]], np.int32), 2, 2)
    with pytest.raises(_capi.ExflowInvalidArgument, match="expert id out of range"):
        affinity.count_transitions(np.array([[0, 2]], np.int32), 2, 1)
    with pytest.raises(_capi.ExflowInvalidArgument, match="num_layers must be >= 2"):
        affinity.count_transitions(np.array([[0]], np.int32), 2, 1)


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (cuobjdump lists the kernels)."""
    import shutil
    import subprocess
    from paper_2401_08383_b200 import _capi
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-lelf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
