"""The C-ABI library loads and exports every symbol include/qcs_b200.h
declares (no device needed: nothing here launches a kernel)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qcs_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qcs_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for need in ("qcs_state_create", "qcs_apply_gate", "qcs_run_program", "qcs_read_stride",
                 "qcs_export_blocks", "qcs_import_blocks", "qcs_state_stats",
                 "qcs_codec_compress", "qcs_codec_decompress", "qcs_state_destroy",
                 "qcs_last_error"):
        assert need in names


def test_library_exports_every_declared_symbol():
    from paper_1811_05140_b200 import build
    if not os.path.exists(build.SO):
        pytest.skip("libqcs_b200.so not built")
    lib = ctypes.CDLL(build.SO)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_device_path_fails_loudly():
    """Without a GPU the engine refuses instead of falling back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1811_05140_b200 import build
    if not os.path.exists(build.SO):
        pytest.skip("libqcs_b200.so not built")
    import paper_1811_05140_b200 as q
    import numpy as np
    with pytest.raises(q.DeviceError):
        q.CompressedState.basis_state(q.StateGeometry.make(4, 2), 0)
    with pytest.raises(q.DeviceError):
        q.compress(np.zeros(8), 0.0)
