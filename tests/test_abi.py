"""The C-ABI library loads without a GPU and exports every declared symbol."""
import ctypes
import os
import re

from conftest import REPO


def declared_functions():
    src = open(os.path.join(REPO, "include", "maya_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(maya_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    from paper_2503_20191_b200 import engine
    L = engine.lib()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(engine.EXPORTED)
    assert L.maya_abi_version() == 1


def test_no_gpu_open_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2503_20191_b200.engine import Engine, EngineError
    import pytest
    with pytest.raises(EngineError):
        Engine(0)
