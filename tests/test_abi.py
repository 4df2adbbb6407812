"""C-ABI boundary checks that need no GPU: the engine library loads, exports
every symbol include/vnt_engine.h declares, and refuses to run without an
sm_100 device (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared(header: Path):
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vnt_[a-z0-9_]+)\s*\(", text)))


def test_engine_exports_every_declared_symbol():
    import paper_2009_09523_b200 as vnt
    lib = ctypes.CDLL(str(vnt.ENGINE_SO))
    names = declared(ROOT / "include" / "vnt_engine.h")
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_host_library_exports_every_declared_symbol():
    import paper_2009_09523_b200 as vnt
    if not vnt.HOST_SO.exists():
        pytest.skip("libvnt.so not built")
    lib = ctypes.CDLL(str(vnt.HOST_SO))
    names = declared(ROOT / "include" / "vnt_trainer.h")
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2009_09523_b200 as vnt
    with pytest.raises(vnt.VntError) as ei:
        vnt.Engine([4, 16, 4])
    assert ei.value.code == 9
    assert "no CPU fallback" in str(ei.value)


def test_build_info():
    import paper_2009_09523_b200 as vnt
    assert b"sm_100a" in vnt.load_engine().vnt_build_info()


def test_uniform_mapping_semantics():
    """make_uniform_mapping (virtual_exec.cpp:71-100) host logic."""
    import numpy as np
    import paper_2009_09523_b200 as vnt
    sizes, dev = vnt.uniform_mapping(16, 16, 4)
    assert list(sizes) == [1] * 16 and list(np.bincount(dev)) == [4] * 4
    sizes, dev = vnt.uniform_mapping(8192, 32, 1, capacity=256)
    assert (sizes == 256).all() and (dev == 0).all()
    with pytest.raises(vnt.VntError) as e:
        vnt.uniform_mapping(64, 4, 2, capacity=8)
    assert e.value.code == 3 and "gpu0" in str(e.value)
    with pytest.raises(vnt.VntError):
        vnt.uniform_mapping(10, 3, 1)
    with pytest.raises(vnt.VntError):
        vnt.uniform_mapping(8, 2, 4)
