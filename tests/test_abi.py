"""The C-ABI library loads (no GPU needed) and exports every symbol the public
header declares; the ctypes binding covers all of them; without a device every
compute entry point fails loudly with a status code (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "morphserve.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ms_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2506_02006_b200 import _native as N
    lib = N.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    bound = {name for name, _, _ in N.SIGNATURES}
    assert set(syms) == bound


def test_host_runtime_libraries_load():
    from paper_2506_02006_b200 import _core
    assert hasattr(_core, "run_simulation") and hasattr(_core, "KvBlockPool")
    C.CDLL(os.path.join(ROOT, "paper_2506_02006_b200", "lib", "libmorphserve_host.so"))


def test_no_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2506_02006_b200 import _native as N
    from paper_2506_02006_b200.device import DeviceModel, LLAMA2_7B, TINY, layer_pages
    assert layer_pages(TINY, 16) == 48 and layer_pages(TINY, 4) == 16
    # Q8 images: 16640-B chunks; Q3 shares the 4-bit container image
    # (32 KiB tiny pages hold one 16640-B chunk each, so tiny Q8 saves nothing)
    assert layer_pages(TINY, 8) == 48 and layer_pages(TINY, 3) == layer_pages(TINY, 4)
    assert layer_pages(LLAMA2_7B, 8) == 25 and layer_pages(LLAMA2_7B, 3) == 13
    with pytest.raises(N.MsError):
        DeviceModel(TINY, arena_pages=64)


def test_validation_without_device():
    from paper_2506_02006_b200 import _native as N
    from paper_2506_02006_b200.device import model_desc, TINY
    d = model_desc(TINY, max_batch=1, max_prefill_tokens=1, max_pos=16, arena_pages=1)
    assert N.lib().ms_layer_pages(C.byref(d), 5) == -1
    d.head_dim = 96
    h = C.c_void_p()
    assert N.lib().ms_ctx_create(0, C.byref(d), C.byref(h)) == N.MS_EVALIDATION
    assert b"head_dim" in N.lib().ms_last_error()
