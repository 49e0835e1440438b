"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/gtap.h declares.

No compute calls here (no GPU in the build container); argument validation that
returns before touching the device is exercised.
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gtap.h")


@pytest.fixture(scope="module")
def libgtap():
    from paper_2604_05982_b200 import build as b
    b.build()
    from paper_2604_05982_b200 import gtap
    return gtap.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gtap_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(libgtap):
    names = declared_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(libgtap, n), f"{n} declared in gtap.h but not exported"
    from paper_2604_05982_b200 import gtap
    assert sorted(gtap.EXPORTS) == names


def test_dynamic_symbols_are_c_abi(libgtap):
    from paper_2604_05982_b200 import gtap
    out = subprocess.run(["nm", "-D", "--defined-only", gtap.LIB_PATH], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for n in declared_functions():
        assert n in syms  # unmangled: extern "C"


def test_sm100a_cubin(libgtap):
    from paper_2604_05982_b200 import gtap
    out = subprocess.run(["cuobjdump", "--list-elf", gtap.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(libgtap):
    from paper_2604_05982_b200 import gtap
    assert libgtap.gtap_abi_version() == 2 == gtap.ABI_VERSION
    assert libgtap.gtap_status_str(5) == b"GTAP_E_POOL_EXHAUSTED"
    assert libgtap.gtap_status_str(0) == b"GTAP_OK"


def test_config_validation_without_gpu(libgtap):
    from paper_2604_05982_b200 import gtap
    cfg = gtap.Config()
    assert libgtap.gtap_config_default(ctypes.byref(cfg), 0, 0) == 0
    assert cfg.struct_size == ctypes.sizeof(gtap.Config)
    assert libgtap.gtap_workspace_bytes(ctypes.byref(cfg)) > 0
    bad = gtap.Config.from_buffer_copy(cfg)
    bad.block_size = 48  # not a multiple of 32
    assert libgtap.gtap_workspace_bytes(ctypes.byref(bad)) == 0
    bad = gtap.Config.from_buffer_copy(cfg)
    bad.max_tasks_per_worker = 1000  # not a power of two
    assert libgtap.gtap_workspace_bytes(ctypes.byref(bad)) == 0
    bad = gtap.Config.from_buffer_copy(cfg)
    bad.struct_size = 4  # ABI guard
    assert libgtap.gtap_workspace_bytes(ctypes.byref(bad)) == 0
    # no device here: init refuses cleanly
    h = ctypes.c_void_p()
    rc = libgtap.gtap_init(ctypes.byref(cfg), None, 0, ctypes.byref(h))
    import torch
    if not torch.cuda.is_available():
        assert rc == 10  # GTAP_E_NO_DEVICE
    assert libgtap.gtap_finalize(None) == 0


def test_table_constructor_validation(libgtap):
    assert libgtap.gtap_table_mergesort(None, None, 16, 128) is None
    assert libgtap.gtap_table_spmv(None, None, None, None, None, 4, 16, 16) is None
    assert libgtap.gtap_table_bfs(None, None, None, 4) is None
    t = libgtap.gtap_table_fib()
    assert t
    libgtap.gtap_table_destroy(t)


def test_workspace_layout_scales(libgtap):
    from paper_2604_05982_b200 import gtap
    cfg = gtap.Config()
    libgtap.gtap_config_default(ctypes.byref(cfg), 0, 0)
    cfg.grid_size, cfg.block_size, cfg.max_tasks_per_worker = 100, 64, 1024
    b1 = libgtap.gtap_workspace_bytes(ctypes.byref(cfg))
    cfg.max_tasks_per_worker = 2048
    b2 = libgtap.gtap_workspace_bytes(ctypes.byref(cfg))
    W = 200
    # records (32 B) + free ring (4 B) + deque ring (4 B, capacity = pool) per slot
    assert b2 - b1 == pytest.approx(W * 1024 * (32 + 4 + 4), rel=0.01)
