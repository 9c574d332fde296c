"""The C-ABI library (libpcc_b200.so) loads without a GPU, exports exactly what
include/pcc_b200.h declares, its pure helpers compute the documented
geometry, device entry points fail loudly (status + message) when no GPU is
present, and the shipped SASS uses the FP64 tensor pipe."""

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest
import torch

from paper_1605_01584_b200 import _lib

from conftest import ROOT

HEADER = ROOT / "include" / "pcc_b200.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(pcc_[a-z0-9_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_symbols() == set(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in header_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode == 0:
        exported = set(re.findall(r"\b(pcc_[a-z0-9_]+)\b", out.stdout))
        assert header_symbols() <= exported


def test_pure_helpers():
    L = _lib.lib()
    assert L.pcc_version() >= 100
    assert L.pcc_ldu(1) == 32 and L.pcc_ldu(32) == 32 and L.pcc_ldu(33) == 64 and L.pcc_ldu(1531) == 1536
    assert L.pcc_rows_padded(1) == 128 and L.pcc_rows_padded(128) == 128 and L.pcc_rows_padded(10007) == 10112
    for n, T in [(1, 1), (128, 1), (129, 3), (2000, 136), (16384, 8256), (10007, 3160), (32768, 32896),
                 (65536, 131328)]:
        assert L.pcc_gpu_tile_count(n) == T  # T at T_g=128


def test_invalid_arguments_rejected_before_any_device_work():
    L = _lib.lib()
    with pytest.raises(ValueError, match="samples"):
        _lib.check(L.pcc_normalize_rows_f64(None, 1, None, 1, None, 1, 0, 1, None))
    with pytest.raises(ValueError, match="ldu"):
        _lib.check(L.pcc_syrk_f64(None, 10, 17, 16, 0, 1, 0, None, 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError, match="n must be"):
        _lib.check(L.pcc_syrk_f64(None, 0, 17, 32, 0, 1, 0, None, 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError, match="tile size"):
        _lib.check(L.pcc_compute_pass_f64(ctypes.c_void_p(16), 10, 5, 32, 0, 0, 1, None, None))
    with pytest.raises(ValueError, match="ldu"):
        _lib.check(L.pcc_syrk_exact_f64(None, 10, 17, 16, 0, 1, 0, None, 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError, match="tile size"):
        _lib.check(L.pcc_compute_pass_exact_f64(ctypes.c_void_p(16), 10, 5, 32, 0, 0, 1, None, None))
    with pytest.raises(ValueError, match="destination count"):
        _lib.check(L.pcc_normalize_rows_bcast_f64(ctypes.c_void_p(16), 4, None, None, 0, 32, 4, 0, 1, None))
    with pytest.raises(ValueError, match="tile range"):
        _lib.check(L.pcc_syrk_launches(100, 0, 10**6, ctypes.byref(ctypes.c_int32())))
    with pytest.raises(ValueError, match="null"):
        _lib.check(L.pcc_ipc_get_handle(None, ctypes.create_string_buffer(64)))
    with pytest.raises(ValueError, match="null"):
        _lib.check(L.pcc_ipc_open_handle(None, None))
    assert L.pcc_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_device_calls_fail_loudly_without_gpu():
    info = _lib.DeviceInfo()
    rc = _lib.lib().pcc_device_info(0, ctypes.byref(info))
    assert rc != 0 and _lib.lib().pcc_last_error()


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not shutil.os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="no cuobjdump")
def test_sass_is_sm100a_and_uses_dmma():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "DMMA.8x8x4" in sass          # FP64 tensor pipe in the contraction
    assert "UTMALDG.2D" in sass          # TMA operand staging (production contraction)
    assert "SYNCS" in sass               # mbarrier ring
    assert "UBLKCP" in sass              # 1-D bulk-copy staging (K1, exact mode)
    assert "DMUL" in sass and "DADD" in sass  # exact mode / K1 chains (no FMA contraction)
    assert "UTCIMMA" in sass             # split mode: tcgen05.mma kind::i8 (int8 tensor cores, TMEM)
    assert "UTMALDG.3D" in sass          # split mode: per-slice TMA boxes of the digit planes
    assert "UTCATOMSWS" in sass          # split mode: tcgen05.alloc (TMEM allocation)


def test_split_entry_points_validate_before_device_work():
    L = _lib.lib()
    W = _lib.SPLIT_ROW_BYTES
    # digit planes: 7 planes x padded rows x l rounded up to the 64-byte row segment
    for n, l in [(1, 2), (300, 77), (16384, 4096), (10007, 1531)]:
        assert L.pcc_split_slice_bytes(n, l) == 7 * L.pcc_rows_padded(n) * (-(-l // W) * W)
    assert L.pcc_split_slice_bytes(0, 5) == 0
    with pytest.raises(ValueError, match="l <= 8192"):
        _lib.check(L.pcc_syrk_split_f64(None, None, 4, 8193, 0, 1, 0, None, 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError, match="NULL"):
        _lib.check(L.pcc_syrk_split_f64(None, None, 4, 100, 0, 1, 0, None, 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError, match="tile size"):
        _lib.check(L.pcc_compute_pass_split_f64(None, None, 10, 100, 0, 0, 1, None, None))


@pytest.mark.parametrize("n", [1, 129, 300, 2000, 10007, 16384])
@pytest.mark.parametrize("group", [1, 3, 12])
def test_tile_schedule_is_a_permutation_of_the_range(n, group):
    """The production contraction's visiting order (head row, grouped body,
    tail row) covers each tile of a partition range exactly once."""
    import numpy as np

    from paper_1605_01584_b200.distributed import partition
    from paper_1605_01584_b200.indexing import sym_job_ids

    L = _lib.lib()
    T = int(L.pcc_gpu_tile_count(n))
    mg = -(-n // 128)
    for p in (1, 2, 3, 8):
        for tb, te in partition(T, p):
            k = te - tb
            ys = np.zeros(max(k, 1), dtype=np.uint64)
            xs = np.zeros(max(k, 1), dtype=np.uint64)
            _lib.check(L.pcc_tile_schedule(n, tb, te, group, ys.ctypes.data, xs.ctypes.data))
            if k == 0:
                continue
            ids = np.sort(sym_job_ids(mg, ys[:k], xs[:k]))
            assert np.array_equal(ids, np.arange(tb, te, dtype=np.uint64))


def _build_capi_example(tmp_path):
    root = Path(__file__).resolve().parent.parent
    exe = tmp_path / "capi_allpairs"
    cmd = ["gcc", "-O2", "-Wall", "-Werror", f"-I{root / 'include'}", "-I/usr/local/cuda/include",
           str(root / "examples" / "capi_allpairs.c"), "-o", str(exe), f"-L{root / 'paper_1605_01584_b200' / 'lib'}",
           "-lpcc_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{root / 'paper_1605_01584_b200' / 'lib'}", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_capi_example_compiles_against_the_header(tmp_path):
    """examples/capi_allpairs.c: the ABI used from plain C (no Python) builds
    against include/pcc_b200.h and links libpcc_b200.so."""
    assert _build_capi_example(tmp_path).exists()


@pytest.mark.gpu
def test_capi_example_runs_on_the_gpu(tmp_path):
    out = subprocess.run([str(_build_capi_example(tmp_path)), "300", "77"], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stdout + out.stderr
