"""Host-side checks of the boundary (no GPU compute): the C-ABI library builds for sm_100a, loads,
exports exactly the entry points include/ldu.h declares, and fails loudly without a GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "ldu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:ldu_status|const char \*|int)\s*\**\s*([a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("ldu_setup", "ldu_amul", "pcg_solve", "pipecg_solve", "ldu_comm_init",
                 "ldu_get_unique_id", "ldu_destroy", "ldu_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_1505_07630_b200 as ldu
    out = subprocess.check_output(["nm", "-D", "--defined-only", ldu.LIB_PATH]).decode()
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    for name in declared_functions():
        assert name in exported, name
        assert name in ldu.SIGNATURES, name
    assert ldu.abi_version() == 2


def test_library_is_sm100a():
    import paper_1505_07630_b200 as ldu
    out = subprocess.check_output(["cuobjdump", "--list-elf", ldu.LIB_PATH]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_links_torch_nccl():
    import paper_1505_07630_b200 as ldu
    out = subprocess.check_output(["readelf", "-d", ldu.LIB_PATH]).decode()
    assert "libnccl.so.2" in out and "nvidia/nccl/lib" in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    import paper_1505_07630_b200 as ldu
    with pytest.raises(ldu.LduError) as ei:
        ldu.LduMatrix(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32), np.ones(3),
                      -np.ones(2))
    assert ei.value.status == ldu.ERR_CUDA


def test_product_never_imports_oracle():
    """The product package and bench's GPU arm must not route through oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1505_07630_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "ldu_oracle" not in txt, f


def test_arg_marshalling_rejects_wrong_dtypes():
    import paper_1505_07630_b200 as ldu
    with pytest.raises(TypeError):
        ldu._ptr(np.zeros(3, np.float32), "f64")
    with pytest.raises(TypeError):
        ldu._ptr(np.zeros(3, np.int64), "i32")
