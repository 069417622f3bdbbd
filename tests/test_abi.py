"""The C-ABI library loads and exports every symbol include/coarse_dslash.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "coarse_dslash.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:cd|coarse)_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_boundary_names():
    names = declared_functions()
    for n in ("coarse_field_alloc", "coarse_links_upload", "coarse_dslash_apply", "coarse_dslash_apply_dagger"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_1612_07873_b200 as cd
    lib = ctypes.CDLL(cd.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(cd.EXPORTS) == declared_functions()


def test_version_and_errors_without_gpu():
    import paper_1612_07873_b200 as cd
    assert "sm_100a" in cd.cd_version()
    # argument errors are reported synchronously with a message (no GPU needed)
    with pytest.raises(cd.CDError) as e:
        cd.cd_context_create((2, 2, 2, 2), 25)
    assert e.value.code in (cd.CD_ERR_UNSUPPORTED, cd.CD_ERR_CUDA)
    with pytest.raises(cd.CDError) as e:
        cd.cd_context_create((3, 2, 2, 2), 24, proc_grid=(2, 1, 1, 1), nranks=2, nccl_id=b"\0" * 128)
    assert e.value.code == cd.CD_ERR_INVALID


def test_sass_is_sm100a_with_tma_and_fhfma():
    """The shipped cubins are sm_100a and contain the Blackwell-native instructions the design
    relies on: UBLKCP (cp.async.bulk / TMA 1-D), mbarrier SYNCS, FHFMA (fp16 x fp16 + fp32)."""
    import shutil
    import subprocess
    import paper_1612_07873_b200 as cd
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-lelf", cd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", cd.LIB_PATH], capture_output=True, text=True).stdout
    for mnem in ("UBLKCP", "SYNCS", "FHFMA"):
        assert mnem in sass, mnem
