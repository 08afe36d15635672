"""CPU-side checks of the C-ABI boundary: libbbf.so builds, loads, exports every function that
include/bbf.h declares, and — with no GPU — refuses to count (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "bbf.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:bbf_status|int|const char\s*\*)\s*(bbf_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2308_07932_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    f = declared_functions()
    for name in ("bbf_graph_load_csr", "bbf_count_global", "bbf_count_per_vertex",
                 "bbf_count_pairs_topk", "bbf_graph_free", "bbf_last_error", "bbf_abi_version",
                 "bbf_nccl_unique_id", "bbf_comm_init", "bbf_comm_free", "bbf_graph_stats"):
        assert name in f


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(bbf_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(libpath)
    for f in declared_functions():
        assert hasattr(lib, f)


def test_sm100a_code_present(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_no_gpu_refusal(libpath):
    import torch
    from paper_2308_07932_b200 import bbf
    assert bbf.abi_version() == 1
    if torch.cuda.is_available():
        pytest.skip("GPU present: refusal path not applicable")
    with pytest.raises(bbf.BBFError) as e:
        bbf.Graph(2, 2, np.array([0, 2, 4], np.uint64), np.array([0, 1, 0, 1], np.uint32),
                  np.ones(4, np.uint8))
    assert e.value.name == "BBF_ECUDA"


def test_null_handle_errors(libpath):
    """Handle-level calls refuse a null graph with BBF_EINVAL (no device needed)."""
    import ctypes as C
    from paper_2308_07932_b200 import bbf
    L = bbf.lib()
    a, b = C.c_uint32(7), C.c_uint32(7)
    assert L.bbf_graph_hybrid_core(None, C.byref(a), C.byref(b)) == 1  # BBF_EINVAL
    assert L.bbf_graph_stats(None, None, None, None, None) == 1


def test_binding_never_imports_oracle():
    src = open(os.path.join(ROOT, "paper_2308_07932_b200", "bbf.py")).read()
    src += open(os.path.join(ROOT, "paper_2308_07932_b200", "__init__.py")).read()
    assert "oracle" not in re.sub(r'""".*?"""', "", src, flags=re.S).replace("Importing this package never imports the CPU oracle", "")
    for f in os.listdir(os.path.join(ROOT, "paper_2308_07932_b200", "csrc")):
        txt = open(os.path.join(ROOT, "paper_2308_07932_b200", "csrc", f)).read()
        assert "oracle" not in txt.lower()


def test_upload_api_argument_errors_without_gpu(libpath):
    """The pipelined-loading entry points validate their arguments before touching a device and,
    with no GPU, refuse (no CPU fallback); freeing a NULL upload is a no-op."""
    import torch
    from paper_2308_07932_b200 import bbf
    L = bbf.lib()
    out = ctypes.c_void_p()
    assert L.bbf_upload_csr(2, 2, None, None, None, 0, ctypes.byref(out)) == bbf.BBF_EINVAL
    rp = np.array([0, 2, 4], np.uint64)
    assert L.bbf_upload_csr(2, 2, rp.ctypes.data_as(ctypes.c_void_p), None, None, 0,
                            ctypes.byref(out)) == bbf.BBF_EINVAL  # nnz > 0 without col / sign
    assert L.bbf_graph_load_upload(None, 0, None, None, ctypes.byref(out)) == bbf.BBF_EINVAL
    assert L.bbf_upload_free(None) == bbf.BBF_OK
    if torch.cuda.is_available():
        pytest.skip("GPU present: refusal path not applicable")
    with pytest.raises(bbf.BBFError) as e:
        bbf.Upload(2, 2, rp, np.array([0, 1, 0, 1], np.uint32), np.ones(4, np.uint8))
    assert e.value.name == "BBF_ECUDA"


def test_build_stamp_records_flags(libpath):
    """The default build's object directory carries a stamp of the flags it was compiled with and
    no extra flags (diagnostic variants build into their own directories, _build_<name>)."""
    import json
    from paper_2308_07932_b200 import build
    stamp = json.load(open(os.path.join(build.BUILD, "flags.json")))
    assert stamp["extra"] == [] and stamp["arch"] == build.ARCH
    assert "-lineinfo" in stamp["flags"]
    assert libpath == build.LIB
