"""C-ABI library checks that need no GPU: it loads, exports every symbol declared in
include/anyseq.h, reports status strings, and refuses to run without a device (no CPU
fallback)."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    import paper_2002_04561_b200 as A
    names = A.header_functions()
    assert "anyseq_align_batch" in names and "anyseq_traceback" in names and \
        "anyseq_align_long" in names
    lib = ctypes.CDLL(A.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(names) <= exported


def test_status_strings_and_version():
    import paper_2002_04561_b200 as A
    assert "sm_100a" in A.version()
    assert A._lib.anyseq_status_str(0) == b"ok"
    assert A._lib.anyseq_status_str(2) == b"invalid sequence byte"
    assert A._lib.anyseq_status_str(99) == b"unknown status"


def test_no_cpu_fallback_without_device():
    import torch
    import paper_2002_04561_b200 as A
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(A.AnyseqError) as e:
        A.Context([0])
    assert e.value.status_name == "E_CUDA"


def test_null_context_is_rejected():
    import paper_2002_04561_b200 as A
    assert A._lib.anyseq_align_batch(None, None, None, None, None) == 1
    assert A._lib.anyseq_traceback(None, None, None, None, None, 0, None) == 1
    assert A._lib.anyseq_sync(None) == 1


def test_sm100a_only_code():
    """The shared library carries sm_100a SASS (and no other architecture)."""
    import paper_2002_04561_b200 as A
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", A.LIB_PATH],
                       capture_output=True, text=True)
    assert r.returncode == 0
    archs = set()
    for line in r.stdout.splitlines():
        for tok in line.replace(".", " ").split():
            if tok.startswith("sm_"):
                archs.add(tok)
    assert archs and all(a.startswith("sm_100") for a in archs), archs
