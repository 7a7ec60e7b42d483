"""CPU checks of the boundary: the C-ABI library builds, loads without a GPU
and exports every function include/hifuse.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2408_08490_b200")
LIB = os.path.join(PKG, "libhifuse.so")


def declared():
    txt = open(os.path.join(ROOT, "include", "hifuse.h")).read()
    return sorted(set(re.findall(r"^\s*(?:hifuse_status|size_t|const char \*|int64_t)\s*\*?\s*(hifuse_\w+)\s*\(",
                                 txt, re.M)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", PKG, "-j8"], stdout=subprocess.DEVNULL)
    names = declared()
    assert len(names) >= 18
    L = ctypes.CDLL(LIB)
    for n in names:
        assert hasattr(L, n), n
    L.hifuse_status_string.restype = ctypes.c_char_p
    assert L.hifuse_status_string(0) == b"ok"


def test_host_only_size_query():
    """hifuse_csr_sizes is host-only: it runs without a device."""
    import numpy as np
    from paper_2408_08490_b200 import hifuse as hf
    sh = hf.Shape([0, 1], [1, 0], [10, 7], [4, 3], 25)
    assert sh.rows == 3 + 4 and sh.S == 10 + 7 and sh.U_max == 17
    assert sh.build_ws > 0


def test_host_side_errors_launch_nothing():
    import numpy as np
    from paper_2408_08490_b200 import hifuse as hf
    with __import__("pytest").raises(hf.HifuseError) as e:
        hf.Shape([0, 5], [1, 0], [10, 7], [4, 3], 25)   # relation type out of range
    assert e.value.code == 1
    with __import__("pytest").raises(hf.HifuseError):
        hf.Shape([0], [0], [3], [4], 5)                 # n_dst > n_src
