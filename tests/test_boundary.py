"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/elmddm.h
declares, validates its configuration synchronously, and the product package never touches
oracle/.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "elmddm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(elmddm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2406_15959_b200 import _lib

    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_status_codes_match_the_header():
    """The binding's status table is the header's enum (incl. the ELMDDM_WRANK warning, SURVEY
    §8(b): rank deficiency is a warning, not an error)."""
    from paper_2406_15959_b200 import _lib

    src = open(os.path.join(ROOT, "include", "elmddm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    body = src[src.index("typedef enum"):src.index("} elmddm_status")]
    enum = {int(v): k for k, v in re.findall(r"\b(ELMDDM_[A-Z]+)\s*=\s*(\d+)", body)}
    assert enum == _lib.STATUS
    assert enum[_lib.WRANK] == "ELMDDM_WRANK" and issubclass(_lib.RankWarning, UserWarning)


def test_config_validation_is_synchronous_and_cpu_safe():
    """Invalid configurations are rejected with ELMDDM_EINVAL before any CUDA call."""
    from paper_2406_15959_b200 import _lib

    L = _lib.load()
    bad = [
        dict(P=2, M=60, p=16, q=16),     # M not a multiple of 8
        dict(P=2, M=64, p=16, q=15),     # q odd
        dict(P=2, M=512, p=16, q=16),    # m < M (underdetermined local LS)
        dict(P=0, M=64, p=16, q=16),
        dict(P=2, M=64, p=16, q=16, s_begin=3, s_end=2),
        dict(P=9, M=64, p=100, q=16),    # ld > ~9.6k (grid panel) with more than 64 subdomains
        dict(P=2, M=64, p=16, q=15, layout=1),   # lattice: needs p == q
        dict(P=2, M=64, p=16, q=16, layout=2),   # unknown layout
        dict(P=2, M=64, p=16, q=16, problem=7, layout=1),   # plate on the lattice: not supported
    ]
    for b in bad:
        cfg = _lib.Config(b["P"], b["M"], b["p"], b["q"], b.get("problem", 0), 0, 0.125, 0.5, 0, b.get("s_begin", 0),
                          b.get("s_end", max(b["P"] ** 2, 1)), 0, b.get("layout", 0))
        h = C.c_void_p()
        assert L.elmddm_create(C.byref(cfg), 0, C.byref(h)) == 1
        assert not h.value
    assert L.elmddm_create(None, 0, C.byref(C.c_void_p())) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2406_15959_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "liboracle" not in txt and "oracle.c" not in txt, f


def test_library_does_not_link_oracle_or_torch():
    import subprocess

    from paper_2406_15959_b200 import _lib

    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "torch" not in out


def test_sass_uses_fp64_tensor_pipe():
    """The GEMM kernels issue DMMA (FP64 tensor pipe) instructions on sm_100a."""
    import shutil
    import subprocess

    from paper_2406_15959_b200 import _lib

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout


def test_partition_covers_all_subdomains():
    from paper_2406_15959_b200 import partition

    import pytest

    from paper_2406_15959_b200 import ElmddmError

    for N in [1, 4, 16, 64, 256, 1024]:
        for world in [1, 2, 3, 4, 8]:
            per = -(-N // world)
            if (world - 1) * per >= N:  # some rank would own nothing: every rank raises
                with pytest.raises(ElmddmError, match="world <= N"):
                    partition(N, world, 0)
                continue
            got = []
            for r in range(world):
                s0, s1 = partition(N, world, r)
                assert 0 <= s0 <= s1 <= N
                got.extend(range(s0, s1))
            assert got == list(range(N))
