"""The C-ABI library loads and exports every symbol include/sg.h declares (no GPU).

Also checks that the product package does not import the oracle and fails
loudly without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2204_05988_b200", "libsg.so")


def declared():
    src = open(os.path.join(ROOT, "include", "sg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        subprocess.check_call([os.path.join(ROOT, "paper_2204_05988_b200", "build.sh")])
    return LIB


def test_exports_every_declared_symbol(built):
    import ctypes
    lib = ctypes.CDLL(built)
    names = declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", built]).decode()
    exported = set(re.findall(r"\bT (sg_[a-z0-9_]+)\b", out))
    assert set(names) <= exported


def test_binding_covers_abi(built):
    from paper_2204_05988_b200 import binding
    lib = binding.load_library()
    for n in declared():
        assert getattr(lib, n).argtypes is not None or n == "sg_last_error", n


def test_no_oracle_in_product():
    pkg = os.path.join(ROOT, "paper_2204_05988_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".sh")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_fails_loudly_without_gpu(built):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2204_05988_b200 import Problem, SGError
    from sginputs import get_config
    with pytest.raises(SGError):
        Problem(get_config("c0_2d_const"))
