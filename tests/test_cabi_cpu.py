"""CPU: the C-ABI library loads without a GPU and exports every symbol include/ltl_core.h declares; without
a device the product path fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2402_12373_b200 import build as B
from paper_2402_12373_b200 import core as K
from paper_2402_12373_b200.errors import BackendUnavailable

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ltl_core.h")).read()
    return sorted(set(re.findall(r"LTL_API\s+[\w\s\*]+?\b(ltl_\w+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(B.build())
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert lib.ltl_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np

    with pytest.raises(BackendUnavailable):
        K.make_core(np.full(4, 2**64 - 1, dtype=np.uint64), 2, 0, K.V_MUELLER)
    from paper_2402_12373_b200.learner import learn

    with pytest.raises(BackendUnavailable):
        learn([(1, 0), (0, 1)], [(0, 0), (1, 1)], 2, max_cost=5)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2402_12373_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), f
                assert "liboracle" not in text, f
