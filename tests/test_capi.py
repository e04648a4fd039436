"""CPU checks of the C ABI: the library loads, exports every declared symbol,
and its host-only functions (hop seeds, child keys) agree with numpy / the oracle."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gfb200.h")


def _declared_functions() -> list[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2311_17410_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        import subprocess

        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2311_17410_b200", "csrc")], check=True)
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    names = _declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2311_17410_b200 import _lib

    assert set(_declared_functions()) == set(_lib.EXPORTED)


def test_hop_seed_matches_numpy(lib):
    from paper_2311_17410_b200 import hop_seed

    assert hop_seed(0, 0) == 15793235383387715774 and hop_seed(0, 1) == 5836529245451711556
    rng = np.random.default_rng(5)
    for s in rng.integers(0, 2**63, 40).tolist() + [2**64 - 1, 2**32, 0]:
        for h in (0, 1, 5, 2**40):
            assert hop_seed(s, h) == int(np.random.SeedSequence([s, h]).generate_state(1, dtype=np.uint64)[0])


def test_child_key_matches_oracle(lib):
    from oracle import child_key

    for p, j in [(0, 0), (1, 9), (2**63, 3), (2**64 - 1, 123456)]:
        assert int(lib.gf_child_key(p, j)) == child_key(p, j)


def test_errors_are_reported_without_gpu(lib):
    h = ctypes.c_void_p()
    assert lib.gf_graph_create(0, 0, 0, 0, 0, ctypes.byref(h)) == 1  # tau < 1 -> EINVAL
    assert b"tau" in lib.gf_last_error()
    assert lib.gf_cache_create(7, 4, 2, 0.5, 0, ctypes.byref(h)) == 1
    assert lib.gf_version().startswith(b"gfb200")


def test_package_imports_without_cuda():
    import paper_2311_17410_b200 as gf

    assert gf.SamplingPolicy("time_window", 5).delta == 5
    with pytest.raises(ValueError):
        gf.SamplingPolicy("time_window", 0)
    with pytest.raises(ValueError):
        gf.SampleRequest([0], [1, 2], [3], gf.SamplingPolicy.recent()).validate()
