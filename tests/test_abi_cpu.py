"""C-ABI library checks that need no GPU: libwq.so builds for sm_100a, loads, exports
every symbol include/wq.h declares, and its two host-only calls agree with the
oracle (thresholds Eq.10-11, byte accounting of D-1)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2605_02262_b200 import build, wq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "wq.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(wq_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    path = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    exported = set(re.findall(r" T (wq_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(wq.exported_symbols()) <= exported
    lib = wq.load()
    for s in declared_symbols():
        assert hasattr(lib, s)
    assert "sm_100a" in wq.wq_version()


def test_library_is_sm100a_only():
    path = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], text=True)
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_host_thresholds_match_oracle(orc):
    s = [0.0, 0.1, 0.5, 0.77, 1.0, -0.2, 1.3]
    for n in (2, 3, 4):
        for alpha in (0.5, 2.0, 5.0):
            assert np.array_equal(wq.wq_thresholds(s, alpha, n), orc.thresholds(s, alpha, n))
    with pytest.raises(wq.WQError):
        wq.wq_thresholds(s, -1.0, 3)


def test_host_packed_bytes_match_oracle(orc):
    for d in (64, 128):
        for S in (16, 32, 64, 128):
            g = wq.geom(1, 4, 28, d, S * 40, S, (2, 4, 8, 16))
            og = orc.geom(1, 4, 28, d, S * 40, S, [2, 4, 8, 16])
            for counts in ([1, 0, 0, 0], [3, 5, 7, 1], [0, 0, 0, 9]):
                for code_only in (False, True):
                    assert wq.wq_packed_bytes(g, counts, code_only) == orc.packed_bytes(og, counts, code_only)


def test_host_packed_bytes_group_granularity(orc):
    """WQ_GRAN_GROUP record sizes (reading Q37) against the oracle's record_bytes(gran=1);
    an unknown granularity is rejected on the host."""
    for d in (64, 128):
        for S in (16, 32, 64, 128):
            g = wq.geom(1, 4, 28, d, S * 40, S, (2, 4, 8, 16))
            for counts in ([1, 0, 0, 0], [3, 5, 7, 1], [0, 0, 0, 9]):
                ref = sum(n * orc.record_bytes(b, d, S, 1) for n, b in zip(counts, (2, 4, 8, 16)))
                assert wq.wq_packed_bytes(g, counts, False, gran=wq.WQ_GRAN_GROUP) == ref
                assert wq.wq_packed_bytes(g, counts, True, gran=wq.WQ_GRAN_GROUP) == wq.wq_packed_bytes(g, counts, True)
    with pytest.raises(wq.WQError):
        wq.wq_packed_bytes(wq.geom(1, 4, 28, 128, 320, 32, (2, 4, 8, 16)), [1, 1, 1, 1], False, gran=7)
