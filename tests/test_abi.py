"""CPU checks of the boundary: librk.so builds, loads, and exports every symbol include/rk.h declares;
host-side helpers (action indexing, shard planning). No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

import paper_1804_06087_b200 as rk
from paper_1804_06087_b200 import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    txt = open(os.path.join(ROOT, "include", "rk.h")).read()
    return sorted(set(re.findall(r"\b(rk_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported():
    L = rk.load_library()
    so = L._name
    out = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    exported = set(re.findall(r" T (rk_\w+)", out))
    want = declared()
    assert want, "no declarations parsed"
    missing = [s for s in want if s not in exported]
    assert not missing, missing
    assert set(rk.rk.EXPORTS) == set(want)


def test_status_strings_without_gpu():
    L = rk.load_library()
    assert L.rk_status_string(0) == b"RK_OK"
    assert L.rk_status_string(7) == b"RK_ENONFINITE"


def test_product_path_does_not_import_oracle():
    """The product package must never import the oracle (parity would be void)."""
    pkg = os.path.join(ROOT, "paper_1804_06087_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in src.replace("oracle-flagged", ""), f


def test_action_index_bijection():
    # |M|=3, |B|=4 -> 28 actions, index 0 <-> (v=0b001, B[0])
    K, nB = 3, 4
    n = ((1 << K) - 1) * nB
    assert n == 28
    assert rk.action_decode(0, K, nB) == (1, 0)
    seen = set()
    for i in range(n):
        v, b = rk.action_decode(i, K, nB)
        assert rk.action_index(v, b, nB) == i
        seen.add((v, b))
    assert len(seen) == n
    with pytest.raises(ValueError):
        rk.action_index(0, 0, nB)


def test_shard_ranges_aligned():
    B = [16, 32, 48, 64]  # the paper's B, lcm 192
    for N in (0, 1, 191, 192, 1000, 50_000, 1_000_000):
        for world in (1, 2, 3, 8):
            rs = shard.shard_ranges(N, world, B)
            assert sum(n for _, n in rs) == N
            pos = 0
            for off, n in rs:
                assert off == pos
                pos += n
            # every boundary except the end is a multiple of lcm(B)
            for off, n in rs:
                if off + n != N:
                    assert (off + n) % 192 == 0
    assert shard.chunk_ranges(0, 1000, 256, [16, 32]) == [(0, 256), (256, 256), (512, 256), (768, 232)]
