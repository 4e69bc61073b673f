"""The native host packer (`_vgpack`, csrc/vg_pack.cpp) of the drop-in APIs,
on the CPU: it writes the same CSR arrays as numpy packing, applies the
reference's row checks (validation.py:12-30; channel range gridgen.py:114-119)
and hands every input it does not take back to the general path (-1)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2211_08506_b200 import ParticleSet, _native, synth


@pytest.fixture(scope="module")
def pk():
    return _native.pack()


def _rows(pb):
    return [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
            for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]


def _bufs(B, n):
    return np.full(B + 1, -7, np.int64), np.full(n, -7, np.int32), np.full((n, 3), np.nan)


def test_rows_pack_equals_numpy_packing(pk):
    pb = synth.packed_batch(synth.CONFIGS[0], range(50))
    X = _rows(pb)
    X[4] = np.zeros((0, 4))
    off_ref = np.concatenate([[0], np.cumsum([len(x) for x in X])])
    rows = np.concatenate(X)
    for a, b in ((0, 50), (3, 17), (4, 5), (49, 50)):
        n = pk.rows_count(X, a, b)
        assert n == off_ref[b] - off_ref[a]
        off, ch, xyz = _bufs(b - a, n)
        assert pk.rows_pack(X, a, b, 5, off.ctypes.data, ch.ctypes.data, xyz.ctypes.data, n) == n
        assert np.array_equal(off, off_ref[a:b + 1] - off_ref[a])
        sl = slice(off_ref[a], off_ref[b])
        assert np.array_equal(ch, rows[sl, 0].astype(np.int32))
        assert np.array_equal(xyz, rows[sl, 1:4])


@pytest.mark.parametrize("row", [[5.0, 1, 1, 1], [-1.0, 1, 1, 1], [0.5, 1, 1, 1],
                                 [1.0, np.nan, 1, 1], [1.0, 1, np.inf, 1], [np.nan, 1, 1, 1]])
def test_rows_pack_rejects_invalid_values(pk, row):
    X = [np.array([[0.0, 1, 2, 3]]), np.array([[1.0, 2, 3, 4], row])]
    off, ch, xyz = _bufs(2, 3)
    assert pk.rows_count(X, 0, 2) == 3
    assert pk.rows_pack(X, 0, 2, 5, off.ctypes.data, ch.ctypes.data, xyz.ctypes.data, 3) == -1


def test_rows_count_hands_other_inputs_to_the_general_path(pk):
    for item in (np.zeros((2, 4), np.float32), [[0.0, 1, 2, 3]], np.zeros((3, 8))[:, ::2],
                 np.zeros(4), np.zeros((2, 3)), np.zeros((0,)), "abcd", None):
        assert pk.rows_count([np.zeros((1, 4)), item], 0, 2) == -1
    assert pk.rows_count([np.zeros((0, 4))], 0, 1) == 0
    # capacity is enforced: -(2 + n) asks for n atoms of staging
    off, ch, xyz = _bufs(2, 1)
    assert pk.rows_pack([np.zeros((1, 4)), np.zeros((2, 4))], 0, 2, 5, off.ctypes.data,
                        ch.ctypes.data, xyz.ctypes.data, 1) == -(2 + 3)


def test_sets_pack_equals_numpy_packing(pk):
    pb = synth.packed_batch(synth.CONFIGS[0], range(30))
    sets = [ParticleSet(pb.channels[a:b], pb.xyz.reshape(-1, 3)[a:b])
            for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
    counts = np.array([len(s) for s in sets], dtype=np.int64)
    counts[7] = 0                                   # a molecule with a recorded error
    off_ref = np.concatenate([[0], np.cumsum(counts)])
    keep = [s for s, c in zip(sets, counts) if c]
    n = int(counts.sum())
    off, ch, xyz = _bufs(30, n)
    assert pk.sets_pack(sets, 0, 30, counts.ctypes.data, off.ctypes.data, ch.ctypes.data,
                        xyz.ctypes.data, n) == 0
    assert np.array_equal(off, off_ref)
    assert np.array_equal(ch, np.concatenate([s.channels for s in keep]).astype(np.int32))
    assert np.array_equal(xyz, np.concatenate([s.positions for s in keep]))
    # a set whose arrays are not contiguous int64 / float64 goes to numpy
    odd = ParticleSet(np.arange(6, dtype=np.int64)[::2] % 3, np.ones((3, 3)))
    c1 = np.array([3], np.int64)
    off, ch, xyz = _bufs(1, 3)
    rc = pk.sets_pack([odd], 0, 1, c1.ctypes.data, off.ctypes.data, ch.ctypes.data,
                      xyz.ctypes.data, 3)
    assert rc in (0, -1)
    if rc == 0:
        assert np.array_equal(ch, odd.channels.astype(np.int32))


def test_numpy_fallback_packer_matches_native(pk):
    """loader._rows_chunk (the general path for inputs the native packer does
    not take: lists, other dtypes) packs the same rows and rejects the same
    values."""
    from paper_2211_08506_b200.loader import _rows_chunk

    pb = synth.packed_batch(synth.CONFIGS[0], range(20))
    X = _rows(pb)
    X32 = [x.astype(np.float32) for x in X]                  # float32 arrays
    assert pk.rows_count(X32, 0, len(X32)) == -1             # not the native packer's
    counts, rows = _rows_chunk(X32, 5)
    assert np.array_equal(counts, np.diff(pb.offsets))
    assert np.array_equal(rows, np.concatenate(X32).astype(np.float64))
    got = _rows_chunk([x.tolist() for x in X[:3]], 5)      # nested lists
    assert got is not None and np.array_equal(got[1], np.concatenate(X[:3]))
    for bad in ([[5.0, 1, 1, 1]], [[0.5, 1, 1, 1]], [[-1.0, 1, 1, 1]], [[1.0, np.inf, 0, 0]],
                [[1.0, 2.0, 3.0]]):
        assert _rows_chunk([X[0], np.array(bad)], 5) is None
