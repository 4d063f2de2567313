"""Pins for the oracle's counter-based RNG.

P1: Philox4x32-10 against the published Random123 known-answer vectors.
P2: uniforms are exactly representable in fp32 (so GPU and oracle consume the
    same numbers); Box-Muller normals have the moments of N(0,1).
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kats():
    out = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        out.append((v[0:4], v[4:6], v[6:10]))
    return out


@pytest.mark.parametrize("ctr,key,expect", _kats())
def test_philox_kat(oracle_lib, ctr, key, expect):
    assert oracle_lib.philox(ctr, key) == expect


def test_draw_addressing(oracle_lib):
    # draw q is word q&3 of block q>>2 of counter (q>>2, phase<<24|sub, gid, iter)
    seed = 0x123456789ABCDEF0
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for q in range(12):
        blk = oracle_lib.philox([q >> 2, (3 << 24) | 7, 42, 9], key)
        assert oracle_lib.draw_u32(seed, 9, 42, 3, 7, q) == blk[q & 3]


def test_uniform_exact_in_fp32(oracle_lib):
    for q in range(2000):
        u = oracle_lib.draw_uniform(5, 1, q, 3, 0, q % 7)
        assert 0.0 < u < 1.0
        assert float(np.float32(u)) == u
        r = oracle_lib.draw_u32(5, 1, q, 3, 0, q % 7)
        assert u == ((r >> 9) + 0.5) / 2 ** 23


def test_uniform_distribution(oracle_lib):
    u = np.array([oracle_lib.draw_uniform(11, 2, g, 4, 1, 0) for g in range(40000)])
    assert abs(u.mean() - 0.5) < 4 * np.sqrt(1 / 12 / u.size)
    assert abs(u.var() - 1 / 12) < 0.003


def test_normals_moments(oracle_lib):
    z = np.concatenate([oracle_lib.draw_normals(3, 1, g, 3, 0, 10) for g in range(8000)])
    n = z.size
    assert abs(z.mean()) < 4 / np.sqrt(n)
    assert abs(z.var() - 1.0) < 4 * np.sqrt(2.0 / n)
    kurt = np.mean(z ** 4) / np.mean(z ** 2) ** 2
    assert abs(kurt - 3.0) < 0.1
    # odd d: the last normal is the cosine branch of the pair
    z5 = oracle_lib.draw_normals(3, 1, 0, 3, 0, 5)
    z6 = oracle_lib.draw_normals(3, 1, 0, 3, 0, 6)
    assert np.array_equal(z5, z6[:5])


def test_streams_independent(oracle_lib):
    a = np.array([oracle_lib.draw_uniform(1, 1, g, 3, 0, 0) for g in range(20000)])
    b = np.array([oracle_lib.draw_uniform(1, 1, g, 3, 1, 0) for g in range(20000)])
    c = np.array([oracle_lib.draw_uniform(1, 2, g, 3, 0, 0) for g in range(20000)])
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.04
    assert abs(np.corrcoef(a, c)[0, 1]) < 0.04
