"""Pins for oracle O-1..O-4 (Philox, draw, bounded draw, Floyd selection).

Each test checks the oracle against something other than itself: published known-answer
vectors, the defining property of a map, exhaustive enumeration, or a statistical law."""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle
from tests._util import GOLDEN


def test_philox_known_answer_vectors():
    """O-1 against Random123's published KATs (tests/golden/philox4x32_10_kat.json)."""
    kat = json.load(open(os.path.join(GOLDEN, "philox4x32_10_kat.json")))
    for vec in kat["vectors"]:
        ctr = [int(x, 16) for x in vec["ctr"]]
        key = [int(x, 16) for x in vec["key"]]
        out = oracle.philox4x32_10(ctr, key)
        assert [f"{x:08x}" for x in out] == vec["out"]


def test_draw_is_keyed_by_seed_pass_hop_node_slot():
    """O-2: u depends on every key component; (ctr=(v,i,hop,pass), key=(seed lo, hi))."""
    base = oracle.draw(4, 0, 1, 17, 3)
    assert base != oracle.draw(5, 0, 1, 17, 3)
    assert base != oracle.draw(4, 1, 1, 17, 3)
    assert base != oracle.draw(4, 0, 2, 17, 3)
    assert base != oracle.draw(4, 0, 1, 18, 3)
    assert base != oracle.draw(4, 0, 1, 17, 4)
    # (seed high word lands in key[1]); check layout against the block function itself is
    # covered by the KAT; here check the packing u = r.y<<32 | r.x on a KAT vector:
    r = oracle.philox4x32_10([0, 0, 0, 0], [0, 0])
    assert oracle.draw(0, 0, 0, 0, 0) == (int(r[1]) << 32) | int(r[0])


def test_draw_counter_layout_pinned_by_kat():
    """O-2 counter layout ctr = (v, i, hop, pass), key = (seed lo32, seed hi32), u = r.y<<32 | r.x,
    pinned by routing Random123 KAT vectors with four DISTINCT counter words through draw():
    any permutation of (v, i, hop, pass), a swapped key half or a swapped output word fails.
    Vector 3: ctr (243f6a88, 85a308d3, 13198a2e, 03707344), key (a4093822, 299f31d0) ->
    out (d16cfe09, 94fdcceb, ...) (tests/golden/philox4x32_10_kat.json)."""
    kat = json.load(open(os.path.join(GOLDEN, "philox4x32_10_kat.json")))
    for vec in kat["vectors"]:
        c = [int(x, 16) for x in vec["ctr"]]
        k = [int(x, 16) for x in vec["key"]]
        o = [int(x, 16) for x in vec["out"]]
        seed = (k[1] << 32) | k[0]
        assert oracle.draw(seed, c[3], c[2], c[0], c[1]) == (o[1] << 32) | o[0]
    # the literal value of the verdict's pin (vector 3), stated once more in full
    assert oracle.draw(0x299F31D0A4093822, 0x03707344, 0x13198A2E, 0x243F6A88, 0x85A308D3) == 0x94FDCCEBD16CFE09


@pytest.mark.parametrize("m", [1, 2, 3, 7, 10, 1000, 65537, 2**31 - 1, 2**32])
def test_bounded_threshold_property(m):
    """O-3: bounded(., m) is the monotone map of [0,2^64) onto [0,m) whose j-th preimage
    starts at ceil(j*2^64/m).  Checked at every threshold for small m and at sampled
    thresholds otherwise (Python big integers, no 128-bit arithmetic)."""
    js = range(1, m) if m <= 1000 else np.random.default_rng(m).integers(1, m, 200)
    for j in js:
        j = int(j)
        start = -(-(j << 64) // m)  # ceil
        assert oracle.bounded(start, m) == j
        assert oracle.bounded(start - 1, m) == j - 1
    assert oracle.bounded(0, m) == 0
    assert oracle.bounded(2**64 - 1, m) == m - 1


@pytest.mark.parametrize("deg", range(1, 8))
def test_floyd_exact_uniformity_bruteforce(deg):
    """O-4: enumerate every tuple of draws t_i in [0, deg-k+i]; every k-subset must be
    produced exactly k! times (Floyd's algorithm is exactly uniform)."""
    for k in range(1, deg + 1):
        counts = {}
        ranges = [range(deg - k + i + 1) for i in range(k)]
        for t in itertools.product(*ranges):
            ch = oracle.floyd_from_draws(deg, list(t))
            assert len(set(ch.tolist())) == k and min(ch) >= 0 and max(ch) < deg
            key = tuple(sorted(ch.tolist()))
            counts[key] = counts.get(key, 0) + 1
        assert len(counts) == math.comb(deg, k)
        assert set(counts.values()) == {math.factorial(k)}


def test_select_small_degree_takes_all_in_order():
    """O-4: deg <= f -> ranks 0..deg-1 (no randomness), deg 0 -> nothing."""
    assert oracle.select(4, 0, 0, 5, 3, 5).tolist() == [0, 1, 2]
    assert oracle.select(4, 0, 0, 5, 5, 5).tolist() == [0, 1, 2, 3, 4]
    assert oracle.select(4, 0, 0, 5, 0, 5).tolist() == []


def test_select_sorted_distinct_and_chi_square_uniform():
    """O-4 with Philox draws: sorted, distinct, in range; rank marginals uniform
    (each rank chosen with probability k/deg) by a chi-square test over 60k nodes, and
    pair frequencies uniform (k=2 subsets) over another 45k."""
    deg, f = 10, 3
    hist = np.zeros(deg)
    for v in range(60_000):
        r = oracle.select(4, 0, 1, v, deg, f)
        assert len(r) == 3 and np.all(np.diff(r) > 0) and r[0] >= 0 and r[-1] < deg
        hist[r] += 1
    p = stats.chisquare(hist).pvalue
    assert p > 1e-4, (hist, p)
    pairs = np.zeros((6, 6))
    for v in range(45_000):
        r = oracle.select(9, 1, 0, v, 6, 2)
        pairs[r[0], r[1]] += 1
    obs = pairs[np.triu_indices(6, 1)]
    assert stats.chisquare(obs).pvalue > 1e-4


def test_select_large_degree_hub():
    """Hub of degree 10^6: k = f draws, all distinct and in range."""
    r = oracle.select(4, 0, 2, 123, 1_000_000, 15)
    assert len(r) == 15 and len(set(r.tolist())) == 15 and r.max() < 1_000_000
    assert np.all(np.diff(r) > 0)
