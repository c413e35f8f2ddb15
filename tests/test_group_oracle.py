"""Pins for the row-f3 oracle (oracle/group.py): the segmented bundles are a stable partition.

Checked against what the definition fixes: a hand-worked example, and on random labels that the
order is a permutation, that each segment holds exactly its bundle's fibers in increasing index,
that the offsets are the prefix of the counts and the summaries those of a direct per-bundle scan.
"""
import numpy as np

from oracle.group import group_by_bundle


def test_hand_example():
    label = np.array([2, -1, 0, 2, 5, 0, 1], np.int32)    # B = 3: label 5 is out of range -> unassigned
    dist = np.array([1.5, np.inf, 0.25, 0.5, 2.0, 3.0, 4.0], np.float32)
    r = group_by_bundle(label, dist, 3)
    assert r["order"].tolist() == [2, 5, 6, 0, 3, 1, 4]
    assert r["offsets"].tolist() == [0, 2, 3, 5, 7]
    assert r["dmin"].tolist() == [0.25, 4.0, 0.5] and r["dmax"].tolist() == [3.0, 4.0, 1.5]
    assert r["dsum"].tolist() == [3.25, 4.0, 2.0]


def test_properties_random():
    rng = np.random.default_rng(3)
    for B in (1, 7, 100):
        label = rng.integers(-1, B + 2, 5000).astype(np.int32)
        dist = rng.uniform(0, 10, 5000).astype(np.float32)
        r = group_by_bundle(label, dist, B)
        order, off = r["order"], r["offsets"]
        assert np.array_equal(np.sort(order), np.arange(5000))
        for b in range(B + 1):
            seg = order[off[b]:off[b + 1]]
            want = np.nonzero(label == b)[0] if b < B else np.nonzero((label < 0) | (label >= B))[0]
            assert np.array_equal(seg, want)
            if b < B and seg.size:
                assert r["dmin"][b] == dist[want].min() and r["dmax"][b] == dist[want].max()
        assert off[-1] == 5000
