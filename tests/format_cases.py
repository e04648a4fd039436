"""Seeded inputs shared by tests/golden/make_golden_formats.py (which runs the reference on
them) and tests/test_formats.py / tests/test_gpu_cluster.py (which run this package on them)."""

from __future__ import annotations

import numpy as np


def wire_messages():
    """(request id, message class name, fields) for every TGRP message type and edge cases."""
    rng = np.random.default_rng(11)
    n = 7
    out = [
        (1, "SampleRequestMsg", dict(targets=rng.integers(0, 1 << 40, n), timestamps=rng.integers(-5, 1 << 50, n),
                                     t_starts=np.full(n, np.iinfo(np.int64).min), fanout=10, policy_kind="uniform",
                                     delta=0, seed=(1 << 64) - 3)),
        (2, "SampleRequestMsg", dict(targets=np.zeros(0, np.int64), timestamps=np.zeros(0, np.int64),
                                     t_starts=np.zeros(0, np.int64), fanout=1, policy_kind="time_window", delta=9,
                                     seed=-1)),
        (3, "SampleResponseMsg", dict(offsets=np.array([0, 2, 2, 5]), neighbors=rng.integers(0, 1000, 5),
                                      edge_ids=rng.integers(0, 1 << 33, 5), timestamps=rng.integers(-9, 1 << 45, 5))),
        (1 << 63, "FeatureRequestMsg", dict(kind=2, ids=rng.integers(0, 1 << 62, 4))),
        (4, "FeatureResponseMsg", dict(dim=3, found=np.array([True, False, True]),
                                       rows=rng.random((3, 3), dtype=np.float32))),
        (5, "FeatureResponseMsg", dict(dim=0, found=np.array([False, True]), rows=np.zeros((2, 0), np.float32))),
        (6, "ErrorMsg", dict(code=7, message="worker failed: é")),
    ]
    return out


def feature_rows(kind: int):
    rng = np.random.default_rng(20 + kind)
    ids = np.sort(rng.choice(10_000, 50, replace=False)).astype(np.int64)
    return ids, rng.random((50, 6), dtype=np.float32)


def metric_inputs():
    return [[5, 1, 0, 9, 3, 3, 2], [4, 4, 4], [0, 0], [1, 2], list(range(1, 40)), []]


def partition_edges():
    rng = np.random.default_rng(3)
    src = rng.integers(0, 40, 300)
    dst = rng.integers(0, 40, 300)
    ts = np.sort(rng.integers(0, 1000, 300))
    return list(zip(src.tolist(), dst.tolist(), ts.tolist()))


def cluster_case(directed: bool):
    rng = np.random.default_rng(7 + int(directed))
    m = 2000
    src = rng.integers(0, 120, m)
    dst = rng.integers(0, 120, m)
    ts = np.sort(rng.integers(0, 5000, m))
    edges = list(zip(src.tolist(), dst.tolist(), ts.tolist()))
    targets = rng.integers(0, 125, 40).tolist()
    times = rng.integers(0, 5200, 40).tolist()
    return edges, targets, times, [4, 3]
