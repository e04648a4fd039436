"""Continuous-learning loop on the GPU: RoundReports equal the reference's modulo wall clock.

Fixtures: tests/golden/harness_reports.json, made by the unmodified reference
run_continuous (recent policy) for three configurations (LRU/LFU/FIFO caches,
reuse/restore on and off, replay, count- and time-based batches, memory).
"""

from __future__ import annotations

import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "harness_reports.json")


def _configs():
    with open(GOLDEN) as fh:
        return json.load(fh)


@pytest.mark.parametrize("key", ["0", "1", "2"])
def test_round_reports_match_reference(cuda_device, key):
    from paper_2311_17410_b200.harness import CacheConfig, RoundReport, RunConfig, reports_equal_modulo_time, run_continuous

    entry = _configs()[key]
    kw = dict(entry["config"])
    cache = CacheConfig(**kw.pop("cache", {}))
    if "fanouts" in kw:
        kw["fanouts"] = tuple(kw["fanouts"])
    cfg = RunConfig(**kw, cache=cache)
    got = list(run_continuous(cfg))
    want = [RoundReport.from_json(line) for line in entry["reports"]]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert reports_equal_modulo_time(g, w), (g, w)
