"""CPU checks of the harness's host-side restatements (config, batching, report metrics)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from paper_2311_17410_b200.harness import (
    RunConfig,
    _fit_or_none,
    _split_batches,
    balance_cv,
    jaccard,
    load_config,
)

REF = "/root/reference/pkg/src"


def test_config_file_and_seed_override(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("generate_nodes = 50\ngenerate_edges = 400\nfanouts = 3,2\ncache_node_policy = lfu\n"
                 "cache_reuse = false\ndirected = yes  # comment\n")
    cfg = load_config(str(p), env={"TG_SEED": "9"})
    assert cfg.generate_nodes == 50 and cfg.fanouts == (3, 2) and cfg.cache.node_policy == "lfu"
    assert cfg.cache.reuse is False and cfg.directed is True and cfg.seed == 9
    p.write_text("bogus = 1\n")
    with pytest.raises(ValueError):
        load_config(str(p), env={})
    with pytest.raises(ValueError):
        RunConfig(initial_fraction=1.0).validate()


def test_split_batches_count_and_time():
    edges = [(i, i + 1, 10 * i) for i in range(25)]
    cfg = RunConfig(initial_fraction=0.2, batch_edges=7)
    init, batches = _split_batches(edges, cfg)
    assert len(init) == 5 and [len(b) for b in batches] == [7, 7, 6]
    cfg = RunConfig(initial_fraction=0.2, batch_by="time", batch_interval=45)
    _, batches = _split_batches(edges, cfg)
    assert sum(len(b) for b in batches) == 20 and all(b[-1][2] - b[0][2] < 45 for b in batches)


def test_report_metrics_basics():
    assert jaccard({1, 2}, {2, 3}) == pytest.approx(1 / 3) and jaccard(set(), set()) == 0.0
    assert _fit_or_none([5, 5, 5]) == (None, None)
    pl, ex = _fit_or_none(list((1000 / np.arange(1, 60) ** 1.5).astype(int) + 1))
    assert pl > 0.9
    assert balance_cv(1, [(0, 1, 0), (2, 3, 1)], False) == (0.0, 0.0)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_helpers_equal_reference():
    sys.path.insert(0, REF)
    from ctdg.harness import RunConfig as RefConfig
    from ctdg.harness import _fit_or_none as ref_fit
    from ctdg.harness import _split_batches as ref_split
    from ctdg.partition import PartitionSpec, balance_stats

    rng = np.random.default_rng(0)
    edges = [(int(a), int(b), int(t)) for a, b, t in zip(rng.integers(0, 40, 500), rng.integers(0, 40, 500),
                                                          np.sort(rng.integers(0, 10_000, 500)))]
    for by in ("count", "time"):
        ours = _split_batches(edges, RunConfig(batch_by=by, batch_edges=37, batch_interval=700))
        theirs = ref_split(edges, RefConfig(batch_by=by, batch_edges=37, batch_interval=700))
        assert ours == theirs
    for p in (1, 2, 3, 4):
        for directed in (True, False):
            st = balance_stats(PartitionSpec(p), edges, directed)
            assert balance_cv(p, edges, directed) == (st.node_cv, st.edge_cv)
    for counts in ([5, 5, 5], [9, 3, 1, 1], list(rng.integers(1, 100, 80))):
        assert _fit_or_none(sorted(counts, reverse=True)) == ref_fit(sorted(counts, reverse=True))
