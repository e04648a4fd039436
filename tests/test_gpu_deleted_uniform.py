"""The post-deletion uniform selection draws a uniform k-subset of the valid candidates.

After deletions the sampler's uniform / time-window selection is this implementation's own procedure
(k_sample_fused_del): Floyd's k positions of the window with the valid ones kept, topped
up by rejection draws over the window, an exact count + Floyd over the valid ranks when the draws run
out, and a validity mask for windows of <= 64 positions.  The parity tests pin it bit for bit to the
oracle; this module checks the law the reference specifies (sampling.py:191-198: k distinct valid
candidates, each with inclusion probability k / n): many identical queries, each with its own query
key, on one node whose list has deleted edges and edges into a deleted node.
"""

from __future__ import annotations

import numpy as np
import pytest
from scipy import stats

from fixtures import TS_MIN

pytestmark = pytest.mark.gpu

P_MIN = 1e-4


def _one_node_graph(n_edges: int, del_frac: float, seed: int):
    import paper_2311_17410_b200 as gf

    rng = np.random.default_rng(seed)
    g = gf.DynamicGraph(directed=True, tau=16)
    src = np.zeros(n_edges, np.int64)
    dst = rng.integers(1, 40, n_edges).astype(np.int64)
    ts = np.arange(n_edges, dtype=np.int64) * 3
    g.add_edges_arrays(src, dst, ts)
    eids = np.arange(n_edges)
    dels = rng.choice(n_edges, size=int(del_frac * n_edges), replace=False)
    if len(dels):
        g.delete_edges(dels)
    g.delete_node(7)  # edges into node 7 stop being candidates
    valid = np.ones(n_edges, bool)
    valid[dels] = False
    valid[dst == 7] = False
    return g, eids[valid], ts


@pytest.mark.parametrize("n_edges,del_frac,fanout", [(400, 0.2, 10), (300, 0.9, 10), (50, 0.3, 7), (1000, 0.05, 16)])
@pytest.mark.parametrize("policy", ["uniform", "time_window"])
def test_post_deletion_uniform_law(cuda_device, n_edges, del_frac, fanout, policy):
    import paper_2311_17410_b200 as gf

    g, valid_eids, ts = _one_node_graph(n_edges, del_frac, seed=n_edges + fanout)
    reps = 20_000
    t_end = int(ts[-1]) + 1
    delta = t_end + 10  # the window covers the whole list
    pol = gf.SamplingPolicy(policy, delta if policy == "time_window" else 0)
    lay = gf.sample_layer(g, np.zeros(reps, np.int64), np.full(reps, TS_MIN, np.int64), np.full(reps, t_end, np.int64),
                          fanout, pol, seed=5)
    offs = np.asarray(lay.offsets.cpu() if hasattr(lay.offsets, "cpu") else lay.offsets)
    eid = np.asarray(lay.edge_ids.cpu() if hasattr(lay.edge_ids, "cpu") else lay.edge_ids)
    nv = len(valid_eids)
    k = min(fanout, nv)
    assert np.all(np.diff(offs) == k)
    picks = eid.reshape(reps, k)
    # only valid candidates, k distinct per query
    assert np.isin(picks, valid_eids).all()
    assert all(len(set(r)) == k for r in picks[:2000].tolist())
    if k == nv:
        return
    # inclusion counts: each valid candidate in reps * k / nv queries
    counts = np.bincount(np.searchsorted(valid_eids, picks.ravel()), minlength=nv)
    expected = np.full(nv, reps * k / nv)
    assert stats.chisquare(counts, expected).pvalue > P_MIN
