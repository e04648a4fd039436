"""GPU: the ClusterSim facade (cluster.py:160-345) and the device feature-table file paths.

* recent sampling through a 3x2 cluster equals the reference ClusterSim's output bit for bit
  (tests/golden/formats.npz, the unmodified reference on the same inputs);
* every policy through the cluster equals sample_khop on one unpartitioned graph bit for bit
  (the reference's tests/test_cluster.py:62-84 property);
* features fetched through the cluster equal one table's rows; telemetry and static scheduling
  follow cluster.py:91-97,329-345; deletes count ids once (cluster.py:206-224).
"""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest

from format_cases import cluster_case, feature_rows

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "formats.npz"))
RES = json.loads(GOLD["results"].tobytes().decode())


@pytest.mark.parametrize("directed", [True, False])
def test_cluster_recent_equals_reference(cuda_device, directed):
    import paper_2311_17410_b200 as gf

    edges, targets, times, fanouts = cluster_case(directed)
    cl = gf.ClusterSim(gf.ClusterSpec(3, 2), directed=directed, tau=8)
    ids = cl.add_edges(edges)
    want = RES[f"cluster_{int(directed)}"]
    assert ids == want["ids"]
    s = cl.sample_khop(gf.SampleRequest(targets, times, fanouts, gf.SamplingPolicy("recent"), 5), gf.Origin(0, 1))
    assert s.to_json_dict() == want["sample"]
    assert [t.requests_served for _, _, t in cl.all_telemetry()] == want["requests"]


@pytest.mark.parametrize("policy", ["recent", "uniform", "time_window"])
@pytest.mark.parametrize("directed", [True, False])
def test_cluster_equals_local(cuda_device, policy, directed):
    import paper_2311_17410_b200 as gf

    src, dst, ts = gf.generate_synthetic_arrays(400, 30_000, 2.2, 100_000, seed=2)
    edges = list(zip(src.tolist(), dst.tolist(), ts.tolist()))
    cl = gf.ClusterSim(gf.ClusterSpec(4, 2), directed=directed, tau=16)
    local = gf.DynamicGraph(directed=directed, tau=16)
    for lo in range(0, len(edges), 7000):
        cl.add_edges(edges[lo:lo + 7000])
        local.add_edges(edges[lo:lo + 7000])
    pol = gf.SamplingPolicy(policy, 5000 if policy == "time_window" else 0)
    rng = np.random.default_rng(1)
    targets = rng.integers(0, 410, 300).tolist()
    times = rng.integers(0, 110_000, 300).tolist()
    req = gf.SampleRequest(targets, times, [5, 3], pol, 77)
    got = cl.sample_khop(req, gf.Origin(1, 0))
    want = gf.sample_khop(local, req)
    assert got == want
    # rank groups: only rank 0 workers served
    tel = {(m, r): t for m, r, t in cl.all_telemetry()}
    assert all(tel[(m, 1)].requests_served == 0 for m in range(4))
    assert sum(tel[(m, 0)].targets_sampled for m in range(4)) == sum(len(lay.source_nodes) for lay in want.layers)
    assert set(cl.rank_group_cv()) == {0, 1}


def test_cluster_static_scheduling_and_failure(cuda_device):
    import torch

    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200.cluster import LayerRequest

    cl = gf.ClusterSim(gf.ClusterSpec(2, 2), directed=True, tau=4)
    cl.add_edges([(0, 1, 1), (1, 2, 2), (2, 3, 3)])
    w = cl.machines[0].workers[1]
    z = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(AssertionError, match="static scheduling"):
        w.serve_sample(gf.Origin(0, 0), LayerRequest(z, z, z, z, 1, gf.SamplingPolicy("recent"), 0))
    cl.machines[0].workers[0].failed = True
    with pytest.raises(gf.RemoteRequestError):
        cl.sample_khop(gf.SampleRequest([0], [10], [1], gf.SamplingPolicy("recent"), 0), gf.Origin(0, 0))
    assert gf.route(cl.spec, gf.Origin(1, 1), 5) == (1, 1)


def test_cluster_deletes_and_features(cuda_device):
    import paper_2311_17410_b200 as gf

    cl = gf.ClusterSim(gf.ClusterSpec(3, 1), directed=False, tau=4, node_dim=3, edge_dim=2)
    ids = cl.add_edges([(0, 1, 1), (1, 2, 2), (2, 4, 3), (4, 4, 5)])
    assert ids == [0, 1, 2, 3]
    assert cl.add_edges([(5, 0, 9)]) == [4]
    assert cl.delete_edges([1, 3, 99]) == 2  # undirected copies on two machines count once
    assert cl.delete_nodes([2, 77]) == 1
    rows = np.arange(30, dtype=np.float32).reshape(10, 3)
    for m in cl.machines:  # node rows sharded by owner (cluster.py:296-309)
        own = np.arange(m.index, 10, 3)
        m.node_features.set_many(own, rows[own])
    got, found = cl.fetch_node_features([0, 4, 9, 12], gf.Origin(0, 0))
    np.testing.assert_array_equal(got[:3], rows[[0, 4, 9]])
    assert found.tolist() == [True, True, True, False]
    cl.machines[2].edge_features.append([5, 8], np.ones((2, 2), np.float32))
    got, found = cl.fetch_edge_features([5, 8, 5], [2, 5, 0], gf.Origin(0, 0))
    assert found.tolist() == [True, True, False]


@pytest.mark.parametrize("kind", [0, 1])
def test_feature_table_files(cuda_device, kind):
    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200 import features as F

    ids, rows = feature_rows(kind)
    if kind == 0:
        t = gf.NodeFeatureTable(6)
        t.set_many(ids[::-1].copy(), rows[::-1].copy())
        assert int(ids[3]) in t and 10_001 not in t
        np.testing.assert_array_equal(t.ids_sorted(), ids)
        buf = io.BytesIO()
        F.save_node_features(t, buf)
    else:
        t = gf.EdgeFeatureTable(6)
        t.append(ids[:20], rows[:20])
        t.append(ids[20:], rows[20:])
        np.testing.assert_array_equal(t.ids, ids)
        np.testing.assert_array_equal(t.values, rows)
        buf = io.BytesIO()
        F.save_edge_features(t, buf)
    assert buf.getvalue() == GOLD["tgff_node" if kind == 0 else "tgff_edge"].tobytes()
    back = F.load_feature_table(io.BytesIO(buf.getvalue()))
    assert type(back) is type(t) and len(back) == len(ids)
    got, found = back.get(np.concatenate([ids, [10_005]]))
    np.testing.assert_array_equal(got[:-1], rows)
    assert found.tolist() == [True] * len(ids) + [False]


def test_node_memory_table(cuda_device):
    import paper_2311_17410_b200 as gf

    m = gf.NodeMemoryTable(4)
    m.update([3, 1], np.ones((2, 4), np.float32), [10, 20])
    m.update([3], np.full((1, 4), 2, np.float32), [30])
    rows, found = m.get([1, 3, 5])
    assert found.tolist() == [True, True, False]
    assert rows[1].tolist() == [2, 2, 2, 2] and m.last_update == {3: 30, 1: 20} and len(m) == 2
    with pytest.raises(ValueError):
        m.update([1], np.ones((1, 3), np.float32), [1])
