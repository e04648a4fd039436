"""K2/K3 parity: the CUDA temporal sampler vs the reference fixtures and the oracle.

recent: bit-exact (offsets, neighbours, edge ids, timestamps) against the
reference's own outputs and the oracle.  uniform/time_window: bit-exact
against the oracle's identical Philox+Floyd stream, exact multisets at
complete fanout against the reference, and the reference's 4-sigma frequency
test (tests/test_sampling.py:93-105).
"""

from __future__ import annotations

from collections import Counter

import numpy as np
import pytest

from fixtures import TS_MIN, load, replay_build

pytestmark = pytest.mark.gpu


def _host(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def test_recent_matches_reference_fixtures(cuda_device):
    import paper_2311_17410_b200 as gf
    from gpu_helpers import gpu_factory

    fx, meta = load("sample_cases.npz")
    for m in meta:
        p = f"s{m['id']}/"
        g, _ = replay_build(gpu_factory, fx, p, {**m, "sizing": "adaptive", "param": 0})
        for f in (1, 3, 10):
            lay = gf.sample_layer(g.g, fx[p + "q_src"], fx[p + "q_t0"], fx[p + "q_t1"], f, gf.SamplingPolicy.recent(), 0)
            for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
                np.testing.assert_array_equal(getattr(lay, nm), fx[p + f"recent_f{f}_{nm}"], err_msg=f"{p} f{f} {nm}")
        req = gf.SampleRequest(fx[p + "khop_roots"].tolist(), fx[p + "khop_ts"].tolist(), [4, 3], gf.SamplingPolicy.recent())
        lays = gf.sample_khop(g.g, req).layers
        for h, lay in enumerate(lays):
            for nm in ("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps"):
                np.testing.assert_array_equal(getattr(lay, nm), fx[p + f"khop{h}_{nm}"], err_msg=f"{p} hop{h} {nm}")


@pytest.mark.parametrize("kind", ["full", "tw"])
def test_complete_fanout_multisets_match_reference(cuda_device, kind):
    import paper_2311_17410_b200 as gf
    from gpu_helpers import gpu_factory

    fx, meta = load("sample_cases.npz")
    for m in meta:
        p = f"s{m['id']}/"
        g, _ = replay_build(gpu_factory, fx, p, {**m, "sizing": "adaptive", "param": 0})
        pol = gf.SamplingPolicy.uniform() if kind == "full" else gf.SamplingPolicy.time_window(m["tw_delta"])
        lay = gf.sample_layer(g.g, fx[p + "q_src"], fx[p + "q_t0"], fx[p + "q_t1"], 10**9, pol, seed=5)
        np.testing.assert_array_equal(lay.offsets, fx[p + f"{kind}_offsets"])
        for i in range(len(lay.offsets) - 1):
            a = slice(lay.offsets[i], lay.offsets[i + 1])
            got = Counter(zip(lay.neighbors[a].tolist(), lay.edge_ids[a].tolist(), lay.timestamps[a].tolist()))
            want = Counter(zip(fx[p + f"{kind}_neighbors"][a].tolist(), fx[p + f"{kind}_edge_ids"][a].tolist(),
                               fx[p + f"{kind}_timestamps"][a].tolist()))
            assert got == want


def _random_graph_pair(rng, directed, tau, n_nodes, m, deletions):
    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    g = gf.DynamicGraph(directed=directed, tau=tau)
    o = OracleGraph(directed, tau)
    src = rng.integers(0, n_nodes, m); dst = rng.integers(0, n_nodes, m)
    ts = np.sort(rng.integers(0, 5 * m, m))
    for chunk in np.array_split(np.arange(m), 3):
        if len(chunk):
            g.add_edges_arrays(src[chunk], dst[chunk], ts[chunk])
            o.add_edges(src[chunk], dst[chunk], ts[chunk])
    if deletions:
        dels = rng.choice(m, size=m // 7, replace=False)
        assert g.delete_edges(dels) == o.delete_edges(dels)
        for v in rng.choice(n_nodes, size=2, replace=False).tolist():
            assert g.delete_node(v) == o.delete_node(v)
    return g, o, ts


@pytest.mark.parametrize("policy", ["recent", "uniform", "time_window"])
@pytest.mark.parametrize("deletions", [False, True])
def test_layer_bitwise_vs_oracle(cuda_device, policy, deletions):
    import paper_2311_17410_b200 as gf

    rng = np.random.default_rng(100 + deletions)
    for case in range(6):
        directed = bool(case % 2)
        tau = int(rng.choice([1, 2, 4, 16, 48, 512]))
        g, o, ts = _random_graph_pair(rng, directed, tau, int(rng.integers(3, 200)), int(rng.integers(50, 6000)),
                                      deletions)
        nq = 3000
        q = rng.integers(-2, g.num_nodes + 2, nq)
        t1 = rng.integers(-5, int(ts[-1]) + 10, nq)
        t0 = np.where(rng.random(nq) < 0.5, TS_MIN, t1 - rng.integers(0, int(ts[-1]) + 1, nq))
        delta = max(1, int(ts[-1]) // 5)
        pol = gf.SamplingPolicy(policy, delta if policy == "time_window" else 0)
        for f in (1, 5, 10, 15, 16, 17, 32, 40):  # fused path up to 16, unfused above
            lay = gf.sample_layer(g, q, t0, t1, f, pol, seed=1234 + f)
            want = o.sample_layer(q, t0, t1, f, policy, delta, seed=1234 + f)
            for nm, w in zip(("offsets", "neighbors", "edge_ids", "timestamps"), want):
                np.testing.assert_array_equal(getattr(lay, nm), w, err_msg=f"case {case} f{f} {nm}")


@pytest.mark.parametrize("policy", ["recent", "uniform", "time_window"])
def test_ingest_after_deletions_bitwise_vs_oracle(cuda_device, policy):
    """Deletions, then more batches (some edges into the deleted nodes), then sampling: the candidate
    bitmap the post-deletion sampler reads is kept current by ingest and rebuilt by every delete."""
    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    rng = np.random.default_rng(77)
    for case in range(4):
        directed = bool(case % 2)
        tau = int(rng.choice([1, 4, 48, 512]))
        n_nodes, m = int(rng.integers(20, 300)), int(rng.integers(2000, 8000))
        g = gf.DynamicGraph(directed=directed, tau=tau)
        o = OracleGraph(directed, tau)
        src = rng.integers(0, n_nodes, m); dst = rng.integers(0, n_nodes, m)
        ts = np.sort(rng.integers(0, 5 * m, m))
        cut = [0, m // 3, 2 * m // 3, m]
        for b in range(3):
            sl = slice(cut[b], cut[b + 1])
            g.add_edges_arrays(src[sl], dst[sl], ts[sl])
            o.add_edges(src[sl], dst[sl], ts[sl])
            if b < 2:  # delete between batches: later batches append behind the deletions
                dels = rng.choice(cut[b + 1], size=cut[b + 1] // 9, replace=False)
                assert g.delete_edges(dels) == o.delete_edges(dels)
                v = int(rng.integers(0, n_nodes))
                assert g.delete_node(v) == o.delete_node(v)
        nq = 4000
        q = rng.integers(0, g.num_nodes, nq)
        t1 = rng.integers(0, int(ts[-1]) + 10, nq)
        t0 = np.where(rng.random(nq) < 0.5, TS_MIN, t1 - rng.integers(0, int(ts[-1]) + 1, nq))
        delta = max(1, int(ts[-1]) // 5)
        pol = gf.SamplingPolicy(policy, delta if policy == "time_window" else 0)
        for f in (1, 7, 10, 16):
            lay = gf.sample_layer(g, q, t0, t1, f, pol, seed=99 + f)
            want = o.sample_layer(q, t0, t1, f, policy, delta, seed=99 + f)
            for nm, w in zip(("offsets", "neighbors", "edge_ids", "timestamps"), want):
                np.testing.assert_array_equal(getattr(lay, nm), w, err_msg=f"case {case} f{f} {nm}")


@pytest.mark.parametrize("policy", ["recent", "uniform"])
def test_khop_bitwise_vs_oracle_and_sharding_invariance(cuda_device, policy):
    import torch

    import paper_2311_17410_b200 as gf

    rng = np.random.default_rng(7)
    src, dst, ts = gf.generate_synthetic_arrays(2000, 200_000, 2.2, 175_200, seed=1, src_skew=2.2)
    from oracle import OracleGraph

    g = gf.DynamicGraph(directed=True, tau=8192)
    o = OracleGraph(True, 8192)
    for lo in range(0, len(src), 50_000):
        g.add_edges_arrays(src[lo:lo + 50_000], dst[lo:lo + 50_000], ts[lo:lo + 50_000])
        o.add_edges(src[lo:lo + 50_000], dst[lo:lo + 50_000], ts[lo:lo + 50_000])
    roots = np.concatenate([src[-2000:], dst[-2000:]])
    rts = np.concatenate([ts[-2000:], ts[-2000:]])
    pick = rng.choice(len(src), 2000, replace=False)
    roots = np.concatenate([roots, src[pick]]); rts = np.concatenate([rts, ts[pick]])
    dev = torch.device("cuda:0")
    full = gf.TemporalSampler(g, [10, 10], policy, seed=3).sample(torch.from_numpy(roots).to(dev),
                                                                 torch.from_numpy(rts).to(dev))
    want = o.sample_khop(roots, rts, [10, 10], policy, seed=3, threads=8)
    for lay, ref in zip(full.layers, want):
        for nm, w in zip(("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps"), ref):
            np.testing.assert_array_equal(_host(getattr(lay, nm)), w, err_msg=nm)
    # the same roots split in 3 shards with their global key bases reproduce the full sample
    parts = np.array_split(np.arange(len(roots)), 3)
    for h in range(2):
        cat = []
        for part in parts:
            sub = gf.TemporalSampler(g, [10, 10], policy, seed=3).sample(
                torch.from_numpy(roots[part]).to(dev), torch.from_numpy(rts[part]).to(dev),
                root_key_base=int(part[0]))
            cat.append(_host(sub.layers[h].neighbors))
        np.testing.assert_array_equal(np.concatenate(cat), _host(full.layers[h].neighbors))


def test_uniform_frequencies_within_4_sigma(cuda_device):
    """Reference tests/test_sampling.py:93-105 on the GPU sampler."""
    import paper_2311_17410_b200 as gf

    g = gf.new_graph(directed=True)
    g.add_edges([(0, i + 1, i) for i in range(20)])
    reps, f, n = 10_000, 5, 20
    counts = Counter()
    for seed in range(reps):
        counts.update(gf.sample_layer(g, [0], [TS_MIN], [100], f, gf.SamplingPolicy.uniform(), seed=seed).neighbors.tolist())
    p = f / n
    sigma = (p * (1 - p) / reps) ** 0.5
    for nbr in range(1, n + 1):
        assert abs(counts[nbr] / reps - p) <= 4 * sigma, nbr


def test_uniform_inclusion_chi2_vs_reference_distribution(cuda_device):
    """Many queries on one hub: per-candidate inclusion counts are uniform (chi^2)."""
    import torch
    from scipy.stats import chisquare

    import paper_2311_17410_b200 as gf

    g = gf.new_graph(directed=True)
    n = 300
    g.add_edges([(0, i + 1, i) for i in range(n)])
    q = 20_000
    dev = torch.device("cuda:0")
    lay = gf.sample_layer(g, torch.zeros(q, dtype=torch.int64, device=dev),
                          torch.full((q,), TS_MIN, dtype=torch.int64, device=dev),
                          torch.full((q,), 10**6, dtype=torch.int64, device=dev), 10, gf.SamplingPolicy.uniform(), seed=11)
    nb = _host(lay.neighbors)
    assert len(nb) == 10 * q
    offs = _host(lay.offsets)
    for i in range(0, q, 997):  # no duplicates inside a query
        s = nb[offs[i]:offs[i + 1]]
        assert len(set(s.tolist())) == len(s)
    cnt = np.bincount(nb, minlength=n + 1)[1:]
    assert chisquare(cnt).pvalue > 1e-4


def test_reference_semantics_goldens(cuda_device):
    """Reference tests/test_sampling.py:44-62,137-167,189-214,245-260 on the GPU path."""
    import paper_2311_17410_b200 as gf

    g = gf.new_graph(directed=False, tau=48)
    A, B, C, D = 0, 1, 2, 3
    g.add_edges([(A, C, 12), (B, C, 14), (C, D, 16), (A, C, 23)])
    lay = gf.sample_layer(g, [A], [TS_MIN], [24], 10, gf.SamplingPolicy.recent(), seed=0)
    assert lay.neighbors.tolist() == [C, C] and sorted(lay.timestamps.tolist()) == [12, 23]
    s = gf.sample_khop(g, gf.SampleRequest([A], [24], [10, 10], gf.SamplingPolicy.recent(), seed=0))
    hop2 = s.layers[1]
    by = {(int(hop2.source_nodes[i]), int(hop2.source_times[i])): sorted(hop2.neighbors[hop2.slice_of(i)].tolist())
          for i in range(len(hop2.source_nodes))}
    assert by[(C, 23)] == [A, B, D] and by[(C, 12)] == []
    assert gf.sample_khop(g, gf.SampleRequest([0], [24], [], gf.SamplingPolicy.recent())).layers == []
    assert gf.random_walk(g, A, 23, 1, gf.SamplingPolicy.recent()) == [(C, 12)]
    assert gf.random_walk(g, B, 14, 3, gf.SamplingPolicy.recent()) == []
    with pytest.raises(ValueError):
        gf.sample_layer(g, [0, 1], [0], [10, 10], 1, gf.SamplingPolicy.recent(), seed=0)
    with pytest.raises(ValueError):
        gf.sample_khop(g, gf.SampleRequest([0], [1], [0], gf.SamplingPolicy.recent()))
    g2 = gf.new_graph(directed=True)
    ids = g2.add_edges([(0, 1, 1), (0, 2, 5), (0, 3, 9)]).accepted_ids
    assert sorted(gf.sample_layer(g2, [0], [TS_MIN], [10], 10**9, gf.SamplingPolicy.time_window(5), 0).timestamps.tolist()) == [5, 9]
    g2.delete_edges([ids[1]])
    assert sorted(gf.sample_layer(g2, [0], [0], [10], 10**9, gf.SamplingPolicy.recent(), 0).timestamps.tolist()) == [1, 9]
    assert gf.sample_layer(g2, [0, 99], [0, 0], [10, 10], 10**9, gf.SamplingPolicy.recent(), 0).offsets.tolist() == [0, 2, 2]
    g3 = gf.new_graph(directed=False)
    g3.add_edges([(0, 1, 1), (0, 2, 2)])
    g3.delete_node(1)
    assert gf.sample_layer(g3, [1], [0], [10], 10**9, gf.SamplingPolicy.recent(), 0).offsets.tolist() == [0, 0]
    assert gf.sample_layer(g3, [0], [0], [10], 10**9, gf.SamplingPolicy.recent(), 0).neighbors.tolist() == [2]


def test_temporal_sampler_north_star_form(cuda_device):
    """TemporalSampler.sample(roots, ts, fanouts, strategy) == the constructor-configured form."""
    import torch

    import paper_2311_17410_b200 as gf

    src, dst, ts = gf.generate_synthetic_arrays(500, 30_000, 2.2, 50_000, seed=4, src_skew=2.2)
    g = gf.DynamicGraph(directed=True, tau=64)
    g.add_edges_arrays(src, dst, ts)
    roots = torch.from_numpy(np.concatenate([src[-300:], dst[-300:]])).cuda()
    rts = torch.from_numpy(np.concatenate([ts[-300:], ts[-300:]])).cuda()
    base = gf.TemporalSampler(g, [5], "recent", seed=2)
    for fo, strat in (([10, 10], "uniform"), ([3], "recent"), ([4, 2], "uniform")):
        a = base.sample(roots, rts, fo, strat)
        b = gf.TemporalSampler(g, fo, strat, seed=2).sample(roots, rts)
        assert len(a.layers) == len(fo)
        for la, lb in zip(a.layers, b.layers):
            for x, y in zip((la.offsets, la.neighbors, la.edge_ids, la.timestamps),
                            (lb.offsets, lb.neighbors, lb.edge_ids, lb.timestamps)):
                assert torch.equal(x, y)


@pytest.mark.parametrize("fanouts", [[15, 10], [3, 5, 2]])
def test_khop_time_window_and_wide_fanouts_vs_oracle(cuda_device, fanouts):
    """Multi-hop time-window and uniform sampling (MAG-style [15, 10], three hops) bit-exact vs the oracle."""
    import torch

    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    src, dst, ts = gf.generate_synthetic_arrays(3000, 120_000, 2.2, 120, seed=9, src_skew=2.2)  # MAG-like ties
    g = gf.DynamicGraph(directed=True, tau=8192)
    o = OracleGraph(True, 8192)
    for lo in range(0, len(src), 40_000):
        g.add_edges_arrays(src[lo:lo + 40_000], dst[lo:lo + 40_000], ts[lo:lo + 40_000])
        o.add_edges(src[lo:lo + 40_000], dst[lo:lo + 40_000], ts[lo:lo + 40_000])
    rng = np.random.default_rng(3)
    pick = rng.integers(0, len(src), 2000)
    roots = np.concatenate([src[pick], dst[pick]])
    rts = np.concatenate([ts[pick], ts[pick] + 1])
    for policy, delta in (("uniform", 0), ("time_window", 30)):
        req = gf.SampleRequest(torch.from_numpy(roots).cuda(), torch.from_numpy(rts).cuda(), fanouts,
                               gf.SamplingPolicy(policy, delta), seed=11)
        got = gf.sample_khop(g, req)
        ref = o.sample_khop(roots, rts, fanouts, policy, delta=delta, seed=11)
        assert len(got.layers) == len(ref)
        for lay, r in zip(got.layers, ref):
            for a, w in zip((lay.offsets, lay.neighbors, lay.edge_ids, lay.timestamps), (r[2], r[3], r[4], r[5])):
                np.testing.assert_array_equal(a.cpu().numpy(), w)


@pytest.mark.parametrize("tau", [1, 2, 4, 48, 8192])
def test_recent_khop_duplicate_heavy_roots_bitwise(cuda_device, tau):
    """The recent policy's per-call boundary memo (gf_sample.cu RecentMemo): roots repeat the same
    (node, t_end) pairs many times, block sizes range from 1 slot (tau 1: every hop-2+ selection
    crosses blocks) to 8192, and the fanout changes per hop ([3, 16, 7]) so memo entries written
    under one fanout are reused under another -- bitwise vs the oracle, hop by hop."""
    import torch

    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    src, dst, ts = gf.generate_synthetic_arrays(300, 40_000, 2.2, 2_000, seed=8, src_skew=2.2)
    g = gf.DynamicGraph(directed=True, tau=tau)
    o = OracleGraph(True, tau)
    for lo in range(0, len(src), 10_000):
        g.add_edges_arrays(src[lo:lo + 10_000], dst[lo:lo + 10_000], ts[lo:lo + 10_000])
        o.add_edges(src[lo:lo + 10_000], dst[lo:lo + 10_000], ts[lo:lo + 10_000])
    rng = np.random.default_rng(tau)
    base = np.concatenate([src[-300:], dst[-300:], np.arange(-2, 302)])
    bts = np.concatenate([ts[-300:], ts[-300:], rng.integers(-5, 2_010, 304)])
    pick = rng.integers(0, len(base), 6_000)
    roots, rts = base[pick], bts[pick]
    dev = torch.device("cuda:0")
    got = gf.TemporalSampler(g, [3, 16, 7], "recent").sample(torch.from_numpy(roots).to(dev),
                                                           torch.from_numpy(rts).to(dev))
    want = o.sample_khop(roots, rts, [3, 16, 7], "recent", threads=8)
    for h, (lay, ref) in enumerate(zip(got.layers, want)):
        for nm, w in zip(("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps"), ref):
            np.testing.assert_array_equal(_host(getattr(lay, nm)), w, err_msg=f"hop{h} {nm}")
    # sample_layer without t_starts (all TS_MIN) also takes the memo path
    lay = gf.sample_layer(g, torch.from_numpy(roots).to(dev), torch.full((len(roots),), TS_MIN, device=dev),
                          torch.from_numpy(rts).to(dev), 10, gf.SamplingPolicy.recent(), 0)
    w = o.sample_layer(roots, np.full(len(roots), TS_MIN), rts, 10, "recent")
    for nm, ww in zip(("offsets", "neighbors", "edge_ids", "timestamps"), w):
        np.testing.assert_array_equal(_host(getattr(lay, nm)), ww)


@pytest.mark.parametrize("policy", ["uniform", "time_window"])
def test_general_path_long_windows_rejection_and_fallback_bitwise(cuda_device, policy):
    """Post-deletion uniform selection over windows of > 64 positions (gf_sample.cu GEN_EXACT):
    rejection draws over the positions when deletions are sparse, the exact count + Floyd
    fallback when most candidates are invalid (a deleted neighbour holding 95% of a hub's
    edges) -- bitwise vs the oracle, which makes the same decisions."""
    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    rng = np.random.default_rng(31)
    n_hub, m = 6, 60_000
    src = rng.integers(0, n_hub, m)
    dst = np.where(rng.random(m) < 0.95, n_hub, rng.integers(n_hub + 1, n_hub + 400, m))  # node n_hub dominates
    ts = np.sort(rng.integers(0, 50_000, m))
    g = gf.DynamicGraph(directed=True, tau=512)
    o = OracleGraph(True, 512)
    for lo in range(0, m, 20_000):
        g.add_edges_arrays(src[lo:lo + 20_000], dst[lo:lo + 20_000], ts[lo:lo + 20_000])
        o.add_edges(src[lo:lo + 20_000], dst[lo:lo + 20_000], ts[lo:lo + 20_000])
    dels = rng.choice(m, m // 50, replace=False)
    assert g.delete_edges(dels) == o.delete_edges(dels)
    q = np.repeat(np.arange(n_hub), 400)
    t1 = rng.integers(10_000, 50_010, len(q))
    t0 = np.full(len(q), TS_MIN)
    delta = 40_000
    pol = gf.SamplingPolicy(policy, delta if policy == "time_window" else 0)
    for case in ("sparse", "dominant_neighbour_deleted"):
        if case == "dominant_neighbour_deleted":
            assert g.delete_node(n_hub) == o.delete_node(n_hub)
        for f in (1, 10, 25):
            lay = gf.sample_layer(g, q, t0, t1, f, pol, seed=77 + f)
            want = o.sample_layer(q, t0, t1, f, policy, delta, seed=77 + f)
            for nm, w in zip(("offsets", "neighbors", "edge_ids", "timestamps"), want):
                np.testing.assert_array_equal(getattr(lay, nm), w, err_msg=f"{case} f{f} {nm}")
            if case == "dominant_neighbour_deleted":
                assert not np.isin(lay.neighbors, [n_hub]).any()
