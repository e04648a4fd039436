"""Adapters used by the -m gpu parity tests (CUDA path vs oracle / golden fixtures)."""

from __future__ import annotations

import numpy as np

import paper_2311_17410_b200 as gf


class GpuGraphAdapter:
    """Wraps gf.DynamicGraph with the array API fixtures.replay_build expects."""

    def __init__(self, directed, tau, sizing="adaptive", param=0):
        sz = {"adaptive": None, "fixed": gf.FixedSizing(max(int(param), 1)), "batch": gf.BatchSizing()}[sizing]
        self.g = gf.DynamicGraph(directed=directed, tau=tau, sizing=sz)

    def add_edges(self, src, dst, ts, edge_ids=None):
        out, _ = self.g.add_edges_arrays(src, dst, ts, edge_ids)
        return out.cpu().numpy()

    def delete_edges(self, ids):
        return self.g.delete_edges(np.asarray(ids, dtype=np.int64))

    def delete_node(self, v):
        return self.g.delete_node(int(v))


def gpu_factory(directed, tau, sizing, param):
    return GpuGraphAdapter(directed, tau, sizing, param)


def export_store(g: gf.DynamicGraph) -> dict:
    f = g.fast
    out = {k: getattr(f, k) for k in ("head", "tail", "num_blocks", "degree", "node_valid", "blk_capacity",
                                       "blk_size", "blk_tmin", "blk_tmax", "blk_prev", "blk_next")}
    arrs = g._block_arrays()
    offs = [0]
    for a, s in zip(arrs, f.blk_size):
        offs.append(offs[-1] + int(s))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    out["slot_offsets"] = np.asarray(offs, np.int64)
    out["slot_nbr"] = cat([a.neighbors[:s] for a, s in zip(arrs, f.blk_size)], np.int64)
    out["slot_eid"] = cat([a.edge_ids[:s] for a, s in zip(arrs, f.blk_size)], np.int64)
    out["slot_ts"] = cat([a.timestamps[:s] for a, s in zip(arrs, f.blk_size)], np.int64)
    out["slot_valid"] = cat([a.valid[:s] for a, s in zip(arrs, f.blk_size)], bool)
    return out


def oracle_store(o) -> dict:
    n = o.export_nodes()
    b = o.export_blocks()
    out = dict(n)
    for ours, theirs in (("capacity", "blk_capacity"), ("size", "blk_size"), ("tmin", "blk_tmin"),
                         ("tmax", "blk_tmax"), ("prev", "blk_prev"), ("next", "blk_next")):
        out[theirs] = b[ours]
    nb, eid, ts, valid, offs = [], [], [], [], [0]
    for h in range(len(b["size"])):
        x = o.block_edges(h)
        nb.append(x[0]); eid.append(x[1]); ts.append(x[2]); valid.append(x[3])
        offs.append(offs[-1] + len(x[0]))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    out.update(slot_offsets=np.asarray(offs, np.int64), slot_nbr=cat(nb, np.int64), slot_eid=cat(eid, np.int64),
               slot_ts=cat(ts, np.int64), slot_valid=cat(valid, bool))
    return out


STORE_KEYS = ("head", "tail", "num_blocks", "degree", "node_valid", "blk_capacity", "blk_size", "blk_tmin",
              "blk_tmax", "blk_prev", "blk_next", "slot_offsets", "slot_nbr", "slot_eid", "slot_ts", "slot_valid")


def assert_store_equal(got: dict, want: dict, msg=""):
    for k in STORE_KEYS:
        np.testing.assert_array_equal(np.asarray(got[k]), np.asarray(want[k]), err_msg=f"{msg} {k}")
