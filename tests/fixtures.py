"""Loaders for the golden fixtures produced by tests/golden/make_golden.py."""

from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TS_MIN = int(np.iinfo(np.int64).min)


@lru_cache(maxsize=None)
def load(name: str):
    d = np.load(os.path.join(GOLDEN, name))
    data = {k: d[k] for k in d.files}
    meta = json.loads(bytes(data.pop("meta")).decode()) if "meta" in data else None
    return data, meta


@lru_cache(maxsize=None)
def misc() -> dict:
    with open(os.path.join(GOLDEN, "misc.json")) as fh:
        return json.load(fh)


def replay_build(make_graph, fx: dict, p: str, m: dict):
    """Rebuild a fixture graph with ``make_graph(directed, tau, sizing, param)``.

    The returned object must offer add_edges(src, dst, ts, edge_ids) -> eids
    array (-1 = rejected), delete_edges(ids), delete_node(v).
    Returns (graph, concatenated eids).
    """
    g = make_graph(m["directed"], m["tau"], m.get("sizing", "adaptive"), m.get("param", 0))
    src, dst, ts = fx[p + "src"], fx[p + "dst"], fx[p + "ts"]
    eids_in = fx.get(p + "eids_in")
    if eids_in is not None and len(eids_in) == 0:
        eids_in = None
    out, pos = [], 0
    for b in fx[p + "batches"].tolist():
        if b == 0:
            continue
        sl = slice(pos, pos + b)
        out.append(np.asarray(g.add_edges(src[sl], dst[sl], ts[sl], None if eids_in is None else eids_in[sl])))
        pos += b
    dele = fx.get(p + "del_edges")
    if dele is not None and len(dele):
        g.delete_edges(dele)
    deln = fx.get(p + "del_nodes")
    if deln is not None:
        for v in deln.tolist():
            g.delete_node(v)
    return g, (np.concatenate(out) if out else np.zeros(0, np.int64))


def replay_offload_case(graph, fx: dict, p: str, m: dict):
    """Replay an offload fixture (tests/golden/make_golden.py offload_cases) on ``graph``.

    ``graph`` offers add_edges(src, dst, ts) -> eids, delete_edges(ids) and
    offload(cutoff) -> (blob bytes, n records).  Yields (what, step, got, want).
    """
    for step in range(3):
        eids = graph.add_edges(fx[p + f"{step}_src"], fx[p + f"{step}_dst"], fx[p + f"{step}_ts"])
        yield "eids", step, np.asarray(eids), fx[p + f"{step}_eids"]
        if step < 2:
            if p + f"{step}_del" in fx:
                graph.delete_edges(fx[p + f"{step}_del"])
            blob, n = graph.offload(m["steps"][step]["cutoff"])
            yield "blob", step, np.frombuffer(blob, np.uint8), fx[p + f"{step}_blob"]
            yield "n", step, n, m["steps"][step]["n"]


def live_layout_from(nodes: dict, blocks: dict, slot_fn, live) -> dict:
    """Live-handle layout (node columns, block columns and slots of `live` handles)."""
    out = {k: nodes[k] for k in ("head", "tail", "num_blocks", "degree", "node_valid")}
    for ours, theirs in (("capacity", "blk_capacity"), ("size", "blk_size"), ("tmin", "blk_tmin"),
                         ("tmax", "blk_tmax"), ("prev", "blk_prev"), ("next", "blk_next")):
        out[theirs] = blocks[ours][live] if len(live) else np.zeros(0, np.int64)
    cols = {"nbr": [], "eid": [], "ts": [], "valid": []}
    offs = [0]
    for h in live:
        nbr, eid, ts, valid = slot_fn(int(h))
        cols["nbr"].append(nbr); cols["eid"].append(eid); cols["ts"].append(ts); cols["valid"].append(valid)
        offs.append(offs[-1] + len(nbr))
    out["slot_offsets"] = np.asarray(offs, np.int64)
    for k, dt in (("nbr", np.int64), ("eid", np.int64), ("ts", np.int64), ("valid", bool)):
        out["slot_" + k] = np.concatenate(cols[k]).astype(dt) if cols[k] else np.zeros(0, dt)
    return out
