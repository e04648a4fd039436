"""CPU: TGRP frames, TGFF files, metrics and partition helpers vs the reference's own outputs
(tests/golden/formats.npz, written by tests/golden/make_golden_formats.py)."""

from __future__ import annotations

import io
import json
import os
import struct

import numpy as np
import pytest

from format_cases import feature_rows, metric_inputs, partition_edges, wire_messages
from paper_2311_17410_b200 import metrics, partition, wire
from paper_2311_17410_b200.features import (KIND_EDGE, KIND_NODE, FeatureFormatError, load_features,
                                            load_features_csv, save_features)

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "formats.npz"))
RES = json.loads(GOLD["results"].tobytes().decode())


def _msg(kind, d):
    return getattr(wire, kind)(**d)


@pytest.mark.parametrize("i", range(len(wire_messages())))
def test_wire_bytes_equal_reference(i):
    rid, kind, d = wire_messages()[i]
    frame = wire.encode_message(rid, _msg(kind, d))
    assert frame == GOLD[f"wire_{i}"].tobytes()
    got_id, back = wire.decode_message(frame)
    assert got_id == rid and type(back).__name__ == kind
    assert wire.encode_message(rid, back) == frame


def test_wire_decoded_types():
    _, req = wire.decode_message(GOLD["wire_0"].tobytes())
    assert req.targets.dtype == np.int64 and req.policy_kind == "uniform" and req.seed == (1 << 64) - 3
    _, resp = wire.decode_message(GOLD["wire_2"].tobytes())
    assert resp.offsets.dtype == np.int64 and resp.offsets.tolist() == [0, 2, 2, 5]
    _, fr = wire.decode_message(GOLD["wire_4"].tobytes())
    assert fr.found.dtype == bool and fr.rows.shape == (3, 3)
    _, fr0 = wire.decode_message(GOLD["wire_5"].tobytes())
    assert fr0.rows.shape == (2, 0)
    _, err = wire.decode_message(GOLD["wire_6"].tobytes())
    assert err.code == 7 and err.message == "worker failed: é"


def test_wire_errors():
    frame = GOLD["wire_2"].tobytes()
    with pytest.raises(wire.WireFormatError, match="magic"):
        wire.decode_message(b"XXXX" + frame[4:])
    with pytest.raises(wire.WireFormatError, match="version"):
        wire.decode_message(frame[:4] + struct.pack("<H", 2) + frame[6:])
    with pytest.raises(wire.WireFormatError, match="header"):
        wire.decode_message(frame[:10])
    with pytest.raises(wire.WireFormatError, match="payload"):
        wire.decode_message(frame[:-1])
    code, payload = wire.encode_payload(_msg(*wire_messages()[2][1:]))
    with pytest.raises(wire.WireFormatError, match="trailing"):
        wire.decode_payload(code, payload + b"\0")
    with pytest.raises(wire.WireFormatError, match="unknown message type"):
        wire.decode_payload(99, payload)
    bad = bytearray(wire.encode_payload(_msg(*wire_messages()[1][1:]))[1])
    bad[-17] = 9  # policy code byte of "<IBqQ"
    with pytest.raises(wire.WireFormatError, match="policy"):
        wire.decode_payload(wire.MSG_SAMPLE_REQUEST, bytes(bad))
    with pytest.raises(TypeError):
        wire.encode_payload(object())


def test_wire_socket_reader():
    frame = GOLD["wire_3"].tobytes()

    class Sock:
        def __init__(self, data, step):
            self.data, self.step = data, step

        def recv(self, n):
            part, self.data = self.data[:min(n, self.step)], self.data[min(n, self.step):]
            return part

    rid, msg = wire.read_message(Sock(frame, 5))
    assert rid == 1 << 63 and msg.kind == 2
    with pytest.raises(ConnectionError):
        wire.read_message(Sock(frame[:-3], 64))


@pytest.mark.parametrize("name,kind", [("tgff_node", KIND_NODE), ("tgff_edge", KIND_EDGE)])
def test_tgff_bytes_equal_reference(name, kind):
    ids, rows = feature_rows(kind)
    buf = io.BytesIO()
    save_features(buf, kind, rows.shape[1], ids, rows)
    assert buf.getvalue() == GOLD[name].tobytes()
    k, dim, ids2, rows2 = load_features(io.BytesIO(GOLD[name].tobytes()))
    assert (k, dim) == (kind, 6)
    np.testing.assert_array_equal(ids2, ids)
    np.testing.assert_array_equal(rows2, rows)


def test_tgff_errors(tmp_path):
    data = GOLD["tgff_node"].tobytes()
    with pytest.raises(FeatureFormatError, match="magic"):
        load_features(b"NOPE" + data[4:])
    with pytest.raises(FeatureFormatError, match="version"):
        load_features(data[:4] + struct.pack("<I", 3) + data[8:])
    with pytest.raises(FeatureFormatError, match="length"):
        load_features(data[:-4])
    p = tmp_path / "f.csv"
    p.write_text("# id,a,b\n1,0.5,2\n7,1,1\n")
    ids, rows = load_features_csv(p, 2)
    assert ids.tolist() == [1, 7] and rows.tolist() == [[0.5, 2.0], [1.0, 1.0]]
    with pytest.raises(FeatureFormatError):
        load_features_csv(p, 3)


def test_metrics_equal_reference():
    for i, counts in enumerate(metric_inputs()):
        want = RES[f"access_{i}"]
        if "error" in want:
            with pytest.raises(ValueError):
                metrics.access_distribution(counts)
        else:
            got = metrics.access_distribution(counts)
            assert repr(got["powerlaw_r2"]) == want["powerlaw_r2"]
            assert repr(got["exponential_r2"]) == want["exponential_r2"]
            assert got["degenerate"] == want["degenerate"]
            assert got["frequencies"].tolist() == want["frequencies"]
        assert repr(metrics.coefficient_of_variation(counts)) == RES[f"cv_{i}"]
    got = [repr(metrics.jaccard(a, b)) for a, b in (([1, 2, 3], [2, 3, 4]), ([], []), ([5], [6]))]
    assert got == RES["jaccard"]


@pytest.mark.parametrize("P", [1, 3, 4])
@pytest.mark.parametrize("directed", [True, False])
def test_partition_equal_reference(P, directed):
    edges = partition_edges()
    spec = partition.PartitionSpec(P)
    want = RES[f"partition_{P}_{int(directed)}"]
    shards = partition.dispatch(spec, edges, directed)
    assert [list(map(list, s.edges)) for s in shards] == want["shards"]
    st = partition.balance_stats(spec, edges, directed)
    assert [list(st.node_counts), list(st.edge_counts), repr(st.node_cv), repr(st.edge_cv)] == want["stats"]
    assert partition.assign(spec, 10) == 10 % P
    with pytest.raises(ValueError):
        partition.PartitionSpec(0)
