"""TGRP frames: the reference's remote sampling / feature RPC encoding (wire.py:1-221).

A frame is a 20-byte little-endian header -- magic ``TGRP``, version (u16),
message type (u16), request id (u64), payload length (u32) -- and a payload
of typed fields; every array is a u32 element count followed by the packed
elements.  The byte layout is the reference's (tests/test_formats.py pins
round trips and byte equality against frames the unmodified reference
encoded, stored as the wire_* entries of tests/golden/formats.npz).

The codec here is table driven: each message type lists its fields as
(name, kind, numpy dtype) and one packer / one reader walk the table.
``response_from_layer`` builds a sample response straight from a device
``SampleLayer`` (one device-to-host copy per array).  Sockets and servers are
not part of this package.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, fields

import numpy as np

WIRE_MAGIC = b"TGRP"
WIRE_VERSION = 1
HEADER_FMT = "<4sHHQI"
HEADER_SIZE = struct.calcsize(HEADER_FMT)

MSG_SAMPLE_REQUEST = 1
MSG_SAMPLE_RESPONSE = 2
MSG_FEATURE_REQUEST = 3
MSG_FEATURE_RESPONSE = 4
MSG_ERROR = 255

POLICY_CODE = {"recent": 0, "uniform": 1, "time_window": 2}
POLICY_NAME = {v: k for k, v in POLICY_CODE.items()}


class WireFormatError(ValueError):
    """Malformed frame or payload."""


@dataclass
class SampleRequestMsg:
    targets: np.ndarray
    timestamps: np.ndarray
    t_starts: np.ndarray
    fanout: int
    policy_kind: str
    delta: int
    seed: int


@dataclass
class SampleResponseMsg:
    offsets: np.ndarray
    neighbors: np.ndarray
    edge_ids: np.ndarray
    timestamps: np.ndarray


@dataclass
class FeatureRequestMsg:
    kind: int  # 0 node, 1 edge, 2 memory
    ids: np.ndarray


@dataclass
class FeatureResponseMsg:
    dim: int
    found: np.ndarray
    rows: np.ndarray


@dataclass
class ErrorMsg:
    code: int
    message: str


# field tables: ("arr", wire dtype, in-memory dtype) | ("fix", struct format over several fields)
_LAYOUT = {
    SampleRequestMsg: (MSG_SAMPLE_REQUEST, [
        ("targets", "arr", "<u8", np.int64), ("timestamps", "arr", "<i8", np.int64),
        ("t_starts", "arr", "<i8", np.int64), (("fanout", "policy_kind", "delta", "seed"), "fix", "<IBqQ", None)]),
    SampleResponseMsg: (MSG_SAMPLE_RESPONSE, [
        ("offsets", "arr", "<u4", np.int64), ("neighbors", "arr", "<u8", np.int64),
        ("edge_ids", "arr", "<u8", np.int64), ("timestamps", "arr", "<i8", np.int64)]),
    FeatureRequestMsg: (MSG_FEATURE_REQUEST, [(("kind",), "fix", "<B", None), ("ids", "arr", "<u8", np.int64)]),
    FeatureResponseMsg: (MSG_FEATURE_RESPONSE, [
        (("dim",), "fix", "<I", None), ("found", "arr", "<u1", bool), ("rows", "arr", "<f4", np.float32)]),
}
_BY_TYPE = {code: (cls, spec) for cls, (code, spec) in _LAYOUT.items()}


def _to_wire(name: str, value):
    if name == "policy_kind":
        return POLICY_CODE[value]
    if name == "seed":
        return int(value) & 0xFFFFFFFFFFFFFFFF
    return int(value)


def _from_wire(name: str, value):
    if name == "policy_kind":
        if value not in POLICY_NAME:
            raise WireFormatError(f"unknown policy code {value}")
        return POLICY_NAME[value]
    return int(value)


def encode_payload(msg) -> tuple[int, bytes]:
    if isinstance(msg, ErrorMsg):
        text = msg.message.encode("utf-8")
        return MSG_ERROR, struct.pack("<HI", msg.code, len(text)) + text
    entry = _LAYOUT.get(type(msg))
    if entry is None:
        raise TypeError(f"cannot encode {type(msg).__name__}")
    code, spec = entry
    out = bytearray()
    for name, kind, fmt, _ in spec:
        if kind == "fix":
            out += struct.pack(fmt, *(_to_wire(n, getattr(msg, n)) for n in name))
        else:
            a = np.asarray(getattr(msg, name))
            if a.ndim > 1:
                a = a.reshape(-1)
            out += struct.pack("<I", a.size)
            out += a.astype(fmt).tobytes()
    return code, bytes(out)


class _Cursor:
    def __init__(self, buf: bytes):
        self.buf, self.at = buf, 0

    def take(self, fmt: str):
        end = self.at + struct.calcsize(fmt)
        if end > len(self.buf):
            raise WireFormatError("truncated payload")
        vals = struct.unpack_from(fmt, self.buf, self.at)
        self.at = end
        return vals

    def array(self, fmt: str) -> np.ndarray:
        (count,) = self.take("<I")
        width = np.dtype(fmt).itemsize
        if self.at + count * width > len(self.buf):
            raise WireFormatError("truncated array")
        a = np.frombuffer(self.buf, dtype=fmt, count=count, offset=self.at).copy()
        self.at += count * width
        return a


def decode_payload(msg_type: int, payload: bytes):
    cur = _Cursor(payload)
    if msg_type == MSG_ERROR:
        code, length = cur.take("<HI")
        text = payload[cur.at:cur.at + length]
        if len(text) != length:
            raise WireFormatError("truncated error message")
        return ErrorMsg(code, text.decode("utf-8"))
    if msg_type not in _BY_TYPE:
        raise WireFormatError(f"unknown message type {msg_type}")
    cls, spec = _BY_TYPE[msg_type]
    vals = {}
    for name, kind, fmt, host in spec:
        if kind == "fix":
            raw = cur.take(fmt)
            vals.update({n: _from_wire(n, v) for n, v in zip(name, raw)})
        else:
            a = cur.array(fmt)
            vals[name] = a.astype(host) if host is not None and a.dtype != host else a
    if cur.at != len(payload):
        raise WireFormatError("trailing bytes in payload")
    if cls is FeatureResponseMsg:
        n, dim = len(vals["found"]), vals["dim"]
        if dim and vals["rows"].size != n * dim:
            raise WireFormatError("feature rows length mismatch")
        vals["rows"] = vals["rows"].reshape(n, dim) if dim else np.zeros((n, 0), dtype=np.float32)
    return cls(**{f.name: vals[f.name] for f in fields(cls)})


def encode_message(request_id: int, msg) -> bytes:
    code, payload = encode_payload(msg)
    return struct.pack(HEADER_FMT, WIRE_MAGIC, WIRE_VERSION, code, request_id, len(payload)) + payload


def _check_header(head: bytes):
    magic, version, code, request_id, length = struct.unpack_from(HEADER_FMT, head, 0)
    if magic != WIRE_MAGIC:
        raise WireFormatError("bad wire magic")
    if version != WIRE_VERSION:
        raise WireFormatError(f"unsupported wire version {version}")
    return code, request_id, length


def decode_message(data: bytes) -> tuple[int, object]:
    if len(data) < HEADER_SIZE:
        raise WireFormatError("truncated header")
    code, request_id, length = _check_header(data)
    payload = data[HEADER_SIZE:HEADER_SIZE + length]
    if len(payload) != length:
        raise WireFormatError("truncated payload")
    return request_id, decode_payload(code, payload)


def read_message(sock) -> tuple[int, object]:
    """One frame from a socket-like object with ``recv``."""
    code, request_id, length = _check_header(_recv_exact(sock, HEADER_SIZE))
    return request_id, decode_payload(code, _recv_exact(sock, length))


def _recv_exact(sock, n: int) -> bytes:
    buf = bytearray()
    while len(buf) < n:
        part = sock.recv(n - len(buf))
        if not part:
            raise ConnectionError("socket closed mid-message")
        buf += part
    return bytes(buf)


def request_from_queries(targets, t_starts, t_ends, fanout: int, policy, seed: int) -> SampleRequestMsg:
    """A sample request for device or host query arrays (policy: SamplingPolicy)."""
    host = [np.asarray(x.cpu() if hasattr(x, "cpu") else x, dtype=np.int64) for x in (targets, t_ends, t_starts)]
    return SampleRequestMsg(host[0], host[1], host[2], int(fanout), policy.kind, int(policy.delta), int(seed))


def response_from_layer(layer) -> SampleResponseMsg:
    """A sample response from a (device or host) SampleLayer."""
    return SampleResponseMsg(*[np.asarray(x.cpu() if hasattr(x, "cpu") else x, dtype=np.int64)
                               for x in (layer.offsets, layer.neighbors, layer.edge_ids, layer.timestamps)])
