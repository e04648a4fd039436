"""The vectorised generator is array-identical to the reference (synth.py:15-53)."""

import hashlib
import json

import numpy as np

from fixtures import misc
from paper_2311_17410_b200.synth import generate_synthetic_arrays


def test_generator_matches_reference_digests():
    for args, digest in misc()["generate_synthetic_sha256"].items():
        nodes, edges, skew, span, seed, src_skew = json.loads(args)
        src, dst, ts = generate_synthetic_arrays(nodes, edges, skew, span, seed, src_skew)
        a = np.stack([src, dst, ts], axis=1).astype(np.int64)
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == digest, args


def test_generator_properties():
    # reference tests/test_metrics.py:50-61: deterministic, sorted, self-loop free
    a = generate_synthetic_arrays(300, 5000, 2.2, 10_000, seed=4)
    b = generate_synthetic_arrays(300, 5000, 2.2, 10_000, seed=4)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    src, dst, ts = a
    assert np.all(np.diff(ts) >= 0) and not np.any(src == dst)
