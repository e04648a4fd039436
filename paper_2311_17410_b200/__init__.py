"""B200-native GNNFlow hot path: device block store, temporal sampler, feature cache.

Drop-in for the hot-path subset of the reference package ``ctdg``
(/root/reference/pkg/src/ctdg/__init__.py:8-44): same class/function names and
semantics, with state on the GPU and the work done by hand-written sm_100a
kernels in libgfb200.so (C ABI: include/gfb200.h).  Importing this package
does not load CUDA; the first graph/cache/sampler call loads libgfb200.so and
fails loudly if it is missing.
"""

from .storage import (  # noqa: F401
    ADJACENCY_LIST_SIZING,
    AdaptiveSizing,
    BatchSizing,
    BlockSizing,
    DynamicGraph,
    FixedSizing,
    GraphFormatError,
    InsertionBatch,
    InsertionResult,
    NodeEntry,
    NodeNotFoundError,
    StorageStats,
    TS_MAX,
    TS_MIN,
    new_graph,
    parse_offload,
    write_offload_records,
)
from .sampling import (  # noqa: F401
    LayeredSample,
    SampleLayer,
    SampleRequest,
    SamplingPolicy,
    TemporalSampler,
    hop_seed,
    random_walk,
    sample_khop,
    sample_khop_device,
    sample_layer,
)
from .cache import CacheSnapshot, VectorCache, load_cache  # noqa: F401
from .features import EdgeFeatureTable, NodeFeatureTable, fetch_features  # noqa: F401
from .synth import generate_synthetic_arrays, generate_synthetic_device  # noqa: F401

__version__ = "0.1.0"
