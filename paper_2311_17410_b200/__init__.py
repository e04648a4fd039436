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
from .features import (  # noqa: F401
    EdgeFeatureTable,
    FeatureFormatError,
    NodeFeatureTable,
    NodeMemoryTable,
    fetch_features,
    load_feature_table,
    save_edge_features,
    save_node_features,
)
from .synth import generate_synthetic, generate_synthetic_arrays, generate_synthetic_device  # noqa: F401
from .metrics import access_distribution, coefficient_of_variation, jaccard  # noqa: F401
from .partition import BalanceStats, PartitionSpec, assign, balance_stats, dispatch  # noqa: F401
from .cluster import ClusterSim, ClusterSpec, Origin, RemoteRequestError, measure_cv, route  # noqa: F401
from .harness import (  # noqa: F401
    CacheConfig,
    IngestFormatError,
    RoundReport,
    RunConfig,
    bench,
    load_config,
    load_edge_csv,
    run_continuous,
    save_edge_csv,
)

__version__ = "0.1.0"
