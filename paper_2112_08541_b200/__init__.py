"""B200-native BGL per-mini-batch preprocessing path.

Drop-in replacements for the reference package's hot-path modules
(`gnnio.sampler`, `gnnio.cachesim`, `gnnio.ordering`) plus the net-new
feature retrieval (`features`) and the fused multi-batch pipeline
(`pipeline`). Every compute step runs in hand-written sm_100a CUDA kernels
behind the C ABI in include/bgl_b200.h (`_lib/libbgl_b200.so`); there is no
CPU fallback.
"""

from . import cachesim, features, graph, ordering, sampler  # noqa: F401
from .cachesim import (  # noqa: F401
    CacheConfig,
    CacheSimReport,
    amortized_update_ops,
    compare_policies,
    simulate,
    warm_static,
)
from .graph import (DeviceGraph, Graph, generate_power_law, generate_power_law_device,  # noqa: F401
                    generate_power_law_exact_device, power_law_edges)
from .ordering import (  # noqa: F401
    BatchSchedule,
    ShufflingErrorReport,
    form_batches,
    generate_bfs_sequences,
    proximity_schedule,
    random_shift,
    random_shuffle_schedule,
    select_num_sequences,
    shuffling_error,
    shuffling_error_threshold,
)
from .sampler import AccessTrace, EpochCommReport, SamplingConfig, sample_batch, simulate_epoch  # noqa: F401

__version__ = "0.1.0"
