"""B200-native ADT codec + AWP controller (arXiv:2004.02297), drop-in for
the reference package `weightpack`'s hot-path API
(/root/reference/pkg/src/weightpack/__init__.py:5-25).

Compute runs in the in-tree sm_100a library libadt.so through a C ABI
(include/adt.h); there is no CPU fallback.
"""

from .codec import (  # noqa: F401
    MAX_ROUND_TO,
    MIN_ROUND_TO,
    STREAM_HEADER_BYTES,
    STREAM_MAGIC,
    STREAM_VERSION,
    VECTOR_GROUP,
    WORD_BYTES,
    MalformedBlock,
    PackedBlock,
    bits_to_round_to,
    blocks_of,
    check_round_to,
    pack,
    pack_many,
    pack_parallel,
    pack_vectorized,
    read_stream,
    truncation_mask,
    unpack,
    unpack_many,
    write_stream,
)
from .layout import PackedLayout  # noqa: F401
from .precision import (  # noqa: F401
    TRACE_HEADER,
    FixedPrecision,
    LayerPrecisionState,
    PrecisionConfig,
    PrecisionController,
    UnknownLayer,
    change_rate,
    l2_norm,
    l2_norm_many,
    write_trace_csv,
)
from .sync import NonFiniteParameters, SyncResult, WeightSync  # noqa: F401
from .grads import GradBucket, GradientSet, ShapeMismatch  # noqa: F401
from .sharded import PeerTimeout, ShardedWeightSync, ShardPlan  # noqa: F401
from .hostsync import HostWeightSync, pack_host  # noqa: F401

__version__ = "0.1.0"
