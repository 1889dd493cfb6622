"""B200-native (sm_100a) lossless homomorphic gradient compression (arXiv 2402.07529).

The hot path of Alg. 1 — compress, aggregate, recover — runs in the
hand-written CUDA kernels of ``csrc/`` behind the C ABI of ``include/lhc.h``
(``liblhc.so``); this package is the thin Python binding over it.
"""
from ._lib import (  # noqa: F401
    LhcError,
    lhc_comm_create,
    lhc_comm_destroy,
    lhc_comm_layout,
    lhc_decompress_workspace,
    lhc_ipc_handle,
    lhc_params,
    lhc_validate,
    last_launch_count,
    lib,
    params,
    read_stats,
    sketch_aggregate,
    sketch_allreduce,
    sketch_clear,
    sketch_compress,
    sketch_compress_coo,
    sketch_decompress,
    sketch_peel,
    sketch_query,
    sketch_hash_rows,
    lhc_shard_layout,
    lhc_shard_comm_create,
    sketch_reduce_scatter,
    sketch_allgather_decoded,
    sketch_clear_batch,
    sketch_compress_batch,
)
from .pipeline import (  # noqa: F401
    Decoder,
    LosslessAllReduce,
    NvlsBuffer,
    NvlsComm,
    PeerComm,
    ShardedAllReduce,
    Sketch,
    aggregate,
)
from .sizing import shard_plan, size_for, size_workload, union_support  # noqa: F401
