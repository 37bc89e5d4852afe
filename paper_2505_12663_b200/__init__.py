"""B200-native (sm_100a) sparse-embedding hot path of MTGenRec (arXiv 2505.12663).

Drop-in for the reference recsparse table/lookup API: the kernels live in
``_lib/librsgpu.so`` (C-ABI: ``include/rsgpu.h``); this package is the host
mirror of the reference interface.  No CPU fallback exists.
"""
from ._lib import (CapacityError, ConfigError, CudaError, InvariantError, IoError, RangeError,
                   RecsparseError, build, lib)
from .batcher import (SequenceBatcher, SequenceSample, closest_prefix, imbalance_report, partition_sequences,
                      weighted_grad_combine)
from .merge import (FeatureConfig, HashTableCollection, MergeGroup, MergePlan, Pooling, Router, catalog_from,
                    collection_lookup, decode_tagged_id, encode_tagged_id, plan_merge)
from .table import (AdagradParams, AdamParams, EmbedTable, SparseStep, TableConfig, Workspace,
                    apply_aggregated, as_keys, hash64_batch, keys_to_numpy, shard_of_batch,
                    sparse_update, stage1_dedup)

__all__ = [
    "SequenceBatcher", "SequenceSample", "closest_prefix", "imbalance_report", "partition_sequences",
    "weighted_grad_combine",
    "FeatureConfig", "HashTableCollection", "MergeGroup", "MergePlan", "Pooling", "Router", "catalog_from",
    "collection_lookup", "decode_tagged_id", "encode_tagged_id", "plan_merge",
    "AdagradParams", "AdamParams", "CapacityError", "ConfigError", "CudaError", "EmbedTable",
    "InvariantError", "IoError", "RangeError", "RecsparseError", "SparseStep", "TableConfig",
    "Workspace", "apply_aggregated", "as_keys", "build", "hash64_batch", "keys_to_numpy", "lib",
    "shard_of_batch", "sparse_update", "stage1_dedup",
]
