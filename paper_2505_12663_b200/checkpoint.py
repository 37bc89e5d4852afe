"""Elastic checkpoint of device tables (host mirror of checkpoint.hpp).

``save_shard`` / ``read_header`` / ``load_shard`` / ``shard_file_name`` keep
the reference's names and file format (checkpoint.hpp:25-54); ``save_cluster``
/ ``load_cluster`` operate on one process's ``ShardedTable`` (every rank
saves / loads its own shard; load_cluster's modulo file selection and
ownership refilter, checkpoint.cpp:194-254).
"""
from __future__ import annotations

import ctypes as C
import os

from . import _lib as L
from ._lib import check


def shard_file_name(rank: int, world_size: int) -> str:
    buf = C.create_string_buffer(256)
    check(L.lib().rs_ckpt_shard_file_name(rank, world_size, buf, len(buf)), "shard_file_name")
    return buf.value.decode()


def save_shard(table, rank: int, world_size: int, path: str) -> None:
    check(L.lib().rs_ckpt_save_shard(table.handle, rank, world_size, os.fspath(path).encode()), "save_shard")


def read_header(path: str) -> L.rs_ckpt_header:
    h = L.rs_ckpt_header()
    check(L.lib().rs_ckpt_read_header(os.fspath(path).encode(), C.byref(h)), "read_shard_file")
    return h


def load_shard(table, directory: str, saved_world: int, new_world: int, rank: int) -> None:
    check(L.lib().rs_ckpt_load_shard(table.handle, os.fspath(directory).encode(), saved_world, new_world, rank),
          "load_cluster")


def save_cluster(sharded, directory: str) -> str:
    """This rank's shard file of a ShardedTable (call on every rank)."""
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, shard_file_name(sharded.rank, sharded.world))
    save_shard(sharded.shard, sharded.rank, sharded.world, path)
    return path


def load_cluster(sharded, directory: str, saved_world: int) -> None:
    """Fill this rank's (empty) shard from a checkpoint saved at saved_world."""
    load_shard(sharded.shard, directory, saved_world, sharded.world, sharded.rank)
