"""Synthetic inputs of the benchmark configs via librsgpu's generator.

Identical (same seed -> same ids) to the reference's generate_workload
(workload.cpp:280-307) and pseudo_sparse_grad (workload.cpp:348-355); the
parity tests check that against the reference itself.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from ._lib import check


def generate(seed: int, num_sequences: int, mean_len: float, max_len: int, sigma: float,
             zipf: float, vocab) -> tuple[np.ndarray, np.ndarray]:
    """-> (lengths[num_sequences] u64, catalog-tagged ids[Σ lengths] u64)."""
    vocab = np.ascontiguousarray(np.atleast_1d(np.asarray(vocab, dtype=np.uint64)))
    lengths = np.zeros(num_sequences, np.uint64)
    cap = int(num_sequences * mean_len * 3) + 4096
    while True:
        ids = np.zeros(cap, np.uint64)
        n = C.c_uint64()
        st = L.lib().rs_workload_generate(seed, num_sequences, mean_len, max_len, sigma, zipf, len(vocab),
                                          vocab.ctypes.data, lengths.ctypes.data, ids.ctypes.data, cap,
                                          C.byref(n))
        if st == L.RS_OK:
            return lengths, ids[: n.value].copy()
        if cap >= num_sequences * max_len:
            check(st, "generate")
        cap = min(cap * 2, num_sequences * max_len)


def write_workload_file(path: str, seed: int, num_sequences: int, mean_len: float, max_len: int, sigma: float,
                        zipf: float, vocab) -> None:
    """generate_workload_file (workload.cpp:280-315): the reference's text format."""
    vocab = np.ascontiguousarray(np.atleast_1d(np.asarray(vocab, dtype=np.uint64)))
    check(L.lib().rs_workload_write(str(path).encode(), seed, num_sequences, mean_len, max_len, sigma, zipf,
                                    len(vocab), vocab.ctypes.data), "write_workload_file")


def read_workload_file(path: str) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """read_workload_file (workload.cpp:317-339) -> (sample_ids u64, labels f64,
    lengths u64, ids u64 concatenated in file order); IoError on a bad file."""
    ns, nt = C.c_uint64(), C.c_uint64()
    p = str(path).encode()
    check(L.lib().rs_workload_read(p, 0, 0, None, None, None, None, C.byref(ns), C.byref(nt)), "read_workload_file")
    sid = np.zeros(max(ns.value, 1), np.uint64)
    lab = np.zeros(max(ns.value, 1), np.float64)
    ln = np.zeros(max(ns.value, 1), np.uint64)
    ids = np.zeros(max(nt.value, 1), np.uint64)
    check(L.lib().rs_workload_read(p, len(sid), len(ids), sid.ctypes.data, lab.ctypes.data, ln.ctypes.data,
                                   ids.ctypes.data, C.byref(ns), C.byref(nt)), "read_workload_file")
    return sid[: ns.value], lab[: ns.value], ln[: ns.value], ids[: nt.value]


def sample_of_tokens(lengths, first_sample_id: int = 1) -> np.ndarray:
    lengths = np.asarray(lengths, np.int64)
    return np.repeat(np.arange(first_sample_id, first_sample_id + len(lengths), dtype=np.uint64), lengths)


def pseudo_grads(sample_of: torch.Tensor, step: int, dim: int) -> torch.Tensor:
    """per-token pseudo_sparse_grad(sample_id, step) generated on the device."""
    s = sample_of.to(device="cuda", dtype=torch.int64).contiguous()
    out = torch.empty((s.numel(), dim), dtype=torch.float32, device="cuda")
    check(L.lib().rs_pseudo_grads(s.data_ptr(), s.numel(), step, dim, out.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream), "pseudo_grads")
    return out


def pseudo_grads_jagged(lengths: torch.Tensor, step: int, dim: int, n_tokens: int,
                        first_sample_id: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """pseudo_sparse_grad rows of a jagged batch from its sequence lengths
    (device tensor): one row per sample broadcast to its tokens."""
    ln = lengths.to(device="cuda", dtype=torch.int64).contiguous()
    if out is None:
        out = torch.empty((n_tokens, dim), dtype=torch.float32, device="cuda")
    check(L.lib().rs_pseudo_grads_jagged(ln.data_ptr(), ln.numel(), first_sample_id, step, dim, n_tokens,
                                         out.data_ptr(), torch.cuda.current_stream().cuda_stream),
          "pseudo_grads_jagged")
    return out
