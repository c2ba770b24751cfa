"""Multi-GPU composition of the search path: one process per GPU, library sharded by contiguous
m/z slices of every charge bucket, queries replicated, ONE exchange step.

    rank r:  candidates_r = search(shard r)            16-byte records, [nq, k]
    all:     gathered = all_gather(candidates_r)       [world, nq, k]  (NCCL over NVLink; gloo in tests)
    all:     merged = k-way lexicographic merge        == the single-GPU answer

The reference has no distributed layer; the rule that makes this exact is that a
query's answer is the minimum of a total-order key over its window (src/search.cpp:133-146) and a
minimum is associative.  The shard engine is anything with `search_shard / merge / decode`:
`GpuShardEngine` wraps a `Context` (the product); the CPU tests plug a host stand-in into the same
class to exercise the exchange with the gloo backend.
"""
from __future__ import annotations

import numpy as np

# wire format of one candidate == homs_b200_candidate (include/homs_b200.h)
CANDIDATE_DTYPE = np.dtype([("distance", "<u4"), ("id_rank", "<u4"), ("abs_diff_bits", "<u8")])
NO_CANDIDATE = 0xFFFFFFFF


def shard_range(bucket_size: int, shard_index: int, shard_count: int) -> tuple[int, int]:
    """Rows [begin, end) of a charge bucket (in its m/z-sorted order) that shard `shard_index`
    keeps -- the same arithmetic as csrc/library.cu."""
    return bucket_size * shard_index // shard_count, bucket_size * (shard_index + 1) // shard_count


def empty_candidates(n: int, k: int) -> np.ndarray:
    rec = np.zeros((n, k), CANDIDATE_DTYPE)
    rec["distance"] = NO_CANDIDATE
    rec["id_rank"] = NO_CANDIDATE
    rec["abs_diff_bits"] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return rec


class GpuShardEngine:
    """Shard engine on one CUDA device (torch tensors are only device buffers here).

    Stream order: the context's kernels, the collective and the merge must run in ONE order.  The
    context is therefore put on a real (non-NULL) torch stream that is also made torch's current
    stream for this device, which is the stream torch.distributed's NCCL ops synchronise with: the
    all-gather cannot start before the search kernels have written `mine`, and the merge kernel cannot
    read `gathered` before the all-gather has finished."""

    def __init__(self, ctx, device):
        import torch
        self.ctx, self.torch, self.device = ctx, torch, torch.device(device)
        self.nq = 0
        self.stream = torch.cuda.Stream(self.device)
        assert self.stream.cuda_stream != 0
        torch.cuda.set_stream(self.stream)
        ctx.set_stream(self.stream.cuda_stream)

    def set_queries(self, dim, q_words, q_mz, q_charge) -> int:
        self.nq = self.ctx.queries_upload(dim, q_words, q_mz, q_charge)
        return self.nq

    def search_shard(self, tol, k):
        with self.torch.cuda.stream(self.stream):
            rec = self.torch.empty(self.nq * k * 16, dtype=self.torch.uint8, device=self.device)
            self.ctx.search_resident_dev(tol, k, rec.data_ptr())
        return rec

    def new_buffer(self, n_bytes):
        with self.torch.cuda.stream(self.stream):
            return self.torch.empty(n_bytes, dtype=self.torch.uint8, device=self.device)

    def merge(self, gathered, nq, k, world):
        with self.torch.cuda.stream(self.stream):
            out = self.new_buffer(nq * k * 16)
            self.ctx.merge_candidates_dev(nq, k, world, gathered.data_ptr(), out.data_ptr())
        return out

    def collective_stream(self):
        """The stream collectives must be issued on (torch's current stream inside this context)."""
        return self.torch.cuda.stream(self.stream)

    def decode(self, records, nq, k):
        return self.ctx.candidates_decode(nq, k, records.data_ptr())


class ShardedSearcher:
    """search_batch over a library sharded across the ranks of a torch.distributed group."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist
        self.engine, self.dist, self.group = engine, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def search_batch(self, dim, q_words, q_mz, q_charge, tol, k: int = 1):
        """-> (raw_score u32[nq, k], ordinal u32[nq, k]) identical on every rank."""
        nq = self.engine.set_queries(dim, q_words, q_mz, q_charge)
        mine = self.engine.search_shard(tol, k)
        if self.world == 1:
            return self.engine.decode(mine, nq, k)
        gathered = self.engine.new_buffer(self.world * nq * k * 16)  # [world][nq][k] records
        import contextlib
        on_stream = getattr(self.engine, "collective_stream", contextlib.nullcontext)
        with on_stream():  # NCCL orders itself against torch's current stream == the context's stream
            self.dist.all_gather_into_tensor(gathered, mine, group=self.group)
        merged = self.engine.merge(gathered, nq, k, self.world)
        return self.engine.decode(merged, nq, k)
