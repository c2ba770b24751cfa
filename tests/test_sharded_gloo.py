"""CPU, world_size = 2, gloo: the exchange/merge plumbing of the multi-GPU path
(paper_2211_16422_b200/sharded.py).  The shard engine here is a host stand-in built on the oracle
(test infrastructure); what is under test is the sharding arithmetic, the wire format of the
16-byte candidate, the all-gather layout and that merged shards equal the unsharded answer."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleShardEngine:
    """Same protocol as sharded.GpuShardEngine, computed with the C oracle on the host."""

    def __init__(self, oracle, dim, words, mz, charge, ids, rank, world):
        from paper_2211_16422_b200 import host, sharded
        self.sharded, self.dim, self.mz = sharded, dim, mz
        self.id_rank = host.id_ranks(ids)
        order = np.lexsort((np.arange(len(mz)), self.id_rank, mz, charge))  # build_index order
        keep = []
        for c in np.unique(charge):
            rows = order[charge[order] == c]
            b, e = sharded.shard_range(len(rows), rank, world)
            keep.append(rows[b:e])
        self.keep = np.sort(np.concatenate(keep))  # original ordinals this shard holds
        self.ix = oracle.build_index(dim, words[self.keep], mz[self.keep], charge[self.keep], None,
                                     [ids[i] for i in self.keep])
        self.q = None

    def set_queries(self, dim, q_words, q_mz, q_charge):
        self.q = (q_words, q_mz, q_charge)
        return len(q_mz)

    def search_shard(self, tol, k):
        qw, qmz, qch = self.q
        score, ordinal = self.ix.search_topk(qw, qmz, qch, tol, k)
        rec = self.sharded.empty_candidates(len(qmz), k)
        hit = ordinal != 0xFFFFFFFF
        glob = self.keep[np.where(hit, ordinal, 0)]
        rec["distance"][hit] = (self.dim - score)[hit]
        rec["id_rank"][hit] = self.id_rank[glob][hit]
        diff = np.abs(np.broadcast_to(qmz[:, None], glob.shape) - self.mz[glob])
        rec["abs_diff_bits"][hit] = diff.view(np.uint64)[hit]
        return torch.from_numpy(rec.view(np.uint8).reshape(-1).copy())

    def new_buffer(self, n_bytes):
        return torch.empty(n_bytes, dtype=torch.uint8)

    def merge(self, gathered, nq, k, world):
        parts = gathered.numpy().view(self.sharded.CANDIDATE_DTYPE).reshape(world, nq, k)
        allc = np.concatenate(list(parts), axis=1)  # [nq, world * k]
        order = np.lexsort((allc["id_rank"], allc["abs_diff_bits"], allc["distance"]), axis=1)[:, :k]
        out = np.take_along_axis(allc, order, axis=1)
        return torch.from_numpy(out.view(np.uint8).reshape(-1).copy())

    def decode(self, records, nq, k):
        rec = records.numpy().view(self.sharded.CANDIDATE_DTYPE).reshape(nq, k)
        hit = rec["distance"] != 0xFFFFFFFF
        ord_of_rank = np.argsort(self.id_rank).astype(np.uint32)
        score = np.where(hit, self.dim - rec["distance"], 0).astype(np.uint32)
        ordinal = np.where(hit, ord_of_rank[np.where(hit, rec["id_rank"], 0)], 0xFFFFFFFF).astype(np.uint32)
        return score, ordinal


def _case():
    rng = np.random.default_rng(77)
    dim, n, nq = 256, 1200, 90
    words = rng.integers(0, 2**64, (n, dim // 64), dtype=np.uint64)
    words[1000:] = words[:200]  # clones: ties must resolve identically across shard boundaries
    mz = np.round(rng.uniform(400.0, 1200.0, n), 2)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    ids = [f"s{rng.integers(0, 400)}" for _ in range(n)]
    qw = words[rng.integers(0, n, nq)]
    qmz = mz[rng.integers(0, n, nq)] + rng.choice([0.0, 0.01, 40.0], nq)
    qch = rng.integers(2, 4, nq).astype(np.uint8)
    return dim, words, mz, charge, ids, qw, qmz, qch


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.binding import Oracle
    from paper_2211_16422_b200 import sharded
    oracle = Oracle("port")
    dim, words, mz, charge, ids, qw, qmz, qch = _case()
    eng = OracleShardEngine(oracle, dim, words, mz, charge, ids, rank, world)
    searcher = sharded.ShardedSearcher(eng)
    res = {}
    for name, tol, k in (("open1", ("da", 500.0), 1), ("open4", ("da", 500.0), 4), ("ppm", ("ppm", 50.0), 3)):
        score, ordinal = searcher.search_batch(dim, qw, qmz, qch, tol, k)
        res[name + "_score"], res[name + "_ordinal"] = score, ordinal
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_merge_equals_unsharded(tmp_path, port):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    free_port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, free_port, str(tmp_path)), nprocs=2, join=True)
    dim, words, mz, charge, ids, qw, qmz, qch = _case()
    ix = port.build_index(dim, words, mz, charge, None, ids)
    r0, r1 = np.load(tmp_path / "rank0.npz"), np.load(tmp_path / "rank1.npz")
    for name, tol, k in (("open1", ("da", 500.0), 1), ("open4", ("da", 500.0), 4), ("ppm", ("ppm", 50.0), 3)):
        score, ordinal = ix.search_topk(qw, qmz, qch, tol, k)
        for r in (r0, r1):  # every rank ends with the single-GPU answer
            assert np.array_equal(r[name + "_ordinal"], ordinal), name
            assert np.array_equal(r[name + "_score"], score), name


def test_shard_ranges_partition_every_bucket():
    from paper_2211_16422_b200 import sharded
    for size in (0, 1, 7, 1000, 1_200_001):
        for world in (1, 2, 3, 8):
            edges = [sharded.shard_range(size, g, world) for g in range(world)]
            assert edges[0][0] == 0 and edges[-1][1] == size
            assert all(edges[g][1] == edges[g + 1][0] for g in range(world - 1))
            assert max(e - b for b, e in edges) - min(e - b for b, e in edges) <= 1
    assert sharded.CANDIDATE_DTYPE.itemsize == 16
