"""GPU: the multi-device context (homs_b200_ctx_create_multi, csrc/group.cu) behind the unchanged
search / cascade / encode entry points.  On a one-GPU box the devices are aliases of device 0 --
the same shard / peer-store / merge code path that runs across 8 GPUs -- and every answer must equal
the plain single-device context's bit for bit.  With >= 2 GPUs visible the same tests also run on
distinct devices, and ShardedSearcher(GpuShardEngine) runs under real NCCL, one process per GPU."""
import os
import socket
import sys

import numpy as np
import pytest

from oracle.binding import PreCfg, SynthCfg
from tests import _util as U

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _device_sets(hb):
    sets = [[0, 0], [0, 0, 0], [0] * 8]
    n = hb.device_count()
    if n >= 2:
        sets.append(list(range(n)))
    return sets


def _case(seed=91, dim=1024, n=9000, nq=700):
    rng = np.random.default_rng(seed)
    words = U.random_hvs(rng, n, dim)
    words[n - 1500:] = words[:1500]  # clones: ties across shard boundaries
    mz = np.round(rng.uniform(400.0, 1200.0, n), 2)
    charge = rng.integers(1, 4, n).astype(np.uint8)
    ids = [f"e{rng.integers(0, 2500)}" for _ in range(n)]
    decoy = (rng.random(n) < 0.5).astype(np.uint8)
    qw = words[rng.integers(0, n, nq)] ^ (U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim))
    qmz = mz[rng.integers(0, n, nq)] + rng.choice([0.0, 0.004, 15.0, -79.97 / 2], nq)
    qch = rng.integers(0, 4, nq).astype(np.uint8)
    return dim, words, mz, charge, ids, decoy, qw, qmz, qch


@pytest.mark.parametrize("engine", ["auto", "tensor_fp4", "popc", "direct"])
def test_group_search_and_cascade_equal_single_device(hb, engine):
    dim, words, mz, charge, ids, decoy, qw, qmz, qch = _case()
    tols = [hb.Tolerance("dalton", 500.0), hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 2.5)]
    with hb.Context(0) as one:
        one.set_engine(engine)
        one.build_index(dim, words, mz, charge, ids=ids, is_decoy=decoy)
        want = {(i, k): one.search_batch(qw, qmz, qch, t, k=k) for i, t in enumerate(tols) for k in (1, 4)}
        want_c = one.cascade_search(qw, qmz, qch, tols[1], tols[0], 0.05)
        want_b = one.buckets()
    for devs in _device_sets(hb):
        with hb.Context(devices=devs) as grp:
            grp.set_engine(engine)
            grp.build_index(dim, words, mz, charge, ids=ids, is_decoy=decoy)
            for (i, k), w in want.items():
                got = grp.search_batch(qw, qmz, qch, tols[i], k=k)
                assert np.array_equal(got.ordinal, w.ordinal), (devs, i, k)
                assert np.array_equal(got.raw_score, w.raw_score), (devs, i, k)
                assert np.array_equal(got.first, w.first) and np.array_equal(got.last, w.last)
            got_c = grp.cascade_search(qw, qmz, qch, tols[1], tols[0], 0.05)
            for key in ("query", "ordinal", "stage", "raw_score"):
                assert np.array_equal(got_c[key], want_c[key]), (devs, key)
            assert np.array_equal(got_c["q_value"].view(np.uint64), want_c["q_value"].view(np.uint64))
            # resident form and the candidate-record form
            grp.queries_upload(dim, qw, qmz, qch)
            res = grp.search_resident(tols[0], k=4, nq=len(qmz))
            assert np.array_equal(res.ordinal, want[(0, 4)].ordinal)
            # the index as a whole: same buckets, rows gathered back from all members in order
            got_b = grp.buckets()
            assert len(got_b) == len(want_b)
            for a, b in zip(got_b, want_b):
                assert a["charge"] == b["charge"] and a["shard_begin"] == 0 and a["shard_end"] == len(b["precursor_mz"])
                assert np.array_equal(a["precursor_mz"], b["precursor_mz"]) and np.array_equal(a["ordinal"], b["ordinal"])
                assert np.array_equal(a["words"], b["words"])
            f1, l1, h1 = grp.select_candidates(qmz, qch, tols[2])
            assert np.array_equal(f1, want[(2, 1)].first) and np.array_equal(l1, want[(2, 1)].last)


def test_group_raw_spectra_paths_equal_single_device(hb, best_oracle):
    """codebook replicas, encode_batch split across the members, fused index / query builds, cache loader."""
    synth = best_oracle.synth(SynthCfg(n_library=1500, n_query=300, peaks_per_spectrum=50, fraction_modified=0.6, seed=23))
    L, Q = synth["library"], synth["queries"]
    # a few unprocessable spectra (too few peaks) in both lists
    for S in (L, Q):
        S["intensity"] = S["intensity"].copy()
        for i in (3, 50, 51, 200):
            a, b = int(S["offsets"][i]), int(S["offsets"][i + 1])
            S["intensity"][a + 5:b] = 0.0
    pre = hb.PreprocessConfig()
    enc = hb.EncoderConfig(dim=2048, step_flips=1024, levels=16, seed=1)
    cb = hb.make_codebook(hb.dimension(pre), enc)
    narrow, wide = hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 500.0)
    with hb.Context(0) as one:
        one.upload_codebook(cb)
        w_lw, w_lok = one.encode_batch(L["offsets"], L["mz"], L["intensity"], pre)
        one.build_index_from_spectra(L["offsets"], L["mz"], L["intensity"], pre, L["precursor_mz"], L["charge"],
                                     ids=L["ids"], is_decoy=L["is_decoy"])
        one.queries_from_spectra(Q["offsets"], Q["mz"], Q["intensity"], pre, Q["precursor_mz"], Q["charge"])
        want = one.search_resident(wide, k=2)
        want_c = one.cascade_resident(narrow, wide, 0.01)
        kept = np.flatnonzero(w_lok)
        image = one.cache_write(pre, enc, w_lw[kept], L["precursor_mz"][kept], L["charge"][kept], L["is_decoy"][kept],
                                [L["ids"][i] for i in kept], ["PEP"] * len(kept))
    for devs in _device_sets(hb):
        with hb.Context(devices=devs) as grp:
            grp.upload_codebook(cb)
            lw, lok = grp.encode_batch(L["offsets"], L["mz"], L["intensity"], pre)
            assert np.array_equal(lok, w_lok) and np.array_equal(lw, w_lw), devs
            ok = grp.build_index_from_spectra(L["offsets"], L["mz"], L["intensity"], pre, L["precursor_mz"],
                                              L["charge"], ids=L["ids"], is_decoy=L["is_decoy"])
            assert np.array_equal(ok, w_lok)
            grp.queries_from_spectra(Q["offsets"], Q["mz"], Q["intensity"], pre, Q["precursor_mz"], Q["charge"])
            got = grp.search_resident(wide, k=2)
            assert np.array_equal(got.ordinal, want.ordinal) and np.array_equal(got.raw_score, want.raw_score), devs
            got_c = grp.cascade_resident(narrow, wide, 0.01)
            for key in ("query", "ordinal", "stage", "raw_score"):
                assert np.array_equal(got_c[key], want_c[key]), (devs, key)
            # read_cache + build_index straight onto the members
            grp.load_cache(image, pre, enc)
            again = grp.search_resident(wide, k=2)
            assert np.array_equal(again.ordinal, want.ordinal) and np.array_equal(again.raw_score, want.raw_score)


def test_group_rejects_external_sharding_and_reports_devices(hb):
    from paper_2211_16422_b200 import capi
    rng = np.random.default_rng(5)
    with hb.Context(devices=[0, 0]) as grp:
        assert capi.ctx_device_count(grp.handle) == 2
        with pytest.raises(hb.HomsError):
            grp.build_index(256, U.random_hvs(rng, 10, 256), np.linspace(500, 600, 10), [2] * 10,
                            shard_index=0, shard_count=2)
    with hb.Context(devices=[0]) as plain:
        assert capi.ctx_device_count(plain.handle) == 1
    with pytest.raises(hb.HomsError):
        hb.Context(devices=[])
    with pytest.raises(hb.HomsError):
        hb.Context(devices=[0, 10_000])


# ---- one process per GPU, real NCCL --------------------------------------------------------------

def _nccl_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_2211_16422_b200 as hb
    from paper_2211_16422_b200 import sharded
    dim, words, mz, charge, ids, decoy, qw, qmz, qch = _case()
    ctx = hb.Context(rank)
    ctx.build_index(dim, words, mz, charge, ids=ids, shard_index=rank, shard_count=world)
    searcher = sharded.ShardedSearcher(sharded.GpuShardEngine(ctx, f"cuda:{rank}"))
    res = {}
    for name, tol, k in (("open1", hb.Tolerance("dalton", 500.0), 1), ("open4", hb.Tolerance("dalton", 500.0), 4),
                         ("ppm", hb.Tolerance("ppm", 20.0), 3)):
        for rep in range(3):  # back to back: a missing stream dependency shows up as a stale buffer
            score, ordinal = searcher.search_batch(dim, qw, qmz, qch, tol, k)
        res[name + "_score"], res[name + "_ordinal"] = score, ordinal
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


def test_sharded_searcher_under_nccl(hb, tmp_path):
    import torch
    import torch.multiprocessing as mp
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("needs >= 2 CUDA devices (NCCL cannot put two ranks on one GPU)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_nccl_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    dim, words, mz, charge, ids, decoy, qw, qmz, qch = _case()
    with hb.Context(0) as one:
        one.build_index(dim, words, mz, charge, ids=ids)
        for name, tol, k in (("open1", hb.Tolerance("dalton", 500.0), 1), ("open4", hb.Tolerance("dalton", 500.0), 4),
                             ("ppm", hb.Tolerance("ppm", 20.0), 3)):
            want = one.search_batch(qw, qmz, qch, tol, k=k)
            for r in range(world):
                got = np.load(tmp_path / f"rank{r}.npz")
                assert np.array_equal(got[name + "_ordinal"], want.ordinal), (name, r)
                assert np.array_equal(got[name + "_score"], want.raw_score), (name, r)


def test_gpu_shard_engine_single_process_stream_order(hb):
    """GpuShardEngine on one device, world = 1 and a hand-made 2-part gather: the engine's stream is the
    context's stream and torch's current stream, so search -> (collective) -> merge is one order."""
    import torch
    from paper_2211_16422_b200 import sharded
    dim, words, mz, charge, ids, decoy, qw, qmz, qch = _case(nq=3000)
    tol, k = hb.Tolerance("dalton", 500.0), 2
    with hb.Context(0) as one:
        one.build_index(dim, words, mz, charge, ids=ids)
        want = one.search_batch(qw, qmz, qch, tol, k=k)
    parts = []
    ctxs = [hb.Context(0) for _ in range(2)]
    engines = []
    for g, c in enumerate(ctxs):
        c.build_index(dim, words, mz, charge, ids=ids, shard_index=g, shard_count=2)
        e = sharded.GpuShardEngine(c, "cuda:0")
        e.set_queries(dim, qw, qmz, qch)
        engines.append(e)
    for rep in range(4):
        parts = [e.search_shard(tol, k) for e in engines]
        e0 = engines[0]
        with e0.collective_stream():
            # stand-in for the all-gather, on the engine's stream like NCCL would be; part 1 comes from the
            # other engine's stream: order it explicitly, as the collective's own stream semantics would
            e0.stream.wait_stream(engines[1].stream)
            gathered = torch.cat(parts)
        merged = e0.merge(gathered, len(qmz), k, 2)
        score, ordinal = e0.decode(merged, len(qmz), k)
        assert np.array_equal(ordinal, want.ordinal) and np.array_equal(score, want.raw_score), rep
    for c in ctxs:
        c.close()
