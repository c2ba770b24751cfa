#!/usr/bin/env python
"""BASELINE config 5: dimension sweep D in {1024 ... 16384} x {standard 20 ppm, open +-500 Da} on the config-3
library (4.3 M rows, reference generator seed 3) re-encoded at every D (flips = D/2).

    python tools/config5_sweep.py [--dims 1024,2048,4096,8192,16384] [--queries 65536] [--steps 5]
    python -m torch.distributed.run --nproc-per-node N ... tools/config5_sweep.py     # N GPUs: library sharded

The workload is generated ONCE; per D: codebook -> library and queries encoded on the GPU -> resident index ->
device-timed search of the resident queries (CUDA events on the context's stream, max over ranks) for both
tolerances -> a bounded sample checked bit for bit against the compiled reference (oracle/_ref, rank 0).
One JSON line per (D, tolerance) on stdout; bench.py's own line for a single point is
`python bench.py --workload hek293 --dim D --tol ppm:20`.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="1024,2048,4096,8192,16384")
    ap.add_argument("--workload", default="hek293")
    ap.add_argument("--queries", type=int, default=65536, help="query prefix searched per step")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--parity-queries", type=int, default=48)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2211_16422_b200 as hb
    from paper_2211_16422_b200 import capi
    import workload as wl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    t = time.time()
    lib, qry, _, gen = wl.make(args.workload, "auto")
    n_lib = len(lib["precursor_mz"])
    nq = min(args.queries, len(qry["precursor_mz"]))
    q_end = int(qry["offsets"][nq])
    qry = dict(offsets=qry["offsets"][:nq + 1], mz=qry["mz"][:q_end], intensity=qry["intensity"][:q_end],
               precursor_mz=qry["precursor_mz"][:nq], charge=qry["charge"][:nq])
    id_rank = hb.id_ranks(lib["ids"])
    log(f"[config5] {args.workload}: {n_lib} library / {nq} query spectra from the {gen} generator in {time.time() - t:.0f}s")
    pre = hb.PreprocessConfig()
    oracle = None
    if rank == 0 and args.parity_queries:
        from oracle import binding as ob
        kind = "ref_v3" if ob.available("ref_v3") else "ref" if ob.available("ref") else "port"
        oracle = ob.Oracle(kind)

    for dim in [int(x) for x in args.dims.split(",")]:
        W = dim // 64
        ctx = hb.Context(local_rank)
        ctx.set_stream(stream.cuda_stream)
        ctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1)))

        def encode(spec, chunk=200_000):
            n = len(spec["offsets"]) - 1
            out = torch.empty((n, W), dtype=torch.int64, device=dev)
            ok = torch.empty(n, dtype=torch.uint8, device=dev)
            for a in range(0, n, chunk):
                b = min(n, a + chunk)
                p0, p1 = int(spec["offsets"][a]), int(spec["offsets"][b])
                off = torch.from_numpy((spec["offsets"][a:b + 1] - spec["offsets"][a]).astype(np.int64)).to(dev)
                mz = torch.from_numpy(spec["mz"][p0:p1]).to(dev)
                it = torch.from_numpy(spec["intensity"][p0:p1]).to(dev)
                ctx.encode_batch_dev(pre, b - a, p1 - p0, off.data_ptr(), mz.data_ptr(), it.data_ptr(),
                                     out[a:b].data_ptr(), ok[a:b].data_ptr())
                ctx.synchronize()
            assert int(ok.sum().item()) == n
            return out

        t = time.time()
        lib_words = encode(lib)
        ctx.build_index_dev(dim, lib_words.data_ptr(), n_lib, lib["precursor_mz"], lib["charge"], is_decoy=lib["is_decoy"],
                            id_rank=id_rank, shard_index=rank, shard_count=world)
        lw_host = lib_words.cpu().numpy().view(np.uint64) if oracle is not None else None
        del lib_words
        torch.cuda.empty_cache()
        q_words = encode(qry)
        d_qmz = torch.from_numpy(qry["precursor_mz"]).to(dev)
        d_qch = torch.from_numpy(qry["charge"]).to(dev)
        ctx.queries_upload_dev(dim, nq, q_words.data_ptr(), d_qmz.data_ptr(), d_qch.data_ptr())
        ctx.synchronize()
        log(f"[config5] D={dim}: encoded + indexed in {time.time() - t:.1f}s")
        oix = None
        if oracle is not None:
            oix = oracle.build_index(dim, lw_host, lib["precursor_mz"], lib["charge"], lib["is_decoy"], lib["ids"])
        rec = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
        gathered = torch.empty(world * nq * 16, dtype=torch.uint8, device=dev) if world > 1 else None
        merged = torch.empty(nq * 16, dtype=torch.uint8, device=dev) if world > 1 else None

        for tol_name, tol in (("ppm:20", hb.Tolerance("ppm", 20.0)), ("da:500", hb.Tolerance("dalton", 500.0))):
            def step():
                ctx.search_resident_dev(tol, 1, rec.data_ptr())
                if world > 1:
                    dist.all_gather_into_tensor(gathered, rec)
                    ctx.merge_candidates_dev(nq, 1, world, gathered.data_ptr(), merged.data_ptr())

            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            ctx.profile(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1)
            k_ms, k_n = ctx.kernel_time(capi.KERNEL_SEARCH)
            ctx.profile(False)
            if world > 1:
                tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
                dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
                ms = float(tmax.item())
            score, ordinal = ctx.candidates_decode(nq, 1, (merged if world > 1 else rec).data_ptr())
            first, last, _ = ctx.select_candidates(qry["precursor_mz"], qry["charge"], tol)
            pairs = int((last - first).sum())
            parity = None
            if oix is not None:
                m = min(nq, args.parity_queries)
                qh = q_words[:m].cpu().numpy().view(np.uint64)
                has, s_ref, o_ref, _ = oix.search_batch(qh, qry["precursor_mz"][:m], qry["charge"][:m],
                                                        ("ppm", 20.0) if tol_name == "ppm:20" else ("da", 500.0),
                                                        threads=os.cpu_count() or 1, batch=4)
                hit = has.astype(bool)
                same = (np.array_equal(ordinal[:m, 0] != 0xFFFFFFFF, hit) and np.array_equal(score[:m, 0][hit], s_ref[hit])
                        and np.array_equal(ordinal[:m, 0][hit], o_ref[hit]))
                parity = f"{m} queries bit-exact vs {oracle.kind}" if same else "MISMATCH"
                if not same:
                    raise AssertionError(f"D={dim} {tol_name}: GPU differs from the reference")
            if rank == 0:
                ms_step = ms / args.steps
                print(json.dumps({
                    "config": f"config 5: {args.workload} library {n_lib} rows re-encoded at D={dim}, {nq} queries, {tol_name}",
                    "dim": dim, "tol": tol_name, "n_gpus": world, "engine": ctx.last_engine(), "ms_per_step": ms_step,
                    "queries_per_s": nq / (ms_step * 1e-3), "kernel_ms_per_step": k_ms / args.steps,
                    "search_launches_per_step": k_n / args.steps, "candidate_pairs_per_step": pairs,
                    "pairs_per_s": pairs / (ms_step * 1e-3),
                    "hbm_view_gbs": pairs * (dim // 8 + 8) / (ms_step * 1e-3) / 1e9,
                    "tensor_tops": (2.0 * pairs / world * ((dim + 255) // 256 * 256) / (k_ms / args.steps * 1e-3) / 1e12
                                    if ctx.last_engine() == "tensor_fp4" and k_ms > 0 else None),
                    "parity": parity, "generator": gen}), flush=True)
        if oix is not None:
            oix.close()
        ctx.close()
        del q_words, rec
        torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
