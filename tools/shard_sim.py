#!/usr/bin/env python
"""Strong-scaling projection of the sharded search on ONE GPU.

Only one B200 is visible to this run, so the N-GPU step cannot be timed directly.  Every rank of the
N-GPU job runs exactly `search_resident_dev` on its own shard (contiguous m/z slice of every charge
bucket, queries replicated) followed by one all-gather of nq*k 16-byte candidates and the merge
kernel; the ranks never wait for each other before the gather.  This tool builds each shard g of G
in turn on the one device, times its step with CUDA events (same code path, same kernels) and
prints  max_g(step) + merge  -- the device-time critical path of the G-GPU job without the gather's
wire time (256 KB per rank at config 2: launch-latency sized).  It also checks that the merged
candidates of the G shards equal the single-shard answer bit for bit.

    python tools/shard_sim.py [--workload iprg2012] [--shards 1,2,4,8] [--steps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="iprg2012")
    ap.add_argument("--shards", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch

    import paper_2211_16422_b200 as hb
    from paper_2211_16422_b200 import capi
    import workload as wl

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    n_targets, n_query, dim, peaks, seed = wl.WORKLOADS[args.workload]
    lib = wl.synth_library(n_targets, peaks, 1.0, seed)
    qry = wl.synth_queries(lib, n_query, seed=seed)
    n_lib, nq = len(lib["precursor_mz"]), n_query
    W = hb.words_for(dim)
    pre = hb.PreprocessConfig()
    tol = hb.Tolerance("dalton", 500.0)
    cb = hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1))

    enc = hb.Context(0)
    enc.set_stream(stream.cuda_stream)
    enc.upload_codebook(cb)

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
            enc.encode_batch_dev(pre, b - a, p1 - p0, off.data_ptr(), mz.data_ptr(), it.data_ptr(),
                                 out[a:b].data_ptr(), ok[a:b].data_ptr())
            enc.synchronize()
        return out

    lib_words, q_words = encode(lib), encode(qry)
    enc.close()
    id_rank = hb.id_ranks(lib["ids"])
    d_qmz = torch.from_numpy(qry["precursor_mz"]).to(dev)
    d_qch = torch.from_numpy(qry["charge"]).to(dev)

    rows = []
    single = None
    for G in [int(x) for x in args.shards.split(",")]:
        per_shard, per_kernel, recs = [], [], []
        for g in range(G):
            ctx = hb.Context(0)
            ctx.set_stream(stream.cuda_stream)
            ctx.build_index_dev(dim, lib_words.data_ptr(), n_lib, lib["precursor_mz"], lib["charge"],
                                is_decoy=lib["is_decoy"], id_rank=id_rank, shard_index=g, shard_count=G)
            ctx.queries_upload_dev(dim, nq, q_words.data_ptr(), d_qmz.data_ptr(), d_qch.data_ptr())
            rec = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
            for _ in range(args.warmup):
                ctx.search_resident_dev(tol, 1, rec.data_ptr())
            torch.cuda.synchronize(dev)
            ctx.profile(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                ctx.search_resident_dev(tol, 1, rec.data_ptr())
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / args.steps
            kms, kl = ctx.kernel_time(capi.KERNEL_SEARCH)
            ctx.profile(False)
            per_shard.append(ms)
            per_kernel.append(kms / max(1, kl))
            recs.append(rec)
            if g == G - 1:  # merge on the last context (any rank does the same)
                gathered = torch.cat(recs)
                merged = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
                for _ in range(3):
                    ctx.merge_candidates_dev(nq, 1, G, gathered.data_ptr(), merged.data_ptr())
                torch.cuda.synchronize(dev)
                m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                m0.record(stream)
                for _ in range(10):
                    ctx.merge_candidates_dev(nq, 1, G, gathered.data_ptr(), merged.data_ptr())
                m1.record(stream)
                torch.cuda.synchronize(dev)
                merge_ms = m0.elapsed_time(m1) / 10
                score, ordinal = ctx.candidates_decode(nq, 1, merged.data_ptr())
            ctx.close()
        if single is None:
            single = (score.copy(), ordinal.copy(), max(per_shard))
        same = bool(np.array_equal(score, single[0]) and np.array_equal(ordinal, single[1]))
        crit = max(per_shard) + (merge_ms if G > 1 else 0.0)
        row = {"shards": G, "step_ms_per_shard": [round(x, 3) for x in per_shard],
               "search_kernel_ms_per_shard": [round(x, 3) for x in per_kernel],
               "merge_ms": round(merge_ms, 4), "critical_path_ms": round(crit, 3),
               "queries_per_s": nq / (crit * 1e-3), "speedup_vs_1": single[2] / crit,
               "balance_mean_over_max": float(np.mean(per_shard) / max(per_shard)),
               "merged_equals_single_shard": same}
        rows.append(row)
        print(json.dumps(row), flush=True)
        assert same, "merged candidates differ from the single-shard answer"
    print(json.dumps({"workload": args.workload, "nq": nq, "library": n_lib, "dim": dim,
                      "note": "one GPU, shards timed one after another; all-gather wire time not included",
                      "rows": rows}))


if __name__ == "__main__":
    main()
