#!/usr/bin/env python
"""Library start-up path: cache image -> resident index.

ours:       homs_b200_library_load_cache  (block -> HBM, FNV-1a-64 on the device, device gather, tensor image)
reference:  read_cache + build_index of the compiled reference (oracle/_ref), same image, host cores
Prints one JSON line.  Usage: python tools/bench_loader.py [n_library] [dim]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2211_16422_b200 as hb  # noqa: E402
from paper_2211_16422_b200 import capi  # noqa: E402


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_200_000
    dim = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    rng = np.random.default_rng(1)
    W = dim // 64
    pre, enc = hb.PreprocessConfig(), hb.EncoderConfig(dim, dim // 2, 16, 1)
    d_words = torch.randint(-2**63, 2**63 - 1, (n, W), dtype=torch.int64, device="cuda")
    mz = rng.uniform(380.0, 1070.0, n)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    decoy = (np.arange(n) % 2).astype(np.uint8)
    ids = [("DECOY_%07d" if i % 2 else "LIB_%07d") % i for i in range(n)]
    peps = ["PEPTIDEK"] * n
    out = {"n_library": n, "dim": dim}
    with hb.Context(0) as ctx:
        t = time.perf_counter()
        image = ctx.cache_write(pre, enc, None, mz, charge, decoy, ids, peps, d_words=d_words.data_ptr())
        out["write_from_device_s"] = time.perf_counter() - t
        out["image_bytes"] = len(image)
        del d_words
        buf = np.frombuffer(image, np.uint8)
        cnt = capi.C.c_uint64()
        for rep in range(2):  # the C-ABI call alone (what a C++ host pays); second run is warm
            t = time.perf_counter()
            rc = capi.library_load_cache(ctx.handle, buf.ctypes.data, len(buf), capi.C.byref(pre.pod()),
                                         capi.C.byref(enc.pod()), 0, 1, capi.C.byref(cnt))
            ctx.synchronize()
            assert rc == 0 and cnt.value == n
            out["load_s"] = time.perf_counter() - t
            print(json.dumps(out), file=sys.stderr, flush=True)
        # checksum alone, device resident
        blk = torch.frombuffer(bytearray(image[-(n * W * 8 + 8):-8]), dtype=torch.uint8).cuda()
        dig = capi.C.c_uint64()
        torch.cuda.synchronize()
        t = time.perf_counter()
        capi.fnv1a64_dev(ctx.handle, blk.data_ptr(), blk.numel(), capi.C.byref(dig))
        out["fnv_device_s"] = time.perf_counter() - t
        out["fnv_device_GBps"] = blk.numel() / out["fnv_device_s"] / 1e9
    print(json.dumps(out), file=sys.stderr, flush=True)
    from oracle import binding as ob
    if ob.available("ref") and "--no-reference" not in sys.argv:
        o = ob.Oracle("ref")
        C = capi.C
        cbuf = (C.c_ubyte * len(image)).from_buffer_copy(image)
        t = time.perf_counter()  # validation-only form: exactly one homs::read_cache of the image
        got = o._cache_read(cbuf, len(image), C.byref(ob.PreCfg()), C.byref(ob.EncCfg(dim, dim // 2, 16, 1)),
                            *([None] * 8))
        out["reference_read_cache_s"] = time.perf_counter() - t
        assert got == n
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
