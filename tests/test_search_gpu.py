"""GPU: index build, candidate windows, windowed Hamming top-k, sharded merge and the cascade,
bit for bit against the oracle and the golden fixtures, through the C ABI."""
import numpy as np
import pytest

from oracle.binding import PreCfg, SynthCfg, fnv1a64_words
from tests import _util as U

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["tensor_fp4", "popc", "direct", "auto"])
def ctx(hb, request):
    """Every search test runs on all engines: tcgen05 mxf4 (e2m1), XOR+POPC, the warp-per-query
    direct engine, and AUTO (which picks direct or tensor_fp4 per call)."""
    c = hb.Context(0)
    c.set_engine(request.param)
    c.engine_name = request.param
    yield c
    c.close()


def _index(ctx, c):
    dim = int(c["dim"][0])
    ids = [x.decode() for x in c["ids"]]
    ctx.build_index(dim, c["words"], c["mz"], c["charge"], ids=ids, is_decoy=c["decoy"])
    return dim, ids


def test_golden_search_cases(hb, ctx):
    for name, c in U.search_cases().items():
        dim, ids = _index(ctx, c)
        for bi, b in enumerate(ctx.buckets()):  # build_index order, search.cpp:37-46
            assert b["charge"] == int(c[f"bucket{bi}"]["charge"][0])
            assert np.array_equal(b["ordinal"], c[f"bucket{bi}"]["ordinal"]), name
            assert np.array_equal(b["words"], c["words"][b["ordinal"]]), name
            assert np.array_equal(b["precursor_mz"], c["mz"][b["ordinal"]]), name
        for tname, tol in U.TOLS.items():
            g = c[tname]
            first, last, has_b = ctx.select_candidates(c["q_mz"], c["q_charge"], U.product_tol(tol))
            nonempty = g["last"] > g["first"]
            assert np.array_equal(last - first, g["last"] - g["first"]), (name, tname)
            assert np.array_equal(first[nonempty], g["first"][nonempty]), (name, tname)
            assert np.array_equal(has_b, g["has_bucket"])
            m = ctx.search_batch(c["q_words"], c["q_mz"], c["q_charge"], U.product_tol(tol))
            assert np.array_equal(m.has_hit[:, 0], g["has"].astype(bool)), (name, tname)
            assert np.array_equal(m.raw_score[:, 0], g["score"]), (name, tname)
            assert np.array_equal(m.ordinal[:, 0], g["ordinal"]), (name, tname)
        for cname, narrow, wide, fq in (("c1", ("ppm", 150.0), ("da", 30.0), 0.05),
                                        ("c2", ("da", 0.3), ("da", 500.0), 0.5)):
            got = ctx.cascade_search(c["q_words"], c["q_mz"], c["q_charge"], U.product_tol(narrow),
                                     U.product_tol(wide), fq)
            for k in got:
                assert np.array_equal(got[k], c[cname][k]), (name, cname, k)


def test_reference_known_answers(hb, ctx):
    """test_search.cpp:116-171 windows, :205-243 tie-breaks, :173-203 self / empty / mismatch."""
    rng = np.random.default_rng(5)
    ctx.build_index(256, U.random_hvs(rng, 5, 256), [999.9799, 999.98, 1000.0, 1000.02, 1000.0201], [2] * 5)
    f, l, has = ctx.select_candidates([1000.0], [2], hb.Tolerance("ppm", 20.0))
    assert (f[0], l[0]) == (1, 4)
    f, l, has = ctx.select_candidates([1000.0], [2], hb.Tolerance("dalton", 500.0))
    assert l[0] - f[0] == 5
    f, l, has = ctx.select_candidates([1000.0, 1000.0], [5, 0], hb.Tolerance("ppm", 20.0))
    assert not has.any() and (l == f).all()
    ctx.build_index(256, U.random_hvs(rng, 4, 256), [499.99, 500.0, 1500.0, 1500.01], [2] * 4)
    f, l, _ = ctx.select_candidates([1000.0], [2], hb.Tolerance("dalton", 500.0))
    assert (f[0], l[0]) == (1, 3)

    shared = U.random_hvs(rng, 1, 256)
    two = np.repeat(shared, 2, 0)
    da1 = hb.Tolerance("dalton", 1.0)
    ctx.build_index(256, two, [1000.30, 1000.10], [2, 2], ids=["far", "near"])
    assert ctx.search_batch(shared, [1000.0], [2], da1).ordinal[0, 0] == 1
    ctx.build_index(256, two, [999.75, 1000.25], [2, 2], ids=["zz", "aa"])
    assert ctx.search_batch(shared, [1000.0], [2], da1).ordinal[0, 0] == 1
    ctx.build_index(256, two, [1000.0, 1000.0], [2, 2], ids=["dup", "dup"])
    assert ctx.search_batch(shared, [1000.0], [2], da1).ordinal[0, 0] == 0

    refs = U.random_hvs(rng, 50, 256)
    mz = rng.uniform(400, 1200, 50)
    ch = rng.integers(2, 4, 50).astype(np.uint8)
    ctx.build_index(256, refs, mz, ch)
    m = ctx.search_batch(refs[17:18], mz[17:18], ch[17:18], hb.Tolerance("ppm", 20.0))
    assert m.ordinal[0, 0] == 17 and m.raw_score[0, 0] == 256
    m = ctx.search_batch(refs[:1], [2000.0], [2], hb.Tolerance("ppm", 20.0))
    assert not m.has_hit[0, 0] and m.raw_score[0, 0] == 0
    with pytest.raises(hb.InvariantError):  # search.cpp:107-109
        ctx.search_batch(U.random_hvs(rng, 1, 128), [800.0], [2], hb.Tolerance("ppm", 20.0), query_dim=128)
    with pytest.raises(hb.InvariantError):  # search.cpp:18
        ctx.build_index(256, np.zeros((0, 4), np.uint64), [], [])
    with pytest.raises(hb.ConfigError):  # search.cpp:13-15 through cascade :223-224
        ctx.cascade_search(refs[:1], [800.0], [2], hb.Tolerance("ppm", 0.0), hb.Tolerance("dalton", 5.0), 0.01)
    assert ctx.search_batch(np.zeros((0, 4), np.uint64), [], [], da1).ordinal.shape == (0, 1)


def test_config1_search_and_cascade(hb, ctx, best_oracle):
    """BASELINE config 1 end to end on the device: synth -> encode -> index -> open / narrow
    search -> cascade; compared with the golden fingerprints and with the live oracle."""
    fp = U.fingerprints()["config1"]
    s = best_oracle.synth(SynthCfg(n_library=5000, n_query=1000, fraction_modified=0.6, seed=1))
    L, Q = s["library"], s["queries"]
    pre = hb.PreprocessConfig()
    ctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(2048, 1024, 16, 1)))
    lw, _ = ctx.encode_batch(L["offsets"], L["mz"], L["intensity"], pre)
    qw, _ = ctx.encode_batch(Q["offsets"], Q["mz"], Q["intensity"], pre)
    ctx.build_index(2048, lw, L["precursor_mz"], L["charge"], ids=L["ids"], is_decoy=L["is_decoy"])
    m = ctx.search_batch(qw, Q["precursor_mz"], Q["charge"], hb.Tolerance("dalton", 500.0))
    assert int((m.last - m.first).sum()) == fp["open_candidates_total"]
    assert int(m.has_hit.sum()) == fp["open_hits"]
    assert f"{fnv1a64_words(m.raw_score[:, 0].astype(np.uint64)):016x}" == fp["open_score_fnv"]
    assert f"{fnv1a64_words(m.ordinal[:, 0].astype(np.uint64)):016x}" == fp["open_ordinal_fnv"]
    n = ctx.search_batch(qw, Q["precursor_mz"], Q["charge"], hb.Tolerance("ppm", 20.0))
    assert int(n.has_hit.sum()) == fp["narrow_hits"]
    assert f"{fnv1a64_words(n.ordinal[:, 0].astype(np.uint64)):016x}" == fp["narrow_ordinal_fnv"]
    c = ctx.cascade_search(qw, Q["precursor_mz"], Q["charge"], hb.Tolerance("ppm", 20.0),
                           hb.Tolerance("dalton", 500.0), 0.01)
    assert (len(c["query"]), int((c["stage"] == 0).sum()), int((c["stage"] == 1).sum())) == (1000, 385, 615)
    assert f"{fnv1a64_words(c['ordinal'].astype(np.uint64)):016x}" == fp["cascade_ordinal_fnv"]
    assert f"{fnv1a64_words(c['q_value'].view(np.uint64)):016x}" == fp["cascade_qvalue_fnv"]


def test_cascade_behaviours(hb, ctx, best_oracle):
    """The reference's cascade tests (test_search.cpp:329-421) on every engine: exact matches are
    accepted in the narrow stage with score D and q = 0; a +79.97 precursor shift strands the query
    in the wide stage; stages whose top hits are all decoys accept nothing; every query is accepted
    at most once, never on a decoy -- and the accepted list equals the oracle's each time."""
    rng = np.random.default_rng(14)
    dim = 1024
    narrow, wide = hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 500.0)

    def refs(n, decoy_fraction):
        words = U.random_hvs(rng, n, dim)
        mz = rng.uniform(400.0, 1200.0, n)
        charge = rng.integers(2, 4, n).astype(np.uint8)
        decoy = (rng.uniform(0, 1, n) < decoy_fraction).astype(np.uint8)
        return words, mz, charge, decoy, [f"ref_{i}" for i in range(n)]

    def both(lib, qw, qmz, qch, fdr_q):
        words, mz, charge, decoy, ids = lib
        ctx.build_index(dim, words, mz, charge, ids=ids, is_decoy=decoy)
        oix = best_oracle.build_index(dim, words, mz, charge, decoy, ids)
        got = ctx.cascade_search(qw, qmz, qch, narrow, wide, fdr_q)
        want = oix.cascade_search(qw, qmz, qch, ("ppm", 20.0), ("da", 500.0), fdr_q)
        oix.close()
        for key in ("query", "ordinal", "stage", "raw_score"):
            assert np.array_equal(got[key], want[key]), key
        assert np.array_equal(got["q_value"].view(np.uint64), want["q_value"].view(np.uint64))
        return got

    lib = refs(30, 0.0)                                   # :329-346
    got = both(lib, lib[0][[3, 9]], lib[1][[3, 9]], lib[2][[3, 9]], 0.01)
    assert list(got["query"]) == [0, 1] and list(got["ordinal"]) == [3, 9]
    assert (got["stage"] == 0).all() and (got["raw_score"] == dim).all() and (got["q_value"] == 0.0).all()

    lib = refs(30, 0.0)                                   # :348-375
    got = both(lib, lib[0][[5]], lib[1][[5]] + 79.97, lib[2][[5]], 0.01)
    assert list(got["ordinal"]) == [5] and list(got["stage"]) == [1] and list(got["raw_score"]) == [dim]

    lib = refs(20, 1.0)                                   # :377-385 decoys only
    got = both(lib, lib[0][[0, 7, 13]], lib[1][[0, 7, 13]], lib[2][[0, 7, 13]], 0.01)
    assert len(got["query"]) == 0

    lib = refs(200, 0.5)                                  # :387-421
    pick = rng.integers(0, 200, 120)
    qw, qmz, qch = lib[0][pick].copy(), lib[1][pick].copy(), lib[2][pick].copy()
    qmz[1::3] += 40.0
    noise = np.arange(2, 120, 3)
    qw[noise] = U.random_hvs(rng, len(noise), dim)
    qmz[noise] = rng.uniform(450.0, 1150.0, len(noise))
    qch[noise] = 2
    got = both(lib, qw, qmz, qch, 0.05)
    assert len(set(got["query"])) == len(got["query"]) <= 120
    assert not lib[3][got["ordinal"]].any()
    assert set(got["stage"]) <= {0, 1}


@pytest.mark.parametrize("dim", [64, 1024, 2048, 4096, 8192, 16384, 32768, 65536])
def test_random_library_vs_oracle(hb, ctx, best_oracle, dim):
    """Dimension sweep (BASELINE config 5 shapes, small n): random hypervectors, both tolerance
    kinds, clones for ties; top-1 vs the oracle's search_batch."""
    rng = np.random.default_rng(dim)
    n, nq = 3000, 300
    words = U.random_hvs(rng, n, dim)
    words[n - 200:] = words[:200]  # clones -> exact score ties resolved by |diff| / id
    mz = np.round(rng.uniform(400.0, 1200.0, n), 3)
    charge = rng.integers(1, 4, n).astype(np.uint8)
    ids = [f"e{rng.integers(0, 500)}" for _ in range(n)]  # many duplicate ids
    qw = U.random_hvs(rng, nq, dim)
    qw[:100] = words[rng.integers(0, n, 100)]
    qmz = np.round(rng.uniform(380.0, 1220.0, nq), 3)
    qch = rng.integers(0, 5, nq).astype(np.uint8)
    ctx.build_index(dim, words, mz, charge, ids=ids)
    oix = best_oracle.build_index(dim, words, mz, charge, None, ids)
    for tol in (("da", 500.0), ("ppm", 2000.0), ("da", 0.0005)):
        m = ctx.search_batch(qw, qmz, qch, U.product_tol(tol))
        has, score, ordinal, _ = oix.search_batch(qw, qmz, qch, tol, threads=8)
        assert np.array_equal(m.has_hit[:, 0], has.astype(bool)), tol
        assert np.array_equal(m.raw_score[:, 0], score), tol
        assert np.array_equal(m.ordinal[:, 0], ordinal), tol
    oix.close()


def test_topk_vs_port(hb, ctx, port):
    """k > 1 (north-star top-k): equals a full sort of the window on the reference key."""
    rng = np.random.default_rng(17)
    dim, n, nq = 512, 1500, 120
    words = U.random_hvs(rng, n, dim)
    words[1000:] = words[:500]
    mz = np.round(rng.uniform(500.0, 600.0, n), 2)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    ids = [f"id{rng.integers(0, 300)}" for _ in range(n)]
    qw = words[rng.integers(0, n, nq)]
    qmz = np.round(rng.uniform(495.0, 605.0, nq), 2)
    qch = rng.integers(2, 4, nq).astype(np.uint8)
    ctx.build_index(dim, words, mz, charge, ids=ids)
    oix = port.build_index(dim, words, mz, charge, None, ids)
    for tol, k in ((("da", 500.0), 5), (("da", 0.05), 8), (("ppm", 50.0), 3), (("da", 2.0), 1)):
        m = ctx.search_batch(qw, qmz, qch, U.product_tol(tol), k=k)
        score, ordinal = oix.search_topk(qw, qmz, qch, tol, k)
        assert np.array_equal(m.ordinal, ordinal), (tol, k)
        assert np.array_equal(m.raw_score, score), (tol, k)


def test_topk_many_work_items_vs_port(hb, ctx, port):
    """Top-k where every query tile is cut into many work items (20k rows: ~12 strips of at most 8
    row tiles per query tile), so that the tensor engines' per-item k-lists, the published k-th-best
    floor and the list merge are all exercised; heavy score ties (rows duplicated four times, few
    distinct m/z values and ids).  One pass of the tensor / direct engines keeps 32 candidates per query
    (register lists of depth 4 / 8 / 16 / 32); k = 33 ... 64 take a second pass bounded below by the first
    pass's last key -- with rows duplicated four times that key sits inside a run of equal scores, so
    the (|mass diff|, id, ordinal) part of the bound decides."""
    rng = np.random.default_rng(29)
    dim, n, nq = 256, 20000, 300
    base = U.random_hvs(rng, n // 4, dim)
    words = np.concatenate([base, base, base, base])
    mz = np.round(rng.uniform(500.0, 520.0, n), 1)
    charge = np.full(n, 2, np.uint8)
    ids = [f"id{rng.integers(0, 50)}" for _ in range(n)]
    qw = base[rng.integers(0, n // 4, nq)] ^ (U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim)
                                               & U.random_hvs(rng, nq, dim))
    qmz = np.round(rng.uniform(495.0, 525.0, nq), 1)
    qch = np.full(nq, 2, np.uint8)
    ctx.build_index(dim, words, mz, charge, ids=ids)
    oix = port.build_index(dim, words, mz, charge, None, ids)
    ks = ((("da", 500.0), 2), (("da", 500.0), 16), (("da", 3.0), 7), (("da", 500.0), 17), (("da", 500.0), 32),
          (("da", 500.0), 33), (("da", 500.0), 64), (("da", 0.3), 64), (("ppm", 200.0), 40))
    if ctx.engine_name == "popc":  # k full passes on the XOR+POPC engine: keep it short
        ks = ks[:4] + ((("da", 0.3), 64),)
    for tol, k in ks:
        m = ctx.search_batch(qw, qmz, qch, U.product_tol(tol), k=k)
        score, ordinal = oix.search_topk(qw, qmz, qch, tol, k)
        assert np.array_equal(m.ordinal, ordinal), (tol, k)
        assert np.array_equal(m.raw_score, score), (tol, k)
        if ctx.engine_name in ("tensor_fp4", "direct"):  # no fall-back to another engine at any depth
            assert ctx.last_engine() == ctx.engine_name, (tol, k)
    oix.close()


def test_search_fuzz_vs_port(hb, ctx, port):
    """Randomised differential test against the full-sort oracle: random sizes, dimensions (also
    not multiples of 64), k, tolerance kinds and widths (empty windows included), charges with
    missing buckets and charge 0, few distinct hypervectors / m/z values / ids so that every level
    of the tie-break key decides somewhere."""
    rng = np.random.default_rng(20221116)
    for case in range(24):
        dim = int(rng.choice([64, 100, 256, 500, 1024, 2048]))
        n = int(rng.integers(1, 2500))
        nq = int(rng.integers(1, 300))
        k = int(rng.choice([1, 1, 2, 3, 5, 16, 17, 20, 33, 48, 64]))
        distinct = max(1, int(n * rng.choice([0.02, 0.3, 1.0])))
        pool = U.random_hvs(rng, distinct, dim)
        words = pool[rng.integers(0, distinct, n)]
        mz = np.round(rng.uniform(300.0, 300.0 + rng.choice([0.5, 20.0, 900.0]), n), int(rng.choice([0, 1, 3])))
        charge = rng.choice([1, 2, 3, 4], n, p=[0.05, 0.5, 0.4, 0.05]).astype(np.uint8)
        ids = [f"p{rng.integers(0, max(1, n // int(rng.choice([1, 7, 400]))))}" for _ in range(n)]
        flip = U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim)
        qw = pool[rng.integers(0, distinct, nq)] ^ (flip if case % 2 else 0)
        qmz = mz[rng.integers(0, n, nq)] + rng.choice([0.0, 0.0, 0.001, 0.5, -3.0, 450.0], nq)
        qch = rng.choice([0, 1, 2, 3, 5], nq, p=[0.05, 0.05, 0.5, 0.35, 0.05]).astype(np.uint8)
        tol = [("da", 500.0), ("da", 0.0005), ("da", 2.0), ("ppm", 10.0), ("ppm", 5000.0), ("da", 40.0)][case % 6]
        ctx.build_index(dim, words, mz, charge, ids=ids)
        oix = port.build_index(dim, words, mz, charge, None, ids)
        m = ctx.search_batch(qw, qmz, qch, U.product_tol(tol), k=k)
        score, ordinal = oix.search_topk(qw, qmz, qch, tol, k)
        oix.close()
        assert np.array_equal(m.ordinal, ordinal), (case, dim, n, nq, k, tol)
        assert np.array_equal(m.raw_score, score), (case, dim, n, nq, k, tol)


def test_sharded_search_merges_to_single(hb):
    """Multi-GPU path on one device: G contexts each hold slice g of every bucket; per-shard
    candidates -> concatenate (what the all-gather yields) -> merge == unsharded result."""
    import torch
    rng = np.random.default_rng(23)
    dim, n, nq = 1024, 4000, 200
    words = U.random_hvs(rng, n, dim)
    words[3500:] = words[:500]
    mz = np.round(rng.uniform(400.0, 1200.0, n), 2)
    charge = rng.integers(2, 5, n).astype(np.uint8)
    ids = [f"x{rng.integers(0, 900)}" for _ in range(n)]
    qw = words[rng.integers(0, n, nq)]
    qmz = mz[rng.integers(0, n, nq)] + rng.choice([0.0, 0.01, 40.0], nq)
    qch = rng.integers(2, 5, nq).astype(np.uint8)
    with hb.Context(0) as single:
        single.build_index(dim, words, mz, charge, ids=ids)
        # k = 3 keeps per-item k-lists in the tensor engine's drain, k = 1 is the plain top-1 path
        for tol, k in ((hb.Tolerance("dalton", 500.0), 3), (hb.Tolerance("ppm", 30.0), 3),
                       (hb.Tolerance("dalton", 500.0), 1), (hb.Tolerance("ppm", 30.0), 1)):
            want = single.search_batch(qw, qmz, qch, tol, k=k)
            for G in (2, 3, 8):
                gathered = torch.zeros(G, nq * k * 16, dtype=torch.uint8, device="cuda")
                shards = [hb.Context(0) for _ in range(G)]
                covered = 0
                for g, c in enumerate(shards):
                    c.build_index(dim, words, mz, charge, ids=ids, shard_index=g, shard_count=G)
                    covered += sum(b["shard_end"] - b["shard_begin"] for b in c.buckets())
                    c.queries_upload(dim, qw, qmz, qch)
                    c.search_resident_dev(tol, k, gathered[g].data_ptr())
                    c.synchronize()
                assert covered == n  # the slices partition the library
                out = torch.zeros(nq * k * 16, dtype=torch.uint8, device="cuda")
                shards[0].merge_candidates_dev(nq, k, G, gathered.data_ptr(), out.data_ptr())
                score, ordinal = shards[0].candidates_decode(nq, k, out.data_ptr())
                for c in shards:
                    c.close()
                assert np.array_equal(ordinal, want.ordinal), (tol, k, G)
                assert np.array_equal(score, want.raw_score), (tol, k, G)


def test_large_open_search_properties(hb, ctx):
    """Size-independent properties at a larger scale (D = 8192, 60k rows, many work items):
    self-search returns the entry itself with score D, and widening the tolerance never lowers
    the best score (test_search.cpp:280-296)."""
    rng = np.random.default_rng(31)
    dim, n, nq = 8192, 60000, 512
    words = U.random_hvs(rng, n, dim)
    mz = rng.uniform(400.0, 1200.0, n)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    ctx.build_index(dim, words, mz, charge)
    pick = rng.integers(0, n, nq)
    m = ctx.search_batch(words[pick], mz[pick], charge[pick], hb.Tolerance("dalton", 500.0))
    assert (m.raw_score[:, 0] == dim).all()
    # the entry itself or an exact duplicate position cannot exist in a random library
    assert np.array_equal(m.ordinal[:, 0], pick.astype(np.uint32))
    qw = U.random_hvs(rng, nq, dim)
    prev = np.zeros(nq, np.uint32)
    for da in (1.0, 5.0, 25.0, 125.0, 700.0):
        s = ctx.search_batch(qw, mz[pick], charge[pick], hb.Tolerance("dalton", da)).raw_score[:, 0]
        assert (s >= prev).all()
        prev = s


@pytest.mark.parametrize("dim", [128, 2048])
def test_many_queries_span_planning_batches(hb, best_oracle, dim):
    """More than 65536 queries: the tensor engine plans in batches of 64k sorted slots (single CTAs with resident
    query chunks at D = 128, CTA pairs at D = 2048); results must equal the POPC engine's and (on a sample) the
    oracle's.  Also: a query set that reaches no bucket at all (no work items)."""
    rng = np.random.default_rng(41)
    n, nq = 3000, 70000
    words = U.random_hvs(rng, n, dim)
    words[2500:] = words[:500]
    mz = np.round(rng.uniform(400.0, 1200.0, n), 2)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    ids = [f"m{rng.integers(0, 700)}" for _ in range(n)]
    qw = words[rng.integers(0, n, nq)] ^ U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim)
    qmz = np.round(rng.uniform(380.0, 1220.0, nq), 2)
    qch = rng.integers(1, 4, nq).astype(np.uint8)
    got = {}
    for eng in ("tensor_fp4", "popc", "direct"):
        with hb.Context(0) as c:
            c.set_engine(eng)
            c.build_index(dim, words, mz, charge, ids=ids)
            got[eng] = c.search_batch(qw, qmz, qch, hb.Tolerance("dalton", 3.0))
            got[eng + "/k3"] = c.search_batch(qw, qmz, qch, hb.Tolerance("dalton", 3.0), k=3)
            none = c.search_batch(qw[:300], qmz[:300], np.zeros(300, np.uint8), hb.Tolerance("dalton", 3.0))
            assert not none.has_hit.any()
    for eng in ("tensor_fp4", "direct"):
        assert np.array_equal(got[eng].ordinal, got["popc"].ordinal), eng
        assert np.array_equal(got[eng].raw_score, got["popc"].raw_score), eng
        # top-3 across planning batches: per-item lists, class-slot floors and the list merge
        assert np.array_equal(got[eng + "/k3"].ordinal, got["popc/k3"].ordinal), eng
        assert np.array_equal(got[eng + "/k3"].raw_score, got["popc/k3"].raw_score), eng
        assert np.array_equal(got[eng + "/k3"].ordinal[:, 0], got["popc"].ordinal[:, 0]), eng
    oix = best_oracle.build_index(dim, words, mz, charge, None, ids)
    sample = rng.integers(0, nq, 2000)
    has, score, ordinal, _ = oix.search_batch(qw[sample], qmz[sample], qch[sample], ("da", 3.0), threads=8)
    assert np.array_equal(got["tensor_fp4"].ordinal[sample, 0], ordinal)
    assert np.array_equal(got["tensor_fp4"].raw_score[sample, 0], score)
    oix.close()


def test_planner_under_a_tight_item_capacity(hb, monkeypatch):
    """The device planner must never emit more work items than the item / partial arrays hold: with
    the capacity forced far below what the shape asks for (the path a huge top-16 search takes when
    4 GB of partials is the limit) the strips get longer and the answers stay the same -- also when
    the capacity is down at the planner's slack (2 items per query tile + 16) and every query tile
    becomes a single item."""
    rng = np.random.default_rng(61)
    dim, n, nq = 256, 40000, 3000
    words = U.random_hvs(rng, n, dim)
    words[30000:] = words[:10000]
    mz = np.round(rng.uniform(400.0, 1200.0, n), 2)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    qw = words[rng.integers(0, n, nq)]
    qmz = np.round(rng.uniform(380.0, 1220.0, nq), 2)
    qch = rng.integers(2, 4, nq).astype(np.uint8)
    tol = hb.Tolerance("dalton", 500.0)
    with hb.Context(0) as c:
        c.set_engine("tensor_fp4")
        c.build_index(dim, words, mz, charge)
        want = {k: c.search_batch(qw, qmz, qch, tol, k=k) for k in (1, 3)}
    for cap in ("400", "120", "10"):
        monkeypatch.setenv("HOMS_B200_TC_ITEM_CAP", cap)  # read once, when the context is created
        with hb.Context(0) as c:
            c.set_engine("tensor_fp4")
            c.build_index(dim, words, mz, charge)
            for k in (1, 3):
                got = c.search_batch(qw, qmz, qch, tol, k=k)
                assert np.array_equal(got.ordinal, want[k].ordinal), (cap, k)
                assert np.array_equal(got.raw_score, want[k].raw_score), (cap, k)
    monkeypatch.delenv("HOMS_B200_TC_ITEM_CAP")


def test_concurrent_callers(hb):
    """The reference's calls are synchronous and re-entrant.  Here: threads that
    share ONE context are serialised by its mutex, threads with their OWN contexts run on their own
    streams; either way every call returns the serial answer."""
    import threading
    rng = np.random.default_rng(53)
    dim, n, nq = 1024, 30000, 2000
    words = U.random_hvs(rng, n, dim)
    words[25000:] = words[:5000]
    mz = np.round(rng.uniform(400.0, 1200.0, n), 2)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    qw = words[rng.integers(0, n, nq)] ^ (U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim))
    qmz = np.round(rng.uniform(380.0, 1220.0, nq), 2)
    qch = rng.integers(2, 4, nq).astype(np.uint8)
    tols = [hb.Tolerance("dalton", 500.0), hb.Tolerance("ppm", 30.0), hb.Tolerance("dalton", 5.0)]
    shared = hb.Context(0)
    shared.build_index(dim, words, mz, charge)
    want = [shared.search_batch(qw, qmz, qch, t, k=2) for t in tols]
    own = [hb.Context(0) for _ in range(3)]
    for c in own:
        c.build_index(dim, words, mz, charge)
    errors = []

    def worker(c, i):
        try:
            for rep in range(6):
                j = (i + rep) % len(tols)
                got = c.search_batch(qw, qmz, qch, tols[j], k=2)
                if not (np.array_equal(got.ordinal, want[j].ordinal) and np.array_equal(got.raw_score, want[j].raw_score)):
                    errors.append((i, rep, j))
        except Exception as exc:  # surfaced below: an exception in a thread would otherwise be lost
            errors.append((i, repr(exc)))

    threads = [threading.Thread(target=worker, args=(shared, i)) for i in range(3)]
    threads += [threading.Thread(target=worker, args=(c, i)) for i, c in enumerate(own)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for c in own + [shared]:
        c.close()
    assert not errors, errors


def test_engine_selection_errors(hb):
    with hb.Context(0) as c:
        with pytest.raises(hb.HomsError):
            c.set_engine(7)
        c.set_engine("popc")
        rng = np.random.default_rng(3)
        c.build_index(256, U.random_hvs(rng, 10, 256), np.linspace(500, 600, 10), [2] * 10)
        with pytest.raises(hb.HomsError):  # no tensor image was built for this library
            c.set_engine("tensor_fp4")
        c.set_engine("auto")
        c.build_index(256, U.random_hvs(rng, 10, 256), np.linspace(500, 600, 10), [2] * 10)
        c.set_engine("tensor_fp4")  # auto builds the e2m1 image
        c.set_engine("tensor")      # ABI 1's int8 code: now an alias of tensor_fp4
        got = c.search_batch(U.random_hvs(rng, 4, 256), [550.0] * 4, [2] * 4, hb.Tolerance("dalton", 500.0))
        assert c.last_engine() == "tensor_fp4" and got.has_hit.all()


@pytest.mark.parametrize("mode", ["default", "collect", "collect_overflow", "collect_tiny_stage", "lists"])
def test_tensor_topk_modes_vs_port(hb, port, monkeypatch, mode):
    """The tensor engine's top-k paths against the full-sort oracle on tie-heavy data: collect + select (default),
    the same with a candidate buffer so small that (nearly) every query overflows and the fix-up list passes
    produce the answer, a buffer that holds everything but far more survivors than the selection stages
    (rows duplicated: hundreds of equal scores), and the register-list passes alone."""
    if mode.startswith("collect"):
        monkeypatch.setenv("HOMS_B200_TC_TOPK", "collect")  # also for the shallow k the default serves from lists
    if mode == "collect_overflow":
        monkeypatch.setenv("HOMS_B200_TC_CCAP", "24")
    elif mode == "collect_tiny_stage":
        monkeypatch.setenv("HOMS_B200_TC_CCAP", "8192")
    elif mode == "lists":
        monkeypatch.setenv("HOMS_B200_TC_TOPK", "lists")
    rng = np.random.default_rng(37)
    dim, n, nq = 256, 24000, 400
    n_base = n // 600 if mode == "collect_tiny_stage" else n // 4  # 600 copies of every row: > 256 ties at the top
    base = U.random_hvs(rng, n_base, dim)
    words = base[np.arange(n) % n_base]
    mz = np.round(rng.uniform(500.0, 520.0, n), 1)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    ids = [f"id{rng.integers(0, 50)}" for _ in range(n)]
    qw = base[rng.integers(0, n_base, nq)] ^ (U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim)
                                               & U.random_hvs(rng, nq, dim))
    qmz = np.round(rng.uniform(495.0, 525.0, nq), 1)
    qch = rng.integers(1, 4, nq).astype(np.uint8)
    oix = port.build_index(dim, words, mz, charge, None, ids)
    with hb.Context(0) as c:
        c.set_engine("tensor_fp4")
        c.build_index(dim, words, mz, charge, ids=ids)
        for tol, k in ((("da", 500.0), 2), (("da", 500.0), 16), (("da", 500.0), 33), (("da", 500.0), 64), (("da", 2.0), 5),
                       (("ppm", 300.0), 64)):
            m = c.search_batch(qw, qmz, qch, U.product_tol(tol), k=k)
            score, ordinal = oix.search_topk(qw, qmz, qch, tol, k)
            assert np.array_equal(m.ordinal, ordinal), (mode, tol, k)
            assert np.array_equal(m.raw_score, score), (mode, tol, k)
            assert c.last_engine() == "tensor_fp4"
        # the cascade and top-1 do not go through this path; a sharded library (two members on one device) does
        with hb.Context(devices=[0, 0]) as grp:
            grp.set_engine("tensor_fp4")
            grp.build_index(dim, words, mz, charge, ids=ids)
            got = grp.search_batch(qw, qmz, qch, hb.Tolerance("dalton", 500.0), k=40)
            score, ordinal = oix.search_topk(qw, qmz, qch, ("da", 500.0), 40)
            assert np.array_equal(got.ordinal, ordinal) and np.array_equal(got.raw_score, score), mode
    oix.close()


@pytest.mark.parametrize("n", [1, 2, 511, 512, 513, 4095, 4096, 4097, 12289])
def test_index_order_at_sort_tile_boundaries(hb, port, n):
    """build_index's (charge, precursor m/z, id, ordinal) order comes from the library's own stable LSD radix sort
    (csrc/radix.cu: 512-element warp chunks, 4096-element tiles): sizes around those boundaries, heavy ties on
    every key level (few distinct m/z values incl. -0.0 / +0.0 and negative ones, duplicate ids, one or many
    charges), against the oracle's comparison sort (search.cpp:37-46)."""
    rng = np.random.default_rng(1000 + n)
    dim = 128
    words = U.random_hvs(rng, n, dim)
    mz = rng.choice(np.array([-3.5, -0.0, 0.0, 1e-300, 380.25, 380.25000000000006, 1070.5, 1e9]), n)
    charge = rng.integers(1, 6 if n > 100 else 2, n).astype(np.uint8)
    ids = [f"s{rng.integers(0, max(2, n // 3))}" for _ in range(n)]
    oix = port.build_index(dim, words, mz, charge, None, ids)
    with hb.Context(0) as c:
        c.build_index(dim, words, mz, charge, ids=ids)
        got = c.buckets()
        want = oix.buckets()
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert g["charge"] == w["charge"]
            assert np.array_equal(g["ordinal"], w["ordinal"]), (n, g["charge"])
            assert np.array_equal(g["precursor_mz"], w["precursor_mz"]), (n, g["charge"])
            assert np.array_equal(g["words"], w["words"]), (n, g["charge"])
    oix.close()


@pytest.mark.parametrize("form,dim", [("pair", 256), ("pair", 1024), ("single", 2048), ("single", 8192)])
def test_tensor_kernel_forms_vs_port(hb, port, monkeypatch, form, dim):
    """Both forms of the tensor search kernel whatever the dimension: one CTA per SM (M = 128 tiles) and CTA pairs
    (cta_group::2, M = 256 tiles over a 2-CTA cluster, default from D = 2048 up).  An odd number of 128-query
    tiles (the pair's second half is empty), several planning tiles, top-1, collected top-k, the register-list
    passes and a sharded group -- against the full-sort oracle."""
    monkeypatch.setenv("HOMS_B200_TC_PAIR", "1" if form == "pair" else "0")
    rng = np.random.default_rng(91 + dim)
    n, nq = (24000, 700) if dim < 8192 else (6000, 300)
    base = U.random_hvs(rng, n // 4, dim)
    words = base[np.arange(n) % (n // 4)]  # every row four times: ties on the score
    mz = np.round(rng.uniform(500.0, 530.0, n), 2)
    charge = rng.integers(2, 4, n).astype(np.uint8)
    ids = [f"id{rng.integers(0, 80)}" for _ in range(n)]
    qw = base[rng.integers(0, n // 4, nq)] ^ (U.random_hvs(rng, nq, dim) & U.random_hvs(rng, nq, dim))
    qmz = np.round(rng.uniform(495.0, 535.0, nq), 2)
    qch = rng.integers(1, 4, nq).astype(np.uint8)
    oix = port.build_index(dim, words, mz, charge, None, ids)
    with hb.Context(0) as c:
        c.set_engine("tensor_fp4")
        c.build_index(dim, words, mz, charge, ids=ids)
        for tol, k in ((("da", 500.0), 1), (("da", 3.0), 1), (("da", 500.0), 5), (("ppm", 4000.0), 40)):
            m = c.search_batch(qw, qmz, qch, U.product_tol(tol), k=k)
            score, ordinal = oix.search_topk(qw, qmz, qch, tol, k)
            assert np.array_equal(m.ordinal, ordinal), (form, dim, tol, k)
            assert np.array_equal(m.raw_score, score), (form, dim, tol, k)
            assert c.last_engine() == "tensor_fp4"
    monkeypatch.setenv("HOMS_B200_TC_TOPK", "lists")
    with hb.Context(devices=[0, 0, 0]) as grp:
        grp.set_engine("tensor_fp4")
        grp.build_index(dim, words, mz, charge, ids=ids)
        got = grp.search_batch(qw, qmz, qch, hb.Tolerance("dalton", 500.0), k=7)
        score, ordinal = oix.search_topk(qw, qmz, qch, ("da", 500.0), 7)
        assert np.array_equal(got.ordinal, ordinal) and np.array_equal(got.raw_score, score), (form, dim)
    oix.close()


def test_tensor_cta_pairs_by_dimension(hb, monkeypatch):
    """homs_b200_ctx_tensor_cta_pairs: CTA pairs (cta_group::2) serve the resident library from D = 2048 up on a
    device that co-schedules a 2-CTA cluster on every SM pair (a B200 does); HOMS_B200_TC_PAIR forces either form."""
    rng = np.random.default_rng(3)
    for dim, want in ((256, False), (1024, False), (2048, True), (8192, True)):
        with hb.Context(0) as c:
            c.build_index(dim, U.random_hvs(rng, 64, dim), np.linspace(500.0, 600.0, 64), np.full(64, 2, np.uint8))
            assert c.tensor_cta_pairs() == want, dim
    monkeypatch.setenv("HOMS_B200_TC_PAIR", "0")
    with hb.Context(0) as c:
        c.build_index(4096, U.random_hvs(rng, 64, 4096), np.linspace(500.0, 600.0, 64), np.full(64, 2, np.uint8))
        assert not c.tensor_cta_pairs()
    monkeypatch.setenv("HOMS_B200_TC_PAIR", "1")
    with hb.Context(0) as c:
        c.build_index(256, U.random_hvs(rng, 64, 256), np.linspace(500.0, 600.0, 64), np.full(64, 2, np.uint8))
        assert c.tensor_cta_pairs()
