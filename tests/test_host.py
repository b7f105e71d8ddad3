"""CPU tests of the product's host side: the C-ABI library loads and exports
every declared symbol, the CSR/CSC build is bit-exact against the oracle
(ratings.cpp:28-89), random_init and the backtracking search match, and the
synthetic BASELINE generator meets its contract.  No device calls."""
import os
import re

import numpy as np
import pytest

import paper_1508_03110_b200 as P
from oracle.pyoracle import Oracle, OracleRatings
from support import movielens_like, random_ratings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "alsncg_capi.h")).read()
    declared = set(re.findall(r"\b(alsncg_[a-z0-9_]+)\s*\(", header))
    declared -= {"alsncg_snapshot_fn"}
    lib = P.lib()
    missing = [name for name in sorted(declared) if not hasattr(lib, name)]
    assert not missing, missing
    assert declared <= set(P._lib.SIGNATURES), declared - set(P._lib.SIGNATURES)
    assert lib.alsncg_abi_version() == 1
    assert lib.alsncg_row_stride(25) == 26 and lib.alsncg_row_stride(100) == 100
    assert lib.alsncg_max_rank() >= 200


def _csr_equal(R, O):
    for a, b in [(R.uptr, O.uptr), (R.iptr, O.iptr), (R.uidx, O.uidx), (R.iidx, O.iidx),
                 (R.uval, O.uval), (R.ival, O.ival)]:
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_csr_csc_bit_exact_vs_oracle(seed):
    T = movielens_like(60, 25, 0.3, 50 + seed)
    perm = np.random.default_rng(seed).permutation(len(T))  # input order must not matter
    R = P.RatingsMatrix.from_triples(T.n_u, T.n_m, users=T.users[perm], items=T.items[perm],
                                     values=T.values[perm])
    O = OracleRatings(T.n_u, T.n_m, T.users, T.items, T.values)
    _csr_equal(R, O)
    R.check_consistent()


def test_csr_single_precision_and_empty_rows():
    # test_core.cpp:134-142; rows/columns with no ratings
    T = random_ratings(7, 9, 0.2, 3)
    R = P.RatingsMatrix.from_triples(T.n_u + 2, T.n_m + 3, users=T.users, items=T.items,
                                     values=T.values + 0.1, single_precision_storage=True)
    O = OracleRatings(T.n_u + 2, T.n_m + 3, T.users, T.items, T.values + 0.1, single=True)
    _csr_equal(R, O)
    assert R.user_count(T.n_u + 1) == 0 and R.item_count(T.n_m + 2) == 0
    r1 = P.RatingsMatrix.from_triples(1, 1, [(0, 0, 0.1)], True)
    assert r1.user_values(0)[0] == np.float32(0.1)
    empty = P.RatingsMatrix.from_triples(3, 2, [])
    assert empty.nnz() == 0 and list(empty.uptr) == [0, 0, 0, 0]


def test_csr_rejects_bad_input():
    # test_core.cpp:125-132
    with pytest.raises(P.DataError):
        P.RatingsMatrix.from_triples(2, 2, [(0, 2, 1.0)])
    with pytest.raises(P.DataError):
        P.RatingsMatrix.from_triples(2, 2, [(-1, 0, 1.0)])
    with pytest.raises(P.DataError):
        P.RatingsMatrix.from_triples(2, 2, [(0, 0, float("nan"))])
    with pytest.raises(P.DuplicateRatingError) as e:
        P.RatingsMatrix.from_triples(2, 2, [(1, 1, 1.0), (0, 1, 2.0), (1, 1, 3.0), (0, 1, 4.0)])
    assert (e.value.user, e.value.item) == (0, 1)  # first duplicate in (user,item) order


def test_random_init_matches_reference_stream():
    o = Oracle("port").random_init(7, 13, 5, 42)
    m = P.random_init(7, 13, 5, 42)
    assert np.array_equal(np.concatenate([m.user_data, m.item_data]), o)


def test_backtracking_kats():
    # test_linesearch.cpp:98-138
    ls = P.linesearch
    r = ls.backtracking_search(P.QuarticPoly([1.0, -2.0, 1.0, 0.0, 0.0]), -2.0, 10.0, 0.5, 0.9, 100)
    assert r.status == ls.LineSearchStatus.kAccepted and r.backtracks == 22
    a = 10.0
    for _ in range(22):
        a *= 0.9
    assert r.alpha == a
    r = ls.backtracking_search(P.QuarticPoly([5.0, -1.0, 0, 0, 0]), -1.0, 2.0, 0.5, 0.9, 100)
    assert (r.status, r.alpha, r.backtracks) == (ls.LineSearchStatus.kAccepted, 2.0, 0)
    q = P.QuarticPoly([1.0, 1.0, 0, 0, 0])
    assert ls.backtracking_search(q, 0.0, 1.0, 0.5, 0.9, 10).status == ls.LineSearchStatus.kNotDescent
    assert ls.backtracking_search(q, 1.0, 1.0, 0.5, 0.9, 10).status == ls.LineSearchStatus.kNotDescent
    r = ls.backtracking_search(P.QuarticPoly([3.0, 0, 0, 0, 0]), -1.0, 1.0, 0.5, 0.9, 10)
    assert r.status == ls.LineSearchStatus.kMaxBacktracks and r.backtracks == 10
    with pytest.raises(ValueError):
        ls.backtracking_search(q, -1.0, 0.0, 0.5, 0.9, 10)


def test_backtracking_random_vs_oracle():
    rng = np.random.default_rng(0)
    orc = Oracle("port")
    for _ in range(300):
        c = rng.normal(size=5)
        c[1] = -abs(c[1])
        slope = c[1]
        st, a, k = orc.backtracking(c, slope, 10.0, 0.5, 0.9, 100)
        r = P.linesearch.backtracking_search(P.QuarticPoly(list(c)), slope, 10.0, 0.5, 0.9, 100)
        assert (int(r.status), r.alpha, r.backtracks) == (st, a, k)


def test_solver_config_validation():
    # test_core.cpp:160-174
    c = P.SolverConfig()
    c.validate()
    c.tau = 1.5
    with pytest.raises(ValueError):
        c.validate()
    c = P.SolverConfig(lambda_=-0.1)
    with pytest.raises(ValueError):
        c.validate()
    assert P.SolverConfig(n_blocks=0, n_workers=3).resolved_blocks() == 3


def test_trace_ordering_invariants():
    # test_core.cpp:150-158
    t = P.ConvergenceTrace()
    t.append(P.TraceRecord(0, 1.0, 1.0, 0.0))
    t.append(P.TraceRecord(1, 0.5, 0.5, 0.1))
    with pytest.raises(AssertionError):
        t.append(P.TraceRecord(1, 0.4, 0.4, 0.2))
    with pytest.raises(AssertionError):
        t.append(P.TraceRecord(2, 0.4, 0.4, 0.05))


def test_quartic_poly_horner():
    q = P.QuarticPoly([1.0, -2.0, 3.0, 0.5, 0.25])
    for a in (0.0, 0.3, 1.0, 2.7):
        d = 1.0 - 2.0 * a + 3.0 * a * a + 0.5 * a ** 3 + 0.25 * a ** 4
        assert abs(q(a) - d) <= 1e-14 * max(1.0, abs(d))


def test_synth_generator_contract():
    R = P.generate(0)
    assert (R.n_users(), R.n_items(), R.nnz()) == (1000, 500, 20000)
    assert np.all(np.diff(R.uptr) == 20)  # config 0: exactly 20 per user
    v = R.uval
    assert v.min() >= 0.5 and v.max() <= 5.0 and np.all(v * 2 == np.round(v * 2))
    cnt = np.diff(R.iptr)
    assert cnt[0] > cnt[50] > cnt[400]  # Zipf head
    again = P.generate(0)
    assert again.uidx.tobytes() == R.uidx.tobytes() and again.uval.tobytes() == R.uval.tobytes()
    u, i, val = P.synth.generate_triples(300, 200, 300 * 20 + 4567, 7)
    assert len(u) == 300 * 20 + 4567 and np.bincount(u).min() >= 20


def _big_triples(seed, n_u=40_000, n_m=3_000, nnz=1_500_000):
    """A ~1.5M-rating instance (multi-threaded CSR build), shuffled input order."""
    rng = np.random.default_rng(seed)
    key = rng.choice(n_u * n_m, size=nnz, replace=False)
    rng.shuffle(key)
    users = (key // n_m).astype(np.int32)
    items = (key % n_m).astype(np.int32)
    values = np.round(rng.uniform(0.5, 5.0, nnz) * 2) / 2
    return n_u, n_m, users, items, values


def test_csr_threaded_build_bit_exact_and_errors_vs_oracle():
    n_u, n_m, u, i, v = _big_triples(5)
    R = P.RatingsMatrix.from_triples(n_u, n_m, users=u, items=i, values=v)
    O = OracleRatings(n_u, n_m, u, i, v)
    _csr_equal(R, O)
    # the first bad triple in INPUT order is the one reported
    u2, v2 = u.copy(), v.copy()
    u2[900_000] = n_u + 5
    v2[300_000] = np.nan
    with pytest.raises(P.DataError, match="non-finite"):
        P.RatingsMatrix.from_triples(n_u, n_m, users=u2, items=i, values=v2)
    with pytest.raises(P.DataError, match=f"user {n_u + 5}"):
        P.RatingsMatrix.from_triples(n_u, n_m, users=u2, items=i, values=v)
    # duplicates: the first one in (user, item) order is reported (ratings.cpp:47-51)
    u3, i3 = u.copy(), i.copy()
    for a, b in ((1_200_000, 10), (50, 700_000)):
        u3[a], i3[a] = u3[b], i3[b]
    first = min((int(u3[b]), int(i3[b])) for b in (10, 700_000))
    with pytest.raises(P.DuplicateRatingError, match=f"user {first[0]}, item {first[1]}"):
        P.RatingsMatrix.from_triples(n_u, n_m, users=u3, items=i3, values=v)


def test_threaded_generator_bitwise_vs_sequential_oracle():
    # odd truth-normal count (spare carried into the rating noise) and a
    # multi-chunk stream: 97 users x 61 items, then 50k users
    from oracle.pyoracle import synth_triples
    for (n_u, n_m, nnz, seed) in ((97, 61, 2_100, 7), (50_001, 2_001, 3_000_000, 11)):
        a = synth_triples(n_u, n_m, nnz, seed)
        b = P.synth.generate_triples(n_u, n_m, nnz, seed)
        for x, y in zip(a, b):
            assert x.tobytes() == y.tobytes()


def test_mt_jump_table_jumps_the_generator():
    # csrc/mt_jump_table.inc (tools/gen_mt_jump.py): g(T) s for the first two
    # polynomials equals stepping std::mt19937_64 by 312*256 and 8*312*256
    # draws; the other two are the 8th powers of their predecessors mod phi
    # (checked when the table is generated).
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gen_mt_jump", os.path.join(root, "tools", "gen_mt_jump.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    polys = g.read_table(os.path.join(root, "paper_1508_03110_b200", "csrc", "mt_jump_table.inc"))
    s0 = g.seed_state(20260101)
    ref = g.words(s0, g.JUMPS[1] + g.N)
    for p in (0, 1):
        assert g.same_state(g.jump(s0, polys[p]), ref[g.JUMPS[p]:g.JUMPS[p] + g.N])
