"""The CUDA path against the committed goldens that the REFERENCE ITSELF
produced (tests/golden/, tests/golden/make_golden.py, oracle/_ref):

  * config 0: ALS-NCG and ALS traces (iteration, backtracks, restarts,
    shuffled columns identical; loss within 1e-9, grad norm within 1e-7
    relative), final model within 1e-8;
  * config 0 at x0: loss 1e-12, gradient 1e-11, quartic 1e-12, user
    half-sweep 1e-9 relative;
  * config 1 to (1/N)||g|| < 1e-6 (ncg.cpp:283-286) against the reference's
    run: the same decision sequence over a 60-iteration prefix, end state and
    iteration count within 10 % (see the test's docstring for why the count
    itself is rounding-sensitive on this problem).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1508_03110_b200 as P

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("algo", ["ncg", "als"])
def test_config0_trace_matches_reference_golden(algo):
    g = load("c0_trace.json")
    c, s = g["config"], g[algo]["solver"]
    R = P.generate(0)
    cfg = P.SolverConfig(lambda_=c["lam"], n_f=c["n_f"], max_iters=s["max_iters"], tol=s["tol"],
                         seed=s["seed"], n_blocks=s["n_blocks"])
    res = (P.ncg.als_ncg_solve if algo == "ncg" else P.als.als_solve)(R, cfg)
    recs = res.trace.records
    assert len(recs) == len(g[algo]["trace"])
    for a, b in zip(recs, g[algo]["trace"]):
        assert (a.iter, a.backtracks, a.restarted, a.shuffled_columns) == \
            (b["iter"], b["backtracks"], b["restarted"], b["shuffled_columns"])
        assert abs(a.loss - b["loss"]) <= 1e-9 * abs(b["loss"])
        assert abs(a.grad_norm - b["grad_norm"]) <= 1e-7 * b["grad_norm"]
    x = np.concatenate([res.model.user_data, res.model.item_data])
    assert abs(np.linalg.norm(x) - g[algo]["model_norm"]) <= 1e-8 * g[algo]["model_norm"]
    assert np.allclose(x[:16], g[algo]["model_head"], rtol=1e-8, atol=0)


def test_config0_kernels_at_x0_match_reference_golden():
    g = load("c0_trace.json")
    c, k = g["config"], g["x0"]
    n_f, n_u, n_m, lam = c["n_f"], c["n_u"], c["n_m"], c["lam"]
    R = P.generate(0)
    x0 = P.random_init(n_f, n_u, n_m, k["seed"])
    xa = np.concatenate([x0.user_data, x0.item_data])
    assert hashlib.sha256(xa.tobytes()).hexdigest() == k["sha256"]
    X = P.FlatVector.from_array(xa, n_f, n_u, n_m)
    assert abs(P.ncg.loss(X, R, lam) - k["loss"]) <= 1e-12 * abs(k["loss"])
    gr = P.ncg.gradient(X, R, lam).array()
    assert abs(np.linalg.norm(gr) - k["gradient_norm"]) <= 1e-11 * k["gradient_norm"]
    assert np.max(np.abs(gr[:16] - k["gradient_head"])) <= 1e-11 * np.max(np.abs(gr))
    p = np.random.default_rng(k["quartic_p_seed"]).standard_normal(xa.size) * k["quartic_p_scale"]
    q = P.linesearch.quartic_coefficients(X, P.FlatVector.from_array(p, n_f, n_u, n_m), R, lam)
    want = np.asarray(k["quartic_n_chunks_1"])
    assert np.max(np.abs(np.asarray(q.c) - want)) <= 1e-12 * np.max(np.abs(want))
    users = P.als.update_users(x0, R, lam)
    assert abs(np.linalg.norm(users) - k["user_half_sweep_norm"]) <= 1e-9 * k["user_half_sweep_norm"]
    assert np.allclose(users[:16], k["user_half_sweep_head"], rtol=1e-9, atol=0)


def test_config1_to_tolerance_matches_reference_trace():
    """Config 1 to (1/N)||g|| < 1e-6 against the reference's own run.

    Measured (profiles/r02_c1_ttt_vs_reference.txt): the two runs take the
    same decisions (backtrack counts, no restarts, no fallback steps) for the
    first 85 iterations; the relative gradient-norm difference starts at
    ~1e-14 and grows by ~1.5x per iteration (4e-9 at k = 20, 1e-4 at k = 50),
    the rounding-level differences of two FP64 implementations amplified by
    the iteration (the reference's own count moves with its n_blocks, which
    only reorders the quartic's sums).  So the test pins the decision
    sequence over a prefix well inside that horizon, the losses along it, and
    the end state: converged, no restarts, the same fallback steps, the
    iteration count within 10 %, and the final loss on the reference's
    trajectory (its loss at the same iteration) within 1e-5."""
    path = os.path.join(GOLD, "c1_ttt_trace.json")
    if not os.path.exists(path):
        pytest.skip("c1_ttt_trace.json not generated yet")
    g = load("c1_ttt_trace.json")
    c, s = g["config"], g["solver"]
    R = P.generate(1)
    cfg = P.SolverConfig(lambda_=c["lam"], n_f=c["n_f"], max_iters=len(g["trace"]) + 100,
                         tol=s["tol"], seed=s["seed"], n_blocks=s["n_blocks"], trace_every=1,
                         paper_timing=True)
    res = P.ncg.als_ncg_solve(R, cfg)
    recs = res.trace.records
    ref = g["trace"]
    PREFIX = 60
    for a, b in zip(recs[:PREFIX + 1], ref[:PREFIX + 1]):
        assert (a.iter, a.backtracks, a.restarted) == (b["iter"], b["backtracks"], b["restarted"]), \
            (a.iter, a.backtracks, b["backtracks"], a.restarted, b["restarted"])
        assert abs(a.loss - b["loss"]) <= 1e-8 * abs(b["loss"]), (a.iter, a.loss, b["loss"])
    want = g["result"]
    assert res.converged and want["converged"]
    assert res.restarts == want["restarts"] == 0
    assert res.fallback_steps == want["fallback_steps"]
    assert abs(res.iterations - want["iterations"]) <= 0.1 * want["iterations"], (res.iterations, want)
    # the end state sits on the reference's trajectory: the loss at the GPU's
    # last iteration equals the reference's loss at that iteration to 1e-5
    k = min(res.iterations, len(ref) - 1)
    assert abs(res.final_loss - ref[k]["loss"]) <= 1e-5 * ref[k]["loss"], (k, res.final_loss, ref[k]["loss"])
