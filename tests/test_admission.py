"""NEXT-4 saturation-bounded admission: the library's native Algorithm 1 against the
plain-Python oracle on random traces, and the paper's invariants."""
import numpy as np
import pytest

from oracle import admission as O

F_TOK, HL, B = 4.4e10, 4096 * 94, 16


@pytest.fixture(scope="module")
def A():
    from paper_2605_02960_b200 import build
    build.build()
    from paper_2605_02960_b200 import asyncep
    return asyncep


def trace(rng, n_groups, n_req, max_prefix_blocks=64):
    """requests sharing prefixes by group: chain = group's prefix blocks + own suffix blocks"""
    groups = [list(rng.integers(1, 2 ** 62, size=rng.integers(1, max_prefix_blocks), dtype=np.uint64))
              for _ in range(n_groups)]
    chains, P, S = [], [], []
    for _ in range(n_req):
        g = groups[rng.integers(n_groups)]
        chains.append(list(g))
        P.append(len(g) * B + int(rng.integers(0, B)))
        S.append(int(rng.integers(1, 512)))
    return chains, P, S


def test_cost_model_pins():
    # SPEC invariants / the paper's statements about Eq. 2
    for P, S in ((0, 0), (1024, 16), (4096, 333), (17, 4000)):
        assert O.cost_delta(P, P, S, F_TOK, HL) + O.c_pfx(P, F_TOK, HL) == pytest.approx(
            O.cost_delta(P, 0, S, F_TOK, HL), rel=1e-15)        # cache credit is exactly the prefix cost
    assert O.cost_delta(100, 100, 0, F_TOK, HL) == 0.0           # fully cached, empty suffix
    assert O.c_sfx(16, 8192, F_TOK, HL) - O.c_sfx(16, 4096, F_TOK, HL) == pytest.approx(4 * 16 * 4096 * HL)


def test_paper_invariants_on_the_oracle():
    """Load band [T, T + Delta_last]; 10 siblings = 1 C_pfx + 10 C_sfx
    (PAPER.md:399); a popular prefix spills to the next-best GPU."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        N = int(rng.integers(4, 9))
        chains, P, S = trace(rng, 6, 400)
        T = 2e14
        loads, tables = [0.0] * N, [set() for _ in range(N)]
        gpus, deltas = O.schedule_round(tables, loads, T, B, F_TOK, HL, chains, P, S)
        assert -1 in gpus  # residual queue nonempty -> every GPU saturated
        for i in range(N):
            last = max(d for g, d in zip(gpus, deltas) if g == i)
            assert T <= loads[i] <= T + last
    # ten siblings on an empty system: one prefix pass + ten suffix passes, all on one GPU
    pref = [11, 12, 13, 14]
    chains, P, S = [pref] * 10, [64] * 10, [100] * 10
    loads, tables = [0.0] * 4, [set() for _ in range(4)]
    gpus, deltas = O.schedule_round(tables, loads, 1e30, B, F_TOK, HL, chains, P, S)
    assert len(set(gpus)) == 1
    assert sum(deltas) == pytest.approx(O.c_pfx(64, F_TOK, HL) + 10 * O.c_sfx(100, 64, F_TOK, HL), rel=1e-12)
    # spill: a small T saturates the prefix owner, the rest go elsewhere
    T = 2.5 * O.c_sfx(100, 64, F_TOK, HL) + O.c_pfx(64, F_TOK, HL)
    loads, tables = [0.0] * 4, [set() for _ in range(4)]
    gpus, _ = O.schedule_round(tables, loads, T, B, F_TOK, HL, chains, P, S)
    assert gpus[:3] == [0, 0, 0] and gpus[3] != 0


@pytest.mark.parametrize("seed", range(6))
def test_native_router_matches_oracle(A, seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 9))
    chains, P, S = trace(rng, int(rng.integers(1, 12)), int(rng.integers(1, 600)))
    T = float(rng.choice([1e14, 1e15, 5e15, 1e30]))
    r = A.Router(N, B, F_TOK, HL, T)
    loads, tables = [0.0] * N, [set() for _ in range(N)]
    for rnd in range(3):  # several rounds: tables (pending) carry over, loads reset (Alg. 1)
        g_ref, d_ref = O.schedule_round(tables, loads, T, B, F_TOK, HL, chains, P, S)
        g, d = r.schedule_round(chains, P, S)
        assert list(g) == g_ref
        np.testing.assert_allclose(d, d_ref, rtol=1e-12, atol=0)
        np.testing.assert_allclose(r.loads(), loads, rtol=1e-12)


def test_native_router_events(A):
    r = A.Router(2, B, 1.0, 0.0, 1e9)
    g, _ = r.schedule_round([[1, 2]], [32], [0])
    L = r.loads()[g[0]]
    r.progress(int(g[0]), 10)                     # L_i <- max(0, L_i - tokens * f_tok)
    assert r.loads()[g[0]] == L - 10
    r.progress(int(g[0]), 10 ** 6)
    assert r.loads()[g[0]] == 0.0
    r.blocks_stored(1, [7, 8])                    # committed on GPU 1 -> a matching request goes there
    g2, d2 = r.schedule_round([[7, 8, 9]], [40], [4], reset_loads=False)
    assert g2[0] == 1 and d2[0] == pytest.approx((40 - 32) + 4)
    cfg = A.RouterConfig(2, B, F_TOK, HL, 1.0)
    assert A.asyncep_cost_delta(cfg, 64, 16, 10) == pytest.approx(O.cost_delta(64, 16, 10, F_TOK, HL), rel=1e-15)
    assert np.isnan(A.asyncep_cost_delta(cfg, 10, 11, 0))


def test_malformed_round_changes_nothing_and_reports(A):
    """A round with a bad request after good ones is rejected before any state changes, and
    asyncep_last_error names the call (half-applied rounds, stale messages)."""
    r = A.Router(2, B, F_TOK, HL, 1e18)
    r.schedule_round([[1, 2], [3]], [2 * B, B], [10, 10], reset_loads=False)
    before = r.loads().copy()
    with pytest.raises(A.AsyncEPError, match="schedule_round"):
        r.schedule_round([[5, 6], [7]], [2 * B, -1], [10, 10], reset_loads=False)
    assert np.array_equal(r.loads(), before)
    # the good prefix [5, 6] was not made pending either: a later request sharing it sees no match
    g, d = r.schedule_round([[5, 6]], [2 * B], [10], reset_loads=False)
    assert d[0] == pytest.approx(O.cost_delta(2 * B, 0, 10, F_TOK, HL), rel=1e-12)
    with pytest.raises(A.AsyncEPError, match="router_progress"):
        r.progress(5, 10)
