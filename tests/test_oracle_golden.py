"""Pin the O2 oracle (the GPU's checker) against the unmodified reference.

Golden vectors in tests/golden/ref_golden.npz were produced by oracle/make_golden.py
from oracle/_ref (the reference headers compiled in place). Each test names the
reference lines it re-hosts. CPU only.
"""
import os

import numpy as np
import pytest

import oracle

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.npz"))


def test_euc2d_matches_reference():
    """instance.hpp:33-37; KATs of test_instance.cpp:136-145 (5, 1, 1 (.5 up), 10, 0)."""
    pts, ref = GOLD["euc2d_pts"], GOLD["euc2d_ref"]
    assert list(ref[:5]) == [5, 1, 1, 10, 0]
    got = np.array([oracle.euc2d(*p) for p in pts], dtype=np.int32)
    assert np.array_equal(got, ref)


def test_power_matches_reference():
    """construction.hpp:19-44 (repeated squaring for integral exponents, std::pow otherwise)."""
    args, ref = GOLD["power_args"], GOLD["power_ref"]
    got = np.array([oracle.power(e, x) for e, x in args])
    assert np.array_equal(got, ref)
    assert oracle.power(5.0, 2.0) == 32.0 and oracle.power(0.0, 123.4) == 1.0  # test_construction.cpp:35-44


@pytest.mark.parametrize("case", list(GOLD["tau_cases"]))
def test_tau_alpha_matches_colony_pheromone(case):
    """ColonyPheromone::begin_step/tau_alpha after update_l_best/update_g_best in ant order:
    acc summed per ant in ant order, tau^alpha = Power(alpha)(tau0 + acc) -- bit-exact."""
    x, y, tours = GOLD[f"tau{case}_x"], GOLD[f"tau{case}_y"], GOLD[f"tau{case}_tours"]
    alpha = float(GOLD[f"tau{case}_alpha"])
    m, n = tours.shape
    o = oracle.O2(x, y, m=m, k=min(16, n - 1), alpha=alpha, beta=2.0)
    for a in range(m):
        o.offer_tour(a, tours[a])
    assert o.g_best()[1] == int(GOLD[f"tau{case}_glen"])
    ref = GOLD[f"tau{case}_ref"]
    for i in range(n):
        assert np.array_equal(o.tau_row(i), ref[i]), f"row {i}"
    # Colony::pheromone (colony.hpp:145-155) sums tau0 first: agree within 1e-12 (colony tests tolerance)
    direct = GOLD[f"tau{case}_direct"]
    if alpha == 1.0:
        for i in range(n):
            mask = np.arange(n) != i
            assert np.allclose(o.tau_row(i)[mask], direct[i][mask], rtol=1e-12, atol=0)


def test_tau_bounds_property():
    """tau0 <= tau <= tau0 + m (SPEC colony-model invariants; test_colony.cpp:145-180)."""
    for case in GOLD["tau_cases"]:
        if float(GOLD[f"tau{case}_alpha"]) != 1.0:
            continue
        ref = GOLD[f"tau{case}_ref"]
        m = GOLD[f"tau{case}_tours"].shape[0]
        assert ref.min() >= 1.0 and ref.max() <= 1.0 + m


def test_rectangle_pheromone_kats():
    """test_colony.cpp:43-60: rectangle 3x4, tours of length 14 (g_best) and 16 share edges."""
    x = np.array([0.0, 3.0, 3.0, 0.0])
    y = np.array([0.0, 0.0, 4.0, 4.0])
    o = oracle.O2(x, y, m=2, k=3, alpha=1.0, beta=1.0)
    assert o.offer_tour(0, [0, 1, 2, 3]) and o.offer_tour(1, [0, 1, 3, 2])
    r0, r2, r1 = o.tau_row(0), o.tau_row(2), o.tau_row(1)
    assert r0[1] == pytest.approx(2.875, abs=1e-12)
    assert r2[3] == pytest.approx(2.875, abs=1e-12)
    assert r0[3] == pytest.approx(2.0, abs=1e-12)
    assert r1[3] == pytest.approx(1.875, abs=1e-12)
    assert r0[2] == pytest.approx(1.875, abs=1e-12)  # diagonal {0,2} only in the 16-tour


@pytest.mark.parametrize("tag", ["table", "fly"])
@pytest.mark.parametrize("beta", [2, 5])
def test_eta_beta_against_heuristic(tag, beta):
    """Heuristic (construction.hpp:49-82): the engine stores eta^beta as f32 = the reference's
    table value exactly; on the on-the-fly path the reference keeps the double, which rounds
    to the same f32. The d = 0 duplicate pair is clamped to eta = 1."""
    x, y, pairs = GOLD[f"eta_{tag}_x"], GOLD[f"eta_{tag}_y"], GOLD[f"eta_{tag}_pairs"]
    ref = GOLD[f"eta_{tag}_b{beta}_ref"]
    got = []
    for i, j in pairs:
        d = max(oracle.euc2d(x[i], y[i], x[j], y[j]), 1)
        got.append(np.float32(oracle.power(float(beta), 1.0 / d)))
    got = np.array(got, dtype=np.float32)
    assert np.array_equal(got, ref.astype(np.float32))
    assert ref[0] == 1.0


def test_update_sequence_matches_colony():
    """update_l_best strict improvement + update_g_best (colony.hpp:115-139), replayed in order."""
    x, y = GOLD["offer_x"], GOLD["offer_y"]
    tours, ants = GOLD["offer_tours"], GOLD["offer_ants"]
    o = oracle.O2(x, y, m=int(ants.max()) + 1, k=4)
    for q in range(len(ants)):
        assert o.offer_tour(int(ants[q]), tours[q]) == bool(GOLD["offer_flags"][q]), q
        assert o.g_best()[1] == int(GOLD["offer_g"][q]), q
    with pytest.raises(ValueError):
        o.offer_tour(0, np.array([0, 1, 2, 2, 4, 5, 6, 7, 8]))


def test_classic_update_matches_pheromone_matrix():
    """PheromoneMatrix evaporate+deposit (construction.hpp:160-213). With k = n-1 every edge is a
    candidate edge, so the O2 candidate-edge table must equal the full reference matrix."""
    ct, cl, ref = GOLD["classic_tours"], GOLD["classic_lens"], GOLD["classic_ref"]
    n = ct.shape[2]
    x = np.arange(n, dtype=np.float64)
    y = np.zeros(n)
    o = oracle.O2(x, y, m=ct.shape[1], k=n - 1, mode="classic", rho=float(GOLD["classic_rho"]),
                  tau_max=float(GOLD["classic_tau"]))
    for r in range(ct.shape[0]):
        o.classic_apply(ct[r], cl[r])
    T, knn = o.T(), o.knn()
    for i in range(n):
        for r in range(n - 1):
            assert T[i, r] == ref[i, knn[i, r]], (i, r)


def test_classic_kats():
    """test_construction.cpp:300-351: evaporation 2 -> 1 at rho = 0.5 (single entry view), floor 1e-6
    at rho = 1, edge shared by tours of length 10 and 20 gains 0.15."""
    n = 4
    x = np.array([0.0, 1.0, 2.0, 3.0]); y = np.zeros(4)
    o = oracle.O2(x, y, m=2, k=3, mode="classic", rho=0.5, tau_max=2.0)
    o.classic_apply(np.zeros((0, n), np.uint32), np.zeros(0, np.int64))
    assert np.all(o.T() == 1.0)
    o1 = oracle.O2(x, y, m=2, k=3, mode="classic", rho=1.0, tau_max=1.0)
    o1.classic_apply(np.zeros((0, n), np.uint32), np.zeros(0, np.int64))
    assert np.all(o1.T() == 1e-6)
    o2 = oracle.O2(x, y, m=2, k=3, mode="classic", rho=0.0, tau_max=1.0)
    o2.classic_apply(np.array([[0, 1, 2, 3], [1, 0, 3, 2]], np.uint32), np.array([10, 20], np.int64))
    T, knn = o2.T(), o2.knn()
    r = int(np.nonzero(knn[0] == 1)[0][0])
    assert T[0, r] == pytest.approx(1.15, abs=1e-15)


def test_philox_known_answers():
    """Random123 Philox4x32-10 known-answer vectors."""
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_draw_schedule_slots():
    """slot s of (seed, ant, iter) = word s%4 of Philox(ctr=(s/4, ant, iter), key=seed)."""
    w = oracle.philox([1, 3, 7, 0], [99, 0])
    for s in range(4, 8):
        assert oracle.draw_word(99, 3, 7, s) == w[s - 4]


def test_roulette_two_to_one_weights():
    """SPEC.md:200 / test_construction.cpp:101-119 analogue for the north-star rule: with
    weights 2:1 the roulette picks the heavier candidate with p = 2/3 (IR would give 3/4)."""
    wins, N = 0, 30000
    for t in range(N):
        lane, _ = oracle.roulette([2.0, 1.0], oracle.draw_word(5, 0, 0, 4 + t))
        wins += lane == 0
    p = wins / N
    sigma = (2 / 3 * 1 / 3 / N) ** 0.5
    assert abs(p - 2 / 3) < 4 * sigma


def test_roulette_feasibility_and_fallback():
    assert oracle.roulette([0.0, 0.0, 0.0], 123)[0] == -1          # all visited -> fallback
    assert oracle.roulette([0.0, 5.0, 0.0], 0xFFFFFFFF)[0] == 1     # only feasible lane wins
    for word in (0, 1 << 31, 0xFFFFFF00):
        assert oracle.roulette([0.0] * 7 + [1e-30] + [0.0] * 8, word)[0] == 7
    # u = 0 picks the lowest feasible lane
    assert oracle.roulette([0.0, 3.0, 1.0], 0)[0] == 1


def test_partial_construction_structure():
    """construction.hpp:312-350 / test_construction.cpp:177-258 on the north-star rule:
    preserved cyclic segment verbatim, m_mod = 0 identity, m_mod = 1 rotation, m_mod = n
    anchored at l_best[start_pos], always a permutation."""
    from paper_1709_03187_b200.instances import grid_instance
    inst = grid_instance(6, 5)
    rng = np.random.default_rng(4)
    o = oracle.O2(inst.xs, inst.ys, m=1, k=8, alpha=5.0, beta=5.0)
    order = rng.permutation(30).astype(np.uint32)
    assert o.offer_tour(0, order)
    words = rng.integers(0, 2**32, 64, dtype=np.uint64).astype(np.uint32)
    base_len = oracle.cycle_length(inst.xs, inst.ys, order)
    for start, m_mod in [(7, 0), (4, 1), (11, 2), (11, 15), (11, 29), (13, 30)]:
        t, ln = o.construct_at(0, start, m_mod, words)
        assert sorted(t.tolist()) == list(range(30))
        keep = 30 - m_mod
        assert np.array_equal(t[:keep], order[(start + np.arange(keep)) % 30])
        assert ln == oracle.cycle_length(inst.xs, inst.ys, t)
        if m_mod <= 1:
            assert ln == base_len
        if m_mod == 30:
            assert t[0] == order[13]


def test_fallback_grid_search_equals_brute_force():
    """The oracle's exact nearest-unvisited grid search against an O(n) scan, on a clustered
    instance with duplicates (fallback-heavy)."""
    from paper_1709_03187_b200.instances import make_config_instance
    inst = make_config_instance("C3", n=1500)
    a = oracle.O2(inst.xs, inst.ys, m=12, k=8, seed=3)
    b = oracle.O2(inst.xs, inst.ys, m=12, k=8, seed=3, fallback_brute=True)
    for _ in range(6):
        a.iterate(); b.iterate()
        assert np.array_equal(a.tours()[0], b.tours()[0])
    assert a.counters()["fallbacks"] > 100


def test_oracle_run_invariants():
    """Every tour a permutation with the recomputed length; g_best monotone and equal to min l_best."""
    from paper_1709_03187_b200.instances import cycle_length, is_permutation_of_n, make_config_instance
    inst = make_config_instance("C1", n=400)
    o = oracle.O2(inst.xs, inst.ys, m=16, k=12, seed=2)
    prev = None
    for _ in range(15):
        o.iterate()
        t, l = o.tours()
        for a in range(16):
            assert is_permutation_of_n(inst.n, t[a]) and cycle_length(inst, t[a]) == l[a]
        g = o.g_best()[1]
        assert g == o.l_best()[1].min()
        assert prev is None or g <= prev
        prev = g
    c = o.counters()
    assert c["decisions"] == c["full_builds"] * (inst.n - 1) + (c["decisions"] - c["full_builds"] * (inst.n - 1))


def test_partial_prob_zero_equals_paco_full():
    """test_engine.cpp:107-118: partial mode with partial_prob = 0 == paco mode, bit for bit."""
    from paper_1709_03187_b200.instances import make_config_instance
    inst = make_config_instance("C1", n=300)
    a = oracle.O2(inst.xs, inst.ys, m=8, k=10, seed=9, partial_prob=0.0)
    b = oracle.O2(inst.xs, inst.ys, m=8, k=10, seed=9, mode="paco")
    for _ in range(5):
        a.iterate(); b.iterate()
    assert np.array_equal(a.tours()[0], b.tours()[0])


def test_oracle_independent_of_thread_count():
    """test_engine.cpp:75-95 analogue: sync results do not depend on the worker count."""
    from paper_1709_03187_b200.instances import make_config_instance
    inst = make_config_instance("C1", n=500)
    a = oracle.O2(inst.xs, inst.ys, m=16, k=16, seed=4, threads=1)
    b = oracle.O2(inst.xs, inst.ys, m=16, k=16, seed=4, threads=7)
    for _ in range(6):
        a.iterate(); b.iterate()
    assert np.array_equal(a.tours()[0], b.tours()[0])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_live_reference_colony_random():
    """Live O1 cross-check beyond the fixtures: random colonies, tau rows bit-exact."""
    rng = np.random.default_rng(77)
    for n, m in [(15, 6), (40, 10)]:
        x = rng.integers(0, 500, n).astype(float)
        y = rng.integers(0, 500, n).astype(float)
        tours = np.stack([rng.permutation(n) for _ in range(m)]).astype(np.uint32)
        ref, _ = oracle.ref_colony_tau(x, y, tours, 1.0, 1.0)
        o = oracle.O2(x, y, m=m, k=8)
        for a in range(m):
            o.offer_tour(a, tours[a])
        for i in range(n):
            assert np.array_equal(o.tau_row(i), ref[i])


def test_two_opt_matches_reference():
    """two_opt (two_opt.hpp:28-67): the square KAT of test_two_opt.cpp:11-21 (48 -> 40) and random
    tours with and without a window, move sequence identical to the reference."""
    assert list(GOLD["twoopt_sq"]) == [0, 1, 2, 3]
    sq_x = np.array([0.0, 10.0, 10.0, 0.0]); sq_y = np.array([0.0, 0.0, 10.0, 10.0])
    o, d = oracle.two_opt(sq_x, sq_y, [0, 2, 1, 3])
    assert d == -8 and list(o) == [0, 1, 2, 3]
    for ti in GOLD["twoopt_cases"]:
        x, y = GOLD[f"twoopt{ti}_x"], GOLD[f"twoopt{ti}_y"]
        o, d = oracle.two_opt(x, y, GOLD[f"twoopt{ti}_in"], int(GOLD[f"twoopt{ti}_window"]))
        assert np.array_equal(o, GOLD[f"twoopt{ti}_out"])
        assert oracle.cycle_length(x, y, o) == int(GOLD[f"twoopt{ti}_len"])
