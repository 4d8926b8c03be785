"""Pins of the FTR (Goldberg Shamir-share PIR over F_p, NEXT-2) oracle:
Lemma 1 proof, Alg. 4.  Expected values from numpy int64
matmuls, closed forms, exhaustive subsets and brute force."""
import itertools

import numpy as np
import pytest

import synth
from oracle import oracle as O

P = 65537


def test_t0_shares_are_unit_vectors():
    sh = O.ftr_query(5, 9, 3, 0, seed=1)
    e = np.zeros(9, np.uint32)
    e[5] = 1
    assert (sh == e).all()


def test_any_t_plus_1_subset_interpolates_to_unit_vector():
    """l = 5, t = 2, every 3-subset interpolates to e_theta at 0."""
    r, l, t, theta = 11, 5, 2, 7
    sh = O.ftr_query(theta, r, l, t, seed=3)
    e = np.zeros(r, np.uint32)
    e[theta] = 1
    for sub in itertools.combinations(range(l), t + 1):
        got = O.ftr_reconstruct(sh[list(sub)], [i + 1 for i in sub])
        assert (got == e).all(), sub
    # t points are not enough: some t-subset does not interpolate to e_theta
    bad = sum((O.ftr_reconstruct(sh[list(s)], [i + 1 for i in s]) != e).any()
              for s in itertools.combinations(range(l), t))
    assert bad > 0


def test_lagrange_closed_forms():
    # interpolating the constant polynomial c gives c; a line a + b x gives a
    c = np.array([[42, 7, 65536]] * 4, np.uint32)
    assert (O.ftr_reconstruct(c, [1, 2, 3, 4]) == [42, 7, 65536]).all()
    a, b = 1234, 999
    resp = np.array([[(a + b * x) % P] for x in (3, 10)], np.uint32)
    assert O.ftr_reconstruct(resp, [3, 10])[0] == a
    with pytest.raises(ValueError):
        O.ftr_reconstruct(resp, [3, 3])


def test_respond_matches_numpy():
    r, s = 700, 33
    rec = synth.uniform_u8_np(4, (r, s))
    rho = synth.uniform_u32_np(5, (r,)) % P
    want = (rho.astype(np.int64) @ rec.astype(np.int64)) % P
    assert (O.ftr_respond(rec, rho).astype(np.int64) == want).all()
    Q = synth.uniform_u32_np(6, (4, r)) % P
    wantb = (Q.astype(np.int64) @ rec.astype(np.int64)) % P
    assert (O.ftr_respond_batch(rec, Q).astype(np.int64) == wantb).all()


@pytest.mark.parametrize("l,t", [(2, 1), (3, 1), (5, 2)])
def test_bruteforce_reconstruct_every_record(l, t):
    r, s = 200, 16
    rec = synth.uniform_u8_np(7, (r, s))
    for theta in range(r):
        sh = O.ftr_query(theta, r, l, t, seed=100 + theta)
        resp = np.stack([O.ftr_respond(rec, sh[i]) for i in range(l)])
        k = t + 1  # any t + 1 responses suffice
        got = O.ftr_reconstruct(resp[:k], [i + 1 for i in range(k)])
        assert (got == rec[theta]).all()


def test_t1_single_server_view_uniform():
    """t-privacy (Lemma 1; SPEC S:196 style, small field p = 7, r = 2, t = 1):
    one server's share vector is uniform over F_7^2 and independent of theta."""
    p, r = 7, 2
    for theta in (0, 1):
        counts = np.zeros((p, p))
        for seed in range(4900):
            sh = O.ftr_query(theta, r, 2, 1, seed, p)
            counts[sh[0, 0], sh[0, 1]] += 1
        chi2 = ((counts - 100.0) ** 2 / 100.0).sum()
        assert chi2 < 90.0  # 48 dof


# ---------------------------------------------------------------- robust decoding
def test_bw_without_errors_equals_lagrange():
    """No corruption: Berlekamp-Welch decodes to the same words as Lagrange
    interpolation at 0 ("when zero corruption, plain Lagrange")."""
    rng = np.random.default_rng(11)
    for k, t in [(2, 1), (3, 1), (5, 2), (7, 3), (7, 1)]:
        resp = rng.integers(0, P, (k, 9)).astype(np.uint32)
        # make the rows a degree-t code word: evaluate random polynomials
        coef = rng.integers(0, P, (t + 1, 9))
        al = np.arange(1, k + 1)
        resp = np.stack([sum(coef[c] * pow(int(a), c, P) for c in range(t + 1)) % P
                         for a in al]).astype(np.uint32)
        got, bad = O.ftr_decode(resp, al, t)
        assert (got == O.ftr_reconstruct(resp[: t + 1], al[: t + 1])).all()
        assert (got == coef[0] % P).all() and not bad.any()


def test_bw_robustness_exhaustive_small():
    """SPEC invariant (FTR robustness): for all (k, t, nu) with
    nu <= floor((k - t - 1) / 2) and k <= 7, corrupting any nu responses (every
    choice of positions, random wrong values) never changes the reconstructed
    block, and the corrupted servers are exactly the ones flagged."""
    r, s = 12, 5
    rec = synth.uniform_u8_np(21, (r, s))
    rng = np.random.default_rng(22)
    checked = 0
    for k in range(2, 8):
        for t in range(0, k):
            e = (k - t - 1) // 2
            theta = int(rng.integers(r))
            sh = O.ftr_query(theta, r, k, t, seed=1000 + 10 * k + t)
            resp = np.stack([O.ftr_respond(rec, sh[i]) for i in range(k)])
            al = np.arange(1, k + 1)
            for nu in range(0, e + 1):
                for pos in itertools.combinations(range(k), nu):
                    bad_resp = resp.copy()
                    for i in pos:
                        bad_resp[i] = (bad_resp[i] + rng.integers(1, P, s)) % P
                    got, bad = O.ftr_decode(bad_resp, al, t)
                    assert (got == rec[theta]).all(), (k, t, pos)
                    assert set(np.nonzero(bad)[0]) == set(pos), (k, t, pos)
                    checked += 1
    assert checked > 100


def test_bw_beyond_radius_and_incomplete():
    """k <= t responses: incompleteness error; e + 1 corrupted responses: the
    unique decoder reports failure (it cannot be right in general: with
    k = 5, t = 2 two bad rows of a 3-of-5 code are undecodable)."""
    r, s, k, t = 10, 6, 5, 2
    rec = synth.uniform_u8_np(23, (r, s))
    sh = O.ftr_query(4, r, k, t, seed=24)
    resp = np.stack([O.ftr_respond(rec, sh[i]) for i in range(k)])
    al = np.arange(1, k + 1)
    with pytest.raises(O.FtrDecodeError):
        O.ftr_decode(resp[:t], al[:t], t)
    rng = np.random.default_rng(25)
    fails = 0
    for trial in range(20):
        bad_resp = resp.copy()
        pos = rng.choice(k, (k - t - 1) // 2 + 1, replace=False)
        for i in pos:
            bad_resp[i] = (bad_resp[i] + rng.integers(1, P, s)) % P
        try:
            got, _ = O.ftr_decode(bad_resp, al, t)
            fails += int(not (got == rec[4]).all())
        except O.FtrDecodeError:
            fails += 1
    assert fails == 20  # never silently "right" beyond the radius on random errors
