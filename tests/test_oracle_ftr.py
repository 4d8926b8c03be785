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
