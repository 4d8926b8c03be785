"""Pins of the ENS (Chor XOR PIR, NEXT-1) oracle: Lemma 1 proof,
Alg. 3.  Expected values from numpy XOR folds, closed forms and brute
force, never from the oracle itself."""
import numpy as np
import pytest

import synth
from oracle import oracle as O


def _bits(v, r):
    return np.unpackbits(v, bitorder="little")[:r]


def test_shares_xor_to_unit_vector():
    for r, l, theta in [(4, 2, 2), (13, 3, 12), (1000, 5, 517), (64, 2, 0)]:
        sh = O.ens_query(theta, r, l, seed=11)
        x = np.bitwise_xor.reduce(sh, axis=0)
        e = np.zeros(r, np.uint8)
        e[theta] = 1
        assert (_bits(x, r) == e).all()
        # padding bits beyond r are zero in every share
        if r % 8:
            assert (sh[:, -1] >> (r % 8) == 0).all()


def test_share_marginals_uniform():
    """Any l-1 shares are uniform and independent of theta (Lemma 1): for r = 4,
    the first share over many seeds hits all 16 values about equally often, and
    the last share's distribution does not depend on theta."""
    counts = {0: np.zeros(16), 3: np.zeros(16)}
    for theta in (0, 3):
        for seed in range(4000):
            sh = O.ens_query(theta, 4, 2, seed)
            counts[theta][sh[1, 0] & 15] += 1
    for c in counts.values():
        chi2 = ((c - 250.0) ** 2 / 250.0).sum()
        assert chi2 < 45.0  # 15 dof, p ~ 1e-4
    first = np.zeros(16)
    for seed in range(4000):
        first[O.ens_query(1, 4, 3, seed)[0, 0] & 15] += 1
    assert ((first - 250.0) ** 2 / 250.0).sum() < 45.0


def test_respond_closed_forms_and_numpy_fold():
    r, d = 300, 40
    rec = synth.uniform_u8_np(3, (r, d))
    nb = (r + 7) // 8
    assert (O.ens_respond(rec, np.zeros(nb, np.uint8)) == 0).all()
    for j in (0, 77, 299):
        e = np.zeros(nb, np.uint8)
        e[j >> 3] = 1 << (j & 7)
        assert (O.ens_respond(rec, e) == rec[j]).all()
    q = synth.uniform_u8_np(4, (nb,))
    q[-1] &= (1 << (r % 8)) - 1
    sel = _bits(q, r).astype(bool)
    assert (O.ens_respond(rec, q) == np.bitwise_xor.reduce(rec[sel], axis=0)).all()
    Q = synth.uniform_u8_np(5, (6, nb))
    Q[:, -1] &= (1 << (r % 8)) - 1
    got = O.ens_respond_batch(rec, Q)
    for b in range(6):
        s = _bits(Q[b], r).astype(bool)
        assert (got[b] == np.bitwise_xor.reduce(rec[s], axis=0)).all()


@pytest.mark.parametrize("l", [2, 3, 5])
def test_bruteforce_reconstruct_every_record(l):
    """Def. 1 / Lemma 1: XOR of the l responses = record theta, for every theta."""
    r, d = 512, 24
    rec = synth.uniform_u8_np(6, (r, d))
    for theta in range(r):
        sh = O.ens_query(theta, r, l, seed=1000 + theta)
        resp = np.stack([O.ens_respond(rec, sh[i]) for i in range(l)])
        assert (O.ens_reconstruct(resp) == rec[theta]).all()
