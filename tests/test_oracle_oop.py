"""Pins of the OOP (CIP-PIR offline-online, NEXT-3) oracle: Lemma 2 proof
(P:1258).  Expected values from brute force, cross-scheme
equivalence with ENS, and numpy XOR folds."""
import numpy as np
import pytest

import synth
from oracle import oracle as O


@pytest.mark.parametrize("n", [2, 3, 4])
def test_bruteforce_reconstruct_every_block(n):
    B, d = 96, 20
    rec = synth.uniform_u8_np(n, (B, d))
    for theta in range(B):
        seeds = np.arange(n, dtype=np.uint64) * 1000 + theta * 7 + 1
        A = [O.oop_preprocess(rec, n, i, int(seeds[i])) for i in range(n)]  # offline
        q = O.oop_query(theta, B, n, seeds)
        resp = np.stack([O.oop_respond(rec, n, i, q[i], A[i]) for i in range(n)])
        assert (np.bitwise_xor.reduce(resp, axis=0) == rec[theta]).all()
        # same block as ENS retrieval (cross-scheme equivalence)
        sh = O.ens_query(theta, B, 2, 5)
        ens = O.ens_reconstruct(np.stack([O.ens_respond(rec, sh[j]) for j in range(2)]))
        assert (ens == rec[theta]).all()


def test_online_touches_only_the_flip_chunk():
    """online work covers 1/n of the DB -- corrupting the other chunks
    after preprocessing does not change server i's response."""
    B, d, n, i = 64, 16, 4, 2
    rec = synth.uniform_u8_np(1, (B, d))
    A = O.oop_preprocess(rec, n, i, 99)
    q = O.oop_query(5, B, n, np.array([1, 2, 99, 4], np.uint64))
    k = B // n
    bad = rec.copy()
    mask = np.ones(B, bool)
    mask[i * k:(i + 1) * k] = False
    bad[mask] ^= 0xA5
    assert (O.oop_respond(rec, n, i, q[i], A) == O.oop_respond(bad, n, i, q[i], A)).all()


def test_preprocess_is_xor_of_prg_selected_nonflip_blocks():
    """A_i = q . (non-flip chunks): the XOR over the selected blocks equals the XOR
    of all selected minus none from the flip chunk; check with an independent
    numpy fold over the bit vector recovered from a unit-record DB."""
    B, n, i = 48, 3, 1
    k = B // n
    # records = unit rows e_b (d = B bytes): A_i then *is* the selection bit vector
    rec = np.eye(B, dtype=np.uint8)
    A = O.oop_preprocess(rec, n, i, 1234)
    sel = A.astype(bool)
    assert not sel[i * k:(i + 1) * k].any()            # flip chunk never selected
    assert 0.2 < sel.mean() < 0.5                      # ~half of (n-1)/n of the blocks
    rnd = synth.uniform_u8_np(2, (B, 8))
    assert (O.oop_preprocess(rnd, n, i, 1234) == np.bitwise_xor.reduce(rnd[sel], axis=0)).all()
