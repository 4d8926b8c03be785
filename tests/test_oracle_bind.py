"""NEXT-4 oracle pins: HCT.Puzzle.Gen and PSD.Puzzle.Bind (Alg. 1 step 1,
P:553-566) with the record layout of P:1686 (DESIGN R11, R21)."""
import numpy as np
import pytest

import synth
from oracle import oracle as O

M32 = 0xFFFFFFFF


def test_puzzle_field_sizes_match_the_paper():
    # "a lambda-bit nonce (n_s), a 4-byte difficulty (kappa), and a
    # 1-byte level (n_l), totaling 37 bytes"; 560 bytes of spectrum data
    assert O.HCT_PUZZLE_BYTES == 37 and O.SPECTRUM_BYTES == 560
    assert synth.PAPER_RECORD_BYTES >= 560 + 37 + 2420  # + ML-DSA signature
    pz = O.hct_puzzle_gen(1, 0, 20, 3)
    assert pz.shape == (37,)
    assert int.from_bytes(pz[32:36].tobytes(), "little") == 20 and pz[36] == 3


def test_nonce_is_philox_of_seed_and_theta():
    """n_s word w = Philox(key = seed, ctr = (theta_lo, theta_hi, w >> 2, 0x48))[w & 3]
    (R21) through the KAT-pinned Philox; theta > 2^32 exercises the high counter word."""
    seed = 0x0123456789ABCDEF
    key = [seed & M32, seed >> 32]
    for theta in (0, 7, 2**32 + 5):
        pz = O.hct_puzzle_gen(seed, theta, 0xDEADBEEF, 9)
        words = pz[:32].view("<u4")
        for w in range(8):
            r = O.philox4x32_10([theta & M32, theta >> 32, w >> 2, 0x48], key)
            assert words[w] == r[w & 3], (theta, w)
        assert int.from_bytes(pz[32:36].tobytes(), "little") == 0xDEADBEEF and pz[36] == 9


def test_nonces_are_distinct_and_uniform():
    """n_s <-$ {0,1}^256: 4096 puzzles -> all distinct, and the 131072 nonce bytes
    pass a chi-square test against the uniform byte distribution (df 255,
    p = 1e-6 bound ~ 370)."""
    pz = np.stack([O.hct_puzzle_gen(99, t, 20, 3) for t in range(4096)])
    nonces = {bytes(p[:32]) for p in pz}
    assert len(nonces) == 4096
    counts = np.bincount(pz[:, :32].reshape(-1), minlength=256).astype(np.float64)
    exp = counts.sum() / 256
    assert ((counts - exp) ** 2 / exp).sum() < 370
    # different PSD seeds give different puzzles for the same record
    assert (O.hct_puzzle_gen(98, 5, 20, 3)[:32] != pz[5, :32]).any()


@pytest.mark.parametrize("d", [597, 3072, 4000])
def test_bind_layout(d):
    """Record = spectrum (560 B, verbatim) || puzzle (37 B) || zero signature
    slot / padding to d, for every record of a ragged range."""
    n, theta0 = 13, 1000
    spec = synth.uniform_u8_np(7, (n, 600))  # stride 600 >= 560: only 560 bytes used
    rec = O.puzzle_bind_hct(spec, theta0, 5, 20, 3, d)
    assert rec.shape == (n, d)
    for i in range(n):
        assert (rec[i, :560] == spec[i, :560]).all()
        assert (rec[i, 560:597] == O.hct_puzzle_gen(5, theta0 + i, 20, 3)).all()
        assert not rec[i, 597:].any()
