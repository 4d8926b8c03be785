"""The seeded input generator: deterministic, counter-based, paper-shaped."""
import torch

import synth


def test_records_deterministic_and_subsettable():
    a = synth.records(9, 0, 200, 3072, 40)
    b = synth.records(9, 150, 50, 3072, 40)
    assert torch.equal(a[150:], b)
    assert not torch.equal(synth.records(10, 0, 4, 3072, 40), a[:4])
    th = torch.tensor([3, 77, 199])
    for bidx in (0, 9, 13, 14, 593, 596, 1000, 3016, 3071):
        assert torch.equal(synth.byte_column(9, th, bidx, 3072, 40), a[th, bidx])


def test_paper_shaped_fields():
    n_ch, n_cols = 40, 512
    r = synth.records(9, 0, 2000, 3072, n_ch, n_cols)
    theta = torch.arange(2000)
    cell = theta // n_ch
    le = lambda x, o, k: sum(x[:, o + i].long() << (8 * i) for i in range(k))
    assert torch.equal(le(r, 0, 4), cell % n_cols)
    assert torch.equal(le(r, 4, 4), cell // n_cols)
    assert torch.equal(le(r, 8, 2), theta % n_ch)
    assert (le(r, 592, 4) == 20).all() and (r[:, 596] == 3).all()
    assert (r[:, 3017:] == 0).all()
    assert set(r[:, 14].tolist()) <= {0, 1}
    # payload bytes look uniform
    pay = r[:, 600:3000].float()
    assert abs(pay.mean().item() - 127.5) < 1.0


def test_uniform_u32_range():
    q = synth.uniform_u32_np(3, (1 << 16,))
    assert q.dtype.name == "uint32"
    assert q.max() > (1 << 31) and q.min() < (1 << 24)
