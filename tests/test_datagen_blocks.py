"""datagen.generate_blocks (the block-major bench's data path) on CPU: blocks drawn on
different 'ranks' are the blocks of one node matrix (column-normalised per block), and the
labels formed from partial products summed over the ranks equal the labels formed with all
blocks local."""
import torch

from paper_2405_16267_b200 import datagen as dg


def _two_rank_labels(loss, C=1):
    N, m, n, kappa = 2, 300, 96, 7
    cs = dg.block_partition(n, 4)
    full_A, full_b, xt = dg.generate_blocks(N, m, n, kappa, loss, cs, [(i, j) for i in range(N) for j in range(4)],
                                            C=C, seed=11, device="cpu")
    parts = {}

    def keep(tag):
        def f(plist):
            parts[tag] = [p.clone() for p in plist]
        return f

    r0 = [(i, j) for i in range(N) for j in (0, 1)]
    r1 = [(i, j) for i in range(N) for j in (2, 3)]
    A0, _, xt0 = dg.generate_blocks(N, m, n, kappa, loss, cs, r0, C=C, seed=11, device="cpu", sum_products=keep(0))
    A1, _, xt1 = dg.generate_blocks(N, m, n, kappa, loss, cs, r1, C=C, seed=11, device="cpu", sum_products=keep(1))
    summed = [a + b for a, b in zip(parts[0], parts[1])]

    def sum_into(plist):
        for k, p in enumerate(plist):
            p.copy_(summed[k])

    _, b0, _ = dg.generate_blocks(N, m, n, kappa, loss, cs, r0, C=C, seed=11, device="cpu", sum_products=sum_into)
    return full_A, full_b, xt, A0, A1, b0, xt0, xt1


def test_blocks_are_placement_independent_and_unit_norm():
    full_A, full_b, xt, A0, A1, b0, xt0, xt1 = _two_rank_labels("ls")
    assert torch.equal(xt, xt0) and torch.equal(xt, xt1)
    for ij, a in list(A0.items()) + list(A1.items()):
        assert torch.equal(a, full_A[ij])
        assert torch.allclose(torch.linalg.vector_norm(a, dim=0), torch.ones(a.shape[1], dtype=a.dtype))


def test_labels_from_summed_partial_products_match_all_local():
    for loss, C in (("ls", 1), ("logistic", 1), ("hinge", 1), ("softmax", 4)):
        full_A, full_b, xt, A0, A1, b0, _, _ = _two_rank_labels(loss, C)
        for i in range(2):
            if loss == "ls":
                assert torch.allclose(b0[i], full_b[i], rtol=0, atol=1e-12)
            else:
                assert torch.mean((b0[i] == full_b[i]).double()) >= 0.999
