"""CPU pins of the oracle's Eq. 8 heterogeneity prior:
het_j = ||H_j - C||_F (Frobenius per SPEC.md:203 / App. B), C = global Hbar
(Eq. 6, Eq. 8 literal) or the group mean Hbar^(g) (App. B), and the routing score
r_ij = s Qbar_i.Kbar_j + log(het_j + eps) (softmax dropped, R-8).

Pins: a NumPy brute force through a different arrangement (einsum per block,
np.linalg.norm), the SPEC Pythagorean example, the degenerate cases G = 1 and
G >= N_K, the within-group variance lemma, and the routing
examples of SPEC.md:242-243 (all-equal statistics -> index order; larger
heterogeneity strictly raises the score)."""
import numpy as np
import pytest

import oracle
from oracle import brute


def _kv(seed, S=300, D=8, scale=1.0):
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((S, D)) * scale
    v = rng.standard_normal((S, D)) + 0.5 * k
    return k, v


@pytest.mark.parametrize("S,D,Bk,G", [(300, 8, 64, 2), (257, 4, 16, 3), (128, 16, 64, 32)])
@pytest.mark.parametrize("mode", ["global", "group"])
def test_het_matches_brute_force(S, D, Bk, G, mode):
    k, v = _kv(S + D, S, D)
    got = oracle.heterogeneity(k, v, Bk=Bk, G=G, mode=mode)
    H = brute.block_H(k, v, Bk)                       # [N_K, D, D], einsum form
    NK = H.shape[0]
    if mode == "global":
        C = np.broadcast_to(H.mean(axis=0), H.shape)
    else:
        C = np.stack([H[(j // G) * G:min((j // G + 1) * G, NK)].mean(axis=0) for j in range(NK)])
    want = np.array([np.linalg.norm(H[j] - C[j]) for j in range(NK)])
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


def test_het_pythagorean_example():
    """H_j - Hbar = [[3,4],[0,0]] -> 5.  Block 0 (2 tokens,
    key deviations +-e_0) has H_0 = e_0^T (v_1 - v_2) = [[6,8],[0,0]]; block 1 has
    constant keys, H_1 = 0; Hbar = [[3,4],[0,0]], so both norms are 5."""
    k = np.array([[1.0, 0.0], [-1.0, 0.0], [2.0, 2.0], [2.0, 2.0]])
    v = np.array([[7.0, 9.0], [1.0, 1.0], [5.0, -3.0], [0.5, 4.0]])
    het = oracle.heterogeneity(k, v, Bk=2, G=32, mode="global")
    assert het.tolist() == [5.0, 5.0]


def test_het_identical_blocks_zero():
    rng = np.random.default_rng(3)
    kb, vb = rng.standard_normal((64, 8)), rng.standard_normal((64, 8))
    k, v = np.tile(kb, (4, 1)), np.tile(vb, (4, 1))   # 4 blocks: sums and means exact
    for mode in ("global", "group"):
        assert np.all(oracle.heterogeneity(k, v, Bk=64, G=2, mode=mode) == 0.0)


def test_het_group_degenerate_cases():
    k, v = _kv(11, 400, 8)
    # G = 1: every block is its own group -> deviation from the group mean is 0
    assert np.all(oracle.heterogeneity(k, v, Bk=32, G=1, mode="group") == 0.0)
    # G >= N_K: one group whose mean is the global Hbar
    a = oracle.heterogeneity(k, v, Bk=32, G=1000, mode="group")
    b = oracle.heterogeneity(k, v, Bk=32, G=1000, mode="global")
    assert np.allclose(a, b, rtol=1e-13, atol=0)


def test_het_group_variance_lemma():
    """SPEC.md:473 (App. B): within each group, sum ||H_j - Hbar^(g)||^2 <=
    sum ||H_j - Hbar||^2 (the group mean minimises the within-group spread)."""
    k, v = _kv(5, 1000, 8)
    G = 3
    hg = oracle.heterogeneity(k, v, Bk=32, G=G, mode="group")
    hl = oracle.heterogeneity(k, v, Bk=32, G=G, mode="global")
    for g0 in range(0, len(hg), G):
        assert (hg[g0:g0 + G] ** 2).sum() <= (hl[g0:g0 + G] ** 2).sum() * (1 + 1e-12)


def test_route_prior_all_equal_is_index_order():
    """all K-bar equal and all het equal -> every row constant ->
    top-k by ascending block index (beta = 0)."""
    S, D = 512, 8
    q = np.random.default_rng(1).standard_normal((1, S, 1, D))
    k = np.zeros((1, S, 1, D)) + 0.25
    het = np.full((1, S // 64), 3.0)
    r = oracle.route(q, k, Bq=64, Bk=64, beta=0.0, kk=3, het=het)
    assert np.all(r["idx"][0] == np.array([0, 1, 2]))


def test_route_prior_monotone_and_additive():
    """raising het_j strictly raises r_.j; the prior enters as an
    additive log term (beta = 0 scores)."""
    rng = np.random.default_rng(2)
    S, D = 640, 8
    q, k = rng.standard_normal((1, S, 1, D)), rng.standard_normal((1, S, 1, D))
    NK = S // 64
    het = rng.uniform(0.5, 2.0, (1, NK))
    base = oracle.route(q, k, Bq=64, Bk=64, beta=0.0, kk=NK, want_scores=True)["scores"]
    with_p = oracle.route(q, k, Bq=64, Bk=64, beta=0.0, kk=NK, want_scores=True, het=het,
                          eps=1e-6)["scores"]
    assert np.allclose(with_p - base, np.log(het + 1e-6)[:, None, :], rtol=0, atol=1e-12)
    het2 = het.copy()
    het2[0, 4] *= 3.0
    up = oracle.route(q, k, Bq=64, Bk=64, beta=0.0, kk=NK, want_scores=True, het=het2)["scores"]
    assert np.all(up[0, :, 4] > with_p[0, :, 4])
    assert np.array_equal(np.delete(up, 4, axis=2), np.delete(with_p, 4, axis=2))


def test_route_prior_changes_selection_towards_heterogeneous_blocks():
    """With equal centroid scores the prior alone decides: the k most
    heterogeneous blocks are kept."""
    S, D = 1024, 8
    q = np.random.default_rng(4).standard_normal((1, S, 1, D))
    k = np.zeros((1, S, 1, D))
    het = np.array([[1.0, 9.0, 2.0, 8.0, 3.0, 7.0, 4.0, 6.0, 5.0, 0.5, 0.1, 0.2, 10.0, 1.5, 2.5,
                     3.5]])
    r = oracle.route(q, k, Bq=64, Bk=64, beta=0.0, kk=4, het=het)
    assert np.all(r["idx"][0] == np.array([1, 3, 5, 12]))
