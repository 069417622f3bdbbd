"""Pins of the transfer-operator oracle (§3.4, §6.6).

Every expected value here comes from an independent route: numpy reshape / sum / repeat of the
4-D fine field, numpy.linalg.qr, dense matrices assembled by applying the oracle to unit vectors
(checked against algebraic identities, not against the oracle's own formula)."""
import itertools

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def blocks4(x, cdims, block, tail):
    """[Vf, *tail] in canonical fine order -> [Lc3, B3, Lc2, B2, Lc1, B1, Lc0, B0, *tail] (numpy only)."""
    sh = []
    for mu in (3, 2, 1, 0):
        sh += [cdims[mu], block[mu]]
    return x.reshape(*sh, *tail)


def rnd(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


@pytest.mark.parametrize("Ns,Nc,Nvec", [(2, 5, 5), (4, 3, 6)])
def test_unit_block_identity_basis_is_a_reshape(Ns, Nc, Nvec):
    """B = 1 and W(s, a, k) = delta(row within chirality, k): P is the reshape coarse dof
    i = chi*Nvec + (s - chi*Ns/2)*Nc + a -> fine dof (s, a); bit-exact both ways."""
    cd_ = (3, 2, 1, 2)
    V = int(np.prod(cd_))
    W = np.zeros((V, Ns, Nc, Nvec), complex)
    for s, a in itertools.product(range(Ns), range(Nc)):
        W[:, s, a, (s % (Ns // 2)) * Nc + a] = 1
    vc = rnd((V, 2 * Nvec), 1)
    vf = oracle.prolong(cd_, (1, 1, 1, 1), Ns, Nc, Nvec, W, vc)
    np.testing.assert_array_equal(vf, vc.reshape(V, Ns, Nc))
    np.testing.assert_array_equal(oracle.restrict(cd_, (1, 1, 1, 1), Ns, Nc, Nvec, W, vf), vc)


@pytest.mark.parametrize("cdims,block,Ns", [((2, 3, 1, 2), (2, 1, 3, 2), 4), ((3, 1, 2, 2), (1, 2, 2, 3), 2)])
def test_constant_basis_is_block_sum_and_broadcast(cdims, block, Ns):
    """W = delta(a, k) on every fine site: the restrictor sums each aggregate hypercube and each
    chirality's spins (numpy reshape + sum over the block axes); the prolongator broadcasts."""
    Nc = Nvec = 3
    Vc = int(np.prod(cdims))
    Vf = Vc * int(np.prod(block))
    W = np.zeros((Vf, Ns, Nc, Nvec), complex)
    for a in range(Nc):
        W[:, :, a, a] = 1
    vf = rnd((Vf, Ns, Nc), 2)
    b = blocks4(vf, cdims, block, (Ns, Nc)).sum(axis=(1, 3, 5, 7))            # [Lc3, Lc2, Lc1, Lc0, Ns, Nc]
    want = b.reshape(Vc, 2, Ns // 2, Nc).sum(axis=2).reshape(Vc, 2 * Nvec)
    got = oracle.restrict(cdims, block, Ns, Nc, Nvec, W, vf)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)
    vc = rnd((Vc, 2 * Nvec), 3)
    c = vc.reshape(cdims[3], 1, cdims[2], 1, cdims[1], 1, cdims[0], 1, 2, 1, Nc)
    c = np.broadcast_to(c, (cdims[3], block[3], cdims[2], block[2], cdims[1], block[1], cdims[0], block[0], 2,
                            Ns // 2, Nc))
    np.testing.assert_array_equal(oracle.prolong(cdims, block, Ns, Nc, Nvec, W, vc), c.reshape(Vf, Ns, Nc))


def _dense_P(cdims, block, Ns, Nc, Nvec, W):
    Vc = int(np.prod(cdims))
    cols = []
    for i in range(Vc * 2 * Nvec):
        e = np.zeros(Vc * 2 * Nvec, complex)
        e[i] = 1
        cols.append(oracle.prolong(cdims, block, Ns, Nc, Nvec, W, e).reshape(-1))
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("cdims,block,Ns,Nc,Nvec", [((2, 1, 2, 1), (2, 2, 1, 2), 4, 3, 6),
                                                     ((1, 2, 1, 3), (2, 1, 2, 1), 2, 4, 3)])
def test_orthonormal_basis_gives_PdagP_identity_and_restrict_is_Pdag(cdims, block, Ns, Nc, Nvec):
    """After block orthonormalisation P^dagger P = I, and restrict == P^dagger:
    both checked on dense matrices assembled column by column."""
    Vf = int(np.prod(cdims)) * int(np.prod(block))
    W = oracle.block_orthonormalise(cdims, block, Ns, Nc, Nvec, rnd((Vf, Ns, Nc, Nvec), 4))
    P = _dense_P(cdims, block, Ns, Nc, Nvec, W)
    np.testing.assert_allclose(P.conj().T @ P, np.eye(P.shape[1]), atol=1e-12)
    vf = rnd((Vf, Ns, Nc), 5)
    np.testing.assert_allclose(oracle.restrict(cdims, block, Ns, Nc, Nvec, W, vf).reshape(-1),
                               P.conj().T @ vf.reshape(-1), rtol=1e-12, atol=1e-12)
    # adjointness on a non-orthonormal basis too
    W2 = rnd((Vf, Ns, Nc, Nvec), 6)
    vc = rnd((int(np.prod(cdims)), 2 * Nvec), 7)
    lhs = np.vdot(vc, oracle.restrict(cdims, block, Ns, Nc, Nvec, W2, vf))
    rhs = np.vdot(oracle.prolong(cdims, block, Ns, Nc, Nvec, W2, vc), vf)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_block_qr_matches_numpy_qr():
    """Gram-Schmidt Q == numpy.linalg.qr Q with the phases that make diag(R) positive real, block by
    block; the blocks are gathered by numpy reshape/transpose (aggregate, chirality)."""
    cdims, block, Ns, Nc, Nvec = (2, 1, 1, 2), (2, 2, 1, 1), 4, 3, 5
    Vc = int(np.prod(cdims))
    Vf = Vc * int(np.prod(block))
    W0 = rnd((Vf, Ns, Nc, Nvec), 8)
    Q = oracle.block_orthonormalise(cdims, block, Ns, Nc, Nvec, W0)

    def gather(x):
        b = blocks4(x, cdims, block, (2, Ns // 2, Nc, Nvec))             # chirality axis split from spin
        b = b.transpose(0, 2, 4, 6, 8, 1, 3, 5, 7, 9, 10, 11)            # [Lc.., chi, B.., s', a, k]
        return b.reshape(Vc * 2, -1, Nvec)

    A, G = gather(W0), gather(Q)
    for blk in range(Vc * 2):
        q, r = np.linalg.qr(A[blk])
        ph = np.diag(r) / np.abs(np.diag(r))
        np.testing.assert_allclose(G[blk], q * ph, atol=1e-12)


def test_rank_deficient_block_raises():
    cdims, block = (1, 1, 1, 2), (1, 1, 1, 1)
    W = rnd((2, 2, 2, 2), 9)
    W[1, 0, :, 1] = W[1, 0, :, 0] * (2 - 1j)          # chirality 0 of site 1: dependent columns
    with pytest.raises(ValueError):
        oracle.block_orthonormalise(cdims, block, 2, 2, 2, W)


def test_galerkin_coarse_operator_stays_nearest_neighbour():
    """P^dagger D P of a nearest-neighbour fine operator (here a coarse-type operator, Ns = 2)
    couples an aggregate only to itself and its +-mu neighbours; the other blocks vanish."""
    cdims, block = (3, 2, 1, 1), (2, 1, 2, 1)
    Ns, Nc, Nvec = 2, 2, 2
    fdims = oracle.fine_dims(cdims, block)
    Vf, Vc, Nf = int(np.prod(fdims)), int(np.prod(cdims)), Ns * Nc
    D = oracle.dense(fdims, synth.links(fdims, Nf))
    W = oracle.block_orthonormalise(cdims, block, Ns, Nc, Nvec, rnd((Vf, Ns, Nc, Nvec), 10))
    P = _dense_P(cdims, block, Ns, Nc, Nvec, W)
    Mc = (P.conj().T @ D @ P).reshape(Vc, 2 * Nvec, Vc, 2 * Nvec)
    xs = [np.array(synth.site_coords(cdims, s)) for s in range(Vc)]
    for a in range(Vc):
        for b in range(Vc):
            d = [(xs[b][m] - xs[a][m]) % cdims[m] for m in range(4)]
            near = sum(1 for m in range(4) if d[m] not in (0,)) <= 1 and all(
                d[m] in (0, 1, cdims[m] - 1) for m in range(4))
            if not near:
                assert np.abs(Mc[a, :, b, :]).max() < 1e-12, (a, b)
    assert np.abs(Mc).max() > 0.1
