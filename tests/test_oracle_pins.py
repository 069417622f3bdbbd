"""Pins of the float64 oracle against what the paper and the mathematics fix.

Every oracle function is checked here against something other than itself: closed forms
(plane waves), library routines (numpy.roll, numpy.matmul, numpy float16 casts, numpy
slicing), invariants (linearity, <w, D v> = <D^H w, v>, tau3-hermiticity) and special
cases (identity, impulse, L = 1 self hops).  A plausible mistake -- a dropped term, a
swapped hop direction, a transposed link, a wrong axis order -- fails at least one test.
"""
import numpy as np
import pytest

import oracle
import synth

rng = np.random.default_rng(20161226)


def crandn(*shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def vol(d):
    return int(np.prod(d))


def as4d(v, dims):
    """[V, N] -> [L3, L2, L1, L0, N] (x0 fastest, Listing 2)."""
    return v.reshape(dims[3], dims[2], dims[1], dims[0], v.shape[-1])


def axis_of(mu):
    return 3 - mu


# ---------------------------------------------------------------- P1 brute force (dense)
@pytest.mark.parametrize("dims,N", [((2, 2, 2, 2), 48), ((3, 3, 3, 3), 6), ((1, 2, 3, 4), 4),
                                    ((2, 3, 4, 5), 2)])
def test_dense_matches_apply(dims, N):
    L = crandn(vol(dims), 9, N, N)
    v = crandn(vol(dims), N)
    D = oracle.dense(dims, L)
    y = oracle.apply(dims, L, v)
    ref = (D @ v.reshape(-1)).reshape(y.shape)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_dense_block_structure():
    """Every block row has exactly the 9 blocks of Eq. 3 (L >= 3: all neighbours distinct)."""
    dims, N = (3, 3, 3, 3), 2
    L = crandn(vol(dims), 9, N, N)
    D = oracle.dense(dims, L)
    V = vol(dims)
    nz = np.abs(D.reshape(V, N, V, N)).sum(axis=(1, 3)) > 0
    assert (nz.sum(axis=1) == 9).all()
    # the forward hop block of site s is L_{2mu}(s) at column block s+mu  (R3/R8)
    s = 17
    x = synth.site_coords(dims, s)
    for mu in range(4):
        xf = x.copy(); xf[mu] = (xf[mu] + 1) % dims[mu]
        sf = int(synth.site_index(dims, xf))
        np.testing.assert_array_equal(D[s * N:(s + 1) * N, sf * N:(sf + 1) * N], L[s, 2 * mu])


def test_dense_double_hops_L2():
    """L_mu = 2: x+mu == x-mu, both terms are added (R10)."""
    dims, N = (2, 1, 1, 1), 2
    L = crandn(2, 9, N, N)
    D = oracle.dense(dims, L)
    blk01 = D[0:N, N:2 * N]
    np.testing.assert_allclose(blk01, L[0, 0] + L[0, 1], rtol=0, atol=1e-15)
    blk00 = D[0:N, 0:N]
    np.testing.assert_allclose(blk00, L[0, 8] + sum(L[0, k] for k in range(2, 8)), rtol=0, atol=1e-14)


# ---------------------------------------------------------------- P2 linearity
def test_linearity():
    dims, N = (2, 3, 2, 4), 8
    L = crandn(vol(dims), 9, N, N)
    u, v = crandn(vol(dims), N), crandn(vol(dims), N)
    a, b = 0.3 - 1.1j, -2.0 + 0.25j
    lhs = oracle.apply(dims, L, a * u + b * v)
    rhs = a * oracle.apply(dims, L, u) + b * oracle.apply(dims, L, v)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)


# ---------------------------------------------------------------- adjoint / P3 tau3-hermiticity
def test_adjoint_identity_general_links():
    """<w, D v> = <D^H w, v> for arbitrary links (pins oracle.adjoint)."""
    dims, N = (3, 2, 4, 3), 6
    L = crandn(vol(dims), 9, N, N)
    v, w = crandn(vol(dims), N), crandn(vol(dims), N)
    lhs = np.vdot(w, oracle.apply(dims, L, v))
    rhs = np.vdot(oracle.adjoint(dims, L, w), v)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(w) * np.linalg.norm(oracle.apply(dims, L, v))
    D = oracle.dense(dims, L)
    np.testing.assert_allclose(oracle.adjoint(dims, L, w).reshape(-1), D.conj().T @ w.reshape(-1),
                               rtol=0, atol=1e-12 * np.abs(D).max() * 50)


@pytest.mark.parametrize("dims", [(2, 2, 2, 2), (3, 4, 2, 3), (1, 2, 1, 3)])
def test_tau3_hermiticity(dims):
    """On tau3-hermitian links (chirality-preserving aggregation, PAPER.md:121 fn. 1) the
    library's dagger tau3 D tau3 is the true adjoint; on general links it is not."""
    N = 8
    Lh = synth.links(dims, N, kind="hermitian")
    v = synth.vector(dims, N)
    w = synth.vector(dims, N, tag=synth.TAG_W)
    Dv = oracle.apply(dims, Lh, v)
    lhs = np.vdot(w, Dv)
    rhs = np.vdot(oracle.apply_dagger_tau3(dims, Lh, w), v)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(w) * np.linalg.norm(Dv)
    np.testing.assert_allclose(oracle.apply_dagger_tau3(dims, Lh, w), oracle.adjoint(dims, Lh, w),
                               rtol=0, atol=1e-13)
    D = oracle.dense(dims, Lh)
    t3 = np.tile(synth.tau3_signs(N), vol(dims))
    np.testing.assert_allclose(t3[:, None] * D * t3[None, :], D.conj().T, rtol=0, atol=1e-15)
    # negative control: general links
    Lg = synth.links(dims, N, kind="general")
    diff = oracle.apply_dagger_tau3(dims, Lg, w) - oracle.adjoint(dims, Lg, w)
    assert np.linalg.norm(diff) > 0.1 * np.linalg.norm(w)


def test_dagger_wiring():
    """P11: dagger(w) = tau3 apply(tau3 w), bit-exact."""
    dims, N = (2, 2, 3, 2), 8
    L = crandn(vol(dims), 9, N, N)
    w = crandn(vol(dims), N)
    t = synth.tau3_signs(N)
    ref = t * oracle.apply(dims, L, t * w)
    np.testing.assert_array_equal(oracle.apply_dagger_tau3(dims, L, w), ref)


# ---------------------------------------------------------------- P4 plane waves (closed form)
@pytest.mark.parametrize("dims,n", [((3, 4, 5, 3), (1, 2, 3, 1)), ((4, 3, 3, 5), (0, 1, 2, 4)),
                                    ((5, 3, 4, 6), (2, 2, 1, 5))])
def test_plane_wave_closed_form(dims, n):
    N = 6
    L = synth.links(dims, N, kind="ti_general")
    u = crandn(N)
    p = 2 * np.pi * np.asarray(n) / np.asarray(dims)
    x = synth.site_coords(dims, np.arange(vol(dims)))
    phase = np.exp(1j * (x @ p))
    v = phase[:, None] * u[None, :]
    M = L[0, 8].copy()
    for mu in range(4):
        M += L[0, 2 * mu] * np.exp(1j * p[mu]) + L[0, 2 * mu + 1] * np.exp(-1j * p[mu])
    ref = phase[:, None] * (M @ u)[None, :]
    y = oracle.apply(dims, L, v)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


# ---------------------------------------------------------------- P5 unit impulse
def test_unit_impulse():
    dims, N = (3, 4, 3, 5), 4
    L = crandn(vol(dims), 9, N, N)
    x0 = np.array([1, 2, 0, 4])
    s0 = int(synth.site_index(dims, x0))
    j0 = 3
    v = np.zeros((vol(dims), N), complex)
    v[s0, j0] = 1.0
    y = oracle.apply(dims, L, v)
    ref = np.zeros_like(y)
    ref[s0] += L[s0, 8][:, j0]
    for mu in range(4):
        xm = x0.copy(); xm[mu] = (xm[mu] - 1) % dims[mu]
        xp = x0.copy(); xp[mu] = (xp[mu] + 1) % dims[mu]
        sm, sp = int(synth.site_index(dims, xm)), int(synth.site_index(dims, xp))
        ref[sm] += L[sm, 2 * mu][:, j0]       # y(x0 - mu) = L_{2mu}(x0 - mu) v(x0)
        ref[sp] += L[sp, 2 * mu + 1][:, j0]   # y(x0 + mu) = L_{2mu+1}(x0 + mu) v(x0)
    np.testing.assert_array_equal(y, ref)


# ---------------------------------------------------------------- P6 shifts == numpy.roll
@pytest.mark.parametrize("mu", [0, 1, 2, 3])
@pytest.mark.parametrize("dirn", [0, 1])
def test_shift_is_roll(mu, dirn):
    dims, N = (3, 4, 5, 6), 4
    V = vol(dims)
    L = np.zeros((V, 9, N, N), complex)
    L[:, 2 * mu + dirn] = np.eye(N)
    v = crandn(V, N)
    y = oracle.apply(dims, L, v)
    # forward hop: y(x) = v(x + mu) = roll by -1 ; backward: roll by +1
    ref = np.roll(as4d(v, dims), -1 if dirn == 0 else +1, axis=axis_of(mu)).reshape(V, N)
    np.testing.assert_array_equal(y, ref)


# ---------------------------------------------------------------- P7 / P8 / P9
def test_block_diagonal_is_batched_matmul():
    dims, N = (2, 3, 2, 2), 48
    V = vol(dims)
    L = np.zeros((V, 9, N, N), complex)
    L[:, 8] = crandn(V, N, N)
    v = crandn(V, N)
    ref = np.matmul(L[:, 8], v[:, :, None])[:, :, 0]
    y = oracle.apply(dims, L, v)
    assert np.max(np.abs(y - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_identity():
    dims, N = (2, 2, 2, 2), 48
    V = vol(dims)
    L = np.zeros((V, 9, N, N), complex)
    L[:, 8] = np.eye(N)
    v = synth.vector(dims, N)
    np.testing.assert_array_equal(oracle.apply(dims, L, v), v)


@pytest.mark.parametrize("dims", [(1, 1, 1, 1), (1, 1, 1, 3), (1, 2, 1, 1)])
def test_L1_self_hops(dims):
    """L_mu = 1: both hops of mu land on x itself (R10)."""
    N = 6
    V = vol(dims)
    L = crandn(V, 9, N, N)
    v = crandn(V, N)
    y = oracle.apply(dims, L, v)
    x = synth.site_coords(dims, np.arange(V))
    for s in range(V):
        ref = L[s, 8] @ v[s]
        for mu in range(4):
            for dirn, step in ((0, 1), (1, -1)):
                xn = x[s].copy(); xn[mu] = (xn[mu] + step) % dims[mu]
                ref = ref + L[s, 2 * mu + dirn] @ v[int(synth.site_index(dims, xn))]
        assert np.max(np.abs(y[s] - ref)) <= 1e-13 * np.max(np.abs(ref))


# ---------------------------------------------------------------- neighbours / site_apply
def test_site_apply_and_neighbours():
    dims, N = (3, 2, 4, 5), 8
    L = crandn(vol(dims), 9, N, N)
    v = crandn(vol(dims), N)
    y = oracle.apply(dims, L, v)
    for s in (0, 7, 63, vol(dims) - 1):
        nb = oracle.neighbours(dims, s)
        x = synth.site_coords(dims, s)
        for mu in range(4):
            xp = x.copy(); xp[mu] = (xp[mu] + 1) % dims[mu]
            xm = x.copy(); xm[mu] = (xm[mu] - 1) % dims[mu]
            assert nb[2 * mu] == synth.site_index(dims, xp)
            assert nb[2 * mu + 1] == synth.site_index(dims, xm)
        assert nb[8] == s
        np.testing.assert_array_equal(oracle.site_apply(L[s], v[nb]), y[s])


# ---------------------------------------------------------------- P10 partition emulation
@pytest.mark.parametrize("dims,P", [((2, 2, 4, 8), (1, 1, 1, 2)), ((2, 2, 4, 8), (1, 1, 2, 4)),
                                    ((2, 2, 4, 8), (1, 1, 1, 8)), ((2, 2, 4, 8), (1, 1, 4, 2)),
                                    ((3, 2, 2, 6), (1, 1, 2, 3)), ((4, 3, 2, 2), (2, 1, 1, 2))])
def test_partitioned_apply_bit_exact(dims, P):
    N = 8
    L = crandn(vol(dims), 9, N, N)
    v = crandn(vol(dims), N)
    np.testing.assert_array_equal(oracle.partitioned_apply(dims, P, L, v), oracle.apply(dims, L, v))


# ---------------------------------------------------------------- halo layout vs numpy slicing
@pytest.mark.parametrize("split", [(0, 0, 0, 1), (0, 0, 1, 1), (1, 0, 1, 0)])
def test_pack_halo_matches_numpy_slices(split):
    ld, N = (2, 3, 3, 5), 4
    V = vol(ld)
    v = crandn(V, N)
    s = rng.random(V).astype(np.float32)
    buf = oracle.pack_halo(ld, split, v, 16 * N, s, 4)
    v4 = as4d(v, ld)
    s4 = s.reshape(ld[3], ld[2], ld[1], ld[0])
    ref = b""
    for mu in range(4):
        if not split[mu]:
            continue
        ax = axis_of(mu)
        for idx in (ld[mu] - 1, 0):   # block A: face for +mu neighbour, block B: for -mu
            ref += np.ascontiguousarray(np.take(v4, idx, axis=ax)).tobytes()
            ref += np.ascontiguousarray(np.take(s4, idx, axis=ax)).tobytes()
            ref += b"\0" * (-len(ref) % 16)   # blocks padded to 16 bytes (R13)
    assert buf == ref


# ---------------------------------------------------------------- fp16 storage vs numpy
def test_quantise_matches_numpy_float16():
    x = crandn(257, 48) * np.exp(rng.uniform(-20, 5, size=(257, 1)))
    x[3] = 0                      # all-zero record (R12: scale 0, payload +0)
    x[5, 7] = 1e-9                # tiny entries -> fp16 subnormals
    q, s = oracle.quantise_fp16(x, 96)
    xf = x.view(np.float64).reshape(257, 96).astype(np.float32)
    sref = np.abs(xf).max(axis=1)
    np.testing.assert_array_equal(s, sref)
    with np.errstate(invalid="ignore", divide="ignore"):
        qref = np.where(sref[:, None] > 0, xf / sref[:, None], np.float32(0)).astype(np.float16)
    np.testing.assert_array_equal(q.reshape(257, 96), qref.view(np.uint16))
    xd = oracle.dequantise_fp16(q, s, 96).reshape(257, 48)
    np.testing.assert_array_equal(xd.view(np.float64).reshape(257, 96),
                                  (qref.astype(np.float32) * sref[:, None]).astype(np.float64))
    # relative error per record is at most 2^-11 of the record's max |component|
    err = np.abs(xd - x).max(axis=1)
    assert (err <= 2.0 ** -11 * np.abs(x).max(axis=1) * 1.0001 + 1e-300).all()


def test_quantised_hermitian_links_stay_hermitian():
    """Paired tau3-hermitian matrices have equal max-abs, so per-matrix fp16 scaling keeps
    the links exactly tau3-hermitian (R12)."""
    dims, N = (2, 2, 2, 2), 48
    Lh = synth.links(dims, N, kind="hermitian")
    q, s = oracle.quantise_fp16(Lh, 2 * N * N)
    Lq = oracle.dequantise_fp16(q, s, 2 * N * N).reshape(Lh.shape)
    w = synth.vector(dims, N, tag=synth.TAG_W)
    np.testing.assert_allclose(oracle.apply_dagger_tau3(dims, Lq, w), oracle.adjoint(dims, Lq, w),
                               rtol=0, atol=1e-13)


# ---------------------------------------------------------------- matrix-free mode (full-size parity)
@pytest.mark.parametrize("kind", ["general", "hermitian", "ti_general", "ti_hermitian"])
@pytest.mark.parametrize("dims,N", [((2, 3, 2, 3), 48), ((3, 2, 1, 4), 64), ((1, 1, 1, 1), 48)])
def test_apply_generated_is_apply_on_synth_links(kind, dims, N):
    """The matrix-free oracle regenerates the links per site with its own copy of the c.3
    recipe; it must equal oracle.apply on synth.links bit for bit (same values, same term
    order) -- which pins its generator to synth (itself pinned by the splitmix64 test vector)
    and its arithmetic to apply (pinned by P1-P10)."""
    v = synth.vector(dims, N)
    L = synth.links(dims, N, kind=kind, scale_log2=-4)
    ref = oracle.apply(dims, L, v)
    got = oracle.apply_generated(dims, N, v, kind=kind, scale_log2=-4)
    np.testing.assert_array_equal(got, ref)


def test_apply_generated_plane_wave_closed_form():
    """Independent pin: translation-invariant links + a plane wave give the closed form of P4
    (SURVEY c.4), without going through oracle.apply."""
    dims, N = (3, 4, 3, 5), 48
    L1 = synth.links((1, 1, 1, 1), N, kind="ti_general")[0]
    n = np.array([1, 2, 0, 3])
    p = 2 * np.pi * n / np.array(dims)
    x = synth.site_coords(dims, np.arange(synth.volume(dims)))
    u = synth.vector((1, 1, 1, 1), N)[0]
    phase = np.exp(1j * (x @ p))
    v = phase[:, None] * u[None, :]
    M = L1[8] + sum(L1[2 * mu] * np.exp(1j * p[mu]) + L1[2 * mu + 1] * np.exp(-1j * p[mu]) for mu in range(4))
    ref = phase[:, None] * (M @ u)[None, :]
    got = oracle.apply_generated(dims, N, v, kind="ti_general")
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
