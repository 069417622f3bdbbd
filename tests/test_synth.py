"""The seeded input generator (synth/): reference vector, value grid, counters, recipes."""
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vector():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if not l.startswith("#")]
    for a, b in rows:
        assert int(synth.splitmix64(np.uint64(int(a, 16)))) == int(b, 16)


def test_uniform_grid_and_range():
    u = synth.uniform(synth.SEED_VEC, synth.TAG_V, np.arange(200000, dtype=np.uint64))
    assert u.min() >= -1.0 and u.max() < 1.0
    np.testing.assert_array_equal(u * 2 ** 21, np.round(u * 2 ** 21))
    np.testing.assert_array_equal(u.astype(np.float32).astype(np.float64), u)
    assert abs(u.mean()) < 0.01 and abs(u.std() - 1 / np.sqrt(3)) < 0.01


def test_counter_layout_vector():
    dims, N = (2, 3, 2, 2), 48
    v = synth.vector(dims, N)
    s, i = 17, 29
    ctr = np.array([(s * N + i) * 2, (s * N + i) * 2 + 1], dtype=np.uint64)
    u = synth.uniform(synth.SEED_VEC, synth.TAG_V, ctr)
    assert v[s, i] == u[0] + 1j * u[1]
    # sub-selection by global site equals the full field's rows
    np.testing.assert_array_equal(synth.vector(dims, N, sites=[5, 17]), v[[5, 17]])


def test_counter_layout_links():
    dims, N = (2, 2, 2, 2), 48
    L = synth.links(dims, N)
    s, k, i, j = 11, 5, 40, 3
    c = ((((s * 9 + k) * N + i) * N + j) * 2)
    u = synth.uniform(synth.SEED_LINKS, synth.TAG_LINKS, np.array([c, c + 1], dtype=np.uint64))
    assert L[s, k, i, j] == u[0] + 1j * u[1]
    np.testing.assert_array_equal(synth.links(dims, N, sites=[3, 11]), L[[3, 11]])


@pytest.mark.parametrize("dims", [(2, 2, 2, 2), (3, 1, 2, 4)])
def test_hermitian_recipe_relations(dims):
    N = 8
    L = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    sig = synth.tau3_signs(N)
    ss = sig[:, None] * sig[None, :]
    V = int(np.prod(dims))
    x = synth.site_coords(dims, np.arange(V))
    for s in range(V):
        np.testing.assert_array_equal(L[s, 8], ss * L[s, 8].conj().T)
        for mu in range(4):
            xp = x[s].copy(); xp[mu] = (xp[mu] + 1) % dims[mu]
            sp = int(synth.site_index(dims, xp))
            # L_{2mu+1}(x+mu) = tau3 L_{2mu}(x)^H tau3
            np.testing.assert_array_equal(L[sp, 2 * mu + 1], ss * L[s, 2 * mu].conj().T)
    # exact in fp32
    r = L.view(np.float64)
    np.testing.assert_array_equal(r.astype(np.float32).astype(np.float64), r)
