"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle.

Gates (BASELINE.json north_star, R17): relative L2 error <= 1e-5 for fp32 storage,
<= 5e-3 for fp16 storage; bit-exact where no arithmetic happens (layouts, import/export,
quantisation, halo pack buffers) and where a single exact product is summed (impulse, shift,
identity).  All inputs are seeded (synth/), identical on both sides.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1612_07873_b200 as cd  # noqa: E402

TOL = {"fp32": 1e-5, "fp16": 5e-3}


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def vol(d):
    return int(np.prod(d))


def run_apply(ctx, links_np, v_np, prec, dagger=False, variant=None):
    if variant is not None:
        ctx.set_option(cd.CD_OPT_VARIANT, variant)
    L = ctx.links_upload(links_np, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v_np)
    (L.apply_dagger if dagger else L.apply)(fout, fin)
    y = fout.export()
    torch.cuda.synchronize()
    return y


# ---------------------------------------------------------------- data movement (bit-exact)
@pytest.mark.parametrize("nvec", [24, 32])
def test_field_roundtrip_fp32(nvec):
    dims = (2, 3, 2, 2)
    ctx = cd.Context(dims, nvec)
    v = synth.vector(dims, 2 * nvec)
    f = ctx.field("fp32")
    f.import_(v)
    np.testing.assert_array_equal(f.export(), v)
    f.import_(v.astype(np.complex64))
    np.testing.assert_array_equal(f.export(dtype=np.complex64), v.astype(np.complex64))


@pytest.mark.parametrize("nvec", [24, 32])
def test_field_fp16_quantisation_bit_exact(nvec):
    dims = (2, 2, 3, 2)
    N = 2 * nvec
    ctx = cd.Context(dims, nvec)
    rng = np.random.default_rng(7)
    v = (rng.standard_normal((vol(dims), N)) + 1j * rng.standard_normal((vol(dims), N))) * \
        np.exp(rng.uniform(-8, 4, (vol(dims), 1)))
    v[1] = 0
    f = ctx.field("fp16")
    f.import_(v)
    raw = np.frombuffer(f.read_stored(), np.uint8)
    q, s = oracle.quantise_fp16(v, 2 * N)
    np.testing.assert_array_equal(raw[:q.nbytes].view(np.uint16), q)
    np.testing.assert_array_equal(raw[q.nbytes:].view(np.float32), s)
    np.testing.assert_array_equal(f.export(), oracle.dequantise_fp16(q, s, 2 * N).reshape(v.shape))


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_links_upload_stored_bit_exact(prec):
    dims, nvec = (2, 2, 2, 2), 24
    N = 2 * nvec
    ctx = cd.Context(dims, nvec)
    Lh = synth.links(dims, N, kind="general")
    L = ctx.links_upload(Lh, prec)
    raw = np.frombuffer(L.read_stored(), np.uint8)
    if prec == "fp32":
        np.testing.assert_array_equal(raw.view(np.complex64).reshape(Lh.shape), Lh.astype(np.complex64))
    else:
        q, s = oracle.quantise_fp16(Lh, 2 * N * N)
        np.testing.assert_array_equal(raw[:q.nbytes].view(np.uint16), q)
        np.testing.assert_array_equal(raw[q.nbytes:].view(np.float32), s)


@pytest.mark.parametrize("kind", ["general", "hermitian", "ti_general", "ti_hermitian"])
@pytest.mark.parametrize("nvec", [24, 32])
def test_device_generator_matches_synth(kind, nvec):
    """The device generator (independent CUDA implementation) == synth (numpy), bit for bit."""
    dims = (2, 3, 2, 3)
    N = 2 * nvec
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate("fp32", kind=kind, seed=0x1612, scale_log2=-4)
    ref = synth.links(dims, N, kind=kind, scale_log2=-4)
    got = np.frombuffer(L.read_stored(), np.complex64).reshape(ref.shape)
    np.testing.assert_array_equal(got, ref.astype(np.complex64))
    f = ctx.field("fp32")
    f.generate(seed=0x7873, tag=2)
    np.testing.assert_array_equal(f.export(), synth.vector(dims, N))
    # fp16 generation == quantisation of the same values
    L16 = ctx.links_generate("fp16", kind=kind, seed=0x1612, scale_log2=-4)
    raw = np.frombuffer(L16.read_stored(), np.uint8)
    q, s = oracle.quantise_fp16(ref, 2 * N * N)
    # values, not bits: the two recipes may give -0.0 vs +0.0 for an entry that is exactly zero
    np.testing.assert_array_equal(raw[:q.nbytes].view(np.float16), q.view(np.float16))
    np.testing.assert_array_equal(raw[q.nbytes:].view(np.float32), s)


@pytest.mark.parametrize("rank", [0, 1, 2, 3])
def test_device_generator_partitioned_global_indices(rank):
    """Each rank's block of a partitioned lattice equals the corresponding global slice: a
    context for `rank` of proc grid (1, 1, 2, 2) (no communicator is needed to generate)
    generates links and vectors at its grid origin (csrc/fields.cu) bit-exactly."""
    dims, nvec, pgrid = (2, 3, 4, 6), 24, (1, 1, 2, 2)
    N = 2 * nvec
    ctx = cd.Context(dims, nvec, pgrid, nranks=4, rank=rank)
    ld, co = ctx.local_dims, ctx.grid_coords
    assert co == (0, 0, rank % 2, rank // 2) and ld == (2, 3, 2, 3)
    def block(a):
        a4 = a.reshape((dims[3], dims[2], dims[1], dims[0]) + a.shape[1:])
        sl = tuple(slice(co[mu] * ld[mu], (co[mu] + 1) * ld[mu]) for mu in (3, 2, 1, 0))
        return np.ascontiguousarray(a4[sl]).reshape((-1,) + a.shape[1:])
    for kind in ("general", "hermitian"):
        full = synth.links(dims, N, kind=kind, scale_log2=-4)
        L = ctx.links_generate("fp32", kind=kind, scale_log2=-4)
        got = np.frombuffer(L.read_stored(), np.complex64).reshape((ctx.V, 9, N, N))
        np.testing.assert_array_equal(got, block(full).astype(np.complex64))
    f = ctx.field("fp32")
    f.generate(seed=0x7873, tag=2)
    np.testing.assert_array_equal(f.export(), block(synth.vector(dims, N)))


# ---------------------------------------------------------------- operator parity
def _variants(prec, nvec):
    ctx = cd.Context((2, 2, 2, 2), nvec)
    return list(range(len(ctx.variants(prec))))


# (4, 4, 3, 5) Nvec 32: V = 240 > 148 SMs, so the fp32 Nvec-32 ring takes dynamic site tickets
CASES = [((2, 2, 2, 2), 24), ((4, 4, 4, 4), 24), ((3, 4, 5, 2), 24), ((2, 3, 2, 4), 32), ((1, 2, 1, 3), 24),
         ((4, 4, 3, 5), 32)]


@pytest.mark.parametrize("dims,nvec", CASES)
@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_apply_all_variants(dims, nvec, prec):
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="general")
    v = synth.vector(dims, N)
    ref = oracle.apply(dims, Lh, v)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    for var in range(len(ctx.variants(prec))):
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        L.apply(fout, fin)
        y = fout.export()
        err = rel_l2(y, ref)
        assert err <= TOL[prec], (ctx.variants(prec)[var], err)
    ctx.set_option(cd.CD_OPT_VARIANT, -1)   # autotuned choice
    L.apply(fout, fin)
    assert rel_l2(fout.export(), ref) <= TOL[prec]


@pytest.mark.parametrize("prec,nvec", [("fp16", 24), ("fp32", 24), ("fp16", 32), ("fp32", 32)])
@pytest.mark.parametrize("dims", [(4, 4, 4, 4), (3, 4, 5, 2), (8, 8, 4, 6)])
def test_ring_gather4_matches_bulk_copies(dims, prec, nvec, monkeypatch):
    """The nine- and three-matrix rings' producer fetches the neighbour vector records with TMA
    gather4 (nine per stage: two gather4 + one bulk copy; three: one gather4 with a duplicate fourth
    row) or with one bulk copy per record (CD_RING_GATHER=0): the same bytes reach the same shared-
    memory slots, so both results are bit-identical, and match the oracle (apply, dagger)."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian")
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    names = ctx.variants(prec)
    rings = [i for i, n in enumerate(names) if n.startswith(("ring_tma_m9", "ring_tma_m3"))]
    assert rings
    for var in rings:
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        for dag, op in ((False, oracle.apply), (True, oracle.adjoint)):
            got = {}
            for g in ("1", "0"):
                monkeypatch.setenv("CD_RING_GATHER", g)
                (L.apply_dagger if dag else L.apply)(fout, fin)
                got[g] = fout.export()
            np.testing.assert_array_equal(got["1"], got["0"])
            assert rel_l2(got["1"], op(dims, Lh, v)) <= TOL[prec], (names[var], dag)
    ctx.set_option(cd.CD_OPT_VARIANT, -1)


@pytest.mark.parametrize("dims,nvec", [((2, 2, 2, 2), 24), ((3, 2, 4, 3), 32), ((4, 4, 4, 4), 24)])
@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_dagger_is_adjoint_on_hermitian_links(dims, nvec, prec):
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian")
    w = synth.vector(dims, N, tag=synth.TAG_W)
    ref = oracle.adjoint(dims, Lh, w)
    np.testing.assert_allclose(oracle.apply_dagger_tau3(dims, Lh, w), ref, rtol=0, atol=1e-12)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(w)
    for var in range(len(ctx.variants(prec))):
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        L.apply_dagger(fout, fin)
        assert rel_l2(fout.export(), ref) <= TOL[prec], ctx.variants(prec)[var]


def test_dagger_general_links_tau3_wiring():
    dims, nvec = (2, 3, 2, 2), 24
    N = 2 * nvec
    Lg = synth.links(dims, N, kind="general")
    w = synth.vector(dims, N, tag=synth.TAG_W)
    y = run_apply(cd.Context(dims, nvec), Lg, w, "fp32", dagger=True)
    assert rel_l2(y, oracle.apply_dagger_tau3(dims, Lg, w)) <= 1e-5


@pytest.mark.parametrize("variant", [0, 1, 9])
def test_unit_impulse_bit_exact(variant):
    dims, nvec = (3, 4, 3, 5), 24
    N = 2 * nvec
    Lh = synth.links(dims, N)
    v = np.zeros((vol(dims), N), complex)
    s0 = int(synth.site_index(dims, [1, 2, 0, 4]))
    v[s0, 17] = 1.0
    y = run_apply(cd.Context(dims, nvec), Lh, v, "fp32", variant=variant)
    np.testing.assert_array_equal(y, oracle.apply(dims, Lh, v))


@pytest.mark.parametrize("mu", [0, 1, 2, 3])
@pytest.mark.parametrize("dirn", [0, 1])
def test_shift_bit_exact(mu, dirn):
    dims, nvec = (3, 4, 3, 5), 24
    N = 2 * nvec
    L = np.zeros((vol(dims), 9, N, N), complex)
    L[:, 2 * mu + dirn] = np.eye(N)
    v = synth.vector(dims, N)
    y = run_apply(cd.Context(dims, nvec), L, v, "fp32")
    ref = np.roll(v.reshape(dims[3], dims[2], dims[1], dims[0], N), -1 if dirn == 0 else 1,
                  axis=3 - mu).reshape(-1, N)
    np.testing.assert_array_equal(y, ref)


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_identity_bit_exact(prec):
    dims, nvec = (2, 2, 2, 2), 32
    N = 2 * nvec
    L = np.zeros((vol(dims), 9, N, N), complex)
    L[:, 8] = np.eye(N)
    v = synth.vector(dims, N)
    y = run_apply(cd.Context(dims, nvec), L, v, prec)
    if prec == "fp32":
        np.testing.assert_array_equal(y, v)
    else:
        q, s = oracle.quantise_fp16(v, 2 * N)
        np.testing.assert_array_equal(y, oracle.dequantise_fp16(q, s, 2 * N).reshape(v.shape))


def test_linearity_fp32():
    dims, nvec = (2, 2, 3, 2), 24
    N = 2 * nvec
    Lh = synth.links(dims, N)
    u, v = synth.vector(dims, N), synth.vector(dims, N, tag=synth.TAG_W)
    ctx = cd.Context(dims, nvec)
    a, b = 0.5, -0.25   # powers of two: exact scaling
    y1 = run_apply(ctx, Lh, a * u + b * v, "fp32")
    y2 = a * run_apply(ctx, Lh, u, "fp32") + b * run_apply(ctx, Lh, v, "fp32")
    assert rel_l2(y1, y2) <= 1e-6


# ---------------------------------------------------------------- halo path on one GPU (self exchange)
@pytest.mark.parametrize("transport", ["copy", "nccl", "peer"])
@pytest.mark.parametrize("mask", [0b1000, 0b1100, 0b0101, 0b1111])
@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_halo_self_exchange(mask, prec, transport):
    """Route split dims through pack -> exchange -> interior + halo-term kernels with P_mu = 1
    (the +mu neighbour is this rank): results match the oracle and the pack buffer is
    bit-exact against oracle.pack_halo.  transport "nccl": a 1-rank communicator, so the real
    ncclGroupStart/Send/Recv/GroupEnd code runs on one GPU (self send/recv); "peer": the pack
    kernel stores into this rank's own IPC window and the wait kernel checks the counters."""
    dims, nvec = (2, 3, 4, 3), 24
    N = 2 * nvec
    Lh = synth.links(dims, N)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    if transport == "peer":
        ctx.peer_connect([ctx.peer_handle()])
    ctx.set_transport(transport)
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    split = [(mask >> mu) & 1 for mu in range(4)]
    buf = ctx.halo_pack(fin)
    raw = np.frombuffer(fin.read_stored(), np.uint8)
    if prec == "fp32":
        ref_buf = oracle.pack_halo(dims, split, raw.view(np.complex64), 8 * N)
    else:
        nb = vol(dims) * N * 4
        ref_buf = oracle.pack_halo(dims, split, raw[:nb].copy(), 4 * N, raw[nb:].copy(), 4)
    assert buf == ref_buf
    assert ctx.halo_exchange(fin) == ref_buf   # self exchange: what arrives is what was packed
    ref = oracle.apply(dims, Lh, v)
    for var in range(len(ctx.variants(prec))):
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        L.apply(fout, fin)
        assert rel_l2(fout.export(), ref) <= TOL[prec], ctx.variants(prec)[var]
        L.apply_dagger(fout, fin)
        assert rel_l2(fout.export(), oracle.apply_dagger_tau3(dims, Lh, v)) <= TOL[prec]


# ---------------------------------------------------------------- full-size configs, whole field
FULL = [((8, 8, 8, 8), 24, "fp32"), ((8, 8, 8, 8), 24, "fp16"), ((6, 6, 6, 12), 32, "fp32"),
        ((6, 6, 6, 12), 32, "fp16"), ((16, 16, 16, 32), 24, "fp16")]


@pytest.mark.parametrize("dims,nvec,prec", FULL)
def test_full_size_whole_field(dims, nvec, prec):
    """BASELINE.json configs at full size, every output element: links and vectors generated on
    the device (bench recipe: links x 2^-4, fields from torch memory), the autotuned variant
    bench.py times, D v and the tau3 dagger, against the float64 matrix-free oracle on the SEEDED
    (unquantised) inputs at north_star's gates (1e-5 fp32, 5e-3 fp16).  The output fields are
    pre-filled with NaN so a site the kernel skipped cannot pass on stale values."""
    N = 2 * nvec
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate(prec, kind="general", seed=0x1612, scale_log2=-4)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.generate(seed=0x7873, tag=2)
    v = synth.vector(dims, N)
    t = synth.tau3_signs(N)
    ref = oracle.apply_generated(dims, N, v, kind="general", scale_log2=-4)
    refd = t * oracle.apply_generated(dims, N, t * v, kind="general", scale_log2=-4)
    for dagger, r in ((False, ref), (True, refd)):
        fout._mem.fill_(0xFF)   # NaN in fp32 and fp16 payloads and scales
        (L.apply_dagger if dagger else L.apply)(fout, fin)
        y = fout.export()
        assert np.isfinite(y).all(), dagger
        assert rel_l2(y, r) <= TOL[prec], (dagger, rel_l2(y, r))


def test_cuda_graph_chain_matches_eager():
    """Chained applies captured in a CUDA graph (the bench protocol) == eager applies."""
    dims, nvec = (4, 4, 4, 4), 24
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate("fp32", scale_log2=-4)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    v0 = a.export()
    L.apply(b, a)   # tune outside capture
    torch.cuda.synchronize()
    a.import_(v0)
    for _ in range(3):
        L.apply(b, a)
        L.apply(a, b)
    eager = a.export()
    a.import_(v0)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            L.apply(b, a, stream=s)
            L.apply(a, b, stream=s)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.export(), eager)


# ---------------------------------------------------------------- chained applies (one persistent kernel)
@pytest.mark.parametrize("dims,nvec,prec,n", [((2, 2, 2, 2), 24, "fp32", 7), ((2, 2, 2, 2), 24, "fp16", 3),
                                              ((2, 2, 2, 2), 32, "fp32", 4), ((3, 2, 2, 2), 24, "fp32", 5),
                                              ((4, 4, 4, 4), 24, "fp16", 3)])
def test_apply_chain_matches_oracle(dims, nvec, prec, n):
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="general", scale_log2=-4)
    v = synth.vector(dims, N)
    ref = v
    for _ in range(n):
        ref = oracle.apply(dims, Lh, ref)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, prec)
    x, y = ctx.field(prec), ctx.field(prec)
    x.import_(v)
    L.apply_chain(x, y, n)
    got = (y if n % 2 else x).export()
    assert rel_l2(got, ref) <= (2e-6 * n if prec == "fp32" else 2e-3 * n)


def test_apply_chain_dagger_and_bitwise_vs_single_applies():
    dims, nvec = (2, 2, 2, 2), 24
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    w = synth.vector(dims, N, tag=synth.TAG_W)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, "fp32")
    x, y = ctx.field("fp32"), ctx.field("fp32")
    x.import_(w)
    L.apply_chain(x, y, 3, dagger=True)
    got = y.export()
    ref = w
    for _ in range(3):
        ref = oracle.adjoint(dims, Lh, ref)
    assert rel_l2(got, ref) <= 1e-5
    # same variant through single applies: identical arithmetic -> bitwise equal
    var = ctx.chosen_variant("fp32", dagger=True) if False else None
    for v in range(1, len(ctx.variants("fp32"))):
        ctx.set_option(cd.CD_OPT_VARIANT, v)
        x.import_(w)
        try:
            L.apply_chain(x, y, 3, dagger=True)
        except cd.CDError:
            continue
        chain = y.export()
        x.import_(w)
        L.apply_dagger(y, x)
        L.apply_dagger(x, y)
        L.apply_dagger(y, x)
        np.testing.assert_array_equal(chain, y.export())


@pytest.mark.parametrize("nvec,prec,n", [(24, "fp32", 5), (24, "fp16", 3), (32, "fp16", 3)])
def test_cluster_chain_forced(nvec, prec, n):
    """The whole-lattice thread-block-cluster chain (variant 1000) on the 2^4 coarsest grid."""
    dims = (2, 2, 2, 2)
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_VARIANT, 1000)
    L = ctx.links_upload(Lh, prec)
    x, y = ctx.field(prec), ctx.field(prec)
    for dag in (False, True):
        x.import_(v)
        L.apply_chain(x, y, n, dagger=dag)
        ref, prev = v, None
        for _ in range(n):
            prev, ref = ref, (oracle.adjoint if dag else oracle.apply)(dims, Lh, ref)
        last, other = (y, x) if n % 2 else (x, y)
        assert rel_l2(last.export(), ref) <= (2e-6 * n if prec == "fp32" else 2e-3 * n)
        assert rel_l2(other.export(), prev) <= (2e-6 * n if prec == "fp32" else 2e-3 * n)


@pytest.mark.parametrize("dims,n", [((2, 2, 2, 2), 7), ((2, 2, 2, 2), 1), ((2, 2, 2, 2), 2), ((2, 1, 2, 2), 6),
                                    ((3, 3, 1, 1), 5), ((4, 2, 2, 1), 4), ((2, 1, 1, 1), 3), ((3, 1, 5, 1), 6),
                                    ((4, 4, 1, 1), 5), ((16, 1, 1, 1), 3), ((1, 2, 2, 4), 4)])
def test_cpush_chain_forced(dims, n):
    """Cluster push chain (variant 4000; fp32, Nvec 24, V <= 16): receive-slot mapping for
    extents 1 (self hop), 2 (shared +-mu slot) and >= 3 (two slots); apply and dagger, last and
    previous iterate against the oracle, repeated launches (mbarrier phases restart per launch)."""
    nvec = 24
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_VARIANT, 4000)
    L = ctx.links_upload(Lh, "fp32")
    x, y = ctx.field("fp32"), ctx.field("fp32")
    tol = 2e-6 * n
    for dag in (False, True):
        ref, prev = v, v
        for _ in range(n):
            prev, ref = ref, (oracle.adjoint if dag else oracle.apply)(dims, Lh, ref)
        for _rep in range(2):
            x.import_(v)
            L.apply_chain(x, y, n, dagger=dag)
            last, other = (y, x) if n % 2 else (x, y)
            assert rel_l2(last.export(), ref) <= tol, (dims, dag)
            if n > 1:
                assert rel_l2(other.export(), prev) <= tol, (dims, dag)


@pytest.mark.parametrize("dims,nvec,n", [((2, 2, 2, 2), 24, 7), ((2, 2, 2, 2), 24, 1), ((2, 2, 2, 2), 24, 2),
                                         ((2, 1, 2, 2), 24, 6), ((3, 3, 1, 1), 24, 5), ((3, 2, 2, 2), 24, 4),
                                         ((1, 1, 1, 1), 24, 3), ((2, 2, 2, 2), 32, 4), ((2, 1, 2, 3), 32, 5)])
def test_llwarp_chain_forced(dims, nvec, n):
    """LL-warp chain (variant 5000; fp32): one warp per 4 rows with all nine hops in registers;
    record sharing for extents 1 and 2, apply and dagger, last and previous iterate against the
    oracle, repeated launches (epoch continuity)."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_VARIANT, 5000)
    L = ctx.links_upload(Lh, "fp32")
    x, y = ctx.field("fp32"), ctx.field("fp32")
    tol = 2e-6 * n
    for dag in (False, True):
        ref, prev = v, v
        for _ in range(n):
            prev, ref = ref, (oracle.adjoint if dag else oracle.apply)(dims, Lh, ref)
        for _rep in range(2):
            x.import_(v)
            L.apply_chain(x, y, n, dagger=dag)
            last, other = (y, x) if n % 2 else (x, y)
            assert rel_l2(last.export(), ref) <= tol, (dims, dag)
            if n > 1:
                assert rel_l2(other.export(), prev) <= tol, (dims, dag)


@pytest.mark.parametrize("variant", [4000, 3002])
def test_long_chain_matches_oracle(variant):
    """256 chained applies in one launch: epoch / mbarrier-phase wrap-around over many applies,
    both iterates against 256 float64 oracle applies (links x 2^-4: the norm grows ~1.09x per
    apply, 1e9 after 256, well inside fp32); measured 6-7e-7 after 256, gate 1e-5."""
    dims, nvec, n = (2, 2, 2, 2), 24, 256
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="general", scale_log2=-4)
    v = synth.vector(dims, N)
    ref, prev = v, v
    for _ in range(n):
        prev, ref = ref, oracle.apply(dims, Lh, ref)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_VARIANT, variant)
    L = ctx.links_upload(Lh, "fp32")
    x, y = ctx.field("fp32"), ctx.field("fp32")
    x.import_(v)
    L.apply_chain(x, y, n)
    assert rel_l2(x.export(), ref) <= 1e-5   # n even: the last iterate is in x
    assert rel_l2(y.export(), prev) <= 1e-5


def test_cpush_chain_unsupported_shapes():
    """Variant 4000 refuses lattices above one 16-CTA cluster, a single site (st.async needs a
    cluster of >= 2 CTAs), fp16 storage and Nvec 32."""
    for dims, nvec, prec in (((3, 2, 2, 2), 24, "fp32"), ((1, 1, 1, 1), 24, "fp32"), ((2, 2, 2, 2), 24, "fp16"),
                             ((2, 2, 2, 2), 32, "fp32")):
        ctx = cd.Context(dims, nvec)
        ctx.set_option(cd.CD_OPT_VARIANT, 4000)
        L = ctx.links_generate(prec, scale_log2=-4)
        x, y = ctx.field(prec), ctx.field(prec)
        x.generate()
        with pytest.raises(cd.CDError):
            L.apply_chain(x, y, 3)


@pytest.mark.parametrize("dims,nvec,prec,n", [((2, 2, 2, 2), 24, "fp32", 6), ((2, 2, 2, 2), 24, "fp16", 3),
                                              ((3, 2, 2, 2), 32, "fp32", 5), ((2, 2, 2, 2), 32, "fp16", 4)])
def test_ll_chain_all_variants(dims, nvec, prec, n):
    """LL-protocol chain (variants 2000 + fg id): every variant that fits, apply and dagger,
    both iterates (last and previous) against the oracle; repeated calls (epoch continuity)."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, prec)
    x, y = ctx.field(prec), ctx.field(prec)
    tol = 2e-6 * n if prec == "fp32" else 2e-3 * n
    ran = 0
    for var in range(len(ctx.variants(prec))):
        ctx.set_option(cd.CD_OPT_VARIANT, 2000 + var)
        for dag in (False, True):
            for _rep in range(2):
                x.import_(v)
                try:
                    L.apply_chain(x, y, n, dagger=dag)
                except cd.CDError:
                    break
                ran += 1
                ref, prev = v, None
                for _ in range(n):
                    prev, ref = ref, (oracle.adjoint if dag else oracle.apply)(dims, Lh, ref)
                last, other = (y, x) if n % 2 else (x, y)
                assert rel_l2(last.export(), ref) <= tol, (ctx.variants(prec)[var], dag)
                assert rel_l2(other.export(), prev) <= tol, (ctx.variants(prec)[var], dag)
    assert ran > 0


@pytest.mark.parametrize("dims,nvec,n", [((2, 2, 2, 2), 24, 6), ((2, 2, 2, 2), 24, 1), ((3, 2, 2, 2), 24, 5),
                                         ((2, 2, 2, 2), 32, 4), ((2, 1, 2, 2), 32, 7)])
def test_llreg_chain_all_variants(dims, nvec, n):
    """LL-register chain (variants 3001 + i; fp32): every (rows per CTA, lanes per row) variant
    that fits co-resident, apply and dagger, last and previous iterate against the oracle,
    repeated calls (epoch continuity across launches)."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, "fp32")
    x, y = ctx.field("fp32"), ctx.field("fp32")
    tol = 2e-6 * n
    ran = 0
    for var in range(3001, 3001 + 6):
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        for dag in (False, True):
            for _rep in range(2):
                x.import_(v)
                try:
                    L.apply_chain(x, y, n, dagger=dag)
                except cd.CDError:
                    break
                ran += 1
                ref, prev = v, v
                for _ in range(n):
                    prev, ref = ref, (oracle.adjoint if dag else oracle.apply)(dims, Lh, ref)
                last, other = (y, x) if n % 2 else (x, y)
                assert rel_l2(last.export(), ref) <= tol, (var, dag)
                if n > 1:
                    assert rel_l2(other.export(), prev) <= tol, (var, dag)
    assert ran >= 4


def test_llreg_chain_bitwise_vs_single_applies():
    """Variant 3001 (4 rows per CTA, 8 lanes per row) does the per-row arithmetic of the
    fg_kw1_wr1 single-apply kernel in the same order: a chain of n equals n single applies."""
    dims, nvec, n = (2, 2, 2, 2), 24, 5
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="general", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, "fp32")
    x, y = ctx.field("fp32"), ctx.field("fp32")
    ctx.set_option(cd.CD_OPT_VARIANT, 3001)
    x.import_(v)
    L.apply_chain(x, y, n)
    chain = y.export()
    ctx.set_option(cd.CD_OPT_VARIANT, ctx.variants("fp32").index("fg_kw1_wr1_f32_nv24"))
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.import_(v)
    for _ in range(n):
        L.apply(b, a)
        a, b = b, a
    np.testing.assert_array_equal(chain, a.export())


def test_chain_tuner_reports_choice():
    """The chain tuner's pick is queryable (cd_context_chosen_variant with dagger = 2 / 3)."""
    dims, nvec = (2, 2, 2, 2), 24
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate("fp32", scale_log2=-4)
    x, y = ctx.field("fp32"), ctx.field("fp32")
    x.generate()
    assert ctx.chosen_chain_variant("fp32") == -1
    L.apply_chain(x, y, 4)
    vid = ctx.chosen_chain_variant("fp32")
    assert vid in (1000, 4000, 5000) or 2000 <= vid < 2000 + len(ctx.variants("fp32")) or 3001 <= vid < 3007 \
        or 0 <= vid < len(ctx.variants("fp32"))


# ---------------------------------------------------------------- multi-RHS on tcgen05 tensor cores
@pytest.mark.parametrize("variant", ["ts", "ss", "ss2"])
@pytest.mark.parametrize("dims,nvec,nrhs", [((2, 2, 2, 2), 24, 128), ((2, 3, 2, 2), 32, 128),
                                            ((2, 2, 2, 2), 24, 256),
                                            # several items per CTA (V * nrhs / 128 > 148): ring wrap,
                                            # both accumulators, staging-tile reuse
                                            ((4, 4, 4, 3), 24, 128), ((3, 3, 3, 6), 32, 128),
                                            ((4, 3, 4, 4), 24, 256)])
def test_apply_mrhs_tensor_cores(dims, nvec, nrhs, variant, monkeypatch):
    """NEXT-1: out_r = D in_r for 128 right-hand sides per CTA on tcgen05 (fp16 storage, fp32
    accumulate in TMEM) against the oracle applied to every rhs; apply and dagger.  variant "ts":
    links as the A operand built in tensor memory (default); "ss": links as the shared-memory B
    operand (CD_MRHS_TS=0); "ss2": the same with two CTAs per SM (CD_MRHS_2CTA=1, Nvec 24)."""
    monkeypatch.setenv("CD_MRHS_TS", "1" if variant == "ts" else "0")
    monkeypatch.setenv("CD_MRHS_2CTA", "1" if variant == "ss2" else "0")   # Nvec 24: two CTAs per SM
    N = 2 * nvec
    V = vol(dims)
    for kind, dag in (("general", False), ("hermitian", True)):
        Lh = synth.links(dims, N, kind=kind, scale_log2=-4)
        vs = np.stack([synth.vector(dims, N, tag=2 + r) for r in range(nrhs)])   # [rhs][V][N]
        ctx = cd.Context(dims, nvec)
        L = ctx.links_upload(Lh, "fp16")
        fin, fout = ctx.field("fp16", nrhs=nrhs), ctx.field("fp16", nrhs=nrhs)
        fin.import_(np.ascontiguousarray(vs))
        L.apply_mrhs(fout, fin, dagger=dag)
        got = fout.export()
        op = oracle.adjoint if dag else oracle.apply
        ref = np.stack([op(dims, Lh, vs[r]) for r in range(nrhs)])
        err = rel_l2(got, ref)
        assert err <= 5e-3, (kind, err)
        # per-rhs errors are uniform (no rhs block mis-addressed)
        per = [rel_l2(got[r], ref[r]) for r in range(nrhs)]
        assert max(per) <= 5e-3, max(per)


def test_mrhs_field_roundtrip_and_generate():
    dims, nvec, nrhs = (2, 2, 2, 2), 24, 128
    N = 2 * nvec
    ctx = cd.Context(dims, nvec)
    f = ctx.field("fp16", nrhs=nrhs)
    f.generate(seed=0x7873, tag=2)
    got = f.export()
    # tensor-core layout (R22): one scale per (site, block of 128 rhs)
    vs = np.stack([synth.vector(dims, N, tag=2 + r) for r in range(nrhs)])     # [rhs][V][N]
    blocks = np.ascontiguousarray(vs.transpose(1, 0, 2))                        # [V][rhs][N]: one record per site
    q, s = oracle.quantise_fp16(blocks, 2 * N * nrhs)
    want = oracle.dequantise_fp16(q, s, 2 * N * nrhs).reshape(blocks.shape).transpose(1, 0, 2)
    np.testing.assert_array_equal(got, want)
    # import of the same values stores the same bytes; export inverts it
    g = ctx.field("fp16", nrhs=nrhs)
    g.import_(np.ascontiguousarray(vs))
    assert g.read_stored() == f.read_stored()
    with pytest.raises(cd.CDError):
        ctx.field("fp16", nrhs=100)


# ---------------------------------------------------------------- NEXT-2: hermiticity-compressed links
@pytest.mark.parametrize("dims,nvec", [((2, 2, 2, 2), 24), ((3, 4, 2, 5), 24), ((2, 3, 2, 2), 32),
                                       ((1, 2, 3, 1), 24), ((4, 4, 4, 4), 24)])
def test_compressed_hermitian_links(dims, nvec):
    """X + 4 forward links per site; backward hops from the neighbour's forward link (transposed):
    apply and dagger match the oracle on tau3-hermitian links; the deviation check is exact (0) on
    hermitian links and large on general ones; the stored records are the 5 source matrices."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian")
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, "fp32")
    C, dev = L.compress_hermitian()
    assert dev == 0.0
    raw = np.frombuffer(C.read_stored(), np.complex64).reshape(vol(dims), 5, N, N)
    np.testing.assert_array_equal(raw, Lh[:, [8, 0, 2, 4, 6]].astype(np.complex64))
    fin, fout = ctx.field("fp32"), ctx.field("fp32")
    fin.import_(v)
    C.apply(fout, fin)
    assert rel_l2(fout.export(), oracle.apply(dims, Lh, v)) <= 1e-5
    C.apply_dagger(fout, fin)
    assert rel_l2(fout.export(), oracle.adjoint(dims, Lh, v)) <= 1e-5
    _, dev_g = ctx.links_upload(synth.links(dims, N, kind="general"), "fp32").compress_hermitian()
    assert dev_g > 0.1


# ---------------------------------------------------------------- NEXT-3: even-odd Schur complement
@pytest.mark.parametrize("dims,nvec", [((2, 2, 2, 2), 24), ((4, 2, 2, 4), 24), ((2, 4, 2, 2), 32),
                                       ((4, 4, 4, 4), 24)])
def test_even_odd_schur(dims, nvec):
    """M_ee v_e = X_e v_e - D_eo X_o^-1 D_oe v_e against the oracle (fp64 Gauss-Jordan); the
    dagger (tau3 M tau3) against the oracle on tau3-hermitian links = M^H."""
    N = 2 * nvec
    V = vol(dims)
    par = oracle.parity(dims)
    for kind in ("general", "hermitian"):
        Lh = synth.links(dims, N, kind=kind, scale_log2=-4)
        for s in range(V):
            Lh[s, 8] += np.eye(N)        # well-conditioned X (keeps tau3-hermiticity)
        v = synth.vector(dims, N)
        v[par == 1] = 0
        ref = oracle.schur_apply(dims, Lh, v)[par == 0]
        ctx = cd.Context(dims, nvec)
        L = ctx.links_upload(Lh, "fp32")
        E = L.prepare_eo()
        fin, fout = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
        fin.import_(np.ascontiguousarray(v[par == 0]))
        E.apply_eo(fout, fin)
        assert rel_l2(fout.export(), ref) <= 1e-5, kind
        if kind == "hermitian":
            t = synth.tau3_signs(N)
            refd = t * oracle.schur_apply(dims, Lh, t * v)[par == 0]
            E.apply_eo(fout, fin, dagger=True)
            assert rel_l2(fout.export(), refd) <= 1e-5


def test_even_odd_singular_detected():
    """A singular odd-site X (here X = 0 at the first odd site) is reported, not silently inverted."""
    dims, nvec = (2, 2, 2, 2), 24
    N = 2 * nvec
    Lh = synth.links(dims, N, scale_log2=-4)
    odd = int(np.nonzero(oracle.parity(dims) == 1)[0][0])
    Lh[odd, 8] = 0
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, "fp32")
    with pytest.raises(cd.CDError):
        L.prepare_eo()
    with pytest.raises(ValueError):
        oracle.schur_apply(dims, Lh, synth.vector(dims, N))


# ---------------------------------------------------------------- NEXT-4: prolongator / restrictor
TRANSFER_CASES = [
    ((2, 2, 2, 2), (2, 2, 2, 2), 4, 3, 24),      # Wilson fine grid, one CTA per aggregate
    ((1, 1, 2, 2), (4, 4, 2, 4), 4, 3, 24),      # few aggregates -> 4-CTA clusters
    ((2, 1, 1, 1), (4, 4, 4, 4), 4, 3, 32),      # 8-CTA clusters, Nvec 32
    ((3, 1, 1, 1), (1, 1, 1, 5), 4, 3, 24),      # ragged: Vf = 15 fine sites
    ((2, 2, 1, 2), (2, 1, 2, 2), 2, 24, 32),     # a coarse level as the fine grid (Ns 2, Nc 24)
    ((2, 1, 2, 1), (2, 2, 1, 2), 2, 5, 24),      # generic kernel path, odd rows per chirality
    ((1, 2, 1, 2), (2, 2, 2, 1), 4, 2, 24),      # generic kernel path, Ns 4
]


def _transfer_inputs(cdims, block, Ns, Nc, nvec):
    fd = oracle.fine_dims(cdims, block)
    Vf, nf = vol(fd), Ns * Nc
    W0 = synth.vector(fd, nf * nvec, tag=5).reshape(Vf, Ns, Nc, nvec)
    vf = synth.vector(fd, nf, tag=6).reshape(Vf, Ns, Nc)
    return fd, W0, vf


@pytest.mark.parametrize("cdims,block,Ns,Nc,nvec", TRANSFER_CASES)
def test_transfer_restrict_prolong(cdims, block, Ns, Nc, nvec):
    """R = P^dagger and P against the oracle on an orthonormalised basis; fp32 coarse fields
    (rel-L2 <= 1e-5) and fp16 coarse fields (restrict <= 5e-3; prolong of the stored fp16 field)."""
    import torch
    fd, W0, vf = _transfer_inputs(cdims, block, Ns, Nc, nvec)
    W = oracle.block_orthonormalise(cdims, block, Ns, Nc, nvec, W0)
    ctx = cd.Context(cdims, nvec)
    T = ctx.transfer(block, Ns, Nc, W)
    np.testing.assert_array_equal(T.read_basis(), W.astype(np.complex64))
    fin = torch.from_numpy(vf.astype(np.complex64)).cuda()
    ref_r = oracle.restrict(cdims, block, Ns, Nc, nvec, W, vf)
    vc = synth.vector(cdims, 2 * nvec, tag=7)
    ref_p = oracle.prolong(cdims, block, Ns, Nc, nvec, W, vc)
    for prec, tol in (("fp32", 1e-5), ("fp16", 5e-3)):
        c = ctx.field(prec)
        T.restrict(c, fin)
        assert rel_l2(c.export(), ref_r) <= tol, prec
        c.import_(vc)
        fout = T.fine_field()
        T.prolong(fout, c)
        want = oracle.prolong(cdims, block, Ns, Nc, nvec, W, c.export()) if prec == "fp16" else ref_p
        assert rel_l2(fout.cpu().numpy(), want) <= 1e-5, prec
    # R P = I on the orthonormal basis (coarse -> fine -> coarse)
    c, c2 = ctx.field("fp32"), ctx.field("fp32")
    c.import_(vc)
    fout = T.fine_field()
    T.prolong(fout, c)
    T.restrict(c2, fout)
    assert rel_l2(c2.export(), vc) <= 1e-5


def test_transfer_restrict_bitwise_reproducible():
    """Fixed-order reductions (no atomics): two restricts give identical bytes, clusters included."""
    import torch
    cdims, block, Ns, Nc, nvec = (1, 1, 2, 2), (4, 4, 2, 4), 4, 3, 24
    fd, W0, vf = _transfer_inputs(cdims, block, Ns, Nc, nvec)
    ctx = cd.Context(cdims, nvec)
    T = ctx.transfer(block, Ns, Nc, W0)
    fin = torch.from_numpy(vf.astype(np.complex64)).cuda()
    a, b = ctx.field("fp32"), ctx.field("fp32")
    T.restrict(a, fin)
    T.restrict(b, fin)
    assert a.read_stored() == b.read_stored()


@pytest.mark.parametrize("cdims,block,Ns,Nc,nvec", TRANSFER_CASES[:3] + TRANSFER_CASES[4:])
def test_transfer_orthonormalise(cdims, block, Ns, Nc, nvec):
    """Device block Gram-Schmidt == the oracle's within fp32 storage rounding."""
    fd, W0, _ = _transfer_inputs(cdims, block, Ns, Nc, nvec)
    ctx = cd.Context(cdims, nvec)
    T = ctx.transfer(block, Ns, Nc, W0)
    T.orthonormalise()
    ref = oracle.block_orthonormalise(cdims, block, Ns, Nc, nvec, W0)
    assert rel_l2(T.read_basis(), ref) <= 1e-5


def test_transfer_orthonormalise_rank_deficient():
    cdims, block, Ns, Nc, nvec = (1, 1, 1, 2), (1, 1, 2, 2), 4, 3, 24
    fd, W0, _ = _transfer_inputs(cdims, block, Ns, Nc, nvec)
    W0[:, :, :, 5] = W0[:, :, :, 2] * (0.5 + 0.25j)
    ctx = cd.Context(cdims, nvec)
    T = ctx.transfer(block, Ns, Nc, W0)
    with pytest.raises(cd.CDError):
        T.orthonormalise()


@pytest.mark.parametrize("mask", [0b1000, 0b0101, 0b1111])
def test_even_odd_halo_self_exchange(mask):
    """Multi-rank even-odd path on one GPU: the masked dims go through pack -> exchange (self
    copy) -> interior -> halo kernels for both Schur stages; result == the oracle (and dagger)."""
    dims, nvec = (4, 2, 2, 4), 24
    N = 2 * nvec
    V = vol(dims)
    par = oracle.parity(dims)
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    for s in range(V):
        Lh[s, 8] += np.eye(N)
    v = synth.vector(dims, N)
    v[par == 1] = 0
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    L = ctx.links_upload(Lh, "fp32")
    E = L.prepare_eo()
    fin, fout = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
    fin.import_(np.ascontiguousarray(v[par == 0]))
    E.apply_eo(fout, fin)
    assert rel_l2(fout.export(), oracle.schur_apply(dims, Lh, v)[par == 0]) <= 1e-5
    t = synth.tau3_signs(N)
    E.apply_eo(fout, fin, dagger=True)
    assert rel_l2(fout.export(), (t * oracle.schur_apply(dims, Lh, t * v))[par == 0]) <= 1e-5


@pytest.mark.parametrize("dims,nvec", [((2, 2, 2, 2), 24), ((3, 4, 2, 5), 24), ((2, 3, 2, 2), 32), ((4, 4, 4, 4), 24)])
def test_compressed_hermitian_links_fp16(dims, nvec):
    """fp16 compressed links: the deviation check is exact on quantised tau3-hermitian links (paired
    matrices share their scale, R12); apply / dagger match the oracle (fp16 gate) and the
    uncompressed fp16 apply of the same stored links."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian")
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    L = ctx.links_upload(Lh, "fp16")
    C, dev = L.compress_hermitian()
    assert dev == 0.0
    fin, fout, fref = ctx.field("fp16"), ctx.field("fp16"), ctx.field("fp16")
    fin.import_(v)
    C.apply(fout, fin)
    L.apply(fref, fin)
    assert rel_l2(fout.export(), oracle.apply(dims, Lh, v)) <= 5e-3
    assert rel_l2(fout.export(), fref.export()) <= 2e-3
    C.apply_dagger(fout, fin)
    assert rel_l2(fout.export(), oracle.adjoint(dims, Lh, v)) <= 5e-3
    _, dev_g = ctx.links_upload(synth.links(dims, N, kind="general"), "fp16").compress_hermitian()
    assert dev_g > 0.1


@pytest.mark.parametrize("mask,dims,nvec", [(0b1000, (2, 2, 2, 4), 24), (0b0011, (4, 2, 2, 2), 24),
                                            (0b1111, (2, 2, 2, 2), 24), (0b1000, (2, 3, 2, 4), 32)])
def test_apply_mrhs_halo_self_exchange(mask, dims, nvec):
    """Multi-rank multi-RHS path on one GPU: face blocks packed in the tensor-core layout, exchanged
    (self copy), interior sites overlapped with the exchange, face sites read the receive buffer;
    apply and dagger against the oracle per rhs."""
    N = 2 * nvec
    nrhs = 128
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    vs = np.stack([synth.vector(dims, N, tag=2 + r) for r in range(nrhs)])
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    L = ctx.links_upload(Lh, "fp16")
    fin, fout = ctx.field("fp16", nrhs=nrhs), ctx.field("fp16", nrhs=nrhs)
    fin.import_(np.ascontiguousarray(vs))
    for dag, op in ((False, oracle.apply), (True, oracle.adjoint)):
        L.apply_mrhs(fout, fin, dagger=dag)
        got = fout.export()
        ref = np.stack([op(dims, Lh, vs[r]) for r in range(nrhs)])
        assert max(rel_l2(got[r], ref[r]) for r in range(nrhs)) <= 5e-3, dag


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("fp16", 5e-3)])
@pytest.mark.parametrize("mask,dims,nvec", [(0b1000, (2, 2, 2, 4), 24), (0b0101, (4, 2, 3, 2), 24),
                                            (0b1111, (2, 2, 2, 2), 24), (0b1000, (2, 3, 2, 4), 32)])
def test_compressed_links_halo_self_exchange(mask, dims, nvec, prec, tol):
    """Compressed links on the multi-rank path (one GPU, self exchange): the one-time link halo
    carries the -mu neighbours' forward records, the vector halo the usual faces; the deviation
    check sees the remote pairs through the link halo (exactly 0 on hermitian links)."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian")
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    C, dev = ctx.links_upload(Lh, prec).compress_hermitian()
    assert dev == 0.0
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    C.apply(fout, fin)
    assert rel_l2(fout.export(), oracle.apply(dims, Lh, v)) <= tol
    C.apply_dagger(fout, fin)
    assert rel_l2(fout.export(), oracle.adjoint(dims, Lh, v)) <= tol


# ---------------------------------------------------------------- seeded random geometry sweep
def _fuzz_cases(n=24, seed=20261017):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        dims = tuple(int(d) for d in rng.integers(1, 5, size=4))
        nvec = int(rng.choice([24, 32]))
        prec = str(rng.choice(["fp32", "fp16"]))
        mask = int(rng.integers(0, 16))
        mask &= sum(1 << mu for mu in range(4) if dims[mu] >= 2)   # a halo dim needs two faces... or one
        out.append((dims, nvec, prec, mask, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("dims,nvec,prec,mask,vseed", _fuzz_cases())
def test_random_geometry_sweep(dims, nvec, prec, mask, vseed):
    """Random small lattices (extents 1-4, including L = 1 and L = 2 self/double hops), both
    storages, random halo self-exchange masks, a random forced variant: apply and dagger vs the
    oracle."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", seed=vseed)
    v = synth.vector(dims, N, seed=vseed + 1)
    ctx = cd.Context(dims, nvec)
    if mask:
        ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    nvar = len(ctx.variants(prec))
    ctx.set_option(cd.CD_OPT_VARIANT, vseed % nvar)
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    tol = TOL[prec]
    try:
        L.apply(fout, fin)
    except cd.CDError as e:   # a forced variant may not support this geometry: fall back to the tuner
        assert e.code in (cd.CD_ERR_UNSUPPORTED, cd.CD_ERR_INVALID), e
        ctx.set_option(cd.CD_OPT_VARIANT, -1)
        L.apply(fout, fin)
    assert rel_l2(fout.export(), oracle.apply(dims, Lh, v)) <= tol
    L.apply_dagger(fout, fin)
    assert rel_l2(fout.export(), oracle.adjoint(dims, Lh, v)) <= tol


def _fuzz_split_cases(n=16, seed=20261018):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        dims = tuple(int(d) for d in rng.integers(2, 7, size=4))
        prec = str(rng.choice(["fp32", "fp16"]))
        mask = int(rng.integers(1, 16))
        tr = str(rng.choice(["copy", "nccl", "peer", "peer"]))
        out.append((dims, prec, mask, tr, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("dims,prec,mask,transport,vseed", _fuzz_split_cases())
def test_random_split_sweep(dims, prec, mask, transport, vseed):
    """Random lattices with several sites per CTA (extents 2-6), random halo masks routed through
    a random transport, every ring variant (the peer transport runs them as the fused split apply)
    and the tuned choice: apply and dagger vs the oracle."""
    nvec = 24
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", seed=vseed)
    v = synth.vector(dims, N, seed=vseed + 1)
    ref, refd = oracle.apply(dims, Lh, v), oracle.adjoint(dims, Lh, v)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    if transport == "peer":
        ctx.peer_connect([ctx.peer_handle()])
    ctx.set_transport(transport)
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    names = ctx.variants(prec)
    for var in [i for i, nm in enumerate(names) if nm.startswith("ring")] + [-1]:
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        L.apply(fout, fin)
        assert rel_l2(fout.export(), ref) <= TOL[prec], (names[var] if var >= 0 else "tuned")
        L.apply_dagger(fout, fin)
        assert rel_l2(fout.export(), refd) <= TOL[prec], (names[var] if var >= 0 else "tuned")


# ---------------------------------------------------------------- link kinds (wrong kind -> CD_ERR_INVALID)
def test_link_kinds_rejected_synchronously():
    """Calls given a link kind they do not support fail with CD_ERR_INVALID and enqueue nothing
    (an even-odd object holds 9V/2 + 8V/2 records, a compressed one 5V: indexing them as 9V
    full links would read past the allocation)."""
    dims, nvec = (4, 4, 4, 4), 24
    ctx = cd.Context(dims, nvec)
    L32 = ctx.links_generate("fp32", kind="hermitian", scale_log2=-4)
    L16 = ctx.links_generate("fp16", kind="hermitian", scale_log2=-4)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    E = L32.prepare_eo()
    C32, _ = L32.compress_hermitian(check=False)
    C16, _ = L16.compress_hermitian(check=False)
    m1, m2 = ctx.field("fp16", nrhs=128), ctx.field("fp16", nrhs=128)
    bad = [lambda: E.apply(b, a), lambda: E.apply_dagger(b, a), lambda: E.apply_chain(a, b, 2),
           lambda: E.read_stored(), lambda: E.compress_hermitian(), lambda: C32.apply_chain(a, b, 2),
           lambda: C16.apply_mrhs(m2, m1), lambda: C32.compress_hermitian()]
    for i, f in enumerate(bad):
        with pytest.raises(cd.CDError) as ei:
            f()
        assert ei.value.code == cd.CD_ERR_INVALID, i
    torch.cuda.synchronize()
    # the context is still healthy: a good apply after the rejected ones is correct
    C32.apply(b, a)
    y = b.export()
    L32.apply(b, a)
    assert rel_l2(y, b.export()) <= 1e-5


def test_compressed_links_split_mismatch_rejected():
    """Compressed links built with no halo split have no link halo; enabling a halo split
    afterwards must not let an apply dereference it."""
    dims, nvec = (4, 4, 4, 4), 24
    ctx = cd.Context(dims, nvec)
    L = ctx.links_generate("fp32", kind="hermitian", scale_log2=-4)
    C, _ = L.compress_hermitian(check=False)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1000)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    with pytest.raises(cd.CDError) as ei:
        C.apply(b, a)
    assert ei.value.code == cd.CD_ERR_INVALID
    C2, _ = L.compress_hermitian(check=False)   # rebuilt under the split: fine
    C2.apply(b, a)
    y = b.export()
    L.apply(b, a)
    assert rel_l2(y, b.export()) <= 1e-5


def test_entry_points_restore_current_device():
    dev0 = torch.cuda.current_device()
    ctx = cd.Context((2, 2, 2, 2), 24, device=torch.cuda.device_count() - 1)
    L = ctx.links_generate("fp32")
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    L.apply(b, a)
    b.export()
    assert torch.cuda.current_device() == dev0


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("mask,dims", [(0b1000, (4, 4, 4, 6)), (0b1100, (4, 4, 4, 6)), (0b1000, (4, 3, 4, 1)),
                                       (0b1001, (2, 4, 3, 2)), (0b1111, (3, 2, 2, 3))])
def test_fused_split_apply_is_one_launch(prec, mask, dims):
    """Ring variants on the peer transport run a split apply as ONE launch (pack in the prologue,
    face sites read their remote records from the window in the same kernel);
    CD_FUSE_SPLIT-independent result == the oracle; the unfused path launches pack + interior +
    wait + halo-term kernels.  Includes local extent 1 (both hops of every site remote) and 2
    (x+mu == x-mu)."""
    nvec = 24
    N = 2 * nvec
    Lh = synth.links(dims, N, scale_log2=-4)
    v = synth.vector(dims, N)
    ref = oracle.apply(dims, Lh, v)
    ctx = cd.Context(dims, nvec)
    ctx.set_option(cd.CD_OPT_HALO_SELF_MASK, mask)
    ctx.peer_connect([ctx.peer_handle()])
    ctx.set_transport("peer")
    names = ctx.variants(prec)
    rings = [i for i, n in enumerate(names) if n.startswith("ring")]
    L = ctx.links_upload(Lh, prec)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    for var in rings:
        ctx.set_option(cd.CD_OPT_VARIANT, var)
        L.apply(fout, fin)
        torch.cuda.synchronize()
        n0 = cd.cd_launch_count()
        L.apply(fout, fin)
        torch.cuda.synchronize()
        assert cd.cd_launch_count() - n0 == 1, names[var]
        assert rel_l2(fout.export(), ref) <= TOL[prec], names[var]
    fg = [i for i, n in enumerate(names) if n.startswith("fg")][0]
    ctx.set_option(cd.CD_OPT_VARIANT, fg)
    L.apply(fout, fin)
    torch.cuda.synchronize()
    n0 = cd.cd_launch_count()
    L.apply(fout, fin)
    torch.cuda.synchronize()
    assert cd.cd_launch_count() - n0 == 4    # pack, interior, arrival wait, halo term
    assert rel_l2(fout.export(), ref) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("dims,nvec", [((8, 8, 4, 5), 24), ((6, 5, 4, 6), 32), ((3, 8, 5, 6), 24)])
def test_compressed_ring_matches_fine_grained(prec, dims, nvec, monkeypatch):
    """Large lattices (V >= 4 x SMs) run compressed links on the persistent TMA ring
    (dslash_ringh: backward links read transposed from the neighbours' forward records);
    apply and dagger == the oracle on tau3-hermitian links and == the fine-grained compressed
    kernel (CD_COMP_RING=0 path, checked through the uncompressed apply of the same links)."""
    N = 2 * nvec
    Lh = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    v = synth.vector(dims, N)
    ctx = cd.Context(dims, nvec)
    assert ctx.V >= 4 * torch.cuda.get_device_properties(0).multi_processor_count
    L = ctx.links_upload(Lh, prec)
    C, dev = L.compress_hermitian()
    assert dev == 0.0
    fin, fout, fref = ctx.field(prec), ctx.field(prec), ctx.field(prec)
    fin.import_(v)
    n0 = cd.cd_launch_count()
    C.apply(fout, fin)
    torch.cuda.synchronize()
    assert cd.cd_launch_count() - n0 == 1
    L.apply(fref, fin)
    assert rel_l2(fout.export(), oracle.apply(dims, Lh, v)) <= TOL[prec]
    assert rel_l2(fout.export(), fref.export()) <= (1e-6 if prec == "fp32" else 2e-3)
    C.apply_dagger(fout, fin)
    assert rel_l2(fout.export(), oracle.adjoint(dims, Lh, v)) <= TOL[prec]
    # one CTA per SM (CD_COMP_2CTA=0) instead of two: the same operator
    monkeypatch.setenv("CD_COMP_2CTA", "0")
    C.apply(fref, fin)
    monkeypatch.setenv("CD_COMP_2CTA", "1")
    C.apply(fout, fin)
    assert rel_l2(fref.export(), oracle.apply(dims, Lh, v)) <= TOL[prec]
    assert rel_l2(fout.export(), fref.export()) <= (1e-6 if prec == "fp32" else 2e-3)
    # the producer's vector records by TMA gather4 or by one bulk copy each: bit-identical
    for dag in (False, True):
        got = {}
        for g in ("1", "0"):
            monkeypatch.setenv("CD_RING_GATHER", g)
            (C.apply_dagger if dag else C.apply)(fout, fin)
            got[g] = fout.export()
        np.testing.assert_array_equal(got["1"], got["0"])
