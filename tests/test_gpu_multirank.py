"""Multi-rank GPU parity (SURVEY §8(e) "Verification", §4 "Distributed tests").

R processes, one rank each, exchange their halos through the library's transports and the
gathered result is checked against the float64 oracle on the whole global lattice:

* ``peer`` transport: every rank maps its halo neighbours' receive windows
  with CUDA IPC and the pack kernel stores the faces straight into them.  CUDA IPC works
  between processes on the SAME GPU, so these tests run R = 2, 4, 8 ranks on one B200 (the
  processes time-slice the GPU; each apply takes milliseconds, the results are exact) and on
  one rank per GPU when more GPUs are visible.
* ``nccl`` transport: ncclSend/ncclRecv (NCCL refuses two ranks on one GPU), so these cases
  run only with >= R visible GPUs and are skipped otherwise.

Checked per case: global relative L2 (per-rank fp64 partial sums, all-reduced)
of D v and D^dagger v vs the oracle; the received halo bytes == oracle.pack_halo of the
neighbours' stored blocks (bit-exact); device-generated links / vectors == the global synth
slice of this rank's origin (bit-exact: the generator uses global indices); invariance vs the
same lattice on one rank; a unit impulse on a partition face (bit-exact fp32); compressed
links (one-time link halo) and the even-odd Schur operator across ranks.  Full-size configs
M4 (6^3x12, Nvec 32, T2) and M5 (16^3x32, Nvec 24, fp16, T2 / T8 / T4xZ2) are compared on the
whole field against the matrix-free oracle.
"""
import os
import socket
import sys
import time
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"fp32": 1e-5, "fp16": 5e-3}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_block(arr, dims, ldims, coords):
    shp = (dims[3], dims[2], dims[1], dims[0]) + arr.shape[1:]
    a4 = arr.reshape(shp)
    sl = tuple(slice(coords[mu] * ldims[mu], (coords[mu] + 1) * ldims[mu]) for mu in (3, 2, 1, 0))
    return np.ascontiguousarray(a4[sl]).reshape((-1,) + arr.shape[1:])


def _coords(rank, pgrid):
    c = []
    for P in pgrid:
        c.append(rank % P)
        rank //= P
    return tuple(c)


def _rel_l2_global(diff2, ref2):
    t = torch.tensor([diff2, ref2], dtype=torch.float64)
    dist.all_reduce(t)
    return float(np.sqrt(t[0] / t[1]))


def _make_ctx(cd, cfg, rank, world, dev):
    nccl_id = None
    if cfg["transport"] == "nccl":
        obj = [cd.cd_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = cd.Context(cfg["dims"], cfg["nvec"], cfg["pgrid"], device=dev, nranks=world, rank=rank, nccl_id=nccl_id)
    if cfg["transport"] == "peer":
        ctx.connect_peers()
    ctx.set_transport(cfg["transport"])
    return ctx


def _stored_record_bytes(oracle, v_local, prec, N):
    """(payload bytes [V, rec], scale bytes [V, 4] or None) of a local vector block as stored."""
    if prec == "fp32":
        return v_local.astype(np.complex64), 8 * N, None
    q, s = oracle.quantise_fp16(v_local, 2 * N)
    return q, 4 * N, s


def _expected_recv(cd, oracle, cfg, rank, vg, prec):
    """The receive buffer of `rank`: per split dim, block A = block A of the -mu neighbour's
    pack, block B = block B of the +mu neighbour's pack (R13 schedule)."""
    dims, nvec, pgrid = cfg["dims"], cfg["nvec"], cfg["pgrid"]
    N = 2 * nvec
    pl = cd.cd_halo_plan_create(dims, nvec, pgrid, rank, prec)
    out = bytearray(pl.total_bytes)
    split = [(pl.split_mask >> m) & 1 for m in range(4)]
    for mu in range(4):
        if not split[mu]:
            continue
        for blk, src_rank in ((0, pl.nbr_rank[mu][1]), (1, pl.nbr_rank[mu][0])):
            spl = cd.cd_halo_plan_create(dims, nvec, pgrid, src_rank, prec)
            vl = _local_block(vg, dims, tuple(spl.local_dims), tuple(spl.grid_coords))
            payload, rec, scales = _stored_record_bytes(oracle, vl, prec, N)
            buf = oracle.pack_halo(tuple(spl.local_dims), split, payload, rec, scales, 0 if scales is None else 4)
            off, nb = pl.block_offset[mu][blk], pl.block_bytes[mu]
            out[off:off + nb] = buf[off:off + nb]
    return bytes(out)


# ---------------------------------------------------------------- checks (run inside each rank)
def check_operator(rank, world, cfg, cd, oracle, synth, dev):
    dims, nvec, pgrid = cfg["dims"], cfg["nvec"], cfg["pgrid"]
    N = 2 * nvec
    ctx = _make_ctx(cd, cfg, rank, world, dev)
    ld, co = ctx.local_dims, ctx.grid_coords
    assert co == _coords(rank, pgrid)
    Lg = synth.links(dims, N, kind="hermitian", scale_log2=-4)
    vg = synth.vector(dims, N)
    Ll, vl = _local_block(Lg, dims, ld, co), _local_block(vg, dims, ld, co)
    ref = _local_block(oracle.apply(dims, Lg, vg), dims, ld, co)
    refd = _local_block(oracle.adjoint(dims, Lg, vg), dims, ld, co)
    out = {}
    for prec in cfg["precs"]:
        # device generator at this rank's origin == the global synth slice (bit-exact)
        L = ctx.links_generate(prec, kind="hermitian", seed=synth.SEED_LINKS, scale_log2=-4)
        raw = np.frombuffer(L.read_stored(), np.uint8)
        if prec == "fp32":
            np.testing.assert_array_equal(raw.view(np.complex64).reshape(Ll.shape), Ll.astype(np.complex64))
        else:
            q, s = oracle.quantise_fp16(Ll, 2 * N * N)
            # values, not bits: the recipes may give -0.0 vs +0.0 for an entry that is exactly zero
            np.testing.assert_array_equal(raw[:q.nbytes].view(np.float16), q.view(np.float16))
            np.testing.assert_array_equal(raw[q.nbytes:].view(np.float32), s)
        fin, fout = ctx.field(prec), ctx.field(prec)
        fin.generate(seed=synth.SEED_VEC, tag=synth.TAG_V)
        if prec == "fp32":
            np.testing.assert_array_equal(fin.export(), vl)
        # halo bytes over the transport == oracle.pack_halo of the neighbours (bit-exact)
        got = ctx.halo_exchange(fin)
        assert got == _expected_recv(cd, oracle, cfg, rank, vg, prec), f"rank {rank} {prec}: halo bytes differ"
        # D v and D^dagger v, twice (the second call runs the tuned variant, new epoch / slot)
        for _ in range(2):
            L.apply(fout, fin)
            y = fout.export()
            e = _rel_l2_global(float(np.sum(np.abs(y - ref) ** 2)), float(np.sum(np.abs(ref) ** 2)))
            assert e <= TOL[prec], (prec, "apply", e)
            L.apply_dagger(fout, fin)
            yd = fout.export()
            ed = _rel_l2_global(float(np.sum(np.abs(yd - refd) ** 2)), float(np.sum(np.abs(refd) ** 2)))
            assert ed <= TOL[prec], (prec, "dagger", ed)
        out[prec] = (e, ed)
        # invariance vs one rank holding the whole lattice (same GPU as rank 0)
        L.apply(fout, fin)
        ys = [None] * world
        dist.all_gather_object(ys, (co, fout.export()))
        if rank == 0:
            one = cd.Context(dims, nvec, device=dev)
            L1 = one.links_generate(prec, kind="hermitian", seed=synth.SEED_LINKS, scale_log2=-4)
            a, b = one.field(prec), one.field(prec)
            a.generate(seed=synth.SEED_VEC, tag=synth.TAG_V)
            L1.apply(b, a)
            y1 = b.export()
            yg = np.zeros_like(y1)
            yg4 = yg.reshape(dims[3], dims[2], dims[1], dims[0], N)
            for c, yl in ys:
                sl = tuple(slice(c[mu] * ld[mu], (c[mu] + 1) * ld[mu]) for mu in (3, 2, 1, 0))
                yg4[sl] = yl.reshape(ld[3], ld[2], ld[1], ld[0], N)
            inv = np.linalg.norm(yg - y1) / np.linalg.norm(y1)
            assert inv <= (1e-6 if prec == "fp32" else 2e-3), (prec, "invariance", inv)
            del L1, a, b, one
        # compressed links across ranks (one-time link halo, then the vector halo per apply)
        C, dev_h = L.compress_hermitian(check=True)
        assert dev_h == 0.0, dev_h
        C.apply(fout, fin)
        y = fout.export()
        ec = _rel_l2_global(float(np.sum(np.abs(y - ref) ** 2)), float(np.sum(np.abs(ref) ** 2)))
        assert ec <= TOL[prec], (prec, "compressed", ec)
        C.apply_dagger(fout, fin)
        yd = fout.export()
        ecd = _rel_l2_global(float(np.sum(np.abs(yd - refd) ** 2)), float(np.sum(np.abs(refd) ** 2)))
        assert ecd <= TOL[prec], (prec, "compressed dagger", ecd)
        del C, L, fin, fout
    # unit impulse on the lowest-T face of rank 0's block (remote hops into rank 0 and its
    # -T neighbour): bit-exact in fp32 when no global extent is 2 (a single product per output)
    if min(dims) >= 3:
        _impulse(ctx, dims, ld, co, N, oracle, synth)
    # even-odd Schur operator across ranks (every local extent even)
    if all(x % 2 == 0 for x in ld):
        out["eo"] = _even_odd(ctx, dims, ld, co, N, Lg, vg, oracle)
    torch.cuda.synchronize()
    dist.barrier()
    return out


def _impulse(ctx, dims, ld, co, N, oracle, synth):
    Lgen = synth.links(dims, N, kind="general")
    v = np.zeros((synth.volume(dims), N), complex)
    s0 = int(synth.site_index(dims, [0, 0, 0, 0]))
    v[s0, 5] = 1.0
    refi = _local_block(oracle.apply(dims, Lgen, v), dims, ld, co)
    Lu = ctx.links_upload(_local_block(Lgen, dims, ld, co), "fp32")
    fi, fo = ctx.field("fp32"), ctx.field("fp32")
    fi.import_(_local_block(v, dims, ld, co))
    Lu.apply(fo, fi)
    np.testing.assert_array_equal(fo.export(), refi)


def _even_odd(ctx, dims, ld, co, N, Lg, vg, oracle):
    Le = Lg.copy()
    Le[:, 8] += np.eye(N)
    par = oracle.parity(dims)
    ve = vg.copy()
    ve[par == 1] = 0
    refe = oracle.schur_apply(dims, Le, ve)
    Lx = ctx.links_upload(_local_block(Le, dims, ld, co), "fp32")
    E = Lx.prepare_eo()
    lpar = oracle.parity(ld)
    xe, ye = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
    xe.import_(np.ascontiguousarray(_local_block(ve, dims, ld, co)[lpar == 0]))
    E.apply_eo(ye, xe)
    r_e = _local_block(refe, dims, ld, co)[lpar == 0]
    got = ye.export()
    ee = _rel_l2_global(float(np.sum(np.abs(got - r_e) ** 2)), float(np.sum(np.abs(r_e) ** 2)))
    assert ee <= 1e-5, ("even-odd", ee)
    return ee


def check_fullsize(rank, world, cfg, cd, oracle, synth, dev):
    """Whole-field parity at a BASELINE full size in the bench's launch configuration (links and
    vectors generated on the device, links x 2^-4, autotuned variant) vs the matrix-free oracle
    on the seeded (unquantised) inputs; D v and the tau3 dagger."""
    dims, nvec, prec = cfg["dims"], cfg["nvec"], cfg["precs"][0]
    N = 2 * nvec
    ctx = _make_ctx(cd, cfg, rank, world, dev)
    ld, co = ctx.local_dims, ctx.grid_coords
    L = ctx.links_generate(prec, kind="general", seed=synth.SEED_LINKS, scale_log2=-4)
    fin, fout = ctx.field(prec), ctx.field(prec)
    fin.generate(seed=synth.SEED_VEC, tag=synth.TAG_V)
    L.apply(fout, fin)   # tunes
    L.apply(fout, fin)
    y = fout.export(dtype=np.complex64)
    L.apply_dagger(fout, fin)
    yd = fout.export(dtype=np.complex64)
    ys = [None] * world
    dist.all_gather_object(ys, (co, y, yd))
    res = {}
    if rank == 0:
        vg = synth.vector(dims, N)
        t = synth.tau3_signs(N)
        ref = oracle.apply_generated(dims, N, vg, kind="general", scale_log2=-4)
        refd = t * oracle.apply_generated(dims, N, t * vg, kind="general", scale_log2=-4)
        for which, r, i in (("apply", ref, 1), ("dagger", refd, 2)):
            yg = np.zeros(r.shape, np.complex64)
            yg4 = yg.reshape(dims[3], dims[2], dims[1], dims[0], N)
            for item in ys:
                c = item[0]
                sl = tuple(slice(c[mu] * ld[mu], (c[mu] + 1) * ld[mu]) for mu in (3, 2, 1, 0))
                yg4[sl] = item[i].reshape(ld[3], ld[2], ld[1], ld[0], N)
            e = float(np.linalg.norm(yg - r) / np.linalg.norm(r))
            assert np.isfinite(yg).all()
            assert e <= TOL[prec], (which, e)
            res[which] = e
    dist.barrier()
    return res


def check_timeout(rank, world, cfg, cd, oracle, synth, dev):
    """A rank that stops calling the collective applies must not hang its neighbour: rank 1
    connects and then never applies; rank 0's apply waits for rank 1's halo, times out after
    CD_OPT_PEER_TIMEOUT_MS, and the NEXT call on its context reports CD_ERR_COMM."""
    dims, nvec = cfg["dims"], cfg["nvec"]
    ctx = _make_ctx(cd, cfg, rank, world, dev)
    L = ctx.links_generate("fp32", scale_log2=-4)
    a, b = ctx.field("fp32"), ctx.field("fp32")
    a.generate()
    out = {}
    if rank == 0:
        ctx.set_option(cd.CD_OPT_PEER_TIMEOUT_MS, 300)
        t0 = time.time()
        L.apply(b, a)
        torch.cuda.synchronize()
        out["waited_s"] = round(time.time() - t0, 3)
        try:
            L.apply(b, a)
            out["code"] = 0
        except cd.CDError as e:
            out["code"] = e.code
        assert out["code"] == cd.CD_ERR_COMM, out
        assert out["waited_s"] < 30, out
    dist.barrier()
    return out


CHECKS = {"operator": check_operator, "fullsize": check_fullsize, "timeout": check_timeout}


def _worker(rank, world, port, cfg, q):
    try:
        sys.path.insert(0, ROOT)
        import oracle
        import synth
        import paper_1612_07873_b200 as cd
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        dev = rank % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        res = CHECKS[cfg["check"]](rank, world, cfg, cd, oracle, synth, dev)
        q.put((rank, "ok", res))
    except BaseException:  # noqa: BLE001 -- report every rank's failure to the parent
        q.put((rank, "err", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            try:
                dist.destroy_process_group()
            except Exception:
                pass


def _run(world, cfg, timeout=900):
    if cfg["transport"] == "nccl" and torch.cuda.device_count() < world:
        pytest.skip(f"NCCL needs one GPU per rank ({world} ranks, {torch.cuda.device_count()} GPUs visible)")
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    results, t0 = {}, time.time()
    while len(results) < world and time.time() - t0 < timeout:
        if not q.empty():
            r, st, payload = q.get()
            results[r] = (st, payload)
            if st == "err":
                break
        else:
            time.sleep(0.05)
            if all(not p.is_alive() for p in procs) and q.empty():
                break
    for p in procs:
        p.join(timeout=30 if len(results) == world else 1)
        if p.is_alive():
            p.kill()
    errs = [f"rank {r}:\n{payload}" for r, (st, payload) in sorted(results.items()) if st == "err"]
    assert not errs, "\n".join(errs)
    assert len(results) == world, f"only {len(results)} of {world} ranks reported within {timeout} s"
    return {r: payload for r, (st, payload) in results.items()}


# ---------------------------------------------------------------- cases
OPERATOR_CASES = [
    # (world, global dims, proc grid, nvec): T, T with local T = 1 (both hops remote, one peer) and
    # 2, Z x T, 8 ranks; the even-odd stage runs where every local extent is even, the impulse
    # (bit-exact) where every global extent is >= 3 (no double hops)
    (2, (4, 3, 4, 6), (1, 1, 1, 2), 24),
    (2, (4, 2, 2, 4), (1, 1, 1, 2), 24),
    (2, (3, 3, 3, 2), (1, 1, 1, 2), 24),
    (4, (4, 3, 4, 4), (1, 1, 2, 2), 24),
    (4, (4, 2, 4, 4), (1, 1, 2, 2), 32),
    (4, (3, 4, 3, 8), (1, 1, 1, 4), 32),
    (8, (4, 2, 4, 8), (1, 1, 2, 4), 24),
    (8, (3, 3, 3, 16), (1, 1, 1, 8), 24),
]


@pytest.mark.parametrize("transport", ["peer", "nccl"])
@pytest.mark.parametrize("world,dims,pgrid,nvec", OPERATOR_CASES)
def test_multirank_operator(world, dims, pgrid, nvec, transport):
    cfg = {"check": "operator", "dims": dims, "pgrid": pgrid, "nvec": nvec, "precs": ["fp32", "fp16"],
           "transport": transport}
    res = _run(world, cfg)
    print(world, dims, pgrid, transport, res[0])


FULL_CASES = [
    # M4: 6^3 x 12, Nvec 32, T-partitioned on 2 ranks (BASELINE configs[3])
    (2, (6, 6, 6, 12), (1, 1, 1, 2), 32, "fp32"),
    # M5: 16^3 x 32, Nvec 24, fp16, 2 / 8 ranks in T and 8 ranks as T4 x Z2 (BASELINE configs[4])
    (2, (16, 16, 16, 32), (1, 1, 1, 2), 24, "fp16"),
    (8, (16, 16, 16, 32), (1, 1, 1, 8), 24, "fp16"),
    (8, (16, 16, 16, 32), (1, 1, 2, 4), 24, "fp16"),
]


@pytest.mark.parametrize("transport", ["peer", "nccl"])
@pytest.mark.parametrize("world,dims,pgrid,nvec,prec", FULL_CASES)
def test_multirank_fullsize_whole_field(world, dims, pgrid, nvec, prec, transport):
    cfg = {"check": "fullsize", "dims": dims, "pgrid": pgrid, "nvec": nvec, "precs": [prec], "transport": transport}
    res = _run(world, cfg, timeout=1500)
    print(world, dims, pgrid, transport, res[0])


def test_peer_timeout_reports_comm_error():
    cfg = {"check": "timeout", "dims": (4, 4, 4, 4), "pgrid": (1, 1, 1, 2), "nvec": 24, "precs": ["fp32"],
           "transport": "peer"}
    res = _run(2, cfg, timeout=300)
    print(res[0])
