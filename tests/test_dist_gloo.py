"""Multi-rank host logic on CPU: two processes over torch.distributed (gloo, 127.0.0.1).

Every rank takes its decomposition and halo wire layout from the library's host-only
cd_halo_plan_create (the same plan the CUDA path's pack / NCCL exchange / halo-term kernels
use), packs its faces by that plan, exchanges them with the plan's schedule (block A -> +mu,
block B -> -mu) over gloo, applies the stencil reading remote neighbours from the received
blocks, and the gathered result must equal the float64 oracle on the whole lattice.  The packed
buffer is also checked byte-for-byte against oracle.pack_halo.  No GPU is involved.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_block(arr, dims, ldims, coords):
    """Slice the LOCAL block of a global site-major array (x0 fastest)."""
    shp = (dims[3], dims[2], dims[1], dims[0]) + arr.shape[1:]
    a4 = arr.reshape(shp)
    sl = tuple(slice(coords[mu] * ldims[mu], (coords[mu] + 1) * ldims[mu]) for mu in (3, 2, 1, 0))
    return np.ascontiguousarray(a4[sl]).reshape((-1,) + arr.shape[1:])


def _worker(rank, world, port, gdims, pgrid, nvec, prec, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    import paper_1612_07873_b200 as cd
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        N = 2 * nvec
        pl = cd.cd_halo_plan_create(gdims, nvec, pgrid, rank, prec)
        ld = tuple(pl.local_dims)
        co = tuple(pl.grid_coords)
        V = pl.local_volume
        Lg = synth.links(gdims, N)
        vg = synth.vector(gdims, N)
        Ll = _local_block(Lg, gdims, ld, co)
        vl = _local_block(vg, gdims, ld, co)
        # ---- pack by the plan (wire format R13), fp32 records or fp16 payload + scales
        if prec == "fp32":
            payload = vl.astype(np.complex64)
            rec, scales = 8 * N, None
        else:
            qv, sv = oracle.quantise_fp16(vl, 2 * N)
            payload, rec, scales = qv, 4 * N, sv
        assert pl.record_bytes == rec
        send = np.zeros(pl.total_bytes, np.uint8)
        p4 = np.frombuffer(payload.tobytes(), np.uint8).reshape(ld[3], ld[2], ld[1], ld[0], rec)
        s4 = None if scales is None else scales.view(np.uint8).reshape(ld[3], ld[2], ld[1], ld[0], 4)
        for mu in range(4):
            if not (pl.split_mask >> mu) & 1:
                continue
            F = pl.face_sites[mu]
            for blk, idx in ((0, ld[mu] - 1), (1, 0)):
                off = pl.block_offset[mu][blk]
                face = np.take(p4, idx, axis=3 - mu).reshape(-1)
                send[off:off + face.size] = face
                if s4 is not None:
                    sf = np.take(s4, idx, axis=3 - mu).reshape(-1)
                    send[off + F * rec:off + F * rec + sf.size] = sf
        ref = oracle.pack_halo(ld, [(pl.split_mask >> m) & 1 for m in range(4)], payload, rec,
                               scales, 0 if scales is None else 4)
        assert send.tobytes() == ref, "plan layout != oracle.pack_halo"
        # ---- exchange with the plan's schedule
        recv = np.zeros_like(send)
        st, rt = torch.from_numpy(send), torch.from_numpy(recv)
        reqs = []
        for mu in range(4):
            if not (pl.split_mask >> mu) & 1:
                continue
            up, dn = pl.nbr_rank[mu][0], pl.nbr_rank[mu][1]
            oA, oB, nb = pl.block_offset[mu][0], pl.block_offset[mu][1], pl.block_bytes[mu]
            reqs.append(dist.isend(st[oA:oA + nb], up, tag=4 * mu + 0))
            reqs.append(dist.isend(st[oB:oB + nb], dn, tag=4 * mu + 1))
            reqs.append(dist.irecv(rt[oA:oA + nb], dn, tag=4 * mu + 0))
            reqs.append(dist.irecv(rt[oB:oB + nb], up, tag=4 * mu + 1))
        for r in reqs:
            r.wait()
        # ---- local stencil with halos from the receive buffer (fp64 on the stored values)
        if prec == "fp32":
            vloc = payload.astype(np.complex128)

            def halo_rec(off, f):
                return np.frombuffer(recv[off + f * rec: off + (f + 1) * rec].tobytes(), np.complex64).astype(
                    np.complex128)
        else:
            vloc = oracle.dequantise_fp16(qv, sv, 2 * N).reshape(V, N)

            def halo_rec(off, f, mu=None):
                raise AssertionError

        y = np.zeros((V, N), np.complex128)
        for s in range(V):
            x = synth.site_coords(ld, s)
            acc = Ll[s, 8] @ vloc[s]
            for mu in range(4):
                o3 = [nu for nu in range(4) if nu != mu]
                f = (x[o3[2]] * ld[o3[1]] + x[o3[1]]) * ld[o3[0]] + x[o3[0]]
                for dirn, step in ((0, 1), (1, -1)):
                    edge = x[mu] == (ld[mu] - 1 if dirn == 0 else 0)
                    if (pl.split_mask >> mu) & 1 and edge:
                        off = pl.block_offset[mu][1 if dirn == 0 else 0]
                        if prec == "fp32":
                            u = halo_rec(off, f)
                        else:
                            F = pl.face_sites[mu]
                            qq = np.frombuffer(recv[off + f * rec: off + (f + 1) * rec].tobytes(), np.uint16)
                            ss = np.frombuffer(recv[off + F * rec + 4 * f: off + F * rec + 4 * f + 4].tobytes(),
                                               np.float32)
                            u = oracle.dequantise_fp16(qq, ss, 2 * N)
                    else:
                        xn = x.copy()
                        xn[mu] = (xn[mu] + step) % ld[mu]
                        u = vloc[int(synth.site_index(ld, xn))]
                    acc = acc + Ll[s, 2 * mu + dirn] @ u
            y[s] = acc
        ys = [None] * world if rank == 0 else None
        dist.gather_object((co, y), ys, dst=0)
        if rank == 0:
            if prec == "fp32":
                ref_y = oracle.apply(gdims, Lg, vg)
            else:
                qg, s_ = oracle.quantise_fp16(vg, 2 * N)
                ref_y = oracle.apply(gdims, Lg, oracle.dequantise_fp16(qg, s_, 2 * N).reshape(vg.shape))
            got = np.zeros_like(ref_y)
            g4 = got.reshape(gdims[3], gdims[2], gdims[1], gdims[0], N)
            for c, yy in ys:
                sl = tuple(slice(c[mu] * ld[mu], (c[mu] + 1) * ld[mu]) for mu in (3, 2, 1, 0))
                g4[sl] = yy.reshape(ld[3], ld[2], ld[1], ld[0], N)
            err = np.linalg.norm(got - ref_y) / np.linalg.norm(ref_y)
            assert err < 1e-13, err
        # bench plumbing: max over ranks (gloo)
        import bench
        assert bench.dist_max(float(rank + 1), world) == float(world)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("gdims,pgrid", [((2, 3, 2, 4), (1, 1, 1, 2)), ((2, 2, 4, 3), (1, 1, 2, 1)),
                                         ((2, 3, 2, 2), (1, 1, 1, 2))])
@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_two_rank_halo_exchange_gloo(gdims, pgrid, prec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, gdims, pgrid, 24, prec, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_plan_is_host_only_and_consistent():
    import paper_1612_07873_b200 as cd
    pl = cd.cd_halo_plan_create((16, 16, 16, 32), 24, (1, 1, 2, 4), 5, "fp16")
    assert tuple(pl.grid_coords) == (0, 0, 1, 2)
    assert tuple(pl.local_dims) == (16, 16, 8, 8)
    assert pl.split_mask == 0b1100
    assert [tuple(r) for r in pl.nbr_rank][2:] == [(4, 4), (7, 3)]
    assert pl.face_sites[3] == 16 * 16 * 8 and pl.record_bytes == 192 and pl.scale_bytes == 4
    assert pl.block_offset[2][1] == pl.block_bytes[2] and pl.block_offset[3][0] == 2 * pl.block_bytes[2]
    assert pl.total_bytes == 2 * pl.block_bytes[2] + 2 * pl.block_bytes[3]
    with pytest.raises(cd.CDError):
        cd.cd_halo_plan_create((16, 16, 16, 30), 24, (1, 1, 1, 4), 0)
