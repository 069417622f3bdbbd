"""Small invocation of every kernel family (run under compute-sanitizer by tests/test_sanitizers.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1612_07873_b200 as cd  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
os.environ.setdefault("CD_TUNE", "0")
for prec in ("fp32", "fp16"):
    ctx = cd.Context((2, 2, 2, 2), 24)
    L = ctx.links_generate(prec, kind="hermitian", scale_log2=-4)
    a, b = ctx.field(prec), ctx.field(prec)
    a.generate()
    if which in ("all", "apply"):
        for v in range(len(ctx.variants(prec))):
            ctx.set_option(cd.CD_OPT_VARIANT, v)
            L.apply(b, a)
            L.apply_dagger(a, b)
    if which in ("all", "chain"):
        for v in [5000, 4000, 1000, 2001, 2002, 1, 3001, 3002, 3003]:
            ctx.set_option(cd.CD_OPT_VARIANT, v)
            try:
                L.apply_chain(a, b, 3)
            except cd.CDError:
                pass
    if which in ("all", "halo"):
        h = cd.Context((2, 2, 2, 4), 24)
        h.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1100)
        Lh = h.links_generate(prec, scale_log2=-4)
        x, y = h.field(prec), h.field(prec)
        x.generate()
        for v in range(len(h.variants(prec))):
            h.set_option(cd.CD_OPT_VARIANT, v)
            Lh.apply(y, x)
    if which in ("all", "transport"):
        # halo self exchanges through the peer transport (pack kernel -> own IPC window, arrival
        # wait kernel) and through a 1-rank NCCL communicator; the chunked bulk path (compressed
        # links' link halo, multi-RHS faces) under the peer transport
        for tr in ("peer", "nccl"):
            h = cd.Context((2, 2, 2, 4), 24)
            h.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1010)
            if tr == "peer":
                h.peer_connect([h.peer_handle()])
            h.set_transport(tr)
            Lh = h.links_generate(prec, kind="hermitian", scale_log2=-4)
            x, y = h.field(prec), h.field(prec)
            x.generate()
            for v in (-1, 0):   # heuristic choice, and the ring (fused split apply on the peer transport)
                h.set_option(cd.CD_OPT_VARIANT, v)
                Lh.apply(y, x)
                Lh.apply_dagger(x, y)
            h.set_option(cd.CD_OPT_VARIANT, -1)
            h.halo_exchange(x)
            # the fused split apply with several sites per CTA (stage reuse, face sites last)
            fz = cd.Context((8, 8, 4, 5), 24)
            fz.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1000)
            if tr == "peer":
                fz.peer_connect([fz.peer_handle()])
            fz.set_transport(tr)
            Lf = fz.links_generate(prec, kind="hermitian", scale_log2=-4)
            fa, fb = fz.field(prec), fz.field(prec)
            fa.generate()
            for v, nm in enumerate(fz.variants(prec)):
                if nm.startswith("ring"):
                    fz.set_option(cd.CD_OPT_VARIANT, v)
                    Lf.apply(fb, fa)
                    Lf.apply_dagger(fa, fb)
            Ch, _ = Lh.compress_hermitian()
            Ch.apply(y, x)
            if prec == "fp16":
                mx, my = h.field("fp16", nrhs=128), h.field("fp16", nrhs=128)
                mx.generate()
                Lh.apply_mrhs(my, mx)
    if which in ("all", "ring"):
        # every persistent ring variant with several sites per CTA (stage reuse across sites)
        rr = cd.Context((8, 8, 4, 5), 24)
        Lr = rr.links_generate(prec, scale_log2=-4)
        ra, rb = rr.field(prec), rr.field(prec)
        ra.generate()
        for v, nm in enumerate(rr.variants(prec)):
            if nm.startswith("ring"):
                rr.set_option(cd.CD_OPT_VARIANT, v)
                Lr.apply(rb, ra)
                Lr.apply_dagger(ra, rb)
    if which in ("all", "mrhs") and prec == "fp16":
        # 4^4 x 128 rhs: 256 items over 148 CTAs (ring stages and B slots reused)
        mr = cd.Context((4, 4, 4, 4), 24)
        ml4 = mr.links_generate("fp16", kind="hermitian", scale_log2=-4)
        m4x, m4y = mr.field("fp16", nrhs=128), mr.field("fp16", nrhs=128)
        m4x.generate()
        ml4.apply_mrhs(m4y, m4x)
        x, y = ctx.field("fp16", nrhs=128), ctx.field("fp16", nrhs=128)
        x.generate()
        L.apply_mrhs(y, x)
        mc = cd.Context((2, 2, 2, 4), 24)
        mc.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1001)
        ml = mc.links_generate("fp16", kind="hermitian", scale_log2=-4)
        mx, my = mc.field("fp16", nrhs=128), mc.field("fp16", nrhs=128)
        mx.generate()
        ml.apply_mrhs(my, mx)
        ml.apply_mrhs(mx, my, dagger=True)
    if which in ("all", "compressed"):
        C, _ = L.compress_hermitian()
        ctx.set_option(cd.CD_OPT_VARIANT, -1)
        C.apply(b, a)
        C.apply_dagger(a, b)
        cc = cd.Context((2, 2, 2, 4), 24)
        cc.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1001)
        Cc, _ = cc.links_generate(prec, kind="hermitian", scale_log2=-4).compress_hermitian()
        ca, cb = cc.field(prec), cc.field(prec)
        ca.generate()
        Cc.apply(cb, ca)
        Cc.apply_dagger(ca, cb)
        rc = cd.Context((8, 8, 4, 5), 24)   # V >= 4 x SMs: the compressed TMA ring (dslash_ringh)
        Cr, _ = rc.links_generate(prec, kind="hermitian", scale_log2=-4).compress_hermitian()
        ra, rb = rc.field(prec), rc.field(prec)
        ra.generate()
        Cr.apply(rb, ra)
        Cr.apply_dagger(ra, rb)
    if which in ("all", "eo") and prec == "fp32":
        E = L.prepare_eo()
        xe, ye = ctx.field("fp32", parity=0), ctx.field("fp32", parity=0)
        xe.import_(torch.randn(ctx.V // 2, ctx.N, dtype=torch.complex64))
        E.apply_eo(ye, xe)
        E.apply_eo(xe, ye, dagger=True)
        hc = cd.Context((2, 2, 2, 4), 24)
        hc.set_option(cd.CD_OPT_HALO_SELF_MASK, 0b1001)
        He = hc.links_generate("fp32", kind="hermitian", scale_log2=-4).prepare_eo()
        he_x, he_y = hc.field("fp32", parity=0), hc.field("fp32", parity=0)
        he_x.import_(torch.randn(hc.V // 2, hc.N, dtype=torch.complex64))
        He.apply_eo(he_y, he_x)
        He.apply_eo(he_x, he_y, dagger=True)
    if which in ("all", "transfer"):
        for cdims, block, ns, nc in (((2, 1, 1, 1), (4, 4, 2, 4), 4, 3), ((2, 2, 2, 2), (1, 1, 1, 1), 2, 24),
                                     ((1, 1, 1, 2), (2, 2, 1, 2), 2, 5)):
            tc = cd.Context(cdims, 24)
            T = tc.transfer(block, ns, nc, torch.randn(tc.V * int(torch.tensor(block).prod()), ns, nc, 24,
                                                       dtype=torch.complex64, device="cuda"))
            T.orthonormalise()
            f = T.fine_field()
            c = tc.field(prec)
            c.generate()
            T.prolong(f, c)
            T.restrict(c, f)
torch.cuda.synchronize()
print("sanitize run ok")
