// dslash_impl.cuh -- sm_100a kernels of the coarse-grid Dirac operator (Eq. 3).
//
//   y(x) = X(x) v(x) + sum_mu [ L_{2mu}(x) v(x+mu) + L_{2mu+1}(x) v(x-mu) ]      (R1-R10)
//
// Two kernel families, both instantiated per (storage precision, Nvec):
//
//  * RING (large lattices): persistent, one CTA per SM.  One producer thread streams each
//    site's nine link matrices -- and next to each the neighbour vector it multiplies -- into a
//    multi-stage shared-memory ring with cp.async.bulk (TMA 1-D, SASS UBLKCP) completed on
//    mbarriers; N/R consumer warps each own R output rows of the site for all nine hops, so the
//    hop ("stencil direction") sum stays in registers (direction splitting is
//    detrimental on large grids).  Lanes split each row dot product D ways (PAPER.md:227-245,
//    Listing 4) and reduce with xor-shuffles.
//
//  * FG (fine-grained, small lattices): a CTA per (site, row block); warps split the nine hops
//    (KW hops per warp) and the rows (WR row-warps); lanes split the dot product.  All link
//    loads (input independent) are issued before griddepcontrol.wait (PDL), the nine neighbour
//    records are staged once per CTA in shared memory, hop partials are reduced through shared
//    memory by one owner thread per row (§6.2-6.4 mapped onto CTAs: grid parallelism
//    x colour-spin x direction x dot-product split, no integer division in the decode).
//
// Dagger (tau3 D tau3, R5): sign flips of input chunks j >= Nvec and output rows
// i >= Nvec, no extra pass.  fp16 storage: FHFMA (fp16 x fp16 + fp32) on the raw half2 words,
// one multiply by s_L * s_v per (row, hop), and a whole-site max-abs before re-quantising y.
#pragma once

#include "device_common.cuh"

#include <cuda.h>   // CUtensorMap (TMA gather4 of the neighbour vector records)

#include <map>
#include <mutex>
#include <tuple>

namespace cd {

// ------------------------------------------------------------------ shared pieces
template <cd_precision P, int NV>
__device__ __forceinline__ bool is_face(const KGeom &g, const int x[4])
{
#pragma unroll
    for (int mu = 0; mu < 4; mu++)
        if (((g.split >> mu) & 1) && (x[mu] == 0 || x[mu] == g.L[mu] - 1)) return true;
    return false;
}

// Store one site's finished rows.  Called by ALL threads of a group of `nthr` threads (named
// barrier `bar_id`, or __syncthreads when bar_id < 0); thread t < N owns row t (fp16 needs the
// whole site for its scale, R12).  fp32: plain store.
template <cd_precision P, int NV>
__device__ __forceinline__ void store_site(unsigned char *out, int site, int row, bool owner, float re, float im,
                                           float *red, int nthr, int bar_id, bool recip = false)
{
    using Q = Cfg<P, NV>;
    if constexpr (P == CD_FP32) {
        if (owner) reinterpret_cast<float2 *>(out + (size_t)site * Q::VREC)[row] = make_float2(re, im);
    } else {
        float m = owner ? fmaxf(fabsf(re), fabsf(im)) : 0.0f;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, shfl_xor(m, o));
        const int warp = (threadIdx.x >> 5), lane = threadIdx.x & 31;
        const int nw = nthr >> 5;
        const int w0 = (bar_id < 0) ? 0 : warp;  // caller passes warp-relative ids via red layout
        (void)w0;
        if (lane == 0) red[warp] = m;
        if (bar_id < 0) __syncthreads(); else bar_named(bar_id, nthr);
        float s = 0.0f;
        for (int w = 0; w < nw; w++) s = fmaxf(s, red[w]);
        if (owner) {
            __half2 q;
            if (s > 0.0f && recip) {
                const float is = __frcp_rn(s);
                q = __halves2half2(__float2half_rn(re * is), __float2half_rn(im * is));
            } else if (s > 0.0f)
                q = __halves2half2(__float2half_rn(__fdiv_rn(re, s)), __float2half_rn(__fdiv_rn(im, s)));
            else q = __halves2half2(__float2half_rn(0.0f), __float2half_rn(0.0f));
            reinterpret_cast<__half2 *>(out + (size_t)site * Q::VREC)[row] = q;
            if (row == 0) *reinterpret_cast<float *>(out + (size_t)site * Q::VREC + Q::VSCALE) = s;
        }
    }
}

// ------------------------------------------------------------------ halo pack (shared by the
// halo_pack kernel and the fused ring prologue).  Face index f of block (mu, blk) -> site index
// (the other three coordinates lexicographic, lowest fastest; x_mu = L-1 for block A, 0 for B).
__device__ __forceinline__ int face_site(const KGeom &g, int mu, int blk, int f)
{
    const int xm = blk == 0 ? sel4(g.L, mu) - 1 : 0;
    if (mu == 0) return f * g.L[0] + xm;
    if (mu == 1) {
        const int x0 = f % g.L[0], r = f / g.L[0];
        return (r * g.L[1] + xm) * g.L[0] + x0;
    }
    if (mu == 2) {
        const int A = g.L[0] * g.L[1];
        const int lo = f % A, hi = f / A;
        return (hi * g.L[2] + xm) * A + lo;
    }
    return f + xm * g.L[0] * g.L[1] * g.L[2];
}

// PackDst entries without dynamic indexing of a kernel parameter (which would force a stack copy)
__device__ __forceinline__ unsigned char *pd_dst(const PackDst &d, int mu, int blk)
{
    unsigned char *a0 = blk ? d.dst[0][1] : d.dst[0][0], *a1 = blk ? d.dst[1][1] : d.dst[1][0];
    unsigned char *a2 = blk ? d.dst[2][1] : d.dst[2][0], *a3 = blk ? d.dst[3][1] : d.dst[3][0];
    return mu == 0 ? a0 : (mu == 1 ? a1 : (mu == 2 ? a2 : a3));
}
__device__ __forceinline__ unsigned long long *pd_flag(const PackDst &d, int mu, int blk)
{
    unsigned long long *a0 = blk ? d.flag[0][1] : d.flag[0][0], *a1 = blk ? d.flag[1][1] : d.flag[1][0];
    unsigned long long *a2 = blk ? d.flag[2][1] : d.flag[2][0], *a3 = blk ? d.flag[3][1] : d.flag[3][0];
    return mu == 0 ? a0 : (mu == 1 ? a1 : (mu == 2 ? a2 : a3));
}

// Elements [start, ...) with step `stride` of block (mu, blk): payload 16-B chunks (four loads in
// flight per thread before their stores), then (fp16) the F scales and the zero padding to 16 B.
template <cd_precision P, int NV>
__device__ __forceinline__ void pack_block(const unsigned char *field, unsigned char *dst, const KGeom &g, int mu,
                                           int blk, int start, int stride)
{
    using Q = Cfg<P, NV>;
    constexpr int PREC = Q::F16 ? 4 * Q::N : 8 * Q::N;
    constexpr int CPR = PREC / 16;
    const int F = sel4(g.F, mu);
    const int np = F * CPR;
    for (int e0 = start; e0 < np; e0 += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int e = e0 + u * stride;
            if (e < np) {
                const int f = e / CPR, ch = e - f * CPR;
                v[u] = *reinterpret_cast<const uint4 *>(field + (size_t)face_site(g, mu, blk, f) * Q::VREC + ch * 16);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int e = e0 + u * stride;
            if (e < np) *reinterpret_cast<uint4 *>(dst + (size_t)e * 16) = v[u];   // record f, chunk ch
        }
    }
    if constexpr (Q::F16) {
        const int npad = (4 - (F & 3)) & 3;
        for (int e = start; e < F + npad; e += stride)
            *reinterpret_cast<float *>(dst + (size_t)F * PREC + (size_t)e * 4) =
                e < F ? *reinterpret_cast<const float *>(field + (size_t)face_site(g, mu, blk, e) * Q::VREC + Q::VSCALE)
                      : 0.0f;
    }
}

// ------------------------------------------------------------------ fused split apply helpers
// (ring + peer transport).  The pack: every CTA of the persistent ring stores its
// grid-stride slice of every face block (wire format R13: payload records, fp16 scales, zero
// padding) straight into the neighbours' windows.
template <cd_precision P, int NV>
__device__ __forceinline__ void fused_pack(const ApplyArgs &a, int start, int stride)
{
    const unsigned char *field = static_cast<const unsigned char *>(a.in);
#pragma unroll 1
    for (int mu = 0; mu < 4; mu++) {
        if (!((a.g.split >> mu) & 1)) continue;
        pack_block<P, NV>(field, pd_dst(a.pd, mu, 0), a.g, mu, 0, start, stride);
        pack_block<P, NV>(field, pd_dst(a.pd, mu, 1), a.g, mu, 1, start, stride);
    }
}

// Run by lanes 1..31 of the producer warp while lane 0 streams the stencil's records: this CTA's
// slice of the pack, then the last CTA to finish releases kPutCtas per block to the receivers (the
// same total a separate halo_pack launch signals, so ranks may mix fused and unfused applies).
template <cd_precision P, int NV>
__device__ __forceinline__ void fused_pack_lanes(const ApplyArgs &a, int lane)
{
    constexpr unsigned kMask = 0xfffffffeu;   // lanes 1..31
    pdl_wait();   // `in` is written by the previous kernel in the stream
    fused_pack<P, NV>(a, (int)blockIdx.x * 31 + (lane - 1), (int)gridDim.x * 31);
    __syncwarp(kMask);
    if (lane == 1) {
        __threadfence_system();
        if (atomicAdd(a.pack_cnt, 1) == (int)gridDim.x - 1) {
            __threadfence_system();
#pragma unroll 1
            for (int b = 0; b < 8; b++) {
                if (!((a.wmask >> b) & 1)) continue;
                unsigned long long *fl = pd_flag(a.pd, b >> 1, b & 1);
                asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(fl), "l"((unsigned long long)kPutCtas)
                             : "memory");
            }
            atomicExch(a.pack_cnt, 0);   // the next fused launch packs only after this kernel completed
        }
    }
}

// Producer side: spin (acquire, system scope) until this exchange's halo has landed in this
// rank's window; on timeout raise the context's error word and go on (never hang).
__device__ __forceinline__ void wait_arrival(const ApplyArgs &a)
{
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll 1
    for (int b = 0; b < 8; b++) {
        if (!((a.wmask >> b) & 1)) continue;
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.wflag + b) : "memory");
            if (v >= a.wtarget) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > a.wtimeout) {
                atomicExch_system(a.werr, 1);
                break;
            }
            __nanosleep(32);
        }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy arrival -> TMA reads
}

// Face index of x in the block of dim mu (the other three coordinates, lowest fastest).
__device__ __forceinline__ int face_index(const KGeom &g, const int x[4], int mu)
{
    return mu == 0 ? (x[3] * g.L[2] + x[2]) * g.L[1] + x[1]
         : mu == 1 ? (x[3] * g.L[2] + x[2]) * g.L[0] + x[0]
         : mu == 2 ? (x[3] * g.L[1] + x[1]) * g.L[0] + x[0]
                   : (x[2] * g.L[1] + x[1]) * g.L[0] + x[0];
}

// ------------------------------------------------------------------ RING variant
// MPS = link matrices per ring stage.  A site's nine matrices are contiguous in HBM
// ([site][k], k = 0..8), so a stage holding MPS of them is ONE bulk copy (plus the MPS vector
// records they multiply): fewer, larger cp.async.bulk operations per byte (the ring was
// measured to be bound by the bulk-copy count, profiles/r01_summary.md).
template <cd_precision P, int NV, int MPS>
struct RingCfg {
    using Q = Cfg<P, NV>;
    // MPS = matrices per stage, + 100 for two CTAs per SM (MPS = 103)
    static constexpr int M = MPS % 100;                              // matrices per stage
    static constexpr int CPS = 1 + MPS / 100;                        // CTAs per SM
    static constexpr int NCW = Q::N / Q::R;                          // consumer warps
    static constexpr int THREADS = 32 * (NCW + 1);
    // vector records after the matrices, 128-B aligned; with nine per stage they sit in blocks of four
    // (each block 128-B aligned: the gather4 destinations) + one: record j at VOFF + vpos(j)
    static constexpr int VOFF = (M * Q::MREC + 127) / 128 * 128;
    static constexpr int VBLK = (4 * Q::VREC + 127) / 128 * 128;
    static constexpr int VAREA = M == 9 ? 2 * VBLK + Q::VREC : (M == 3 ? VBLK : M * Q::VREC);   // M = 3: + a spare slot
    static constexpr int STAGE = (VOFF + VAREA + 127) / 128 * 128;
    __host__ __device__ static constexpr int vpos(int j) { return M == 9 ? (j >> 2) * VBLK + (j & 3) * Q::VREC : j * Q::VREC; }
    static constexpr int HDR = 1024;                                // barriers + reduction scratch
    static constexpr int MAXS = 32;
    static constexpr int SMEM_BUDGET = CPS == 1 ? 227 * 1024 : 115712;   // latency bound: all of it (per CTA)
    static constexpr int S = ((SMEM_BUDGET - HDR) / STAGE) > MAXS ? MAXS : ((SMEM_BUDGET - HDR) / STAGE);
    static constexpr int SMEM = HDR + S * STAGE;
    static constexpr int SLOTS = 4;                                  // ticket-counter slots (launch % 4)
    static_assert(9 % M == 0, "M must divide 9");
    static_assert(CPS == 1 || MPS == 103, "two CTAs per SM: three matrices per stage");
};


// TMA gather4 (sm_100): four rows of a 2-D tensor map -- here four neighbours' vector records -- land
// back to back in shared memory from ONE instruction (the ring producer's per-copy issue cost is
// its critical path: nine vector copies per site become two gather4 + one bulk copy)
__device__ __forceinline__ void gather4_g2s(void *dst_smem, const CUtensorMap *tm, int r0, int r1, int r2, int r3,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

template <cd_precision P, int NV, int MPS>
__global__ void __launch_bounds__(RingCfg<P, NV, MPS>::THREADS, RingCfg<P, NV, MPS>::CPS) dslash_ring(ApplyArgs a, int slotx, const __grid_constant__ CUtensorMap tmv)
{
    // slotx = ticket slot | diagnostic bits << 8 (CD_RING_EXP, timing experiments only: 1 = no vector
    // copies, 2 = no consumer math (results wrong with either), 4 = static round-robin sites, 8 = IEEE
    // division in the fp16 re-quantisation) | gather4 << 16
    const int slot = slotx & 0xff, rexp = (slotx >> 8) & 0xff;
    const bool g4 = (slotx >> 16) & 1;   // tmv describes `in` as [V][VREC] bytes: gather4 the vector records
    using Q = Cfg<P, NV>;
    using RC = RingCfg<P, NV, MPS>;
    constexpr int M = RC::M;                                         // matrices per stage
    constexpr int S = RC::S;
    constexpr int G = 9 / M;                                       // stages per site
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + RC::MAXS;
    float *red = reinterpret_cast<float *>(smem + 16 * RC::MAXS);        // 2 x 32 floats
    int *siteq = reinterpret_cast<int *>(smem + 16 * RC::MAXS + 256);    // site id per stage
    unsigned char *stages = smem + RC::HDR;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    const unsigned char *in = static_cast<const unsigned char *>(a.in);
    unsigned char *out = static_cast<unsigned char *>(a.out);
    const int V = a.g.V;
    int *tickets = a.work + 2 * slot;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 32 * RC::NCW);   // every consumer thread releases (see below)
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_trigger();

    if (warp == RC::NCW && lane != 0) {
        // fused split apply: the other 31 lanes of the producer warp pack this CTA's slice of the
        // face records straight into the neighbours' windows, overlapped with the stencil
        if (a.fused) fused_pack_lanes<P, NV>(a, lane);
        return;
    }
    if (warp == RC::NCW) {
        // ===== producer: one elected lane takes sites from a global ticket counter (dynamic
        // load balance across SMs) and streams their records into the ring.  Ticket slot
        // `slot` (launch % 4) was reset by the last CTA of the launch 4 before this one, which
        // completed before this launch's predecessor did (stream order / griddepcontrol.wait).
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            // The first site of CTA b is site b (static); its link matrices do not depend on the
            // previous kernel, so their bulk copies go out BEFORE griddepcontrol.wait and overlap
            // that kernel's tail (PDL).  Its vector records (`in`, written by the previous
            // kernel) follow the wait.  Later sites come from the ticket counter (site =
            // gridDim.x + ticket).
            // fused split apply: tickets walk the sites rotated by a.rot, which for a T-only split puts
            // both T faces last (their remote records have long landed by then); otherwise a face
            // site met early just waits for the arrival (once per CTA).  Arithmetic on purpose: the
            // producer thread's per-site latency is the ring's critical path (an index-list load per
            // site measured +22 % at 16^3x32).
            auto order = [&](int t) -> int {
                const int u = t + a.rot;
                return u < V ? u : u - V;
            };
            // The first site's links are prefetched before griddepcontrol.wait (PDL); a fused apply
            // does so too unless that site is a face site (its remote records need the arrival wait)
            const int site0 = order((int)blockIdx.x);
            int x0[4];
            decode(a.g, site0 < V ? site0 : 0, x0);
            const bool pre = (G <= S) && (int)blockIdx.x < V && !(a.fused && is_face<P, NV>(a.g, x0));
            bool landed = false;
            if (pre) {
                const int site = site0;
                int x[4] = {x0[0], x0[1], x0[2], x0[3]};
                const unsigned char *lsite = links + (size_t)site * 9 * Q::MREC;
                for (int gi = 0; gi < G; gi++) {
                    int nvc = 0;
#pragma unroll
                    for (int j = 0; j < M; j++) nvc += !(a.halo && remote_hop(a.g, x, gi * M + j)) && !(rexp & 1);
                    unsigned char *st = stages + (size_t)gi * RC::STAGE;
                    mbar_arrive_expect_tx(&full[gi], M * Q::MREC + nvc * Q::VREC + (gi == 0 ? 4 : 0));
                    if (gi == 0) st_async_u32(&siteq[gi], (uint32_t)site, &full[gi]);
                    bulk_g2s(st, lsite + (size_t)gi * M * Q::MREC, M * Q::MREC, &full[gi]);
                }
                pdl_wait();   // `in` is written by the previous kernel in the stream
                for (int gi = 0; gi < G; gi++) {
                    unsigned char *st = stages + (size_t)gi * RC::STAGE;
#pragma unroll
                    for (int j = 0; j < M; j++) {
                        const int k = gi * M + j;
                        if ((a.halo && remote_hop(a.g, x, k)) || (rexp & 1)) continue;
                        bulk_g2s(st + RC::VOFF + RC::vpos(j), in + (size_t)neighbour(a.g, x, site, k) * Q::VREC,
                                 Q::VREC, &full[gi]);
                    }
                }
                stage = G % S;
                phase = (G == S) ? 1u : 0u;
            } else {
                pdl_wait();   // `in` is written by the previous kernel in the stream
            }
            // without the prefetch (a site needs more stages than the ring holds) the static
            // first site goes through the loop like any other
            bool first = !pre && (int)blockIdx.x < V;
            int nstatic = 0;
            for (;;) {
                // (rexp & 4, diagnostic: static round-robin sites instead of tickets)
                const int tk = first ? (int)blockIdx.x
                                     : ((rexp & 4) ? (int)blockIdx.x + (++nstatic) * (int)gridDim.x
                                                   : (int)gridDim.x + atomicAdd(tickets, 1));
                first = false;
                if (tk >= V) {   // sentinel stage: tells the consumers to stop
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], 4);
                    st_async_u32(&siteq[stage], 0xFFFFFFFFu, &full[stage]);
                    break;
                }
                const int site = order(tk);
                int x[4];
                decode(a.g, site, x);
                const unsigned char *lsite = links + (size_t)site * 9 * Q::MREC;
                constexpr int PREC = Q::F16 ? 4 * Q::N : 8 * Q::N;   // wire payload record
#pragma unroll
                // TMA gather4 of the vector records (nine or three per stage) for a site without remote hops;
                // with three per stage the fourth gathered row is a duplicate landing in the block's spare slot
                const bool gsite = (M == 9 || M == 3) && g4 && !(rexp & 1);
                for (int gi = 0; gi < G; gi++) {
                    // TMA gather4 of the vector records by blocks of four slots (M = 9: slots 0-3 and 4-7, slot 8
                    // by a bulk copy; M = 3: slots 0-2 with a duplicate fourth row into the spare slot) for every
                    // block without a remote hop; a face site's block holding its remote hop(s) keeps per-record copies
                    uint32_t rmask = 0;
#pragma unroll
                    for (int j = 0; j < M; j++)
                        if (a.halo && remote_hop(a.g, x, gi * M + j)) rmask |= 1u << j;
                    const bool gb0 = gsite && !(rmask & (M == 9 ? 0xFu : 0x7u));
                    const bool gb1 = gsite && M == 9 && !(rmask & 0xF0u);
                    uint32_t vbytes = (gb0 && M == 3) ? Q::VREC : 0;
#pragma unroll
                    for (int j = 0; j < M; j++) {
                        const bool rem = (rmask >> j) & 1;
                        vbytes += !rem ? ((rexp & 1) ? 0 : Q::VREC) : (a.fused ? PREC + (Q::F16 ? 16 : 0) : 0);
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char *st = stages + (size_t)stage * RC::STAGE;
                    // the site id travels like the data: an async store counted on the same barrier
                    mbar_arrive_expect_tx(&full[stage], M * Q::MREC + vbytes + (gi == 0 ? 4 : 0));
                    if (gi == 0) st_async_u32(&siteq[stage], (uint32_t)site, &full[stage]);
                    bulk_g2s(st, lsite + (size_t)gi * M * Q::MREC, M * Q::MREC, &full[stage]);
                    unsigned char *vd = st + RC::VOFF;
                    const int k0 = gi * M;
                    if (gb0) {
                        const int n2 = neighbour(a.g, x, site, k0 + 2);
                        gather4_g2s(vd, &tmv, neighbour(a.g, x, site, k0), neighbour(a.g, x, site, k0 + 1), n2,
                                    M == 9 ? neighbour(a.g, x, site, k0 + 3) : n2, &full[stage]);
                    }
                    if (gb1)
                        gather4_g2s(vd + RC::vpos(4), &tmv, neighbour(a.g, x, site, 4), neighbour(a.g, x, site, 5),
                                    neighbour(a.g, x, site, 6), neighbour(a.g, x, site, 7), &full[stage]);
#pragma unroll
                    for (int j = 0; j < M; j++) {
                        if ((gb0 && j < (M == 9 ? 4 : 3)) || (gb1 && j >= 4 && j < 8)) continue;   // gathered
                        const int k = gi * M + j;
                        if ((rmask >> j) & 1) {
                            if (!a.fused) continue;   // unfused: the halo-term kernel adds this hop
                            if (!landed) {
                                wait_arrival(a);
                                landed = true;
                            }
                            // a +mu hop reads block B (the +mu rank's x_mu = 0 face), a -mu hop block A
                            const int mu = k >> 1, blk = (k & 1) ? 0 : 1;
                            const int f = face_index(a.g, x, mu);
                            const unsigned char *rb = static_cast<const unsigned char *>(a.recv) + a.g.blk_off[mu][blk];
                            bulk_g2s(st + RC::VOFF + RC::vpos(j), rb + (size_t)f * PREC, PREC, &full[stage]);
                            // fp16: the 16-B aligned quad of wire scales holding this record's scale lands in
                            // the record's scale slot (+ its 12 pad bytes); the consumer picks 4 * (f & 3) --
                            // no dependent load on the producer thread (its latency is the ring's critical path)
                            if constexpr (Q::F16)
                                bulk_g2s(st + RC::VOFF + RC::vpos(j) + Q::VSCALE,
                                         rb + (size_t)sel4(a.g.F, mu) * PREC + (size_t)(f & ~3) * 4, 16, &full[stage]);
                            continue;
                        }
                        if (rexp & 1) continue;
                        bulk_g2s(st + RC::VOFF + RC::vpos(j), in + (size_t)neighbour(a.g, x, site, k) * Q::VREC,
                                 Q::VREC, &full[stage]);
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
            // the last CTA to finish resets this slot's tickets (for launch + 4)
            if (atomicAdd(tickets + 1, 1) == (int)gridDim.x - 1) {
                tickets[0] = 0;
                tickets[1] = 0;
                __threadfence();
            }
        }
        return;
    }

    // ===== consumers: warp w owns rows [w*R, w*R + R) of the current site, all nine hops
    pdl_wait();   // order our stores after the previous kernel (it may still read `out`)
    const int r = lane / Q::D, d = lane % Q::D;
    const int row = warp * Q::R + r;
    constexpr bool ROT = (Q::ROWB % 128 == 0) && (Q::D * 16 < 128);   // fp16 N=64: avoid 2-way bank conflict
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
        mbar_wait(&full[stage], phase);   // first stage of the next site
        const int site = *reinterpret_cast<volatile int *>(&siteq[stage]);
        if (site < 0) break;
        int x[4];
        decode(a.g, site, x);
        float re = 0.0f, im = 0.0f;
        // one hop: row `row` of matrix j of stage `st` times its vector record
        // fused split apply, fp16: a remote record's scale sits at 4 * (f & 3) in its scale slot
        int sofs[9];
#pragma unroll
        for (int k = 0; k < 9; k++) sofs[k] = 0;
        if constexpr (Q::F16) {
            if (a.fused && is_face<P, NV>(a.g, x)) {
#pragma unroll
                for (int k = 0; k < 8; k++)
                    if (remote_hop(a.g, x, k)) sofs[k] = 4 * (face_index(a.g, x, k >> 1) & 3);
            }
        }
        auto hop = [&](const unsigned char *st, int j, int so) {
            const unsigned char *mrec = st + j * Q::MREC;
            const unsigned char *mrow = mrec + row * Q::ROWB;
            const unsigned char *vrec = st + RC::VOFF + RC::vpos(j);
            if constexpr (P == CD_FP32) {
                float pr[Q::C], pi[Q::C];
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    pr[c] = 0.0f;
                    pi[c] = 0.0f;
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                    cmac2(lds128(mrow + q * 16), vq, pr[c], pi[c]);
                }
#pragma unroll
                for (int c = 0; c < Q::C; c++) { re += pr[c]; im += pi[c]; }
            } else {
                float ra = 0.f, rb = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int cc = ROT ? ((c + (r & 1)) % Q::C) : c;
                    const int q = d + Q::D * cc;
                    uint4 vq = lds128(vrec + q * 16);
                    if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                    hmac4(lds128(mrow + q * 16), vq, ra, rb, ia, ib);
                }
                const float sc = *reinterpret_cast<const float *>(mrec + Q::MSCALE) *
                                 *reinterpret_cast<const float *>(vrec + Q::VSCALE + so);
                re = fmaf(ra - rb, sc, re);
                im = fmaf(ia + ib, sc, im);
            }
        };
        // only face sites of a split dim have remote hops; every other site takes the
        // straight-line path even when the context is split (the interior kernel of run_split)
        const bool checked = a.halo && !a.fused && is_face<P, NV>(a.g, x);
#pragma unroll
        for (int gi = 0; gi < G; gi++) {
            if (gi > 0) mbar_wait(&full[stage], phase);
            const unsigned char *st = stages + (size_t)stage * RC::STAGE;
            if (rexp & 2) {
            } else if (!checked) {
                // straight-line stage (no per-hop branch): the compiler interleaves the M
                // independent hops' loads and FMA chains -- one CTA per SM leaves few consumer
                // warps, so this ILP is what keeps up with HBM at power-capped clocks (m9 fp16 at
                // 16^3x32: 1.69 -> 1.55 ms, profiles/r02/ring_ilp_ab.txt).  Waiting for a whole
                // site's stages before computing (more ILP for m1 / m3) measured slower for fp32.
#pragma unroll
                for (int j = 0; j < M; j++) hop(st, j, sofs[gi * M + j]);
            } else {
#pragma unroll
                for (int j = 0; j < M; j++)
                    if (!remote_hop(a.g, x, gi * M + j)) hop(st, j, 0);
            }
            // release the stage: every consumer thread arrives after its own reads returned (the
            // accumulators depend on every load) -- no reliance on __syncwarp ordering the other
            // lanes' reads before one elected arrive, so compute-sanitizer racecheck can verify
            // the reuse of a stage (round 2; the elected-lane form was flagged)
            asm volatile("" : "+f"(re), "+f"(im)::"memory");
            mbar_arrive(&empty[stage]);
            if (++stage == S) { stage = 0; phase ^= 1; }
        }
#pragma unroll
        for (int m = Q::D / 2; m >= 1; m >>= 1) {
            re += shfl_xor(re, m);
            im += shfl_xor(im, m);
        }
        const bool owner = (d == 0);
        if (checked) {
            if (owner) a.scratch[(size_t)site * Q::N + row] = make_float2(re, im);
        } else {
            const float sg = (a.dagger && row >= NV) ? -1.0f : 1.0f;
            // re-quantise with x * (1/s) (R12: <= 1 ulp fp32 before the fp16 rounding; M5 fp16
            // 1577 -> 1554 us against the IEEE division, which rexp & 8 restores for A/B runs)
            store_site<P, NV>(out, site, row, owner, sg * re, sg * im, red + 32 * (it & 1), 32 * RC::NCW, 1,
                              (rexp & 8) == 0);
        }
    }
}

// ------------------------------------------------------------------ RING variant, compressed links
// tau3-hermiticity-compressed links: a site stores X and its four forward links
// ([site][5]); the backward hop k = 2mu+1 of x uses L_{2mu+1}(x) = tau3 L_{2mu}(x - mu)^H tau3, i.e.
// the -mu neighbour's forward record read transposed.  The persistent TMA ring of dslash_ring with
// one bulk copy per matrix: HBM carries 5 matrices per site (the neighbours' forward records come
// back from L2: with tickets in site order they were streamed a few hundred sites earlier), the
// consumers read a backward matrix by columns.  Unsplit contexts (a split one uses dslash_fgh).
// compressed ring stage slot p -> hop: X (k = 8), the forward hops 0, 2, 4, 6 (records 0-4 of the site,
// contiguous), then the backward hops 1, 3, 5, 7
__host__ __device__ constexpr int kperm(int p) { return p == 0 ? 8 : (p < 5 ? 2 * (p - 1) : 2 * (p - 5) + 1); }

template <cd_precision P, int NV, int MPS>
__global__ void __launch_bounds__(RingCfg<P, NV, MPS>::THREADS, RingCfg<P, NV, MPS>::CPS) dslash_ringh(ApplyArgs a, int slotx, const __grid_constant__ CUtensorMap tmv)
{
    const int slot = slotx & 0xff;
    const bool g4 = (slotx >> 16) & 1;   // tmv describes `in` as [V][VREC]: gather4 the vector records
    using Q = Cfg<P, NV>;
    using RC = RingCfg<P, NV, MPS>;
    constexpr int MM = RC::M;   // matrices per stage
    constexpr int S = RC::S;
    static_assert(S >= 2, "ring needs at least two stages");
    constexpr int G = 9 / MM;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + RC::MAXS;
    float *red = reinterpret_cast<float *>(smem + 16 * RC::MAXS);
    int *siteq = reinterpret_cast<int *>(smem + 16 * RC::MAXS + 256);
    unsigned char *stages = smem + RC::HDR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned char *comp = static_cast<const unsigned char *>(a.links);
    const unsigned char *in = static_cast<const unsigned char *>(a.in);
    unsigned char *out = static_cast<unsigned char *>(a.out);
    const int V = a.g.V;
    int *tickets = a.work + 2 * slot;
    if (threadIdx.x == 0) {
        for (int st = 0; st < S; st++) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 32 * RC::NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_trigger();
    if (warp == RC::NCW) {
        if (lane == 0) {
            pdl_wait();
            int stage = 0;
            uint32_t phase = 0;
            bool first = (int)blockIdx.x < V;
            for (;;) {
                const int site = first ? (int)blockIdx.x : (int)gridDim.x + atomicAdd(tickets, 1);
                first = false;
                if (site >= V) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], 4);
                    st_async_u32(&siteq[stage], 0xFFFFFFFFu, &full[stage]);
                    break;
                }
                int x[4];
                decode(a.g, site, x);
#pragma unroll
                for (int gi = 0; gi < G; gi++) {
                    // stage slots p = gi * MM + j hold hop kperm(p): the site's own five records (X and the
                    // forward hops, contiguous in `comp`) first -- ONE copy per stage for that run -- then the
                    // backward hops (record 1 + mu of x - mu); vectors by gather4 (MM = 9: two + one bulk
                    // copy; MM = 3: one, its fourth row a duplicate into the spare slot)
                    const int p0 = gi * MM;
                    const int nown = p0 < 5 ? (MM < 5 - p0 ? MM : 5 - p0) : 0;
                    const int nvrec = g4 ? (MM == 3 ? 4 : MM) : MM;
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char *st = stages + (size_t)stage * RC::STAGE;
                    mbar_arrive_expect_tx(&full[stage], MM * Q::MREC + nvrec * Q::VREC + (gi == 0 ? 4 : 0));
                    if (gi == 0) st_async_u32(&siteq[stage], (uint32_t)site, &full[stage]);
                    if (nown > 0)
                        bulk_g2s(st, comp + ((size_t)site * 5 + p0) * Q::MREC, nown * Q::MREC, &full[stage]);
                    int n[MM];
#pragma unroll
                    for (int j = 0; j < MM; j++) n[j] = neighbour(a.g, x, site, kperm(p0 + j));
#pragma unroll
                    for (int j = 0; j < MM; j++) {
                        if (j < nown) continue;
                        const int mu = p0 + j - 5;   // backward hop 2mu+1: record 1 + mu of x - mu
                        bulk_g2s(st + j * Q::MREC, comp + ((size_t)n[j] * 5 + 1 + mu) * Q::MREC, Q::MREC, &full[stage]);
                    }
                    unsigned char *vd = st + RC::VOFF;
                    if (g4) {
                        if constexpr (MM == 9) {
                            gather4_g2s(vd, &tmv, n[0], n[1], n[2], n[3], &full[stage]);
                            gather4_g2s(vd + RC::vpos(4), &tmv, n[4], n[5], n[6], n[7], &full[stage]);
                            bulk_g2s(vd + RC::vpos(8), in + (size_t)n[8] * Q::VREC, Q::VREC, &full[stage]);
                        } else {
                            gather4_g2s(vd, &tmv, n[0], n[1], n[2], n[2], &full[stage]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < MM; j++)
                            bulk_g2s(vd + RC::vpos(j), in + (size_t)n[j] * Q::VREC, Q::VREC, &full[stage]);
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
            if (atomicAdd(tickets + 1, 1) == (int)gridDim.x - 1) {
                tickets[0] = 0;
                tickets[1] = 0;
                __threadfence();
            }
        }
        return;
    }
    pdl_wait();
    const int r = lane / Q::D, d = lane % Q::D;
    const int row = warp * Q::R + r;
    const float srow = row >= NV ? -1.0f : 1.0f;   // s_i of the backward hops
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
        mbar_wait(&full[stage], phase);
        const int site = *reinterpret_cast<volatile int *>(&siteq[stage]);
        if (site < 0) break;
        float re = 0.0f, im = 0.0f;
#pragma unroll
        for (int gi = 0; gi < G; gi++) {
            if (gi > 0) mbar_wait(&full[stage], phase);
            const unsigned char *st = stages + (size_t)stage * RC::STAGE;
#pragma unroll
            for (int j = 0; j < MM; j++) {
                const int k = kperm(gi * MM + j);
                const bool bwd = (k != 8) && (k & 1);
                const unsigned char *mrec = st + j * Q::MREC;
                const unsigned char *vrec = st + RC::VOFF + RC::vpos(j);
                if constexpr (P == CD_FP32) {
                    float hr = 0.0f, hi = 0.0f;
#pragma unroll
                    for (int c = 0; c < Q::C; c++) {
                        const int q = d + Q::D * c;
                        uint4 vq = lds128(vrec + q * 16);
                        if (!bwd) {
                            if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                            cmac2(lds128(mrec + row * Q::ROWB + q * 16), vq, hr, hi);
                        } else {
                            // s_j tau3-hermiticity sign, times the dagger's tau3: flip iff j >= NV && !dagger
                            if (!a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                            const float *vf = reinterpret_cast<const float *>(&vq);
#pragma unroll
                            for (int t = 0; t < Q::CPC; t++) {   // conj(M[j][row]) v_j
                                const int jj = q * Q::CPC + t;
                                const float2 m = *reinterpret_cast<const float2 *>(mrec + jj * Q::ROWB + row * 8);
                                hr = fmaf(m.x, vf[2 * t], hr);
                                hr = fmaf(m.y, vf[2 * t + 1], hr);
                                hi = fmaf(m.x, vf[2 * t + 1], hi);
                                hi = fmaf(-m.y, vf[2 * t], hi);
                            }
                        }
                    }
                    if (bwd) {
                        hr *= srow;
                        hi *= srow;
                    }
                    re += hr;
                    im += hi;
                } else {
                    float ra = 0.f, rb = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
                    for (int c = 0; c < Q::C; c++) {
                        const int q = d + Q::D * c;
                        uint4 vq = lds128(vrec + q * 16);
                        if (!bwd) {
                            if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                            hmac4(lds128(mrec + row * Q::ROWB + q * 16), vq, ra, rb, ia, ib);
                        } else {
                            if (!a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                            const uint32_t *vw = &vq.x;
#pragma unroll
                            for (int t = 0; t < Q::CPC; t++) {
                                const int jj = q * Q::CPC + t;
                                hmac1(*reinterpret_cast<const uint32_t *>(mrec + jj * Q::ROWB + row * 4), vw[t], ra, rb,
                                      ia, ib);
                            }
                        }
                    }
                    const float sc = *reinterpret_cast<const float *>(mrec + Q::MSCALE) *
                                     *reinterpret_cast<const float *>(vrec + Q::VSCALE) * (bwd ? srow : 1.0f);
                    // forward: (ra - rb, ia + ib); backward (conjugated matrix): (ra + rb, ia - ib)
                    re = fmaf(bwd ? ra + rb : ra - rb, sc, re);
                    im = fmaf(bwd ? ia - ib : ia + ib, sc, im);
                }
            }
            // the stage's shared-memory reads must have returned before it is released: pin the
            // accumulators (which depend on every load) ahead of the arrive
            asm volatile("" : "+f"(re), "+f"(im)::"memory");
            mbar_arrive(&empty[stage]);   // every consumer thread (see dslash_ring)
            if (++stage == S) { stage = 0; phase ^= 1; }
        }
#pragma unroll
        for (int m = Q::D / 2; m >= 1; m >>= 1) {
            re += shfl_xor(re, m);
            im += shfl_xor(im, m);
        }
        const bool owner = (d == 0);
        const float sg = (a.dagger && row >= NV) ? -1.0f : 1.0f;
        store_site<P, NV>(out, site, row, owner, sg * re, sg * im, red + 32 * (it & 1), 32 * RC::NCW, 1,
                          true);   // x * (1/s) as dslash_ring (R12)
    }
}

// ------------------------------------------------------------------ FG variant
template <cd_precision P, int NV, int KW, int WR>
struct FgCfg {
    using Q = Cfg<P, NV>;
    static constexpr int WK = 9 / KW;
    static constexpr int NW = WK * WR;
    static constexpr int THREADS = 32 * NW;
    static constexpr int ROWS = WR * Q::R;
    static constexpr int NRB = Q::N / ROWS;
    static_assert(WK * KW == 9, "KW must divide 9");
    static_assert(NRB * ROWS == Q::N, "row blocks must tile N");
    static_assert(NW <= 32, "too many warps");
    // fp16 output with the site split over NRB CTAs: the last CTA to finish quantises it
    static constexpr bool SPLIT16 = (P == CD_FP16) && NRB > 1;
    static_assert(!SPLIT16 || THREADS >= Q::N, "the finishing CTA needs a thread per row");
};

template <cd_precision P, int NV, int KW, int WR>
__global__ void __launch_bounds__(FgCfg<P, NV, KW, WR>::THREADS) dslash_fg(ApplyArgs a)
{
    using Q = Cfg<P, NV>;
    using F = FgCfg<P, NV, KW, WR>;
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];
    __shared__ float2 part[F::WK][F::ROWS];
    __shared__ float red[32];

    const int site = blockIdx.x / F::NRB, rb = blockIdx.x - site * F::NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wk = warp / WR, wr = warp - wk * WR;
    const int r = lane / Q::D, d = lane % Q::D;
    const int rowl = wr * Q::R + r, row = rb * F::ROWS + rowl;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    const unsigned char *in = static_cast<const unsigned char *>(a.in);
    unsigned char *out = static_cast<unsigned char *>(a.out);

    int x[4];
    decode(a.g, site, x);

    // 1. link rows: input independent -> issued before the PDL wait
    uint4 Lc[KW][Q::C];
    float sl[KW];
    bool on[KW];
#pragma unroll
    for (int kk = 0; kk < KW; kk++) {
        const int k = kseq(wk * KW + kk);
        on[kk] = !(a.halo && remote_hop(a.g, x, k));
        const unsigned char *m = links + ((size_t)site * 9 + k) * Q::MREC;
#pragma unroll
        for (int c = 0; c < Q::C; c++)
            Lc[kk][c] = on[kk] ? ld_stream(m + row * Q::ROWB + (d + Q::D * c) * 16) : make_uint4(0, 0, 0, 0);
        sl[kk] = (Q::F16 && on[kk]) ? ld_nc_f32(m + Q::MSCALE) : 0.0f;
    }
    // the latency regime (a grid of at most a few CTAs per SM): each lane loads the neighbour
    // chunks it needs straight into registers -- no staging round trip through shared memory
    // and no barrier between the vectors' arrival and the math (the floor of a dependent launch
    // is ~0.82 us; this is on the path after griddepcontrol.wait, profiles/r02/launch_floor.txt)
    // Measured (profiles/r02/fg_direct_ab.txt): 2^4 fp32 kw1_wr2 2.03 -> 1.62 us, fp16 kw1_wr1
    // 4.84 -> 3.79 us; at 4^4 (>= 512 CTAs) the staged path is faster (6.80 vs 7.31 us), so the
    // direct path is gated to grids of at most two CTAs per SM.
    constexpr bool kDirect = KW == 1;   // registers: KW x C chunks more (kw3 would lose occupancy, kw9 spill)
    constexpr int KD = kDirect ? KW : 1;
    const bool direct = kDirect && a.g.V * F::NRB <= 2 * 148;
    const unsigned char *nbrec[KD];
#pragma unroll
    for (int kk = 0; kk < KD; kk++) {
        const int k = kseq(wk * KW + kk);
        nbrec[kk] = in + (size_t)neighbour(a.g, x, site, k) * Q::VREC;
    }
    pdl_trigger();
    pdl_wait();

    uint4 Vd[KD][Q::C];
    float svd[KD];
    if (direct) {
#pragma unroll
        for (int kk = 0; kk < KD; kk++) {
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                Vd[kk][c] = on[kk] ? ld_nc(nbrec[kk] + (d + Q::D * c) * 16) : make_uint4(0, 0, 0, 0);
            svd[kk] = (Q::F16 && on[kk]) ? ld_nc_f32(nbrec[kk] + Q::VSCALE) : 0.0f;
        }
    } else {
        // 2. the nine neighbour records -> shared memory (one 16-B chunk per thread-step)
        for (int t = threadIdx.x; t < 9 * Q::VCH; t += F::THREADS) {
            const int k = t / Q::VCH, e = t - k * Q::VCH;
            if (a.halo && remote_hop(a.g, x, k)) continue;
            const int nb = neighbour(a.g, x, site, k);
            *reinterpret_cast<uint4 *>(vs + k * Q::VREC + e * 16) = ld_nc(in + (size_t)nb * Q::VREC + e * 16);
        }
        __syncthreads();
    }

    // 3. dot products (ILP: one accumulator pair per chunk, Listing 5)
    float re = 0.0f, im = 0.0f;
#pragma unroll
    for (int kk = 0; kk < KW; kk++) {
        if (!on[kk]) continue;
        const int k = kseq(wk * KW + kk);
        const unsigned char *vrec = vs + k * Q::VREC;
        if constexpr (P == CD_FP32) {
            float pr[Q::C], pi[Q::C];
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                pr[c] = 0.0f;
                pi[c] = 0.0f;
                const int q = d + Q::D * c;
                uint4 vq = direct ? Vd[kDirect ? kk : 0][c] : lds128(vrec + q * 16);
                if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                cmac2(Lc[kk][c], vq, pr[c], pi[c]);
            }
#pragma unroll
            for (int c = 0; c < Q::C; c++) { re += pr[c]; im += pi[c]; }
        } else {
            float ra = 0.f, rb2 = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                const int q = d + Q::D * c;
                uint4 vq = direct ? Vd[kDirect ? kk : 0][c] : lds128(vrec + q * 16);
                if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                hmac4(Lc[kk][c], vq, ra, rb2, ia, ib);
            }
            const float sc = sl[kk] * (direct ? svd[kDirect ? kk : 0] : *reinterpret_cast<const float *>(vrec + Q::VSCALE));
            re = fmaf(ra - rb2, sc, re);
            im = fmaf(ia + ib, sc, im);
        }
    }
    // 4. dot-product split: xor-shuffle over the D lanes of a row
#pragma unroll
    for (int m = Q::D / 2; m >= 1; m >>= 1) {
        re += shfl_xor(re, m);
        im += shfl_xor(im, m);
    }
    // 5. direction split: hop-group partials through shared memory, one owner per row
    if (d == 0) part[wk][rowl] = make_float2(re, im);
    __syncthreads();
    const int t = threadIdx.x;
    const bool owner = t < F::ROWS;
    float yr = 0.0f, yi = 0.0f;
    if (owner) {
#pragma unroll
        for (int w = 0; w < F::WK; w++) {
            yr += part[w][t].x;
            yi += part[w][t].y;
        }
    }
    const int orow = rb * F::ROWS + (owner ? t : 0);
    if (a.halo && is_face<P, NV>(a.g, x)) {
        if (owner) a.scratch[(size_t)site * Q::N + orow] = make_float2(yr, yi);
        return;
    }
    const float sg = (a.dagger && orow >= NV) ? -1.0f : 1.0f;
    if constexpr (F::SPLIT16) {
        // fp16 storage needs the whole site's max |y| (R12): every row block parks its
        // fp32 rows in an L2-resident scratch; the last CTA of the site (per-site arrival
        // counter, reset by that CTA) quantises all N rows.  No atomics on data, deterministic.
        __shared__ int last;
        if (owner) a.ysplit[(size_t)site * Q::N + orow] = make_float2(sg * yr, sg * yi);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = (atomicAdd(&a.site_cnt[site], 1) == F::NRB - 1);
        __syncthreads();
        if (!last) return;
        __threadfence();
        const bool own = threadIdx.x < Q::N;
        const float2 v = own ? __ldcg(&a.ysplit[(size_t)site * Q::N + threadIdx.x]) : make_float2(0.f, 0.f);
        if (threadIdx.x == 0) a.site_cnt[site] = 0;
        store_site<P, NV>(out, site, own ? threadIdx.x : 0, own, v.x, v.y, red, F::THREADS, -1);
    } else {
        store_site<P, NV>(out, site, orow, owner, sg * yr, sg * yi, red, F::THREADS, -1);
    }
}

// ------------------------------------------------------------------ compressed (tau3-hermitian) links
// for tau3-hermitian operators L_{2mu+1}(x) = tau3 L_{2mu}(x-mu)^H tau3 (PAPER.md:121
// fn. 1), so only X and the four forward links are stored: record c of a site is
// c = 0: X, c = 1 + mu: L_{2mu}.  The backward hop of x reads the forward link of x - mu
// TRANSPOSED:  w_i = s_i sum_j conj(M_ji) s_j u_j  (s = tau3 signs, M = L_{2mu}(x-mu), u = v(x-mu)),
// with lanes = (4 output rows i) x (8 groups of input rows j): each warp load is 8 rows x a
// 32-byte strip of M (sector-exact), reduced over j with xor-shuffles.  CTA = (site, 4 rows),
// one warp per hop (the fg kw1/wr1 decomposition).  fp32 storage.
template <int NV>
__global__ void __launch_bounds__(288, NV == 24 ? 3 : 2) dslash_fgh(ApplyArgs a)
{
    using Q = Cfg<CD_FP32, NV>;
    constexpr int ROWS = 16;                 // output rows per CTA
    constexpr int NRB = Q::N / ROWS;
    constexpr int RG = ROWS / Q::R;          // forward: row groups of R = 4 rows per warp
    constexpr int TJ = Q::N / 2;             // backward: input rows j per lane (2 j-groups)
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];
    __shared__ float2 part[9][ROWS];
    const int site = blockIdx.x / NRB, rb = blockIdx.x - site * NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = kseq(warp);   // X, then 0..7
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    const unsigned char *in = static_cast<const unsigned char *>(a.in);
    int x[4];
    decode(a.g, site, x);
    const bool fwd = (k == 8) || !(k & 1);
    const bool remote = a.halo && remote_hop(a.g, x, k);   // added by dslash_fgh_halo
    // forward / X hop: own record; backward hop: forward record of the -mu neighbour
    const int msite = fwd ? site : neighbour(a.g, x, site, k);
    const int crec = (k == 8) ? 0 : 1 + (k >> 1);
    const unsigned char *m = links + ((size_t)msite * 5 + crec) * Q::MREC;
    const int r = lane / Q::D, d = lane % Q::D;           // forward mapping: (row, dot chunk)
    const int il = lane & 15, gj = lane >> 4;             // backward mapping: (row i, j group)
    uint4 Lc[RG][Q::C];
    uint2 Mc[TJ];
    if (remote) {
    } else if (fwd) {
#pragma unroll
        for (int g = 0; g < RG; g++)
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                Lc[g][c] = ld_stream(m + (rb * ROWS + g * Q::R + r) * Q::ROWB + (d + Q::D * c) * 16);
    } else {
#pragma unroll
        for (int t = 0; t < TJ; t++) {   // rows j = gj + 2t: 2 x 128-byte column strips per instruction
            const uint2 *p = reinterpret_cast<const uint2 *>(m + (size_t)(gj + 2 * t) * Q::ROWB + (rb * ROWS + il) * 8);
            asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(Mc[t].x), "=r"(Mc[t].y) : "l"(p));
        }
    }
    pdl_trigger();
    pdl_wait();
    for (int t = threadIdx.x; t < 9 * Q::VCH; t += 288) {
        const int kk = t / Q::VCH, e = t - kk * Q::VCH;
        if (a.halo && remote_hop(a.g, x, kk)) continue;
        const int nb = neighbour(a.g, x, site, kk);
        *reinterpret_cast<uint4 *>(vs + kk * Q::VREC + e * 16) = ld_nc(in + (size_t)nb * Q::VREC + e * 16);
    }
    __syncthreads();
    const float2 *vk = reinterpret_cast<const float2 *>(vs + k * Q::VREC);
    if (remote) {
        if (lane < ROWS) part[warp][lane] = make_float2(0.0f, 0.0f);
    } else if (fwd) {
#pragma unroll
        for (int g = 0; g < RG; g++) {
            float re = 0.0f, im = 0.0f;
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                const int q = d + Q::D * c;
                uint4 vq = lds128(reinterpret_cast<const unsigned char *>(vk) + q * 16);
                if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                cmac2(Lc[g][c], vq, re, im);
            }
#pragma unroll
            for (int o = Q::D / 2; o >= 1; o >>= 1) {
                re += shfl_xor(re, o);
                im += shfl_xor(im, o);
            }
            if (d == 0) part[warp][g * Q::R + r] = make_float2(re, im);
        }
    } else {
        float re = 0.0f, im = 0.0f;
#pragma unroll
        for (int t = 0; t < TJ; t++) {
            const int j = gj + 2 * t;
            float2 u = vk[j];
            // s_j of the tau3 structure, times the dagger's tau3 on the input
            const bool neg = (j >= NV) != (a.dagger && j >= NV);
            if (neg) u = make_float2(-u.x, -u.y);
            const float ma = __uint_as_float(Mc[t].x), mb = __uint_as_float(Mc[t].y);
            re = fmaf(ma, u.x, fmaf(mb, u.y, re));    // conj(M) u: (ma - i mb)(ux + i uy)
            im = fmaf(ma, u.y, fmaf(-mb, u.x, im));
        }
        re += shfl_xor(re, 16);
        im += shfl_xor(im, 16);
        const int i = rb * ROWS + il;
        const float si = (i >= NV) ? -1.0f : 1.0f;   // s_i of the tau3 structure
        if (gj == 0) part[warp][il] = make_float2(si * re, si * im);
    }
    __syncthreads();
    if (threadIdx.x < ROWS) {
        float yr = 0.0f, yi = 0.0f;
#pragma unroll
        for (int w = 0; w < 9; w++) {
            yr += part[w][threadIdx.x].x;
            yi += part[w][threadIdx.x].y;
        }
        const int row = rb * ROWS + threadIdx.x;
        if (a.halo && is_face<CD_FP32, NV>(a.g, x)) {   // partial for dslash_fgh_halo (no output sign yet)
            a.scratch[(size_t)site * Q::N + row] = make_float2(yr, yi);
            return;
        }
        const float sg = (a.dagger && row >= NV) ? -1.0f : 1.0f;
        reinterpret_cast<float2 *>(static_cast<unsigned char *>(a.out) + (size_t)site * Q::VREC)[row] =
            make_float2(sg * yr, sg * yi);
    }
}

// fp16 storage: the same decomposition with half2 payloads (FHFMA, one scale product per hop) and
// the whole-site re-quantisation of the fp16 row-split fg variants (fp32 rows parked in an
// L2-resident scratch, the last of the site's CTAs quantises).
template <int NV>
__global__ void __launch_bounds__(288, 3) dslash_fgh16(ApplyArgs a)
{
    using Q = Cfg<CD_FP16, NV>;
    constexpr int ROWS = 16;
    constexpr int NRB = Q::N / ROWS;
    constexpr int RG = ROWS / Q::R;
    constexpr int TJ = Q::N / 8;             // backward: input rows j per lane (8 j-groups), 16 B each
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];
    __shared__ float2 part[9][ROWS];
    __shared__ float red[32];
    __shared__ int last;
    const int site = blockIdx.x / NRB, rb = blockIdx.x - site * NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = kseq(warp);
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    const unsigned char *in = static_cast<const unsigned char *>(a.in);
    int x[4];
    decode(a.g, site, x);
    const bool fwd = (k == 8) || !(k & 1);
    const bool remote = a.halo && remote_hop(a.g, x, k);   // added by dslash_fgh_halo
    const int msite = fwd ? site : neighbour(a.g, x, site, k);
    const int crec = (k == 8) ? 0 : 1 + (k >> 1);
    const unsigned char *m = links + ((size_t)msite * 5 + crec) * Q::MREC;
    const int r = lane / Q::D, d = lane % Q::D;
    const int ic = lane & 3, gj = lane >> 2;   // backward: (4 columns i, j group)
    uint4 Lc[RG][Q::C];
    uint4 Mc[TJ];
    if (remote) {
    } else if (fwd) {
#pragma unroll
        for (int g = 0; g < RG; g++)
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                Lc[g][c] = ld_stream(m + (rb * ROWS + g * Q::R + r) * Q::ROWB + (d + Q::D * c) * 16);
    } else {
#pragma unroll
        for (int t = 0; t < TJ; t++)   // rows j = gj + 8t: 8 x 64-byte column strips per instruction
            Mc[t] = ld_stream(m + (size_t)(gj + 8 * t) * Q::ROWB + (rb * ROWS + 4 * ic) * 4);
    }
    const float msc = remote ? 0.0f : ld_nc_f32(m + Q::MSCALE);
    pdl_trigger();
    pdl_wait();
    for (int t = threadIdx.x; t < 9 * Q::VCH; t += 288) {
        const int kk = t / Q::VCH, e = t - kk * Q::VCH;
        if (a.halo && remote_hop(a.g, x, kk)) continue;
        const int nb = neighbour(a.g, x, site, kk);
        *reinterpret_cast<uint4 *>(vs + kk * Q::VREC + e * 16) = ld_nc(in + (size_t)nb * Q::VREC + e * 16);
    }
    __syncthreads();
    const unsigned char *vrec = vs + k * Q::VREC;
    const float sc = remote ? 0.0f : msc * *reinterpret_cast<const float *>(vrec + Q::VSCALE);
    if (remote) {
        if (lane < ROWS) part[warp][lane] = make_float2(0.0f, 0.0f);
    } else if (fwd) {
#pragma unroll
        for (int g = 0; g < RG; g++) {
            float ra = 0.f, rb2 = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                const int q = d + Q::D * c;
                uint4 vq = lds128(vrec + q * 16);
                if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                hmac4(Lc[g][c], vq, ra, rb2, ia, ib);
            }
            float re = (ra - rb2) * sc, im = (ia + ib) * sc;
#pragma unroll
            for (int o = Q::D / 2; o >= 1; o >>= 1) {
                re += shfl_xor(re, o);
                im += shfl_xor(im, o);
            }
            if (d == 0) part[warp][g * Q::R + r] = make_float2(re, im);
        }
    } else {
        float ra[4] = {0.f, 0.f, 0.f, 0.f}, rb2[4] = {0.f, 0.f, 0.f, 0.f};
        float ia[4] = {0.f, 0.f, 0.f, 0.f}, ib[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t *u32 = reinterpret_cast<const uint32_t *>(vrec);
#pragma unroll
        for (int t = 0; t < TJ; t++) {
            const int j = gj + 8 * t;
            uint32_t u = u32[j];
            if ((j >= NV) != (a.dagger && j >= NV)) u ^= 0x80008000u;   // s_j, times the dagger's tau3
            const uint32_t *mw = &Mc[t].x;                           // M[j][i .. i+3]
#pragma unroll
            for (int q = 0; q < 4; q++) hmac1(mw[q], u, ra[q], rb2[q], ia[q], ib[q]);   // conj(M) u
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            float re = (ra[q] + rb2[q]) * sc, im = (ia[q] - ib[q]) * sc;
#pragma unroll
            for (int o = 4; o <= 16; o <<= 1) {
                re += shfl_xor(re, o);
                im += shfl_xor(im, o);
            }
            const int il = 4 * ic + q;
            const float si = (rb * ROWS + il >= NV) ? -1.0f : 1.0f;
            if (gj == 0) part[warp][il] = make_float2(si * re, si * im);
        }
    }
    __syncthreads();
    if (threadIdx.x < ROWS) {
        float yr = 0.0f, yi = 0.0f;
#pragma unroll
        for (int w = 0; w < 9; w++) {
            yr += part[w][threadIdx.x].x;
            yi += part[w][threadIdx.x].y;
        }
        const int row = rb * ROWS + threadIdx.x;
        const float sg = (a.dagger && row >= NV) ? -1.0f : 1.0f;
        if (a.halo && is_face<CD_FP16, NV>(a.g, x)) a.scratch[(size_t)site * Q::N + row] = make_float2(yr, yi);
        else a.ysplit[(size_t)site * Q::N + row] = make_float2(sg * yr, sg * yi);
    }
    if (a.halo && is_face<CD_FP16, NV>(a.g, x)) return;   // dslash_fgh_halo finishes (and quantises) it
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(&a.site_cnt[site], 1) == NRB - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    const bool own = threadIdx.x < Q::N;
    const float2 v = own ? __ldcg(&a.ysplit[(size_t)site * Q::N + threadIdx.x]) : make_float2(0.f, 0.f);
    if (threadIdx.x == 0) a.site_cnt[site] = 0;
    store_site<CD_FP16, NV>(static_cast<unsigned char *>(a.out), site, own ? threadIdx.x : 0, own, v.x, v.y, red, 288, -1);
}

// hermiticity deviation of fp16 links, on the dequantised values (payload x record scale)
template <int NV>
__global__ void links_herm_dev16_kernel(const unsigned char *full, KGeom g, float *dev, const unsigned char *lhalo,
                                   int64_t o0, int64_t o1, int64_t o2, int64_t o3)
{
    using Q = Cfg<CD_FP16, NV>;
    const int site = blockIdx.x >> 2, mu = blockIdx.x & 3;
    int x[4];
    decode(g, site, x);
    const int nb = neighbour(g, x, site, 2 * mu + 1);
    const unsigned char *Br = full + ((size_t)site * 9 + 2 * mu + 1) * Q::MREC;
    const unsigned char *frec = full + ((size_t)nb * 9 + 2 * mu) * Q::MREC;
    if (lhalo != nullptr && ((g.split >> mu) & 1) && x[mu] == 0) {   // the -mu neighbour is remote: link halo
        const int f = mu == 0 ? (x[3] * g.L[2] + x[2]) * g.L[1] + x[1]
                    : mu == 1 ? (x[3] * g.L[2] + x[2]) * g.L[0] + x[0]
                    : mu == 2 ? (x[3] * g.L[1] + x[1]) * g.L[0] + x[0]
                              : (x[2] * g.L[1] + x[1]) * g.L[0] + x[0];
        frec = lhalo + (mu == 0 ? o0 : mu == 1 ? o1 : mu == 2 ? o2 : o3) + (size_t)f * Q::MREC;
    }
    const unsigned char *Fr = frec;
    const __half2 *B = reinterpret_cast<const __half2 *>(Br);
    const __half2 *F = reinterpret_cast<const __half2 *>(Fr);
    const float sb = *reinterpret_cast<const float *>(Br + Q::MSCALE), sf = *reinterpret_cast<const float *>(Fr + Q::MSCALE);
    float mx = 0.0f;
    for (int e = threadIdx.x; e < Q::N * Q::N; e += blockDim.x) {
        const int i = e / Q::N, j = e - i * Q::N;
        const float s = ((i < NV) == (j < NV)) ? 1.0f : -1.0f;
        const float2 f = __half22float2(F[j * Q::N + i]);
        const float2 b = __half22float2(B[e]);
        // rounded products (no contraction): equal scales and mirrored payloads give exactly 0
        const float bx = __fmul_rn(b.x, sb), by = __fmul_rn(b.y, sb);
        const float fx = __fmul_rn(s * f.x, sf), fy = __fmul_rn(s * f.y, sf);
        mx = fmaxf(mx, fmaxf(fabsf(bx - fx), fabsf(by + fy)));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, shfl_xor(mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int *>(dev), __float_as_int(mx));
}

// Multi-rank compressed operator: one CTA per face site adds the remote hops to the partial of the
// interior kernel.  Forward remote hop (x_mu = L-1): own compressed record x the vector from
// receive block B; backward remote hop (x_mu = 0): the -mu neighbour's forward record from the
// one-time link halo (transposed, tau3) x the vector from receive block A.  Then the final store
// (fp16: whole-site quantisation).
template <cd_precision P, int NV>
__global__ void __launch_bounds__(32 * (2 * NV / Cfg<P, NV>::R)) dslash_fgh_halo(ApplyArgs a)
{
    using Q = Cfg<P, NV>;
    constexpr int NWARP = Q::N / Q::R;
    constexpr int PREC = Q::F16 ? 4 * Q::N : 8 * Q::N;   // vector wire payload record
    __shared__ float red[32];
    const int site = a.face_sites[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = lane / Q::D, d = lane % Q::D;
    const int row = warp * Q::R + r;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    const unsigned char *recv = static_cast<const unsigned char *>(a.recv);
    const unsigned char *lh = static_cast<const unsigned char *>(a.lhalo);
    int x[4];
    decode(a.g, site, x);
    float re = 0.0f, im = 0.0f;
    for (int k = 0; k < 8; k++) {
        if (!remote_hop(a.g, x, k)) continue;
        const int mu = k >> 1;
        const int blk = (k & 1) ? 0 : 1;
        const int f = mu == 0 ? (x[3] * a.g.L[2] + x[2]) * a.g.L[1] + x[1]
                    : mu == 1 ? (x[3] * a.g.L[2] + x[2]) * a.g.L[0] + x[0]
                    : mu == 2 ? (x[3] * a.g.L[1] + x[1]) * a.g.L[0] + x[0]
                              : (x[2] * a.g.L[1] + x[1]) * a.g.L[0] + x[0];
        const unsigned char *vrec = recv + a.g.blk_off[mu][blk] + (size_t)f * PREC;
        float vsc = 1.0f;
        if constexpr (Q::F16)
            vsc = *reinterpret_cast<const float *>(recv + a.g.blk_off[mu][blk] + (size_t)a.g.F[mu] * PREC + (size_t)f * 4);
        if (!(k & 1)) {   // forward: rows of the own record 1 + mu
            const unsigned char *m = links + ((size_t)site * 5 + 1 + mu) * Q::MREC;
            if constexpr (P == CD_FP32) {
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int q = d + Q::D * c;
                    uint4 vq = ld_nc(vrec + q * 16);
                    if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                    cmac2(ld_nc(m + row * Q::ROWB + q * 16), vq, re, im);
                }
            } else {
                float ra = 0.f, rb = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int q = d + Q::D * c;
                    uint4 vq = ld_nc(vrec + q * 16);
                    if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                    hmac4(ld_nc(m + row * Q::ROWB + q * 16), vq, ra, rb, ia, ib);
                }
                const float sc = ld_nc_f32(m + Q::MSCALE) * vsc;
                re = fmaf(ra - rb, sc, re);
                im = fmaf(ia + ib, sc, im);
            }
        } else {          // backward: column `row` of the neighbour's forward record, tau3 on both sides
            const unsigned char *m = lh + a.lhoff[mu] + (size_t)f * Q::MREC;
            const float si = row >= NV ? -1.0f : 1.0f;
            float br = 0.0f, bi = 0.0f;
            if constexpr (P == CD_FP32) {
                for (int j = d; j < Q::N; j += Q::D) {
                    const float2 mm = __ldg(reinterpret_cast<const float2 *>(m + (size_t)j * Q::ROWB) + row);
                    float2 u = __ldg(reinterpret_cast<const float2 *>(vrec) + j);
                    if ((j >= NV) != (a.dagger && j >= NV)) u = make_float2(-u.x, -u.y);
                    br = fmaf(mm.x, u.x, fmaf(mm.y, u.y, br));
                    bi = fmaf(mm.x, u.y, fmaf(-mm.y, u.x, bi));
                }
            } else {
                float ra = 0.f, rb = 0.f, ia = 0.f, ib = 0.f;
                for (int j = d; j < Q::N; j += Q::D) {
                    const uint32_t mm = __ldg(reinterpret_cast<const uint32_t *>(m + (size_t)j * Q::ROWB) + row);
                    uint32_t u = __ldg(reinterpret_cast<const uint32_t *>(vrec) + j);
                    if ((j >= NV) != (a.dagger && j >= NV)) u ^= 0x80008000u;
                    hmac1(mm, u, ra, rb, ia, ib);
                }
                const float sc = ld_nc_f32(m + Q::MSCALE) * vsc;
                br = (ra + rb) * sc;
                bi = (ia - ib) * sc;
            }
            re += si * br;
            im += si * bi;
        }
    }
#pragma unroll
    for (int o = Q::D / 2; o >= 1; o >>= 1) {
        re += shfl_xor(re, o);
        im += shfl_xor(im, o);
    }
    const bool owner = (d == 0);
    if (owner) {
        const float2 p = a.scratch[(size_t)site * Q::N + row];
        re += p.x;
        im += p.y;
    }
    const float sg = (a.dagger && row >= NV) ? -1.0f : 1.0f;
    store_site<P, NV>(static_cast<unsigned char *>(a.out), site, row, owner, sg * re, sg * im, red, 32 * NWARP, -1);
}

// link halo send: forward record L_{2mu}(x) of every x_mu = L-1 face site (compressed record 1 + mu)
template <cd_precision P, int NV>
__global__ void lhalo_pack_kernel(const unsigned char *comp, unsigned char *send, KGeom g, int4 pairs, int64_t o0,
                                  int64_t o1, int64_t o2, int64_t o3)
{
    using Q = Cfg<P, NV>;
    const int pi = blockIdx.y;
    const int mu = pi == 0 ? pairs.x : (pi == 1 ? pairs.y : (pi == 2 ? pairs.z : pairs.w));
    const int64_t off = mu == 0 ? o0 : (mu == 1 ? o1 : (mu == 2 ? o2 : o3));
    const int L = sel4(g.L, mu);
    const int F = g.V / L;
    for (int f = blockIdx.x; f < F; f += gridDim.x) {
        int x[4];
        // face index f: lexicographic over the other three dims (as dslash_fgh_halo)
        if (mu == 0) { x[1] = f % g.L[1]; x[2] = (f / g.L[1]) % g.L[2]; x[3] = f / (g.L[1] * g.L[2]); }
        else if (mu == 1) { x[0] = f % g.L[0]; x[2] = (f / g.L[0]) % g.L[2]; x[3] = f / (g.L[0] * g.L[2]); }
        else if (mu == 2) { x[0] = f % g.L[0]; x[1] = (f / g.L[0]) % g.L[1]; x[3] = f / (g.L[0] * g.L[1]); }
        else { x[0] = f % g.L[0]; x[1] = (f / g.L[0]) % g.L[1]; x[2] = f / (g.L[0] * g.L[1]); }
        if (mu == 0) x[0] = L - 1;
        else if (mu == 1) x[1] = L - 1;
        else if (mu == 2) x[2] = L - 1;
        else x[3] = L - 1;
        const uint4 *src = reinterpret_cast<const uint4 *>(comp + ((size_t)encode(g, x) * 5 + 1 + mu) * Q::MREC);
        uint4 *dst = reinterpret_cast<uint4 *>(send + off + (size_t)f * Q::MREC);
        for (int e = threadIdx.x; e < Q::MREC / 16; e += blockDim.x) dst[e] = src[e];
    }
}

// full links -> compressed records (X, L_0, L_2, L_4, L_6 per site), one CTA per output record
template <cd_precision P, int NV>
__global__ void links_compress_kernel(const unsigned char *full, unsigned char *comp, int64_t nrec)
{
    using Q = Cfg<P, NV>;
    const int64_t rec = blockIdx.x;
    const int64_t site = rec / 5;
    const int c = (int)(rec - site * 5);
    const int k = c == 0 ? 8 : 2 * (c - 1);
    const uint4 *src = reinterpret_cast<const uint4 *>(full + ((size_t)site * 9 + k) * Q::MREC);
    uint4 *dst = reinterpret_cast<uint4 *>(comp + (size_t)rec * Q::MREC);
    for (int e = threadIdx.x; e < Q::MREC / 16; e += blockDim.x) dst[e] = src[e];
}

// max |L_{2mu+1}(x) - tau3 L_{2mu}(x-mu)^H tau3| over the lattice (fp32 links): the validity check
// of the compression.  One CTA per (site, mu); result via an atomic max on the float bits (>= 0).
template <int NV>
__global__ void links_herm_dev_kernel(const unsigned char *full, KGeom g, float *dev, const unsigned char *lhalo,
                                   int64_t o0, int64_t o1, int64_t o2, int64_t o3)
{
    using Q = Cfg<CD_FP32, NV>;
    const int site = blockIdx.x >> 2, mu = blockIdx.x & 3;
    int x[4];
    decode(g, site, x);
    const int nb = neighbour(g, x, site, 2 * mu + 1);
    const float2 *B = reinterpret_cast<const float2 *>(full + ((size_t)site * 9 + 2 * mu + 1) * Q::MREC);
    const unsigned char *frec = full + ((size_t)nb * 9 + 2 * mu) * Q::MREC;
    if (lhalo != nullptr && ((g.split >> mu) & 1) && x[mu] == 0) {   // the -mu neighbour is remote: link halo
        const int f = mu == 0 ? (x[3] * g.L[2] + x[2]) * g.L[1] + x[1]
                    : mu == 1 ? (x[3] * g.L[2] + x[2]) * g.L[0] + x[0]
                    : mu == 2 ? (x[3] * g.L[1] + x[1]) * g.L[0] + x[0]
                              : (x[2] * g.L[1] + x[1]) * g.L[0] + x[0];
        frec = lhalo + (mu == 0 ? o0 : mu == 1 ? o1 : mu == 2 ? o2 : o3) + (size_t)f * Q::MREC;
    }
    const float2 *F = reinterpret_cast<const float2 *>(frec);
    float m = 0.0f;
    for (int e = threadIdx.x; e < Q::N * Q::N; e += blockDim.x) {
        const int i = e / Q::N, j = e - i * Q::N;
        const float s = ((i < NV) == (j < NV)) ? 1.0f : -1.0f;
        const float2 f = F[j * Q::N + i];
        const float2 b = B[e];
        m = fmaxf(m, fmaxf(fabsf(b.x - s * f.x), fabsf(b.y + s * f.y)));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, shfl_xor(m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int *>(dev), __float_as_int(m));
}

// ------------------------------------------------------------------ CHAIN variant (latency regime)
// n chained applies (t even: y = D x, t odd: x = D y) in ONE cooperative launch.  The CTA grid
// is the FG decomposition; every CTA keeps its link rows in registers for all n applies (the
// whole 2^4 operator is 2.7 MB spread over the SMs) and waits point-to-point for the nine
// neighbour sites of the previous apply through per-site counters (release / acquire at gpu
// scope) -- no kernel boundary and no grid-wide barrier between applies.  Waiting for the
// neighbours' counters covers both hazards: their outputs (RAW) and their reads of the buffer
// this CTA is about to overwrite (WAR; the stencil is symmetric).  Counters are monotonic; the
// host passes the base value.
__device__ __forceinline__ uint4 ld_cg(const void *p)
{
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <cd_precision P, int NV, int KW, int WR>
__global__ void __launch_bounds__(FgCfg<P, NV, KW, WR>::THREADS) dslash_chain(ApplyArgs a, int n, unsigned base)
{
    using Q = Cfg<P, NV>;
    using F = FgCfg<P, NV, KW, WR>;
    static_assert(!F::SPLIT16, "fp16 chain needs whole-site CTAs");
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];
    __shared__ float2 part[F::WK][F::ROWS];
    __shared__ float red[32];

    const int site = blockIdx.x / F::NRB, rb = blockIdx.x - site * F::NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wk = warp / WR, wr = warp - wk * WR;
    const int r = lane / Q::D, d = lane % Q::D;
    const int rowl = wr * Q::R + r, row = rb * F::ROWS + rowl;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    unsigned char *const buf0 = const_cast<unsigned char *>(static_cast<const unsigned char *>(a.in));
    unsigned char *const buf1 = static_cast<unsigned char *>(a.out);
    unsigned *cnt = a.chain_cnt;

    int x[4];
    decode(a.g, site, x);
    uint4 Lc[KW][Q::C];
    float sl[KW];
#pragma unroll
    for (int kk = 0; kk < KW; kk++) {
        const int k = kseq(wk * KW + kk);
        const unsigned char *m = links + ((size_t)site * 9 + k) * Q::MREC;
#pragma unroll
        for (int c = 0; c < Q::C; c++) Lc[kk][c] = ld_stream(m + row * Q::ROWB + (d + Q::D * c) * 16);
        sl[kk] = Q::F16 ? ld_nc_f32(m + Q::MSCALE) : 0.0f;
    }

    if (a.dagger) {   // tau3 on the input, folded once into the register-resident links (chunks j >= Nvec)
#pragma unroll
        for (int j = 0; j < KW; j++)
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                if ((d + Q::D * c) * Q::CPC >= NV) Lc[j][c] = neg_chunk<Q::F16>(Lc[j][c]);
    }
    const int t9 = threadIdx.x < 9 ? neighbour(a.g, x, site, threadIdx.x) : 0;

    for (int t = 0; t < n; t++) {
        const unsigned char *in = (t & 1) ? buf1 : buf0;
        unsigned char *out = (t & 1) ? buf0 : buf1;
        if (t > 0 && threadIdx.x < 9) {   // neighbours (and self) finished apply t-1
            const unsigned target = base + (unsigned)(t * F::NRB);
            while ((int)(ld_acquire(&cnt[t9]) - target) < 0) {
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 9 * Q::VCH; e += F::THREADS) {
            const int k = e / Q::VCH, c16 = e - k * Q::VCH;
            const int nb = neighbour(a.g, x, site, k);
            *reinterpret_cast<uint4 *>(vs + k * Q::VREC + c16 * 16) = ld_cg(in + (size_t)nb * Q::VREC + c16 * 16);
        }
        __syncthreads();
        float re = 0.0f, im = 0.0f;
#pragma unroll
        for (int kk = 0; kk < KW; kk++) {
            const int k = kseq(wk * KW + kk);
            const unsigned char *vrec = vs + k * Q::VREC;
            if constexpr (P == CD_FP32) {
                float pr[Q::C], pi[Q::C];
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    pr[c] = 0.0f;
                    pi[c] = 0.0f;
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    cmac2(Lc[kk][c], vq, pr[c], pi[c]);
                }
#pragma unroll
                for (int c = 0; c < Q::C; c++) { re += pr[c]; im += pi[c]; }
            } else {
                float ra = 0.f, rb2 = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    hmac4(Lc[kk][c], vq, ra, rb2, ia, ib);
                }
                const float sc = sl[kk] * *reinterpret_cast<const float *>(vrec + Q::VSCALE);
                re = fmaf(ra - rb2, sc, re);
                im = fmaf(ia + ib, sc, im);
            }
        }
#pragma unroll
        for (int m = Q::D / 2; m >= 1; m >>= 1) {
            re += shfl_xor(re, m);
            im += shfl_xor(im, m);
        }
        if (d == 0) part[wk][rowl] = make_float2(re, im);
        __syncthreads();
        const bool owner = threadIdx.x < F::ROWS;
        float yr = 0.0f, yi = 0.0f;
        if (owner) {
#pragma unroll
            for (int w = 0; w < F::WK; w++) {
                yr += part[w][threadIdx.x].x;
                yi += part[w][threadIdx.x].y;
            }
        }
        const int orow = rb * F::ROWS + (owner ? threadIdx.x : 0);
        const float sg = (a.dagger && orow >= NV) ? -1.0f : 1.0f;
        store_site<P, NV>(out, site, orow, owner, sg * yr, sg * yi, red, F::THREADS, -1);
        __syncthreads();
        if (threadIdx.x == 0)   // publish: this row block finished apply t (release, gpu scope)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&cnt[site]) : "memory");
    }
}

inline cudaError_t launch_ex(const void *fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, void **args,
                             bool cooperative);

// ------------------------------------------------------------------ LL chain (latency regime)
// As dslash_chain, but the intermediate vectors travel in an "LL" format (as NCCL's LL
// protocol): every 4-byte payload word is stored together with its epoch in ONE 8-byte store,
// so a reader polls the data itself -- no separate completion flag, no release fence, one L2
// round trip per apply on the critical path.  Double-buffered: apply t reads LL[t&1] (epoch
// base+t), writes LL[(t+1)&1] (epoch base+t+1); having read all nine neighbour records of
// epoch base+t proves those CTAs finished apply t-1, including their reads of the buffer this
// CTA now overwrites (symmetric stencil).  Every iterate is also stored in the ordinary
// format (x / y ping-pong), off the critical path.
template <cd_precision P, int NV>
struct LLCfg {
    using Q = Cfg<P, NV>;
    static constexpr int W = Q::F16 ? Q::N + 1 : 2 * Q::N;   // payload words per record (+scale for fp16)
    static constexpr int WP = (W + 1) / 2;                     // 16-byte units (2 LL words) per record
    static constexpr int REC = WP * 16;                        // LL record bytes
};

template <cd_precision P, int NV, int KW, int WR>
__global__ void __launch_bounds__(FgCfg<P, NV, KW, WR>::THREADS) dslash_llchain(ApplyArgs a, int n, unsigned base)
{
    using Q = Cfg<P, NV>;
    using F = FgCfg<P, NV, KW, WR>;
    using LL = LLCfg<P, NV>;
    static_assert(!F::SPLIT16, "fp16 chain needs whole-site CTAs");
    constexpr int UNITS = 9 * LL::WP;                               // 16-B LL units to gather
    constexpr int U = (UNITS + F::THREADS - 1) / F::THREADS;       // per thread
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];
    __shared__ float2 part[F::WK][F::ROWS];
    __shared__ float red[32];

    const int site = blockIdx.x / F::NRB, rb = blockIdx.x - site * F::NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wk = warp / WR, wr = warp - wk * WR;
    const int r = lane / Q::D, d = lane % Q::D;
    const int rowl = wr * Q::R + r, row = rb * F::ROWS + rowl;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    unsigned char *const buf0 = const_cast<unsigned char *>(static_cast<const unsigned char *>(a.in));
    unsigned char *const buf1 = static_cast<unsigned char *>(a.out);
    unsigned char *const ll = reinterpret_cast<unsigned char *>(a.llbuf);
    const size_t llhalf = (size_t)a.g.V * LL::REC;

    int x[4];
    decode(a.g, site, x);
    uint4 Lc[KW][Q::C];
    float sl[KW];
#pragma unroll
    for (int kk = 0; kk < KW; kk++) {
        const int k = kseq(wk * KW + kk);
        const unsigned char *m = links + ((size_t)site * 9 + k) * Q::MREC;
#pragma unroll
        for (int c = 0; c < Q::C; c++) Lc[kk][c] = ld_stream(m + row * Q::ROWB + (d + Q::D * c) * 16);
        sl[kk] = Q::F16 ? ld_nc_f32(m + Q::MSCALE) : 0.0f;
    }

    if (a.dagger) {   // tau3 on the input, folded once into the register-resident links (chunks j >= Nvec)
#pragma unroll
        for (int j = 0; j < KW; j++)
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                if ((d + Q::D * c) * Q::CPC >= NV) Lc[j][c] = neg_chunk<Q::F16>(Lc[j][c]);
    }
    // the LL units this thread gathers: (hop k, unit w) -> source site
    int uk[U], uw[U], unb[U];
#pragma unroll
    for (int i = 0; i < U; i++) {
        const int e = threadIdx.x + i * F::THREADS;
        uk[i] = e < UNITS ? e / LL::WP : -1;
        uw[i] = e < UNITS ? e - uk[i] * LL::WP : 0;
        unb[i] = e < UNITS ? neighbour(a.g, x, site, uk[i]) : 0;
    }

    for (int t = 0; t < n; t++) {
        unsigned char *gout = (t & 1) ? buf0 : buf1;
        if (t == 0) {   // the input is ready at launch: ordinary format
            for (int e = threadIdx.x; e < 9 * Q::VCH; e += F::THREADS) {
                const int k = e / Q::VCH, c16 = e - k * Q::VCH;
                *reinterpret_cast<uint4 *>(vs + k * Q::VREC + c16 * 16) =
                    ld_nc(buf0 + (size_t)neighbour(a.g, x, site, k) * Q::VREC + c16 * 16);
            }
        } else {        // poll the LL words of epoch base + t
            const unsigned want = base + (unsigned)t;
            const unsigned char *src = ll + (size_t)(t & 1) * llhalf;
            uint4 v[U];
            bool done[U];
#pragma unroll
            for (int i = 0; i < U; i++) done[i] = uk[i] < 0;
            bool all = false;
            bool first = true;
            while (!all) {
                if (!first && a.poll_ns > 0) __nanosleep(a.poll_ns);   // back off: spinning loads share L2 with the writers
                first = false;
#pragma unroll
                for (int i = 0; i < U; i++)
                    if (!done[i]) v[i] = ld_cg(src + (size_t)unb[i] * LL::REC + uw[i] * 16);
                all = true;
#pragma unroll
                for (int i = 0; i < U; i++) {
                    if (done[i]) continue;
                    const bool last_odd = (LL::W & 1) && uw[i] == LL::WP - 1;   // second word is padding
                    done[i] = v[i].y == want && (last_odd || v[i].w == want);
                    if (done[i]) {   // unpack the (1 or 2) payload words into the ordinary record
                        unsigned *dst = reinterpret_cast<unsigned *>(vs + uk[i] * Q::VREC);
                        const int w0 = 2 * uw[i];
                        if constexpr (Q::F16) {
                            dst[w0 == Q::N ? Q::VSCALE / 4 : w0] = v[i].x;
                            if (!last_odd) dst[w0 + 1 == Q::N ? Q::VSCALE / 4 : w0 + 1] = v[i].z;
                        } else {
                            dst[w0] = v[i].x;
                            dst[w0 + 1] = v[i].z;
                        }
                    }
                    all = all && done[i];
                }
            }
        }
        __syncthreads();
        float re = 0.0f, im = 0.0f;
#pragma unroll
        for (int kk = 0; kk < KW; kk++) {
            const int k = kseq(wk * KW + kk);
            const unsigned char *vrec = vs + k * Q::VREC;
            if constexpr (P == CD_FP32) {
                float pr[Q::C], pi[Q::C];
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    pr[c] = 0.0f;
                    pi[c] = 0.0f;
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    cmac2(Lc[kk][c], vq, pr[c], pi[c]);
                }
#pragma unroll
                for (int c = 0; c < Q::C; c++) { re += pr[c]; im += pi[c]; }
            } else {
                float ra = 0.f, rb2 = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    hmac4(Lc[kk][c], vq, ra, rb2, ia, ib);
                }
                const float sc = sl[kk] * *reinterpret_cast<const float *>(vrec + Q::VSCALE);
                re = fmaf(ra - rb2, sc, re);
                im = fmaf(ia + ib, sc, im);
            }
        }
#pragma unroll
        for (int m = Q::D / 2; m >= 1; m >>= 1) {
            re += shfl_xor(re, m);
            im += shfl_xor(im, m);
        }
        if (d == 0) part[wk][rowl] = make_float2(re, im);
        __syncthreads();
        const bool owner = threadIdx.x < F::ROWS;
        float yr = 0.0f, yi = 0.0f;
        if (owner) {
#pragma unroll
            for (int w = 0; w < F::WK; w++) {
                yr += part[w][threadIdx.x].x;
                yi += part[w][threadIdx.x].y;
            }
        }
        const int orow = rb * F::ROWS + (owner ? threadIdx.x : 0);
        const float sg = (a.dagger && orow >= NV) ? -1.0f : 1.0f;
        yr *= sg;
        yi *= sg;
        const unsigned ep = base + (unsigned)t + 1;
        unsigned char *dst = ll + (size_t)((t + 1) & 1) * llhalf + (size_t)site * LL::REC;
        if constexpr (P == CD_FP32) {
            if (owner) {   // one 16-byte store = two LL words {re, ep}, {im, ep}
                reinterpret_cast<uint4 *>(dst)[orow] = make_uint4(__float_as_uint(yr), ep, __float_as_uint(yi), ep);
                reinterpret_cast<float2 *>(gout + (size_t)site * Q::VREC)[orow] = make_float2(yr, yi);
            }
        } else {
            float mx = owner ? fmaxf(fabsf(yr), fabsf(yi)) : 0.0f;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, shfl_xor(mx, o));
            if (lane == 0) red[warp] = mx;
            __syncthreads();
            float s = 0.0f;
            for (int w = 0; w < F::NW; w++) s = fmaxf(s, red[w]);
            if (owner) {
                __half2 q;
                if (s > 0.0f) q = __halves2half2(__float2half_rn(__fdiv_rn(yr, s)), __float2half_rn(__fdiv_rn(yi, s)));
                else q = __halves2half2(__float2half_rn(0.0f), __float2half_rn(0.0f));
                const unsigned qb = *reinterpret_cast<unsigned *>(&q);
                reinterpret_cast<uint2 *>(dst)[orow] = make_uint2(qb, ep);
                reinterpret_cast<unsigned *>(gout + (size_t)site * Q::VREC)[orow] = qb;
                if (orow == 0) {
                    reinterpret_cast<uint2 *>(dst)[Q::N] = make_uint2(__float_as_uint(s), ep);
                    *reinterpret_cast<float *>(gout + (size_t)site * Q::VREC + Q::VSCALE) = s;
                }
            }
        }
        __syncthreads();   // vs / part / red reuse in the next apply
    }
}

// ------------------------------------------------------------------ LL-register chain (2^4 latency regime)
// The LL protocol of dslash_llchain with the on-chip critical path cut down:
//  * one warp per hop k (the paper's direction split) polls ITS OWN neighbour's LL
//    record (lane-contiguous 16-B units, whole record) -- no CTA barrier before the math; a warp
//    runs its chunk FMAs the moment its neighbour's record lands;
//  * the hop partials meet in shared memory; the hop warps `bar.arrive` (non-blocking), warp 0
//    alone `bar.sync`s, sums the 9 partials in the fixed hop order and stores the LL record;
//  * GATE: the hop warps then wait (second named barrier) until warp 0 has ISSUED that store
//    before they poll the next epoch -- spinning loads of the next epoch would otherwise sit in
//    the SM's L1tex queue in front of warp 0's shared loads and LL store (the critical path;
//    measured 440-1050 cycles of queueing without the gate);
//  * REP: the writer stores its rows to REP replicas of the LL buffer and reader CTA b polls
//    replica b % REP, so each 128-B line has REP x fewer pollers (a hot line is served by one L2
//    slice; 108 warps poll each line per round at 2^4 with 12 CTAs per site).
//  * ROWS rows per CTA (NRB = N / ROWS CTAs per site; ROWS = 6 gives 128 CTAs at 2^4 -- one
//    per SM); WR = ceil(ROWS / 4) warps per hop, surplus rows computed on clamped data, unused.
// Without GATE, the named barriers and the partial buffers alternate with t & 1: a hop warp
// can run at most one apply ahead of warp 0 (its neighbour's epoch t+2 needs this site's epoch
// t+1 record, which warp 0 writes after consuming the partials of apply t).
// The per-row arithmetic (chunk partials, xor-shuffle over the dot split, hop sum from 0 in hop
// order) is that of dslash_fg<kw=1>: the chain is bitwise equal to single applies of it.
// fp32 storage (the fp16 format quantises a whole site, which one CTA of ROWS rows cannot).
struct LLRDesc {
    int rows, ld;   // rows per CTA, lanes per row (dot-product split)
};
constexpr LLRDesc kLLR[] = {{4, 8}, {8, 4}, {6, 4}, {8, 8}, {12, 4}, {16, 2}};
constexpr int kNLLR = sizeof(kLLR) / sizeof(kLLR[0]);
static_assert(kNLLR == kNumLLReg, "LL-register variant count");

template <int NV, int ROWS, int LD>
struct LLRegCfg {
    static constexpr int N = 2 * NV;
    static constexpr int LR = 32 / LD;               // rows per warp
    static constexpr int LC = N / (2 * LD);          // 16-B chunks (2 complex) per lane per row
    static constexpr int WR = (ROWS + LR - 1) / LR;  // warps per hop
    static constexpr int NW = 9 * WR;
    static constexpr int THREADS = 32 * NW;
    static constexpr int NRB = N / ROWS;
    static constexpr bool OK = (N % ROWS == 0) && (LC * LD * 2 == N) && NW <= 32 && ROWS <= 32;
};

__device__ __forceinline__ void spin_until(long long c)
{
    while (clock64() < c) {
    }
}

template <int NV, int ROWS, int LD>
__global__ void __launch_bounds__(LLRegCfg<NV, ROWS, LD>::THREADS) dslash_llreg(ApplyArgs a, int n, unsigned base)
{
    using Q = Cfg<CD_FP32, NV>;
    using F = LLRegCfg<NV, ROWS, LD>;
    using LL = LLCfg<CD_FP32, NV>;
    constexpr int UPL = (LL::WP + 31) / 32;   // LL units per lane (whole record, lane-contiguous)
    __shared__ float2 part[9][F::WR * F::LR];
    __shared__ __align__(16) float2 vst[F::NW][Q::N];

    const int site = blockIdx.x / F::NRB, rb = blockIdx.x - site * F::NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wk = warp / F::WR, wr = warp - wk * F::WR;
    const int r = lane / LD, d = lane % LD;
    const int rowl = wr * F::LR + r;
    const int row = rb * ROWS + (rowl < ROWS ? rowl : ROWS - 1);
    const int k = kseq(wk);
    unsigned char *const buf0 = const_cast<unsigned char *>(static_cast<const unsigned char *>(a.in));
    unsigned char *const buf1 = static_cast<unsigned char *>(a.out);
    unsigned char *const ll = reinterpret_cast<unsigned char *>(a.llbuf);
    const size_t llhalf = (size_t)a.g.V * LL::REC;
    long long *const tr = (a.trace && blockIdx.x == 0 && lane == 0) ? a.trace : nullptr;

    int x[4];
    decode(a.g, site, x);
    const int nb = neighbour(a.g, x, site, k);
    uint4 Lc[F::LC];
    {
        const unsigned char *m = static_cast<const unsigned char *>(a.links) + ((size_t)site * 9 + k) * Q::MREC;
#pragma unroll
        for (int c = 0; c < F::LC; c++) Lc[c] = ld_stream(m + row * Q::ROWB + (d + LD * c) * 16);
    }
    if (a.dagger) {   // tau3 on the input folded into the register-resident links (columns j >= Nvec)
#pragma unroll
        for (int c = 0; c < F::LC; c++)
            if ((d + LD * c) * 2 >= NV) Lc[c] = neg_chunk<false>(Lc[c]);
    }

    for (int t = 0; t < n; t++) {
        // trace (CD_CHAIN_TRACE, CTA 0, lane 0 of the wr == 0 warps): absolute clock64 per event,
        // written at the end of the apply; row 4 * wk + e (e: 0 start, 1 record landed, 2 arrived
        // at the partials barrier (hop warps) / its LDS returned (warp 0)), warp 0 also 36 summed,
        // 37 LL store issued, 38 go barrier arrived, 39 trace written.  (BAR.SYNC defers blocking
        // to the next dependent memory instruction, so warp 0's barrier time is read after a load.)
        long long c_start = 0, c_data = 0, c_bar = 0, c_sum = 0, c_st = 0;
        const long long c_start0 = clock64();
        if (tr) c_start = c_start0;
        uint4 vq[F::LC];
        if (t == 0) {   // the input is ready at launch: ordinary format
#pragma unroll
            for (int c = 0; c < F::LC; c++) vq[c] = ld_nc(buf0 + (size_t)nb * Q::VREC + (d + LD * c) * 16);
        } else {        // poll the neighbour's record of epoch base + t
            const unsigned want = base + (unsigned)t;
            const unsigned char *src = ll + (size_t)(t & 1) * llhalf + (size_t)nb * LL::REC;
            uint4 u[UPL];
            unsigned miss = 0;
#pragma unroll
            for (int i = 0; i < UPL; i++)
                if (lane + 32 * i < LL::WP) miss |= 1u << i;
            // Polls are cheap for the poller but not for the system: every poll of a hot line
            // queues at its L2 slice in front of the writers' stores and the other pollers
            // (measured: two rounds in flight per warp slow the chain by 10 %).  So the first
            // poll waits until the record can plausibly have landed (poll_d0 cycles after this
            // warp's start of the apply) and unsuccessful polls back off poll_d1 cycles.
            if (a.poll_ns > 0) __nanosleep(a.poll_ns);
            if (a.poll_d0 > 0) spin_until(c_start0 + a.poll_d0);
            while (true) {
#pragma unroll
                for (int i = 0; i < UPL; i++)
                    if (miss & (1u << i)) u[i] = ld_cg(src + (lane + 32 * i) * 16);
#pragma unroll
                for (int i = 0; i < UPL; i++)
                    if ((miss & (1u << i)) && u[i].y == want && u[i].w == want) miss &= ~(1u << i);
                if (!__any_sync(0xffffffffu, miss != 0u)) break;
                if (a.poll_d1 > 0) spin_until(clock64() + a.poll_d1);
            }
#pragma unroll
            for (int i = 0; i < UPL; i++)
                if (lane + 32 * i < LL::WP)
                    vst[warp][lane + 32 * i] = make_float2(__uint_as_float(u[i].x), __uint_as_float(u[i].z));
            __syncwarp();
#pragma unroll
            for (int c = 0; c < F::LC; c++) vq[c] = lds128(&vst[warp][2 * (d + LD * c)]);
            __syncwarp();
        }
        if (tr) c_data = clock64();
        float re = 0.0f, im = 0.0f;
        {
            float pr[F::LC], pi[F::LC];
#pragma unroll
            for (int c = 0; c < F::LC; c++) {
                pr[c] = 0.0f;
                pi[c] = 0.0f;
                cmac2(Lc[c], vq[c], pr[c], pi[c]);
            }
#pragma unroll
            for (int c = 0; c < F::LC; c++) { re += pr[c]; im += pi[c]; }
        }
#pragma unroll
        for (int m = LD / 2; m >= 1; m >>= 1) {
            re += shfl_xor(re, m);
            im += shfl_xor(im, m);
        }
        if (d == 0) part[wk][rowl] = make_float2(re, im);
        if (warp != 0) {   // hop warps: arrive, then wait until warp 0 has issued the LL store
            asm volatile("bar.arrive 1, %0;" ::"r"(F::THREADS) : "memory");
            if (tr) c_bar = clock64();
            asm volatile("bar.sync 2, %0;" ::"r"(F::THREADS) : "memory");
            if (tr && wr == 0 && t < 1024) {
                tr[(4 * wk + 0) * 1024 + t] = c_start;
                tr[(4 * wk + 1) * 1024 + t] = c_data;
                tr[(4 * wk + 2) * 1024 + t] = c_bar;
            }
            continue;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(F::THREADS) : "memory");
        if (lane < ROWS) {
            float yr = 0.0f, yi = 0.0f;
#pragma unroll
            for (int w = 0; w < 9; w++) {
                const float2 p = part[w][lane];
                if (w == 0 && tr) c_bar = clock64();
                yr += p.x;
                yi += p.y;
            }
            const int orow = rb * ROWS + lane;
            if (a.dagger && orow >= NV) yr = -yr, yi = -yi;
            if (tr) c_sum = clock64();
            const unsigned ep = base + (unsigned)t + 1;
            reinterpret_cast<uint4 *>(ll + (size_t)((t + 1) & 1) * llhalf + (size_t)site * LL::REC)[orow] =
                make_uint4(__float_as_uint(yr), ep, __float_as_uint(yi), ep);
            if (t >= n - 2) {   // the caller sees the last two iterates (x / y ping-pong)
                unsigned char *gout = (t & 1) ? buf0 : buf1;
                reinterpret_cast<float2 *>(gout + (size_t)site * Q::VREC)[orow] = make_float2(yr, yi);
            }
        }
        if (tr) c_st = clock64();
        asm volatile("bar.arrive 2, %0;" ::"r"(F::THREADS) : "memory");
        if (tr && t < 1024) {
            const long long c_go = clock64();
            tr[0 * 1024 + t] = c_start;
            tr[1 * 1024 + t] = c_data;
            tr[2 * 1024 + t] = c_bar;
            tr[36 * 1024 + t] = c_sum;
            tr[37 * 1024 + t] = c_st;
            tr[38 * 1024 + t] = c_go;
            tr[39 * 1024 + t] = clock64();
        }
    }
}

template <int NV, int I>
cudaError_t launch_llreg_t(const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms)
{
    constexpr LLRDesc D = kLLR[I];
    using F = LLRegCfg<NV, D.rows, D.ld>;
    if constexpr (!F::OK) {
        return cudaErrorNotSupported;
    } else {
        auto fn = dslash_llreg<NV, D.rows, D.ld>;
        const size_t smem = 0;
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, F::THREADS, smem);
        if (e != cudaSuccess) return e;
        if ((int64_t)a.g.V * F::NRB > (int64_t)per_sm * num_sms) return cudaErrorCooperativeLaunchTooLarge;
        ApplyArgs aa = a;
        int nn = n;
        unsigned bb = base;
        void *args[] = {&aa, &nn, &bb};
        return launch_ex((const void *)fn, dim3((unsigned)(a.g.V * F::NRB)), dim3(F::THREADS), smem, s, false, args,
                         true);
    }
}

// LL-register chain variants: id LLREG_CHAIN_ID0 + 1 + index into kLLR
template <cd_precision P, int NV, int I = 0>
cudaError_t dispatch_llreg(int idx, const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms)
{
    if constexpr (P != CD_FP32 || I >= kNLLR) {
        return cudaErrorNotSupported;
    } else {
        if (idx == I) return launch_llreg_t<NV, I>(a, n, base, s, num_sms);
        return dispatch_llreg<P, NV, I + 1>(idx, a, n, base, s, num_sms);
    }
}

template <cd_precision P, int NV, int KW, int WR>
cudaError_t launch_llchain_t(const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms)
{
    using F = FgCfg<P, NV, KW, WR>;
    if constexpr (F::SPLIT16) {
        return cudaErrorNotSupported;
    } else {
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dslash_llchain<P, NV, KW, WR>, F::THREADS, 0);
        if (e != cudaSuccess) return e;
        if ((int64_t)a.g.V * F::NRB > (int64_t)per_sm * num_sms) return cudaErrorCooperativeLaunchTooLarge;
        ApplyArgs aa = a;
        int nn = n;
        unsigned bb = base;
        void *args[] = {&aa, &nn, &bb};
        return launch_ex((const void *)dslash_llchain<P, NV, KW, WR>, dim3((unsigned)(a.g.V * F::NRB)),
                         dim3(F::THREADS), 0, s, false, args, true);
    }
}

// ------------------------------------------------------------------ LL-warp chain (fp32; latency regime)
// The LL protocol of dslash_llchain / dslash_llreg with the work of a row kept in ONE warp:
//   * CTA = one warp = 4 rows of one site (N/4 CTAs per site); lane (row r, d of 8) holds
//     L_k(x)[row][chunks d, d+8, ...] for ALL nine hops in registers (cmac2x / FFMA2 math), so
//     the hop sum never leaves registers and the 8-lane xor-shuffle leaves y(x)[row] in every
//     lane of the row -- no shared-memory reduction, no CTA barrier, no warp hand-off;
//   * the warp polls the distinct neighbour records of the epoch it needs (at L_mu = 2 the
//     +-mu hops share one record, at L_mu = 1 a hop reads the site's own record) with one
//     round of lane-contiguous 16-B LL loads per poll, stages the payload in shared memory and
//     runs the nine mat-vecs; lane d = 0 of each row then stores the row's LL word.
// Critical path per apply: L2 round trip of the LL words + the warp's math + 3 shuffles + one
// store (the LL-register chain adds a cross-warp reduction and a barrier hand-off).  fp32 only.
template <int NV>
struct LLWarpCfg {
    static constexpr int N = 2 * NV;
    static constexpr int LD = 8;              // lanes per row (dot-product split)
    static constexpr int RPW = 32 / LD;       // rows per warp (= per CTA)
    static constexpr int NWS = N / RPW;       // CTAs per site
    static constexpr int LC = N / (2 * LD);   // 16-B link chunks per lane per hop
};

template <int NV>
__global__ void __launch_bounds__(32, 1) dslash_llwarp(ApplyArgs a, int n, unsigned base)
{
    using Q = Cfg<CD_FP32, NV>;
    using K = LLWarpCfg<NV>;
    using LL = LLCfg<CD_FP32, NV>;
    constexpr int UPL = (LL::WP + 31) / 32;   // LL units per lane per record
    __shared__ __align__(16) float2 vst[9][K::N];

    const int site = blockIdx.x / K::NWS, wb = blockIdx.x - site * K::NWS;
    const int lane = threadIdx.x, d = lane % K::LD;
    const int row = wb * K::RPW + lane / K::LD;
    unsigned char *const buf0 = const_cast<unsigned char *>(static_cast<const unsigned char *>(a.in));
    unsigned char *const buf1 = static_cast<unsigned char *>(a.out);
    unsigned char *const ll = reinterpret_cast<unsigned char *>(a.llbuf);
    const size_t llhalf = (size_t)a.g.V * LL::REC;

    int x[4];
    decode(a.g, site, x);
    int nb[9];          // neighbour of hop position i (kseq order: X first)
    uint32_t dup = 0;   // bit i: hop i reads the record staged for hop src(i) (L_mu = 2: i - 1; L_mu = 1: 0)
    uint32_t dsrc1 = 0; // bit i: ... and that source is X (L_mu = 1)
#pragma unroll
    for (int i = 0; i < 9; i++) {
        const int k = kseq(i);
        nb[i] = neighbour(a.g, x, site, k);
        if (k < 8) {
            const int L = sel4(a.g.L, k >> 1);
            if (L == 1) dup |= 1u << i, dsrc1 |= 1u << i;
            else if (L == 2 && (k & 1)) dup |= 1u << i;
        }
    }
    uint4 Lc[9][K::LC];
#pragma unroll
    for (int i = 0; i < 9; i++) {
        const unsigned char *m = static_cast<const unsigned char *>(a.links) + ((size_t)site * 9 + kseq(i)) * Q::MREC +
                                 row * Q::ROWB;
#pragma unroll
        for (int c = 0; c < K::LC; c++) Lc[i][c] = ld_stream(m + (d + K::LD * c) * 16);
    }
    if (a.dagger) {   // tau3 on the input folded into the register-resident links (chunks q >= Nvec/2)
#pragma unroll
        for (int i = 0; i < 9; i++)
#pragma unroll
            for (int c = 0; c < K::LC; c++)
                if ((d + K::LD * c) * 2 >= NV) Lc[i][c] = neg_chunk<false>(Lc[i][c]);
    }
    const float osign = (a.dagger && row >= NV) ? -1.0f : 1.0f;

    for (int t = 0; t < n; t++) {
        const long long c_start = clock64();
        unsigned long long A = 0ull, B = 0ull;
        if (t == 0) {   // the input is ready at launch: ordinary format
#pragma unroll
            for (int i = 0; i < 9; i++) {
                const unsigned char *src = buf0 + (size_t)nb[i] * Q::VREC;
#pragma unroll
                for (int c = 0; c < K::LC; c++) cmac2x(Lc[i][c], ld_nc(src + (d + K::LD * c) * 16), A, B);
            }
        } else {
            const unsigned want = base + (unsigned)t;
            const unsigned char *src = ll + (size_t)(t & 1) * llhalf;
            uint32_t miss = 0;   // bit UPL * i + u: unit lane + 32 u of hop i's record not landed yet
#pragma unroll
            for (int i = 0; i < 9; i++)
#pragma unroll
                for (int u = 0; u < UPL; u++)
                    if (!((dup >> i) & 1u) && lane + 32 * u < LL::WP) miss |= 1u << (UPL * i + u);
            __syncwarp();   // every lane finished reading vst (previous apply)
            if (a.poll_d0 > 0) spin_until(c_start + a.poll_d0);
            while (true) {
                uint4 w[9][UPL];
#pragma unroll
                for (int i = 0; i < 9; i++)
#pragma unroll
                    for (int u = 0; u < UPL; u++)
                        if ((miss >> (UPL * i + u)) & 1u) w[i][u] = ld_cg(src + (size_t)nb[i] * LL::REC + (lane + 32 * u) * 16);
#pragma unroll
                for (int i = 0; i < 9; i++)
#pragma unroll
                    for (int u = 0; u < UPL; u++)
                        if (((miss >> (UPL * i + u)) & 1u) && w[i][u].y == want && w[i][u].w == want) {
                            miss &= ~(1u << (UPL * i + u));
                            vst[i][lane + 32 * u] = make_float2(__uint_as_float(w[i][u].x), __uint_as_float(w[i][u].z));
                        }
                if (!__any_sync(0xffffffffu, miss != 0u)) break;
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 9; i++) {
                const int s = (i > 0 && ((dup >> i) & 1u)) ? (((dsrc1 >> i) & 1u) ? 0 : i - 1) : i;
                const float2 *v = vst[s];
#pragma unroll
                for (int c = 0; c < K::LC; c++) cmac2x(Lc[i][c], lds128(v + 2 * (d + K::LD * c)), A, B);
            }
        }
        float re = __uint_as_float((uint32_t)A) - __uint_as_float((uint32_t)(B >> 32));
        float im = __uint_as_float((uint32_t)(A >> 32)) + __uint_as_float((uint32_t)B);
#pragma unroll
        for (int m = K::LD / 2; m >= 1; m >>= 1) {
            re += shfl_xor(re, m);
            im += shfl_xor(im, m);
        }
        re *= osign;
        im *= osign;
        if (d == 0) {
            const unsigned ep = base + (unsigned)t + 1;
            if (t + 1 < n)
                reinterpret_cast<uint4 *>(ll + (size_t)((t + 1) & 1) * llhalf + (size_t)site * LL::REC)[row] =
                    make_uint4(__float_as_uint(re), ep, __float_as_uint(im), ep);
            if (t >= n - 2) {   // the caller sees the last two iterates (x / y ping-pong)
                unsigned char *gout = (t & 1) ? buf0 : buf1;
                reinterpret_cast<float2 *>(gout + (size_t)site * Q::VREC)[row] = make_float2(re, im);
            }
        }
    }
}

template <cd_precision P, int NV>
cudaError_t launch_llwarp_t(const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms)
{
    if constexpr (P != CD_FP32) {
        return cudaErrorNotSupported;
    } else {
        using K = LLWarpCfg<NV>;
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dslash_llwarp<NV>, 32, 0);
        if (e != cudaSuccess) return e;
        if ((int64_t)a.g.V * K::NWS > (int64_t)per_sm * num_sms) return cudaErrorCooperativeLaunchTooLarge;
        ApplyArgs aa = a;
        int nn = n;
        unsigned bb = base;
        void *args[] = {&aa, &nn, &bb};
        return launch_ex((const void *)dslash_llwarp<NV>, dim3((unsigned)(a.g.V * K::NWS)), dim3(32), 0, s, false, args,
                         true);
    }
}

// ------------------------------------------------------------------ CLUSTER chain (V <= 16 sites)
// The whole lattice in ONE thread-block cluster (non-portable size up to 16, one CTA per site):
// every CTA keeps its site's nine matrices in registers for all n applies and its current
// vector in shared memory; the neighbour records are read through distributed shared memory
// (mapa + ld.shared::cluster) and one cluster barrier per apply orders everything (double-
// buffered vectors: the barrier at the end of apply t lets apply t+1 overwrite the buffer
// apply t read).  Per apply: cluster barrier + one DSMEM round trip + the math -- no HBM/L2
// round trips, no kernel boundary.  Work per CTA: TASKS = 9 hops x (N/R) row groups, spread
// over NW warps (TPW tasks per warp); lanes split each row D ways as everywhere else.
template <cd_precision P, int NV, int NW>
struct ClusterCfg {
    using Q = Cfg<P, NV>;
    static constexpr int RG = Q::N / Q::R;          // row groups
    static constexpr int TASKS = 9 * RG;
    static constexpr int TPW = TASKS / NW;
    static constexpr int THREADS = 32 * NW;
    static_assert(TPW * NW == TASKS, "tasks must tile the warps");
    static_assert(THREADS >= 9 * (Q::VREC / 16), "one 16-B neighbour chunk per thread");
};


template <cd_precision P, int NV, int NW>
__global__ void __launch_bounds__(ClusterCfg<P, NV, NW>::THREADS, 1) dslash_cluster_chain(ApplyArgs a, int n)
{
    using Q = Cfg<P, NV>;
    using K = ClusterCfg<P, NV, NW>;
    __shared__ __align__(16) unsigned char vbuf[2][Q::VREC];   // this site's vector, by apply parity
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];     // the nine neighbour records
    __shared__ float2 part[9][Q::N];
    __shared__ float red[32];

    const int site = (int)cluster_rank();   // grid == one cluster of V CTAs
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = lane / Q::D, d = lane % Q::D;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    unsigned char *const g0 = const_cast<unsigned char *>(static_cast<const unsigned char *>(a.in));
    unsigned char *const g1 = static_cast<unsigned char *>(a.out);
    int x[4];
    decode(a.g, site, x);

    // links -> registers, once for all n applies
    uint4 Lc[K::TPW][Q::C];
    float sl[K::TPW];
#pragma unroll
    for (int j = 0; j < K::TPW; j++) {
        const int task = warp + NW * j;
        const int k = task / K::RG, rg = task - k * K::RG;
        const int row = rg * Q::R + r;
        const unsigned char *m = links + ((size_t)site * 9 + k) * Q::MREC;
#pragma unroll
        for (int c = 0; c < Q::C; c++) Lc[j][c] = ld_stream(m + row * Q::ROWB + (d + Q::D * c) * 16);
        sl[j] = Q::F16 ? ld_nc_f32(m + Q::MSCALE) : 0.0f;
    }

    if (a.dagger) {   // tau3 on the input, folded once into the register-resident links (chunks j >= Nvec)
#pragma unroll
        for (int j = 0; j < K::TPW; j++)
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                if ((d + Q::D * c) * Q::CPC >= NV) Lc[j][c] = neg_chunk<Q::F16>(Lc[j][c]);
    }
    // this thread's neighbour chunk (for the staging step)
    const int sk = threadIdx.x / Q::VCH, se = threadIdx.x - sk * Q::VCH;
    const bool stager = sk < 9;
    const unsigned src_cta = stager ? (unsigned)neighbour(a.g, x, site, sk) : 0u;
    for (int e = threadIdx.x; e < Q::VCH; e += K::THREADS)
        *reinterpret_cast<uint4 *>(vbuf[0] + e * 16) = ld_nc(g0 + (size_t)site * Q::VREC + e * 16);
    cluster_sync_all();

    for (int t = 0; t < n; t++) {
        const int pin = t & 1;
        if (stager)
            *reinterpret_cast<uint4 *>(vs + sk * Q::VREC + se * 16) = ld_dsmem(vbuf[pin] + se * 16, src_cta);
        __syncthreads();
        float rr[K::TPW], ii[K::TPW];
#pragma unroll
        for (int j = 0; j < K::TPW; j++) {
            const int task = warp + NW * j;
            const int k = task / K::RG;
            const unsigned char *vrec = vs + k * Q::VREC;
            float re = 0.0f, im = 0.0f;
            if constexpr (P == CD_FP32) {
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    cmac2(Lc[j][c], vq, re, im);
                }
            } else {
                float ra = 0.f, rb2 = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
                for (int c = 0; c < Q::C; c++) {
                    const int q = d + Q::D * c;
                    uint4 vq = lds128(vrec + q * 16);
                    hmac4(Lc[j][c], vq, ra, rb2, ia, ib);
                }
                const float sc = sl[j] * *reinterpret_cast<const float *>(vrec + Q::VSCALE);
                re = (ra - rb2) * sc;
                im = (ia + ib) * sc;
            }
            rr[j] = re;
            ii[j] = im;
        }
#pragma unroll
        for (int j = 0; j < K::TPW; j++) {
#pragma unroll
            for (int m = Q::D / 2; m >= 1; m >>= 1) {
                rr[j] += shfl_xor(rr[j], m);
                ii[j] += shfl_xor(ii[j], m);
            }
            const int task = warp + NW * j;
            const int k = task / K::RG, rg = task - k * K::RG;
            if (d == 0) part[k][rg * Q::R + r] = make_float2(rr[j], ii[j]);
        }
        __syncthreads();
        const bool owner = threadIdx.x < Q::N;
        float yr = 0.0f, yi = 0.0f;
        if (owner) {
            const float2 p8 = part[8][threadIdx.x];   // X first, then k = 0..7 (R11 order)
            yr = p8.x;
            yi = p8.y;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                yr += part[k][threadIdx.x].x;
                yi += part[k][threadIdx.x].y;
            }
        }
        const int orow = owner ? threadIdx.x : 0;
        const float sg = (a.dagger && orow >= NV) ? -1.0f : 1.0f;
        // new vector -> this CTA's shared buffer (read by the peers next apply) and to HBM
        unsigned char *gout = (t & 1) ? g0 : g1;
        store_site<P, NV>(vbuf[pin ^ 1] - (size_t)0, 0, orow, owner, sg * yr, sg * yi, red, K::THREADS, -1);
        __syncthreads();
        for (int e = threadIdx.x; e < Q::VCH; e += K::THREADS)
            *reinterpret_cast<uint4 *>(gout + (size_t)site * Q::VREC + e * 16) =
                *reinterpret_cast<const uint4 *>(vbuf[pin ^ 1] + e * 16);
        cluster_sync_all();   // everybody's new vector is visible; everybody finished reading the old one
    }
}

template <cd_precision P, int NV>
struct ClusterNW {   // warps per site-CTA (0: the site's links do not fit in one SM's registers)
    static constexpr int nw = (P == CD_FP32 && NV == 24) ? 27 : (P == CD_FP16 && NV == 24) ? 27
                            : (P == CD_FP16 && NV == 32) ? 24 : 0;
};

template <cd_precision P, int NV, int NW>
cudaError_t launch_cluster_chain_t(const ApplyArgs &a, int n, cudaStream_t s)
{
    using K = ClusterCfg<P, NV, NW>;
    if (a.g.V > 16 || a.halo) return cudaErrorNotSupported;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(dslash_cluster_chain<P, NV, NW>,
                                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.g.V);
    cfg.blockDim = dim3(K::THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)a.g.V;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, dslash_cluster_chain<P, NV, NW>, &cfg);
    if (e != cudaSuccess) return e;
    if (nclusters < 1) return cudaErrorCooperativeLaunchTooLarge;
    ApplyArgs aa = a;
    int nn = n;
    void *args[] = {&aa, &nn};
    count_launch();
    return cudaLaunchKernelExC(&cfg, (const void *)dslash_cluster_chain<P, NV, NW>, args);
}

// ------------------------------------------------------------------ CLUSTER push chain (V <= 16, fp32, Nvec 24)
// The whole lattice in ONE thread-block cluster, one CTA per site, the site's nine 48 x 48
// complex matrices in registers for all n applies; no L2 traffic and no polling:
//   * thread (row group rg of 3 rows, chunk q of 24) holds L_k(x)[3 rg + j][chunk q] for all
//     nine hops and j = 0..2 (108 floats): one 16-B shared load of a neighbour record per hop
//     feeds three rows (a shared load costs 4 wavefronts however many lanes share its address,
//     so the earlier one-row-per-thread layout was bound by the shared-memory data pipe);
//     complex MACs on the packed FP32 pipe (cmac2x);
//   * a warp = 4 row groups x 8 chunks; the three warps of a "triple" cover all 24 chunks of the
//     same 12 rows: xor-shuffle reduce-scatter over the 8 lanes, the three partials meet in
//     shared memory behind one 96-thread named barrier;
//   * thread (row r12 of the triple, destination dd) then pushes y(x)[row] to destination dd --
//     this CTA's own slot 8 and the receive slots of the CTAs that read x as a neighbour -- with
//     st.async into their shared memory; one thread per (triple, destination) adds the triple's
//     arrival + 96 bytes of expected transaction on the destination's mbarrier (remote
//     arrive.expect_tx): barrier 0 (own slot) completes when the 4 own triples arrived and 384
//     bytes landed, barrier 1 (all remote slots) when 4 triples of every producing neighbour
//     did -- no local re-arming;
//   * a warp waits for its own record (X hop), then once for the remote records; the X math
//     overlaps the remote wait; on all-extent-2 lattices the slot offsets are compile-time and
//     the +-mu hops share one load.
// Receive slots (consumer c, hop k): k = 8 or L_mu = 1 -> slot 8 (own); L_mu = 2 -> slot 2 mu
// for both hops (x + mu = x - mu: one record); else slot k.  Flow control needs no extra signal:
// a thread pushes epoch t+1 only after its warp received the complete epoch-t records of every
// neighbour, and every triple of a neighbour pushes its part of epoch t only after it finished
// reading epoch t-1 (the slot parity being overwritten) and observed both barrier phases of
// epoch t-1 -- the neighbour relation is symmetric.  The per-triple partial buffer alternates
// with the apply parity (its barrier orders a rewrite after every read of two applies ago).
// Measured (2^4, Nvec 24): 0.841 us per apply = 40.3 % of 8 TB/s, LL-register chain 0.915-0.934.
template <int NV>
struct CPushCfg {
    static constexpr int N = 2 * NV;
    static constexpr int NT = 4;              // warp triples (12 warps)
    static constexpr int RPT = N / NT;        // rows per triple (12): 4 row groups of 3 rows
    static constexpr int THREADS = 32 * 3 * NT;
    static_assert(NV == 24, "layout: 24 chunks per row = 3 warps x 8 lanes, 16 row groups of 3 rows");
};

// wait for a phase, return 0 as a value the dependent shared loads use in their address
__device__ __forceinline__ uint32_t mbar_wait_dep(uint32_t bar, uint32_t parity)
{
    uint32_t z;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "@!p bra WAIT_%=;\n"
        "mov.u32 %0, 0;\n"
        "}\n" : "=r"(z) : "r"(bar), "r"(parity) : "memory");
    return z;
}
// shared load the compiler may schedule freely (ordered only through its address operand)
__device__ __forceinline__ uint4 lds128_dep(uint32_t a)
{
    uint4 v;
    asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, unsigned cta)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
    return r;
}
__device__ __forceinline__ void st_async_f2(uint32_t dst, float a, float b, uint32_t bar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                 ::"r"(dst), "f"(a), "f"(b), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_remote(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

template <int NV, bool TRACE, bool ALL2>
__global__ void __launch_bounds__(CPushCfg<NV>::THREADS, 1) dslash_cpush(ApplyArgs a, int n)
{
    using Q = Cfg<CD_FP32, NV>;
    using K = CPushCfg<NV>;
    __shared__ __align__(16) float2 rec[2][9][K::N];          // receive slots by epoch parity
    __shared__ __align__(8) uint64_t bar[2][2];                // [parity][0: own slot 8, 1: all remote slots]
    __shared__ __align__(16) float part[2][K::NT][3][K::RPT * 2];   // [parity][triple][member][row of triple, re/im]

    const long long c_entry = clock64();
    const int site = (int)cluster_rank();   // grid == one cluster of V CTAs
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tw = warp / 3, m = warp - 3 * tw;                // triple, member (chunk block)
    const int rq = lane >> 3, d = lane & 7;
    const int rg = tw * 4 + rq;                                // row group: rows 3 rg .. 3 rg + 2
    const int q = m * 8 + d;                                   // the 16-B chunk (complex 2q, 2q+1) of this lane
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    unsigned char *const g0 = const_cast<unsigned char *>(static_cast<const unsigned char *>(a.in));
    unsigned char *const g1 = static_cast<unsigned char *>(a.out);
    int x[4];
    decode(a.g, site, x);

    // push role after the triple reduction: row (of the triple's 12) r12, destination dd
    const int tid3 = m * 32 + lane, r12 = tid3 >> 3, dd = tid3 & 7;
    const int prow = tw * K::RPT + r12;
    int dst_cta = -1, dst_slot = 0;   // destination dd: own slot 8, then per mu the -mu / +mu readers
    {
        int i = 0;
        if (dd == i) dst_cta = site, dst_slot = 8;
        i++;
#pragma unroll
        for (int mu = 0; mu < 4; mu++) {
            const int L = sel4(a.g.L, mu);
            if (L >= 2) {   // x - mu reads us through hop 2mu (L = 2: x - mu = x + mu, one push)
                if (dd == i) dst_cta = neighbour(a.g, x, site, 2 * mu + 1), dst_slot = 2 * mu;
                i++;
            }
            if (L >= 3) {   // x + mu reads us through hop 2mu + 1
                if (dd == i) dst_cta = neighbour(a.g, x, site, 2 * mu), dst_slot = 2 * mu + 1;
                i++;
            }
        }
    }
    const uint32_t rec_s = (uint32_t)__cvta_generic_to_shared(&rec[0][0][0]);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar[0][0]);
    uint32_t dst_rec = 0, dst_bar = 0;   // cluster addresses of slot dst_slot / its barrier, parity 0
    if (dst_cta >= 0) {
        dst_rec = mapa_u32(rec_s + (uint32_t)(dst_slot * K::N + prow) * 8u, (unsigned)dst_cta);
        dst_bar = mapa_u32(bar_s + (dst_slot == 8 ? 0u : 8u), (unsigned)dst_cta);
    }
    // the slot each hop reads (kseq order: X first), and the number of remote producers
    uint64_t slotmask = 0;   // 4 bits per hop position
    int nremote = 0;
#pragma unroll
    for (int i = 0; i < 9; i++) {
        const int k = kseq(i);
        int s = 8;
        if (k < 8) {
            const int L = sel4(a.g.L, k >> 1);
            s = L == 1 ? 8 : (L == 2 ? (k & ~1) : k);
            if (L >= 3 || (L == 2 && !(k & 1))) nremote++;
        }
        slotmask |= (uint64_t)s << (4 * i);
    }

    uint32_t hoff[8];   // byte offset of the receive slot of hop position i = 1..8 (k = i - 1)
#pragma unroll
    for (int i = 1; i < 9; i++)   // ALL2 (every extent 2, the 2^4 coarsest grid): compile-time slots 2 mu
        hoff[i - 1] = (ALL2 ? (uint32_t)((i - 1) & ~1) : ((uint32_t)(slotmask >> (4 * i)) & 15u)) * (uint32_t)(K::N * 8);
    // links: chunk q of rows 3 rg + j, all nine hops (108 floats per thread)
    uint4 Lc[9][3];
    // dagger: tau3 on the input (columns of chunks q >= Nvec/2) and on the output (rows >= Nvec)
    // folded into the register-resident links -- no sign work per apply
#pragma unroll
    for (int i = 0; i < 9; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            uint4 l = ld_stream(links + ((size_t)site * 9 + kseq(i)) * Q::MREC + (3 * rg + j) * Q::ROWB + q * 16);
            const bool neg = a.dagger && ((q * 2 >= NV) != (3 * rg + j >= NV));
            Lc[i][j] = neg ? neg_chunk<false>(l) : l;
        }
    if (threadIdx.x == 0) {   // own: 4 producer triples; remote: 4 per producing neighbour
        for (int p = 0; p < 2; p++) {
            mbar_init(&bar[p][0], K::NT);
            mbar_init(&bar[p][1], K::NT * (nremote > 0 ? nremote : 1));
        }
        fence_mbar_init();
    }
    cluster_sync_all();

    long long *const tr = (TRACE && a.trace && blockIdx.x == 0 && lane == 0) ? a.trace : nullptr;
    if (TRACE && tr && warp == 0) {   // prologue: rows 39 (kernel entry), 38 (after the cluster barrier)
        tr[39 * 1024] = c_entry;
        tr[38 * 1024] = clock64();
    }
    for (int t = 0; t < n; t++) {
        const int par = t & 1;
        const bool trt = TRACE && tr && t < 1024 && warp < 8;
        if (trt) tr[(4 * warp) * 1024 + t] = clock64();
        unsigned long long A[3] = {0ull, 0ull, 0ull}, B[3] = {0ull, 0ull, 0ull};   // packed, see cmac2x
        // The triple's arrival (+ its 96 expected bytes) on each destination's barrier for epoch
        // t + 1 goes out early, off the epilogue: it needs no data, and it cannot reach a phase
        // before its time -- the destination finished with that barrier's previous phase (epoch
        // t - 1) before it pushed the epoch-t record this warp has just received, and the new
        // phase still needs every byte of epoch t + 1 to complete.
        const bool early_arrive = t + 1 < n && dst_cta >= 0 && r12 == 0;
        if (t == 0) {   // the input is ready at launch
            if (early_arrive) mbar_arrive_expect_tx_remote(dst_bar + 16u, K::RPT * 8u);
#pragma unroll
            for (int i = 0; i < 9; i++) {
                const uint4 v = ld_nc(g0 + (size_t)neighbour(a.g, x, site, kseq(i)) * Q::VREC + q * 16);
#pragma unroll
                for (int j = 0; j < 3; j++) cmac2x(Lc[i][j], v, A[j], B[j]);
            }
        } else {
            const uint32_t ph = ((t - 1) >> 1) & 1;
            uint32_t z = mbar_wait_dep(bar_s + (uint32_t)(par * 2) * 8u, ph);
            if (TRACE && trt) tr[(4 * warp + 1) * 1024 + t] = clock64();
            {   // X: own slot 8, while the remote records are in flight
                const uint4 v = lds128_dep(rec_s + (uint32_t)((par * 9 + 8) * K::N) * 8u + z + (uint32_t)q * 16u);
#pragma unroll
                for (int j = 0; j < 3; j++) cmac2x(Lc[0][j], v, A[j], B[j]);
            }
            if (nremote > 0) {
                // (not ordered after the X math: forcing that order cost 3 %, the scheduler overlaps
                // the X FFMA2s with the wait on its own)
                z = mbar_wait_dep(bar_s + (uint32_t)(par * 2 + 1) * 8u, ph);
                if (TRACE && trt) tr[(32 + warp) * 1024 + t] = clock64() + z;
            }
            // per-thread part of the address in one register, per-hop part uniform (slot offsets
            // precomputed): one LDS [R + UR] per hop
            const uint32_t tb = rec_s + (uint32_t)q * 16u + z + (uint32_t)(par * 9 * K::N * 8);
            if (early_arrive) mbar_arrive_expect_tx_remote(dst_bar + (uint32_t)(par ^ 1) * 16u + z, K::RPT * 8u);
            uint4 v[8];
#pragma unroll
            for (int i = 1; i < 9; i++) v[i - 1] = lds128_dep(tb + hoff[i - 1]);
#pragma unroll
            for (int i = 1; i < 9; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) cmac2x(Lc[i][j], v[i - 1], A[j], B[j]);
        }
        if (trt) tr[(4 * warp + 2) * 1024 + t] = clock64();
        // 6 values (re, im of rows 3 rg + j) summed over the 8 lanes d by a reduce-scatter:
        // lane d ends with value d (values 6, 7 are padding)
        float w[8];
#pragma unroll
        for (int j = 0; j < 3; j++) {
            w[2 * j] = __uint_as_float((uint32_t)A[j]) - __uint_as_float((uint32_t)(B[j] >> 32));
            w[2 * j + 1] = __uint_as_float((uint32_t)(A[j] >> 32)) + __uint_as_float((uint32_t)B[j]);
        }
        w[6] = 0.0f;
        w[7] = 0.0f;
        {
            const bool hi = d & 4;   // keep values 4..7 (hi) or 0..3
            float u[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const float send = hi ? w[e] : w[e + 4];
                const float keep = hi ? w[e + 4] : w[e];
                u[e] = keep + shfl_xor(send, 4);
            }
            const bool h2 = d & 2;   // keep u[2..3] or u[0..1]
            float u2[2];
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float send = h2 ? u[e] : u[e + 2];
                const float keep = h2 ? u[e + 2] : u[e];
                u2[e] = keep + shfl_xor(send, 2);
            }
            const bool h1 = d & 1;
            const float send = h1 ? u2[0] : u2[1];
            const float keep = h1 ? u2[1] : u2[0];
            const float r = keep + shfl_xor(send, 1);   // value index d
            if (d < 6) part[par][tw][m][rq * 6 + d] = r;   // row 3 rq + d / 2 of the triple, re/im = d & 1
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + tw), "r"(96) : "memory");   // the triple's three members
        {
            const float *pp = &part[par][tw][0][2 * r12];
            float yr = pp[0] + pp[K::RPT * 2] + pp[2 * K::RPT * 2];
            float yi = pp[1] + pp[K::RPT * 2 + 1] + pp[2 * K::RPT * 2 + 1];
            if (t + 1 < n && dst_cta >= 0) {
                const uint32_t off = (uint32_t)(par ^ 1);
                st_async_f2(dst_rec + off * 9u * K::N * 8u, yr, yi, dst_bar + off * 16u);
            }
            if (t >= n - 2 && dd == 0) {   // the caller sees the last two iterates (x / y ping-pong)
                unsigned char *gout = (t & 1) ? g0 : g1;
                reinterpret_cast<float2 *>(gout + (size_t)site * Q::VREC)[prow] = make_float2(yr, yi);
            }
        }
        if (trt) tr[(4 * warp + 3) * 1024 + t] = clock64();
    }
    cluster_sync_all();   // no CTA leaves while a peer may still address its shared memory
}

template <cd_precision P, int NV>
cudaError_t launch_cpush_t(const ApplyArgs &a, int n, cudaStream_t s)
{
    if constexpr (P != CD_FP32 || NV != 24) {
        return cudaErrorNotSupported;
    } else {
        using K = CPushCfg<NV>;
        // st.async needs a real cluster (>= 2 CTAs); one cluster holds at most 16 CTAs
        if (a.g.V < 2 || a.g.V > 16 || a.halo || a.g.split) return cudaErrorNotSupported;
        const bool all2 = a.g.L[0] == 2 && a.g.L[1] == 2 && a.g.L[2] == 2 && a.g.L[3] == 2;
        const void *fns[2][2] = {{(const void *)dslash_cpush<NV, false, false>, (const void *)dslash_cpush<NV, false, true>},
                                 {(const void *)dslash_cpush<NV, true, false>, (const void *)dslash_cpush<NV, true, true>}};
        const void *fn = fns[a.trace ? 1 : 0][all2 ? 1 : 0];
        static bool attr = false;
        if (!attr) {
            for (int i = 0; i < 4; i++) {
                cudaError_t e = cudaFuncSetAttribute(fns[i >> 1][i & 1], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e != cudaSuccess) return e;
            }
            attr = true;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)a.g.V);
        cfg.blockDim = dim3(K::THREADS);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)a.g.V;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        // the occupancy query costs ~10 us of host time: cache it per (kernel, cluster size, device)
        static std::mutex mu;
        static std::map<std::tuple<const void *, int, int>, int> fits;
        int dev = 0;
        cudaGetDevice(&dev);
        const auto key = std::make_tuple(fn, a.g.V, dev);
        int nclusters = -1;
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = fits.find(key);
            if (it != fits.end()) nclusters = it->second;
        }
        if (nclusters < 0) {
            cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
            if (e != cudaSuccess) return e;
            std::lock_guard<std::mutex> lk(mu);
            fits[key] = nclusters;
        }
        if (nclusters < 1) return cudaErrorCooperativeLaunchTooLarge;
        ApplyArgs aa = a;
        int nn = n;
        void *args[] = {&aa, &nn};
        count_launch();
        return cudaLaunchKernelExC(&cfg, fn, args);
    }
}

// ------------------------------------------------------------------ halo term (multi-rank)
// One CTA per face site: y(x) = partial(x) + sum over remote hops L_k(x) v_halo, then the
// final store (fp16: whole-site re-quantisation).  Neighbour records come from the receive
// buffer in the wire order of DESIGN.md R13: a +mu hop reads block B of mu (sent by the +mu
// neighbour from its x_mu = 0 face), a -mu hop reads block A.
template <cd_precision P, int NV>
__global__ void __launch_bounds__(32 * (2 * NV / Cfg<P, NV>::R)) dslash_halo(ApplyArgs a)
{
    using Q = Cfg<P, NV>;
    constexpr int NWARP = Q::N / Q::R;
    constexpr int PREC = Q::F16 ? 4 * Q::N : 8 * Q::N;   // wire payload record
    __shared__ float red[32];
    const int site = a.face_sites[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = lane / Q::D, d = lane % Q::D;
    const int row = warp * Q::R + r;
    const unsigned char *links = static_cast<const unsigned char *>(a.links);
    const unsigned char *recv = static_cast<const unsigned char *>(a.recv);
    int x[4];
    decode(a.g, site, x);
    float re = 0.0f, im = 0.0f;
    for (int k = 0; k < 8; k++) {
        if (!remote_hop(a.g, x, k)) continue;
        const int mu = k >> 1;
        const int blk = (k & 1) ? 0 : 1;
        int o3[3], n = 0;
        for (int nu = 0; nu < 4; nu++)
            if (nu != mu) o3[n++] = nu;
        const int f = (x[o3[2]] * a.g.L[o3[1]] + x[o3[1]]) * a.g.L[o3[0]] + x[o3[0]];
        const unsigned char *vrec = recv + a.g.blk_off[mu][blk] + (size_t)f * PREC;
        const unsigned char *m = links + ((size_t)site * 9 + k) * Q::MREC;
        if constexpr (P == CD_FP32) {
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                const int q = d + Q::D * c;
                uint4 vq = ld_nc(vrec + q * 16);
                if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                cmac2(ld_nc(m + row * Q::ROWB + q * 16), vq, re, im);
            }
        } else {
            float ra = 0.f, rb = 0.f, ia = 0.f, ib = 0.f;
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                const int q = d + Q::D * c;
                uint4 vq = ld_nc(vrec + q * 16);
                if (a.dagger && q * Q::CPC >= NV) vq = neg_chunk<true>(vq);
                hmac4(ld_nc(m + row * Q::ROWB + q * 16), vq, ra, rb, ia, ib);
            }
            const float sv = *reinterpret_cast<const float *>(recv + a.g.blk_off[mu][blk] + (size_t)a.g.F[mu] * PREC +
                                                              (size_t)f * 4);
            const float sc = ld_nc_f32(m + Q::MSCALE) * sv;
            re = fmaf(ra - rb, sc, re);
            im = fmaf(ia + ib, sc, im);
        }
    }
#pragma unroll
    for (int m = Q::D / 2; m >= 1; m >>= 1) {
        re += shfl_xor(re, m);
        im += shfl_xor(im, m);
    }
    const bool owner = (d == 0);
    if (owner) {
        const float2 p = a.scratch[(size_t)site * Q::N + row];
        re += p.x;
        im += p.y;
    }
    const float sg = (a.dagger && row >= NV) ? -1.0f : 1.0f;
    store_site<P, NV>(static_cast<unsigned char *>(a.out), site, row, owner, sg * re, sg * im, red, 32 * NWARP, -1);
}

// ------------------------------------------------------------------ halo pack
// One launch for all split dims: blockIdx.y = (mu, block) pair index,
// threads over the face's 16-B payload chunks and then its scales (fp16).  The destination of
// block (mu, blk) is d.dst[mu][blk]: the local send buffer (NCCL / copy transports) or, for the
// peer transport, the receive slot in the neighbour's window -- the pack IS the transfer (stores
// over NVLink), and each CTA then bumps the receiver's arrival counter for that block.
template <cd_precision P, int NV>
__global__ void halo_pack(const unsigned char *field, PackDst d, KGeom g, int4 pairs)
{
    const int pi = blockIdx.y >> 1, blk = blockIdx.y & 1;
    const int mu = pi == 0 ? pairs.x : (pi == 1 ? pairs.y : (pi == 2 ? pairs.z : pairs.w));
    pack_block<P, NV>(field, pd_dst(d, mu, blk), g, mu, blk, blockIdx.x * blockDim.x + threadIdx.x,
                      gridDim.x * blockDim.x);
    signal_block(pd_flag(d, mu, blk));
}

// ------------------------------------------------------------------ variant table
struct VDesc {
    int kind;  // 0 = ring (kw = matrices per stage), 1 = fg (kw hops per warp, wr row-warps)
    int kw, wr;
};

template <cd_precision P, int NV>
struct Variants;
template <>
struct Variants<CD_FP32, 24> {
    static constexpr int n = 11;
    static constexpr VDesc v[n] = {{0, 1, 0}, {1, 1, 1}, {1, 1, 2}, {1, 1, 3}, {1, 3, 2}, {1, 3, 4},
                                   {1, 3, 6}, {1, 9, 3}, {1, 9, 6}, {1, 9, 12}, {0, 3, 0}};
};
template <>
struct Variants<CD_FP32, 32> {
    static constexpr int n = 9;
    static constexpr VDesc v[n] = {{0, 1, 0}, {1, 1, 1}, {1, 1, 2}, {1, 3, 2}, {1, 3, 4},
                                   {1, 3, 8}, {1, 9, 4}, {1, 9, 8}, {0, 3, 0}};
};
template <>
struct Variants<CD_FP16, 24> {
    // (a ring m9 with two consumer groups splitting each stage's hops was parity-green but measured 6 %
    // slower at M5 under the power cap and removed: profiles/r02/ring_g2_rejected.txt)
    static constexpr int n = 12;
    static constexpr VDesc v[n] = {{0, 1, 0}, {1, 3, 6}, {1, 9, 6}, {1, 1, 1}, {1, 1, 2}, {1, 3, 2},
                                   {1, 3, 3}, {1, 9, 2}, {1, 9, 3}, {0, 3, 0}, {0, 9, 0}, {0, 103, 0}};
};
template <>
struct Variants<CD_FP16, 32> {
    static constexpr int n = 9;
    static constexpr VDesc v[n] = {{0, 1, 0}, {1, 3, 8}, {1, 9, 8}, {1, 1, 1}, {1, 1, 2},
                                   {1, 3, 2}, {1, 3, 4}, {1, 9, 4}, {0, 3, 0}};
};

template <cd_precision P, int NV>
inline const char *variant_name_t(int id)
{
    static char names[16][48];
    static bool init = false;
    if (!init) {
        for (int i = 0; i < Variants<P, NV>::n; i++) {
            const VDesc &v = Variants<P, NV>::v[i];
            if (v.kind == 0 && v.kw > 100)   // two CTAs per SM
                snprintf(names[i], 48, "ring_tma_m%dx2_%s_nv%d", v.kw % 100, P == CD_FP32 ? "f32" : "f16", NV);
            else if (v.kind == 0) snprintf(names[i], 48, "ring_tma_m%d_%s_nv%d", v.kw, P == CD_FP32 ? "f32" : "f16", NV);
            else snprintf(names[i], 48, "fg_kw%d_wr%d_%s_nv%d", v.kw, v.wr, P == CD_FP32 ? "f32" : "f16", NV);
        }
        init = true;
    }
    return (id >= 0 && id < Variants<P, NV>::n) ? names[id] : nullptr;
}

inline cudaError_t launch_ex(const void *fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, void **args,
                             bool cooperative = false)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    at[1].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (or the launch fails)
    at[1].val.cooperative = cooperative ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    count_launch();
    return cudaLaunchKernelExC(&cfg, fn, args);
}

// Host: a 2-D TMA tensor map over a field of V records of `rec` bytes (32-bit elements, one record per
// row, box = one row) for the producer's gather4.  The driver entry point is looked up once through
// the runtime (no link-time libcuda dependency); false if unavailable (the bulk-copy path is used).
inline bool encode_rows_map(CUtensorMap *tm, const void *base, int rec, int V)
{
    typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = []() -> EncodeFn {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    if (!fn || V <= 0 || rec % 16 || rec > 1024) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)(rec / 4), (cuuint64_t)V};   // 32-bit elements: a row <= 256 of them
    const cuuint64_t strides[1] = {(cuuint64_t)rec};
    const cuuint32_t box[2] = {(cuuint32_t)(rec / 4), 1};
    const cuuint32_t estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <cd_precision P, int NV, int MPS>
cudaError_t launch_ring(const ApplyArgs &a, cudaStream_t s, bool pdl, int num_sms)
{
    using RC = RingCfg<P, NV, MPS>;
    static_assert(RC::S >= 2, "ring needs at least two stages");
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(dslash_ring<P, NV, MPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, RC::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    // 2-CTA clusters (148 SMs = 74 TPC pairs): st.async (the site-id handoff) needs a cluster of >= 2
    int grid = a.g.V < RC::CPS * num_sms ? a.g.V : RC::CPS * num_sms;
    grid = (grid + 1) & ~1;
    ApplyArgs aa = a;
    static const int rexp = getenv("CD_RING_EXP") ? atoi(getenv("CD_RING_EXP")) : 0;   // diagnostic only
    // nine matrices per stage: a 2-D tensor map of `in` ([V][VREC] bytes) lets the producer gather four
    // vector records per instruction for every site without remote hops (CD_RING_GATHER=0: nine bulk copies)
    const bool gather_on = !(getenv("CD_RING_GATHER") && atoi(getenv("CD_RING_GATHER")) == 0);
    CUtensorMap tmv;
    memset(&tmv, 0, sizeof(tmv));
    const bool g4 = (RC::M == 9 || RC::M == 3) && gather_on && encode_rows_map(&tmv, a.in, Cfg<P, NV>::VREC, a.g.V);
    int slot = (a.seq & (RC::SLOTS - 1)) | (rexp << 8) | ((g4 ? 1 : 0) << 16);
    void *args[] = {&aa, &slot, &tmv};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(RC::THREADS);
    cfg.dynamicSmemBytes = RC::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 2;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    count_launch();
    return cudaLaunchKernelExC(&cfg, (const void *)dslash_ring<P, NV, MPS>, args);
}

template <cd_precision P, int NV, int MPS>
cudaError_t launch_ringh(const ApplyArgs &a, cudaStream_t s, bool pdl, int num_sms)
{
    using RC = RingCfg<P, NV, MPS>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(dslash_ringh<P, NV, MPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, RC::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    int grid = a.g.V < RC::CPS * num_sms ? a.g.V : RC::CPS * num_sms;
    grid = (grid + 1) & ~1;   // 2-CTA clusters: st.async (the site-id handoff)
    ApplyArgs aa = a;
    const bool gather_on = !(getenv("CD_RING_GATHER") && atoi(getenv("CD_RING_GATHER")) == 0);
    CUtensorMap tmv;
    memset(&tmv, 0, sizeof(tmv));
    const bool g4 = (RC::M == 9 || RC::M == 3) && gather_on && encode_rows_map(&tmv, a.in, Cfg<P, NV>::VREC, a.g.V);
    int slot = (a.seq & (RC::SLOTS - 1)) | ((g4 ? 1 : 0) << 16);
    void *args[] = {&aa, &slot, &tmv};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(RC::THREADS);
    cfg.dynamicSmemBytes = RC::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 2;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    count_launch();
    return cudaLaunchKernelExC(&cfg, (const void *)dslash_ringh<P, NV, MPS>, args);
}

template <cd_precision P, int NV, int KW, int WR>
cudaError_t launch_fg(const ApplyArgs &a, cudaStream_t s, bool pdl)
{
    using F = FgCfg<P, NV, KW, WR>;
    ApplyArgs aa = a;
    void *args[] = {&aa};
    return launch_ex((const void *)dslash_fg<P, NV, KW, WR>, dim3((unsigned)(a.g.V * F::NRB)), dim3(F::THREADS), 0, s,
                     pdl, args);
}

template <cd_precision P, int NV, int KW, int WR>
cudaError_t launch_chain_t(const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms)
{
    using F = FgCfg<P, NV, KW, WR>;
    if constexpr (F::SPLIT16) {
        return cudaErrorNotSupported;
    } else {
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dslash_chain<P, NV, KW, WR>, F::THREADS, 0);
        if (e != cudaSuccess) return e;
        if ((int64_t)a.g.V * F::NRB > (int64_t)per_sm * num_sms) return cudaErrorCooperativeLaunchTooLarge;
        ApplyArgs aa = a;
        int nn = n;
        unsigned bb = base;
        void *args[] = {&aa, &nn, &bb};
        return launch_ex((const void *)dslash_chain<P, NV, KW, WR>, dim3((unsigned)(a.g.V * F::NRB)), dim3(F::THREADS),
                         0, s, false, args, true);
    }
}

template <cd_precision P, int NV, int I>
cudaError_t dispatch_chain(int id, const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms, int *nrb)
{
    if constexpr (I >= Variants<P, NV>::n) {
        return cudaErrorInvalidValue;
    } else {
        if (id == I) {
            constexpr VDesc v = Variants<P, NV>::v[I];
            if constexpr (v.kind == 0) {
                return cudaErrorNotSupported;
            } else {
                *nrb = FgCfg<P, NV, v.kw, v.wr>::NRB;
                return launch_chain_t<P, NV, v.kw, v.wr>(a, n, base, s, num_sms);
            }
        }
        return dispatch_chain<P, NV, I + 1>(id, a, n, base, s, num_sms, nrb);
    }
}

template <cd_precision P, int NV, int I>
cudaError_t dispatch_llchain(int id, const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int num_sms)
{
    if constexpr (I >= Variants<P, NV>::n) {
        return cudaErrorInvalidValue;
    } else {
        if (id == I) {
            constexpr VDesc v = Variants<P, NV>::v[I];
            if constexpr (v.kind == 0) return cudaErrorNotSupported;
            else return launch_llchain_t<P, NV, v.kw, v.wr>(a, n, base, s, num_sms);
        }
        return dispatch_llchain<P, NV, I + 1>(id, a, n, base, s, num_sms);
    }
}

template <cd_precision P, int NV, int I>
cudaError_t dispatch_variant(int id, const ApplyArgs &a, cudaStream_t s, bool pdl, int num_sms)
{
    if constexpr (I >= Variants<P, NV>::n) {
        return cudaErrorInvalidValue;
    } else {
        if (id == I) {
            constexpr VDesc v = Variants<P, NV>::v[I];
            if constexpr (v.kind == 0) return launch_ring<P, NV, v.kw>(a, s, pdl, num_sms);
            else return launch_fg<P, NV, v.kw, v.wr>(a, s, pdl);
        }
        return dispatch_variant<P, NV, I + 1>(id, a, s, pdl, num_sms);
    }
}

template <cd_precision P, int NV>
cudaError_t launch_halo_t(const ApplyArgs &a, cudaStream_t s)
{
    if (a.n_face == 0) return cudaSuccess;
    using Q = Cfg<P, NV>;
    ApplyArgs aa = a;
    void *args[] = {&aa};
    return launch_ex((const void *)dslash_halo<P, NV>, dim3(a.n_face), dim3(32 * (Q::N / Q::R)), 0, s, false, args);
}

template <cd_precision P, int NV>
cudaError_t launch_pack_t(const void *field, const PackDst &d, const KGeom &g, cudaStream_t s)
{
    int4 pairs = make_int4(0, 0, 0, 0);
    int np = 0;
    int *pp = &pairs.x;
    for (int mu = 0; mu < 4; mu++)
        if ((g.split >> mu) & 1) pp[np++] = mu;
    if (np == 0) return cudaSuccess;
    const unsigned char *f = static_cast<const unsigned char *>(field);
    PackDst dd = d;
    KGeom gg = g;
    void *args[] = {&f, &dd, &gg, &pairs};
    return launch_ex((const void *)halo_pack<P, NV>, dim3(kPutCtas, 2 * np), dim3(256), 0, s, false, args);
}

}  // namespace cd

// Per-(P, NV) entry points, defined in the instantiation units.
#define CD_INSTANTIATE(P, NV, TAG)                                                                                 \
    namespace cd {                                                                                                \
    cudaError_t launch_dslash_##TAG(int id, const ApplyArgs &a, cudaStream_t s, bool pdl, int sms)                \
    {                                                                                                             \
        return dispatch_variant<P, NV, 0>(id, a, s, pdl, sms);                                                    \
    }                                                                                                             \
    cudaError_t launch_halo_##TAG(const ApplyArgs &a, cudaStream_t s) { return launch_halo_t<P, NV>(a, s); }      \
    cudaError_t launch_ringh_##TAG(const ApplyArgs &a, cudaStream_t s, bool pdl, int sms, int mps)                \
    {                                                                                                             \
        if (mps == 9) {                                                                                           \
            if constexpr (RingCfg<P, NV, 9>::S >= 2) return launch_ringh<P, NV, 9>(a, s, pdl, sms);                \
            else return cudaErrorNotSupported;                                                                    \
        }                                                                                                         \
        if (mps == 103) {                                                                                         \
            if constexpr (RingCfg<P, NV, 103>::S >= 2) return launch_ringh<P, NV, 103>(a, s, pdl, sms);            \
            else return launch_ringh<P, NV, 3>(a, s, pdl, sms);                                                   \
        }                                                                                                         \
        return launch_ringh<P, NV, 3>(a, s, pdl, sms);                                                            \
    }                                                                                                             \
    cudaError_t launch_fgh_##TAG(const ApplyArgs &a, cudaStream_t s, bool pdl)                                    \
    {                                                                                                             \
        ApplyArgs aa = a;                                                                                         \
        void *args[] = {&aa};                                                                                     \
        const void *fn = P == CD_FP32 ? (const void *)dslash_fgh<NV> : (const void *)dslash_fgh16<NV>;            \
        return launch_ex(fn, dim3((unsigned)(a.g.V * (2 * NV / 16))), dim3(288), 0, s, pdl, args);                \
    }                                                                                                             \
    cudaError_t launch_compress_##TAG(const void *full, void *comp, int64_t nsites, cudaStream_t s)               \
    {                                                                                                             \
        count_launch();                                                                                           \
        links_compress_kernel<P, NV><<<(unsigned)(nsites * 5), 256, 0, s>>>(                                      \
            static_cast<const unsigned char *>(full), static_cast<unsigned char *>(comp), nsites * 5);             \
        return cudaGetLastError();                                                                                \
    }                                                                                                             \
    cudaError_t launch_hermdev_##TAG(const void *full, const KGeom &g, float *dev, cudaStream_t s,                \
                                     const void *lhalo, const int64_t *lo)                                        \
    {                                                                                                             \
        count_launch();                                                                                           \
        const unsigned char *fu = static_cast<const unsigned char *>(full);                                      \
        const unsigned char *lh = static_cast<const unsigned char *>(lhalo);                                     \
        const int64_t z[4] = {0, 0, 0, 0};                                                                        \
        const int64_t *o = lo ? lo : z;                                                                           \
        if constexpr (P == CD_FP32)                                                                               \
            links_herm_dev_kernel<NV><<<(unsigned)(g.V * 4), 256, 0, s>>>(fu, g, dev, lh, o[0], o[1], o[2], o[3]); \
        else                                                                                                      \
            links_herm_dev16_kernel<NV><<<(unsigned)(g.V * 4), 256, 0, s>>>(fu, g, dev, lh, o[0], o[1], o[2], o[3]); \
        return cudaGetLastError();                                                                                \
    }                                                                                                             \
    cudaError_t launch_fgh_halo_##TAG(const ApplyArgs &a, cudaStream_t s)                                         \
    {                                                                                                             \
        if (a.n_face == 0) return cudaSuccess;                                                                    \
        count_launch();                                                                                           \
        dslash_fgh_halo<P, NV><<<(unsigned)a.n_face, 32 * (2 * NV / Cfg<P, NV>::R), 0, s>>>(a);                    \
        return cudaGetLastError();                                                                                \
    }                                                                                                             \
    cudaError_t launch_lhalo_pack_##TAG(const void *comp, void *send, const KGeom &g, const int64_t *o,           \
                                        cudaStream_t s)                                                           \
    {                                                                                                             \
        int4 pairs = make_int4(0, 0, 0, 0);                                                                       \
        int np = 0;                                                                                               \
        for (int mu = 0; mu < 4; mu++)                                                                            \
            if ((g.split >> mu) & 1) (&pairs.x)[np++] = mu;                                                       \
        if (np == 0) return cudaSuccess;                                                                          \
        count_launch();                                                                                           \
        lhalo_pack_kernel<P, NV><<<dim3(296, np), 256, 0, s>>>(static_cast<const unsigned char *>(comp),          \
                                                               static_cast<unsigned char *>(send), g, pairs, o[0], \
                                                               o[1], o[2], o[3]);                                 \
        return cudaGetLastError();                                                                                \
    }                                                                                                             \
    cudaError_t launch_chain_##TAG(int id, const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int sms,     \
                                   int *nrb)                                                                      \
    {                                                                                                             \
        if (id > LLREG_CHAIN_ID0 && id < LLREG_CHAIN_ID0 + 100) {                                                    \
            *nrb = 0;                                                                                             \
            return dispatch_llreg<P, NV>(id - LLREG_CHAIN_ID0 - 1, a, n, base, s, sms);                             \
        }                                                                                                         \
        if (id >= LL_CHAIN_ID0 && id < LL_CHAIN_ID0 + Variants<P, NV>::n) {                                       \
            *nrb = 0;                                                                                             \
            return dispatch_llchain<P, NV, 0>(id - LL_CHAIN_ID0, a, n, base, s, sms);                             \
        }                                                                                                         \
        if (id == LLWARP_CHAIN_ID) {                                                                              \
            *nrb = 0;                                                                                             \
            return launch_llwarp_t<P, NV>(a, n, base, s, sms);                                                    \
        }                                                                                                         \
        if (id == CPUSH_CHAIN_ID) {                                                                               \
            *nrb = 0;                                                                                             \
            return launch_cpush_t<P, NV>(a, n, s);                                                                \
        }                                                                                                         \
        if (id == CLUSTER_CHAIN_ID) {                                                                             \
            *nrb = 0;                                                                                             \
            if constexpr (ClusterNW<P, NV>::nw > 0)                                                               \
                return launch_cluster_chain_t<P, NV, ClusterNW<P, NV>::nw>(a, n, s);                              \
            else                                                                                                  \
                return cudaErrorNotSupported;                                                                     \
        }                                                                                                         \
        return dispatch_chain<P, NV, 0>(id, a, n, base, s, sms, nrb);                                             \
    }                                                                                                             \
    cudaError_t launch_pack_##TAG(const void *f, const PackDst &d, const KGeom &g, cudaStream_t s)                \
    {                                                                                                             \
        return launch_pack_t<P, NV>(f, d, g, s);                                                                  \
    }                                                                                                             \
    int variant_count_##TAG() { return Variants<P, NV>::n; }                                                      \
    const char *variant_name_##TAG(int id) { return variant_name_t<P, NV>(id); }                                  \
    int variant_kind_##TAG(int id, int *kw, int *wr)                                                              \
    {                                                                                                             \
        if (id < 0 || id >= Variants<P, NV>::n) return -1;                                                        \
        *kw = Variants<P, NV>::v[id].kw;                                                                          \
        *wr = Variants<P, NV>::v[id].wr;                                                                          \
        return Variants<P, NV>::v[id].kind;                                                                       \
    }                                                                                                             \
    }
