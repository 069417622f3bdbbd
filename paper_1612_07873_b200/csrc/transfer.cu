// transfer.cu -- prolongator and restrictor of adaptive geometric multigrid (
// PAPER.md:108-121 §3.4, kernels §6.6).
//
// Aggregates are B0 x B1 x B2 x B3 hypercubes of fine sites; fine site x belongs to the
// coarse site floor(x / B).  A fine site has nf = Ns * Nc dofs r = s*Nc + a; chirality
// chi(r) = r >= nf/2 (spins s >= Ns/2, R20; P:121 fn. 1).  Basis W[sf][r][k] (fp32
// complex, k < Nvec) = the prolongator's columns, block-orthonormalised per (aggregate, chi).
//
//   prolong : vf(sf, r) = sum_k W(sf, r, k) vc(agg(sf), chi(r)*Nvec + k)           (gather)
//   restrict: vc(X, chi*Nvec + k) = sum_{sf in X, chi(r) = chi} conj(W(sf, r, k)) vf(sf, r)
//                                                             (restrictor = P^dagger)
//
// Both are streams over W (HBM bound: 8 * nf * Nvec bytes per fine site vs 8 * nf of vector).
// Lane mapping for both: 16-lane row groups, lane g owns the k pair (2g, 2g+1) -- one float4 of a
// basis row, rows contiguous in HBM, so a row group reads a whole row per instruction.
//   prolong : (a gather, no reduction across sites) 4-lane groups per fine site instead, so every
//             lane is busy for Nvec 24 (see prolong_kernel); CTA per (aggregate, split).
//   restrict: "a single aggregate ... mapped exactly to a thread block" -- here to one CTA
//             or a thread-block CLUSTER of CL CTAs (small coarse grids fill the GPU); each lane
//             accumulates its k pair for both chiralities over its rows in registers, then a fixed-
//             order reduction: xor-shuffle -> shared memory across warps -> DSMEM across the
//             cluster (no atomics, bitwise reproducible; the paper used a CUB block reduce).
#include <cuda_fp16.h>
#include <cstdint>

#include "cd_internal.h"
#include "device_common.cuh"

namespace cd {

__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// fine site of block index b in aggregate xc
__device__ __forceinline__ int fine_site(const TGeom &t, const int xc[4], int b)
{
    int bx[4];
    bx[0] = b % t.B[0];
    b /= t.B[0];
    bx[1] = b % t.B[1];
    b /= t.B[1];
    bx[2] = b % t.B[2];
    bx[3] = b / t.B[2];
    const int x0 = xc[0] * t.B[0] + bx[0], x1 = xc[1] * t.B[1] + bx[1];
    const int x2 = xc[2] * t.B[2] + bx[2], x3 = xc[3] * t.B[3] + bx[3];
    return ((x3 * t.Lf[2] + x2) * t.Lf[1] + x1) * t.Lf[0] + x0;
}

// ------------------------------------------------------------------ prolongator
// 4-lane row groups: lane q owns float4 chunks q, q+4, ... of a basis row (NV/8 of them: every lane
// busy for Nvec 24 and 32, each load instruction of a group reads 64 contiguous bytes).  A group
// takes 2 rows of one chirality at a time; a 2-step transposing shuffle reduction leaves row r0 in
// lanes {0,1} and row r0+1 in lanes {2,3}.  A warp works on 8 fine sites at once.
template <int NV, cd_precision PC, int NFH>
__global__ void __launch_bounds__(256, 2) prolong_kernel(const float4 *__restrict__ W, const unsigned char *__restrict__ vc,
                                                      float2 *__restrict__ vf, TGeom t)
{
    constexpr int HG = NV / 2;   // float4 per basis row
    constexpr int KPL = NV / 8;  // float4 per lane per row
    const int q = threadIdx.x & 3;
    // work item = (aggregate, fine site b of the aggregate), aggregate-major: one item per group,
    // 64 consecutive items per CTA, so a CTA streams the basis rows of one (part of an) aggregate
    // and its groups share the coarse vector through L1.
    const int64_t item = (int64_t)blockIdx.x * 64 + (threadIdx.x >> 2);
    const bool valid = item < (int64_t)t.c.V * t.Bvol;
    const int sc = valid ? (int)(item / t.Bvol) : 0;
    const int b0 = valid ? (int)(item - (int64_t)sc * t.Bvol) : 0;
    int xc[4];
    decode(t.c, sc, xc);
    float4 v0[KPL], v1[KPL];   // this lane's k pairs of both chiralities
    if constexpr (PC == CD_FP32) {
        const float4 *r = reinterpret_cast<const float4 *>(vc + (size_t)sc * (8 * 2 * NV));
#pragma unroll
        for (int j = 0; j < KPL; j++) {
            v0[j] = __ldg(r + q + 4 * j);
            v1[j] = __ldg(r + HG + q + 4 * j);
        }
    } else {
        const unsigned char *rec = vc + (size_t)sc * (4 * 2 * NV + 16);
        const float s = __ldg(reinterpret_cast<const float *>(rec + 4 * 2 * NV));
        auto cvt = [s](uint2 h) {
            const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&h.x));
            const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&h.y));
            return make_float4(a.x * s, a.y * s, b.x * s, b.y * s);
        };
#pragma unroll
        for (int j = 0; j < KPL; j++) {
            v0[j] = cvt(__ldg(reinterpret_cast<const uint2 *>(rec) + q + 4 * j));
            v1[j] = cvt(__ldg(reinterpret_cast<const uint2 *>(rec) + HG + q + 4 * j));
        }
    }
    const int nf = t.nf, nfh = NFH > 0 ? NFH : t.nf >> 1;
    const int sf = fine_site(t, xc, b0);
    const float4 *Wr = W + (size_t)sf * nf * HG + q;
    float2 *out = vf + (size_t)sf * nf;
    // two rows of chirality chi: unconditional loads (row index clamped), so the compiler can hoist
    // the loads of several chunks ahead of their math (bytes in flight decide this kernel's speed)
    auto chunk = [&](int chi, int r0) {
        const float4 *v = chi == 0 ? v0 : v1;
        float4 w[2][KPL];
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int rr = chi * nfh + min(r0 + i, nfh - 1);
#pragma unroll
            for (int j = 0; j < KPL; j++) w[i][j] = __ldg(Wr + (size_t)rr * HG + 4 * j);
        }
        float pr[2], pi[2];
#pragma unroll
        for (int i = 0; i < 2; i++) {
            pr[i] = 0.f, pi[i] = 0.f;
#pragma unroll
            for (int j = 0; j < KPL; j++) {
                pr[i] += w[i][j].x * v[j].x - w[i][j].y * v[j].y + w[i][j].z * v[j].z - w[i][j].w * v[j].w;
                pi[i] += w[i][j].x * v[j].y + w[i][j].y * v[j].x + w[i][j].z * v[j].w + w[i][j].w * v[j].z;
            }
        }
        const bool up = (q & 2) != 0;   // lanes 2,3 keep row r0+1
        const float sr = up ? pr[0] : pr[1], si = up ? pi[0] : pi[1];
        float kr = up ? pr[1] : pr[0], ki = up ? pi[1] : pi[0];
        kr += __shfl_xor_sync(0xffffffffu, sr, 2);
        ki += __shfl_xor_sync(0xffffffffu, si, 2);
        kr += __shfl_xor_sync(0xffffffffu, kr, 1);
        ki += __shfl_xor_sync(0xffffffffu, ki, 1);
        const int r = r0 + (up ? 1 : 0);
        if (valid && (q & 1) == 0 && r < nfh) out[chi * nfh + r] = make_float2(kr, ki);
    };
    if constexpr (NFH > 0) {
#pragma unroll
        for (int chi = 0; chi < 2; chi++)
#pragma unroll
            for (int r0 = 0; r0 < NFH; r0 += 2) chunk(chi, r0);
    } else {
#pragma unroll
        for (int chi = 0; chi < 2; chi++)
#pragma unroll 4
            for (int r0 = 0; r0 < nfh; r0 += 2) chunk(chi, r0);
    }
}

// ------------------------------------------------------------------ restrictor
template <int NV, cd_precision PC, int CL>
__global__ void __launch_bounds__(256) restrict_kernel(const float4 *__restrict__ W, const float2 *__restrict__ vf,
                                                       unsigned char *__restrict__ vc, TGeom t)
{
    constexpr int HG = NV / 2;
    constexpr int RB = 8;   // rows in flight per lane
    __shared__ float4 part[8][2][16];
    __shared__ __align__(16) float4 red[2][16];
    const int rank = CL > 1 ? (int)cluster_rank() : 0;
    const int sc = blockIdx.x / CL;
    const int warp = threadIdx.x >> 5, half = (threadIdx.x >> 4) & 1, g = threadIdx.x & 15;
    const int rg = (rank * 8 + warp) * 2 + half;
    int xc[4];
    decode(t.c, sc, xc);
    float4 a[2] = {f4zero(), f4zero()};
    const int nf = t.nf, nfh = nf >> 1;
    if (g < HG) {
        for (int b = rg; b < t.Bvol; b += CL * 16) {
            const int sf = fine_site(t, xc, b);
            const float4 *Wr = W + (size_t)sf * nf * HG + g;
            const float2 *f = vf + (size_t)sf * nf;
#pragma unroll
            for (int chi = 0; chi < 2; chi++) {
                for (int r0 = chi * nfh; r0 < (chi + 1) * nfh; r0 += RB) {
                    float4 w[RB];
                    float2 x[RB];
#pragma unroll
                    for (int i = 0; i < RB; i++) {
                        const bool ok = r0 + i < (chi + 1) * nfh;
                        w[i] = ok ? __ldg(Wr + (size_t)(r0 + i) * HG) : f4zero();
                        x[i] = ok ? __ldg(f + r0 + i) : make_float2(0.f, 0.f);
                    }
#pragma unroll
                    for (int i = 0; i < RB; i++) {   // conj(w) * x
                        a[chi].x += w[i].x * x[i].x + w[i].y * x[i].y;
                        a[chi].y += w[i].x * x[i].y - w[i].y * x[i].x;
                        a[chi].z += w[i].z * x[i].x + w[i].w * x[i].y;
                        a[chi].w += w[i].z * x[i].y - w[i].w * x[i].x;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int chi = 0; chi < 2; chi++) {
        a[chi].x += __shfl_xor_sync(0xffffffffu, a[chi].x, 16);
        a[chi].y += __shfl_xor_sync(0xffffffffu, a[chi].y, 16);
        a[chi].z += __shfl_xor_sync(0xffffffffu, a[chi].z, 16);
        a[chi].w += __shfl_xor_sync(0xffffffffu, a[chi].w, 16);
        if (half == 0) part[warp][chi][g] = a[chi];
    }
    __syncthreads();
    float4 tot = f4zero();
    const int chi = threadIdx.x >> 4;   // threads 0..31: (chi, g)
    if (threadIdx.x < 32) {
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const float4 p = part[w][chi][g];
            tot.x += p.x, tot.y += p.y, tot.z += p.z, tot.w += p.w;
        }
    }
    if constexpr (CL > 1) {
        if (threadIdx.x < 32) red[chi][g] = tot;
        cluster_sync_all();
        if (rank == 0 && threadIdx.x < 32) {
            tot = f4zero();
            for (int c = 0; c < CL; c++) {
                const uint4 u = ld_dsmem(&red[chi][g], (unsigned)c);
                tot.x += __uint_as_float(u.x), tot.y += __uint_as_float(u.y);
                tot.z += __uint_as_float(u.z), tot.w += __uint_as_float(u.w);
            }
        }
        cluster_sync_all();   // peers' shared memory stays alive until rank 0 has read it
        if (rank != 0) return;
    }
    if (threadIdx.x >= 32) return;
    if constexpr (PC == CD_FP32) {
        if (g < HG) reinterpret_cast<float4 *>(vc + (size_t)sc * (8 * 2 * NV))[chi * HG + g] = tot;
    } else {
        // fp16 record: DESIGN.md R12 (s = max |x|, q = fp16_rn(x / s), IEEE division)
        float m = g < HG ? fmaxf(fmaxf(fabsf(tot.x), fabsf(tot.y)), fmaxf(fabsf(tot.z), fabsf(tot.w))) : 0.f;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        unsigned char *rec = vc + (size_t)sc * (4 * 2 * NV + 16);
        if (g < HG) {
            __half2 h0, h1;
            if (m > 0.f) {
                h0 = __halves2half2(__float2half_rn(__fdiv_rn(tot.x, m)), __float2half_rn(__fdiv_rn(tot.y, m)));
                h1 = __halves2half2(__float2half_rn(__fdiv_rn(tot.z, m)), __float2half_rn(__fdiv_rn(tot.w, m)));
            } else {
                h0 = h1 = __halves2half2(__float2half_rn(0.f), __float2half_rn(0.f));
            }
            uint2 u;
            u.x = *reinterpret_cast<unsigned *>(&h0);
            u.y = *reinterpret_cast<unsigned *>(&h1);
            reinterpret_cast<uint2 *>(rec)[chi * HG + g] = u;
        }
        if (threadIdx.x == 0) *reinterpret_cast<float *>(rec + 4 * 2 * NV) = m;
    }
}

// ------------------------------------------------------------------ setup: block orthonormalisation
// Per (aggregate, chirality): modified Gram-Schmidt in column order ("QR decomposition on
// these blocks"), fp64 sums over fp32 storage, fixed-order block reductions; in place.
__device__ double2 block_sum2(double2 v, double2 *buf, double2 *bc)
{
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 s = make_double2(0.0, 0.0);
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s.x += buf[w].x, s.y += buf[w].y;
        *bc = s;
    }
    __syncthreads();
    return *bc;
}

template <int NV>
__global__ void __launch_bounds__(256) orthonormalise_kernel(float2 *__restrict__ W, TGeom t, int *fail)
{
    extern __shared__ int sfs[];   // fine site of every block index b
    __shared__ double2 buf[8];
    __shared__ double2 bc;
    const int sc = blockIdx.x >> 1, chi = blockIdx.x & 1;
    int xc[4];
    decode(t.c, sc, xc);
    for (int b = threadIdx.x; b < t.Bvol; b += blockDim.x) sfs[b] = fine_site(t, xc, b);
    __syncthreads();
    const int nfh = t.nf >> 1, M = t.Bvol * nfh;
    auto row = [&](int m) -> float2 * {
        const int b = m / nfh, r = m - b * nfh;
        return W + ((size_t)sfs[b] * t.nf + chi * nfh + r) * NV;
    };
    for (int k = 0; k < NV; k++) {
        double2 p = make_double2(0.0, 0.0);
        for (int m = threadIdx.x; m < M; m += blockDim.x) {
            const float2 v = row(m)[k];
            p.x += (double)v.x * v.x + (double)v.y * v.y;
        }
        const double nrm0 = block_sum2(p, buf, &bc).x;
        for (int j = 0; j < k; j++) {   // v_k -= <q_j, v_k> q_j
            p = make_double2(0.0, 0.0);
            for (int m = threadIdx.x; m < M; m += blockDim.x) {
                const float2 qj = row(m)[j], v = row(m)[k];
                p.x += (double)qj.x * v.x + (double)qj.y * v.y;
                p.y += (double)qj.x * v.y - (double)qj.y * v.x;
            }
            const double2 d = block_sum2(p, buf, &bc);
            for (int m = threadIdx.x; m < M; m += blockDim.x) {
                float2 *rp = row(m);
                const float2 qj = rp[j], v = rp[k];
                rp[k] = make_float2((float)(v.x - (d.x * qj.x - d.y * qj.y)), (float)(v.y - (d.x * qj.y + d.y * qj.x)));
            }
        }
        p = make_double2(0.0, 0.0);
        for (int m = threadIdx.x; m < M; m += blockDim.x) {
            const float2 v = row(m)[k];
            p.x += (double)v.x * v.x + (double)v.y * v.y;
        }
        const double nrm = sqrt(block_sum2(p, buf, &bc).x);
        if (!(nrm > 1e-5 * sqrt(nrm0))) {   // DESIGN.md R21 (uniform decision: every thread sees nrm)
            if (threadIdx.x == 0) atomicExch(fail, 1);
            return;
        }
        for (int m = threadIdx.x; m < M; m += blockDim.x) {
            float2 *rp = row(m);
            const float2 v = rp[k];
            rp[k] = make_float2((float)(v.x / nrm), (float)(v.y / nrm));
        }
    }
}

__global__ void c128_to_c64_kernel(const double2 *__restrict__ in, float2 *__restrict__ out, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = make_float2((float)in[i].x, (float)in[i].y);
}

// ------------------------------------------------------------------ launchers
int restrict_cluster_size(const TGeom &t, int num_sms)
{
    int cl = 1;
    while (cl < 8 && (int64_t)t.c.V * cl < 4 * num_sms && t.Bvol >= cl * 2 * 16) cl *= 2;
    return cl;
}

template <int NV, cd_precision PC, int CL>
static cudaError_t launch_restrict_t(const void *W, const void *vf, void *vc, const TGeom &t, cudaStream_t s)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(t.c.V * CL));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = CL > 1 ? 1 : 0;
    count_launch();
    return cudaLaunchKernelEx(&cfg, restrict_kernel<NV, PC, CL>, static_cast<const float4 *>(W),
                              static_cast<const float2 *>(vf), static_cast<unsigned char *>(vc), t);
}

template <int NV, cd_precision PC>
static cudaError_t launch_restrict_p(int cl, const void *W, const void *vf, void *vc, const TGeom &t, cudaStream_t s)
{
    switch (cl) {
    case 1: return launch_restrict_t<NV, PC, 1>(W, vf, vc, t, s);
    case 2: return launch_restrict_t<NV, PC, 2>(W, vf, vc, t, s);
    case 4: return launch_restrict_t<NV, PC, 4>(W, vf, vc, t, s);
    case 8: return launch_restrict_t<NV, PC, 8>(W, vf, vc, t, s);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_restrict(cd_precision pc, int nvec, int cl, const void *W, const void *vf, void *vc, const TGeom &t,
                            cudaStream_t s)
{
    if (nvec == 24)
        return pc == CD_FP32 ? launch_restrict_p<24, CD_FP32>(cl, W, vf, vc, t, s)
                             : launch_restrict_p<24, CD_FP16>(cl, W, vf, vc, t, s);
    if (nvec == 32)
        return pc == CD_FP32 ? launch_restrict_p<32, CD_FP32>(cl, W, vf, vc, t, s)
                             : launch_restrict_p<32, CD_FP16>(cl, W, vf, vc, t, s);
    return cudaErrorInvalidValue;
}

template <int NV, cd_precision PC>
static void prolong_dispatch(const dim3 &grid, cudaStream_t s, const float4 *w, const unsigned char *c, float2 *f,
                             const TGeom &t)
{
    // compile-time rows per chirality for the common fine grids: Wilson (Ns 4, Nc 3) and a
    // coarse level of Nvec 24 / 32 as the fine grid (Ns 2)
    switch (t.nf / 2) {
    case 6: prolong_kernel<NV, PC, 6><<<grid, 256, 0, s>>>(w, c, f, t); break;
    case 24: prolong_kernel<NV, PC, 24><<<grid, 256, 0, s>>>(w, c, f, t); break;
    case 32: prolong_kernel<NV, PC, 32><<<grid, 256, 0, s>>>(w, c, f, t); break;
    default: prolong_kernel<NV, PC, 0><<<grid, 256, 0, s>>>(w, c, f, t); break;
    }
}

cudaError_t launch_prolong(cd_precision pc, int nvec, const void *W, const void *vc, void *vf, const TGeom &t,
                           cudaStream_t s)
{
    const dim3 grid((unsigned)(((int64_t)t.c.V * t.Bvol + 63) / 64));
    const float4 *w = static_cast<const float4 *>(W);
    const unsigned char *c = static_cast<const unsigned char *>(vc);
    float2 *f = static_cast<float2 *>(vf);
    count_launch();
    if (nvec == 24) {
        if (pc == CD_FP32) prolong_dispatch<24, CD_FP32>(grid, s, w, c, f, t);
        else prolong_dispatch<24, CD_FP16>(grid, s, w, c, f, t);
    } else if (nvec == 32) {
        if (pc == CD_FP32) prolong_dispatch<32, CD_FP32>(grid, s, w, c, f, t);
        else prolong_dispatch<32, CD_FP16>(grid, s, w, c, f, t);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_orthonormalise(int nvec, void *W, const TGeom &t, int *fail, cudaStream_t s)
{
    const size_t smem = sizeof(int) * (size_t)t.Bvol;
    const dim3 grid((unsigned)(2 * t.c.V)), block(256);
    count_launch();
    if (nvec == 24) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(orthonormalise_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        orthonormalise_kernel<24><<<grid, block, smem, s>>>(static_cast<float2 *>(W), t, fail);
    } else if (nvec == 32) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(orthonormalise_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        orthonormalise_kernel<32><<<grid, block, smem, s>>>(static_cast<float2 *>(W), t, fail);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_c128_to_c64(const void *in, void *out, int64_t n, cudaStream_t s)
{
    count_launch();
    c128_to_c64_kernel<<<1184, 256, 0, s>>>(static_cast<const double2 *>(in), static_cast<float2 *>(out), n);
    return cudaGetLastError();
}

}  // namespace cd
