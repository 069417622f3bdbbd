// comm.cpp -- NCCL point-to-point halo exchange (replaces the paper's pack -> D2H -> MPI ->
// H2D path, with device-to-device NCCL over NVLink / NVSwitch).
//
// libnccl.so.2 is opened with dlopen by soname, so the process uses the NCCL that PyTorch
// has already loaded (one NCCL per process) and the library has no link-time NCCL
// dependency.  Only the handful of entry points below are used.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cd_internal.h"
#include "comm.h"

namespace cd {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;

static bool load_nccl(std::string &err)
{
    if (g_nccl.h) return true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
        return false;
    }
#define SYM(field, name)                                                 \
    *reinterpret_cast<void **>(&g_nccl.field) = dlsym(h, name);          \
    if (!g_nccl.field) {                                                 \
        err = std::string("libnccl.so.2 lacks ") + name;                 \
        return false;                                                    \
    }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    // optional (NCCL >= 2.14): per-communicator CTA cap
    *reinterpret_cast<void **>(&g_nccl.CommInitRankConfig) = dlsym(h, "ncclCommInitRankConfig");
    SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    g_nccl.h = h;
    return true;
}

struct Comm {
    ncclComm_t comm = nullptr;
};

int nccl_unique_id(uint8_t out[128], std::string &err)
{
    if (!load_nccl(err)) return CD_ERR_NCCL;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) {
        err = std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r);
        return CD_ERR_NCCL;
    }
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return CD_OK;
}

int comm_create(const uint8_t id_bytes[128], int nranks, int rank, Comm **out, std::string &err)
{
    if (!load_nccl(err)) return CD_ERR_NCCL;
    ncclUniqueId id;
    memcpy(&id, id_bytes, 128);
    Comm *c = new Comm();
    ncclResult_t r;
    if (g_nccl.CommInitRankConfig) {
        // cap NCCL's CTAs (CD_NCCL_MAX_CTAS, default 4) so its send/recv kernels fit in the SMs the
        // persistent interior leaves free (CD_OPT_NCCL_SM_RESERVE, default 8): a halo of <= 1.6 MB
        // per rank does not need more, and the stencil keeps the rest of the GPU
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        const char *ev = getenv("CD_NCCL_MAX_CTAS");
        cfg.maxCTAs = ev ? atoi(ev) : 4;
        cfg.minCTAs = 1;
        r = g_nccl.CommInitRankConfig(&c->comm, nranks, id, rank, &cfg);
    } else {
        r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
    }
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r);
        delete c;
        return CD_ERR_NCCL;
    }
    *out = c;
    return CD_OK;
}

void comm_destroy(Comm *c)
{
    if (!c) return;
    if (c->comm) g_nccl.CommDestroy(c->comm);
    delete c;
}

int comm_check(Comm *c, std::string &err)
{
    if (!c) return CD_OK;
    ncclResult_t a = ncclSuccess;
    g_nccl.CommGetAsyncError(c->comm, &a);
    if (a != ncclSuccess && a != ncclInProgress) {
        err = std::string("NCCL async error: ") + g_nccl.GetErrorString(a);
        return CD_ERR_NCCL;
    }
    return CD_OK;
}

int comm_create_self(Comm **out, std::string &err)
{
    uint8_t id[128];
    int r = nccl_unique_id(id, err);
    if (r != CD_OK) return r;
    return comm_create(id, 1, 0, out, err);
}

int transport_of(const cd_context *c)
{
    if (c->transport != TR_AUTO) return c->transport;
    if (c->peer_ready) return TR_PEER;
    if (c->comm) return TR_NCCL;
    return TR_COPY;
}

int transport_check(cd_context *c, std::string &err)
{
    if (c->err_host && *reinterpret_cast<volatile int *>(c->err_host)) {
        err = "halo transport: an in-kernel wait for a neighbour's halo timed out (a rank stopped calling the "
              "collective applies, or the ranks issued them in different orders); the context's results are invalid";
        return CD_ERR_COMM;
    }
    return comm_check(c->comm, err);
}

static bool nccl_ok(ncclResult_t r, const char *what, std::string &err)
{
    if (r == ncclSuccess || r == ncclInProgress) return true;
    err = std::string(what) + ": " + g_nccl.GetErrorString(r);
    return false;
}

// NCCL / device-copy exchange of the blocks of `pl` (R13): block A of every split
// dim goes to the +mu neighbour's block A, block B to the -mu neighbour's block B.  Self
// neighbours (P_mu = 1 forced through the halo path) are a device copy under TR_COPY and an
// NCCL self send/recv under TR_NCCL (the real group code on one GPU).
static int exchange_nccl_copy(cd_context *ctx, const cd_halo_plan &pl, const unsigned char *send, unsigned char *recv,
                              int tr, cudaStream_t s, std::string &err)
{
    bool group = false;
    int rc = CD_OK;
    for (int mu = 0; mu < 4 && rc == CD_OK; mu++) {
        if (!((pl.split_mask >> mu) & 1)) continue;
        const size_t blk = (size_t)pl.block_bytes[mu];
        const int64_t offA = pl.block_offset[mu][0], offB = pl.block_offset[mu][1];
        const int up = pl.nbr_rank[mu][0], dn = pl.nbr_rank[mu][1];
        const bool self = up == ctx->rank && dn == ctx->rank;
        if (tr == TR_COPY) {
            if (!self) {
                err = "the device-copy transport only serves self exchanges (P_mu = 1); multi-rank contexts need "
                      "NCCL (nccl_id) or the peer transport (cd_context_peer_connect)";
                return CD_ERR_INVALID;
            }
            cudaError_t e = cudaMemcpyAsync(recv + offA, send + offA, 2 * blk, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) {
                err = std::string("halo self copy: ") + cudaGetErrorString(e);
                return CD_ERR_CUDA;
            }
            continue;
        }
        if (!ctx->comm) {
            err = "NCCL transport requested but the context has no communicator";
            return CD_ERR_INVALID;
        }
        if (!group) {
            if (!nccl_ok(g_nccl.GroupStart(), "ncclGroupStart", err)) return CD_ERR_NCCL;
            group = true;
        }
        // fixed issue order: sends (A -> +mu, B -> -mu) then receives (A <- -mu, B <- +mu); with
        // P_mu = 2 (or 1: self) both peers coincide and NCCL matches per-peer operations in order
        ncclComm_t cm = ctx->comm->comm;
        const int pu = self ? 0 : up, pd = self ? 0 : dn;   // a 1-rank communicator's self is rank 0
        if (!nccl_ok(g_nccl.Send(send + offA, blk, ncclUint8, pu, cm, s), "ncclSend", err) ||
            !nccl_ok(g_nccl.Send(send + offB, blk, ncclUint8, pd, cm, s), "ncclSend", err) ||
            !nccl_ok(g_nccl.Recv(recv + offA, blk, ncclUint8, pd, cm, s), "ncclRecv", err) ||
            !nccl_ok(g_nccl.Recv(recv + offB, blk, ncclUint8, pu, cm, s), "ncclRecv", err))
            rc = CD_ERR_NCCL;
    }
    if (group) {
        std::string e2;
        if (!nccl_ok(g_nccl.GroupEnd(), "ncclGroupEnd", e2) && rc == CD_OK) {
            err = e2;
            rc = CD_ERR_NCCL;
        }
    }
    return rc;
}

// ---- peer transport (CUDA IPC windows) -------------------------------------------------------
static unsigned split_blocks(const cd_halo_plan &pl)
{
    unsigned m = 0;
    for (int mu = 0; mu < 4; mu++)
        if ((pl.split_mask >> mu) & 1) m |= 3u << (2 * mu);
    return m;
}
static unsigned char *slot_of(unsigned char *win, size_t slot_bytes, uint64_t epoch)
{
    return win + kWinHeader + (size_t)(epoch & 1) * slot_bytes;
}
static unsigned long long *flag_of(unsigned char *win, int mu, int blk)
{
    return reinterpret_cast<unsigned long long *>(win) + 2 * mu + blk;
}

int halo_begin(cd_context *ctx, const cd_halo_plan &pl, HaloX *x, std::string &err)
{
    memset(x, 0, sizeof(*x));
    x->transport = transport_of(ctx);
    x->mask = split_blocks(pl);
    if (x->transport != TR_PEER) {
        for (int mu = 0; mu < 4; mu++)
            for (int b = 0; b < 2; b++)
                x->pd.dst[mu][b] = static_cast<unsigned char *>(ctx->send_buf) + pl.block_offset[mu][b];
        x->recv = ctx->recv_buf;
        return CD_OK;
    }
    if (!ctx->peer_ready) {
        err = "peer transport requested but cd_context_peer_connect has not been called";
        return CD_ERR_INVALID;
    }
    if ((size_t)pl.total_bytes > ctx->win_slot) {
        err = "halo larger than the peer window slot";
        return CD_ERR_INVALID;
    }
    const uint64_t e = ++ctx->epoch;
    for (int mu = 0; mu < 4; mu++)
        for (int b = 0; b < 2; b++) {
            if (!((x->mask >> (2 * mu + b)) & 1)) continue;
            unsigned char *pw = ctx->peer_win[mu][b];   // block A -> the +mu rank, block B -> the -mu rank
            x->pd.dst[mu][b] = slot_of(pw, ctx->win_slot, e) + pl.block_offset[mu][b];
            x->pd.flag[mu][b] = flag_of(pw, mu, b);
        }
    x->recv = slot_of(ctx->win, ctx->win_slot, e);
    x->target = (unsigned long long)kPutCtas * e;
    return CD_OK;
}

int halo_post(cd_context *ctx, const cd_halo_plan &pl, const HaloX &x, cudaStream_t comm, std::string &err)
{
    if (x.transport == TR_PEER) return CD_OK;
    return exchange_nccl_copy(ctx, pl, static_cast<const unsigned char *>(ctx->send_buf),
                              static_cast<unsigned char *>(ctx->recv_buf), x.transport, comm, err);
}

int halo_finish(cd_context *ctx, const HaloX &x, cudaStream_t s, std::string &err)
{
    if (x.transport != TR_PEER) return CD_OK;
    PeerWait w{reinterpret_cast<const unsigned long long *>(ctx->win), x.mask, x.target, ctx->err_dev,
               ctx->peer_timeout_ns};
    cudaError_t e = launch_peer_wait(w, s);
    if (e != cudaSuccess) {
        err = std::string("peer wait kernel: ") + cudaGetErrorString(e);
        return CD_ERR_CUDA;
    }
    return CD_OK;
}

int halo_exchange_buf(cd_context *ctx, const cd_halo_plan &pl, const void *send_, void *recv_, cudaStream_t s,
                      std::string &err)
{
    const unsigned char *send = static_cast<const unsigned char *>(send_);
    unsigned char *recv = static_cast<unsigned char *>(recv_);
    const int tr = transport_of(ctx);
    if (tr != TR_PEER) return exchange_nccl_copy(ctx, pl, send, recv, tr, s, err);
    if (!ctx->peer_ready) {
        err = "peer transport requested but cd_context_peer_connect has not been called";
        return CD_ERR_INVALID;
    }
    // chunk every block through its sub-window of a slot; the 2-slot reuse argument of
    // halo_begin holds because put -> wait -> copy-out of every chunk are stream-ordered on s
    const unsigned mask = split_blocks(pl);
    const int nblk = __builtin_popcount(mask);
    if (!nblk) return CD_OK;
    const int64_t sub = (int64_t)(ctx->win_slot / nblk) & ~int64_t(255);
    int64_t maxb = 0;
    for (int mu = 0; mu < 4; mu++) maxb = std::max<int64_t>(maxb, pl.block_bytes[mu]);
    const int64_t nch = (maxb + sub - 1) / sub;
    for (int64_t ch = 0; ch < nch; ch++) {
        const uint64_t e = ++ctx->epoch;
        PackDst pd{};
        const unsigned char *src[4][2] = {};
        unsigned char *mine[4][2] = {}, *dst[4][2] = {};
        int64_t len[4][2] = {};
        int i = 0;
        for (int mu = 0; mu < 4; mu++)
            for (int b = 0; b < 2; b++) {
                if (!((mask >> (2 * mu + b)) & 1)) continue;
                const int64_t off = ch * sub;
                len[mu][b] = std::max<int64_t>(0, std::min<int64_t>(sub, pl.block_bytes[mu] - off));
                src[mu][b] = send + pl.block_offset[mu][b] + off;
                pd.dst[mu][b] = slot_of(ctx->peer_win[mu][b], ctx->win_slot, e) + i * sub;
                pd.flag[mu][b] = flag_of(ctx->peer_win[mu][b], mu, b);
                mine[mu][b] = slot_of(ctx->win, ctx->win_slot, e) + i * sub;
                dst[mu][b] = recv + pl.block_offset[mu][b] + off;
                i++;
            }
        cudaError_t ce = launch_peer_put(src, len, mask, pd, s);
        PeerWait w{reinterpret_cast<const unsigned long long *>(ctx->win), mask, (unsigned long long)kPutCtas * e,
                   ctx->err_dev, ctx->peer_timeout_ns};
        if (ce == cudaSuccess) ce = launch_peer_wait(w, s);
        if (ce == cudaSuccess) ce = launch_copy_blocks(mine, dst, len, mask, s);
        if (ce != cudaSuccess) {
            err = std::string("peer bulk exchange: ") + cudaGetErrorString(ce);
            return CD_ERR_CUDA;
        }
    }
    return CD_OK;
}

int peer_window_export(cd_context *ctx, size_t slot_bytes, unsigned char out[64], std::string &err)
{
    if (!ctx->win) {
        const size_t slot = (std::max<size_t>(slot_bytes, 4096) + 255) & ~size_t(255);
        void *w = nullptr;
        cudaError_t e = cudaMalloc(&w, kWinHeader + 2 * slot);
        if (e == cudaSuccess) e = cudaMemset(w, 0, kWinHeader + 2 * slot);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();   // counters are zero before any peer can map them
        if (e != cudaSuccess) {
            if (w) cudaFree(w);
            err = std::string("peer window: ") + cudaGetErrorString(e);
            return CD_ERR_CUDA;
        }
        ctx->win = static_cast<unsigned char *>(w);
        ctx->win_slot = slot;
    }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, ctx->win);
    if (e != cudaSuccess) {
        err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
        return CD_ERR_CUDA;
    }
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(out, &h, 64);
    return CD_OK;
}

int peer_connect(cd_context *ctx, const unsigned char *handles, int n, std::string &err)
{
    if (!ctx->win) {
        err = "cd_context_peer_handle must be called (on every rank) before cd_context_peer_connect";
        return CD_ERR_INVALID;
    }
    if (n != ctx->nranks) {
        err = "need one 64-byte handle per rank";
        return CD_ERR_INVALID;
    }
    std::vector<unsigned char *> by_rank(ctx->nranks, nullptr);
    by_rank[ctx->rank] = ctx->win;
    for (int mu = 0; mu < 4; mu++)
        for (int d = 0; d < 2; d++) {
            if (!((ctx->kg.split >> mu) & 1)) continue;
            const int r = ctx->nbr_rank[mu][d];
            if (!by_rank[r]) {
                cudaIpcMemHandle_t h;
                memcpy(&h, handles + 64 * (size_t)r, 64);
                void *p = nullptr;
                cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
                if (e != cudaSuccess) {
                    err = std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(r) + "): " + cudaGetErrorString(e);
                    return CD_ERR_CUDA;
                }
                ctx->ipc_opened.push_back(p);
                by_rank[r] = static_cast<unsigned char *>(p);
            }
            ctx->peer_win[mu][d] = by_rank[r];
        }
    ctx->peer_ready = true;
    return CD_OK;
}

void peer_release(cd_context *ctx)
{
    for (void *p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    ctx->ipc_opened.clear();
    if (ctx->win) cudaFree(ctx->win);
    ctx->win = nullptr;
    ctx->peer_ready = false;
}

}  // namespace cd
