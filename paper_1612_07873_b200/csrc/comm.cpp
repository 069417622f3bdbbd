// comm.cpp -- NCCL point-to-point halo exchange (replaces the paper's pack -> D2H -> MPI ->
// H2D path, with device-to-device NCCL over NVLink / NVSwitch).
//
// libnccl.so.2 is opened with dlopen by soname, so the process uses the NCCL that PyTorch
// has already loaded (one NCCL per process) and the library has no link-time NCCL
// dependency.  Only the handful of entry points below are used.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "cd_internal.h"
#include "comm.h"

namespace cd {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
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
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
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

// Exchange the packed faces (R13): block A of every split dim goes to the +mu
// neighbour's block A, block B to the -mu neighbour's block B.  Dims whose neighbours are
// this rank itself (P_mu = 1, forced through the halo path) are copied device-to-device.
int halo_exchange(cd_context *ctx, const cd_halo_plan &pl, cudaStream_t s, std::string &err)
{
    return halo_exchange_buf(ctx, pl, ctx->send_buf, ctx->recv_buf, s, err);
}

int halo_exchange_buf(cd_context *ctx, const cd_halo_plan &pl, const void *send_, void *recv_, cudaStream_t s,
                      std::string &err)
{
    const unsigned char *send = static_cast<const unsigned char *>(send_);
    unsigned char *recv = static_cast<unsigned char *>(recv_);
    bool group = false;
    for (int mu = 0; mu < 4; mu++) {
        if (!((pl.split_mask >> mu) & 1)) continue;
        const size_t blk = (size_t)pl.block_bytes[mu];
        const int64_t offA = pl.block_offset[mu][0], offB = pl.block_offset[mu][1];
        const int up = pl.nbr_rank[mu][0], dn = pl.nbr_rank[mu][1];
        if (up == ctx->rank && dn == ctx->rank) {
            cudaError_t e = cudaMemcpyAsync(recv + offA, send + offA, 2 * blk, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) {
                err = std::string("halo self copy: ") + cudaGetErrorString(e);
                return CD_ERR_CUDA;
            }
            continue;
        }
        if (!ctx->comm) {
            err = "halo exchange across ranks needs a NCCL communicator";
            return CD_ERR_NCCL;
        }
        if (!group) {
            g_nccl.GroupStart();
            group = true;
        }
        // fixed issue order: sends (A -> +mu, B -> -mu) then receives (A <- -mu, B <- +mu);
        // with P_mu = 2 both peers coincide and NCCL matches per-peer operations in order.
        g_nccl.Send(send + offA, blk, ncclUint8, up, ctx->comm->comm, s);
        g_nccl.Send(send + offB, blk, ncclUint8, dn, ctx->comm->comm, s);
        g_nccl.Recv(recv + offA, blk, ncclUint8, dn, ctx->comm->comm, s);
        g_nccl.Recv(recv + offB, blk, ncclUint8, up, ctx->comm->comm, s);
    }
    if (group) {
        ncclResult_t r = g_nccl.GroupEnd();
        if (r != ncclSuccess && r != ncclInProgress) {
            err = std::string("NCCL halo exchange: ") + g_nccl.GetErrorString(r);
            return CD_ERR_NCCL;
        }
    }
    return CD_OK;
}

}  // namespace cd
