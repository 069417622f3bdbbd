// comm.h -- NCCL halo exchange (internal).
#pragma once
#include <string>

#include "cd_internal.h"

namespace cd {
int nccl_unique_id(uint8_t out[128], std::string &err);
int comm_create(const uint8_t id[128], int nranks, int rank, Comm **out, std::string &err);
void comm_destroy(Comm *c);
int comm_check(Comm *c, std::string &err);
int comm_create_self(Comm **out, std::string &err);   // 1-rank communicator (NCCL self send/recv)

// The transport an exchange on this context uses now (resolves CD_OPT_TRANSPORT = auto).
int transport_of(const cd_context *ctx);

// One vector-halo exchange (apply / dagger / compressed / even-odd stage), DESIGN.md §7:
//   halo_begin  -- where the pack kernel writes (send buffer, or the peers' windows) and which
//                  buffer the halo kernel reads; the peer transport advances the epoch;
//   halo_post   -- after the pack on the comm stream: NCCL group / device copy (peer: nothing,
//                  the pack was the transfer);
//   halo_finish -- on the compute stream before the halo kernel (peer: the wait kernel).
struct HaloX {
    PackDst pd;
    const void *recv;
    int transport;
    unsigned mask;          // blocks in flight, bit 2mu+blk
    unsigned long long target;
};
int halo_begin(cd_context *ctx, const cd_halo_plan &plan, HaloX *x, std::string &err);
int halo_post(cd_context *ctx, const cd_halo_plan &plan, const HaloX &x, cudaStream_t comm, std::string &err);
int halo_finish(cd_context *ctx, const HaloX &x, cudaStream_t s, std::string &err);

// A whole-buffer exchange between caller-given send / receive buffers laid out by `plan`
// (one-time link halo, multi-RHS faces), all on stream s.  NCCL / copy: direct; peer: chunked
// through the windows (put -> wait -> copy out per chunk).
int halo_exchange_buf(cd_context *ctx, const cd_halo_plan &plan, const void *send, void *recv, cudaStream_t s,
                      std::string &err);

// Peer windows: allocate + export this rank's window; map the neighbours' windows.
int peer_window_export(cd_context *ctx, size_t slot_bytes, unsigned char out[64], std::string &err);
int peer_connect(cd_context *ctx, const unsigned char *handles, int n, std::string &err);
void peer_release(cd_context *ctx);
int transport_check(cd_context *ctx, std::string &err);   // async transport faults (NCCL, peer timeouts)
}  // namespace cd
