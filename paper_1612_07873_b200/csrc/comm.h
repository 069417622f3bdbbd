// comm.h -- NCCL halo exchange (internal).
#pragma once
#include <string>

#include "cd_internal.h"

namespace cd {
int nccl_unique_id(uint8_t out[128], std::string &err);
int comm_create(const uint8_t id[128], int nranks, int rank, Comm **out, std::string &err);
void comm_destroy(Comm *c);
int comm_check(Comm *c, std::string &err);
int halo_exchange(cd_context *ctx, const cd_halo_plan &plan, cudaStream_t s, std::string &err);
// the same exchange between caller-given send / receive buffers laid out by `plan`
int halo_exchange_buf(cd_context *ctx, const cd_halo_plan &plan, const void *send, void *recv, cudaStream_t s,
                      std::string &err);
}  // namespace cd
