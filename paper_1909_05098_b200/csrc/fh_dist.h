// Multi-GPU halo exchange helpers (fh_dist.cu).
#pragma once
#include "fh_internal.h"

namespace fh {

struct NcclUniqueId {
  char internal[128];  // layout of ncclUniqueId (nccl.h, NCCL_UNIQUE_ID_BYTES)
};

// file to dlopen for NCCL before the default sonames (empty / null: sonames only); no effect once NCCL is loaded
void nccl_set_library(const char *path);
void nccl_unique_id(NcclUniqueId *id);
void *nccl_comm_init(const NcclUniqueId &id, int rank, int world);
void nccl_comm_destroy(void *comm);
// grouped point-to-point exchange of halo temperatures with every peer
void nccl_exchange(void *comm, const void *sendbuf, void *recvbuf, size_t elem, const std::vector<int32_t> &peers,
                   const std::vector<int64_t> &send_offs, const std::vector<int64_t> &recv_offs, cudaStream_t s);
void nccl_min_u64(void *comm, unsigned long long *dev_value, cudaStream_t s);

template <typename S>
void halo_pack(const S *T, const int32_t *nodes, int64_t n, S *buf, cudaStream_t s);
template <typename S>
void halo_unpack(S *T, const int32_t *nodes, int64_t n, const S *buf, cudaStream_t s);

}  // namespace fh
