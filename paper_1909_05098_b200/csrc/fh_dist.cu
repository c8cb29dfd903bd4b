// Multi-GPU halo exchange: NCCL (loaded with dlopen when a multi-GPU engine
// attaches, so single-GPU use never touches it) and the pack / unpack kernels.
//
// Per step and rank (fh_api.cu tiled_run):
//   compute stream: interior tiles -> [wait halo(s-1)] -> boundary tiles -> pack
//   comm stream:    [wait pack] -> ncclGroup{Send/Recv per peer} -> unpack
// The interior tiles of step s+1 overlap the NCCL transfer of step s.
#include <dlfcn.h>

#include "fh_dist.h"

namespace fh {

namespace {
struct NcclApi {
  void *h = nullptr;
  int (*GetUniqueId)(NcclUniqueId *) = nullptr;
  int (*CommInitRank)(void **, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(void *) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*Recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*AllReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(int) = nullptr;
};
NcclApi g_nccl;
std::string g_nccl_path;  // preferred library file (nccl_set_library), tried before the sonames

void load_nccl() {
  if (g_nccl.h) return;
  // a libnccl.so.2 the process already holds (e.g. the one bundled with
  // PyTorch) is reused by soname; otherwise the preferred file comes first, so
  // that a framework imported LATER finds the version it was built against
  // under that soname instead of an older system copy
  const char *names[] = {g_nccl_path.empty() ? nullptr : g_nccl_path.c_str(), "libnccl.so.2", "libnccl.so"};
  if ((g_nccl.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD)) == nullptr)
    for (const char *n : names)
      if (n && (g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!g_nccl.h) fail(FH_ERR_DEVICE, std::string("cannot load NCCL: ") + dlerror());
  auto sym = [](const char *s) {
    void *p = dlsym(g_nccl.h, s);
    if (!p) fail(FH_ERR_DEVICE, std::string("NCCL symbol missing: ") + s);
    return p;
  };
  g_nccl.GetUniqueId = (int (*)(NcclUniqueId *))sym("ncclGetUniqueId");
  g_nccl.CommInitRank = (int (*)(void **, int, NcclUniqueId, int))sym("ncclCommInitRank");
  g_nccl.CommDestroy = (int (*)(void *))sym("ncclCommDestroy");
  g_nccl.GroupStart = (int (*)())sym("ncclGroupStart");
  g_nccl.GroupEnd = (int (*)())sym("ncclGroupEnd");
  g_nccl.Send = (int (*)(const void *, size_t, int, int, void *, cudaStream_t))sym("ncclSend");
  g_nccl.Recv = (int (*)(void *, size_t, int, int, void *, cudaStream_t))sym("ncclRecv");
  g_nccl.AllReduce = (int (*)(const void *, void *, size_t, int, int, void *, cudaStream_t))sym("ncclAllReduce");
  g_nccl.GetErrorString = (const char *(*)(int))sym("ncclGetErrorString");
}

void nccl_check(int rc, const char *what) {
  if (rc != 0) fail(FH_ERR_DEVICE, std::string(what) + ": " + g_nccl.GetErrorString(rc));
}

// ncclDataType_t / ncclRedOp_t values of nccl.h
constexpr int kNcclUint64 = 5, kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclMin = 3;
}  // namespace

void nccl_set_library(const char *path) { g_nccl_path = path ? path : ""; }

void nccl_unique_id(NcclUniqueId *id) {
  load_nccl();
  nccl_check(g_nccl.GetUniqueId(id), "ncclGetUniqueId");
}

void *nccl_comm_init(const NcclUniqueId &id, int rank, int world) {
  load_nccl();
  void *comm = nullptr;
  nccl_check(g_nccl.CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
  return comm;
}

void nccl_comm_destroy(void *comm) {
  if (comm && g_nccl.h) g_nccl.CommDestroy(comm);
}

void nccl_exchange(void *comm, const void *sendbuf, void *recvbuf, size_t elem, const std::vector<int32_t> &peers,
                   const std::vector<int64_t> &send_offs, const std::vector<int64_t> &recv_offs, cudaStream_t s) {
  const int dtype = elem == 4 ? kNcclFloat32 : kNcclFloat64;
  nccl_check(g_nccl.GroupStart(), "ncclGroupStart");
  for (size_t q = 0; q < peers.size(); ++q) {
    const size_t ns = (size_t)(send_offs[q + 1] - send_offs[q]), nr = (size_t)(recv_offs[q + 1] - recv_offs[q]);
    if (ns)
      nccl_check(g_nccl.Send((const char *)sendbuf + elem * send_offs[q], ns, dtype, peers[q], comm, s), "ncclSend");
    if (nr) nccl_check(g_nccl.Recv((char *)recvbuf + elem * recv_offs[q], nr, dtype, peers[q], comm, s), "ncclRecv");
  }
  nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd");
}

void nccl_min_u64(void *comm, unsigned long long *dev_value, cudaStream_t s) {
  nccl_check(g_nccl.AllReduce(dev_value, dev_value, 1, kNcclUint64, kNcclMin, comm, s), "ncclAllReduce");
}

template <typename S>
__global__ void k_gather_nodes(const S *__restrict__ T, const int32_t *__restrict__ nodes, int64_t n,
                               S *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = T[nodes[i]];
}

template <typename S>
__global__ void k_scatter_nodes(S *__restrict__ T, const int32_t *__restrict__ nodes, int64_t n,
                                const S *__restrict__ in) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) T[nodes[i]] = in[i];
}

template <typename S>
void halo_pack(const S *T, const int32_t *nodes, int64_t n, S *buf, cudaStream_t s) {
  if (n <= 0) return;
  k_gather_nodes<S><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(T, nodes, n, buf);
  FH_CUDA(cudaGetLastError());
}

template <typename S>
void halo_unpack(S *T, const int32_t *nodes, int64_t n, const S *buf, cudaStream_t s) {
  if (n <= 0) return;
  k_scatter_nodes<S><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(T, nodes, n, buf);
  FH_CUDA(cudaGetLastError());
}

template void halo_pack<float>(const float *, const int32_t *, int64_t, float *, cudaStream_t);
template void halo_pack<double>(const double *, const int32_t *, int64_t, double *, cudaStream_t);
template void halo_unpack<float>(float *, const int32_t *, int64_t, const float *, cudaStream_t);
template void halo_unpack<double>(double *, const int32_t *, int64_t, const double *, cudaStream_t);

}  // namespace fh
