// ATOMIC assembly: element kernel with warp-aggregated global atomics + node
// kernel (fh_atomic.cu).  Shares the TILED engine's numbering and node arrays.
#pragma once
#include "fh_tiled.cuh"

namespace fh {

struct AtomicState {
  const int32_t *tet_conn = nullptr, *hex_conn = nullptr;  // N new node ids per element, sorted by smallest id
  const void *tet_G = nullptr, *hex_G = nullptr;           // [6][n] metric components (S)
  int64_t n_tet = 0, n_hex = 0, V = 0;
  const uint8_t *cls = nullptr;  // per node: 0 updated, 1 updated + Robin, 2 Dirichlet (kept)
  const void *hA = nullptr, *hAT = nullptr;  // per node (S), Robin nodes only read
};

template <typename S>
void atomic_step(const TiledArgs<S> &g, const AtomicState &a, S *F, cudaStream_t s);
template <typename S>
void atomic_pack(const int32_t *elem, int64_t n, const double *G, double scale, const double *kf, S *out,
                 cudaStream_t s);

}  // namespace fh
