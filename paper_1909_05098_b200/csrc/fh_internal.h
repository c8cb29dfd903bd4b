// Internal declarations shared by the engine's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <stdexcept>
#include <string>
#include <vector>

#include "fedheat_b200.h"

namespace fh {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error(code, msg); }

// record `code`'s printf-style message as the calling thread's fh_last_error(); returns code
int set_error(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));

#define FH_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t _e = (x);                                                                   \
    if (_e != cudaSuccess)                                                                  \
      ::fh::fail(FH_ERR_DEVICE, std::string(#x) + ": " + cudaGetErrorString(_e) + " (" + \
                                    __FILE__ + ":" + std::to_string(__LINE__) + ")");     \
  } while (0)

// --------------------------------------------------------------------------
// device buffer (owned)
template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) FH_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void upload(const T *h, size_t count, cudaStream_t s = 0) {
    alloc(count);
    if (count) FH_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T> &v, cudaStream_t s = 0) { upload(v.data(), v.size(), s); }
  void zero(cudaStream_t s = 0) {
    if (n) FH_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
  }
  size_t bytes() const { return sizeof(T) * n; }
};

// --------------------------------------------------------------------------
// property curve passed by value in kernel parameters (constant bank)
template <typename S>
struct Curve {
  int n;
  S x[FH_MAX_KNOTS];
  S y[FH_MAX_KNOTS];
  S slope[FH_MAX_KNOTS];  // slope[j] = (y[j+1]-y[j])/(x[j+1]-x[j]), computed in fp64 on the host
};

template <typename S>
struct Mat {
  Curve<S> rho, c, k, wb;
  int td_perf;  // wb curve active
  S wbcb;       // perfusion_rate * blood_specific_heat (constant perfusion)
  S cb, Ta, Qm;
};

constexpr int kMaxRegions = 4;

template <typename S>
struct MatSet {
  int n;
  Mat<S> m[kMaxRegions];
};

// fast-path clamped interpolation (FMA allowed).  Branch-free for the common
// one- and two-knot curves (the clamped end values are selected, so they are
// returned exactly like the reference's kernels.py:61-73).
template <typename S>
__device__ __forceinline__ S interp(const Curve<S> &c, S x) {
  if (c.n == 1) return c.y[0];
  if (c.n == 2) {
    S r = c.slope[0] * (x - c.x[0]) + c.y[0];
    r = (x >= c.x[1]) ? c.y[1] : r;
    return (x <= c.x[0]) ? c.y[0] : r;
  }
  if (x <= c.x[0]) return c.y[0];
  if (x >= c.x[c.n - 1]) return c.y[c.n - 1];
  int j = 0;
  while (c.x[j + 1] <= x) ++j;
  return c.slope[j] * (x - c.x[j]) + c.y[j];
}

// exact-path interpolation: kernels.py:61-73 with separate roundings
__device__ __forceinline__ double interp_rn(const Curve<double> &c, double x) {
  if (c.n == 1 || x <= c.x[0]) return c.y[0];
  if (x >= c.x[c.n - 1]) return c.y[c.n - 1];
  int j = 0;
  while (c.x[j + 1] <= x) ++j;
  return __dadd_rn(__dmul_rn(c.slope[j], __dsub_rn(x, c.x[j])), c.y[j]);
}

// Device-side bounds checks of the checked build (scripts/build_variant.sh
// checked "-DFH_CHECKS"; compute-sanitizer is not available on this GPU pool):
// a failed check prints the site and traps.  Compiled out otherwise.
#ifdef FH_CHECKS
#define FH_DEV_CHECK(cond, what)                                                                      \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("FH_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                       \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define FH_DEV_CHECK(cond, what) \
  do {                           \
  } while (0)
#endif

struct FailFlag {
  unsigned long long step;  // ~0ull = none
};

// --------------------------------------------------------------------------
// host-side partition of the mesh into tiles ("parts") for the fused step
struct PartitionInput {
  int64_t V, n_tet, n_hex;
  const double *xyz;
  const int64_t *tets, *hexes;
  const uint8_t *node_class;  // 0 free, 1 robin, 2 dirichlet
  int target_part_nodes;
  int batch;          // slots per batch (== kernel block size)
  int n_domains;      // top-level domain count (parts never straddle domains)
  int slab_axis;      // -1 RCB, else domains are slabs along this axis
  int hex_color = 0;  // 0: colour hexes only when not corner-unique; 1: always
  int first_touch = 0;  // renumber each tile's nodes in first-touch order of its batches (measured neutral)
  int tet_rows = 1;     // tet colour classes may touch a node up to tet_rows times (one accumulator row each)
};

struct Partition {
  int n_parts = 0;
  std::vector<int64_t> new_of_old, old_of_new;          // node permutation
  std::vector<int32_t> part_node_start;                  // P+1
  std::vector<int32_t> part_n_free;                      // nodes updated (free + robin)
  std::vector<int32_t> part_robin_start;                 // local index of first robin node
  std::vector<int32_t> part_tet_start, part_hex_start;   // P+1 each (slot ranges per kind, 4-aligned)
  std::vector<int32_t> part_tet_count, part_hex_count;   // real slots per part (rest is padding)
  std::vector<int32_t> part_halo_start, halo_nodes;      // halo (non-owned) nodes per part, sorted
  std::vector<uint16_t> tet_conn16, hex_conn16;          // tile-local node index per slot corner
  std::vector<int32_t> part_domain;                      // domain of each part
  std::vector<int32_t> domain_part_start;                // n_domains+1
  std::vector<int32_t> tet_slot_elem, hex_slot_elem;     // original element id per slot (-1 = padding)
  std::vector<int32_t> tet_conn, hex_conn;               // new node ids per slot
  std::vector<uint8_t> tet_rank, hex_rank;               // per slot corner phase (ranked mode)
  bool corner_unique = false;                            // phases == corner index
  int max_phase_tet = 0, max_phase_hex = 0;
  int max_part_nodes = 0;
  int max_local_nodes = 0;  // owned + halo
  int max_part_free = 0;
  // colouring: slots of one colour share no updated node; slots are sorted by
  // colour inside each tile, phase = colour index inside the batch
  bool colored_ok = false;
  bool hex_colored = false;  // hex slots colour-sorted (only when hexes are not corner-unique)
  int max_colors = 0, max_nph_tet = 0, max_nph_hex = 0;
  std::vector<uint8_t> tet_color, hex_color, tet_phase, hex_phase;
  std::vector<uint8_t> tet_batch_nph, hex_batch_nph;  // phases per batch (index = slot / B)
  // tet accumulator rows: 1, or 4 when every tile's tet colour classes were
  // built with up to 4 writes per node (row r = the write's rank in its
  // class; stored in bits 14-15 of tet_conn16, local index in bits 0-13)
  int tet_rows = 1;
  int batch = 256;  // slots per batch the slot ranges are aligned to
};

void build_partition(const PartitionInput &in, Partition &out);

// Multi-GPU halo bookkeeping for `rank` of `world` ranks; rank r owns domains
// [r*D/W, (r+1)*D/W).  Lists hold new node ids, ascending; Dirichlet nodes are
// never exchanged (their values are constant on every rank).
struct Exchange {
  int rank = 0, world = 1;
  int part_lo = 0, part_hi = 0;      // parts owned by this rank
  int64_t node_lo = 0, node_hi = 0;  // owned new node ids
  std::vector<int32_t> peers;        // ranks we talk to, ascending
  std::vector<int64_t> send_offs, recv_offs;  // per peer (size peers+1)
  std::vector<int32_t> send_nodes, recv_nodes;
  std::vector<int32_t> part_order;   // owned parts: boundary parts first, then interior
  int n_boundary = 0;
};
void build_exchange(const Partition &P, const uint8_t *is_dirichlet_new, int n_domains, int world, int rank,
                    Exchange &X);
// rank-local view of P for X's parts (X's lists are rewritten to local ids)
void localize_partition(const Partition &P, Exchange &X, Partition &L);

// node -> incident conn positions (ascending), positions of the flat
// tets-then-hexes connectivity (exact order of the reference's conn_data)
void build_node_csr(int64_t V, int64_t n_tet, const int64_t *tets, int64_t n_hex, const int64_t *hexes,
                    std::vector<int32_t> &offs, std::vector<int32_t> &pos);

// --------------------------------------------------------------------------
// device precompute (fh_precompute.cu)
struct GeomOut {
  double *A;        // sum N^2 or nullptr
  double *row_abs;  // nconn or nullptr
  double *G;        // 6 * E or nullptr (G = w inv inv^T, upper triangle 00 01 02 11 12 22)
  double *vol;      // E
  int *bad;         // first degenerate element (atomicMin), init INT_MAX
};
void launch_geometry(const double *xyz, const int32_t *conn, int64_t n_tet, int64_t n_hex, GeomOut out,
                     cudaStream_t s);
void launch_node_volumes(const int32_t *csr_offs, const int32_t *csr_pos, int64_t V, int64_t n_tet,
                         const double *vol, double *node_vol, cudaStream_t s);

}  // namespace fh
