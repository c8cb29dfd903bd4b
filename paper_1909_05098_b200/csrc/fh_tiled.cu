// TILED mode: the whole explicit step (north_star (ii)-(iv)) as ONE kernel.
//
// One CTA per tile ("part", fh_partition.cpp) of owned nodes:
//   0. thread 0 starts a kStages-deep ring of TMA bulk copies
//      (cp.async.bulk + mbarrier complete_tx) of the tile's element-slot
//      stream -- 16-bit tile-local connectivity, the 6-value metric tensor G
//      (A = D G D^T), the conductivity factor -- batch by batch;
//   1. meanwhile all threads stage the tile's temperatures in shared memory:
//      the owned node range (coalesced) and the halo list (gathered), and zero
//      the nodal load accumulators;
//   2. per batch (one thread per element slot): corner temperatures from
//      shared memory, k(T) per corner (TD) for kbar_e, g = D^T (T - T_0),
//      f = G g, c_a = kbar * D_a . f; then -c_a is added into the owned
//      corners' accumulators phase by phase, a barrier per phase, so each
//      node's sum has a fixed order: deterministic without atomics;
//   3. every owned non-Dirichlet node: T' = T + dt (F - kb T + qb + qm + q_ext
//      [+ Robin]) / C with C = rho(T) c(T) v and kb = w_b(T) c_b v, written to
//      the other temperature buffer; runaway check.
// HBM traffic per step: the slot stream once (duplicated halo elements
// included), the node streams (T, v, [q, xyz]) once, T' once, halo T from L2.
#include <cstdio>
#include <type_traits>
#include <algorithm>

#include "fh_tiled.cuh"

namespace fh {

constexpr unsigned long long kNone = ~0ull;

// minimum resident CTAs per SM requested from ptxas for the fp32 step kernel
// (caps registers; the default is the measured best, see scripts/sweep.py)
// (5 since the tiles stage T alone: 48 registers without spills and ~43 KB of
// shared memory per 1536-node tile; cfg4 0.2623 -> 0.2484 ms/step over 4)
#ifndef FH_MIN_BLOCKS_F32
#define FH_MIN_BLOCKS_F32 5
#endif
constexpr int kMinBlocksF32 = FH_MIN_BLOCKS_F32;
#ifndef FH_MIN_BLOCKS_TET
#define FH_MIN_BLOCKS_TET 6
#endif
constexpr int kMinBlocksTet = FH_MIN_BLOCKS_TET;  // tet-only fp32 kernels: smaller tiles, more CTAs
// tet-only fp64 kernels: 3 resident CTAs (<= 80 registers; cfg3 fp64 runs 4 waves of 3 CTAs/SM)
constexpr int kMinBlocksTetF64 = 3;
// global loads kept in flight per thread in the staging and node-update loops
#ifndef FH_STAGE_UNROLL
#define FH_STAGE_UNROLL 8
#endif
#ifndef FH_PREFETCH_NODES
#define FH_PREFETCH_NODES 1
#endif
#ifndef FH_NODE_UNROLL
#define FH_NODE_UNROLL 2
#endif
#ifndef FH_HEX_TM_CONST
#define FH_HEX_TM_CONST 0
#endif
#ifndef FH_STAGE_UNROLL_TET
#define FH_STAGE_UNROLL_TET 4
#endif
#ifndef FH_NODE_UNROLL_TET
#define FH_NODE_UNROLL_TET 1
#endif
// per-tile material / single-RF node bodies (0: the general body whenever node regions exist)
#ifndef FH_PART_MAT
#define FH_PART_MAT 1
#endif
// corner phases: predicated accumulation (0) or unpredicated into a trash slot (1)
#ifndef FH_TRASH_SLOT
#define FH_TRASH_SLOT 0
#endif

// (T, k(T)) of a tile-local node, staged once per tile in shared memory
template <typename S>
struct __align__(2 * sizeof(S)) TK {
  S t, k;
};

// What a tile stages per node.  Two-knot laws (LIN) and TI runs stage T alone:
// k is linear between the knots, so an element's mean conductivity is k(mean
// T) unless a staged temperature lies outside them (`kclamp`, tile-uniform,
// found while staging; then the corner values are interpolated one by one).
// Laws with more knots (KST) stage (T, k(T)) pairs.
template <typename S, bool KST>
using Staged = std::conditional_t<KST, TK<S>, S>;
template <typename S>
__device__ __forceinline__ S st_T(const S *sT, int i) { return sT[i]; }
template <typename S>
__device__ __forceinline__ S st_T(const TK<S> *sT, int i) { return sT[i].t; }

// products that must not be contracted into an FMA (keeps T == Ta a bitwise
// fixed point: kb*T and qb = kb*Ta round identically)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// ---- TMA bulk copy / mbarrier helpers (sm_90+ PTX, sm_100a target) ----------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a 16-byte aligned range (no shared memory, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// any range: widened to 16-byte boundaries (allocations are 256-byte granular), 32 KB pieces
__device__ __forceinline__ void prefetch_range(const void *p, size_t bytes) {
  if (!p || bytes == 0) return;
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  for (; a < e; a += 32768) {
    const uintptr_t n = e - a < 32768 ? e - a : 32768;
    bulk_prefetch_l2(reinterpret_cast<const void *>(a), (uint32_t)n);
  }
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// stage layout for one batch of B slots of a kind with N corners
template <typename S>
struct StageLayout {
  int conn, G, kf, region, rank, phase;
  __host__ __device__ StageLayout(int N, bool has_kf, bool has_rank, bool has_region) {
    conn = 0;
    G = kBatch * N * 2;
    kf = G + 6 * kBatch * (int)sizeof(S);
    region = kf + (has_kf ? kBatch * (int)sizeof(S) : 0);  // material byte per slot (several materials only)
    rank = region + (has_region ? kBatch : 0);
    phase = rank + (has_rank ? kBatch * N : 0);  // colored mode only (no rank block then)
  }
};

// LIN: every curve has two knots (one-knot curves were normalised on the host
// to y1 = y0, slope 0), so the clamped interpolation is two selects and an FMA
template <bool LIN, typename S>
__device__ __forceinline__ S ip(const Curve<S> &c, S x) {
  if (!LIN) return interp(c, x);
  S r = c.slope[0] * (x - c.x[0]) + c.y[0];
  r = (x >= c.x[1]) ? c.y[1] : r;
  return (x <= c.x[0]) ? c.y[0] : r;
}

template <bool LIN, typename S>
__device__ __forceinline__ S kbar_from(const Curve<S> &kc, const S *Tn, int n, S kf) {
  S s = S(0);
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if (b < n) s += ip<LIN>(kc, Tn[b]);
  return s / S(n) * kf;
}

// material-0 mean conductivity of a slot from its corner temperatures (two-knot law kc)
template <typename S, int N>
__device__ __forceinline__ S kbar_lin(const Curve<S> &kc, const S (&T)[N], bool kclamp, S kf) {
  if (!kclamp) {
    S sum;
    if constexpr (N == 8) sum = ((T[0] + T[1]) + (T[2] + T[3])) + ((T[4] + T[5]) + (T[6] + T[7]));
    else sum = (T[0] + T[1]) + (T[2] + T[3]);
    return (kc.slope[0] * (sum * S(1.0 / N) - kc.x[0]) + kc.y[0]) * kf;
  }
  S K[N];
#pragma unroll
  for (int b = 0; b < N; ++b) K[b] = ip<true>(kc, T[b]);
  S sum;
  if constexpr (N == 8) sum = ((K[0] + K[1]) + (K[2] + K[3])) + ((K[4] + K[5]) + (K[6] + K[7]));
  else sum = (K[0] + K[1]) + (K[2] + K[3]);
  return sum * S(1.0 / N) * kf;
}

__device__ __forceinline__ float fast_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fast_div(double a, double b) { return a / b; }
__device__ __forceinline__ void load_xyzv(const float *p, float &x, float &y, float &z, float &v) {
  const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
  x = a.x; y = a.y; z = a.z; v = a.w;
}
__device__ __forceinline__ void load_xyzv(const double *p, double &x, double &y, double &z, double &v) {
  const double2 a = __ldg(reinterpret_cast<const double2 *>(p)), b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
  x = a.x; y = a.y; z = b.x; v = b.y;
}
// fp32: hardware ex2 (2 ulp, well inside the 1e-4 fp32 tolerance); fp64: libm
__device__ __forceinline__ float fast_exp(float x) { return __expf(x); }
__device__ __forceinline__ double fast_exp(double x) { return exp(x); }

// F - kb T + qb + qm + q_ext with C, kb from the material laws (TD) or the
// frozen arrays (TI); returns the rate, writes the capacity
// INSIDE: x lies strictly between the knots of every two-knot law of the
// material (the tile's `kclamp` flag is clear), so the clamps of ip<true> are
// skipped -- the remaining FMA is ip<true>'s own, bit for bit
template <bool LIN, bool INSIDE, typename S>
__device__ __forceinline__ S ipn(const Curve<S> &c, S x) {
  if (LIN && INSIDE) return c.slope[0] * (x - c.x[0]) + c.y[0];
  return ip<LIN>(c, x);
}

template <typename S, bool TD, bool LIN, bool INSIDE = false>
__device__ __forceinline__ S node_rate(const Mat<S> &m, S x, S F, S v, S q, S cfrozen, S kbfrozen, S &cap) {
  S kb;
  if (TD) {
    cap = ipn<LIN, INSIDE>(m.rho, x) * ipn<LIN, INSIDE>(m.c, x) * v;
    kb = m.td_perf ? ipn<LIN, INSIDE>(m.wb, x) * m.cb * v : m.wbcb * v;
  } else {
    cap = cfrozen;
    kb = m.td_perf ? kbfrozen : m.wbcb * v;
  }
  return (((F - mul_rn(kb, x)) + mul_rn(kb, m.Ta)) + m.Qm * v) + q;
}

template <typename S>
__device__ __forceinline__ S sources_at(const TiledArgs<S> &g, const S *xyz) {
  // the host passes the active sources only, Gaussians first
  const S x = xyz[0], y = xyz[1], z = xyz[2];
  if (g.n_src == 1 && g.n_gauss == 1) {  // the common single-Gaussian case, straight-line
    const SourceT<S> &s = g.src[0];
    const S dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
    return s.amp * fast_exp(-((dx * dx + dy * dy) + dz * dz) * s.inv2s2);
  }
  S q = S(0);
#pragma unroll 1
  for (int k = 0; k < g.n_gauss; ++k) {
    const SourceT<S> &s = g.src[k];
    const S dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
    const S r2 = (dx * dx + dy * dy) + dz * dz;
    q += s.amp * fast_exp(-r2 * s.inv2s2);
  }
#pragma unroll 1
  for (int k = g.n_gauss; k < g.n_src; ++k) {
    const SourceT<S> &s = g.src[k];
    const S dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
    const S r2 = (dx * dx + dy * dy) + dz * dz;
    q += r2 > S(0) ? min(s.cap, fast_div(s.inv4pi_amp, r2)) : s.cap;
  }
  return q;
}

// Issue the bulk copies of batch j of part p into stage buffer `st`.
template <typename S>
__device__ void issue_batch(const TiledArgs<S> &g, int p, int j, int nbt, unsigned char *stage, uint64_t *bar,
                            bool with_region = true) {
  const bool tet = j < nbt;
  const int N = tet ? 4 : 8;
  const int b = tet ? j : j - nbt;
  const int s0 = (tet ? g.part_tet_start[p] : g.part_hex_start[p]) + b * kBatch;
  const int cnt = (tet ? g.part_tet_count[p] : g.part_hex_count[p]) - b * kBatch;
  const int k = cnt < kBatch ? cnt : kBatch;
  const int kr = (k + 3) & ~3;
  const unsigned char *rec = (tet ? g.tet_rec : g.hex_rec) + (size_t)(s0 / kBatch) * RecBytes<S>(N);
  const S *kf = tet ? g.tet_kf : g.hex_kf;
  const uint8_t *rank = tet ? g.tet_rank : g.hex_rank;
  const uint8_t *phase = tet ? g.tet_phase : g.hex_phase;
  const uint8_t *region_s = tet ? g.tet_region : g.hex_region;
  const StageLayout<S> L(N, kf != nullptr, rank != nullptr, region_s != nullptr);
  const uint8_t *region = with_region ? region_s : nullptr;  // uniform tiles: nothing to stage
  const int kp = (k + 15) & ~15;  // bulk copies move multiples of 16 bytes
  uint32_t bytes = (uint32_t)(kr * N * 2 + 6 * kr * sizeof(S));
  if (kf) bytes += kr * sizeof(S);
  if (rank) bytes += kr * N;
  if (phase) bytes += kp;
  if (region) bytes += kp;
  mbar_expect_tx(bar, bytes);
  if (phase) bulk_g2s(stage + L.phase, phase + s0, kp, bar);
  if (region) bulk_g2s(stage + L.region, region + s0, kp, bar);
  if (kr == kBatch) {  // a full batch: one copy of the whole record (conn16 + 6 G rows)
    bulk_g2s(stage + L.conn, rec, RecBytes<S>(N), bar);
  } else {
    bulk_g2s(stage + L.conn, rec, kr * N * 2, bar);
    const unsigned char *Gb = rec + kBatch * N * 2;
#pragma unroll
    for (int c = 0; c < 6; ++c)
      bulk_g2s(stage + L.G + c * kBatch * sizeof(S), Gb + c * kBatch * sizeof(S), kr * sizeof(S), bar);
  }
  if (kf) bulk_g2s(stage + L.kf, kf + s0, kr * sizeof(S), bar);
  if (rank) bulk_g2s(stage + L.rank, rank + (size_t)N * s0, kr * N, bar);
}

// LEAN loops: the whole batch record (padding slots included) and, for tets,
// the 256 phase bytes of batch j of the tile whose slots start at s_start
template <typename S, int N>
__device__ __forceinline__ void lean_issue(const TiledArgs<S> &g, int s_start, int j, unsigned char *stage,
                                           uint64_t *bar) {
  const unsigned char *rec = (N == 4 ? g.tet_rec : g.hex_rec) + (size_t)(s_start / kBatch + j) * RecBytes<S>(N);
  mbar_expect_tx(bar, (uint32_t)(RecBytes<S>(N) + (N == 4 ? kBatch : 0)));
  bulk_g2s(stage, rec, RecBytes<S>(N), bar);
  if (N == 4) bulk_g2s(stage + RecBytes<S>(N), g.tet_phase + s_start + j * kBatch, kBatch, bar);
}

// LEAN 3 (mixed tiles): batch j of the tile is a tet batch while j < nbt, then a hex batch
template <typename S>
__device__ __forceinline__ void lean_issue_mixed(const TiledArgs<S> &g, int t_start, int h_start, int nbt, int j,
                                                 unsigned char *stage, uint64_t *bar) {
  if (j < nbt) lean_issue<S, 4>(g, t_start, j, stage, bar);
  else lean_issue<S, 8>(g, h_start, j - nbt, stage, bar);
}

// element loads of staged slot i of the batch ------------------------------------
template <typename S, bool TD, bool LIN>
__device__ __forceinline__ void hex_loads(const TiledArgs<S> &g, const unsigned char *stage,
                                          const Staged<S, TD && !LIN> *sT, bool kclamp, int reg, bool has_kf, int i,
                                          uint16_t nd[8], S c[8]) {
  constexpr bool KST = TD && !LIN;
  const StageLayout<S> L(8, has_kf, g.hex_rank != nullptr, g.hex_region != nullptr);
  const uint4 w = reinterpret_cast<const uint4 *>(stage + L.conn)[i];
  nd[0] = w.x & 0xffff; nd[1] = w.x >> 16; nd[2] = w.y & 0xffff; nd[3] = w.y >> 16;
  nd[4] = w.z & 0xffff; nd[5] = w.z >> 16; nd[6] = w.w & 0xffff; nd[7] = w.w >> 16;
  S T[8], K[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if constexpr (KST) {
      const TK<S> q = sT[nd[b]];
      T[b] = q.t;
      K[b] = q.k;
    } else {
      T[b] = sT[nd[b]];
      K[b] = S(0);
    }
  }
  const S *G = reinterpret_cast<const S *>(stage + L.G);
  const S g00 = G[i], g01 = G[kBatch + i], g02 = G[2 * kBatch + i], g11 = G[3 * kBatch + i],
          g12 = G[4 * kBatch + i], g22 = G[5 * kBatch + i];
  const S kf = has_kf ? reinterpret_cast<const S *>(stage + L.kf)[i] : S(1);
  S kb = kf;
  if (TD) {
    if (reg == 0 && !KST) {  // two-knot law of material 0
      kb = kbar_lin<S, 8>(g.mats.m[0].k, T, kclamp, kf);
    } else if (reg == 0) {  // k(T) of material 0 staged per node: kbar = mean of the corner values
      const S sum = ((K[0] + K[1]) + (K[2] + K[3])) + ((K[4] + K[5]) + (K[6] + K[7]));
      kb = sum * S(0.125) * kf;
    } else {  // other materials (rare slots): the element's own curve at each corner
      kb = kbar_from<LIN>(g.mats.m[reg].k, T, 8, kf);
    }
  }
  // g = sum_b s_b (T_b - T_0) with the corner signs of element.py HEX_VERTEX_SIGNS
  // (the T_0 shifts cancel pairwise except where written explicitly)
  const S gx = ((T[1] - T[0]) + (T[2] - T[3])) + ((T[5] - T[4]) + (T[6] - T[7]));
  const S gy = ((T[3] - T[0]) + (T[2] - T[1])) + ((T[7] - T[4]) + (T[6] - T[5]));
  const S gz = ((T[4] - T[0]) + (T[5] - T[1])) + ((T[6] - T[2]) + (T[7] - T[3]));
  const S u = kb * (g00 * gx + g01 * gy + g02 * gz);
  const S v = kb * (g01 * gx + g11 * gy + g12 * gz);
  const S w2 = kb * (g02 * gx + g12 * gy + g22 * gz);
  const S a = u + v, b2 = u - v;
  c[0] = -a - w2; c[1] = b2 - w2; c[2] = a - w2; c[3] = -b2 - w2;
  c[4] = -a + w2; c[5] = b2 + w2; c[6] = a + w2; c[7] = -b2 + w2;
}

// with accumulator rows (g.tet_rows > 1) each 16-bit word is row << 14 | local
// index; rofs[a] = row * row_stride locates the corner's accumulator
template <typename S, bool TD, bool LIN>
__device__ __forceinline__ void tet_loads(const TiledArgs<S> &g, const unsigned char *stage,
                                          const Staged<S, TD && !LIN> *sT, bool kclamp, int reg, bool has_kf, int i,
                                          uint16_t nd[4], S c[4], int rofs[4], uint32_t idx_mask, int row_stride) {
  constexpr bool KST = TD && !LIN;
  const StageLayout<S> L(4, has_kf, g.tet_rank != nullptr, g.tet_region != nullptr);
  const uint2 w = reinterpret_cast<const uint2 *>(stage + L.conn)[i];
  const uint32_t raw[4] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16};
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    nd[a] = (uint16_t)(raw[a] & idx_mask);
    rofs[a] = (int)(raw[a] >> 14) * row_stride;
  }
  S T[4], K[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if constexpr (KST) {
      const TK<S> q = sT[nd[b]];
      T[b] = q.t;
      K[b] = q.k;
    } else {
      T[b] = sT[nd[b]];
      K[b] = S(0);
    }
  }
  const S *G = reinterpret_cast<const S *>(stage + L.G);
  const S g00 = G[i], g01 = G[kBatch + i], g02 = G[2 * kBatch + i], g11 = G[3 * kBatch + i],
          g12 = G[4 * kBatch + i], g22 = G[5 * kBatch + i];
  const S kf = has_kf ? reinterpret_cast<const S *>(stage + L.kf)[i] : S(1);
  S kb = kf;
  if (TD) {
    if (reg == 0 && !KST) {
      kb = kbar_lin<S, 4>(g.mats.m[0].k, T, kclamp, kf);
    } else if (reg == 0) {
      kb = ((K[0] + K[1]) + (K[2] + K[3])) * S(0.25) * kf;
    } else {
      kb = kbar_from<LIN>(g.mats.m[reg].k, T, 4, kf);
    }
  }
  const S d1 = T[1] - T[0], d2 = T[2] - T[0], d3 = T[3] - T[0];
  c[1] = kb * (g00 * d1 + g01 * d2 + g02 * d3);
  c[2] = kb * (g01 * d1 + g11 * d2 + g12 * d3);
  c[3] = kb * (g02 * d1 + g12 * d2 + g22 * d3);
  c[0] = -((c[1] + c[2]) + c[3]);
}

// accumulation modes (deterministic in all three):
//   kRanked      phase = rank of the slot among the node's slots of the batch
//   kCornerPhase corner-unique tiles: phase = corner index (N barriers/batch)
// Each thread carries kSPT slots of the batch (i = q * kTileThreads + tid).
//   kColored     slots sorted by colour (no two slots of a colour share an
//                updated node): phase = colour index inside the batch, so a
//                batch needs as many barriers as it holds colours (1-2)
//   kSharedAtomic  red.shared.add per corner, one barrier per batch: fastest
//                but the summation order is not fixed (tolerance-only, opt-in)
//   kCornerPhase2  corner phases with two accumulator rows (corners a and
//                a + N/2 share a phase): half the barriers, 2x accumulator smem
// (round 1 also measured one accumulator row per corner and four-row corner
// phases: both slower, the extra rows cost a resident CTA per SM; removed)
enum { kRanked = 0, kCornerPhase = 1, kCornerSlot = 2, kColored = 3, kSharedAtomic = 4, kCornerPhase2 = 5,
       kCornerPhase4 = 6 };

template <typename S, int N, int MODE>
__device__ __forceinline__ void accumulate(S *acc, const uint16_t (&nd)[kSPT][N], const S (&c)[kSPT][N], int nfree,
                                           const bool (&valid)[kSPT], const uint8_t (&rank)[kSPT][N], int n_phase) {
  int loc[kSPT][N];
#pragma unroll
  for (int q = 0; q < kSPT; ++q)
#pragma unroll
    for (int a = 0; a < N; ++a) loc[q][a] = (valid[q] && nd[q][a] < nfree) ? (int)nd[q][a] : -1;
  if (MODE == kSharedAtomic) {
    // non-deterministic (summation order varies run to run; tolerance-only)
#pragma unroll
    for (int q = 0; q < kSPT; ++q)
#pragma unroll
      for (int a = 0; a < N; ++a)
        if (loc[q][a] >= 0) atomicAdd(&acc[loc[q][a]], -c[q][a]);
    __syncthreads();  // stage buffer fully consumed before it is refilled
  } else if (MODE == kCornerPhase2) {
    // two accumulator rows: corner a (< N/2) into row 0, corner a + N/2 into
    // row 1 in the same phase -> N/2 barriers per batch; F = row0 + row1
    S *acc1 = acc + nfree;
#pragma unroll
    for (int a = 0; a < N / 2; ++a) {
#pragma unroll
      for (int q = 0; q < kSPT; ++q) {
        if (loc[q][a] >= 0) acc[loc[q][a]] -= c[q][a];
        if (loc[q][a + N / 2] >= 0) acc1[loc[q][a + N / 2]] -= c[q][a + N / 2];
      }
      __syncthreads();
    }
  } else if (MODE == kCornerPhase && !FH_TRASH_SLOT) {
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int q = 0; q < kSPT; ++q)
        if (loc[q][a] >= 0) acc[loc[q][a]] -= c[q][a];
      __syncthreads();
    }
  } else if (MODE == kCornerPhase) {
    // corners the tile does not update (halo, Dirichlet, padding slots) add
    // into the trash slot acc[nfree] (never read): no predicates per phase
    int tl[kSPT][N];
#pragma unroll
    for (int q = 0; q < kSPT; ++q)
#pragma unroll
      for (int a = 0; a < N; ++a) tl[q][a] = valid[q] ? min((int)nd[q][a], nfree) : nfree;
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int q = 0; q < kSPT; ++q) acc[tl[q][a]] -= c[q][a];
      __syncthreads();
    }
  } else {
    for (int ph = 0; ph < n_phase; ++ph) {
#pragma unroll
      for (int q = 0; q < kSPT; ++q)
#pragma unroll
        for (int a = 0; a < N; ++a)
          if (rank[q][a] == ph && loc[q][a] >= 0) acc[loc[q][a]] -= c[q][a];
      __syncthreads();
    }
  }
}
// colour phases: all corners of a slot share its colour's phase, so a thread
// does its N read-modify-writes once, in its phase (warps are mostly one
// colour: slots are colour-sorted)
static_assert(kSPT == 1, "accumulate_colored handles one slot per thread");
template <typename S, int N>
__device__ __forceinline__ void accumulate_colored(S *acc, const uint16_t (&nd)[N], const S (&c)[N], int nfree,
                                                   bool valid, int myph, int n_phase, const int *rofs = nullptr) {
  int loc[N];
#pragma unroll
  for (int a = 0; a < N; ++a) loc[a] = (valid && nd[a] < nfree) ? (int)nd[a] + (rofs ? rofs[a] : 0) : -1;
  for (int ph = 0; ph < n_phase; ++ph) {
    if (myph == ph) {
#pragma unroll
      for (int a = 0; a < N; ++a)
        if (loc[a] >= 0) acc[loc[a]] -= c[a];
    }
    __syncthreads();
  }
}

// KINDS: 0 hex-only, 1 tet-only, 2 mixed mesh (the absent kind's path is compiled out).
// LEAN: the batch loop specialised for the common tiles -- tet-only colour
// phases or hex-only two-row corner phases, every slot in material 0, no
// per-slot kf / region / rank streams -- with every per-batch flag and stage
// offset a compile-time constant (same arithmetic, same bits).  LEAN 1: the
// whole launch (fp32 records with paired G rows); LEAN 2: the material-0
// hex-only tiles of a mixed mesh or a mesh with regions (component-row G, like
// the general kernel's tiles of the same launch family); LEAN 3: the
// material-0 tiles of such a mesh that hold tets and hexes (one-row colour
// phases for the tet batches, then the hex batches).
template <typename S, bool TD, int MODE, int KINDS, bool LIN, int LEAN = 0>
__global__ void __launch_bounds__(kTileThreads, sizeof(S) == 4 ? (KINDS == 1 ? kMinBlocksTet : kMinBlocksF32)
                                                                : (KINDS == 1 ? kMinBlocksTetF64 : 2))
    k_tiled_step(const __grid_constant__ TiledArgs<S> g) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr bool KST = TD && !LIN;  // stage (T, k(T)) pairs; otherwise T alone (see Staged)
  using ST = Staged<S, KST>;
  S *acc = reinterpret_cast<S *>(smem + g.smem_T);
  unsigned char *ring = smem + g.smem_T + g.smem_acc;
  const int kStages = g.n_stages;
  __shared__ __align__(8) uint64_t bars[kMaxStages];
  __shared__ __align__(8) uint64_t hbar;  // halo id list copy
  __shared__ __align__(8) uint64_t tbar;  // owned temperature range copy (T-only staging)
  __shared__ int s_bad;
  // phases per batch of the tile (colour modes), read once instead of per batch
  constexpr int kNphCache = kTileThreads;  // one phase-count byte per batch, filled by one thread each
  __shared__ uint8_t s_nph[kNphCache];
  // skip only when an EARLIER step failed: every CTA of the failing step still
  // writes its tile, so the field after a runaway is that whole step's output
  if (g.flag->step < g.step_no) return;
  const int p = g.part_list ? g.part_list[g.part_begin + blockIdx.x] : g.part_begin + (int)blockIdx.x;
  const int tid = threadIdx.x;
  const int n0 = g.part_node_start[p];
  const int nn = g.part_node_start[p + 1] - n0;
  const int nfree = g.part_n_free[p];
  // T-only staging: the owned range Tin[n0, n0 + nn) is one bulk copy from the
  // 16-byte boundary below n0, so the tile's node 0 sits `lead` elements into
  // the staging region (the elements before it are never referenced)
  constexpr int kVec = 16 / (int)sizeof(S);
  const int lead = KST ? 0 : (n0 & (kVec - 1));
  ST *sT = reinterpret_cast<ST *>(smem) + lead;
  const int n_bulk = KST ? 0 : ((lead + nn) & ~(kVec - 1));  // elements the bulk copy brings (from n0 - lead)
  // tile tables read once (the batch loop would otherwise re-load them every iteration)
  const int t_cnt = __ldg(g.part_tet_count + p), h_cnt = __ldg(g.part_hex_count + p);
  const int t_start = __ldg(g.part_tet_start + p), h_start = __ldg(g.part_hex_start + p);
  const int nbt = (t_cnt + kBatch - 1) / kBatch;
  // several materials: the tile's slots may all share one region (then no
  // region bytes are staged and every slot uses it), else -1
  const int preg = g.part_region ? (int)g.part_region[p] : -1;
  const int nbh = (g.part_hex_count[p] + kBatch - 1) / kBatch;
  const int nb = nbt + nbh;
  // the tile's halo id list is bulk-copied into the (not yet used) accumulator
  // region first thing, so the halo gather waits one round trip, not two.
  // The copy is widened to 16-byte boundaries (the list is padded at its end).
  const int h0 = g.part_halo_start[p], nh = g.part_halo_start[p + 1] - h0;
  const int hs = h0 & ~3, hoff = h0 - hs;
  FH_DEV_CHECK(nn + nh <= g.max_local && nfree <= nn && n0 + nn <= g.n_nodes, "tile node ranges");
  int32_t *s_ids = reinterpret_cast<int32_t *>(acc);
  {
    const uint8_t *bn = (KINDS == 0) ? nullptr : g.tet_bnph;
    if (bn && tid < nbt && tid < kNphCache) s_nph[tid] = __ldg(bn + t_start / kBatch + tid);
    const uint8_t *hn = (KINDS == 1 || MODE != kColored) ? nullptr : g.hex_bnph;
    if (hn && tid < nbh && nbt + tid < kNphCache) s_nph[nbt + tid] = __ldg(hn + h_start / kBatch + tid);
  }
  if (tid == 0) {
    s_bad = 0;
#pragma unroll
    for (int q = 0; q < kStages; ++q) mbar_init(&bars[q], 1);
    mbar_init(&hbar, 1);
    mbar_init(&tbar, 1);
    fence_barrier_init();
  }
  __syncthreads();  // the mbarriers are initialised before anyone waits on them
  if (tid == 0) {
    const uint32_t hbytes = (uint32_t)((((h0 + nh + 3) & ~3) - hs) * 4);
    mbar_expect_tx(&hbar, hbytes);
    if (hbytes) bulk_g2s(s_ids, g.halo_nodes + hs, hbytes, &hbar);
    if constexpr (!KST) {
      mbar_expect_tx(&tbar, (uint32_t)(n_bulk * sizeof(S)));
      if (n_bulk) bulk_g2s(smem, g.Tin + (n0 - lead), (uint32_t)(n_bulk * sizeof(S)), &tbar);
    }
    for (int j = 0; j < kStages && j < nb; ++j) {
      if constexpr (LEAN && KINDS == 2)
        lean_issue_mixed<S>(g, t_start, h_start, nbt, j, ring + j * g.stage_bytes, &bars[j]);
      else if constexpr (LEAN)
        lean_issue<S, KINDS == 1 ? 4 : 8>(g, KINDS == 1 ? t_start : h_start, j, ring + j * g.stage_bytes, &bars[j]);
      else
        issue_batch(g, p, j, nbt, ring + j * g.stage_bytes, &bars[j], preg < 0);
    }
#if FH_PREFETCH_NODES
    // the node update's per-node streams, pulled into L2 while the batches run
    if (g.n_src) prefetch_range(g.xyzv + 4 * (size_t)n0, 4 * sizeof(S) * nfree);
    else prefetch_range(g.vol + n0, sizeof(S) * nfree);
    prefetch_range(g.q_ext ? g.q_ext + n0 : nullptr, sizeof(S) * nfree);
#endif
  }
  // stage temperatures: owned range + halo list; zero accumulators.  Loads
  // are clamped to valid addresses and only the shared stores are predicated,
  // so the unrolled rounds stay branch-free.  Two-knot laws stage T alone and
  // note whether any staged temperature lies outside material 0's conductivity
  // knots (kout -> kclamp); laws with more knots stage k(T) of material 0 too.
  // (kout is set by any staged temperature that is not strictly inside
  // (g.lin_lo, g.lin_hi), the intersection of the knot ranges of material 0's
  // sloped laws -- k, rho, c, w_b -- so the flag also lets the node update of
  // LEAN tiles skip its clamps; NaN counts as outside)
  const Curve<S> &k0 = g.mats.m[0].k;
  const S kx0 = g.lin_lo, kx1 = g.lin_hi;
  const bool ksloped = TD && LIN;
  bool kout = false;
  auto staged = [&](S x) -> ST {
    if constexpr (KST) {
      return TK<S>{x, interp(k0, x)};
    } else {
      if (TD && LIN) kout |= !((x > kx0) & (x < kx1));
      return x;
    }
  };
  // loads in flight per thread while staging (tet-only tiles: 4, measured
  // 1% faster on cfg3; hex tiles: 8)
  constexpr int U = KINDS == 1 ? FH_STAGE_UNROLL_TET : FH_STAGE_UNROLL;
  if constexpr (KST) {
    for (int base = tid; base < nn; base += U * kTileThreads) {
      S x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = __ldg(g.Tin + n0 + min(base + u * kTileThreads, nn - 1));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * kTileThreads;
        const ST v = staged(x[u]);
        if (i < nn) sT[i] = v;
      }
    }
  } else {
    // the (at most kVec - 1) owned nodes past the bulk copy's last 16 bytes
    const int i = n_bulk - lead + tid;
    if (i < nn) sT[i] = staged(__ldg(g.Tin + n0 + i));
  }
  mbar_wait(&hbar, 0);
  for (int base = tid; base < nh; base += U * kTileThreads) {
    int id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      id[u] = s_ids[hoff + min(base + u * kTileThreads, nh - 1)];
      FH_DEV_CHECK(id[u] >= 0 && id[u] < g.n_nodes, "halo node id");
    }
    S x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = __ldg(g.Tin + id[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * kTileThreads;
      const ST v = staged(x[u]);
      if (i < nh) sT[nn + i] = v;
    }
  }
  if constexpr (!KST) {
    mbar_wait(&tbar, 0);
    if (ksloped) {  // knots check of the bulk-copied owned nodes (16 bytes per load)
      for (int v = tid; v < n_bulk / kVec; v += kTileThreads) {
        S x[kVec];
        if constexpr (sizeof(S) == 4) {
          const float4 q = reinterpret_cast<const float4 *>(smem)[v];
          x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
        } else {
          const double2 q = reinterpret_cast<const double2 *>(smem)[v];
          x[0] = q.x; x[1] = q.y;
        }
#pragma unroll
        for (int c = 0; c < kVec; ++c) kout |= !((x[c] > kx0) & (x[c] < kx1)) & (v * kVec + c >= lead);
      }
    }
  }
  if (tid == 0) sT[nn + nh] = ST{};  // the padding slots' dummy node (partition step 5): T = 0
  // every halo id has been read: the accumulators may be zeroed
  const bool kclamp = __syncthreads_or(kout && ksloped) != 0;
  const int acc_rows = max(MODE == kCornerPhase2 ? 2 : 1,
                           KINDS == 2 ? 1 : g.tet_rows);
  for (int i = tid; i < acc_rows * nfree; i += kTileThreads) acc[i] = S(0);
  __syncthreads();

  // uniform per launch: stage layouts and which optional streams exist
  const bool t_kf = g.tet_kf != nullptr, h_kf = g.hex_kf != nullptr;
  // stage layouts follow the global streams; t_reg / h_reg: this tile reads
  // its slots' region bytes (otherwise they all use tile_reg)
  const bool t_rs = g.tet_region != nullptr, h_rs = g.hex_region != nullptr;
  const bool t_reg = t_rs && preg < 0, h_reg = h_rs && preg < 0;
  const int tile_reg = preg < 0 ? 0 : preg;
  const bool t_col = g.tet_phase != nullptr;
  const uint32_t t_mask = g.tet_rows > 1 ? 0x3fffu : 0xffffu;  // row-tagged tet connectivity
  const StageLayout<S> Lt(4, t_kf, !t_col, t_rs);
  const StageLayout<S> Lh(8, h_kf, MODE == kRanked, h_rs);
  auto batch_nph = [&](int jj, const uint8_t *bn, int slot0) -> int {
    return jj < kNphCache ? (int)s_nph[jj] : (int)__ldg(bn + slot0 / kBatch);
  };
  if constexpr (LEAN) {
    // stage layout without kf / region / rank blocks: conn16 | G | phase (tets)
    constexpr int kGt = kBatch * 4 * 2, kGh = kBatch * 8 * 2, kPhase = kGt + 6 * kBatch * (int)sizeof(S);
    const int sbytes = g.stage_bytes;
    const uint32_t bar0 = smem_u32(&bars[0]);
    const int cnt = KINDS == 1 ? t_cnt : h_cnt;
    int st = 0;
    uint32_t par = 0;
    for (int j = 0; j < nb; ++j) {
      unsigned char *stage = ring + st * sbytes;
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "LWAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra LWAIT_%=;\n}" ::"r"(bar0 + 8u * (uint32_t)st),
          "r"(par)
          : "memory");
      // the whole batch record was copied: padding slots point at the dummy node
      const bool valid = true;
      const int i = tid;
      // every thread has read its slot from the stage once the batch's first
      // accumulation barrier is passed: the refill goes out right there
      auto refill = [&]() {
        if (tid == 0 && j + kStages < nb) {
          fence_proxy_async();
          if constexpr (KINDS == 2) lean_issue_mixed<S>(g, t_start, h_start, nbt, j + kStages, stage, &bars[st]);
          else lean_issue<S, KINDS == 1 ? 4 : 8>(g, KINDS == 1 ? t_start : h_start, j + kStages, stage, &bars[st]);
        }
      };
      // mixed tiles (LEAN 3): the tile's tet batches come first
      const bool tet_batch = KINDS == 1 || (KINDS == 2 && j < nbt);
      const int kG = tet_batch ? kGt : kGh;
      // fp32: paired G rows (k_pack_slots) (00,01) (02,11) (12,22), one 8-byte
      // load each; fp64: the 6 component rows
      S g00, g01, g02, g11, g12, g22;
      if constexpr (sizeof(S) == 4 && LEAN == 1) {
        const float2 *G2 = reinterpret_cast<const float2 *>(stage + kG);
        const float2 p0 = G2[i], p1 = G2[kBatch + i], p2 = G2[2 * kBatch + i];
        g00 = p0.x; g01 = p0.y; g02 = p1.x; g11 = p1.y; g12 = p2.x; g22 = p2.y;
      } else {
        const S *G = reinterpret_cast<const S *>(stage + kG);
        g00 = G[i]; g01 = G[kBatch + i]; g02 = G[2 * kBatch + i];
        g11 = G[3 * kBatch + i]; g12 = G[4 * kBatch + i]; g22 = G[5 * kBatch + i];
      }
      // Node references are used as BYTE offsets into sT and the accumulator
      // rows.  The fp32 LEAN 1 records store them pre-multiplied by 4
      // (k_scale_conn; no shift per corner), the others hold plain indices.
      constexpr bool SCALED = LEAN == 1 && sizeof(S) == 4;
      constexpr int SH = SCALED ? 0 : (sizeof(S) == 4 ? 2 : 3);
      const unsigned char *sTb = reinterpret_cast<const unsigned char *>(sT);
      unsigned char *accb = reinterpret_cast<unsigned char *>(acc);
      const uint32_t nfreeb = (uint32_t)nfree * (uint32_t)sizeof(S);
      if (KINDS != 0 && tet_batch) {
        const uint2 w = reinterpret_cast<const uint2 *>(stage)[i];
        const uint32_t raw[4] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16};
        uint32_t nd[4], rofs[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {  // LEAN tets always carry row-tagged connectivity (host condition)
          nd[a] = (raw[a] & 0x3fffu) << SH;
          rofs[a] = (raw[a] >> 14) * nfreeb;
        }
        S T[4];
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) T[b2] = *reinterpret_cast<const S *>(sTb + nd[b2]);
        // tet_loads with reg == 0 and kf == 1
        const S kb = kbar_lin<S, 4>(k0, T, kclamp, S(1));
        const S d1 = T[1] - T[0], d2 = T[2] - T[0], d3 = T[3] - T[0];
        S c[4];
        c[1] = kb * (g00 * d1 + g01 * d2 + g02 * d3);
        c[2] = kb * (g01 * d1 + g11 * d2 + g12 * d3);
        c[3] = kb * (g02 * d1 + g12 * d2 + g22 * d3);
        c[0] = -((c[1] + c[2]) + c[3]);
        const int ph = stage[kPhase + i];
        const int nph = s_nph[j];  // LEAN tiles have at most kNphCache batches (host condition)
        // colour phases (accumulate_colored): the slot's 4 corners are 4
        // distinct nodes, so the 4 read-modify-writes are issued together;
        // the first two phases are unrolled (1.3 phases per batch on cfg3)
        int loc[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) loc[a] = nd[a] < nfreeb ? (int)(nd[a] + rofs[a]) : -1;
        auto rmw = [&]() {
          S old[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) old[a] = loc[a] >= 0 ? *reinterpret_cast<S *>(accb + loc[a]) : S(0);
#pragma unroll
          for (int a = 0; a < 4; ++a)
            if (loc[a] >= 0) *reinterpret_cast<S *>(accb + loc[a]) = old[a] - c[a];
        };
        (void)valid;
        if (ph == 0) rmw();
        __syncthreads();
        refill();
        if (nph > 1) {
          if (ph == 1) rmw();
          __syncthreads();
          for (int q = 2; q < nph; ++q) {
            if (ph == q) rmw();
            __syncthreads();
          }
        }
      } else {
        const uint4 w = reinterpret_cast<const uint4 *>(stage)[i];
        uint32_t nd[kSPT][8];
        nd[0][0] = (w.x & 0xffff) << SH; nd[0][1] = (w.x >> 16) << SH; nd[0][2] = (w.y & 0xffff) << SH;
        nd[0][3] = (w.y >> 16) << SH; nd[0][4] = (w.z & 0xffff) << SH; nd[0][5] = (w.z >> 16) << SH;
        nd[0][6] = (w.w & 0xffff) << SH; nd[0][7] = (w.w >> 16) << SH;
        S T[8];
#pragma unroll
        for (int b2 = 0; b2 < 8; ++b2) T[b2] = *reinterpret_cast<const S *>(sTb + nd[0][b2]);
        // hex_loads with reg == 0 and kf == 1
        const S kb = kbar_lin<S, 8>(k0, T, kclamp, S(1));
        const S gx = ((T[1] - T[0]) + (T[2] - T[3])) + ((T[5] - T[4]) + (T[6] - T[7]));
        const S gy = ((T[3] - T[0]) + (T[2] - T[1])) + ((T[7] - T[4]) + (T[6] - T[5]));
        const S gz = ((T[4] - T[0]) + (T[5] - T[1])) + ((T[6] - T[2]) + (T[7] - T[3]));
        const S u = kb * (g00 * gx + g01 * gy + g02 * gz);
        const S v = kb * (g01 * gx + g11 * gy + g12 * gz);
        const S w2 = kb * (g02 * gx + g12 * gy + g22 * gz);
        const S a0 = u + v, b0 = u - v;
        S c[kSPT][8];
        c[0][0] = -a0 - w2; c[0][1] = b0 - w2; c[0][2] = a0 - w2; c[0][3] = -b0 - w2;
        c[0][4] = -a0 + w2; c[0][5] = b0 + w2; c[0][6] = a0 + w2; c[0][7] = -b0 + w2;
        // two-row corner phases (accumulate<kCornerPhase2>): corners a and a+4
        // go to different rows, so both read-modify-writes issue together
        (void)valid;
        unsigned char *acc1b = accb + nfreeb;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const bool u0 = nd[0][a] < nfreeb, u1 = nd[0][a + 4] < nfreeb;
          S *p0 = reinterpret_cast<S *>(accb + nd[0][a]), *p1 = reinterpret_cast<S *>(acc1b + nd[0][a + 4]);
          const S o0 = u0 ? *p0 : S(0), o1 = u1 ? *p1 : S(0);
          if (u0) *p0 = o0 - c[0][a];
          if (u1) *p1 = o1 - c[0][a + 4];
          __syncthreads();
          if (a == 0) refill();
        }
      }
      if (++st == kStages) {
        st = 0;
        par ^= 1u;
      }
    }
    (void)cnt;
  } else {
  int st = 0;
  uint32_t parity = 0;
  for (int j = 0; j < nb; ++j) {
    unsigned char *stage = ring + st * g.stage_bytes;
    mbar_wait(&bars[st], parity);
    const bool tet = KINDS == 1 || (KINDS == 2 && j < nbt);
    const int b = tet ? j : j - nbt;
    const int cnt = tet ? t_cnt : h_cnt;
    bool valid[kSPT];
#pragma unroll
    for (int q = 0; q < kSPT; ++q) valid[q] = b * kBatch + q * kTileThreads + tid < cnt;
    if (tet) {
      uint16_t nd[kSPT][4];
      S c[kSPT][4];
      uint8_t rk[kSPT][4];
      int rofs[kSPT][4];
#pragma unroll
      for (int q = 0; q < kSPT; ++q) {
        // slots past the end of a partial batch read slot 0 (always present)
        // instead of branching; only their accumulation is predicated off
        const int i = valid[q] ? q * kTileThreads + tid : 0;
        const int reg = t_reg ? (int)stage[Lt.region + i] : tile_reg;
        tet_loads<S, TD, LIN>(g, stage, sT, kclamp, reg, t_kf, i, nd[q], c[q], rofs[q], t_mask, nfree);
        FH_DEV_CHECK(nd[q][0] < nn + nh && nd[q][1] < nn + nh && nd[q][2] < nn + nh && nd[q][3] < nn + nh,
                     "tet corner outside the tile's staged nodes");
        // tets are never corner-unique: colour phases (phase byte per slot) or,
        // if the colouring overflowed, ranked phases (rank byte per corner)
        if (t_col) {
          const uint8_t ph = stage[Lt.phase + i];
#pragma unroll
          for (int a = 0; a < 4; ++a) rk[q][a] = ph;
        } else {
          const uint32_t w = reinterpret_cast<const uint32_t *>(stage + Lt.rank)[i];
          rk[q][0] = w & 0xff; rk[q][1] = (w >> 8) & 0xff; rk[q][2] = (w >> 16) & 0xff; rk[q][3] = w >> 24;
        }
      }
      if (t_col)
        accumulate_colored<S, 4>(acc, nd[0], c[0], nfree, valid[0], rk[0][0],
                                 batch_nph(j, g.tet_bnph, t_start + b * kBatch), rofs[0]);
      else
        accumulate<S, 4, kRanked>(acc, nd, c, nfree, valid, rk, g.max_phase_tet);
    } else {
      uint16_t nd[kSPT][8];
      S c[kSPT][8];
      uint8_t rk[kSPT][8];
#pragma unroll
      for (int q = 0; q < kSPT; ++q) {
        const int i = valid[q] ? q * kTileThreads + tid : 0;
        const int reg = h_reg ? (int)stage[Lh.region + i] : tile_reg;
        hex_loads<S, TD, LIN>(g, stage, sT, kclamp, reg, h_kf, i, nd[q], c[q]);
#ifdef FH_CHECKS
        for (int a = 0; a < 8; ++a) FH_DEV_CHECK(nd[q][a] < nn + nh, "hex corner outside the tile's staged nodes");
#endif
        if (MODE == kRanked) {
          const uint2 w = reinterpret_cast<const uint2 *>(stage + Lh.rank)[i];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            rk[q][a] = (w.x >> (8 * a)) & 0xff;
            rk[q][a + 4] = (w.y >> (8 * a)) & 0xff;
          }
        } else if (MODE == kColored) {
          const uint8_t ph = stage[Lh.phase + i];
#pragma unroll
          for (int a = 0; a < 8; ++a) rk[q][a] = ph;
        } else {
#pragma unroll
          for (int a = 0; a < 8; ++a) rk[q][a] = 0;
        }
      }
      if (MODE == kColored)
        accumulate_colored<S, 8>(acc, nd[0], c[0], nfree, valid[0], rk[0][0],
                                 batch_nph(j, g.hex_bnph, h_start + b * kBatch));
      else
        accumulate<S, 8, MODE>(acc, nd, c, nfree, valid, rk, g.max_phase_hex);
    }
    // every thread passed the last phase barrier: the stage can be refilled
    if (tid == 0 && j + kStages < nb) {
      fence_proxy_async();
      issue_batch(g, p, j + kStages, nbt, stage, &bars[st], preg < 0);
    }
    if (++st == kStages) {
      st = 0;
      parity ^= 1u;
    }
  }
  }  // generic batch loop
  __syncthreads();

  // lumped nodal update of the owned free nodes.  The per-tile uniform
  // decisions (material lookup, source kinds, Robin rows) pick one of four
  // loop bodies, so the common ones are branch-free and the UN nodes of a
  // round interleave: 0 general, 1 single material / no dynamic source / no
  // Robin row in the tile, 2 the same with exactly one Gaussian source, 3 the
  // same with exactly one RF source.  `tm` is the tile's material.
  bool bad = false;
  const int rstart = g.part_robin_start[p];
  // LEAN tet tiles: the one material's laws as direct constant-bank operands
  // (measured: cfg3 0.0712 -> 0.0707 ms/step; the hex loop measured 1.5%
  // slower with it, so it keeps the indexed loads)
  const int tm = (LEAN && (KINDS == 1 || FH_HEX_TM_CONST)) ? 0
                                                          : (g.node_region ? (FH_PART_MAT ? (int)g.part_mat[p] : -1) : 0);
  // nodes per thread per round: their global loads are issued together
  constexpr int UN = KINDS == 1 ? FH_NODE_UNROLL_TET : FH_NODE_UNROLL;
  auto node_loop = [&](auto kind_tag, auto inside_tag) {
    constexpr int KIND = decltype(kind_tag)::value;
    constexpr bool INSIDE = decltype(inside_tag)::value;
    for (int base = tid; base < nfree; base += UN * kTileThreads) {
      S v[UN], q[UN], cf[UN], kf[UN], px[UN], py[UN], pz[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int loc = base + u * kTileThreads;
        const bool ok = loc < nfree;
        const int n = n0 + (ok ? loc : 0);
        q[u] = g.q_ext ? __ldg(g.q_ext + n) : S(0);
        cf[u] = TD ? S(0) : __ldg(g.cap_frozen + n);
        kf[u] = (!TD && g.kb_frozen) ? __ldg(g.kb_frozen + n) : S(0);
        if (KIND >= 2 || (KIND == 0 && g.n_src)) {  // packed (x, y, z, v): one vector load per node
          load_xyzv(g.xyzv + 4 * (size_t)n, px[u], py[u], pz[u], v[u]);
        } else {
          v[u] = __ldg(g.vol + n);
          px[u] = py[u] = pz[u] = S(0);
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        // straight-line body for every lane (index clamped), predicated store
        const bool ok = base + u * kTileThreads < nfree;
        const int loc = ok ? base + u * kTileThreads : 0;
        const int n = n0 + loc;
        const S x = st_T(sT, loc);
        S Fsum;
        if (MODE == kCornerPhase2) {
          Fsum = acc[loc] + acc[nfree + loc];
        } else if (KINDS == 1 && g.tet_rows > 1) {  // tet accumulator rows, summed in row order
          const S r01 = acc[loc] + acc[nfree + loc];
          Fsum = g.tet_rows == 4   ? r01 + (acc[2 * nfree + loc] + acc[3 * nfree + loc])
                 : g.tet_rows == 3 ? r01 + acc[2 * nfree + loc]
                                   : r01;
        } else {
          Fsum = acc[loc];
        }
        S rate;
        S cap;
        if (KIND != 0)  // single material: curve parameters are uniform operands
          rate = node_rate<S, TD, LIN, INSIDE>(g.mats.m[tm], x, Fsum, v[u], q[u], cf[u], kf[u], cap);
        else if (!g.node_region)
          rate = node_rate<S, TD, LIN>(g.mats.m[0], x, Fsum, v[u], q[u], cf[u], kf[u], cap);
        else
          rate = node_rate<S, TD, LIN>(g.mats.m[g.node_region[n]], x, Fsum, v[u], q[u], cf[u], kf[u], cap);
        if (KIND == 2) {
          const SourceT<S> &sr = g.src[0];
          const S dx = px[u] - sr.cx, dy = py[u] - sr.cy, dz = pz[u] - sr.cz;
          rate += sr.amp * fast_exp(-((dx * dx + dy * dy) + dz * dz) * sr.inv2s2) * v[u];
        } else if (KIND == 3) {  // min(P / (4 pi r^2), cap), the cap at r = 0 (sources_at)
          const SourceT<S> &sr = g.src[0];
          const S dx = px[u] - sr.cx, dy = py[u] - sr.cy, dz = pz[u] - sr.cz;
          const S r2 = (dx * dx + dy * dy) + dz * dz;
          rate += (r2 > S(0) ? min(sr.cap, fast_div(sr.inv4pi_amp, r2)) : sr.cap) * v[u];
        } else if (KIND == 0 && g.n_src) {
          const S xyz[3] = {px[u], py[u], pz[u]};
          rate += sources_at(g, xyz) * v[u];
        }
        if (KIND == 0 && loc >= rstart) {
          const int rb = g.part_robin_base[p] + (loc - rstart);
          rate += g.robin_hAT[rb] - g.robin_hA[rb] * x;
        }
        const S xn = x + fast_div(g.dt * rate, cap);
        if (ok) {
          if (g.F_out) g.F_out[n] = Fsum;
          g.Tout[n] = xn;
          bad |= !(fabs(xn) <= g.runaway_limit);  // also catches NaN
        }
      }
    }
  };
  const bool simple = tm >= 0 && rstart >= nfree;
  // LEAN tiles (material 0 throughout) whose staged temperatures all lie inside the laws' knots skip the clamps
  const bool inside = LEAN != 0 && TD && LIN && tm == 0 && !kclamp;
  auto node_kind = [&](auto inside_tag) {
    if (simple && g.n_src == 0)
      node_loop(std::integral_constant<int, 1>{}, inside_tag);
    else if (simple && g.n_src == 1 && g.n_gauss == 1)
      node_loop(std::integral_constant<int, 2>{}, inside_tag);
    else if (simple && g.n_src == 1)
      node_loop(std::integral_constant<int, 3>{}, inside_tag);
    else
      node_loop(std::integral_constant<int, 0>{}, std::false_type{});
  };
  if constexpr (LEAN != 0) {
    if (inside) node_kind(std::true_type{});
    else node_kind(std::false_type{});
  } else {
    node_kind(std::false_type{});
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) s_bad = 1;
  __syncthreads();
  if (tid == 0 && s_bad) atomicMin(&g.flag->step, g.step_no);
}

// the step kernel instance for these arguments, with `smem` bytes of dynamic
// shared memory allowed
template <typename S>
void (*pick_step_kernel(const TiledArgs<S> &g, bool td, int mode_sel, size_t smem))(TiledArgs<S>) {
  using K = void (*)(TiledArgs<S>);
  // [lin][td][kinds][hex mode]; tet-only meshes ignore the hex mode.  LIN
  // only matters with temperature-dependent laws (TI never interpolates).
#define FH_MODES(TDV, KV, L)                                                                       \
  {k_tiled_step<S, TDV, kRanked, KV, L>, k_tiled_step<S, TDV, kCornerPhase, KV, L>,                 \
   k_tiled_step<S, TDV, kRanked, KV, L>, k_tiled_step<S, TDV, kColored, KV, L>,                     \
   k_tiled_step<S, TDV, kSharedAtomic, KV, L>, k_tiled_step<S, TDV, kCornerPhase2, KV, L>,          \
   k_tiled_step<S, TDV, kRanked, KV, L>}
#define FH_TETONLY(TDV, L)                                                                         \
  {k_tiled_step<S, TDV, kRanked, 1, L>, k_tiled_step<S, TDV, kRanked, 1, L>,                        \
   k_tiled_step<S, TDV, kRanked, 1, L>, k_tiled_step<S, TDV, kRanked, 1, L>,                        \
   k_tiled_step<S, TDV, kRanked, 1, L>, k_tiled_step<S, TDV, kRanked, 1, L>,                        \
   k_tiled_step<S, TDV, kRanked, 1, L>}
  static const K table[2][2][3][7] = {
      {{FH_MODES(false, 0, false), FH_TETONLY(false, false), FH_MODES(false, 2, false)},
       {FH_MODES(true, 0, false), FH_TETONLY(true, false), FH_MODES(true, 2, false)}},
      {{FH_MODES(false, 0, false), FH_TETONLY(false, false), FH_MODES(false, 2, false)},
       {FH_MODES(true, 0, true), FH_TETONLY(true, true), FH_MODES(true, 2, true)}}};
#undef FH_MODES
#undef FH_TETONLY
  const int mode = mode_sel < 0 || mode_sel > 6 ? 0 : mode_sel;
  const int kinds = (g.tet_rec && g.hex_rec) ? 2 : (g.hex_rec ? 0 : 1);
  const int lin = g.lin ? 1 : 0;
  K kern = table[lin][td ? 1 : 0][kinds][mode];
  // the LEAN batch loops (see k_tiled_step)
  // decided at setup (TiledState::lean), which also packed the records' G in pairs
  int lean = 0;
  if (g.lean == 1 && kinds == 1) {
    kern = k_tiled_step<S, true, kRanked, 1, true, 1>;
    lean = 1;
  } else if (g.lean == 1 && kinds == 0) {
    kern = k_tiled_step<S, true, kCornerPhase2, 0, true, 1>;
    lean = 2;
  } else if (g.lean == 2 && kinds == 0) {
    kern = k_tiled_step<S, true, kCornerPhase2, 0, true, 2>;
    lean = 3;
  } else if (g.lean == 3 && kinds == 2) {
    kern = k_tiled_step<S, true, kCornerPhase2, 2, true, 3>;
    lean = 4;
  }
  static size_t configured[5][2][2][3][7] = {};
  size_t &cfg = configured[lean][lin][td ? 1 : 0][kinds][mode];
  if (smem > cfg) {
    FH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cfg = smem;
  }
  return kern;
}

template <typename S>
void tiled_step(const TiledArgs<S> &g, int n_parts, bool td, int mode_sel, size_t smem, cudaStream_t s) {
  if (n_parts <= 0) return;
  pick_step_kernel<S>(g, td, mode_sel, smem)<<<n_parts, kTileThreads, smem, s>>>(g);
  FH_CUDA(cudaGetLastError());
}
template void tiled_step<float>(const TiledArgs<float> &, int, bool, int, size_t, cudaStream_t);
template void tiled_step<double>(const TiledArgs<double> &, int, bool, int, size_t, cudaStream_t);

template <typename S>
int tiled_occupancy(const TiledArgs<S> &g, bool td, int mode_sel, size_t smem) {
  int bps = 0;
  FH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pick_step_kernel<S>(g, td, mode_sel, smem),
                                                        kTileThreads, smem));
  return bps;
}
template int tiled_occupancy<float>(const TiledArgs<float> &, bool, int, size_t);
template int tiled_occupancy<double>(const TiledArgs<double> &, bool, int, size_t);

// ---- TI freeze ---------------------------------------------------------------
template <typename S, int N>
__global__ void k_freeze_slots(const TiledArgs<S> g, const int32_t *__restrict__ conn, const uint8_t *region,
                               int64_t n_slots, const S *__restrict__ kf, S *__restrict__ kbar) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_slots) return;
  const Curve<S> &kc = g.mats.m[region ? region[s] : 0].k;
  S T[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) T[b] = b < N ? g.Tin[conn[N * s + b]] : S(0);
  kbar[s] = kbar_from<false>(kc, T, N, kf ? kf[s] : S(1));
}

template <typename S>
__global__ void k_freeze_nodes(const TiledArgs<S> g, int64_t V, S *__restrict__ cap, S *__restrict__ kb) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= V) return;
  const Mat<S> &m = g.mats.m[g.node_region ? g.node_region[n] : 0];
  const S x = g.Tin[n], v = g.vol[n];
  cap[n] = interp(m.rho, x) * interp(m.c, x) * v;
  kb[n] = m.td_perf ? interp(m.wb, x) * m.cb * v : m.wbcb * v;
}

template <typename S>
void tiled_freeze(const TiledArgs<S> &g, const int32_t *tet_conn, const int32_t *hex_conn, int64_t nt, int64_t nh,
                  int64_t V, const S *kf_tet, const S *kf_hex, S *kbar_tet, S *kbar_hex, S *cap, S *kb,
                  cudaStream_t s) {
  if (nt) k_freeze_slots<S, 4><<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(g, tet_conn, g.tet_region, nt, kf_tet, kbar_tet);
  if (nh) k_freeze_slots<S, 8><<<(unsigned)((nh + 255) / 256), 256, 0, s>>>(g, hex_conn, g.hex_region, nh, kf_hex, kbar_hex);
  if (V) k_freeze_nodes<S><<<(unsigned)((V + 255) / 256), 256, 0, s>>>(g, V, cap, kb);
  FH_CUDA(cudaGetLastError());
}
template void tiled_freeze<float>(const TiledArgs<float> &, const int32_t *, const int32_t *, int64_t, int64_t,
                                  int64_t, const float *, const float *, float *, float *, float *, float *,
                                  cudaStream_t);
template void tiled_freeze<double>(const TiledArgs<double> &, const int32_t *, const int32_t *, int64_t, int64_t,
                                   int64_t, const double *, const double *, double *, double *, double *, double *,
                                   cudaStream_t);

template <typename S>
__global__ void k_probes_t(const S *__restrict__ T, const int32_t *__restrict__ probes, int64_t np,
                           double *__restrict__ out, const FailFlag *flag) {
  if (flag && flag->step != kNone) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < np) out[q] = probes[q] >= 0 ? (double)T[probes[q]] : __longlong_as_double(0x7ff8000000000000ll);
}

template <typename S>
void gather_probes_t(const S *T, const int32_t *probes, int64_t np, double *out, const FailFlag *flag,
                     cudaStream_t s) {
  if (np <= 0) return;
  k_probes_t<S><<<(unsigned)((np + 127) / 128), 128, 0, s>>>(T, probes, np, out, flag);
  FH_CUDA(cudaGetLastError());
}
template void gather_probes_t<float>(const float *, const int32_t *, int64_t, double *, const FailFlag *, cudaStream_t);
template void gather_probes_t<double>(const double *, const int32_t *, int64_t, double *, const FailFlag *,
                                      cudaStream_t);

}  // namespace fh
